"""Cartesian domain decomposition on the B200 path (parallel.py:45-547 of the
reference).

Two executions of ``run_parallel`` share one contract -- bitwise identical to
the serial solver for every rank layout (tests/test_parallel.py:192-212 of
the reference):

* one device (default): the subdomains are instances of ONE batched device
  run; before every stage a face-only halo kernel copies each subdomain's
  boundary slabs into its neighbours' ghost cells, all subdomains share one
  step state, so dt is the global max-reduction (parallel.py:498-501) and
  the whole loop stays on the GPU (CUDA-graph batches, no host sync).
* one process per GPU (``torch.distributed`` initialised, world size ==
  number of ranks): ``run_parallel_nccl`` -- halo slabs packed by
  fvb_halo_pack, exchanged with NCCL send/recv, unpacked by fvb_halo_unpack;
  dt from an all-reduce(MAX) of the per-axis maxima.

``exchange_halos`` keeps the reference's message-level API (sequential
axes, full padded extents, tags) with device pack/unpack.
"""

from __future__ import annotations

import math
import queue
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .grid import Field, GridSpec, make_field
from .solver import DeviceField, DeviceRun, TYPES, _raise_run_error, _v, check_scheme, make_layout

_RECV_TIMEOUT = 60.0


@dataclass(frozen=True)
class RankTopology:
    """Cartesian layout of ranks; rank 0 at the origin, x fastest."""

    ranks_per_axis: tuple

    def __post_init__(self):
        object.__setattr__(self, "ranks_per_axis", tuple(int(r) for r in self.ranks_per_axis))
        if any(r < 1 for r in self.ranks_per_axis):
            raise E.ConfigError(f"ranks per axis must be >= 1, got {self.ranks_per_axis}")

    @property
    def dim(self) -> int:
        return len(self.ranks_per_axis)

    @property
    def size(self) -> int:
        return math.prod(self.ranks_per_axis)

    def coords(self, rank: int) -> tuple:
        out = []
        for r in self.ranks_per_axis:
            out.append(rank % r)
            rank //= r
        return tuple(out)

    def rank_of(self, coords) -> int:
        rank = 0
        for c, r in zip(reversed(coords), reversed(self.ranks_per_axis)):
            rank = rank * r + c
        return rank

    def neighbor(self, rank: int, axis: int, side: int, periodic: bool):
        c = list(self.coords(rank))
        c[axis] += 1 if side else -1
        r = self.ranks_per_axis[axis]
        if 0 <= c[axis] < r:
            return self.rank_of(c)
        if not periodic:
            return None
        c[axis] %= r
        return self.rank_of(c)


@dataclass(frozen=True)
class Subdomain:
    rank: int
    grid: GridSpec
    offset: tuple


def decompose(grid, topo: RankTopology) -> list:
    """Exact tiling; local grids inherit the global deltas (parallel.py:99-124)."""
    if topo.dim != grid.dim:
        raise E.ConfigError(f"topology dim {topo.dim} does not match grid dim {grid.dim}")
    for axis, (n, r) in enumerate(zip(grid.cells, topo.ranks_per_axis)):
        if n % r:
            raise E.ConfigError(f"{n} cells on axis {axis} not divisible by {r} ranks")
    local = tuple(n // r for n, r in zip(grid.cells, topo.ranks_per_axis))
    out = []
    for rank in range(topo.size):
        off = tuple(c * m for c, m in zip(topo.coords(rank), local))
        origin = tuple(grid.origin[k] + off[k] * grid.deltas[k] for k in range(grid.dim))
        extent = tuple(m * d for m, d in zip(local, grid.deltas))
        g = GridSpec(grid.dim, local, origin, extent, ghost_width=grid.ghost_width, deltas=grid.deltas)
        out.append(Subdomain(rank, g, off))
    return out


def _box(part) -> tuple:
    d = part.grid.dim
    return (slice(None),) + tuple(
        slice(part.offset[d - 1 - j], part.offset[d - 1 - j] + part.grid.cells[d - 1 - j]) for j in range(d))


def scatter_field(global_field, parts) -> list:
    src = global_field.interior
    out = []
    for part in parts:
        loc = make_field(part.grid, global_field.ncomp, 0.0)
        loc.interior[...] = src[_box(part)]
        out.append(loc)
    return out


def stitch_fields(global_grid, parts, locals_) -> Field:
    out = make_field(global_grid, locals_[0].ncomp, 0.0)
    for part, loc in zip(parts, locals_):
        out.interior[_box(part)] = loc.interior
    cls = TYPES["Field"] or Field
    return cls(out.grid, out.ncomp, out.data) if cls is not Field else out


@dataclass
class RankRecord:
    step: int
    t: float
    dt: float
    seconds: float


# ---------------------------------------------------------------------------
# message-level halo API (parallel.py:127-254)
# ---------------------------------------------------------------------------

@dataclass
class HaloMessage:
    source: int
    dest: int
    axis: int
    side: int
    tag: int
    payload: object


class Transport:
    def send(self, msg: HaloMessage) -> None:
        raise NotImplementedError

    def receive(self, source: int, dest: int, axis: int, side: int, tag: int):
        raise NotImplementedError


class InProcessTransport(Transport):
    """Per-pair FIFO with strictly increasing tags (parallel.py:147-182)."""

    def __init__(self, size: int):
        self.size = size
        self._queues = {(s, d): queue.SimpleQueue() for s in range(size) for d in range(size)}
        self._last_tag = {}

    def send(self, msg: HaloMessage) -> None:
        key = (msg.source, msg.dest)
        last = self._last_tag.get(key)
        if last is not None and msg.tag <= last:
            raise E.ProtocolError(f"tag {msg.tag} not increasing on pair {key} (last {last})")
        self._last_tag[key] = msg.tag
        self._queues[key].put(msg)

    def receive(self, source, dest, axis, side, tag):
        try:
            msg = self._queues[(source, dest)].get(timeout=_RECV_TIMEOUT)
        except queue.Empty:
            raise E.ProtocolError(f"timed out waiting for message {source}->{dest} tag {tag}") from None
        if (msg.axis, msg.side, msg.tag) != (axis, side, tag):
            raise E.ProtocolError(
                f"message mismatch on pair ({source}, {dest}): expected (axis={axis}, side={side}, tag={tag}), "
                f"got (axis={msg.axis}, side={msg.side}, tag={msg.tag})")
        return msg.payload


def _desc(grid, ncomp, halo_all=True):
    s = N.Scheme()
    s.dim, s.ncomp, s.ghost, s.rk_order = grid.dim, ncomp, grid.ghost_width, 1
    s.eq = 0 if ncomp == grid.dim + 2 else 1
    for k in range(3):
        s.cells[k] = grid.cells[k] if k < grid.dim else 1
        s.deltas[k] = grid.deltas[k] if k < grid.dim else 1.0
        s.bc[k] = N.BC_HALO if (halo_all and k < grid.dim) else N.BC_PERIODIC
    return s


def exchange_halos(field, rank: int, topo: RankTopology, transport: Transport, bc, tag: int):
    """parallel.py:201-254: sequential axis passes over the full padded extent
    (corners propagate), two directional sub-passes per axis; slabs are
    packed/unpacked on the GPU (fvb_halo_pack/unpack)."""
    import torch

    dev, was_dev = (field, True) if isinstance(field, DeviceField) else (DeviceField.from_host(field), False)
    grid = dev.grid
    ctx = N.context()
    s = _desc(grid, dev.ncomp)
    L = make_layout(grid, dev.ncomp)
    ptr = N.C.c_void_p(dev.data.data_ptr())
    for axis in range(grid.dim):
        periodic = _v(bc[axis]) == "periodic"
        nb = {side: topo.neighbor(rank, axis, side, periodic) for side in (0, 1)}
        if nb[0] == rank and nb[1] == rank:  # single rank along a periodic axis: plain wrap
            _fill_one_axis(dev, axis, "periodic")
            continue
        count = int(ctx.lib.fvb_halo_count(N.C.byref(s), axis))
        for d in (0, 1):
            send_nb, recv_nb = nb[d], nb[1 - d]
            subtag = (tag * grid.dim + axis) * 2 + d
            if send_nb is not None:
                buf = torch.empty(count, dtype=torch.float64, device=dev.data.device)
                ctx.check(ctx.lib.fvb_halo_pack(ctx.h, N.C.byref(s), N.C.byref(L), ptr, axis, d,
                                                N.C.c_void_p(buf.data_ptr())))
                transport.send(HaloMessage(rank, send_nb, axis, 1 - d, subtag, buf.cpu().numpy()))
            if recv_nb is None:
                _fill_one_side(dev, axis, 1 - d)
            else:
                payload = transport.receive(recv_nb, rank, axis, 1 - d, subtag)
                buf = torch.as_tensor(np.ascontiguousarray(payload), dtype=torch.float64).to(dev.data.device)
                ctx.check(ctx.lib.fvb_halo_unpack(ctx.h, N.C.byref(s), N.C.byref(L), ptr, axis, 1 - d,
                                                  N.C.c_void_p(buf.data_ptr())))
    if not was_dev:
        field.data[...] = dev.data.cpu().numpy()
        return field
    return dev


def _fill_one_axis(dev, axis, kind):
    ctx = N.context()
    s = _desc(dev.grid, dev.ncomp, halo_all=False)
    for k in range(3):
        s.bc[k] = N.BC_HALO
    s.bc[axis] = N.BC_PERIODIC if kind == "periodic" else N.BC_OUTFLOW
    L = make_layout(dev.grid, dev.ncomp)
    ctx.check(ctx.lib.fvb_fill_ghosts(ctx.h, N.C.byref(s), N.C.byref(L), N.C.c_void_p(dev.data.data_ptr()), 1))


def _fill_one_side(dev, axis, side):
    """_fill_outflow_side (parallel.py:189-198): copy the nearest interior
    layer into the ghost slab of one side (a broadcast device copy)."""
    grid = dev.grid
    g = grid.ghost_width
    idx = [slice(None)] * dev.data.dim()
    ax = grid.dim - axis
    n = grid.cells[axis]
    src = [slice(None)] * dev.data.dim()
    if side == 0:
        idx[ax] = slice(0, g)
        src[ax] = slice(g, g + 1)
    else:
        idx[ax] = slice(n + g, n + 2 * g)
        src[ax] = slice(n + g - 1, n + g)
    dev.data[tuple(idx)] = dev.data[tuple(src)].expand_as(dev.data[tuple(idx)])


# ---------------------------------------------------------------------------
# run_parallel (parallel.py:430-521)
# ---------------------------------------------------------------------------

def run_parallel(init, cfg, ranks_per_axis, n_steps: int | None = None, overlap: bool = True, *,
                 arith: str | None = None):
    """Decomposed run; returns (stitched final Field, per-rank records)."""
    import torch

    check_scheme(init.grid, cfg)
    topo = RankTopology(tuple(ranks_per_axis))
    parts = decompose(init.grid, topo)
    if torch.distributed.is_available() and torch.distributed.is_initialized() \
            and torch.distributed.get_world_size() == topo.size and topo.size > 1:
        cpu = torch.distributed.get_backend() == "gloo"
        return run_parallel_nccl(init, cfg, topo, parts, n_steps, arith=arith, cpu_comm=cpu, overlap=overlap)
    locals_ = scatter_field(init, parts)
    grid = parts[0].grid
    ncomp = init.ncomp
    host = torch.from_numpy(np.stack([np.asarray(f.data) for f in locals_]))
    b0 = host.to("cuda")
    bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
    ctx = N.context()
    ranks = (N.C.c_int32 * 3)(*(list(topo.ranks_per_axis) + [1] * (3 - grid.dim)))
    per = (N.C.c_int32 * 3)(*[int(_v(cfg.bc[k]) == "periodic") if k < grid.dim else 1 for k in range(3)])
    ctx.check(ctx.lib.fvb_run_set_topology(ctx.h, ranks, per))
    split = tuple(k for k in range(grid.dim) if topo.ranks_per_axis[k] > 1)
    mode = N.MODE_FIXED if n_steps is not None else N.MODE_PAR_T_END
    run = DeviceRun(grid, cfg, bufs, topo.size, mode, n_steps, arith, halo_axes=split, ctx=ctx)
    records = []
    while True:
        infos, done = run.poll()
        if infos[0].err or done[0]:
            break
        n = 256 if n_steps is None else max(1, n_steps - int(infos[0].steps))
        if n_steps is None and infos[0].dt > 0:
            n = int(min(n, max(1, math.ceil((cfg.t_end - infos[0].t) / infos[0].dt) + 2)))
        tic = time.perf_counter()
        run.steps(n)
        infos, done = run.poll()
        run.read_log(infos, (time.perf_counter() - tic) / max(1, int(infos[0].steps) - run._seen[0]))
    info = run.end()[0]
    if info.err:
        try:
            _raise_run_error(info, grid, ncomp)
        except E.ConslawError as exc:
            raise E.SimulationError(f"rank 0 failed: {exc}") from exc
    final = bufs[int(info.steps) % 2] if cfg.rk_order == 1 else bufs[0]
    finals = [DeviceField(grid, ncomp, final[r]).to_host() for r in range(topo.size)]
    recs = [RankRecord(r.step, r.t, r.dt, r.seconds) for r in run.records[0]]
    return stitch_fields(init.grid, parts, finals), [list(recs) for _ in range(topo.size)]


def start_halo_exchange(topo: RankTopology, rank: int, periodic, pack, alloc, dist, group=None, axes=None):
    """Post the face-only halo sends/receives of one rank over
    torch.distributed P2P (NCCL on GPUs; gloo in the CPU tests) and return
    a handle for ``finish_halo_exchange``.

    ``pack(axis, side)`` returns the slab(s) of the g interior layers next to
    face (axis, side) -- one contiguous tensor or a list of them;
    ``alloc(axis, side)`` the matching receive buffer(s) for the ghosts of
    that side.  Axes are exchanged concurrently (the residual never reads
    corner ghosts, solver.py:99-104).  Ordering rule so that a pair of ranks
    that are mutual neighbours on both sides (2 ranks on a periodic axis,
    parallel.py:227-230) match: sends are issued by side (low, high),
    receives by the SENDER's side, i.e. high ghosts first.  World-edge sides
    without a neighbour are left to the caller (outflow)."""
    ops, recvs = [], []

    def _list(x):
        return x if isinstance(x, (list, tuple)) else [x]

    for axis in (range(topo.dim) if axes is None else axes):
        if topo.ranks_per_axis[axis] == 1:
            continue
        nb = [topo.neighbor(rank, axis, side, bool(periodic[axis])) for side in (0, 1)]
        for side in (0, 1):
            if nb[side] is not None:
                for t in _list(pack(axis, side)):
                    ops.append(dist.P2POp(dist.isend, t, nb[side], group))
        for side in (1, 0):
            if nb[side] is not None:
                buf = alloc(axis, side)
                for t in _list(buf):
                    ops.append(dist.P2POp(dist.irecv, t, nb[side], group))
                recvs.append((axis, side, buf))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    return reqs, recvs


def finish_halo_exchange(handle, unpack):
    """Complete the exchange: NCCL works make the current stream wait (no
    host block); then ``unpack(axis, side, buf)`` places each slab."""
    reqs, recvs = handle
    for req in reqs:
        req.wait()
    for axis, side, buf in recvs:
        unpack(axis, side, buf)


def halo_exchange_dist(topo: RankTopology, rank: int, periodic, pack, unpack, alloc, dist, group=None, axes=None):
    """Blocking face-only halo exchange (start + finish)."""
    finish_halo_exchange(start_halo_exchange(topo, rank, periodic, pack, alloc, dist, group, axes), unpack)


class _Halos:
    """Persistent halo buffers of one rank's subdomain.

    The march axis (z in 3D, y in 2D) -- the split bench.py uses -- needs no
    packing: for every component the g send layers and the g ghost layers
    are contiguous slices of the field buffer, so NCCL reads and writes them
    in place (ncomp messages per side).  Other axes go through fvb_halo_pack
    / fvb_halo_unpack into buffers allocated once."""

    def __init__(self, ctx, scheme, layout, grid, ncomp, split, cpu_comm):
        import torch

        self.ctx, self.s, self.L = ctx, scheme, layout
        self.grid, self.ncomp, self.cpu = grid, ncomp, cpu_comm
        self.march = grid.dim - 1
        g = grid.ghost_width
        self.g = g
        n = grid.cells[self.march]
        self.direct = (not cpu_comm) and self.march in split and n >= g
        self.bufs = {}
        for axis in split:
            if self.direct and axis == self.march:
                continue
            cnt = int(ctx.lib.fvb_halo_count(N.C.byref(scheme), axis))
            dev = "cpu" if cpu_comm else "cuda"
            for side in (0, 1):
                self.bufs[(axis, side, "send")] = torch.empty(cnt, dtype=torch.float64, device="cuda")
                self.bufs[(axis, side, "recv")] = torch.empty(cnt, dtype=torch.float64, device=dev,
                                                              pin_memory=cpu_comm)
                if cpu_comm:
                    self.bufs[(axis, side, "host_send")] = torch.empty(cnt, dtype=torch.float64, pin_memory=True)

    def _slab(self, u, side, ghost):
        """Per-component contiguous views of the march-axis layers: the g
        interior layers next to face `side` (ghost=False) or its g ghosts."""
        g, n = self.g, self.grid.cells[self.march]
        lo = (g if side == 0 else n) if not ghost else (0 if side == 0 else n + g)
        return [u[0, c, lo:lo + g] for c in range(self.ncomp)]

    def movers(self, u):
        ctx, s, L = self.ctx, self.s, self.L
        ptr = N.C.c_void_p(u.data_ptr())

        def pack(axis, side):
            if self.direct and axis == self.march:
                return self._slab(u, side, ghost=False)
            buf = self.bufs[(axis, side, "send")]
            ctx.check(ctx.lib.fvb_halo_pack(ctx.h, N.C.byref(s), N.C.byref(L), ptr, axis, side,
                                            N.C.c_void_p(buf.data_ptr())))
            if self.cpu:
                host = self.bufs[(axis, side, "host_send")]
                host.copy_(buf)
                return host
            return buf

        def alloc(axis, side):
            if self.direct and axis == self.march:
                return self._slab(u, side, ghost=True)  # received straight into the ghost layers
            return self.bufs[(axis, side, "recv")]

        def unpack(axis, side, buf):
            if self.direct and axis == self.march:
                return
            b = buf.to("cuda", non_blocking=False) if self.cpu else buf
            ctx.check(ctx.lib.fvb_halo_unpack(ctx.h, N.C.byref(s), N.C.byref(L), ptr, axis, side,
                                              N.C.c_void_p(b.data_ptr())))

        return pack, unpack, alloc


class DecomposedRun:
    """The per-rank loop of run_parallel (parallel.py:479-521) for one
    subdomain on this process's GPU, device resident.

    ``local`` is this rank's subdomain (a host ``Field`` or a ``DeviceField``
    with its own GridSpec, ghosts included).  Every stage: halo exchange of
    the stage input over torch.distributed P2P (NCCL; march-axis layers in
    place, other axes packed into persistent buffers), then the fused stage
    kernel -- with ``overlap`` and a split march axis, the inner rows [g,
    n-g) run while the halos are in flight and the two shell slabs after
    they land (overlapped_residual, parallel.py:325-361).  Every step: one
    all-reduce(MAX) of [maxima, error flags] and a device finalisation that
    all ranks evaluate identically (global dt, parallel.py:498-501).  All of
    it is stream ordered on the run's own stream: the host reads the device
    state only every ``poll_every`` steps and at the end.  ``cpu_comm``
    stages the exchanged slabs and the reduce through host memory (gloo),
    e.g. to test several ranks on one GPU.

    ``peer_halos`` (NCCL groups, march axis the only split axis, one GPU per
    rank): the fused halo exchange -- the three field buffers live in
    symmetric memory (torch.distributed._symmetric_memory, NVLink peer
    mappings), every stage kernel also stores its first / last g march rows
    into the neighbours' ghost rows (``fvb_run_set_peers``), and a device
    barrier after each stage orders the ranks; no pack, no NCCL message per
    stage.  "auto" uses it when available.

    ``advance(n)`` enqueues up to n more steps; ``finish()`` returns
    (DeviceField of the final subdomain, [RankRecord])."""

    def __init__(self, local, cfg, topo: RankTopology, n_steps=None, *, arith=None, group=None,
                 cpu_comm: bool = False, overlap: bool = True, poll_every: int = 64, log: bool = True,
                 peer_halos="auto"):
        import torch
        import torch.distributed as dist

        self.dist, self.group, self.cfg, self.topo = dist, group, cfg, topo
        self.rank = dist.get_rank(group)
        self.n_steps = n_steps
        self.poll_every = max(1, int(poll_every))
        self.stream = torch.cuda.Stream()
        with torch.cuda.stream(self.stream):  # NCCL orders after the library's kernels on this stream
            dev = local if isinstance(local, DeviceField) else DeviceField.from_host(local)
            self.grid, self.ncomp = dev.grid, dev.ncomp
            grid = self.grid
            self.split = tuple(k for k in range(grid.dim) if topo.ranks_per_axis[k] > 1)
            self.periodic = [int(_v(cfg.bc[k]) == "periodic") for k in range(grid.dim)]
            self.march = grid.dim - 1
            self.symm = None
            if self._peer_ok(peer_halos, cpu_comm):
                try:
                    import torch.distributed._symmetric_memory as symm_mem

                    # the three RK buffers in one symmetric allocation: every rank
                    # maps its neighbours' copies (same layout, same offsets)
                    block = symm_mem.empty((3, 1) + tuple(dev.data.shape), dtype=torch.float64, device="cuda")
                    hdl = symm_mem.rendezvous(block, group or dist.group.WORLD)
                    base = int(getattr(hdl, "offset", 0) or 0)
                    if int(hdl.buffer_ptrs[self.rank]) + base != block.data_ptr():
                        raise RuntimeError("symmetric buffer pointers do not match the local block")
                    self.symm = hdl
                    block[0, 0].copy_(dev.data)
                    self.bufs = [block[k] for k in range(3)]
                except Exception as exc:  # no peer mappings here: the NCCL exchange instead
                    if peer_halos is True:
                        raise
                    import warnings

                    warnings.warn(f"fused peer halos unavailable ({exc}); using NCCL halo messages")
                    self.symm = None
            if self.symm is None:
                b0 = dev.data.unsqueeze(0).contiguous()
                self.bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
            self.ctx = ctx = N.context()
            ctx.check(ctx.lib.fvb_run_set_external_reduce(ctx.h, 1))
            mode = N.MODE_FIXED if n_steps is not None else N.MODE_PAR_T_END
            self.run = DeviceRun(grid, cfg, self.bufs, 1, mode, n_steps, arith, halo_axes=self.split, ctx=ctx,
                                 log=log)
            self.halos = _Halos(ctx, self.run.scheme, self.run.layout, grid, self.ncomp, self.split, cpu_comm)
            self.cpu_comm = cpu_comm
            self.red = torch.zeros(grid.dim + 2, dtype=torch.float64, device="cuda")
            self.red_host = torch.zeros(grid.dim + 2, dtype=torch.float64, pin_memory=True) if cpu_comm else None
            self.g = grid.ghost_width
            if self.symm is not None:
                self._set_peers()
            # overlap schedule: every split axis long enough for an inner box
            self.ovl = overlap and grid.dim >= 2 and bool(self.split) and \
                all(grid.cells[a] > 2 * self.g for a in self.split)
            self.boxes = self._boxes() if self.ovl else None
            self.nst = 1 if cfg.rk_order == 1 else cfg.rk_order
            self.steps = 0
            self.done = False
            self._tic = time.perf_counter()
            self._last = 0
            self._reduce_and_finalize(0)

    def _peer_ok(self, peer_halos, cpu_comm) -> bool:
        """Fused halo exchange applicable: asked for (or auto), NCCL group,
        only the march axis split, symmetric memory available."""
        if not peer_halos or cpu_comm or self.split != (self.march,) or self.march == 0:
            return False
        if self.dist.get_backend(self.group) != "nccl":
            return False
        try:
            import torch.distributed._symmetric_memory  # noqa: F401
        except Exception:
            if peer_halos == "auto":
                return False
            raise
        return True

    def _set_peers(self):
        """Neighbours' buffer pointers (symmetric memory) -> fvb_run_set_peers."""
        ctx = self.ctx
        nbytes = self.bufs[0].numel() * 8
        base = int(getattr(self.symm, "offset", 0) or 0)  # the block's offset in each rank's allocation
        ptrs = [int(q) + base for q in self.symm.buffer_ptrs]
        per = bool(self.periodic[self.march])
        lo = self.topo.neighbor(self.rank, self.march, 0, per)
        hi = self.topo.neighbor(self.rank, self.march, 1, per)

        def arr(r):
            if r is None:
                return None
            return (N.C.c_void_p * 3)(*[N.C.c_void_p(int(ptrs[r]) + k * nbytes) for k in range(3)])

        self._peer_arrays = (arr(lo), arr(hi))  # keep alive
        ctx.check(ctx.lib.fvb_run_set_peers(ctx.h, self._peer_arrays[0], self._peer_arrays[1]))
        self._peer_primed = False  # the first stage input's ghosts come from one regular exchange

    def _reduce_and_finalize(self, post: int):
        ctx, dist, red = self.ctx, self.dist, self.red
        ctx.check(ctx.lib.fvb_run_export(ctx.h, N.C.c_void_p(red.data_ptr())))
        if self.cpu_comm:
            self.red_host.copy_(red)
            dist.all_reduce(self.red_host, op=dist.ReduceOp.MAX, group=self.group)
            red.copy_(self.red_host)
        else:
            dist.all_reduce(red, op=dist.ReduceOp.MAX, group=self.group)
        ctx.check(ctx.lib.fvb_run_finalize(ctx.h, N.C.c_void_p(red.data_ptr()), post))

    def _outflow_edges(self, u, axes):
        # world edges of split, non-periodic axes: outflow ghosts (parallel.py:246-247)
        view = DeviceField(self.grid, self.ncomp, u[0])
        for axis in axes:
            for side in (0, 1):
                if self.topo.neighbor(self.rank, axis, side, bool(self.periodic[axis])) is None:
                    _fill_one_side(view, axis, side)

    def _boxes(self):
        """Inner box (cells >= g from every split face) and the disjoint
        shell slabs that complete the subdomain (parallel.py:288-322): per
        split axis two slabs of thickness g, each spanning what is left of
        the other axes."""
        g, dim = self.g, self.grid.dim
        n = list(self.grid.cells)
        lo, hi = [0] * dim, list(n)
        inner_lo = [g if a in self.split else 0 for a in range(dim)]
        inner_hi = [n[a] - g if a in self.split else n[a] for a in range(dim)]
        shells = []
        for a in self.split:
            for side_lo, side_hi in ((0, g), (n[a] - g, n[a])):
                blo, bhi = list(lo), list(hi)
                blo[a], bhi[a] = side_lo, side_hi
                shells.append((blo, bhi))
            lo[a], hi[a] = g, n[a] - g
        arr = lambda v: (N.C.c_int64 * 3)(*(list(v) + [0] * (3 - dim)))  # noqa: E731
        return (arr(inner_lo), arr(inner_hi)), [(arr(a), arr(b)) for a, b in shells]

    def _stage(self, st, u):
        ctx, dist, topo, rank, per, grp = self.ctx, self.dist, self.topo, self.rank, self.periodic, self.group
        pack, unpack, alloc = self.halos.movers(u)
        if self.symm is not None:
            if not self._peer_primed:  # ghosts of the very first stage input
                halo_exchange_dist(topo, rank, per, pack, unpack, alloc, dist, grp)
                self._peer_primed = True
            self._outflow_edges(u, self.split)
            ctx.check(ctx.lib.fvb_run_stage(ctx.h, st))  # also stores the neighbours' ghost rows
            self.symm.barrier(channel=0)  # every rank's stage (and its peer stores) done
            return
        if not self.ovl:
            halo_exchange_dist(topo, rank, per, pack, unpack, alloc, dist, grp)
            self._outflow_edges(u, self.split)
            ctx.check(ctx.lib.fvb_run_stage(ctx.h, st))
            return
        # every split axis's halos travel while the inner box is computed
        handle = start_halo_exchange(topo, rank, per, pack, alloc, dist, grp, axes=self.split)
        (ilo, ihi), shells = self.boxes
        ctx.check(ctx.lib.fvb_run_stage_box(ctx.h, st, ilo, ihi, 0))
        finish_halo_exchange(handle, unpack)
        self._outflow_edges(u, self.split)
        for i, (blo, bhi) in enumerate(shells):
            ctx.check(ctx.lib.fvb_run_stage_box(ctx.h, st, blo, bhi, int(i == len(shells) - 1)))

    def _poll(self):
        infos, done = self.run.poll()
        self.run.read_log(infos, (time.perf_counter() - self._tic) / max(1, self.steps - self._last))
        self._tic, self._last = time.perf_counter(), self.steps
        self.done = self.done or done[0]
        return infos

    def advance(self, n: int | None = None) -> int:
        """Enqueue up to ``n`` more steps (None: to the end); returns how
        many were enqueued."""
        import torch

        k = 0
        with torch.cuda.stream(self.stream):
            while not self.done and (n is None or k < n):
                if self.n_steps is not None and self.steps >= self.n_steps:
                    break
                if self.steps % self.poll_every == 0 and self.steps > self._last:
                    self._poll()  # (the step log ring holds 4096 entries)
                    if self.done:
                        break
                elif self.steps == 0 and self.n_steps is None:
                    self._poll()
                    if self.done:
                        break
                for st in range(self.nst):
                    self._stage(st, self.bufs[self.steps % 2] if self.nst == 1 else self.bufs[st])
                self._reduce_and_finalize(1)
                self.steps += 1
                k += 1
        return k

    def finish(self):
        import torch

        with torch.cuda.stream(self.stream):
            if self.n_steps is None:
                self.advance()
            info = self._poll()[0]
            info = self.run.end()[0]
            if info.err:
                try:
                    _raise_run_error(info, self.grid, self.ncomp)
                except E.ConslawError as exc:
                    raise E.SimulationError(f"rank {self.rank} failed: {exc}") from exc
            final = self.bufs[int(info.steps) % 2] if self.cfg.rk_order == 1 else self.bufs[0]
            recs = [RankRecord(r.step, r.t, r.dt, r.seconds) for r in self.run.records[0]]
            out = DeviceField(self.grid, self.ncomp, final[0])
        torch.cuda.current_stream().wait_stream(self.stream)
        return out, recs


def run_decomposed(local, cfg, topo: RankTopology, n_steps=None, *, arith=None, group=None,
                   cpu_comm: bool = False, overlap: bool = True, poll_every: int = 64):
    """Run one rank's subdomain to the end (see DecomposedRun); returns
    (DeviceField of the final subdomain, [RankRecord])."""
    r = DecomposedRun(local, cfg, topo, n_steps, arith=arith, group=group, cpu_comm=cpu_comm, overlap=overlap,
                      poll_every=poll_every)
    r.advance()
    return r.finish()


def run_parallel_nccl(init, cfg, topo, parts, n_steps, *, arith=None, group=None, cpu_comm: bool = False,
                      overlap: bool = True):
    """One subdomain per process (rank r of the torch.distributed group owns
    part r): ``run_decomposed`` on the scattered subdomain, then the
    subdomains travel to rank 0 one at a time (device send/recv, one D2H
    each) and are stitched there; every rank gets all ranks' records.

    Rank 0 returns the stitched global Field; the other ranks return their
    own final subdomain (a process-per-GPU caller has no single owner of the
    global result)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    local = scatter_field(init, [parts[rank]])[0]
    dev, recs = run_decomposed(local, cfg, topo, n_steps, arith=arith, group=group, cpu_comm=cpu_comm,
                               overlap=overlap)
    mine = dev.to_host()
    allrecs = [None] * world
    dist.all_gather_object(allrecs, recs, group=group)
    if world == 1:
        return stitch_fields(init.grid, parts, [mine]), allrecs
    if rank == 0:
        locs = [mine]
        buf = torch.empty(tuple(mine.data.shape), dtype=torch.float64, device="cpu" if cpu_comm else "cuda")
        for r in range(1, world):
            dist.recv(buf, src=r, group=group)
            locs.append(Field(parts[r].grid, init.ncomp, buf.cpu().numpy().copy()))
        return stitch_fields(init.grid, parts, locs), allrecs
    dist.send(torch.from_numpy(np.ascontiguousarray(mine.data)) if cpu_comm else dev.data.contiguous(),
              dst=0, group=group)
    return mine, allrecs


# ---------------------------------------------------------------------------
# overhead metric (parallel.py:529-547)
# ---------------------------------------------------------------------------

@dataclass
class OverheadReport:
    ranks: int
    mean_seconds: float
    baseline_seconds: float
    overhead_fraction: float


def overhead_metric(times_K, times_1, ranks: int) -> OverheadReport:
    times_K, times_1 = list(times_K), list(times_1)
    if not times_K or not times_1:
        raise E.ConfigError("overhead metric needs non-empty timing series")
    mk = sum(times_K) / len(times_K)
    m1 = sum(times_1) / len(times_1)
    return OverheadReport(ranks, mk, m1, (mk - m1) / m1)
