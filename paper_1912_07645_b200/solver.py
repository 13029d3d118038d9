"""Drop-in solver API of the reference (solver.py:36-246) on the B200 path.

Every function keeps the reference signature and return type; the work runs
in libfvb200.so (csrc/):

* ``run_simulation``   -> fvb_run_begin/steps/poll/end: fused stage kernels,
  CFL reduction and loop control resident on the GPU, CUDA-graph batches.
* ``spatial_residual`` -> fvb_spatial_residual (stage kernel, kind L)
* ``wave_speed_maxima`` / ``stable_dt`` -> fvb_wave_speed_maxima
* ``ssp_rk_step``      -> fvb_ssp_rk_step
* ``fill_boundary``    -> fvb_fill_ghosts

Objects are duck-typed: the reference's own ``Field``/``GridSpec``/
``SchemeConfig`` instances are accepted unchanged (enums are read by
``.value``), and results are built with the caller's classes.

Arithmetic: ``arith="exact"`` (default) is bitwise identical to the
reference; ``arith="fast"`` removes divides/contracts FMAs (relative L1
<= 1e-12 over the test windows).  Default from ``FVB_ARITH``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from . import errors as E
from .equations import EULER, EquationModel
from .grid import BoundaryKind, Field, GridSpec
from .numerics import FluxKind, Reconstruction


def _v(x):
    return x.value if hasattr(x, "value") else str(x)


@dataclass(frozen=True)
class SchemeConfig:
    model: EquationModel
    flux: FluxKind = FluxKind.RUSANOV
    recon: Reconstruction = Reconstruction()
    rk_order: int = 2
    cfl: float = 0.475
    t_end: float = 1.0
    bc: tuple = ()

    def __post_init__(self):
        if self.rk_order not in (1, 2, 3):
            raise E.ConfigError(f"rk_order must be 1, 2 or 3, got {self.rk_order}")
        if not 0.0 < self.cfl <= 1.0:
            raise E.ConfigError(f"cfl must lie in (0, 1], got {self.cfl}")
        if self.t_end < 0.0:
            raise E.ConfigError(f"t_end must be >= 0, got {self.t_end}")
        if _v(self.flux) == "hllc" and self.model.kind != EULER:
            raise E.ConfigError("HLLC flux requires the Euler equations")
        if not self.bc:
            object.__setattr__(self, "bc", (BoundaryKind.PERIODIC,) * self.model.dim)
        if len(self.bc) != self.model.dim:
            raise E.ConfigError(f"need {self.model.dim} boundary kinds, got {len(self.bc)}")


@dataclass
class TimeStepRecord:
    step: int
    t: float
    dt: float
    seconds: float


# the result types can be rebound to the reference's classes (compat.py)
TYPES = {"Field": None, "TimeStepRecord": TimeStepRecord}


def _radius(cfg) -> int:
    return 1 if _v(cfg.recon.kind) == "none" else 2


def check_scheme(grid, cfg) -> None:
    """solver.py:73-79."""
    if _radius(cfg) > grid.ghost_width:
        raise E.ConfigError(
            f"ghost_width {grid.ghost_width} too small for reconstruction radius {_radius(cfg)}")


def _check_periodic(grid, bc) -> None:
    # fill_axis raises before the first residual (grid.py:153-157)
    for axis in range(grid.dim):
        if _v(bc[axis]) == "periodic" and grid.cells[axis] < grid.ghost_width:
            raise E.ConfigError(
                f"periodic axis {axis} needs cells >= ghost_width ({grid.cells[axis]} < {grid.ghost_width})")


# ---------------------------------------------------------------------------
# C-ABI descriptors
# ---------------------------------------------------------------------------

def make_scheme(grid, cfg, arith: str | None = None, halo_axes=(), all_halo: bool = False) -> N.Scheme:
    m = cfg.model
    s = N.Scheme()
    s.dim = grid.dim
    s.ncomp = grid.dim + 2 if m.kind == EULER else 1
    s.eq = N.EQ[m.kind]
    s.flux = N.FLUX[_v(cfg.flux)]
    s.recon = N.RECON[_v(cfg.recon.kind)]
    s.rk_order = int(cfg.rk_order)
    s.arith = N.ARITH[arith or N.default_arith()]
    s.ghost = int(grid.ghost_width)
    for k in range(3):
        if k < grid.dim:
            if all_halo or k in halo_axes:
                s.bc[k] = N.BC_HALO
            else:
                s.bc[k] = N.BC_PERIODIC if _v(cfg.bc[k]) == "periodic" else N.BC_OUTFLOW
            s.cells[k] = int(grid.cells[k])
            s.deltas[k] = float(grid.deltas[k])
        else:
            s.bc[k] = N.BC_PERIODIC
            s.cells[k] = 1
            s.deltas[k] = 1.0
    s.gamma = float(m.gamma)
    s.weno_eps = float(cfg.recon.epsilon)
    s.cfl = float(cfg.cfl)
    s.t_end = float(cfg.t_end)
    for k in range(3):
        s.adv[k] = float(m.advection_speed[k]) if (m.kind == "advection" and k < grid.dim) else 0.0
    return s


def make_layout(grid, ncomp: int) -> N.Layout:
    """Strides of a contiguous (ninst, ncomp, *grid.data_shape) buffer."""
    P = list(grid.padded) + [1] * (3 - grid.dim)
    g = grid.ghost_width
    L = N.Layout()
    L.sy = P[0]
    L.sz = P[0] * P[1]
    L.sc = P[0] * P[1] * P[2]
    L.si = L.sc * ncomp
    L.origin = g + (g * L.sy if grid.dim >= 2 else 0) + (g * L.sz if grid.dim >= 3 else 0)
    return L


# ---------------------------------------------------------------------------
# device-resident fields
# ---------------------------------------------------------------------------

class DeviceField:
    """A field resident in HBM: ``data`` is a CUDA float64 tensor of shape
    (ncomp, *grid.data_shape) -- the reference layout, ghosts included."""

    def __init__(self, grid, ncomp: int, data):
        self.grid = grid
        self.ncomp = ncomp
        self.data = data

    @classmethod
    def from_host(cls, field, device=None, pin: bool = False):
        """H2D copy of ``field.data`` (one DMA; asynchronous when the numpy
        buffer lives in pinned memory, e.g. ``pinned_field``)."""
        import torch

        N._require_cuda()  # no CPU fallback: fail loudly without a GPU
        src = torch.from_numpy(np.ascontiguousarray(field.data, dtype=np.float64))
        pinned = src.is_pinned()
        staged = not pinned
        if staged:  # stage pageable input through a reused (per-thread) pinned buffer
            stage = _staging(("h2d", tuple(src.shape)), tuple(src.shape))
            stage.copy_(src)  # multi-threaded host copy
            src = stage
        dev = torch.empty(src.shape, dtype=torch.float64, device=device or "cuda")
        # the staging buffer is reused by the next call: copy synchronously
        dev.copy_(src, non_blocking=not staged)
        return cls(field.grid, field.ncomp, dev)

    @property
    def interior(self):
        g = self.grid.ghost_width
        return self.data[(slice(None),) + tuple(slice(g, g + n) for n in self.grid.interior_shape)]

    def to_host(self, like=None):
        """Reference Field with zero ghosts (solver.py:196 field_from_interior):
        one contiguous DMA into a reused pinned staging buffer, one host copy
        into the returned array, ghosts zeroed on the host."""
        a = _d2h(self.data)
        g = self.grid.ghost_width
        for j, n in enumerate(self.grid.interior_shape):  # zero the ghost slabs on the host
            lo = [slice(None)] * a.ndim
            hi = [slice(None)] * a.ndim
            lo[1 + j] = slice(0, g)
            hi[1 + j] = slice(n + g, n + 2 * g)
            a[tuple(lo)] = 0.0
            a[tuple(hi)] = 0.0
        cls = type(like) if like is not None and not isinstance(like, DeviceField) else (TYPES["Field"] or Field)
        return cls(self.grid, self.ncomp, a)

    def copy(self):
        return DeviceField(self.grid, self.ncomp, self.data.clone())


_STAGING_TLS = __import__("threading").local()  # per-thread pinned staging buffers (ranks may be threads)


def _staging(key, shape):
    import torch

    cache = getattr(_STAGING_TLS, "bufs", None)
    if cache is None:
        cache = _STAGING_TLS.bufs = {}
    buf = cache.get(key)
    if buf is None:
        buf = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        cache[key] = buf
    return buf


def _d2h(t):
    """Device tensor -> fresh numpy array: one DMA straight into pinned host
    memory that the returned array owns (pageable D2H of a fresh allocation
    runs at ~2 GB/s: page faults).  The pinned block comes from torch's
    caching host allocator, so steady-state calls allocate nothing and no
    host-side copy follows the DMA; it returns to the cache when the caller
    drops the array."""
    import os

    import torch

    mode = os.environ.get("FVB_D2H", "pinned")
    if mode == "pageable":
        return t.cpu().numpy()
    if mode == "staged":  # reused staging buffer + host copy (the previous scheme)
        buf = _staging(("d2h", tuple(t.shape), t.device.index), tuple(t.shape))
        buf.copy_(t)
        out = np.empty(tuple(t.shape))
        torch.from_numpy(out).copy_(buf)
        return out
    buf = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    buf.copy_(t)
    return buf.numpy()


def pinned_field(field):
    """Copy of a host Field whose data lives in pinned (page-locked) memory,
    so run_simulation's host<->device copies are single DMAs."""
    import torch

    t = torch.empty(tuple(field.data.shape), dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = field.data
    return type(field)(field.grid, field.ncomp, t.numpy())


def _ptr(t) -> int:
    return t.data_ptr()


def _as_device(field):
    if isinstance(field, DeviceField):
        return field, True
    return DeviceField.from_host(field), False


# ---------------------------------------------------------------------------
# error messages in the reference's shapes
# ---------------------------------------------------------------------------

def _cell_index(grid, flat: int) -> tuple:
    """Flat (z*ny + y)*nx + x -> numpy index tuple over interior_shape."""
    return tuple(int(i) for i in np.unravel_index(int(flat), grid.interior_shape))


def _raise_run_error(info: N.RunInfo, grid, ncomp: int, dev=None):
    sub = info.errsub
    if info.err == N.E_STATIC:
        raise E.StaticFieldError("static field: all wave speeds vanish")
    if sub == N.SUB_INIT_UNPHYS:
        raise E.SimulationError("initial field contains unphysical states")
    if sub == N.SUB_STAGE_UNPHYS:
        raise E.SimulationError(f"unphysical state in interior cell {_cell_index(grid, info.errcell)}")
    if sub == N.SUB_NONFINITE:
        ncell = math.prod(grid.cells)
        bad = _cell_index(grid, int(info.errcell) % ncell)
        raise E.SimulationError(f"non-finite value after step {info.steps} (t = {info.t:.6g}) at cell {bad}")
    if sub == N.SUB_POST_UNPHYS:
        raise E.SimulationError(f"unphysical state after step {info.steps} (t = {info.t:.6g})")
    if sub == N.SUB_HLLC:
        raise E.UnphysicalStateError("degenerate HLLC wave fan (sL >= sR)")
    if sub == N.SUB_REMOTE:
        raise E.SimulationError("another rank of the decomposed run failed")
    if sub == N.SUB_SPEED_UNPHYS:
        if not 0 <= int(info.errcell) < math.prod(grid.cells):
            raise E.UnphysicalStateError("unphysical state on another rank")
        idx = _cell_index(grid, info.errcell)
        val = ""
        if dev is not None:
            val = f": u = {dev.interior[(slice(None),) + idx].cpu().numpy()}"
        raise E.UnphysicalStateError(f"unphysical state at cell {idx}{val}")
    raise N.status_error(info.err, f"run failed (code {info.err}, detail {sub})")


# ---------------------------------------------------------------------------
# run_simulation (solver.py:199-246)
# ---------------------------------------------------------------------------

class DeviceRun:
    """Drives the device-resident loop of fvb_run_begin/steps/poll/end over
    one or more instances that share a scheme (batched ensembles)."""

    LOG_RING = 4096

    def __init__(self, grid, cfg, bufs, ninst: int = 1, mode: int = N.MODE_T_END, max_steps=None,
                 arith=None, halo_axes=(), log: bool = True, ctx=None):
        self.ctx = ctx or N.context()
        self.grid = grid
        self.cfg = cfg
        self.ncomp = cfg.model.ncomp
        self.ninst = ninst
        self.bufs = bufs
        self.scheme = make_scheme(grid, cfg, arith, halo_axes)
        self.layout = make_layout(grid, self.ncomp)
        self.mode = mode
        ms = -1 if max_steps is None else int(max_steps)
        self.max_steps = ms
        arr = (N.C.c_void_p * 3)(*[N.C.c_void_p(_ptr(b)) for b in bufs])
        self._arr = arr
        lib = self.ctx.lib
        self.log_ring = self.LOG_RING if log else 0
        self.ctx.check(lib.fvb_run_set_log(self.ctx.h, self.log_ring, ninst))
        self.ctx.check(lib.fvb_run_begin(self.ctx.h, N.C.byref(self.scheme), N.C.byref(self.layout), arr,
                                         ninst, mode, ms))
        self.enqueued = 0
        self.records = [[] for _ in range(ninst)]
        self._seen = [0] * ninst

    def steps(self, n: int):
        self.ctx.check(self.ctx.lib.fvb_run_steps(self.ctx.h, int(n)))
        self.enqueued += int(n)

    def poll(self):
        infos = (N.RunInfo * self.ninst)()
        done = (N.C.c_int32 * self.ninst)()
        self.ctx.check(self.ctx.lib.fvb_run_poll(self.ctx.h, infos, done))
        return list(infos), [bool(d) for d in done]

    def read_log(self, infos, seconds_per_step: float):
        """Append TimeStepRecords for steps completed since the last read."""
        if not self.log_ring:
            return
        rec_cls = TYPES["TimeStepRecord"]
        need = [(i, self._seen[i], int(infos[i].steps)) for i in range(self.ninst) if infos[i].steps > self._seen[i]]
        if not need:
            return
        import torch

        # the ring lives in the context; fetch it through run_end-less poll:
        # copy the whole ring (ninst * ring * 16 B) once per batch
        buf = (N.C.c_double * (2 * self.log_ring * self.ninst))()
        # fvb_run_end would deactivate the plan; use a dedicated read
        self._read_ring(buf)
        for i, lo, hi in need:
            if hi - lo > self.log_ring:
                raise RuntimeError("step log overrun")
            for s in range(lo, hi):
                j = s % self.log_ring
                t = buf[2 * (i * self.log_ring + j)]
                dt = buf[2 * (i * self.log_ring + j) + 1]
                self.records[i].append(rec_cls(s + 1, t, dt, seconds_per_step))
            self._seen[i] = hi

    def _read_ring(self, buf):
        self.ctx.check(self.ctx.lib.fvb_run_read_log(self.ctx.h, buf, self.log_ring))

    def end(self):
        infos = (N.RunInfo * self.ninst)()
        rc = self.ctx.lib.fvb_run_end(self.ctx.h, infos, None, 0)
        if rc not in (N.OK,) and not any(i.err for i in infos):
            self.ctx.check(rc)
        return list(infos)

    def result_buffer(self, info) -> int:
        if self.cfg.rk_order == 1:
            return int(info.steps) % 2
        return 0


_LAZY_TYPES: dict = {}


def _lazy_host_field(grid, ncomp, dev_data, like):
    """Host Field for an observer whose ``data`` is copied to the host only
    when first read.  The step's state is kept by a device-to-device copy
    (~10 us for KH2D 1024^2), so an observer that reads the field rarely --
    the CLI's snapshot observer writes only at snapshot times (cli.py:110-118)
    -- costs a stream sync per step instead of a 34 MB D2H; a field kept
    past the observer call still holds that step's values."""
    base = type(like) if like is not None and not isinstance(like, DeviceField) else (TYPES["Field"] or Field)
    cls = _LAZY_TYPES.get(base)
    if cls is None:
        def _get(self):
            d = self.__dict__.get("_host")
            if d is None:
                d = DeviceField(self.grid, self.ncomp, self.__dict__["_dev"]).to_host().data
                self.__dict__["_host"] = d
                self.__dict__["_dev"] = None
            return d

        def _set(self, value):
            self.__dict__["_host"] = value
            self.__dict__["_dev"] = None

        cls = _LAZY_TYPES[base] = type(base.__name__, (base,), {
            "data": property(_get, _set), "__module__": base.__module__,
            "__doc__": base.__doc__})
    f = object.__new__(cls)
    f.__dict__.update(grid=grid, ncomp=ncomp, _dev=dev_data.clone(), _host=None)
    return f


def run_simulation(init, cfg, observers: Sequence[Callable] = (), max_steps: int | None = None, *,
                   arith: str | None = None, batch: int = 256):
    """Advance from t = 0 to t_end on the GPU (solver.py:199-246).

    ``init`` may be a host Field (reference or ours) or a DeviceField; the
    result has the same kind.  Observers are called as in the reference
    (initial state, then after every accepted step) with host Fields.
    """
    import torch

    grid = init.grid
    check_scheme(grid, cfg)
    _check_periodic(grid, cfg.bc)
    dev, was_dev = _as_device(init)
    b0 = dev.data.clone() if was_dev else dev.data
    bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
    run = DeviceRun(grid, cfg, bufs, 1, N.MODE_T_END, max_steps, arith)
    if observers:
        infos, done = run.poll()
        if infos[0].err:
            run.end()
            _raise_run_error(infos[0], grid, dev.ncomp, dev)
        first = init.copy() if not was_dev else _lazy_host_field(grid, dev.ncomp, b0, init)
        for obs in observers:
            obs(0, 0.0, first)
    step_batch = 1 if observers else batch
    last_obs = 0
    while True:
        infos, done = run.poll()
        if infos[0].err or done[0]:
            break
        n = step_batch
        if max_steps is not None:
            n = min(n, max(1, int(max_steps) - int(infos[0].steps)))
        if infos[0].dt > 0 and not observers:
            # about the steps left to t_end (+ slack); extra launches exit early
            left = (cfg.t_end - infos[0].t) / infos[0].dt
            n = int(min(n, max(1, math.ceil(left) + 2)))
        tic = time.perf_counter()
        run.steps(n)
        infos, done = run.poll()
        secs = (time.perf_counter() - tic) / max(1, infos[0].steps - run._seen[0])
        run.read_log(infos, secs)
        if infos[0].err:
            break
        if observers and infos[0].steps > last_obs:
            last_obs = int(infos[0].steps)
            host = _lazy_host_field(grid, dev.ncomp, bufs[run.result_buffer(infos[0])], init)
            for obs in observers:
                obs(last_obs, float(infos[0].t), host)
    final_info = run.end()[0]
    if final_info.err:
        _raise_run_error(final_info, grid, dev.ncomp, DeviceField(grid, dev.ncomp, bufs[run.result_buffer(final_info)]))
    out = DeviceField(grid, dev.ncomp, bufs[run.result_buffer(final_info)])
    if not was_dev:
        return out.to_host(init), run.records[0]  # ghosts zeroed on the host copy
    keep = out.interior.clone()  # zero ghosts like field_from_interior (solver.py:196)
    out.data.zero_()
    out.interior.copy_(keep)
    return out, run.records[0]


# ---------------------------------------------------------------------------
# single-shot kernels
# ---------------------------------------------------------------------------

def spatial_residual(field, cfg, *, arith: str | None = None) -> np.ndarray:
    """solver.py:82-113.  Ghost cells are taken from ``field`` as given
    (the caller fills them), exactly like the reference."""
    import torch

    grid = field.grid
    check_scheme(grid, cfg)
    ctx = N.context()
    dev, was_dev = _as_device(field)
    out = torch.empty_like(dev.data)
    s = make_scheme(grid, cfg, arith, all_halo=True)
    L = make_layout(grid, dev.ncomp)
    ctx.check(ctx.lib.fvb_spatial_residual(ctx.h, N.C.byref(s), N.C.byref(L), N.C.c_void_p(_ptr(dev.data)),
                                           N.C.c_void_p(_ptr(out)), 1))
    res = DeviceField(grid, dev.ncomp, out).interior
    return res if was_dev else res.cpu().numpy().copy()


def wave_speed_maxima(field, cfg, *, arith: str | None = None) -> np.ndarray:
    """solver.py:128-136 (check=True)."""
    grid = field.grid
    ctx = N.context()
    dev, _ = _as_device(field)
    s = make_scheme(grid, cfg, arith)
    L = make_layout(grid, dev.ncomp)
    out = (N.C.c_double * grid.dim)()
    rc = ctx.lib.fvb_wave_speed_maxima(ctx.h, N.C.byref(s), N.C.byref(L), N.C.c_void_p(_ptr(dev.data)), 1, out)
    if rc == N.E_UNPHYSICAL:
        msg = ctx.message()
        flat = int(msg.split("cell ")[1].split(" ")[0])
        idx = _cell_index(grid, flat)
        val = dev.interior[(slice(None),) + idx].cpu().numpy()
        raise E.UnphysicalStateError(f"unphysical state at cell {idx}: u = {val}")
    ctx.check(rc)
    return np.array([out[k] for k in range(grid.dim)])


def dt_from_maxima(maxima, deltas, cfl: float, remaining: float | None = None) -> float:
    """solver.py:139-149 (host scalar arithmetic, same operation order)."""
    denom = 0.0
    for k in range(len(deltas)):
        denom += maxima[k] / deltas[k]
    if denom == 0.0:
        raise E.StaticFieldError("static field: all wave speeds vanish")
    dt = cfl / denom
    if remaining is not None:
        dt = min(dt, remaining)
    return dt


def stable_dt(field, cfg, remaining: float | None = None, *, arith: str | None = None) -> float:
    return dt_from_maxima(wave_speed_maxima(field, cfg, arith=arith), field.grid.deltas, cfg.cfl, remaining)


def ssp_rk_advance(u, dt: float, L: Callable, order: int):
    """solver.py:158-173 for any array type (numpy or CUDA tensors)."""
    if order == 1:
        return u + dt * L(u)
    if order == 2:
        u1 = u + dt * L(u)
        return 0.5 * u + 0.5 * (u1 + dt * L(u1))
    if order == 3:
        u1 = u + dt * L(u)
        u2 = 0.75 * u + 0.25 * (u1 + dt * L(u1))
        return (1.0 / 3.0) * u + (2.0 / 3.0) * (u2 + dt * L(u2))
    raise E.ConfigError(f"unsupported rk order {order}")


def ssp_rk_step(field, dt: float, cfg, fill_ghosts=None, residual=None, *, arith: str | None = None):
    """solver.py:176-196.  Without hooks: one fused kernel per stage
    (fvb_ssp_rk_step).  With hooks (parallel.py passes them) the stages run
    through the hooks, the combination on the GPU via torch tensors."""
    import torch

    grid = field.grid
    check_scheme(grid, cfg)
    dev, was_dev = _as_device(field)
    if fill_ghosts is None and residual is None:
        _check_periodic(grid, cfg.bc)
        ctx = N.context()
        s = make_scheme(grid, cfg, arith)
        L = make_layout(grid, dev.ncomp)
        un = dev.data.clone()
        w1, w2 = torch.empty_like(un), torch.empty_like(un)
        ctx.check(ctx.lib.fvb_ssp_rk_step(ctx.h, N.C.byref(s), N.C.byref(L), N.C.c_void_p(_ptr(un)),
                                          N.C.c_void_p(_ptr(w1)), N.C.c_void_p(_ptr(w2)), 1, float(dt)))
        out = DeviceField(grid, dev.ncomp, un)
    else:
        fill = fill_ghosts or (lambda f: fill_boundary_device(f, cfg.bc))
        resid = residual or (lambda f, c: spatial_residual(f, c, arith=arith))

        def L(inner):
            stage = DeviceField(grid, dev.ncomp, torch.zeros_like(dev.data))
            stage.interior.copy_(inner)
            host_hook = not isinstance(fill_ghosts, type(None)) or residual is not None
            f = stage.to_host() if host_hook else stage
            if host_hook:
                f.data[...] = 0.0
                f.interior[...] = inner.cpu().numpy()
            fill(f)
            r = resid(f, cfg)
            return torch.as_tensor(np.asarray(r) if not torch.is_tensor(r) else r, device=dev.data.device)

        new = ssp_rk_advance(dev.interior.clone(), dt, L, cfg.rk_order)
        out = DeviceField(grid, dev.ncomp, torch.zeros_like(dev.data))
        out.interior.copy_(new)
    keep = out.interior.clone()
    out.data.zero_()
    out.interior.copy_(keep)
    return out if was_dev else out.to_host(field)


def fill_boundary_device(dev: DeviceField, bc):
    grid = dev.grid
    bc = tuple(bc)
    if len(bc) != grid.dim:
        raise E.ConfigError(f"need {grid.dim} boundary kinds, got {len(bc)}")
    _check_periodic(grid, bc)

    class _Cfg:  # minimal scheme carrier for the descriptor
        pass

    ctx = N.context()
    s = N.Scheme()
    s.dim = grid.dim
    s.ncomp = dev.ncomp
    s.eq = 0 if dev.ncomp == grid.dim + 2 else 1
    s.ghost = grid.ghost_width
    s.rk_order = 1
    for k in range(3):
        s.cells[k] = grid.cells[k] if k < grid.dim else 1
        s.deltas[k] = grid.deltas[k] if k < grid.dim else 1.0
        s.bc[k] = (N.BC_PERIODIC if _v(bc[k]) == "periodic" else N.BC_OUTFLOW) if k < grid.dim else 0
    s.gamma = 1.4
    L = make_layout(grid, dev.ncomp)
    ctx.check(ctx.lib.fvb_fill_ghosts(ctx.h, N.C.byref(s), N.C.byref(L), N.C.c_void_p(_ptr(dev.data)), 1))
    return dev


def _device_fill_boundary(field, bc):
    """grid.fill_boundary: mutates ``field`` (host or device) and returns it."""
    if isinstance(field, DeviceField):
        return fill_boundary_device(field, bc)
    dev = DeviceField.from_host(field)
    fill_boundary_device(dev, bc)
    field.data[...] = dev.data.cpu().numpy()
    return field
