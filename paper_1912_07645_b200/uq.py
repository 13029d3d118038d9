"""On-GPU Monte Carlo / quasi-Monte Carlo statistics (uq.py:25-322 of the
reference) on the B200 path.

* Sampling (``SamplePlan``, ``draw_sample``, Halton) stays on the host and is
  the reference algorithm unchanged, so sample vectors are identical.
* Each batch of samples runs as ONE batched device run (one instance per
  sample, per-instance dt/t/stop flag, csrc/fvb_state.cuh); final fields
  never leave HBM: ``FieldMoments`` and ``StructureFunctionAccumulator`` are
  updated by CUDA kernels (fvb_moments_push / fvb_structure_push) in
  sample-index order, which reproduces run_mc's ordered merge
  (uq.py:318-321) bitwise on one GPU.
* Under ``torch.distributed`` (one process per GPU) samples are sharded in
  contiguous blocks and the per-rank accumulators are merged once at the end
  in rank order (one all_gather; Chan merge on the GPU).

Functionals are duck-typed by ``name`` like write_stats dispatches them
(output.py:158-191); the reference's own FieldMoments /
StructureFunctionAccumulator prototypes are accepted and returned filled.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .solver import DeviceField, DeviceRun, _raise_run_error, check_scheme, make_layout, make_scheme

MC = "mc"
QMC = "qmc"
_PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53)


@dataclass(frozen=True)
class SamplePlan:
    method: str = MC
    samples: int = 1
    seed: int = 0
    stochastic_dim: int = 1

    def __post_init__(self):
        if self.method not in (MC, QMC):
            raise E.ConfigError(f"unknown sampling method {self.method!r}")
        if self.samples < 1:
            raise E.ConfigError(f"sample count must be >= 1, got {self.samples}")
        if self.stochastic_dim < 1:
            raise E.ConfigError(f"stochastic_dim must be >= 1, got {self.stochastic_dim}")


@dataclass(frozen=True)
class MlmcPlan:
    """Level grids coarsest to finest; every axis equal or doubled per level
    (uq.py:47-76)."""

    grids: tuple
    samples_per_level: tuple
    method: str = MC
    seed: int = 0
    stochastic_dim: int = 1

    def __post_init__(self):
        if len(self.grids) != len(self.samples_per_level):
            raise E.ConfigError("need one sample count per level")
        if len(self.grids) < 1:
            raise E.ConfigError("MLMC needs at least one level")
        if any(m < 1 for m in self.samples_per_level):
            raise E.ConfigError("per-level sample counts must be >= 1")
        for lvl in range(1, len(self.grids)):
            coarse, fine = self.grids[lvl - 1], self.grids[lvl]
            same = all(f == c for f, c in zip(fine.cells, coarse.cells))
            doubled = all(f == 2 * c for f, c in zip(fine.cells, coarse.cells))
            if not (same or doubled):
                raise E.ConfigError(f"level {lvl} cells {fine.cells} are neither equal to nor double the "
                                    f"level {lvl - 1} cells {coarse.cells}")

    @property
    def levels(self) -> int:
        return len(self.grids)


def radical_inverse(index: int, base: int) -> float:
    """Van der Corput radical inverse (uq.py:79-87)."""
    inv, factor = 0.0, 1.0 / base
    while index > 0:
        inv += factor * (index % base)
        index //= base
        factor /= base
    return inv


def halton_point(index: int, dim: int) -> np.ndarray:
    if dim > len(_PRIMES):
        raise E.ConfigError(f"Halton supports up to {len(_PRIMES)} dimensions")
    return np.array([radical_inverse(index, _PRIMES[d]) for d in range(dim)])


def draw_sample(plan, k: int, level: int = 0) -> np.ndarray:
    """uq.py:97-106: Philox keyed by (seed, level<<48 + k) or Halton k+1."""
    samples = plan.samples_per_level[level] if hasattr(plan, "samples_per_level") else plan.samples
    if not 0 <= k < samples:
        raise E.ConfigError(f"sample index {k} out of range [0, {samples})")
    if plan.method == QMC:
        return halton_point(k + 1, plan.stochastic_dim)
    key = [np.uint64(plan.seed), np.uint64((level << 48) + k)]
    return np.random.Generator(np.random.Philox(key=key)).random(plan.stochastic_dim)


# ---------------------------------------------------------------------------
# GPU-resident functionals
# ---------------------------------------------------------------------------

class MomentAccumulator:
    """Host view with the reference's fields (uq.py:114-158)."""

    def __init__(self, shape):
        self.count = 0
        self.mean = np.zeros(shape)
        self.m2 = np.zeros(shape)

    def variance(self, ddof: int = 1) -> np.ndarray:
        if self.count <= ddof:
            return np.zeros_like(self.m2)
        return self.m2 / (self.count - ddof)

    def second_moment(self) -> np.ndarray:
        if self.count == 0:
            return np.zeros_like(self.m2)
        return self.m2 / self.count + self.mean ** 2


class FieldMoments:
    """Per-cell mean and M2 of the conserved field, kept in HBM."""

    name = "moments"

    def __init__(self, grid, ncomp: int):
        self.grid = grid
        self.ncomp = ncomp
        self.count = 0
        self._mean = None
        self._m2 = None

    def fresh(self):
        return FieldMoments(self.grid, self.ncomp)

    def _alloc(self):
        import torch

        if self._mean is None:
            shape = (self.ncomp,) + tuple(self.grid.interior_shape)
            self._mean = torch.zeros(shape, dtype=torch.float64, device="cuda")
            self._m2 = torch.zeros(shape, dtype=torch.float64, device="cuda")

    def push_device(self, ctx, scheme, layout, buf, inst: int):
        """Merge one sample's final field (instance ``inst`` of ``buf``)."""
        self._alloc()
        ctx.check(ctx.lib.fvb_moments_push(ctx.h, N.C.byref(scheme), N.C.byref(layout), N.C.c_void_p(buf.data_ptr()),
                                           inst, N.C.c_void_p(self._mean.data_ptr()),
                                           N.C.c_void_p(self._m2.data_ptr()), self.count))
        self.count += 1

    def push_device_batch(self, ctx, scheme, layout, buf, inst: int, n: int):
        """Merge instances inst .. inst+n-1 of ``buf`` in that order: one
        kernel, (mean, M2) read and written once (bitwise equal to n pushes)."""
        self._alloc()
        ctx.check(ctx.lib.fvb_moments_push_batch(ctx.h, N.C.byref(scheme), N.C.byref(layout),
                                                 N.C.c_void_p(buf.data_ptr()), inst, int(n),
                                                 N.C.c_void_p(self._mean.data_ptr()),
                                                 N.C.c_void_p(self._m2.data_ptr()), self.count))
        self.count += int(n)

    def update(self, field) -> None:
        """FieldMoments.update (uq.py:174-175) for one field."""
        dev = field if isinstance(field, DeviceField) else DeviceField.from_host(field)
        ctx = N.context()
        s = _descriptor(dev.grid, dev.ncomp)
        self.push_device(ctx, s, make_layout(dev.grid, dev.ncomp), dev.data, 0)

    def merge(self, other: "FieldMoments") -> None:
        """MomentAccumulator.merge (uq.py:135-148) on the GPU."""
        if other.count == 0:
            return
        self._alloc()
        ctx = N.context()
        ctx.check(ctx.lib.fvb_moments_merge(ctx.h, N.C.c_void_p(self._mean.data_ptr()),
                                            N.C.c_void_p(self._m2.data_ptr()), self.count,
                                            N.C.c_void_p(other._mean.data_ptr()), N.C.c_void_p(other._m2.data_ptr()),
                                            other.count, self._mean.numel()))
        self.count += other.count

    @property
    def acc(self) -> MomentAccumulator:
        a = MomentAccumulator((self.ncomp,) + tuple(self.grid.interior_shape))
        a.count = self.count
        if self._mean is not None:
            a.mean = self._mean.cpu().numpy()
            a.m2 = self._m2.cpu().numpy()
        return a


class StructureFunctionAccumulator:
    """Mean |u(x + h e_k) - u(x)|^p over positions and axes (uq.py:231-273);
    the per-sample sums are computed by fvb_structure_push on the GPU."""

    name = "structure_function"

    def __init__(self, p: float, max_offset: int, component: int = 0):
        if p < 1:
            raise E.ConfigError(f"structure-function exponent must be >= 1, got {p}")
        if max_offset < 0:
            raise E.ConfigError(f"max offset must be >= 0, got {max_offset}")
        self.p = float(p)
        self.max_offset = int(max_offset)
        self.component = int(component)
        self.samples = 0
        self._sums = None

    def fresh(self):
        return StructureFunctionAccumulator(self.p, self.max_offset, self.component)

    def _alloc(self):
        import torch

        if self._sums is None:
            self._sums = torch.zeros(self.max_offset + 1, dtype=torch.float64, device="cuda")

    def push_device(self, ctx, scheme, layout, buf, inst: int):
        self._alloc()
        ctx.check(ctx.lib.fvb_structure_push(ctx.h, N.C.byref(scheme), N.C.byref(layout),
                                             N.C.c_void_p(buf.data_ptr()), inst, self.component, self.p,
                                             self.max_offset, N.C.c_void_p(self._sums.data_ptr())))
        self.samples += 1

    def update(self, field) -> None:
        dev = field if isinstance(field, DeviceField) else DeviceField.from_host(field)
        ctx = N.context()
        self.push_device(ctx, _descriptor(dev.grid, dev.ncomp), make_layout(dev.grid, dev.ncomp), dev.data, 0)

    def merge(self, other: "StructureFunctionAccumulator") -> None:
        if other.max_offset != self.max_offset or other.p != self.p:
            raise E.ConfigError("structure-function specs do not match")
        self._alloc()
        if other._sums is not None:
            self._sums += other._sums
        self.samples += other.samples

    @property
    def sums(self) -> np.ndarray:
        return np.zeros(self.max_offset + 1) if self._sums is None else self._sums.cpu().numpy()

    def values(self) -> np.ndarray:
        if self.samples == 0:
            return np.zeros(self.max_offset + 1)
        return self.sums / self.samples


class Histogram:
    """Per-probe histogram of one component with under/overflow bins
    (uq.py:181-228).  Only the probe values of each sample leave the GPU (a
    gather of len(probe_cells) doubles); binning follows the reference
    expression by expression."""

    name = "histogram"

    def __init__(self, probe_cells, component: int, lo: float, hi: float, bins: int = 64):
        if hi <= lo:
            raise E.ConfigError(f"histogram range [{lo}, {hi}) is empty")
        if bins < 1:
            raise E.ConfigError(f"histogram needs >= 1 bins, got {bins}")
        self.probe_cells = tuple(tuple(int(i) for i in p) for p in probe_cells)
        self.component = component
        self.lo = float(lo)
        self.hi = float(hi)
        self.bins = int(bins)
        self.counts = np.zeros((len(self.probe_cells), bins + 2), dtype=np.int64)
        self.samples = 0

    @property
    def edges(self) -> np.ndarray:
        return np.linspace(self.lo, self.hi, self.bins + 1)

    def fresh(self):
        return Histogram(self.probe_cells, self.component, self.lo, self.hi, self.bins)

    def add_values(self, values) -> None:
        width = (self.hi - self.lo) / self.bins
        for p, v in enumerate(values):
            v = float(v)
            if v < self.lo:
                self.counts[p, 0] += 1
            elif v >= self.hi:
                self.counts[p, -1] += 1
            else:
                self.counts[p, 1 + min(int((v - self.lo) / width), self.bins - 1)] += 1
        self.samples += 1

    def gather(self, data, grid):
        """Probe values of one padded (ncomp, *data_shape) field (host or device)."""
        g = grid.ghost_width
        idx = [(self.component,) + tuple(g + i for i in reversed(cell)) for cell in self.probe_cells]
        if isinstance(data, np.ndarray):
            return [data[i] for i in idx]
        import torch

        cols = list(zip(*idx))
        return data[tuple(torch.tensor(c, device=data.device) for c in cols)].cpu().numpy()

    def update(self, field) -> None:
        self.add_values(self.gather(field.data, field.grid))

    def merge(self, other: "Histogram") -> None:
        if other.counts.shape != self.counts.shape:
            raise E.ConfigError("histogram shapes do not match")
        self.counts += other.counts
        self.samples += other.samples


def _descriptor(grid, ncomp):
    s = N.Scheme()
    s.dim = grid.dim
    s.ncomp = ncomp
    s.eq = 0 if ncomp == grid.dim + 2 else 1
    s.ghost = grid.ghost_width
    s.rk_order = 1
    for k in range(3):
        s.cells[k] = grid.cells[k] if k < grid.dim else 1
        s.deltas[k] = grid.deltas[k] if k < grid.dim else 1.0
    return s


# ---------------------------------------------------------------------------
# estimator
# ---------------------------------------------------------------------------

class _Slot:
    """One requested functional: our GPU accumulator + how to hand it back."""

    def __init__(self, proto, grid, ncomp):
        self.proto = proto
        name = getattr(proto, "name", None)
        self.kind = name
        if name == "moments":
            self.gpu = FieldMoments(grid, ncomp)
        elif name == "structure_function":
            self.gpu = StructureFunctionAccumulator(proto.p, proto.max_offset, getattr(proto, "component", 0))
        elif name == "histogram":
            self.gpu = None
            self.hist = Histogram(proto.probe_cells, proto.component, proto.lo, proto.hi, proto.bins)
        else:
            self.gpu = None  # other host functionals: fed host fields
            self.host = proto.fresh()

    def push(self, ctx, scheme, layout, buf, inst, grid, ncomp, like):
        if self.gpu is not None:
            self.gpu.push_device(ctx, scheme, layout, buf, inst)
        elif self.kind == "histogram":
            self.hist.add_values(self.hist.gather(buf[inst], grid))
        else:
            one = DeviceField(grid, ncomp, buf[inst]).to_host(like)
            c = self.proto.fresh()
            c.update(one)
            self.host.merge(c)

    def result(self):
        """Return an object of the caller's functional type."""
        if self.kind == "histogram":
            if isinstance(self.proto, Histogram):
                return self.hist
            out = self.proto.fresh()
            out.counts, out.samples = self.hist.counts, self.hist.samples
            return out
        if self.gpu is None:
            return self.host
        if isinstance(self.proto, (FieldMoments, StructureFunctionAccumulator)):
            return self.gpu
        out = self.proto.fresh()  # reference class: fill its public fields
        if self.kind == "moments":
            acc = self.gpu.acc
            out.acc.count, out.acc.mean, out.acc.m2 = acc.count, acc.mean, acc.m2
        else:
            out.sums = self.gpu.sums
            out.samples = self.gpu.samples
        return out


def shard_range(n: int, world: int, rank: int):
    """Contiguous sample block of ``rank``: [rank*n//world, (rank+1)*n//world)."""
    return (rank * n) // world, ((rank + 1) * n) // world


def default_batch(grid, ncomp: int) -> int:
    """Samples per device batch: ~16M cell-components (KH2D 512^2: 16,
    Burgers 2048^2: 4), at most 64; even when possible (the scalar ring
    kernel marches two instances per block)."""
    cells = math.prod(grid.cells)
    b = int(max(1, min(64, (16 << 20) // max(1, cells * ncomp))))
    return b - (b % 2) if b > 1 else b


def run_mc(plan, grid, cfg, evaluate_init, functionals, workers: int = 1, *, batch: int | None = None,
           arith: str | None = None, group=None, max_steps: int | None = None):
    """Single-level estimate (uq.py:302-322) on the GPU.

    ``workers`` sizes the host pool that evaluates a host ``evaluate_init``
    a batch ahead (the GPU batch replaces the reference's per-sample thread
    pool).  Under an initialised torch.distributed group the samples are
    sharded over the ranks (contiguous blocks) and every rank returns the
    merged result.  ``max_steps`` caps the steps of every sample
    (run_simulation's max_steps, solver.py:199-246) -- bench.py uses it for
    fixed-work timing.
    """
    import torch

    check_scheme(grid, cfg)
    ncomp = cfg.model.ncomp
    world, rank = 1, 0
    dist = None
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        dist = torch.distributed
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = shard_range(plan.samples, world, rank)
    slots = [_Slot(f, grid, ncomp) for f in functionals]
    _ensemble(plan, 0, grid, cfg, evaluate_init, slots, lo, hi, batch, arith, workers, max_steps)
    if dist is not None and world > 1:
        _merge_ranks(slots, dist, group, world)
    return [s.result() for s in slots]


def gather_ordered(tensors, count: int, dist, group, world):
    """All-gather one rank's (count, tensors) block; returns the blocks of all
    ranks in rank order -- the order run_mc merges samples in."""
    import torch

    dev = tensors[0].device
    # gloo moves host tensors only: stage device data through host memory
    host = dist.get_backend(group) == "gloo" and dev.type == "cuda"
    cnt = torch.tensor([int(count)], dtype=torch.int64, device="cpu" if host else dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    gathered = []
    for t in tensors:
        src = t.contiguous().cpu() if host else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src, group=group)
        gathered.append([x.to(dev) for x in parts] if host else parts)
    return [(int(cnts[r].item()), [g[r] for g in gathered]) for r in range(world)]


_PINNED: dict = {}
_PINNED_LOCK = threading.Lock()


def _pinned_stage(key):
    """Persistent pinned host buffer for (owner thread, parity, shape)."""
    import torch

    with _PINNED_LOCK:
        buf = _PINNED.get(key)
        if buf is None:
            buf = _PINNED[key] = torch.empty(key[2], dtype=torch.float64, pin_memory=True)
        return buf


def _ensemble(plan, level, grid, cfg, evaluate_init, slots, lo, hi, batch=None, arith=None, workers=1,
              max_steps=None):
    """Samples [lo, hi) of one level: batched device runs (one instance per
    sample), each final field pushed into every slot in sample order.

    The host-side initial data of batch b+1 (the caller's ``evaluate_init``,
    stacked into pinned memory) is prepared on helper threads while batch b
    runs on the GPU -- ``workers`` of them evaluate samples concurrently, the
    role the reference gives its thread pool (uq.py:302-322); a failing
    sample raises at the same point, with the same message, as without the
    overlap (the lowest failing sample of the batch, after batch b has been
    pushed)."""
    import concurrent.futures as cf

    import torch

    ncomp = cfg.model.ncomp
    B = batch or default_batch(grid, ncomp)
    ctx = N.context()
    layout = make_layout(grid, ncomp)
    desc = make_scheme(grid, cfg, arith)
    mlmc = hasattr(plan, "samples_per_level")
    where = f"level {level}, " if mlmc else ""
    batches = [list(range(k, min(hi, k + B))) for k in range(lo, hi, B)]

    nw = max(1, int(workers or 1))
    evals = cf.ThreadPoolExecutor(max_workers=nw) if nw > 1 else None

    def one(j):
        try:
            return evaluate_init(grid, draw_sample(plan, j, level)), None
        except Exception as exc:  # reported in sample order by prepare()
            return None, exc

    owner = threading.get_ident()

    def prepare(ks, parity):
        outs = list(evals.map(one, ks)) if evals else [one(j) for j in ks]
        for j, (_, exc) in zip(ks, outs):
            if exc is not None:
                raise E.SimulationError(f"{where}sample {j} failed: {exc}") from exc
        first = outs[0][0]
        a0 = np.asarray(first.data, dtype=np.float64)
        # two persistent pinned staging buffers per shape, alternating by
        # batch: buffer b % 2 is rewritten only after batch b ran to the end
        host = _pinned_stage((owner, parity, (len(ks),) + a0.shape))
        hv = host.numpy()
        for i, (f0, _) in enumerate(outs):
            hv[i] = np.asarray(f0.data, dtype=np.float64)
        return host, first

    from .initdev import DeviceInit

    on_device = isinstance(evaluate_init, DeviceInit)  # initial data evaluated on the GPU: no host side at all
    try:
        _run_batches(plan, level, grid, cfg, evaluate_init, slots, batches, prepare, on_device, ctx, layout, desc,
                     ncomp, where, arith, max_steps)
    finally:
        if evals:
            evals.shutdown(cancel_futures=True)


def _run_batches(plan, level, grid, cfg, evaluate_init, slots, batches, prepare, on_device, ctx, layout, desc,
                 ncomp, where, arith, max_steps):
    """_ensemble's batch loop: batch b+1's host initial data is prepared on a
    helper thread while batch b runs."""
    import concurrent.futures as cf

    import torch

    like = None
    with cf.ThreadPoolExecutor(max_workers=1) as pool:
        nxt = pool.submit(prepare, batches[0], 0) if batches and not on_device else None
        for b, ks in enumerate(batches):
            if on_device:
                b0 = torch.empty((len(ks), ncomp) + tuple(grid.padded[::-1]), dtype=torch.float64, device="cuda")
                errs = evaluate_init.evaluate_batch(grid, [draw_sample(plan, j, level) for j in ks], b0)
                for j, exc in zip(ks, errs):
                    if exc is not None:
                        raise E.SimulationError(f"{where}sample {j} failed: {exc}") from exc
            else:
                host, first = nxt.result()
                like = like or first
                b0 = host.to("cuda", non_blocking=True)
                nxt = pool.submit(prepare, batches[b + 1], (b + 1) % 2) if b + 1 < len(batches) else None
            bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
            run = DeviceRun(grid, cfg, bufs, len(ks), N.MODE_T_END, max_steps, arith, log=False, ctx=ctx)
            while True:
                infos, done = run.poll()
                if all(done):
                    break
                left = max(((cfg.t_end - i.t) / i.dt) if (i.dt > 0 and not d) else 1 for i, d in zip(infos, done))
                n = min(512, max(1, math.ceil(left) + 2))
                if max_steps is not None:  # no launches past the cap (they would be no-ops)
                    n = min(n, max(1, int(max_steps) - min(int(i.steps) for i, d in zip(infos, done) if not d)))
                run.steps(int(n))
            infos = run.end()
            for j, info in zip(ks, infos):
                if info.err:
                    try:
                        _raise_run_error(info, grid, ncomp)
                    except E.ConslawError as exc:
                        raise E.SimulationError(f"{where}sample {j} failed: {exc}") from exc
            where_ = [int(infos[i].steps) % 2 if cfg.rk_order == 1 else 0 for i in range(len(ks))]
            for s in slots:  # each slot sees the batch's samples in sample order
                if isinstance(s.gpu, FieldMoments) and len(set(where_)) == 1:
                    s.gpu.push_device_batch(ctx, desc, layout, bufs[where_[0]], 0, len(ks))  # one kernel per batch
                    continue
                for i in range(len(ks)):
                    s.push(ctx, desc, layout, bufs[where_[i]], i, grid, ncomp, like)


@dataclass
class MlmcMoments:
    """Telescoped first/second moments on the finest grid (uq.py:325-331)."""

    mean: np.ndarray
    second_moment: np.ndarray
    variance: np.ndarray


def prolong(values, factor_per_axis):
    """Piecewise-constant injection onto a finer grid (uq.py:334-345);
    works on numpy arrays and on device tensors (component axis first, x last,
    factors x-first)."""
    dim = len(factor_per_axis)
    out = values
    for j in range(dim):
        f = factor_per_axis[dim - 1 - j]
        if f != 1:
            out = np.repeat(out, f, axis=1 + j) if isinstance(out, np.ndarray) else out.repeat_interleave(f, dim=1 + j)
    return out


def _second_moment(fm):
    """m2 / count + mean**2 (uq.py:155-158) on the device.  The count is a
    full tensor: torch turns division by a host scalar into a multiplication
    by its (rounded) reciprocal, which would not be bitwise."""
    import torch

    return fm._m2 / torch.full_like(fm._m2, float(fm.count)) + fm._mean * fm._mean


def run_mlmc(plan, make_cfg, evaluate_init, workers: int = 1, *, batch: int | None = None,
             arith: str | None = None):
    """Multilevel estimate of the field mean and variance (uq.py:348-419):
    every level's fine and coarse ensembles run as batched device runs with
    on-GPU moment accumulation; the telescoping sums stay on the device."""
    finest = plan.grids[-1]
    mean_total = second_total = None
    acc0 = None
    for level in range(plan.levels):
        grid_f = plan.grids[level]
        cfg_f = make_cfg(grid_f)
        slot = _Slot(FieldMoments(grid_f, cfg_f.model.ncomp), grid_f, cfg_f.model.ncomp)
        _ensemble(plan, level, grid_f, cfg_f, evaluate_init, [slot], 0, plan.samples_per_level[level], batch, arith,
                  workers)
        acc_f = slot.gpu
        if level == 0:
            acc0 = acc_f
        factor_f = tuple(nf // nl for nf, nl in zip(finest.cells, grid_f.cells))
        mean_l = prolong(acc_f._mean, factor_f)
        second_l = prolong(_second_moment(acc_f), factor_f)
        if level > 0:
            grid_c = plan.grids[level - 1]
            cfg_c = make_cfg(grid_c)
            slot_c = _Slot(FieldMoments(grid_c, cfg_c.model.ncomp), grid_c, cfg_c.model.ncomp)
            _ensemble(plan, level, grid_c, cfg_c, evaluate_init, [slot_c], 0, plan.samples_per_level[level], batch,
                      arith, workers)
            fc = slot_c.gpu
            factor_c = tuple(nf // nl for nf, nl in zip(finest.cells, grid_c.cells))
            mean_l = mean_l - prolong(fc._mean, factor_c)
            second_l = second_l - prolong(_second_moment(fc), factor_c)
        if mean_total is None:
            mean_total, second_total = mean_l, second_l
        else:
            mean_total = mean_total + mean_l
            second_total = second_total + second_l
    if plan.levels == 1:
        variance = acc0.acc.variance(ddof=1)  # telescoping degenerates to single-level sampling
    else:
        variance = (second_total - mean_total * mean_total).cpu().numpy()
    return MlmcMoments(mean_total.cpu().numpy(), second_total.cpu().numpy(), variance)


def _merge_ranks(slots, dist, group, world):
    """Deterministic cross-rank reduce: one all_gather per statistic, then a
    fold in rank order (rank 0's sample block first)."""
    import torch

    for s in slots:
        g = s.gpu
        if isinstance(g, FieldMoments):
            g._alloc()
            tot = FieldMoments(g.grid, g.ncomp)
            for cnt, (mean, m2) in gather_ordered([g._mean, g._m2], g.count, dist, group, world):
                part = FieldMoments(g.grid, g.ncomp)
                part.count, part._mean, part._m2 = cnt, mean, m2
                tot.merge(part)  # Chan merge on the GPU (fvb_moments_merge)
            s.gpu = tot
        elif isinstance(g, StructureFunctionAccumulator):
            g._alloc()
            tot = g.fresh()
            tot._alloc()
            for cnt, (sums,) in gather_ordered([g._sums], g.samples, dist, group, world):
                tot._sums += sums
                tot.samples += cnt
            s.gpu = tot
        elif s.kind == "histogram":
            # counts and sample totals add (uq.py:221-228): all-gather, sum in rank order
            h = s.hist
            counts = torch.as_tensor(np.ascontiguousarray(h.counts), dtype=torch.int64)
            counts = counts.to("cuda") if dist.get_backend(group) == "nccl" else counts
            blocks = gather_ordered([counts], h.samples, dist, group, world)
            tot = np.zeros_like(h.counts)
            for cnt, (c,) in blocks:
                tot = tot + c.cpu().numpy().astype(h.counts.dtype)
            h.counts = tot
            h.samples = sum(cnt for cnt, _ in blocks)
        else:
            # any other host functional: gather the objects, merge in rank order
            objs = [None] * world
            dist.all_gather_object(objs, s.host, group=group)
            tot = s.proto.fresh()
            for o in objs:
                tot.merge(o)
            s.host = tot
