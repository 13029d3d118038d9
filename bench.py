"""Benchmark: Gcell-updates/s per SSP-RK stage (BASELINE.json metric).

Default workload (BASELINE.json configs[1], "C2"): 2D Kelvin-Helmholtz Euler,
WENO2 + HLLC, SSP-RK3, 1024x1024 periodic, fp64 -- the KH2D preset
(presets.py:65-104) with reconstruction=weno2 and the MC seed-42 sample-0
random vector; synthetic data, no checkpoint.  One bench "step" is one full
SSP-RK3 time step (3 fused stage launches, CFL reduction fused into the last
stage, dt computed on the device), timed from the developed state at
t ~ 1 (rolled-up shear layers).  L2 is flushed (256 MiB write) before every
timed step; each step is timed with CUDA events on the launching stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--arith fast|exact] [--config kh2d|mc|kh3d|bqmc]

Multi-GPU: ``--gpus N`` launched without torchrun re-executes itself under
``torch.distributed.run`` with N processes (one per GPU, NCCL).  Per config:

* kh2d (C2, single domain): N independent replicas ("replicas only").
* mc (C3): one "step" = one sharded ``run_mc`` over the whole ensemble
  (default 1024 KH2D samples at 512^2, --mc-steps RK3 steps each, initial
  data evaluated on the GPU), contiguous sample blocks per rank, the moment
  statistics merged across ranks (NCCL all-gather + rank-ordered Chan merge)
  inside the timed region; strong scaling (fixed total samples).
* kh3d (C4): ``DecomposedRun`` -- z-slab domain decomposition, one 512^3
  subdomain per GPU (weak scaling), NCCL halo exchange of the march-axis
  layers in place overlapped with the inner box, one all-reduce(MAX) per
  step for the global dt; one "step" = one RK3 step of the whole domain.
* bqmc (C5 shape): batched Burgers QMC ensemble replicas + on-GPU statistics.

``--impl reference`` times the reference's own CPU implementation on the
host cores: the UNMODIFIED ``conslaw`` package from ``baseline/_ref``
stepping with its own ``ssp_rk_step``/``stable_dt``, its residual seam
(``residual=``) fed by the reference's ``spatial_residual`` evaluated in
row bands by a process pool over all host cores (plus the stock
single-process ``run_simulation`` for one step); the numpy oracle port when
``baseline/_ref`` is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gcell-updates/s per SSP-RK stage"
UNIT = "Gcell-stage/s"
KH_VECTOR = [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203]
N_CELLS = 1024
# the KH presets' initial data (presets.py:65-145), evaluated on the GPU by initdev.DeviceInit
KH_EXPRS = [
    "y < 0.25 + 0.01 * sin(2 * pi * (x + X0)) ? 1.0 : (y < 0.75 + 0.01 * sin(2 * pi * (x + X1)) ? 2.0 : 1.0)",
    "y < 0.25 + 0.01 * sin(2 * pi * (x + X2)) ? -0.5 : (y < 0.75 + 0.01 * sin(2 * pi * (x + X3)) ? 0.5 : -0.5)",
]
REF_PATH = ROOT / "baseline" / "_ref"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _hbm_peak():
    pk = _peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------

class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/fvb_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": float(np.median(loaded or sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# our arm: shared plumbing
# ---------------------------------------------------------------------------

class Env:
    """Device, stream and (for N > 1, or kh3d) the process group."""

    def __init__(self, ws, rank, local, need_group=False):
        import torch

        self.ws, self.rank = ws, rank
        ndev = torch.cuda.device_count()
        self.dev_index = local % max(1, ndev)
        torch.cuda.set_device(self.dev_index)
        self.dist = None
        if ws > 1 or need_group:
            import torch.distributed as dist

            if ws == 1 and "MASTER_ADDR" not in os.environ:  # a one-rank group (kh3d at N = 1)
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
                                  WORLD_SIZE="1")
            if ws <= ndev:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.dev_index))
            else:  # more ranks than GPUs (a smoke run on a small box): gloo for the host-side reduces only
                dist.init_process_group("gloo")
            self.dist = dist
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)

    @property
    def nccl(self):
        return self.dist is not None and self.dist.get_backend() == "nccl"

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        if self.dist is not None:
            if self.nccl:
                self.dist.barrier(device_ids=[self.dev_index])
            else:
                self.dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        import torch

        if self.dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if self.nccl else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.barrier()
            self.dist.destroy_process_group()


def _timed(env, fn, reps, flush=None, stream=None):
    """reps x fn() between CUDA events on the stream the work is issued on
    (env.stream unless given), barrier + sync on both sides; returns
    (per-rep ms, max-over-ranks total ms)."""
    import torch

    stream = stream or env.stream
    evs = []
    env.barrier()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
            stream.wait_stream(env.stream)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    env.barrier()
    per = [a.elapsed_time(b) for a, b in evs]
    return per, env.max_over_ranks(float(sum(per)))


def _roofline(bytes_per_cell_stage, cell_stages, seconds, kernel, traffic=None, compute=None):
    peak, src = _hbm_peak()
    achieved = bytes_per_cell_stage * cell_stages / seconds / 1e9
    r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": src, "kernel": kernel,
         "algorithmic_bytes_per_cell_stage": round(bytes_per_cell_stage, 2)}
    if compute:
        r["compute"] = compute
    return r


def _profile_json(name):
    p = ROOT / "profiles" / name
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def _traffic_key(roof, name):
    """ncu DRAM bytes per stage launch of the same kernel and workload (profiles/)."""
    t = _profile_json(name)
    if t:
        roof["traffic"] = t.get("stage_bytes_per_launch")
        roof["traffic_source"] = t.get("source")


def _kh2d_profile_keys(roof):
    """traffic (ncu dram bytes per stage launch) and the FP64 roof from the
    committed captures of the same kernel (profiles/)."""
    t = _profile_json("traffic.json")
    if t:
        roof["traffic"] = t.get("stage_bytes_per_launch")
    f = _profile_json("fp64_roof.json")
    if f:
        try:
            st = f["ring_kernel_stages"]
            ach = sum(x["fp64_tflops"] * x["us"] for x in st) / sum(x["us"] for x in st)
            pk = f["measured_peak"]["dfma_peak_tflops"]
            roof["compute"] = {"bound": "fp64", "achieved": round(ach, 2), "peak": pk, "unit": "TFLOP/s",
                               "frac": round(ach / pk, 4),
                               "fp64_pipe_pct": round(sum(x["fp64_pipe_pct"] for x in st) / len(st), 1),
                               "source": "profiles/fp64_roof.json (ncu, tools/fp64_peak.cu)"}
        except Exception:
            pass


# ---------------------------------------------------------------------------
# kh2d (C2) and bqmc (C5 shape): replicas of one device run per rank
# ---------------------------------------------------------------------------

def bench_single(args, env):
    import torch

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import _native as N
    from paper_1912_07645_b200.initial import kelvin_helmholtz
    from paper_1912_07645_b200.solver import DeviceField, DeviceRun

    n = args.cells
    grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    burgers = args.config == "bqmc"
    if burgers:  # configs[4]: the authored Burgers QMC scheme (Rusanov, WENO2, RK3, CFL 0.475)
        cfg = P.SchemeConfig(P.EquationModel("burgers", 2), P.FluxKind.RUSANOV,
                             P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
        from paper_1912_07645_b200.initial import burgers_sines
        from paper_1912_07645_b200.uq import SamplePlan, draw_sample

        ninst = args.samples
        plan = SamplePlan("qmc", ninst, 42, 2)
        inits = [burgers_sines(grid, draw_sample(plan, k)) for k in range(ninst)]
        init = inits[0]
        b0 = torch.from_numpy(np.stack([f.data for f in inits])).to("cuda")
    else:
        cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                             P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
        ninst = 1
        init = kelvin_helmholtz(grid, KH_VECTOR)
        if args.state_file and Path(args.state_file).exists():
            init = P.Field(grid, 4, np.load(args.state_file))  # developed state saved by tools/make_state.py
            args.warm_time = 0.0
        b0 = DeviceField.from_host(init).data
    bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
    run = DeviceRun(grid, cfg, bufs, ninst, N.MODE_FIXED, 1 << 40, args.arith, log=False)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    cells = n * n * ninst
    ncomp = 1 if burgers else 4

    run.steps(args.warmup)
    # advance to a developed state (KH roll-up under way) before timing, so
    # the timed steps are representative of a run to t_end rather than of the
    # piecewise-constant initial bands
    while True:
        infos, _ = run.poll()
        if infos[0].err or infos[0].t >= args.warm_time:
            break
        run.steps(256)
    t_start = float(infos[0].t)
    developed = bufs[run.result_buffer(infos[0])].clone() if not burgers else None
    torch.cuda.synchronize()
    with Clocks(env.dev_index) as clk:
        tic = time.perf_counter()  # sustained load so the clock sampler sees the part under this kernel
        while time.perf_counter() - tic < args.sustain:
            run.steps(64)
            torch.cuda.synchronize()
        l0 = run.ctx.launches()
        step_ms, t_ms = _timed(env, lambda: run.steps(1), args.steps, flush)
        launches = run.ctx.launches() - l0
    stats = None
    if burgers:  # the on-GPU statistics of configs[4]: moments + structure functions of every sample
        from paper_1912_07645_b200.solver import make_layout
        from paper_1912_07645_b200.uq import FieldMoments, StructureFunctionAccumulator, _descriptor

        mom, sf = FieldMoments(grid, 1), StructureFunctionAccumulator(2.0, 8)
        sch, lay = _descriptor(grid, 1), make_layout(grid, 1)
        buf = bufs[run.result_buffer(infos[0])]
        mom.push_device(run.ctx, sch, lay, buf, 0)  # warm: accumulator / partials allocations
        sf.push_device(run.ctx, sch, lay, buf, 0)

        def push_all():
            for k in range(ninst):
                mom.push_device(run.ctx, sch, lay, buf, k)
                sf.push_device(run.ctx, sch, lay, buf, k)

        _, ms = _timed(env, push_all, 1)
        stats = {"ms_per_sample": round(ms / ninst, 4),
                 "what": "FieldMoments + StructureFunctionAccumulator(p=2, H=8) push of one final sample field"}
    infos, done = run.poll()
    run.end()
    if infos[0].err:
        raise RuntimeError(f"bench run failed: err {infos[0].err}/{infos[0].errsub}")
    ms_per_step = t_ms / args.steps
    value = env.ws * cells * 3 * args.steps / (t_ms * 1e-3) / 1e9
    bps = 8 * ncomp * (2 + 3 + 3) / 3  # stage 1: r us, w out; stages 2-3: r us, un, w out
    kern = "pair_kernel" if args.arith == "fast" else "ring_kernel"  # fvb_capi.cu stage_grid defaults
    kname = (f"{kern}<BURGERS,RUSANOV,WENO2> (batched)" if burgers else f"{kern}<EULER,HLLC,WENO2>")
    roof = _roofline(bps, cells * 3 * args.steps, t_ms * 1e-3, kname + " (3 launches/step)")
    if not burgers:
        _kh2d_profile_keys(roof)
    else:
        _traffic_key(roof, "traffic_bqmc.json")

    # e2e through the public API with host buffers, from the same developed
    # state the kernel timing starts at: run_simulation(host Field) with the
    # input in pinned memory (and, beside it, a pageable numpy Field)
    e2e = None
    if burgers:
        # e2e: the reference-facing run_mc with the caller's host numpy
        # initial data (H2D of every sample) and the statistics read back
        from paper_1912_07645_b200 import uq

        m = args.e2e_steps

        def e2e_call():
            mo, sfa = uq.run_mc(plan, grid, cfg, burgers_sines,
                                [uq.FieldMoments(grid, 1), uq.StructureFunctionAccumulator(2.0, 8)],
                                workers=args.workers, arith=args.arith, max_steps=m)
            return float(mo.acc.mean.sum() + mo.acc.m2.sum() + np.sum(sfa.sums))  # D2H of the statistics

        e2e_call()
        env.barrier()
        tic = time.perf_counter()
        for _ in range(args.e2e_reps):
            e2e_call()
        torch.cuda.synchronize()
        el = env.max_over_ranks(time.perf_counter() - tic)
        e2e = {"value": round(env.ws * cells * 3 * m * args.e2e_reps / el / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(ninst * init.data.nbytes), "d2h_bytes_per_step": int(2 * n * n * 8 + 9 * 8),
               "step": f"one run_mc call ({ninst} QMC samples, host numpy initial data, max_steps={m}) with "
                       "moments + structure functions read back",
               "calls": args.e2e_reps}
    if not burgers:
        from paper_1912_07645_b200.solver import pinned_field

        m = args.e2e_steps
        cfg_e = P.SchemeConfig(cfg.model, cfg.flux, cfg.recon, 3, 0.475, 2.0)
        state = P.Field(grid, 4, DeviceField(grid, 4, developed.reshape((4,) + tuple(developed.shape[-2:])))
                        .to_host().data)
        pinned = pinned_field(state)
        warm = [P.run_simulation(pinned, cfg_e, max_steps=2, arith=args.arith)[0] for _ in range(2)]
        del warm

        def e2e_rate(field, reps):
            env.barrier()
            tic = time.perf_counter()
            for _ in range(reps):
                out, recs = P.run_simulation(field, cfg_e, max_steps=m, arith=args.arith)
            torch.cuda.synchronize()
            el = env.max_over_ranks(time.perf_counter() - tic)
            return env.ws * cells * 3 * m * reps / el / 1e9

        e2e_rate(pinned, 1)  # warm both paths (staging buffers, host allocator) before timing
        e2e_rate(state, 1)
        e2e = {"value": round(e2e_rate(pinned, args.e2e_reps), 4), "unit": UNIT,
               "h2d_bytes_per_step": int(init.data.nbytes), "d2h_bytes_per_step": int(init.data.nbytes),
               "step": f"one run_simulation(host Field, max_steps={m}) call from the developed state "
                       f"(t = {t_start:.3f}), input in pinned memory",
               "calls": args.e2e_reps,
               "pageable_value": round(e2e_rate(state, args.e2e_reps), 4)}
    return {"value": value, "ms_per_step": ms_per_step, "roofline": roof, "e2e": e2e, "launches": launches,
            "clocks": clk.summary(), "t_start": t_start, "stats": stats,
            "state": f"timed from simulated t = {t_start:.3f}" + ("" if burgers else " (KH roll-up developed)"),
            "parallelism": f"replicas x{env.ws}" if env.ws > 1 else "single GPU",
            "scaling": "weak"}


# ---------------------------------------------------------------------------
# mc (C3): sharded run_mc over the ranks
# ---------------------------------------------------------------------------

def bench_mc(args, env):
    import torch

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initdev import DeviceInit
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    n = args.cells
    grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
    M = args.mc_samples
    S = args.mc_steps
    plan = uq.SamplePlan("mc", M, 42, 4)
    init = DeviceInit(KH_EXPRS + ["0.0", "2.5"], cfg.model, primitive=True)
    group = env.dist.group.WORLD if env.dist is not None else None
    result = {}

    def one():
        m, = uq.run_mc(plan, grid, cfg, init, [uq.FieldMoments(grid, 4)], arith=args.arith, max_steps=S,
                       group=group)
        result["m"] = m

    from paper_1912_07645_b200 import _native as N

    one()  # compile the initial-data program, allocate batch buffers
    with Clocks(env.dev_index) as clk:
        for _ in range(max(0, args.warmup - 1)):
            one()
        l0 = N.context().launches()
        step_ms, t_ms = _timed(env, one, args.steps)
        launches = N.context().launches() - l0
    cell_stages = M * S * 3 * n * n  # all ranks together, per run_mc call
    ms_per_step = t_ms / args.steps
    value = cell_stages * args.steps / (t_ms * 1e-3) / 1e9
    assert result["m"].acc.count == M
    bps = 85.33 + 160.0 / (3 * S)  # + the per-sample moments update (read field, rmw mean and M2)
    roof = _roofline(bps, cell_stages * args.steps, t_ms * 1e-3,
                     ("pair_kernel" if args.arith == "fast" else "ring_kernel")
                     + "<EULER,HLLC,WENO2> (batched) + moments_push_kernel")

    # e2e: the same sharded run_mc with the caller's host evaluate_init (the
    # reference-style numpy initial data, H2D of every sample) and the
    # statistics read back to the host
    lo, hi = uq.shard_range(M, env.ws, env.rank)

    def e2e_call():
        m, = uq.run_mc(plan, grid, cfg, kelvin_helmholtz, [uq.FieldMoments(grid, 4)], workers=args.workers,
                       arith=args.arith, max_steps=S, group=group)
        return m.acc.mean.sum() + m.acc.m2.sum()  # D2H of the statistics

    e2e_call()
    env.barrier()
    tic = time.perf_counter()
    e2e_call()
    torch.cuda.synchronize()
    el = env.max_over_ranks(time.perf_counter() - tic)
    field_bytes = 4 * (n + 4) * (n + 4) * 8
    e2e = {"value": round(cell_stages / el / 1e9, 4), "unit": UNIT,
           "h2d_bytes_per_step": int((hi - lo) * field_bytes), "d2h_bytes_per_step": int(2 * 4 * n * n * 8),
           "step": f"one run_mc call with host numpy initial data (rank {env.rank}: samples {lo}..{hi - 1})"}
    return {"value": value, "ms_per_step": ms_per_step, "roofline": roof, "e2e": e2e, "launches": launches,
            "clocks": clk.summary(), "t_start": 0.0, "stats": None,
            "state": f"every sample from t = 0 for {S} RK3 steps (run_mc max_steps)",
            "parallelism": f"sample sharding x{env.ws} (contiguous blocks, NCCL merge)" if env.ws > 1
            else "single GPU",
            "scaling": "strong"}


# ---------------------------------------------------------------------------
# kh3d (C4): z-slab decomposition over NCCL, one subdomain per rank
# ---------------------------------------------------------------------------

def bench_kh3d(args, env):
    import torch

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200.initdev import DeviceInit
    from paper_1912_07645_b200.parallel import DecomposedRun, RankTopology
    from paper_1912_07645_b200.solver import DeviceField, pinned_field

    n, ws, rank = args.cells, env.ws, env.rank
    # global grid n x n x (n ws), unit spacing 1/n; rank r owns z in [r, r+1)
    local = P.GridSpec(3, (n, n, n), (0.0, 0.0, float(rank)), (1.0, 1.0, 1.0), ghost_width=2,
                       deltas=(1.0 / n,) * 3)
    cfg = P.SchemeConfig(P.EquationModel("euler", 3), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
    topo = RankTopology((1, 1, ws))
    init = DeviceInit(KH_EXPRS + ["0.0", "0.0", "2.5"], cfg.model, primitive=True)
    buf = torch.empty((1, 5) + tuple(local.padded[::-1]), dtype=torch.float64, device="cuda")
    err = init.evaluate_batch(local, [KH_VECTOR], buf)[0]
    if err is not None:
        raise err
    dev = DeviceField(local, 5, buf[0])
    total = args.warmup + args.steps
    run = DecomposedRun(dev, cfg, topo, n_steps=total + 1, arith=args.arith, group=None, log=False,
                        poll_every=1 << 30, peer_halos={"auto": "auto", "peer": True, "nccl": False}[args.halo])
    halo_path = ("fused peer stores (symmetric memory over NVLink) + device barrier per stage"
                 if run.symm is not None else "NCCL P2P messages, inner box overlapped")
    run.advance(args.warmup)
    with Clocks(env.dev_index) as clk:
        l0 = run.ctx.launches()
        step_ms, t_ms = _timed(env, lambda: run.advance(1), args.steps, stream=run.stream)
        launches = run.ctx.launches() - l0
    run.advance(1)
    final, _ = run.finish()
    cells = n ** 3
    field_bytes = 5 * (n + 4) ** 3 * 8
    ms_per_step = t_ms / args.steps
    value = ws * cells * 3 * args.steps / (t_ms * 1e-3) / 1e9
    roof = _roofline(8 * 5 * 8 / 3, ws * cells * 3 * args.steps, t_ms * 1e-3,
                     ("ring3i_kernel" if args.arith == "fast" else "ring3_kernel")
                     + "<EULER,HLLC,WENO2> (3+ launches/step)")
    if args.arith == "fast":
        _traffic_key(roof, "traffic_kh3d.json")
    roof["achieved"] = round(roof["achieved"] / ws, 1)  # per GPU (the peak is one GPU's)
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["per"] = "GPU"

    # e2e: this rank's subdomain from pinned host memory through DecomposedRun
    # (H2D inside), e2e_steps RK3 steps, final subdomain back to the host --
    # for subdomains up to 8 GB (a 1024^3 subdomain would need 43 GB of
    # pinned host memory per rank and a second set of device buffers)
    e2e = None
    if field_bytes <= 8 << 30:
        host = pinned_field(final.to_host())
        del final, run
        m = max(1, args.e2e_steps // 2)
        env.barrier()
        tic = time.perf_counter()
        r2 = DecomposedRun(host, cfg, topo, n_steps=m, arith=args.arith, log=False)
        r2.advance()
        out, _ = r2.finish()
        out.to_host()
        torch.cuda.synchronize()
        el = env.max_over_ranks(time.perf_counter() - tic)
        e2e = {"value": round(ws * cells * 3 * m / el / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(host.data.nbytes), "d2h_bytes_per_step": int(host.data.nbytes),
               "step": f"one DecomposedRun of {m} RK3 steps per rank from a pinned host subdomain, result to host"}
    return {"value": value, "ms_per_step": ms_per_step, "roofline": roof, "e2e": e2e, "launches": launches,
            "clocks": clk.summary(), "t_start": 0.0, "stats": None,
            "state": f"KH3D from t = 0 after {args.warmup} warm-up steps",
            "parallelism": f"z-slab decomposition x{ws}, halos: {halo_path}" if ws > 1
            else "single GPU (one-rank group: same code path)",
            "scaling": "weak"}


# ---------------------------------------------------------------------------
# CPU reference path
# ---------------------------------------------------------------------------

_SH = {}


def _ref_importable() -> bool:
    if not (REF_PATH / "conslaw").exists():
        return False
    if str(REF_PATH) not in sys.path:
        sys.path.insert(0, str(REF_PATH))
    try:
        import conslaw  # noqa: F401

        return True
    except Exception:
        return False


def _band_residual(job):
    """Residual of rows [y0, y1) of the shared padded stage array, computed
    by the reference's own spatial_residual (or the oracle port) on the
    band's padded sub-array (its ghost rows are the neighbouring rows)."""
    from multiprocessing import shared_memory

    kind, name, shape, n, y0, y1, out_name = job
    shm = _SH.get(name) or shared_memory.SharedMemory(name=name)
    _SH[name] = shm
    a = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
    oshm = _SH.get(out_name) or shared_memory.SharedMemory(name=out_name)
    _SH[out_name] = oshm
    L = np.ndarray((shape[0], n, n), dtype=np.float64, buffer=oshm.buf)
    g = 2
    band = a[:, y0:y1 + 2 * g, :]  # padded rows y0 .. y1+2g (ghost rows included)
    if kind == "reference":
        from conslaw import solver as RS
        from conslaw.grid import Field as RField, GridSpec as RGrid

        h = y1 - y0
        grid = RGrid(2, (n, h), (0.0, y0 / n), (1.0, h / n), ghost_width=g, deltas=(1.0 / n, 1.0 / n))
        L[:, y0:y1, :] = RS.spatial_residual(RField(grid, 4, band), _ref_cfg())
    else:
        from oracle import fv_oracle as O

        sc = O.Scheme(dim=2, cells=(n, y1 - y0), deltas=(1.0 / n, 1.0 / n), eq="euler", flux="hllc",
                      recon="weno2", rk=3, cfl=0.475, t_end=2.0)
        L[:, y0:y1, :] = O.residual(band, sc)
    return y1 - y0


def _ref_cfg():
    from conslaw.equations import EquationModel
    from conslaw.numerics import FluxKind, Reconstruction, ReconstructionKind
    from conslaw.solver import SchemeConfig

    return SchemeConfig(EquationModel("euler", 2), FluxKind.HLLC, Reconstruction(ReconstructionKind.WENO2),
                        rk_order=3, cfl=0.475, t_end=2.0)


def bench_cpu(n, steps, workers, warmup=1, budget_s=180.0, kind=None):
    """Returns (Gcell-stage/s, seconds per step, steps timed, kind) of the CPU
    reference on the host: ``workers`` processes evaluate the residual in row
    bands (bitwise equal to the serial residual).  kind "reference": the
    unmodified conslaw package (baseline/_ref) steps with its own
    ssp_rk_step / stable_dt and its residual seam; kind "port": the oracle.

    ``warmup`` untimed steps, then up to ``steps`` timed RK3 steps; the timed
    loop stops early once ``budget_s`` seconds are spent (a bounded sample on
    slow hosts) and the number of steps actually timed is returned."""
    import multiprocessing as mp
    from multiprocessing import shared_memory

    kind = kind or ("reference" if _ref_importable() else "port")
    g = 2
    shape = (4, n + 2 * g, n + 2 * g)
    shm_in = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * 8)
    shm_out = shared_memory.SharedMemory(create=True, size=4 * n * n * 8)
    a = np.ndarray(shape, dtype=np.float64, buffer=shm_in.buf)
    Lout = np.ndarray((4, n, n), dtype=np.float64, buffer=shm_out.buf)
    edges = np.linspace(0, n, workers + 1).astype(int)
    jobs = [(kind, shm_in.name, shape, n, int(edges[i]), int(edges[i + 1]), shm_out.name)
            for i in range(workers) if edges[i + 1] > edges[i]]
    ctx = mp.get_context("fork")
    try:
        with ctx.Pool(workers) as pool:
            if kind == "reference":
                from conslaw import solver as RS
                from conslaw.grid import Field as RField, GridSpec as RGrid

                from paper_1912_07645_b200.initial import kelvin_helmholtz as kh
                import paper_1912_07645_b200 as P

                cfg = _ref_cfg()
                grid = RGrid(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=g)
                init = kh(P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=g), KH_VECTOR)
                field = RField(grid, 4, np.array(init.data))

                def residual(stage, cfg_):  # the reference's seam (solver.py:176-193)
                    a[...] = stage.data
                    list(pool.map(_band_residual, jobs))
                    return Lout.copy()

                def step(f):
                    dt = RS.stable_dt(f, cfg, cfg.t_end)
                    return RS.ssp_rk_step(f, dt, cfg, residual=residual)
            else:
                from oracle import fv_oracle as O

                sc = O.Scheme(dim=2, cells=(n, n), deltas=(1.0 / n, 1.0 / n), eq="euler", flux="hllc",
                              recon="weno2", rk=3, cfl=0.475, t_end=2.0)
                field = O.kelvin_helmholtz((n, n), KH_VECTOR)

                def Lfun(inner):
                    a[...] = 0.0
                    O.interior(a, sc)[...] = inner
                    O.ghost_fill(a, sc)
                    list(pool.map(_band_residual, jobs))
                    return Lout.copy()

                def step(u):
                    dt = O.cfl_dt(O.speed_maxima(u, sc), sc, None)
                    return O.padded_from_interior(sc, O.rk_combine(O.interior(u, sc).copy(), dt, Lfun, 3))
            cur = field
            for _ in range(max(1, warmup)):  # warm the pool (untimed)
                cur = step(cur)
            done = 0
            tic = time.perf_counter()
            while done < steps:
                cur = step(cur)
                done += 1
                if time.perf_counter() - tic > budget_s:
                    break
            el = time.perf_counter() - tic
    finally:
        for s in (shm_in, shm_out):
            s.close()
            s.unlink()
    return n * n * 3 * done / el / 1e9, el / done, done, kind


def bench_cpu_stock(n):
    """The stock single-process path: conslaw.run_simulation(init, cfg,
    max_steps=1) (baseline/_ref), one RK3 step of KH2D n^2."""
    if not _ref_importable():
        return None
    from conslaw.grid import Field as RField, GridSpec as RGrid
    from conslaw.solver import run_simulation

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200.initial import kelvin_helmholtz as kh

    init = kh(P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2), KH_VECTOR)
    f = RField(RGrid(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2), 4, np.array(init.data))
    tic = time.perf_counter()
    run_simulation(f, _ref_cfg(), max_steps=1)
    el = time.perf_counter() - tic
    return {"value": round(n * n * 3 / el / 1e9, 7), "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"stock conslaw.run_simulation(max_steps=1), KH2D {n}^2, one process, {el:.1f} s"}


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------

def _relaunch(args_list, n):
    """--gpus N without torchrun: re-execute under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())]
    return subprocess.call(cmd + args_list)


PARITY = {  # what tests/test_gpu_benchsize.py checks for each bench configuration
    "kh2d": "exact: bitwise == reference; fast: relative L1 <= 1e-12 per conserved component "
            "(sum|a-b|/sum|b|) vs the oracle from this developed state after 1/3/10 steps "
            "(tests/test_gpu_benchsize.py)",
    "mc": "C3 shape, 16 samples x 512^2: exact moments bitwise == the sample-order merge of the oracle's "
          "per-sample finals; fast: means <= 1e-12 per component, variances <= 1e-10 relative L1 "
          "(tests/test_gpu_benchsize.py)",
    "kh3d": "KH3D 128^3: exact bitwise == oracle (1 RK3 step from t = 0 and from a developed state with flow "
            "along all three axes); fast relative L1 <= 1e-12 per conserved component from that state after 1 "
            "and 3 steps (tests/test_gpu_benchsize.py)",
    "bqmc": "C5 shape, 4 Burgers QMC samples x 2048^2: exact moments bitwise == oracle, structure functions "
            "within 1e-13; fast: mean and structure functions <= 1e-12, variance <= 1e-10 relative L1 "
            "(tests/test_gpu_benchsize.py)",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arith", default=os.environ.get("FVB_BENCH_ARITH", "fast"), choices=["fast", "exact"])
    ap.add_argument("--cells", type=int, default=None, help="cells per axis (1024 kh2d, 512 mc/kh3d, 2048 bqmc)")
    ap.add_argument("--config", default="kh2d", choices=["kh2d", "mc", "kh3d", "bqmc"],
                    help="kh2d: BASELINE configs[1] (headline); mc: sharded run_mc (configs[2]); kh3d: z-slab "
                         "decomposition over NCCL (configs[3]); bqmc: batched Burgers QMC (configs[4] shape)")
    ap.add_argument("--samples", type=int, default=4, help="bqmc: samples per GPU batch")
    ap.add_argument("--mc-samples", type=int, default=1024, help="mc: total samples (sharded over the ranks)")
    ap.add_argument("--mc-steps", type=int, default=20, help="mc: RK3 steps per sample (run_mc max_steps)")
    ap.add_argument("--workers", type=int, default=max(1, min(16, os.cpu_count() or 1)),
                    help="mc e2e: host threads evaluating the numpy initial data")
    ap.add_argument("--halo", default="auto", choices=["auto", "peer", "nccl"],
                    help="kh3d: fused peer-memory halo stores (auto when symmetric memory works) or NCCL messages")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sustain", type=float, default=1.5, help="seconds of untimed load for the clock sampler")
    ap.add_argument("--warm-time", type=float, default=1.0, help="simulated time reached before timing")
    ap.add_argument("--state-file", default=None, help="start from a saved developed state (profiling)")
    args = ap.parse_args()
    ws, rank, local = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(sys.argv[1:], args.gpus))
    if args.steps is None:
        args.steps = {"mc": 5, "kh3d": 10}.get(args.config, 50)
    if args.warmup is None:
        args.warmup = 3 if args.config in ("mc", "kh3d") else 5
    if args.cells is None:
        args.cells = {"kh2d": N_CELLS, "mc": 512, "kh3d": 512, "bqmc": 2048}[args.config]
    if args.config == "bqmc" and args.warm_time == 1.0:
        args.warm_time = 0.01  # the authored config runs to t = 0.02
    workload = {
        "kh2d": f"KH2D {args.cells}x{args.cells} Euler, WENO2 + HLLC, SSP-RK3, periodic, fp64 "
                "(BASELINE configs[1]); step = one RK3 time step (3 stages)",
        "mc": f"KH2D MC ensemble (BASELINE configs[2]): {args.mc_samples} samples x {args.cells}^2, WENO2 + HLLC, "
              f"SSP-RK3, fp64, {args.mc_steps} RK3 steps per sample, on-GPU mean/variance; step = one sharded "
              "run_mc call over the whole ensemble",
        "kh3d": f"KH3D Euler, WENO2 + HLLC, SSP-RK3, fp64, {args.cells}^3 per GPU, z-slab domain decomposition "
                "(BASELINE configs[3]); step = one RK3 time step of the whole domain",
        "bqmc": f"Burgers 2D QMC ensemble, {args.samples} samples/GPU x {args.cells}^2, WENO2 + Rusanov, SSP-RK3, "
                "fp64, batched (configs[4] shape); step = one RK3 step of every sample",
    }[args.config]
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        workers = max(1, cores)
        # W untimed full RK3 steps, then K timed ones (cut short after 180 s on
        # a slow host; "steps" says how many), on the kh2d workload
        n = args.cells if args.config == "kh2d" else N_CELLS
        val, sps, done, kind = bench_cpu(n, max(1, args.steps), workers, warmup=max(1, args.warmup))
        stock = bench_cpu_stock(n)
        what = ("the unmodified conslaw package (baseline/_ref): its ssp_rk_step / stable_dt, the residual seam "
                "fed by its spatial_residual in row bands" if kind == "reference" else
                "the numpy oracle port (baseline/_ref absent), residual in row bands")
        line = {
            "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": UNIT, "n_gpus": ws,
            "steps": done, "warmup": max(1, args.warmup), "ms_per_step": round(sps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (KH2D preset, MC seed 42 sample 0)",
            "config": {"workload": workload if args.config == "kh2d" else workload + " [reference arm: kh2d]",
                       "arith": "numpy (reference op order)",
                       "state": "from t = 0 (numpy evaluates every branch of every cell: its cost does not depend "
                                "on the state)"},
            "cpu_baseline": {"value": round(val, 6), "unit": UNIT, "cores": workers, "kind": kind,
                             "sample": f"{done} timed RK3 step(s) of KH2D {n}^2: {what}, {workers} processes"},
            "e2e": {"value": round(val, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        if stock:
            line["single_process"] = stock
        print(json.dumps(line))
        return

    import torch  # noqa: F401

    env = Env(ws, rank, local, need_group=args.config == "kh3d")
    try:
        fn = {"kh2d": bench_single, "bqmc": bench_single, "mc": bench_mc, "kh3d": bench_kh3d}[args.config]
        res = fn(args, env)
    finally:
        env.close()
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu and args.config == "kh2d":
        # bounded CPU sample beside the GPU number: one RK3 step of the same
        # workload through the reference in ONE process (numpy is single threaded)
        val, sps, _, kind = bench_cpu(args.cells, max(1, args.cpu_steps), 1)
        cpu = {"value": round(val, 6), "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"1 RK3 step of KH2D {args.cells}^2 through "
                         + ("the unmodified conslaw package (baseline/_ref)" if kind == "reference"
                            else "the numpy oracle port") + f", 1 process, {sps:.1f} s"}
    line = {
        "metric": METRIC, "value": round(res["value"], 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 4),
        "higher_is_better": True, "scaling": res["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": {"kh2d": "synthetic (KH2D preset initial data, MC seed 42 sample 0)",
                 "mc": "synthetic (KH2D preset initial data evaluated on the GPU, MC seed 42 samples 0..M-1)",
                 "kh3d": "synthetic (KH3D preset initial data evaluated on the GPU, MC seed 42 sample 0)",
                 "bqmc": "synthetic (Burgers QMC initial data, Halton samples 0..n-1)"}[args.config],
        "config": {"workload": workload, "arith": args.arith,
                   "parity": PARITY[args.config],
                   "l2": ("flushed (256 MiB write) before every timed step" if args.config in ("kh2d", "bqmc")
                          else "inputs larger than L2 (" + ("1024 x 8.5 MB sample fields" if args.config == "mc"
                                                            else "5.5 GB subdomain per GPU") + ")"),
                   "state": res["state"], "parallelism": res["parallelism"]},
        **({"uq_stats": res["stats"]} if res.get("stats") else {}),
        "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
        "clocks": res["clocks"],
    }
    if res.get("launches") is not None:
        line["gpu_launches"] = int(res["launches"])
    print(json.dumps(line))


if __name__ == "__main__":
    main()
