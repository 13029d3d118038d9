"""Benchmark: Gcell-updates/s per SSP-RK stage (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): 2D Kelvin-Helmholtz Euler,
WENO2 + HLLC, SSP-RK3, 1024x1024 periodic, fp64 -- the KH2D preset
(presets.py:65-104) with reconstruction=weno2 and the MC seed-42 sample-0
random vector; synthetic data, no checkpoint.  One bench "step" is one full
SSP-RK3 time step (3 fused stage launches, CFL reduction fused into the last
stage, dt computed on the device).  L2 is flushed (256 MiB write) before
every timed step; each step is timed with CUDA events on the launching
stream and the sum is the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--arith fast|exact]

N > 1 (torchrun, one process per GPU): C2 is a single-domain config, so the
ranks run independent replicas (weak scaling, no data-path collective); the
step time is the max over ranks and ``value`` counts all ranks' cells.

``--impl reference`` times the CPU reference path -- the numpy oracle
restatement (oracle/fv_oracle.py, bitwise equal to the reference package) --
on the host cores, row-band decomposed over a process pool, on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
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
# our arm
# ---------------------------------------------------------------------------

def bench_ours(args, ws, rank, local):
    import torch

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import _native as N
    from paper_1912_07645_b200.initial import kelvin_helmholtz
    from paper_1912_07645_b200.solver import DeviceField, DeviceRun

    ndev = torch.cuda.device_count()
    dev_index = local % max(1, ndev)
    torch.cuda.set_device(dev_index)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        # one rank per GPU over NCCL; more ranks than GPUs (a smoke run on a
        # small box) falls back to gloo for the barrier/timing reduce only --
        # the replicas never exchange data
        if ws <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    n = args.cells
    dim = 3 if args.config == "kh3d" else 2
    grid = P.GridSpec(dim, (n,) * dim, (0.0,) * dim, (1.0,) * dim, ghost_width=2)
    burgers = args.config == "bqmc"
    if burgers:  # configs[4]: the Burgers QMC preset scheme (Rusanov, WENO2, RK3, CFL 0.475)
        cfg = P.SchemeConfig(P.EquationModel("burgers", dim), P.FluxKind.RUSANOV,
                             P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
    else:
        cfg = P.SchemeConfig(P.EquationModel("euler", dim), P.FluxKind.HLLC,
                             P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
    ninst = args.samples if args.config in ("mc", "bqmc") else 1
    if burgers:
        from paper_1912_07645_b200.initial import burgers_sines
        from paper_1912_07645_b200.uq import SamplePlan, draw_sample

        plan = SamplePlan("qmc", ninst, 42, 2)
        inits = [burgers_sines(grid, draw_sample(plan, k)) for k in range(ninst)]
        init = inits[0]
        b0 = torch.from_numpy(np.stack([f.data for f in inits])).to("cuda")
    elif args.config == "mc":
        from paper_1912_07645_b200.uq import SamplePlan, draw_sample

        plan = SamplePlan("mc", ninst, 42, 4)
        inits = [kelvin_helmholtz(grid, draw_sample(plan, k)) for k in range(ninst)]
        init = inits[0]
        b0 = torch.from_numpy(np.stack([f.data for f in inits])).to("cuda")
    else:
        init = kelvin_helmholtz(grid, KH_VECTOR)
        if args.state_file and Path(args.state_file).exists():
            init = P.Field(grid, dim + 2, np.load(args.state_file))  # developed state saved by tools/make_state.py
            args.warm_time = 0.0
        b0 = DeviceField.from_host(init).data
    bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
    total_steps = args.warmup + args.steps
    run = DeviceRun(grid, cfg, bufs, ninst, N.MODE_FIXED, 1 << 40, args.arith, log=False)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    cells = n ** dim * ninst
    ncomp = 1 if burgers else dim + 2

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
    torch.cuda.synchronize()
    evs = []
    with Clocks(dev_index) as clk:
        # sustained load so the clock sampler sees the part under this kernel
        tic = time.perf_counter()
        while time.perf_counter() - tic < args.sustain:
            run.steps(64)
            torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = run.ctx.launches()
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run.steps(1)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
    launches = run.ctx.launches() - l0 - 0
    stats = None
    if burgers:  # the on-GPU statistics of configs[4]: moments + structure functions of every sample
        from paper_1912_07645_b200.solver import make_layout
        from paper_1912_07645_b200.uq import FieldMoments, StructureFunctionAccumulator, _descriptor

        mom, sf = FieldMoments(grid, 1), StructureFunctionAccumulator(2.0, 8)
        sch, lay = _descriptor(grid, 1), make_layout(grid, 1)
        buf = bufs[run.result_buffer(infos[0])]
        mom.push_device(run.ctx, sch, lay, buf, 0)  # warm: accumulator / partials allocations
        sf.push_device(run.ctx, sch, lay, buf, 0)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(ninst):
            mom.push_device(run.ctx, sch, lay, buf, k)
            sf.push_device(run.ctx, sch, lay, buf, k)
        b.record(stream)
        torch.cuda.synchronize()
        stats = {"ms_per_sample": round(a.elapsed_time(b) / ninst, 4),
                 "what": "FieldMoments + StructureFunctionAccumulator(p=2, H=8) push of one final sample field"}
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = float(sum(step_ms))
    infos, done = run.poll()
    run.end()
    if infos[0].err:
        raise RuntimeError(f"bench run failed: err {infos[0].err}/{infos[0].errsub}")
    if dist:
        on_gpu = dist.get_backend() == "nccl"
        tt = torch.tensor([t_ms], device="cuda" if on_gpu else "cpu", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = ws * cells * 3 * args.steps / (t_ms * 1e-3) / 1e9

    # roofline: the 3 fused stage launches of a step (the only kernels in it)
    bytes_step = cells * 8 * ncomp * (2 + 3 + 3)  # stage1: r us, w out; stages 2-3: r us, un, w out
    kname = {"kh2d": "ring_kernel<EULER,HLLC,WENO2>", "mc": "ring_kernel<EULER,HLLC,WENO2> (batched)",
             "kh3d": "ring3_kernel<EULER,HLLC,WENO2>",
             "bqmc": "ring_kernel<BURGERS,RUSANOV,WENO2> (batched)"}[args.config]
    peak, peak_src = _hbm_peak()
    achieved = bytes_step / (ms_per_step * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                "kernel": kname + " (3 launches/step)",
                "algorithmic_bytes_per_cell_stage": round(bytes_step / cells / 3, 2)}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists() and args.config == "kh2d":
        try:
            roofline["traffic"] = json.loads(prof.read_text()).get("stage_bytes_per_launch")
        except Exception:
            pass
    fp64 = ROOT / "profiles" / "fp64_roof.json"
    if fp64.exists() and args.config == "kh2d":
        # the roof that binds in practice: FP64 throughput (from the committed
        # ncu capture and the measured DFMA peak, not from this run)
        try:
            f = json.loads(fp64.read_text())
            st = f["ring_kernel_stages"]
            ach = sum(x["fp64_tflops"] * x["us"] for x in st) / sum(x["us"] for x in st)
            pk = f["measured_peak"]["dfma_peak_tflops"]
            roofline["compute"] = {"bound": "fp64", "achieved": round(ach, 2), "peak": pk, "unit": "TFLOP/s",
                                   "frac": round(ach / pk, 4),
                                   "fp64_pipe_pct": round(sum(x["fp64_pipe_pct"] for x in st) / len(st), 1),
                                   "source": "profiles/fp64_roof.json (ncu, tools/fp64_peak.cu)"}
        except Exception:
            pass

    # e2e through the public API with host buffers: run_simulation(host Field)
    e2e = None
    if (rank == 0 or ws > 1) and args.config == "kh2d":
        m = args.e2e_steps
        cfg_e = P.SchemeConfig(cfg.model, cfg.flux, cfg.recon, 3, 0.475, 2.0)
        from paper_1912_07645_b200.solver import pinned_field

        pinned = pinned_field(init)  # host input in pinned memory (contract: H2D from pinned)
        # warm: kernels, graphs, and two result buffers in the pinned host cache
        # (a loop holds the previous result while the next call returns)
        warm = [P.run_simulation(pinned, cfg_e, max_steps=2, arith=args.arith)[0] for _ in range(2)]
        del warm
        torch.cuda.synchronize()
        tic = time.perf_counter()
        reps = args.e2e_reps
        for _ in range(reps):
            out, recs = P.run_simulation(pinned, cfg_e, max_steps=m, arith=args.arith)
        torch.cuda.synchronize()
        el = time.perf_counter() - tic
        e2e = {"value": round(cells * 3 * m * reps / el / 1e9 * ws, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(init.data.nbytes), "d2h_bytes_per_step": int(init.data.nbytes),
               "step": f"one run_simulation(host Field, max_steps={m}) call", "calls": reps}

    if dist:
        dist.barrier()
    return {
        "value": value, "ms_per_step": ms_per_step, "roofline": roofline, "e2e": e2e,
        "launches": launches, "clocks": clk.summary(), "step_ms": step_ms, "t_start": t_start, "stats": stats,
    }


# ---------------------------------------------------------------------------
# CPU reference path: the oracle, row-band decomposed over host processes
# ---------------------------------------------------------------------------

_SH = {}


def _band_residual(job):
    """Residual of rows [y0, y1) of the shared padded stage array."""
    from multiprocessing import shared_memory

    from oracle import fv_oracle as O

    name, shape, n, y0, y1, out_name = job
    shm = _SH.get(name) or shared_memory.SharedMemory(name=name)
    _SH[name] = shm
    a = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
    oshm = _SH.get(out_name) or shared_memory.SharedMemory(name=out_name)
    _SH[out_name] = oshm
    L = np.ndarray((shape[0], n, n), dtype=np.float64, buffer=oshm.buf)
    g = 2
    band = a[:, y0:y1 + 2 * g, :]  # padded rows y0 .. y1+2g (ghost rows included)
    sc = O.Scheme(dim=2, cells=(n, y1 - y0), deltas=(1.0 / n, 1.0 / n), eq="euler", flux="hllc",
                  recon="weno2", rk=3, cfl=0.475, t_end=2.0)
    L[:, y0:y1, :] = O.residual(band, sc)
    return y1 - y0


def cpu_reference_step(pool, u_pad, n, workers, shm_in, shm_out):
    """One SSP-RK3 step of the oracle (solver.py:164-173) with the residual
    evaluated in row bands by `workers` processes (bitwise equal to serial)."""
    from oracle import fv_oracle as O

    sc = O.Scheme(dim=2, cells=(n, n), deltas=(1.0 / n, 1.0 / n), eq="euler", flux="hllc", recon="weno2",
                  rk=3, cfl=0.475, t_end=2.0)
    a = np.ndarray(u_pad.shape, dtype=np.float64, buffer=shm_in.buf)
    L = np.ndarray((4, n, n), dtype=np.float64, buffer=shm_out.buf)
    edges = np.linspace(0, n, workers + 1).astype(int)
    jobs = [(shm_in.name, u_pad.shape, n, int(edges[i]), int(edges[i + 1]), shm_out.name)
            for i in range(workers) if edges[i + 1] > edges[i]]

    def Lfun(inner):
        a[...] = 0.0
        O.interior(a, sc)[...] = inner
        O.ghost_fill(a, sc)
        list(pool.map(_band_residual, jobs))
        return L.copy()

    dt = O.cfl_dt(O.speed_maxima(u_pad, sc), sc, None)
    return O.padded_from_interior(sc, O.rk_combine(O.interior(u_pad, sc).copy(), dt, Lfun, 3))


def bench_cpu(n, steps, workers, warmup=1, budget_s=180.0):
    """Returns (Gcell-stage/s, seconds per step, steps timed) of the oracle on the host.

    ``warmup`` untimed steps, then up to ``steps`` timed RK3 steps; the timed
    loop stops early once ``budget_s`` seconds are spent (a bounded sample
    on slow hosts), and the number of steps actually timed is returned."""
    import multiprocessing as mp
    from multiprocessing import shared_memory

    from oracle import fv_oracle as O

    u = O.kelvin_helmholtz((n, n), KH_VECTOR)
    shm_in = shared_memory.SharedMemory(create=True, size=u.nbytes)
    shm_out = shared_memory.SharedMemory(create=True, size=4 * n * n * 8)
    ctx = mp.get_context("fork")
    try:
        with ctx.Pool(workers) as pool:
            cur = u
            for _ in range(max(1, warmup)):  # warm the pool (untimed)
                cur = cpu_reference_step(pool, cur, n, workers, shm_in, shm_out)
            done = 0
            tic = time.perf_counter()
            while done < steps:
                cur = cpu_reference_step(pool, cur, n, workers, shm_in, shm_out)
                done += 1
                if time.perf_counter() - tic > budget_s:
                    break
            el = time.perf_counter() - tic
    finally:
        shm_in.close()
        shm_in.unlink()
        shm_out.close()
        shm_out.unlink()
    return n * n * 3 * done / el / 1e9, el / done, done


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arith", default=os.environ.get("FVB_BENCH_ARITH", "fast"), choices=["fast", "exact"])
    ap.add_argument("--cells", type=int, default=None, help="cells per axis (default 1024 kh2d, 512 mc, 256 kh3d)")
    ap.add_argument("--config", default="kh2d", choices=["kh2d", "mc", "kh3d", "bqmc"],
                    help="kh2d: BASELINE configs[1] (headline); mc: batched KH2D ensemble (configs[2] "
                         "shape); kh3d: KH3D single domain (configs[3] shape); bqmc: batched Burgers QMC "
                         "ensemble + structure functions (configs[4] shape)")
    ap.add_argument("--samples", type=int, default=None, help="mc / bqmc: samples per GPU batch (16 / 4)")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sustain", type=float, default=1.5, help="seconds of untimed load for the clock sampler")
    ap.add_argument("--warm-time", type=float, default=1.0, help="simulated time reached before timing")
    ap.add_argument("--state-file", default=None, help="start from a saved developed state (profiling)")
    args = ap.parse_args()
    if args.cells is None:
        args.cells = {"kh2d": N_CELLS, "mc": 512, "kh3d": 256, "bqmc": 2048}[args.config]
    if args.samples is None:
        args.samples = 4 if args.config == "bqmc" else 16
    if args.config == "bqmc" and args.warm_time == 1.0:
        args.warm_time = 0.01  # the preset runs to t = 0.02
    ws, rank, local = _dist()
    workload = {
        "kh2d": f"KH2D {args.cells}x{args.cells} Euler, WENO2 + HLLC, SSP-RK3, periodic, fp64 "
                "(BASELINE configs[1]); step = one RK3 time step (3 stages)",
        "mc": f"KH2D MC ensemble, {args.samples} samples/GPU x {args.cells}^2, WENO2 + HLLC, SSP-RK3, fp64, "
              "batched (one instance per sample; configs[2] shape); step = one RK3 step of every sample",
        "kh3d": f"KH3D {args.cells}^3 Euler, WENO2 + HLLC, SSP-RK3, periodic, fp64 (configs[3] shape, "
                "single domain); step = one RK3 time step",
        "bqmc": f"Burgers 2D QMC ensemble, {args.samples} samples/GPU x {args.cells}^2, WENO2 + Rusanov, SSP-RK3, "
                "fp64, batched (configs[4] shape); step = one RK3 step of every sample",
    }[args.config]
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        workers = max(1, cores)
        # the driver's --steps K --warmup W: W untimed full RK3 steps, then K
        # timed ones (cut short after 180 s on a slow host; "steps" says how many)
        val, sps, done = bench_cpu(args.cells, max(1, args.steps), workers, warmup=max(1, args.warmup))
        line = {
            "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": UNIT, "n_gpus": ws,
            "steps": done, "warmup": max(1, args.warmup), "ms_per_step": round(sps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (KH2D preset, MC seed 42 sample 0)",
            "config": {"workload": workload, "arith": "numpy (reference op order)"},
            "cpu_baseline": {"value": round(val, 6), "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": f"{done} timed RK3 step(s) of KH2D {args.cells}^2 through the "
                                       f"numpy oracle, residual row-band split over {workers} processes"},
            "e2e": {"value": round(val, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    res = bench_ours(args, ws, rank, local)
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu and args.config == "kh2d":
        # bounded CPU sample: 1 RK3 step of the same workload, single process
        # (numpy is single threaded), the oracle = reference op order
        val, sps, _ = bench_cpu(args.cells, max(1, args.cpu_steps), 1)
        cpu = {"value": round(val, 6), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"1 RK3 step of KH2D {args.cells}^2 through the numpy oracle (oracle/fv_oracle.py), "
                         f"1 process, {sps:.1f} s"}
    line = {
        "metric": METRIC, "value": round(res["value"], 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": {"kh2d": "synthetic (KH2D preset initial data, MC seed 42 sample 0)",
                 "mc": "synthetic (KH2D preset initial data, MC seed 42 samples 0..n-1)",
                 "kh3d": "synthetic (KH3D initial data, MC seed 42 sample 0)",
                 "bqmc": "synthetic (Burgers QMC preset initial data, Halton samples 0..n-1)"}[args.config],
        "config": {"workload": workload, "arith": args.arith,
                   "parity": "exact: bitwise == reference; fast: rel L1 <= 1e-12 (tests/test_gpu_parity.py)",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "state": (f"timed from the saved state {args.state_file} (+ t = {res['t_start']:.3f})"
                             if args.state_file else
                             f"timed from simulated t = {res['t_start']:.3f}"
                             + ("" if args.config == "bqmc" else " (KH roll-up developed)")),
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        **({"uq_stats": res["stats"]} if res.get("stats") else {}),
        "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
        "clocks": res["clocks"], "gpu_launches": int(res["launches"]),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
