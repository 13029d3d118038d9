"""Per-block timeline of the 2D pair kernel (diagnostic; needs the variant
library built with -DFVB_BLOCK_TIMES=1: python tools/variant.py bt --dims 2
-DFVB_BLOCK_TIMES=1, run with FVB_LIB=build/bt/libfvb200.so).

Advances KH2D 1024^2 (fast) to t ~ 1, runs a few RK3 steps, then reads the
[start, end] globaltimer stamps and SM of every block of the last launch of
each stage and summarises: kernel span, block durations, start skew,
resident blocks over time (how much of the span runs below full
occupancy -- the one-wave tail)."""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1912_07645_b200 as P  # noqa: E402
from paper_1912_07645_b200 import _native as N  # noqa: E402
from paper_1912_07645_b200.initial import kelvin_helmholtz  # noqa: E402
from paper_1912_07645_b200.solver import DeviceRun  # noqa: E402

VEC = [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203]


def main(out_path):
    grid = P.GridSpec(2, (1024, 1024), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
    b0 = torch.from_numpy(kelvin_helmholtz(grid, VEC).data).to("cuda")
    bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
    run = DeviceRun(grid, cfg, bufs, 1, N.MODE_FIXED, 1 << 40, "fast", log=False)
    while True:
        infos, _ = run.poll()
        if infos[0].t >= 1.0:
            break
        run.steps(256)
    run.steps(8)
    run.poll()
    torch.cuda.synchronize()
    lib = N.context().lib
    buf = (ctypes.c_ulonglong * (3 * 8192 * 3))()
    assert lib.fvb_debug_block_times(buf) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(3, 8192, 3).astype(np.int64)
    run.end()
    np.save(str(Path(out_path).with_suffix(".npy")), a)  # raw [stage][block][t0, t1, sm]
    res = {}
    for k in range(3):
        rows = a[k]
        rows = rows[rows[:, 1] > 0]
        t0, t1, sm = rows[:, 0], rows[:, 1], rows[:, 2]
        span = t1.max() - t0.min()
        dur = t1 - t0
        # resident blocks over time (1 ns resolution on a 1000-point grid)
        grid_t = np.linspace(t0.min(), t1.max(), 1000)
        resident = np.array([np.count_nonzero((t0 <= g) & (t1 > g)) for g in grid_t])
        per_sm_end = np.array([t1[sm == s].max() for s in np.unique(sm)])
        per_sm_n = np.array([np.count_nonzero(sm == s) for s in np.unique(sm)])
        res[f"stage{k + 1}"] = {
            "blocks": int(len(rows)), "span_us": round(span / 1e3, 2),
            "block_us": {q: round(float(np.percentile(dur, p)) / 1e3, 2) for q, p in
                         (("min", 0), ("p10", 10), ("p50", 50), ("p90", 90), ("max", 100))},
            "start_skew_us": round(float(t0.max() - t0.min()) / 1e3, 2),
            "mean_resident_blocks": round(float(resident.mean()), 1),
            "max_resident_blocks": int(resident.max()),
            "frac_span_above_95pct_of_max": round(float(np.mean(resident >= 0.95 * resident.max())), 3),
            "sm_end_spread_us": round(float(per_sm_end.max() - per_sm_end.min()) / 1e3, 2),
            "blocks_per_sm": {"min": int(per_sm_n.min()), "max": int(per_sm_n.max())},
            "mean_block_over_span": round(float(dur.mean() / span), 3),
        }
    Path(out_path).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "block_times.json")
