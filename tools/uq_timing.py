"""Wall-clock breakdown of run_mc (the public UQ API) on one GPU: host-side
initial-data evaluation vs the batched device runs + statistics.

    python tools/uq_timing.py [--cells 512] [--samples 64] [--t-end 0.05]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_07645_b200 as P  # noqa: E402
from paper_1912_07645_b200 import uq  # noqa: E402
from paper_1912_07645_b200.initial import kelvin_helmholtz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=512)
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--t-end", type=float, default=0.05)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--cached-init", action="store_true", help="evaluate_init returns one precomputed field")
    ap.add_argument("--device-init", action="store_true", help="initial data evaluated on the GPU (DeviceInit)")
    a = ap.parse_args()
    n = a.cells
    grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=a.t_end)
    plan = uq.SamplePlan("mc", a.samples, 42, 4)
    t_init = [0.0]

    cached = kelvin_helmholtz(grid, (0.1, 0.2, 0.3, 0.4)) if a.cached_init else None

    def init(g, vec):
        t0 = time.perf_counter()
        f = cached if cached is not None else kelvin_helmholtz(g, vec)
        t_init[0] += time.perf_counter() - t0
        return f

    if a.device_init:  # the KH2D preset program, evaluated by fvb_init_eval
        kh = ["y < 0.25 + 0.01 * sin(2.0 * pi * (x + X0)) ? 1.0 : y < 0.75 + 0.01 * sin(2.0 * pi * (x + X1)) ? 2.0 : 1.0",
              "y < 0.25 + 0.01 * sin(2.0 * pi * (x + X2)) ? -0.5 : y < 0.75 + 0.01 * sin(2.0 * pi * (x + X3)) ? 0.5 : -0.5",
              "0.0", "2.5"]
        init = P.DeviceInit(kh, cfg.model, primitive=True)
    # warm (kernels, allocator)
    uq.run_mc(uq.SamplePlan("mc", 2, 42, 4), grid, cfg, init, [uq.FieldMoments(grid, 4)], arith="fast")
    t_init[0] = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = uq.run_mc(plan, grid, cfg, init, [uq.FieldMoments(grid, 4), uq.StructureFunctionAccumulator(2.0, 8)],
                    workers=a.workers, arith="fast", batch=a.batch)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"run_mc {a.samples} x {n}^2 to t={a.t_end}, workers={a.workers}: wall {wall:.3f} s, host init {t_init[0]:.3f} s "
          f"({100 * t_init[0] / wall:.0f} %), {a.samples / wall:.1f} samples/s; "
          f"mean[0] sum {float(np.asarray(res[0].acc.mean).sum()):.6e}")


if __name__ == "__main__":
    main()
