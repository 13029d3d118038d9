"""Small workloads for per-kernel ncu captures (profiles/r02_*): each mode
runs the kernel of interest a few times after a warm-up.

  python tools/profile_kernels.py bqmc     # scalar ring kernel (Burgers, 2 instances/block) + moments + structure fn
  python tools/profile_kernels.py mc       # init_eval_kernel (device initial data) + batched Euler ring kernel
  python tools/profile_kernels.py halo     # halo_instances_kernel (one-device run_parallel, 2x2 subdomains)
  python tools/profile_kernels.py kh3d     # ring3_kernel at 512^3
  python tools/profile_kernels.py kh2d     # the headline ring kernel from the developed state
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_07645_b200 as P  # noqa: E402
from paper_1912_07645_b200 import _native as N  # noqa: E402
from paper_1912_07645_b200 import uq  # noqa: E402
from paper_1912_07645_b200.initdev import DeviceInit  # noqa: E402
from paper_1912_07645_b200.solver import DeviceRun, make_layout  # noqa: E402

KH = ["y < 0.25 + 0.01 * sin(2 * pi * (x + X0)) ? 1.0 : (y < 0.75 + 0.01 * sin(2 * pi * (x + X1)) ? 2.0 : 1.0)",
      "y < 0.25 + 0.01 * sin(2 * pi * (x + X2)) ? -0.5 : (y < 0.75 + 0.01 * sin(2 * pi * (x + X3)) ? 0.5 : -0.5)"]
VEC = [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203]


def euler(dim, t_end=2.0):
    return P.SchemeConfig(P.EquationModel("euler", dim), P.FluxKind.HLLC,
                          P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=t_end)


def main(mode):
    t0 = time.time()
    if mode == "bqmc":
        grid = P.GridSpec(2, (2048, 2048), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
        cfg = P.SchemeConfig(P.EquationModel("burgers", 2), P.FluxKind.RUSANOV,
                             P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=0.02)
        init = DeviceInit(["1.0 + 0.5 * sin(2 * pi * (x + X0)) * sin(2 * pi * (y + X1))"], cfg.model, primitive=False)
        plan = uq.SamplePlan("qmc", 4, 42, 2)
        for _ in range(2):
            uq.run_mc(plan, grid, cfg, init, [uq.FieldMoments(grid, 1), uq.StructureFunctionAccumulator(2.0, 8)],
                      arith="fast", max_steps=4)
    elif mode == "mc":
        grid = P.GridSpec(2, (512, 512), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
        cfg = euler(2)
        init = DeviceInit(KH + ["0.0", "2.5"], cfg.model, primitive=True)
        plan = uq.SamplePlan("mc", 32, 42, 4)
        for _ in range(2):
            uq.run_mc(plan, grid, cfg, init, [uq.FieldMoments(grid, 4)], arith="fast", max_steps=4)
    elif mode == "halo":
        from paper_1912_07645_b200.initial import kelvin_helmholtz
        from paper_1912_07645_b200.parallel import run_parallel

        grid = P.GridSpec(2, (1024, 1024), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
        init = kelvin_helmholtz(grid, VEC)
        for _ in range(2):
            run_parallel(init, euler(2), (2, 2), n_steps=3, arith="fast")
    elif mode == "kh3d":
        n = 512
        grid = P.GridSpec(3, (n, n, n), (0.0,) * 3, (1.0,) * 3, ghost_width=2)
        cfg = euler(3)
        buf = torch.empty((1, 5) + tuple(grid.padded[::-1]), dtype=torch.float64, device="cuda")
        DeviceInit(KH + ["0.0", "0.0", "2.5"], cfg.model, primitive=True).evaluate_batch(grid, [VEC], buf)
        bufs = [buf, torch.empty_like(buf), torch.empty_like(buf)]
        run = DeviceRun(grid, cfg, bufs, 1, N.MODE_FIXED, 1 << 40, "fast", log=False)
        run.steps(3)
        run.poll()
        run.end()
    elif mode == "kh2d":
        state = Path("/tmp/kh2d_t1.npy")
        grid = P.GridSpec(2, (1024, 1024), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
        if state.exists():
            b0 = torch.from_numpy(np.load(state)).to("cuda")
        else:
            from paper_1912_07645_b200.initial import kelvin_helmholtz

            b0 = torch.from_numpy(kelvin_helmholtz(grid, VEC).data).to("cuda")
        bufs = [b0, torch.empty_like(b0), torch.empty_like(b0)]
        run = DeviceRun(grid, euler(2), bufs, 1, N.MODE_FIXED, 1 << 40, "fast", log=False)
        run.steps(3)
        run.poll()
        run.end()
    torch.cuda.synchronize()
    print(mode, "ok", round(time.time() - t0, 2), "s")


if __name__ == "__main__":
    main(sys.argv[1])
