"""Per-step cost of run_simulation observers (lazy host fields) on KH2D
1024^2: none, a no-op observer, and one reading the field every 50 steps."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1912_07645_b200 as P
from paper_1912_07645_b200.initial import kelvin_helmholtz
from paper_1912_07645_b200.solver import pinned_field
n = 1024
grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC, P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=2.0)
init = pinned_field(kelvin_helmholtz(grid, (0.82, 0.19, 0.87, 0.39)))
P.run_simulation(init, cfg, max_steps=5, arith="fast")
for name, obs in (("none", []), ("no-op", [lambda s, t, f: None]),
                  ("reads every 50th", [lambda s, t, f: f.interior.sum() if s % 50 == 0 else None])):
    for rep in range(2):  # report the warm repetition
        torch.cuda.synchronize(); t0 = time.perf_counter()
        P.run_simulation(init, cfg, observers=obs, max_steps=200, arith="fast")
        torch.cuda.synchronize(); ms = (time.perf_counter() - t0) / 200 * 1e3
    print(f"observer {name}: {ms:.3f} ms/step")
