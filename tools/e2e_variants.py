"""Time run_simulation(host Field, max_steps=10) end to end."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1912_07645_b200 as P
from paper_1912_07645_b200.initial import kelvin_helmholtz
from paper_1912_07645_b200.solver import pinned_field

n = 1024
grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC, P.Reconstruction(P.ReconstructionKind.WENO2),
                     rk_order=3, cfl=0.475, t_end=2.0)
init = pinned_field(kelvin_helmholtz(grid, [0.82, 0.19, 0.87, 0.39]))
for _ in range(3):
    out, _ = P.run_simulation(init, cfg, max_steps=10, arith="fast")
torch.cuda.synchronize()
a = time.perf_counter()
for _ in range(20):
    out, _ = P.run_simulation(init, cfg, max_steps=10, arith="fast")
torch.cuda.synchronize()
print(sys.argv[1:], f"{(time.perf_counter() - a) / 20 * 1e3:.2f} ms per call")
import numpy as np

pageable = P.Field(grid, 4, np.array(init.data))
for _ in range(2):
    P.run_simulation(pageable, cfg, max_steps=10, arith="fast")
torch.cuda.synchronize()
a = time.perf_counter()
for _ in range(20):
    out, _ = P.run_simulation(pageable, cfg, max_steps=10, arith="fast")
torch.cuda.synchronize()
print("pageable input", f"{(time.perf_counter() - a) / 20 * 1e3:.2f} ms per call")
