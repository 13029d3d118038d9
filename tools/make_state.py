"""Advance KH2D 1024^2 (WENO2/HLLC/RK3) to t >= T and save the padded field
(profiling runs then start from a developed state without the warm loop)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_1912_07645_b200 as P
from paper_1912_07645_b200.initial import kelvin_helmholtz

T = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/kh2d_t1.npy"
n = 1024
grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC, P.Reconstruction(P.ReconstructionKind.WENO2),
                     rk_order=3, cfl=0.475, t_end=T)
init = kelvin_helmholtz(grid, [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203])
final, recs = P.run_simulation(init, cfg, arith="exact")
np.save(out, final.data)
print("saved", out, "t =", recs[-1].t, "steps", len(recs))
