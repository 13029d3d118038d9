"""C1 parity gate timing: Sod 1024, HLLC, no reconstruction, RK1, CFL 0.4,
t_end 0.2 (1119 steps) through run_simulation, exact arithmetic."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import hashlib

import paper_1912_07645_b200 as P
from paper_1912_07645_b200.initial import sod

grid = P.GridSpec(1, (1024,), (0.0,), (1.0,), ghost_width=1)
cfg = P.SchemeConfig(P.EquationModel("euler", 1), P.FluxKind.HLLC, P.Reconstruction(), rk_order=1, cfl=0.4,
                     t_end=0.2, bc=(P.BoundaryKind.OUTFLOW,))
init = sod(grid)
P.run_simulation(init, cfg)
for _ in range(3):
    a = time.perf_counter()
    final, recs = P.run_simulation(init, cfg)
    el = time.perf_counter() - a
sha = hashlib.sha256(final.interior.tobytes()).hexdigest()[:16]
print(f"C1: {len(recs)} steps, dt1={recs[0].dt!r}, sha={sha}, {el*1e3:.2f} ms wall "
      f"({1024*len(recs)/el/1e9:.4f} Gcell-stage/s)")
