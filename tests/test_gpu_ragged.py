"""Ragged grids: extents that are not multiples of any tile, strip, chunk or
warp size (the pair kernel's 62-cell strips and row chunks, ring3i's 30 x 8
tiles), tiny extents, mixed periodic / outflow boundaries.  Exact mode is
bitwise equal to the oracle (fields and dt); fast mode within relative L1
1e-12 per component.  The oracle is the golden-pinned numpy restatement
(oracle/fv_oracle.py); KH / Burgers initial data as in the presets."""
import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import oracle_scheme, product_objects, rel_l1_field

pytestmark = pytest.mark.gpu

KH_VEC = [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203]

CASES = [
    # name, eq, flux, recon, rk, cells, bcs, steps
    ("kh2d_1000x37", "euler", "hllc", "weno2", 3, (1000, 37), ("periodic", "periodic"), 3),
    ("kh2d_63x130_outflow_x", "euler", "hllc", "weno2", 3, (63, 130), ("outflow", "periodic"), 3),
    ("kh2d_129x67_weno3", "euler", "hllc", "weno3", 3, (129, 67), ("periodic", "periodic"), 3),
    ("kh2d_125x3_rusanov_rk2", "euler", "rusanov", "weno2", 2, (125, 3), ("periodic", "periodic"), 4),
    ("kh2d_7x5_none_rk1", "euler", "hllc", "none", 1, (7, 5), ("periodic", "outflow"), 5),
    ("burgers2d_517x130", "burgers", "rusanov", "weno2", 3, (517, 130), ("periodic", "periodic"), 3),
    ("kh3d_45x33x29", "euler", "hllc", "weno2", 3, (45, 33, 29), ("periodic", "periodic", "periodic"), 2),
    ("kh3d_31x9x70_mixed", "euler", "hllc", "weno2", 3, (31, 9, 70), ("outflow", "periodic", "outflow"), 2),
    ("kh3d_61x17x5_rusanov", "euler", "rusanov", "weno3", 2, (61, 17, 5), ("periodic", "periodic", "periodic"), 2),
]


def _scheme(eq, flux, recon, rk, cells, bcs):
    return dict(dim=len(cells), cells=list(cells), deltas=[1.0 / n for n in cells], eq=eq, gamma=1.4, adv=[],
                flux=flux, recon=recon, eps=1e-6, rk=rk, cfl=0.475, t_end=10.0, bcs=list(bcs),
                ghost=1 if recon == "none" else 2)


def _init(eq, cells, ghost):
    if eq == "euler":
        return O.kelvin_helmholtz(tuple(cells), KH_VEC, ghost=ghost)
    return O.burgers_sines(tuple(cells), KH_VEC[:2], ghost=ghost)


@pytest.fixture(scope="module")
def P():
    import paper_1912_07645_b200 as P

    return P


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_ragged_grid(P, case, arith):
    _, eq, flux, recon, rk, cells, bcs, steps = case
    d = _scheme(eq, flux, recon, rk, cells, bcs)
    grid, cfg = product_objects(d)
    sc = oracle_scheme(d)
    u0 = _init(eq, cells, sc.ghost)
    ref, log = O.simulate(np.array(u0), sc, steps)
    out, recs = P.run_simulation(P.Field(grid, u0.shape[0], u0.copy()), cfg, max_steps=steps, arith=arith)
    assert len(recs) == steps
    if arith == "exact":
        assert [r.dt for r in recs] == [dt for (_, _, dt) in log]
        assert O.sha16(out.interior) == O.sha16(O.interior(ref, sc)), case[0]
    else:
        assert max(abs(r.dt - dt) / dt for r, (_, _, dt) in zip(recs, log)) <= 1e-12
        assert rel_l1_field(out.interior, O.interior(ref, sc)) <= 1e-12, case[0]
