"""Domain decomposition on the GPU: run_parallel must be bitwise equal to the
serial solver for every rank layout (reference tests/test_parallel.py:
192-212), in n_steps and t_end modes, and exchange_halos must reproduce the
serial ghost fill (tests/test_parallel.py:120-154)."""
import threading

import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import oracle_scheme, product_objects

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1912_07645_b200 as P

    return P


CASES = [("kh2d64_weno2_50", [(2, 1), (1, 2), (2, 2), (4, 1), (4, 4)]),
         ("euler2d_hllc_weno3_outflow", [(2, 1), (2, 2)]),
         ("euler2d_rusanov_none_outflow", [(2, 2)]),
         ("advection2d_weno3_rk3", [(2, 2)]),
         ("burgers1d_weno2_rk1_periodic", [(2,), (4,)]),
         ("burgers1d_none_rk2_outflow", [(3,)]),
         ("kh3d16_weno2_5", [(2, 2, 2), (1, 1, 4)]),
         ("euler3d_hllc_none_outflow", [(2, 1, 2)])]


@pytest.mark.parametrize("name,layouts", CASES)
def test_run_parallel_fixed_bitwise(P, golden, golden_arrays, name, layouts):
    from paper_1912_07645_b200.parallel import run_parallel

    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(golden_arrays[name + "__init"])
    init = P.Field(grid, data.shape[0], data)
    sc = oracle_scheme(case["scheme"])
    n = 6
    ref, log = O.simulate_fixed(init.data, sc, n)
    for lay in layouts:
        if any(c % r for c, r in zip(grid.cells, lay)):
            continue
        out, recs = run_parallel(init, cfg, lay, n_steps=n, arith="exact")
        assert len(recs) == int(np.prod(lay)) and len(recs[0]) == n
        assert [r.dt for r in recs[0]] == [d for (_, _, d) in log], (name, lay)
        assert O.sha16(out.interior) == O.sha16(O.interior(ref, sc)), (name, lay)


def test_run_parallel_t_end_matches_serial(P, golden, golden_arrays):
    from paper_1912_07645_b200.parallel import run_parallel

    for name in ("burgers1d_weno3_rk3_outflow", "euler2d_hllc_weno2_periodic"):
        case = next(r for r in golden["runs"] if r["name"] == name)
        grid, cfg = product_objects(case["scheme"])
        data = np.array(golden_arrays[name + "__init"])
        init = P.Field(grid, data.shape[0], data)
        lay = (2,) if grid.dim == 1 else (2, 2)
        out, recs = run_parallel(init, cfg, lay, arith="exact")
        assert len(recs[0]) == case["steps"]
        assert O.sha16(out.interior) == case["final_sha"], name


def test_exchange_halos_matches_serial_fill(P, golden, golden_arrays):
    from paper_1912_07645_b200 import parallel as PP

    for name, lay in (("kh2d32_weno3_20", (2, 2)), ("euler2d_hllc_weno2_outflow", (2, 2)),
                      ("kh3d8_weno3_full", (2, 1, 2)), ("burgers1d_weno2_rk1_outflow", (4,))):
        case = next(r for r in golden["runs"] if r["name"] == name)
        grid, cfg = product_objects(case["scheme"])
        sc = oracle_scheme(case["scheme"])
        data = np.array(golden_arrays[name + "__final"])
        glob = P.Field(grid, data.shape[0], data.copy())
        want = O.ghost_fill(data.copy(), sc)
        topo = PP.RankTopology(lay)
        parts = PP.decompose(grid, topo)
        locs = PP.scatter_field(glob, parts)
        tr = PP.InProcessTransport(topo.size)
        errs = []

        def work(r):
            try:
                PP.exchange_halos(locs[r], r, topo, tr, cfg.bc, tag=1)
            except BaseException as e:  # surfaced below
                errs.append(e)

        ths = [threading.Thread(target=work, args=(r,)) for r in range(topo.size)]
        [t.start() for t in ths]
        [t.join() for t in ths]
        assert not errs, errs
        g = grid.ghost_width
        for part, loc in zip(parts, locs):
            sl = (slice(None),) + tuple(
                slice(part.offset[grid.dim - 1 - j], part.offset[grid.dim - 1 - j] + part.grid.padded[grid.dim - 1 - j])
                for j in range(grid.dim))
            assert np.array_equal(loc.data, want[sl]), (name, part.rank)


def test_protocol_errors(P):
    from paper_1912_07645_b200 import parallel as PP

    tr = PP.InProcessTransport(2)
    tr.send(PP.HaloMessage(0, 1, 0, 1, 5, np.zeros(1)))
    with pytest.raises(P.ProtocolError):
        tr.send(PP.HaloMessage(0, 1, 0, 1, 5, np.zeros(1)))
    with pytest.raises(P.ProtocolError):
        tr.receive(0, 1, 1, 1, 5)


@pytest.mark.parametrize("name,layouts", [("kh2d64_weno2_50", [(2, 1), (1, 2), (2, 2)]),
                                          ("euler2d_hllc_weno3_outflow", [(2, 1), (2, 2)]),
                                          ("kh3d16_weno2_5", [(2, 2, 2), (1, 2, 1)])])
def test_run_parallel_fast_decomposition_invariant(P, golden, golden_arrays, name, layouts):
    """Fast mode (the pair kernel in 2D, ring3i in 3D, ghosts of split axes
    read from memory incl. the 16-byte ring copies): a decomposed run equals
    the undecomposed fast run bitwise -- the reference's decomposition
    invariance (tests/test_parallel.py:192-212) holds in both modes."""
    from paper_1912_07645_b200.parallel import run_parallel

    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(golden_arrays[name + "__init"])
    init = P.Field(grid, data.shape[0], data)
    whole, _ = run_parallel(init, cfg, (1,) * grid.dim, n_steps=5, arith="fast")
    for lay in layouts:
        out, recs = run_parallel(init, cfg, lay, n_steps=5, arith="fast")
        assert O.sha16(out.interior) == O.sha16(whole.interior), (name, lay)
