"""Parity at the sizes bench.py measures (BASELINE configs[1]-[4]).

* KH2D 1024^2 (C2), exact mode: 2 RK3 steps from t = 0 and 2 steps from the
  developed state bench.py times (t ~ 1, rolled-up shear layers), bitwise
  equal to the oracle (fields and dt sequences).
* KH2D 1024^2 fast mode from that state after 1, 3 and 10 steps: relative
  L1 <= 1e-12 per component (sum|a-b| / sum|b| of each conserved
  component, no floor), dt within 1e-12.
* KH3D 128^3 (C4 shape), exact, 1 step: bitwise; and from a developed state
  with flow along all three axes (t = 0.5, averaged with its y<->z
  transpose): exact 1 step bitwise, fast after 1 and 3 steps <= 1e-12 per
  component.
* C3: run_mc over 16 KH2D samples at 512^2 and C5: 4 Burgers QMC samples at
  2048^2 (truncated t_end, two steps each), exact mode: moments bitwise equal
  to the sequential sample-order merge of the oracle's per-sample finals,
  structure functions within 1e-13; fast mode within the tolerance.

The oracle references (test infrastructure) run concurrently in spawned
host processes (tests/oracle_jobs.py) while the GPU computes.
"""
import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import fv_oracle as O
from tests import oracle_jobs as J
from tests.helpers import rel_l1

pytestmark = pytest.mark.gpu

KH_VEC = [0.8201981478608876, 0.18924562408645496, 0.8676608148821462, 0.3945814702827203]
KH_SCHEME = dict(eq="euler", flux="hllc", recon="weno2", rk=3, cfl=0.475, t_end=2.0)
C3_TEND = 4.0e-4   # dt_1 ~ 2.19e-4 at 512^2: two steps
C5_TEND = 1.5e-4   # dt_1 ~ 7.7e-5 at 2048^2: two steps
FAST_CHECKPOINTS = (1, 3, 10)
KH3D_CHECKPOINTS = (1, 3)


def rel_l1_components(a, b):
    """max over components of sum|a_c - b_c| / sum|b_c| (no floor)."""
    return max(float(np.abs(a[c] - b[c]).sum() / np.abs(b[c]).sum()) for c in range(b.shape[0]))


def _kh_objects(P, n, dim=2, t_end=2.0):
    grid = P.GridSpec(dim, (n,) * dim, (0.0,) * dim, (1.0,) * dim, ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", dim), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=t_end)
    return grid, cfg


def _burgers_objects(P, n, t_end):
    grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("burgers", 2), P.FluxKind.RUSANOV,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=t_end)
    return grid, cfg


@pytest.fixture(scope="module")
def P():
    import paper_1912_07645_b200 as P

    return P


@pytest.fixture(scope="module")
def pool():
    ex = cf.ProcessPoolExecutor(max_workers=max(2, min(24, os.cpu_count() or 2)),
                                mp_context=mp.get_context("spawn"))
    yield ex
    ex.shutdown(cancel_futures=True)


@pytest.fixture(scope="module")
def jobs(P, pool):
    """Submit every oracle reference up front; the tests wait on theirs."""
    from paper_1912_07645_b200.initial import kelvin_helmholtz
    from paper_1912_07645_b200.uq import SamplePlan, draw_sample

    f = {}
    n = 1024
    s2 = dict(dim=2, cells=(n, n), deltas=(1.0 / n, 1.0 / n), **KH_SCHEME)
    grid, cfg = _kh_objects(P, n)
    init = kelvin_helmholtz(grid, KH_VEC)
    f["kh_t0"] = pool.submit(J.simulate_checkpoints, init.data, s2, (2,))
    s3 = dict(dim=3, cells=(128,) * 3, deltas=(1.0 / 128,) * 3, **KH_SCHEME)
    f["kh3d"] = pool.submit(J.simulate_checkpoints, O.kelvin_helmholtz((128,) * 3, KH_VEC), s3, (1,))
    # C3 / C5 per-sample finals (merged in sample order by the tests)
    c3 = dict(dim=2, cells=(512, 512), deltas=(1.0 / 512,) * 2, **dict(KH_SCHEME, t_end=C3_TEND))
    plan3 = SamplePlan("mc", 16, 42, 4)
    f["c3"] = [pool.submit(J.sample_final, "kh", (512, 512), draw_sample(plan3, k), c3) for k in range(16)]
    c5 = dict(dim=2, cells=(2048, 2048), deltas=(1.0 / 2048,) * 2, eq="burgers", flux="rusanov", recon="weno2",
              rk=3, cfl=0.475, t_end=C5_TEND)
    plan5 = SamplePlan("qmc", 4, 42, 2)
    f["c5"] = [pool.submit(J.sample_final, "burgers", (2048, 2048), draw_sample(plan5, k), c5) for k in range(4)]
    # the developed state bench.py times: advanced on the GPU (an input only)
    gcfg = P.SchemeConfig(cfg.model, cfg.flux, cfg.recon, 3, 0.475, 1.0)
    state, recs = P.run_simulation(init, gcfg, arith="fast")
    assert recs[-1].t >= 1.0 - 1e-12
    f["state"] = state
    f["kh_t1"] = pool.submit(J.simulate_checkpoints, state.data, s2, (2,))
    for k in FAST_CHECKPOINTS:  # separate jobs: they run side by side
        f[f"kh_t1_{k}"] = pool.submit(J.simulate_checkpoints, state.data, s2, (k,))
    # a developed 3D state with flow in all three directions: KH3D 128^3 run
    # to t = 0.5 on the GPU (z-uniform, vz = 0 -- the preset is extruded), then
    # averaged with its y<->z transpose (axes and momenta swapped): a convex
    # combination of physical states, non-trivial along every axis
    g3, c3cfg = _kh_objects(P, 128, dim=3)
    st3, _ = P.run_simulation(kelvin_helmholtz(g3, KH_VEC),
                              P.SchemeConfig(c3cfg.model, c3cfg.flux, c3cfg.recon, 3, 0.475, 0.5), arith="fast")
    d = st3.data
    mix = np.ascontiguousarray(0.5 * (d + d.transpose(0, 2, 1, 3)[[0, 1, 3, 2, 4]]))
    f["state3"] = mix
    for k in KH3D_CHECKPOINTS:
        f[f"kh3d_mix_{k}"] = pool.submit(J.simulate_checkpoints, mix, s3, (k,))
    return f


def _moments_ref(finals):
    mom = O.Moments(finals[0].shape)
    for a in finals:
        mom.push(a)
    return mom


def test_kh2d_1024_exact_from_t0(P, jobs):
    grid, cfg = _kh_objects(P, 1024)
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    out, recs = P.run_simulation(kelvin_helmholtz(grid, KH_VEC), cfg, max_steps=2, arith="exact")
    ref, dts = jobs["kh_t0"].result()[2]
    assert [r.dt for r in recs] == dts
    assert np.array_equal(out.interior, ref), "KH2D 1024^2 exact differs from the oracle (t = 0)"


def test_kh2d_1024_exact_from_developed_state(P, jobs):
    grid, cfg = _kh_objects(P, 1024)
    state = jobs["state"]
    out, recs = P.run_simulation(P.Field(grid, 4, state.data.copy()), cfg, max_steps=2, arith="exact")
    ref, dts = jobs["kh_t1"].result()[2]
    assert [r.dt for r in recs] == dts
    assert O.sha16(out.interior) == O.sha16(ref), "KH2D 1024^2 exact differs from the oracle (t ~ 1)"


@pytest.mark.parametrize("steps", FAST_CHECKPOINTS)
def test_kh2d_1024_fast_from_developed_state(P, jobs, steps):
    grid, cfg = _kh_objects(P, 1024)
    state = jobs["state"]
    out, recs = P.run_simulation(P.Field(grid, 4, state.data.copy()), cfg, max_steps=steps, arith="fast")
    ref, dts = jobs[f"kh_t1_{steps}"].result()[steps]
    err = rel_l1_components(out.interior, ref)
    assert err <= 1e-12, f"fast mode relative L1 {err:.3e} after {steps} steps"
    assert max(abs(r.dt - d) / d for r, d in zip(recs, dts)) <= 1e-12


def test_kh3d_128_exact_one_step(P, jobs):
    grid, cfg = _kh_objects(P, 128, dim=3)
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    out, recs = P.run_simulation(kelvin_helmholtz(grid, KH_VEC), cfg, max_steps=1, arith="exact")
    ref, dts = jobs["kh3d"].result()[1]
    assert [r.dt for r in recs] == dts
    assert np.array_equal(out.interior, ref), "KH3D 128^3 exact differs from the oracle"


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c3_run_mc_512_16_samples(P, jobs, arith):
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    grid, cfg = _kh_objects(P, 512, t_end=C3_TEND)
    plan = uq.SamplePlan("mc", 16, 42, 4)
    m, = uq.run_mc(plan, grid, cfg, kelvin_helmholtz, [uq.FieldMoments(grid, 4)], arith=arith)
    ref = _moments_ref([f.result() for f in jobs["c3"]])
    assert m.acc.count == 16
    if arith == "exact":
        assert O.sha16(m.acc.mean) == O.sha16(ref.mean)
        assert O.sha16(m.acc.variance(ddof=1)) == O.sha16(ref.variance())
    else:
        assert rel_l1_components(m.acc.mean, ref.mean) <= 1e-12
        assert rel_l1(m.acc.variance(ddof=1), ref.variance()) <= 1e-10


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c5_burgers_qmc_2048_4_samples(P, jobs, pool, arith):
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import burgers_sines

    grid, cfg = _burgers_objects(P, 2048, C5_TEND)
    plan = uq.SamplePlan("qmc", 4, 42, 2)
    m, s = uq.run_mc(plan, grid, cfg, burgers_sines,
                     [uq.FieldMoments(grid, 1), uq.StructureFunctionAccumulator(2.0, 8)], arith=arith)
    finals = [f.result() for f in jobs["c5"]]
    ref = _moments_ref(finals)
    sf = sum(pool.map(J.structure_sums, [a[0] for a in finals], [2.0] * 4, [8] * 4))
    if arith == "exact":
        assert O.sha16(m.acc.mean) == O.sha16(ref.mean)
        assert O.sha16(m.acc.variance(ddof=1)) == O.sha16(ref.variance())
        assert rel_l1(s.sums, sf) <= 1e-13
    else:
        assert rel_l1(m.acc.mean, ref.mean) <= 1e-12
        assert rel_l1(m.acc.variance(ddof=1), ref.variance()) <= 1e-10
        assert rel_l1(s.sums, sf) <= 1e-12
    assert s.samples == 4


def test_kh3d_128_fast_one_step(P, jobs):
    """The fast-mode 3D default (ring3i) at 128^3 against the oracle.  At t = 0
    the y/z momenta are pure pressure round-off (vy = vz = 0), so their error
    is measured against 1e-3 of the largest component's norm (helpers.rel_l1_field)."""
    from paper_1912_07645_b200.initial import kelvin_helmholtz
    from tests.helpers import rel_l1_field

    grid, cfg = _kh_objects(P, 128, dim=3)
    out, recs = P.run_simulation(kelvin_helmholtz(grid, KH_VEC), cfg, max_steps=1, arith="fast")
    ref, dts = jobs["kh3d"].result()[1]
    assert rel_l1_field(out.interior, ref) <= 1e-12
    assert abs(recs[0].dt - dts[0]) <= 1e-12 * dts[0]


def test_kh3d_128_exact_from_developed_3d_state(P, jobs):
    """KH3D 128^3 exact mode, 1 step from the developed three-direction state:
    bitwise equal to the oracle (fields and dt)."""
    grid, cfg = _kh_objects(P, 128, dim=3)
    out, recs = P.run_simulation(P.Field(grid, 5, jobs["state3"].copy()), cfg, max_steps=1, arith="exact")
    ref, dts = jobs["kh3d_mix_1"].result()[1]
    assert [r.dt for r in recs] == dts
    assert O.sha16(out.interior) == O.sha16(ref), "KH3D 128^3 exact differs from the oracle (developed state)"


@pytest.mark.parametrize("steps", KH3D_CHECKPOINTS)
def test_kh3d_128_fast_from_developed_3d_state(P, jobs, steps):
    """The fast 3D default (ring3i) from the developed three-direction state:
    relative L1 <= 1e-12 per conserved component, no floor (every momentum
    component is O(1) here), dt within 1e-12."""
    grid, cfg = _kh_objects(P, 128, dim=3)
    out, recs = P.run_simulation(P.Field(grid, 5, jobs["state3"].copy()), cfg, max_steps=steps, arith="fast")
    ref, dts = jobs[f"kh3d_mix_{steps}"].result()[steps]
    err = rel_l1_components(out.interior, ref)
    assert err <= 1e-12, f"fast mode relative L1 {err:.3e} after {steps} steps"
    assert max(abs(r.dt - d) / d for r, d in zip(recs, dts)) <= 1e-12
