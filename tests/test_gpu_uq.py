"""GPU UQ parity: run_mc with on-GPU moments / structure functions against
the golden statistics of the reference's run_mc (tests/golden)."""
import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import product_objects, rel_l1

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1912_07645_b200 as P

    return P


def _setup(P, case):
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import burgers_sines, kelvin_helmholtz

    grid, cfg = product_objects(case["scheme"])
    fn = kelvin_helmholtz if case["scheme"]["eq"] == "euler" else burgers_sines
    plan = uq.SamplePlan(case["method"], case["samples"], case["seed"], case["stochastic_dim"])
    fm = uq.FieldMoments(grid, cfg.model.ncomp)
    sf = uq.StructureFunctionAccumulator(case["sf_p"], case["sf_H"])
    return uq, grid, cfg, fn, plan, fm, sf


@pytest.mark.parametrize("name", ["kh2d128_mc8", "kh2d128_qmc8", "burgers128_qmc8"])
@pytest.mark.parametrize("batch", [1, 3, 8])
def test_run_mc_matches_reference(P, golden, name, batch):
    case = next(u for u in golden["uq"] if u["name"] == name)
    uq, grid, cfg, fn, plan, fm, sf = _setup(P, case)
    m, s = uq.run_mc(plan, grid, cfg, fn, [fm, sf], batch=batch, arith="exact")
    acc = m.acc
    assert acc.count == case["samples"]
    # moments: bitwise (same per-sample merge order as the reference)
    assert O.sha16(acc.mean) == case["mean_sha"]
    assert O.sha16(acc.variance(ddof=1)) == case["var_sha"]
    assert O.sha16(acc.m2) == case["m2_sha"]
    # structure functions: summation order differs from numpy's pairwise mean
    assert rel_l1(s.sums, np.array(case["sf_sums"])) <= 1e-13
    assert s.samples == case["samples"]


def test_run_mc_fast_within_tolerance(P, golden):
    case = next(u for u in golden["uq"] if u["name"] == "kh2d128_mc8")
    uq, grid, cfg, fn, plan, fm, sf = _setup(P, case)
    m, s = uq.run_mc(plan, grid, cfg, fn, [fm, sf], arith="fast")
    ref_m, ref_sf = O.mc_moments_and_sf(lambda v: O.kelvin_helmholtz(tuple(grid.cells), v), 
                                        __import__("tests.helpers", fromlist=["x"]).oracle_scheme(case["scheme"]),
                                        case["method"], case["seed"], case["samples"], case["stochastic_dim"])
    acc = m.acc
    for c in range(acc.mean.shape[0]):
        assert rel_l1(acc.mean[c], ref_m.mean[c]) <= 1e-12
    assert rel_l1(acc.variance(), ref_m.variance()) <= 1e-10
    assert rel_l1(s.sums, ref_sf) <= 1e-12


def test_functionals_update_merge(P, golden, golden_arrays):
    """FieldMoments.update/merge and StructureFunctionAccumulator.update on
    single fields (uq.py:174-178, 254-268) against the oracle formulas."""
    from paper_1912_07645_b200 import uq

    case = next(r for r in golden["runs"] if r["name"] == "kh2d64_weno2_50")
    grid, cfg = product_objects(case["scheme"])
    a = np.array(golden_arrays["kh2d64_weno2_50__init"])
    b = np.array(golden_arrays["kh2d64_weno2_50__final"])
    fa, fb = P.Field(grid, 4, a), P.Field(grid, 4, b)
    sc = __import__("tests.helpers", fromlist=["x"]).oracle_scheme(case["scheme"])
    ref = O.Moments(O.interior(a, sc).shape)
    for x in (a, b, a):
        ref.push(np.asarray(O.interior(x, sc)))
    m1, m2 = uq.FieldMoments(grid, 4), uq.FieldMoments(grid, 4)
    m1.update(fa)
    m1.update(fb)
    m2.update(fa)
    m1.merge(m2)
    ref2 = O.Moments(ref.mean.shape)
    ref2.push(np.asarray(O.interior(a, sc)))
    ref2.push(np.asarray(O.interior(b, sc)))
    r3 = O.Moments(ref.mean.shape)
    r3.push(np.asarray(O.interior(a, sc)))
    ref2.merge(r3)
    assert np.array_equal(m1.acc.mean, ref2.mean) and np.array_equal(m1.acc.m2, ref2.m2)
    sf = uq.StructureFunctionAccumulator(2.0, 8)
    sf.update(fb)
    want = O.structure_sums(np.asarray(O.interior(b, sc)[0]), 2.0, 8)
    assert rel_l1(sf.sums, want) <= 1e-13
    sf3 = uq.StructureFunctionAccumulator(1.5, 5, component=3)
    sf3.update(fb)
    want3 = O.structure_sums(np.asarray(O.interior(b, sc)[3]), 1.5, 5)
    assert rel_l1(sf3.sums, want3) <= 1e-13


@pytest.mark.parametrize("name", ["kh2d_mlmc_2lvl", "kh2d_mlmc_1lvl", "kh2d_mlmc_qmc_2lvl"])
def test_run_mlmc_matches_reference(P, golden, name):
    """run_mlmc (uq.py:348-419): batched GPU ensembles per level, telescoping
    on the device; bitwise against the reference's run_mlmc."""
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    case = next(u for u in golden["mlmc"] if u["name"] == name)
    _, cfg = product_objects(case["scheme"])
    grids = tuple(P.GridSpec(2, tuple(c), (0.0, 0.0), (1.0, 1.0), ghost_width=2) for c in case["cells"])
    plan = uq.MlmcPlan(grids, tuple(case["samples"]), method=case["method"], seed=case["seed"],
                       stochastic_dim=case["stochastic_dim"])
    res = uq.run_mlmc(plan, lambda g: cfg, kelvin_helmholtz, arith="exact")
    assert O.sha16(res.mean) == case["mean_sha"]
    assert O.sha16(res.second_moment) == case["second_sha"]
    assert O.sha16(res.variance) == case["var_sha"]


@pytest.mark.parametrize("name", ["kh2d_mlmc_2lvl", "kh2d_mlmc_qmc_2lvl"])
def test_run_mlmc_fast_within_tolerance(P, golden, name):
    """run_mlmc in fast arithmetic (the fast-mode default kernels on every
    level) against the exact run, which test_run_mlmc_matches_reference pins
    bitwise to the reference: mean and second moment within relative L1
    1e-12, the variance (a difference of moments) within 1e-10."""
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    case = next(u for u in golden["mlmc"] if u["name"] == name)
    _, cfg = product_objects(case["scheme"])
    grids = tuple(P.GridSpec(2, tuple(c), (0.0, 0.0), (1.0, 1.0), ghost_width=2) for c in case["cells"])
    plan = uq.MlmcPlan(grids, tuple(case["samples"]), method=case["method"], seed=case["seed"],
                       stochastic_dim=case["stochastic_dim"])
    ref = uq.run_mlmc(plan, lambda g: cfg, kelvin_helmholtz, arith="exact")
    assert O.sha16(ref.mean) == case["mean_sha"]
    got = uq.run_mlmc(plan, lambda g: cfg, kelvin_helmholtz, arith="fast")
    assert rel_l1(got.mean, ref.mean) <= 1e-12
    assert rel_l1(got.second_moment, ref.second_moment) <= 1e-12
    assert rel_l1(got.variance, ref.variance) <= 1e-10


def test_histogram_functional_matches_reference(P, golden):
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    case = golden["histogram"]
    grid, cfg = product_objects(case["scheme"])
    h = uq.Histogram([tuple(p) for p in case["probes"]], case["component"], case["lo"], case["hi"], case["bins"])
    (res,) = uq.run_mc(uq.SamplePlan("mc", 8, 42, 4), grid, cfg, kelvin_helmholtz, [h], arith="exact")
    assert res.samples == case["samples"]
    assert res.counts.tolist() == case["counts"]


@pytest.mark.parametrize("workers", [1, 3])
def test_run_mc_workers_and_failing_sample(P, golden, workers):
    """Concurrent initial-data evaluation (workers > 1, prefetched a batch
    ahead) leaves the statistics bitwise unchanged, and a failing sample
    raises the reference's message for the lowest failing index
    (uq.py:281-288, pool.map order)."""
    case = next(u for u in golden["uq"] if u["name"] == "kh2d128_mc8")
    uq, grid, cfg, fn, plan, fm, sf = _setup(P, case)
    m, s = uq.run_mc(plan, grid, cfg, fn, [fm, sf], workers=workers, batch=3, arith="exact")
    assert O.sha16(m.acc.mean) == case["mean_sha"]
    assert O.sha16(m.acc.variance(ddof=1)) == case["var_sha"]

    seen = []

    def bad(g, vec):
        k = plan_vectors.index(tuple(vec))
        seen.append(k)
        if k in (5, 7):
            raise ValueError(f"boom {k}")
        return fn(g, vec)

    plan_vectors = [tuple(uq.draw_sample(plan, k)) for k in range(plan.samples)]
    with pytest.raises(P.SimulationError, match=r"^sample 5 failed: boom 5$"):
        uq.run_mc(plan, grid, cfg, bad, [uq.FieldMoments(grid, cfg.model.ncomp)], workers=workers, batch=3,
                  arith="exact")
    assert 5 in seen


@pytest.mark.parametrize("ni", ["1", "2", "4"])
def test_scalar_instances_per_block_bitwise(P, golden, monkeypatch, ni):
    """The scalar ring kernel marching 1, 2 or 4 ensemble instances per block
    (FVB_RING_NI) gives the reference's statistics bitwise."""
    monkeypatch.setenv("FVB_RING_NI", ni)
    case = next(u for u in golden["uq"] if u["name"] == "burgers128_qmc8")
    uq, grid, cfg, fn, plan, fm, sf = _setup(P, case)
    m, s = uq.run_mc(plan, grid, cfg, fn, [fm, sf], batch=4, arith="exact")
    assert O.sha16(m.acc.mean) == case["mean_sha"]
    assert O.sha16(m.acc.variance(ddof=1)) == case["var_sha"]


def test_run_mlmc_with_device_init(P, golden):
    """run_mlmc fed by the device initial-data evaluator (every level's
    samples evaluated on the GPU) against the reference's run_mlmc."""
    from paper_1912_07645_b200 import uq

    case = next(u for u in golden["mlmc"] if u["name"] == "kh2d_mlmc_2lvl")
    _, cfg = product_objects(case["scheme"])
    grids = tuple(P.GridSpec(2, tuple(c), (0.0, 0.0), (1.0, 1.0), ghost_width=2) for c in case["cells"])
    plan = uq.MlmcPlan(grids, tuple(case["samples"]), method=case["method"], seed=case["seed"],
                       stochastic_dim=case["stochastic_dim"])
    src = next(r for r in golden["runs"] if r["name"] == "kh2d64_weno2_50")  # the KH2D preset program
    dev = P.DeviceInit(src["init_exprs"], cfg.model, primitive=src["primitive"])
    res = uq.run_mlmc(plan, lambda g: cfg, dev, arith="exact")
    ref = uq.run_mlmc(plan, lambda g: cfg, __import__("paper_1912_07645_b200.initial", fromlist=["x"]).kelvin_helmholtz,
                      arith="exact")
    # KH initial values are discrete (thresholds): bitwise unless a cell centre
    # sits within an ulp of the perturbed interface
    if O.sha16(res.mean) != case["mean_sha"]:
        assert rel_l1(res.mean, ref.mean) <= 1e-12
    assert rel_l1(res.variance, ref.variance) <= 1e-10


@pytest.mark.parametrize("H,p", [(70, 2.0), (9, 1.0), (12, 1.5)])
def test_structure_function_any_max_offset(P, H, p):
    """StructureFunctionAccumulator.update (uq.py:254-262) with max offsets
    past the old 63 limit, offsets longer than the grid (np.roll wraps) and
    p != 2, against the oracle's numpy restatement."""
    from paper_1912_07645_b200 import uq

    rng = np.random.default_rng(H)
    grid = P.GridSpec(2, (48, 40), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    data = np.zeros((1, 44, 52))
    data[0, 2:42, 2:50] = rng.standard_normal((40, 48))
    sf = uq.StructureFunctionAccumulator(p, H)
    sf.update(P.Field(grid, 1, data))
    ref = O.structure_sums(data[0, 2:42, 2:50], p, H)
    assert sf.samples == 1 and len(sf.sums) == H + 1
    assert rel_l1(sf.sums, ref) <= 1e-13
