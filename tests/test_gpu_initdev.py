"""Device initial data (initdev.DeviceInit -> fvb_init_eval) against the
reference's eval_init output stored in the golden fixtures, and run_mc fed
from it."""
import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import GOLDEN_RUN_NAMES, product_objects, rel_l1_field

pytestmark = pytest.mark.gpu

TRANSCENDENTAL = ("sin", "cos", "exp", "^")


@pytest.fixture(scope="module")
def P():
    import paper_1912_07645_b200 as P

    return P


def _grid(P, case):
    grid, cfg = product_objects(case["scheme"])
    d = case["scheme"]
    if any(case["origin"]):
        grid = P.GridSpec(d["dim"], tuple(d["cells"]), tuple(case["origin"]),
                          tuple(o + c * dl for o, c, dl in zip(case["origin"], d["cells"], d["deltas"])),
                          ghost_width=d["ghost"], deltas=tuple(d["deltas"]))
    return grid, cfg


@pytest.mark.parametrize("name", GOLDEN_RUN_NAMES)
def test_device_init_matches_reference_eval_init(P, golden, golden_arrays, name):
    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = _grid(P, case)
    dev = P.DeviceInit(case["init_exprs"], cfg.model, primitive=case["primitive"])
    f = dev(grid, case["vector"])
    key = name + "__init"
    if key in golden_arrays:
        ref = np.asarray(golden_arrays[key])
        g = case["scheme"]["ghost"]
        sl = (slice(None),) + tuple(slice(g, g + n) for n in reversed(case["scheme"]["cells"]))
        ref_in, got = ref[sl], f.data[sl]
        assert np.isfinite(f.data).all()
        # ghosts are zero, like make_field(grid, ncomp, 0.0)
        mask = np.ones(f.data.shape, dtype=bool)
        mask[sl] = False
        assert not np.any(f.data[mask])
    else:  # KH presets: the product's bitwise host restatement is the reference
        from paper_1912_07645_b200.initial import kelvin_helmholtz

        ref_in = kelvin_helmholtz(grid, case["vector"]).interior
        got = f.interior
    if not any(op in t for t in case["init_exprs"] for op in TRANSCENDENTAL):
        assert O.sha16(np.ascontiguousarray(got)) == case["init_sha"], name  # IEEE ops only: bitwise
    else:
        assert rel_l1_field(got, ref_in) <= 1e-14, name
        assert O.sha16(np.ascontiguousarray(got)) == case["init_sha"] or np.max(np.abs(got - ref_in)) <= 1e-13


def test_device_init_errors(P):
    grid = P.GridSpec(2, (8, 6), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    euler = P.EquationModel("euler", 2)
    with pytest.raises(P.ExprError, match=r"^component 1 evaluates to a non-finite value at cell \(0, 3\): "
                                          r"1.0 / \(x - 0.4375\)$"):
        P.DeviceInit(["1", "1 / (x - 0.4375)", "0", "1"], euler)(grid)
    with pytest.raises(P.UnphysicalStateError, match="^non-positive density or pressure in primitive state$"):
        P.DeviceInit(["x - 0.5", "0", "0", "1"], euler)(grid)
    with pytest.raises(P.UnphysicalStateError, match="^initial data is unphysical$"):
        P.DeviceInit(["1", "0", "0", "0.1 - x"], euler, primitive=False)(grid)
    with pytest.raises(P.ExprError, match="random symbol X2 exceeds the stochastic dimension"):
        P.DeviceInit(["1 + X2", "0", "0", "1"], euler)(grid, (0.1, 0.2))
    with pytest.raises(P.ExprError, match="need 4 component expressions, got 1"):
        P.DeviceInit(["1"], euler)(grid)


@pytest.mark.parametrize("name", ["kh2d128_mc8", "kh2d128_qmc8", "burgers128_qmc8"])
def test_run_mc_with_device_init(P, golden, name):
    from paper_1912_07645_b200 import uq

    case = next(u for u in golden["uq"] if u["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    # the same preset programs, as the reference printed them for the runs
    src = next(r for r in golden["runs"]
               if r["name"] == ("burgers2d64_qmc0" if case["scheme"]["eq"] == "burgers" else "kh2d64_weno2_50"))
    exprs, primitive = src["init_exprs"], src["primitive"]
    dev = P.DeviceInit(exprs, cfg.model, primitive=primitive)
    plan = uq.SamplePlan(case["method"], case["samples"], case["seed"], case["stochastic_dim"])
    m, s = uq.run_mc(plan, grid, cfg, dev, [uq.FieldMoments(grid, cfg.model.ncomp),
                                            uq.StructureFunctionAccumulator(case["sf_p"], case["sf_H"])],
                     batch=3, arith="exact")
    acc = m.acc
    assert acc.count == case["samples"]
    # the KH / Burgers programs use sin: bitwise when no value moves by an ulp,
    # else rounding-level close
    if O.sha16(acc.mean) != case["mean_sha"]:
        assert float(acc.variance(ddof=1)[0].max()) == pytest.approx(case["max_var0"], rel=1e-10)
    assert np.allclose(s.values(), case["sf"], rtol=1e-10, atol=0)
