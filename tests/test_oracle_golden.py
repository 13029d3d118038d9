"""Pin the CPU oracle to the reference: every golden fingerprint produced by
running the reference package (tests/golden/make_golden.py) must be
reproduced bitwise by oracle/fv_oracle.py."""
import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import GOLDEN_RUN_NAMES, oracle_scheme

FAST_RUNS = None


def _runs(golden):
    return [r for r in golden["runs"] if r["name"] != "sod1024_c1"]


def test_sod_c1_gate(golden, golden_arrays):
    case = next(r for r in golden["runs"] if r["name"] == "sod1024_c1")
    sc = oracle_scheme(case["scheme"])
    init = golden_arrays["sod1024_c1__init"]
    final, log = O.simulate(init, sc, case["max_steps"])
    assert len(log) == case["steps"] == 1119
    assert log[0][2] == case["dts"][0] == 3.301383807533268e-4
    assert O.sha16(O.interior(final, sc)) == case["final_sha"] == "9c0cbfebb9424977"


@pytest.mark.parametrize("name", [n for n in GOLDEN_RUN_NAMES if n != "sod1024_c1"])
def test_oracle_runs_bitwise(golden, golden_arrays, name):
    case = next(r for r in _runs(golden) if r["name"] == name)
    sc = oracle_scheme(case["scheme"])
    key = case["name"] + "__init"
    if key in golden_arrays:
        init = golden_arrays[key]
    else:
        init = O.kelvin_helmholtz(tuple(sc.cells), case["vector"], ghost=sc.ghost)
    assert O.sha16(O.interior(init, sc)) == case["init_sha"]
    final, log = O.simulate(init, sc, case["max_steps"])
    assert len(log) == case["steps"]
    assert [d for (_, _, d) in log[:8]] == case["dts"]
    assert O.sha16(np.array([d for (_, _, d) in log])) == case["dt_sha"]
    assert O.sha16(O.interior(final, sc)) == case["final_sha"], case["name"]
    assert O.sha16(final) == case["data_sha"]


def test_residual_cases_bitwise(golden, golden_arrays):
    for case in golden["residuals"]:
        sc = oracle_scheme(case["scheme"])
        u = golden_arrays[case["name"] + "__u"].copy()
        # the stored array is already ghost-filled; re-fill to check ghost_fill
        raw = O.padded_from_interior(sc, O.interior(u, sc))
        O.ghost_fill(raw, sc)
        assert O.sha16(raw) == case["filled_sha"], case["name"]
        L = O.residual(raw, sc)
        assert O.sha16(L) == case["L_sha"], case["name"]
        assert list(O.speed_maxima(raw, sc)) == case["max"], case["name"]


def test_error_cases(golden):
    errs = {e["name"]: e for e in golden["errors"]}
    sc = O.Scheme(dim=1, cells=(8,), deltas=(1 / 8,), eq="euler", flux="hllc", rk=1, t_end=0.1)
    u = np.zeros((3, 8))
    u[0] = 1.0
    u[2] = 2.5
    u[0, 5] = -1.0
    with pytest.raises(O.OracleError) as ei:
        O.simulate(O.padded_from_interior(sc, u), sc)
    assert ei.value.kind == errs["unphysical_init"]["kind"]
    sc = O.Scheme(dim=2, cells=(6, 5), deltas=(1 / 6, 1 / 5), eq="burgers", recon="weno2", rk=3, t_end=0.1)
    with pytest.raises(O.OracleError) as ei:
        O.simulate(O.padded_from_interior(sc, np.zeros((1, 5, 6))), sc)
    assert ei.value.kind == errs["static_field"]["kind"] == "StaticFieldError"
    sc = O.Scheme(dim=1, cells=(16,), deltas=(1 / 16,), eq="burgers", rk=1, t_end=1.0)
    u = np.ones((1, 16))
    u[0, 9] = 1e200
    with np.errstate(all="ignore"), pytest.raises(O.OracleError) as ei:
        O.simulate(O.padded_from_interior(sc, u), sc)
    assert "non-finite value after step 1" in str(ei.value)
    assert "(8,)" in errs["nonfinite"]["msg"] and "(8,)" in str(ei.value)


def test_sample_vectors(golden):
    s = golden["samples"]
    for k in range(8):
        assert list(O.sample_vector("mc", 42, k, 4)) == s["mc_seed42_dim4"][k]
        assert list(O.sample_vector("qmc", 42, k, 4)) == s["qmc_dim4"][k]
    assert list(O.sample_vector("mc", 7, 1000, 16)) == s["mc_seed7_dim16_k1000"]
    assert list(O.sample_vector("qmc", 7, 1000, 16)) == s["qmc_dim16_k1000"]


def test_kh_initial_data(golden):
    vec = golden["samples"]["mc_seed42_dim4"][0]
    init = O.kelvin_helmholtz((1024, 1024), vec)
    sc = O.Scheme(dim=2, cells=(1024, 1024), deltas=(1 / 1024,) * 2, eq="euler", recon="weno2")
    assert O.sha16(O.interior(init, sc)) == golden["kh2d1024_init_sha"]


@pytest.mark.parametrize("name", ["kh2d128_mc8", "kh2d128_qmc8", "burgers128_qmc8"])
def test_uq_gates(golden, name):
    case = next(u for u in golden["uq"] if u["name"] == name)
    sc = oracle_scheme(case["scheme"])
    if sc.eq == "euler":
        init_fn = lambda v: O.kelvin_helmholtz(tuple(sc.cells), v, ghost=sc.ghost)
    else:
        init_fn = lambda v: O.burgers_sines(tuple(sc.cells), v, ghost=sc.ghost)
    mom, sf = O.mc_moments_and_sf(init_fn, sc, case["method"], case["seed"], case["samples"],
                                  case["stochastic_dim"], case["sf_p"], case["sf_H"])
    assert O.sha16(mom.mean) == case["mean_sha"]
    assert O.sha16(mom.variance()) == case["var_sha"]
    assert O.sha16(mom.m2) == case["m2_sha"]
    assert list(sf) == case["sf_sums"]
