"""The product's initial data (paper_1912_07645_b200/initial.py) must be
bitwise equal to the reference's eval_init on the same random vectors
(golden SHAs from tests/golden/make_golden.py).  Host-only: runs on CPU."""
import numpy as np

import paper_1912_07645_b200 as P
from oracle import fv_oracle as O
from paper_1912_07645_b200.initial import burgers_sines, kelvin_helmholtz, sod
from paper_1912_07645_b200.uq import SamplePlan, draw_sample


def test_kh2d_1024(golden):
    vec = golden["samples"]["mc_seed42_dim4"][0]
    grid = P.GridSpec(2, (1024, 1024), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    f = kelvin_helmholtz(grid, vec)
    assert O.sha16(f.interior) == golden["kh2d1024_init_sha"]


def test_kh3d_64(golden):
    vec = golden["samples"]["mc_seed42_dim4"][0]
    grid = P.GridSpec(3, (64, 64, 64), (0.0,) * 3, (1.0,) * 3, ghost_width=2)
    assert O.sha16(kelvin_helmholtz(grid, vec).interior) == golden["kh3d64_init_sha"]


def test_burgers_qmc(golden):
    grid = P.GridSpec(2, (256, 256), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    vec = draw_sample(SamplePlan("qmc", 256, 0, 2), 5)
    assert O.sha16(burgers_sines(grid, vec).interior) == golden["burgers256_qmc5_init_sha"]


def test_uq_case_inits(golden):
    for case in golden["uq"]:
        d = case["scheme"]
        grid = P.GridSpec(2, tuple(d["cells"]), (0.0, 0.0), (1.0, 1.0), ghost_width=d["ghost"])
        fn = kelvin_helmholtz if d["eq"] == "euler" else burgers_sines
        for k, vec in enumerate(case["vectors"][:3]):
            ours = fn(grid, vec)
            ref = (O.kelvin_helmholtz if d["eq"] == "euler" else O.burgers_sines)(tuple(d["cells"]), vec)
            assert np.array_equal(ours.data, ref), (case["name"], k)


def test_sod_matches_golden_init(golden, golden_arrays):
    case = next(r for r in golden["runs"] if r["name"] == "sod1024_c1")
    grid = P.GridSpec(1, (1024,), (0.0,), (1.0,), ghost_width=1)
    assert O.sha16(sod(grid).interior) == case["init_sha"]


def test_draw_sample_matches_reference(golden):
    s = golden["samples"]
    for k in range(8):
        assert list(draw_sample(SamplePlan("mc", 8, 42, 4), k)) == s["mc_seed42_dim4"][k]
        assert list(draw_sample(SamplePlan("qmc", 8, 42, 4), k)) == s["qmc_dim4"][k]
    assert list(draw_sample(SamplePlan("mc", 2000, 7, 16), 1000)) == s["mc_seed7_dim16_k1000"]
    assert list(draw_sample(SamplePlan("qmc", 2000, 7, 16), 1000)) == s["qmc_dim16_k1000"]
