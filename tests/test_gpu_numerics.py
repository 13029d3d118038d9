"""The function-level numerics API on the GPU (numerics.py:64-210 of the
reference): WENO weights / face values, reconstruct_axis, Rusanov and HLLC
fluxes through the FLUX_FUNCTIONS registry -- bitwise equal to the oracle
(pinned to the reference) in exact arithmetic, and to the reference package
itself when baseline/_ref is installed; the reference's error behaviour
(degenerate HLLC fan, unphysical states, HLLC on a scalar law)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import fv_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def NM():
    from paper_1912_07645_b200 import numerics

    return numerics


def _states(rng, dim, n, ncomp=None):
    """Random physical Euler states (rho, m, E) with a few exactly equal pairs."""
    rho = rng.uniform(0.2, 3.0, n)
    v = rng.uniform(-2.0, 2.0, (dim, n))
    p = rng.uniform(0.1, 5.0, n)
    u = np.empty((dim + 2, n))
    u[0] = rho
    u[1:1 + dim] = rho * v
    u[1 + dim] = p / 0.4 + 0.5 * rho * (v * v).sum(axis=0)
    return u


@pytest.mark.parametrize("dim", [1, 2, 3])
@pytest.mark.parametrize("flux", ["hllc", "rusanov"])
def test_euler_flux_bitwise(NM, dim, flux):
    import paper_1912_07645_b200 as P

    rng = np.random.default_rng(dim * 7 + len(flux))
    uL, uR = _states(rng, dim, 5000), _states(rng, dim, 5000)
    uR[:, ::17] = uL[:, ::17]  # exact consistency F(u, u) = f(u) (numerics.py:195-196)
    uR[1:, 3::29] = uL[1:, 3::29] * 1.25  # equal momenta/energy ratios, different states
    uR[0, 3::29] = uL[0, 3::29] * 1.25
    model = P.EquationModel("euler", dim)
    sc = O.Scheme(dim=dim, cells=(4,) * dim, deltas=(0.25,) * dim, eq="euler", flux=flux)
    for axis in range(dim):
        got = NM.FLUX_FUNCTIONS[P.FluxKind(flux)](model, NM.FacePair(uL, uR), axis)
        ref = O._FLUX[flux](sc, uL, uR, axis)
        assert np.array_equal(got, ref), (flux, dim, axis)
        # numerical_flux dispatch, trailing shape kept
        got2 = NM.numerical_flux(model, P.FluxKind(flux), NM.FacePair(uL.reshape(dim + 2, 50, 100),
                                                                      uR.reshape(dim + 2, 50, 100)), axis)
        assert got2.shape == (dim + 2, 50, 100) and np.array_equal(got2.reshape(dim + 2, -1), ref)


@pytest.mark.parametrize("eq", ["burgers", "advection"])
def test_scalar_rusanov_bitwise(NM, eq):
    import paper_1912_07645_b200 as P

    rng = np.random.default_rng(3)
    uL, uR = rng.uniform(-2, 2, (1, 4000)), rng.uniform(-2, 2, (1, 4000))
    adv = (0.7, -1.3) if eq == "advection" else ()
    model = P.EquationModel(eq, 2, advection_speed=adv)
    sc = O.Scheme(dim=2, cells=(4, 4), deltas=(0.25, 0.25), eq=eq, adv=adv, flux="rusanov")
    for axis in range(2):
        assert np.array_equal(NM.rusanov_flux(model, NM.FacePair(uL, uR), axis), O.flux_rusanov(sc, uL, uR, axis))


@pytest.mark.parametrize("kind", ["weno2", "weno3"])
def test_weno_weights_and_faces_bitwise(NM, kind):
    import paper_1912_07645_b200 as P

    rng = np.random.default_rng(5)
    um, uc, up = (rng.standard_normal(20000) for _ in range(3))
    uc[::11] = um[::11]
    up[::13] = uc[::13]
    k = P.ReconstructionKind(kind)
    w0, w1 = NM.weno_weights(um, uc, up, k, 1e-6)
    d0, d1 = {"weno2": (0.5, 0.5), "weno3": (1.0 / 3.0, 2.0 / 3.0)}[kind]
    a0 = d0 / (1e-6 + (uc - um) ** 2) ** 2  # numerics.py:74-78
    a1 = d1 / (1e-6 + (up - uc) ** 2) ** 2
    assert np.array_equal(w0, a0 / (a0 + a1)) and np.array_equal(w1, a1 / (a0 + a1))
    assert np.array_equal(NM.weno_face_value(um, uc, up, k, 1e-6), O.weno_face(um, uc, up, kind, 1e-6))
    # reconstruct_axis on a padded 2D array, both axes
    data = rng.uniform(0.5, 1.5, (1, 12, 14))
    for ax, n in ((2, 10), (1, 8)):
        pair = NM.reconstruct_axis(data, ax, n, 2, P.Reconstruction(k))
        ref = O.faces_along(data, ax, n, 2, kind, 1e-6)
        assert np.array_equal(pair.uL, ref[0]) and np.array_equal(pair.uR, ref[1])


def test_errors(NM):
    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import errors as E

    model = P.EquationModel("euler", 2)
    # rho = inf is physical (p = 0.4 > floor) but has c = 0 and v = 0 on both
    # sides: sR - sL = 0 -> the reference raises (numerics.py:166-167)
    u = np.array([[np.inf], [0.0], [0.0], [1.0]])
    with pytest.raises(E.UnphysicalStateError, match=r"degenerate HLLC wave fan \(sL >= sR\)"):
        NM.hllc_flux(model, NM.FacePair(u, u), 0)
    # an unphysical state: physical_flux's check (equations.py:77-86), uL first
    good = _states(np.random.default_rng(1), 2, 6)
    bad = good.copy()
    bad[3, 4] = 0.0  # p < 0 at face 4 of uR
    with pytest.raises(E.UnphysicalStateError, match=r"unphysical state at cell \(4,\)"):
        NM.rusanov_flux(model, NM.FacePair(good, bad), 1)
    with pytest.raises(E.ConfigError, match="HLLC flux is only defined for the Euler equations"):
        NM.hllc_flux(P.EquationModel("burgers", 1), NM.FacePair(np.ones((1, 3)), np.ones((1, 3))), 0)
    with pytest.raises(E.ConfigError, match="weno_weights needs WENO2 or WENO3"):
        NM.weno_weights(1.0, 2.0, 3.0, P.ReconstructionKind.NONE)


def _reference():
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "conslaw").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import conslaw.numerics as RN

    return RN


def test_against_reference_package(NM):
    """The reference's own functions on the same inputs (baseline/_ref)."""
    RN = _reference()
    if RN is None:
        pytest.skip("baseline/_ref (the reference package) is not installed")
    from conslaw.equations import EquationModel as REM

    rng = np.random.default_rng(9)
    for dim in (1, 2, 3):
        uL, uR = _states(rng, dim, 3000), _states(rng, dim, 3000)
        for fk in (RN.FluxKind.HLLC, RN.FluxKind.RUSANOV):
            for axis in range(dim):
                ref = RN.numerical_flux(REM("euler", dim), fk, RN.FacePair(uL, uR), axis)
                got = NM.numerical_flux(REM("euler", dim), fk, NM.FacePair(uL, uR), axis)
                assert np.array_equal(got, ref)
    um, uc, up = (rng.standard_normal(5000) for _ in range(3))
    for k in (RN.ReconstructionKind.WENO2, RN.ReconstructionKind.WENO3):
        assert np.array_equal(NM.weno_face_value(um, uc, up, k, 1e-6), RN.weno_face_value(um, uc, up, k, 1e-6))
        for a, b in zip(NM.weno_weights(um, uc, up, k), RN.weno_weights(um, uc, up, k)):
            assert np.array_equal(a, b)
