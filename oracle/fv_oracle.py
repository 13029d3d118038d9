"""CPU oracle for the finite-volume stage hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `conslaw` algorithm for
the path the B200 build replaces.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it, and there only as
the checker or the timed CPU baseline.  The product path
(``paper_1912_07645_b200``) never imports it.

Parity pin: every function follows the reference operation by operation
(numpy evaluates each binary op as one IEEE-754 binary64 pass, no FMA), so the
oracle is bitwise equal to the reference.  That claim is checked against the
golden fingerprints in ``tests/golden/golden.json`` produced by importing the
reference itself (``tests/golden/make_golden.py``) -- see
``tests/test_oracle_golden.py``.

Citations are ``/root/reference/pkg/src/conslaw/<file>:<line>``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import numpy as np

FLOOR = 1e-12  # equations.py:20


class OracleError(Exception):
    """Raised where the reference raises; ``kind`` names the reference class."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


@dataclass
class Scheme:
    """Flat description of one run (SchemeConfig + GridSpec + EquationModel).

    ``eq`` in {"euler", "burgers", "advection"}; ``flux`` in {"hllc",
    "rusanov"}; ``recon`` in {"none", "weno2", "weno3"}; ``bcs`` entries in
    {"periodic", "outflow"} (x first).
    """

    dim: int
    cells: tuple
    deltas: tuple
    eq: str = "euler"
    gamma: float = 1.4
    adv: tuple = ()
    flux: str = "rusanov"
    recon: str = "none"
    eps: float = 1e-6
    rk: int = 2
    cfl: float = 0.475
    t_end: float = 1.0
    bcs: tuple = ()
    ghost: int = dc_field(default=0)

    def __post_init__(self):
        if not self.bcs:
            self.bcs = ("periodic",) * self.dim
        if self.ghost == 0:
            self.ghost = max(self.radius, 1)  # iodsl/config.py:359

    @property
    def ncomp(self) -> int:
        return self.dim + 2 if self.eq == "euler" else 1  # equations.py:51-53

    @property
    def radius(self) -> int:
        return 1 if self.recon == "none" else 2  # numerics.py:45-47

    def np_axis(self, axis: int) -> int:
        return 1 + (self.dim - 1 - axis)  # grid.py:28-30


def _cut(nd, ax, lo, hi):
    s = [slice(None)] * nd
    s[ax] = slice(lo, hi)
    return tuple(s)


# ---------------------------------------------------------------------------
# ghost fill  (grid.py:147-175)
# ---------------------------------------------------------------------------

def ghost_fill(data: np.ndarray, sc: Scheme) -> np.ndarray:
    g = sc.ghost
    nd = data.ndim
    for axis in range(sc.dim):
        n = sc.cells[axis]
        ax = sc.np_axis(axis)
        if sc.bcs[axis] == "periodic":
            if n < g:
                raise OracleError("ConfigError", "periodic axis shorter than ghost width")
            data[_cut(nd, ax, 0, g)] = data[_cut(nd, ax, n, n + g)]
            data[_cut(nd, ax, n + g, n + 2 * g)] = data[_cut(nd, ax, g, 2 * g)]
        else:
            data[_cut(nd, ax, 0, g)] = data[_cut(nd, ax, g, g + 1)]
            data[_cut(nd, ax, n + g, n + 2 * g)] = data[_cut(nd, ax, n + g - 1, n + g)]
    return data


def interior(data: np.ndarray, sc: Scheme) -> np.ndarray:
    g = sc.ghost
    return data[(slice(None),) + tuple(slice(g, g + n) for n in reversed(sc.cells))]


def padded_from_interior(sc: Scheme, inner: np.ndarray) -> np.ndarray:
    shape = (inner.shape[0],) + tuple(n + 2 * sc.ghost for n in reversed(sc.cells))
    out = np.zeros(shape)
    interior(out, sc)[...] = inner
    return out


# ---------------------------------------------------------------------------
# equation of state and physics  (equations.py:62-129)
# ---------------------------------------------------------------------------

def euler_pressure(sc: Scheme, u):
    # Python's sum() starts from int 0: 0 + m0^2 is exact  (equations.py:65)
    msq = 0
    for k in range(sc.dim):
        msq = msq + u[1 + k] ** 2
    return (sc.gamma - 1.0) * (u[1 + sc.dim] - msq / (2.0 * u[0]))


def physical(sc: Scheme, u):
    if sc.eq != "euler":
        return np.ones(np.shape(u)[1:], dtype=bool)
    return (u[0] > FLOOR) & (euler_pressure(sc, u) > FLOOR)


def _assert_physical(sc: Scheme, u):
    ok = np.atleast_1d(physical(sc, u))
    if not ok.all():
        raise OracleError("UnphysicalStateError", "unphysical state")


def phys_flux(sc: Scheme, u, axis: int, check: bool = True):
    u = np.asarray(u, dtype=float)
    if sc.eq == "burgers":
        return 0.5 * u * u
    if sc.eq == "advection":
        return sc.adv[axis] * u
    if check:
        _assert_physical(sc, u)
    vel = u[1 + axis] / u[0]
    p = euler_pressure(sc, u)
    f = np.empty_like(u)
    f[0] = u[1 + axis]
    for j in range(sc.dim):
        f[1 + j] = u[1 + j] * vel
    f[1 + axis] = f[1 + axis] + p
    f[1 + sc.dim] = (u[1 + sc.dim] + p) * vel
    return f


def wave_speed(sc: Scheme, u, axis: int, check: bool = True):
    u = np.asarray(u, dtype=float)
    if sc.eq == "burgers":
        return np.abs(u[0])
    if sc.eq == "advection":
        return np.broadcast_to(abs(sc.adv[axis]), u.shape[1:]).copy()
    if check:
        _assert_physical(sc, u)
    c = np.sqrt(sc.gamma * euler_pressure(sc, u) / u[0])
    return np.abs(u[1 + axis] / u[0]) + c


def sound(sc: Scheme, u):
    return np.sqrt(sc.gamma * euler_pressure(sc, u) / u[0])


# ---------------------------------------------------------------------------
# reconstruction  (numerics.py:51-118)
# ---------------------------------------------------------------------------

_IDEAL = {"weno2": (0.5, 0.5), "weno3": (1.0 / 3.0, 2.0 / 3.0)}


def weno_face(um, uc, up, kind: str, eps: float):
    d0, d1 = _IDEAL[kind]
    b0 = (uc - um) ** 2
    b1 = (up - uc) ** 2
    a0 = d0 / (eps + b0) ** 2
    a1 = d1 / (eps + b1) ** 2
    s = a0 + a1
    w0, w1 = a0 / s, a1 / s
    return uc + 0.5 * (w0 * (uc - um) + w1 * (up - uc))


def faces_along(data, ax: int, n: int, g: int, recon: str, eps: float):
    """(uL, uR) at the n+1 interfaces; interface j between padded g-1+j, g+j."""
    nd = data.ndim

    def sh(k):  # padded cells g-1+k+j for j = 0..n
        return data[_cut(nd, ax, g - 1 + k, g + n + k)]

    if recon == "none":
        return sh(0), sh(1)
    left = weno_face(sh(-1), sh(0), sh(1), recon, eps)
    right = weno_face(sh(2), sh(1), sh(0), recon, eps)
    return left, right


# ---------------------------------------------------------------------------
# numerical fluxes  (numerics.py:133-196)
# ---------------------------------------------------------------------------

def flux_rusanov(sc: Scheme, uL, uR, axis):
    fL = phys_flux(sc, uL, axis)
    fR = phys_flux(sc, uR, axis)
    s = np.maximum(wave_speed(sc, uL, axis, False), wave_speed(sc, uR, axis, False))
    return 0.5 * (fL + fR) - 0.5 * s * (uR - uL)


def flux_hllc(sc: Scheme, uL, uR, axis):
    if sc.eq != "euler":
        raise OracleError("ConfigError", "HLLC needs Euler")
    uL = np.asarray(uL, dtype=float)
    uR = np.asarray(uR, dtype=float)
    fL = phys_flux(sc, uL, axis)
    fR = phys_flux(sc, uR, axis)
    d = sc.dim
    rL, rR = uL[0], uR[0]
    vL = uL[1 + axis] / rL
    vR = uR[1 + axis] / rR
    pL = euler_pressure(sc, uL)
    pR = euler_pressure(sc, uR)
    cL = sound(sc, uL)
    cR = sound(sc, uR)
    sL = np.minimum(vL - cL, vR - cR)
    sR = np.maximum(vL + cL, vR + cR)
    if np.any(sR - sL <= 0):
        raise OracleError("UnphysicalStateError", "degenerate HLLC wave fan")
    den = rL * (sL - vL) - rR * (sR - vR)
    sM = (pR - pL + rL * vL * (sL - vL) - rR * vR * (sR - vR)) / den

    def star(u, rho, v, p, E, sK):
        fac = rho * (sK - v) / (sK - sM)
        st = np.empty_like(u)
        st[0] = fac
        for j in range(d):
            st[1 + j] = fac * (u[1 + j] / rho)
        st[1 + axis] = fac * sM
        st[1 + d] = fac * (E / rho + (sM - v) * (sM + p / (rho * (sK - v))))
        return st

    with np.errstate(all="ignore"):
        FsL = fL + sL * (star(uL, rL, vL, pL, uL[1 + d], sL) - uL)
        FsR = fR + sR * (star(uR, rR, vR, pR, uR[1 + d], sR) - uR)
    out = np.where(sL >= 0, fL, np.where(sM >= 0, FsL, np.where(sR > 0, FsR, fR)))
    same = np.all(uL == uR, axis=0)
    return np.where(same, fL, out)


_FLUX = {"rusanov": flux_rusanov, "hllc": flux_hllc}


# ---------------------------------------------------------------------------
# residual, CFL, SSP-RK, driver  (solver.py:82-246)
# ---------------------------------------------------------------------------

def residual(data: np.ndarray, sc: Scheme) -> np.ndarray:
    """Interior time derivative of a ghost-filled padded array."""
    g = sc.ghost
    if sc.radius > g:
        raise OracleError("ConfigError", "ghost width too small")
    nd = data.ndim
    ok = physical(sc, interior(data, sc))
    if not ok.all():
        bad = tuple(int(i) for i in np.argwhere(~np.atleast_1d(ok))[0])
        raise OracleError("SimulationError", f"unphysical state in interior cell {bad}")
    L = np.zeros((data.shape[0],) + tuple(reversed(sc.cells)))
    fallback = sc.eq == "euler" and sc.recon != "none"
    for axis in range(sc.dim):
        ax = sc.np_axis(axis)
        sub = data
        for other in range(sc.dim):
            if other != axis:
                sub = sub[_cut(nd, sc.np_axis(other), g, g + sc.cells[other])]
        n = sc.cells[axis]
        uL, uR = faces_along(sub, ax, n, g, sc.recon, sc.eps)
        if fallback:
            good = physical(sc, uL) & physical(sc, uR)
            if not good.all():
                pL, pR = faces_along(sub, ax, n, g, "none", sc.eps)
                uL = np.where(good, uL, pL)
                uR = np.where(good, uR, pR)
        F = _FLUX[sc.flux](sc, uL, uR, axis)
        L -= (F[_cut(nd, ax, 1, None)] - F[_cut(nd, ax, None, -1)]) / sc.deltas[axis]
    return L


def speed_maxima(data: np.ndarray, sc: Scheme) -> np.ndarray:
    inner = interior(data, sc)
    return np.array([float(np.max(wave_speed(sc, inner, k))) for k in range(sc.dim)])


def cfl_dt(maxima, sc: Scheme, remaining=None) -> float:
    den = 0.0
    for k in range(sc.dim):
        den += maxima[k] / sc.deltas[k]
    if den == 0.0:
        raise OracleError("StaticFieldError", "static field: all wave speeds vanish")
    dt = sc.cfl / den
    if remaining is not None:
        dt = min(dt, remaining)
    return dt


def rk_combine(u, dt, L, order):
    """SSP-RK as convex combinations (solver.py:158-173)."""
    if order == 1:
        return u + dt * L(u)
    if order == 2:
        u1 = u + dt * L(u)
        return 0.5 * u + 0.5 * (u1 + dt * L(u1))
    u1 = u + dt * L(u)
    u2 = 0.75 * u + 0.25 * (u1 + dt * L(u1))
    return (1.0 / 3.0) * u + (2.0 / 3.0) * (u2 + dt * L(u2))


def step(data: np.ndarray, dt: float, sc: Scheme, fill=None, resid=None) -> np.ndarray:
    """One SSP-RK step on a padded array; returns a new padded array with
    zero ghosts (solver.py:176-196)."""
    fill = fill or (lambda a: ghost_fill(a, sc))
    resid = resid or residual

    def L(inner):
        a = padded_from_interior(sc, inner)
        fill(a)
        return resid(a, sc)

    return padded_from_interior(sc, rk_combine(interior(data, sc).copy(), dt, L, sc.rk))


def simulate(data: np.ndarray, sc: Scheme, max_steps=None):
    """run_simulation (solver.py:199-246): returns (padded final, [(step,t,dt)])."""
    if sc.radius > sc.ghost:
        raise OracleError("ConfigError", "ghost width too small")
    if not physical(sc, interior(data, sc)).all():
        raise OracleError("SimulationError", "initial field contains unphysical states")
    cur = data.copy()
    t = 0.0
    n = 0
    log = []
    while t < sc.t_end:
        rem = sc.t_end - t
        if rem <= 1e-14 * sc.t_end:
            break
        if max_steps is not None and n >= max_steps:
            break
        dt = cfl_dt(speed_maxima(cur, sc), sc, rem)
        cur = step(cur, dt, sc)
        n += 1
        t += dt
        inner = interior(cur, sc)
        if not np.isfinite(inner).all():
            bad = tuple(int(i) for i in np.argwhere(~np.isfinite(inner))[0][1:])
            raise OracleError("SimulationError", f"non-finite value after step {n} at cell {bad}")
        if not physical(sc, inner).all():
            raise OracleError("SimulationError", f"unphysical state after step {n}")
        log.append((n, t, dt))
    return cur, log


def simulate_fixed(data: np.ndarray, sc: Scheme, n_steps: int):
    """run_parallel's n_steps mode (parallel.py:490-520): dt is not capped by
    t_end and only finiteness is checked after each step."""
    cur = data.copy()
    t = 0.0
    log = []
    for n in range(1, n_steps + 1):
        dt = cfl_dt(speed_maxima(cur, sc), sc, None)
        cur = step(cur, dt, sc)
        t += dt
        if not np.isfinite(interior(cur, sc)).all():
            raise OracleError("SimulationError", f"non-finite value after step {n}")
        log.append((n, t, dt))
    return cur, log


# ---------------------------------------------------------------------------
# UQ statistics  (uq.py:114-273)
# ---------------------------------------------------------------------------

class Moments:
    """Per-cell count/mean/M2 merged one sample at a time (uq.py:135-148)."""

    def __init__(self, shape):
        self.count = 0
        self.mean = np.zeros(shape)
        self.m2 = np.zeros(shape)

    def push(self, value: np.ndarray):
        # a fresh accumulator updated with one value has count 1, mean v, m2 0
        # (uq.py:125-133 with count 0); merging it is uq.py:143-148.
        one_mean = np.zeros(value.shape) + (value - np.zeros(value.shape)) / 1
        one_m2 = np.zeros(value.shape) + (value - np.zeros(value.shape)) * (value - one_mean)
        if self.count == 0:
            self.count, self.mean, self.m2 = 1, one_mean.copy(), one_m2.copy()
            return
        tot = self.count + 1
        delta = one_mean - self.mean
        frac = 1 / tot
        self.mean = self.mean + delta * frac
        self.m2 = self.m2 + one_m2 + delta ** 2 * self.count * frac
        self.count = tot

    def merge(self, other: "Moments"):
        if other.count == 0:
            return
        if self.count == 0:
            self.count, self.mean, self.m2 = other.count, other.mean.copy(), other.m2.copy()
            return
        tot = self.count + other.count
        delta = other.mean - self.mean
        frac = other.count / tot
        self.mean = self.mean + delta * frac
        self.m2 = self.m2 + other.m2 + delta ** 2 * self.count * frac
        self.count = tot

    def variance(self, ddof=1):
        if self.count <= ddof:
            return np.zeros_like(self.m2)
        return self.m2 / (self.count - ddof)


def structure_sums(w: np.ndarray, p: float, H: int) -> np.ndarray:
    """Per-sample contribution to StructureFunctionAccumulator.sums
    (uq.py:254-262): for h, mean over numpy axes of |roll(w,-h) - w|^p."""
    out = np.zeros(H + 1)
    dim = w.ndim
    for h in range(H + 1):
        acc = 0.0
        for j in range(dim):
            acc += float(np.mean(np.abs(np.roll(w, -h, axis=j) - w) ** p))
        out[h] += acc / dim
    return out


# ---------------------------------------------------------------------------
# sampling (uq.py:79-106) -- needed to build identical inputs in tests
# ---------------------------------------------------------------------------

_PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53)


def sample_vector(method: str, seed: int, k: int, dim: int, level: int = 0) -> np.ndarray:
    if method == "qmc":
        out = []
        for b in _PRIMES[:dim]:
            idx, inv, f = k + 1, 0.0, 1.0 / b
            while idx > 0:
                inv += f * (idx % b)
                idx //= b
                f /= b
            out.append(inv)
        return np.array(out)
    key = [np.uint64(seed), np.uint64((level << 48) + k)]
    return np.random.Generator(np.random.Philox(key=key)).random(dim)


def mc_moments_and_sf(init_fn, sc: Scheme, method, seed, samples, sdim, p=2.0, H=8,
                      comp=0, want_sf=True):
    """run_mc (uq.py:302-322) for FieldMoments (+ structure function)."""
    mom = None
    sf = np.zeros(H + 1)
    for k in range(samples):
        vec = sample_vector(method, seed, k, sdim)
        final, _ = simulate(init_fn(vec), sc)
        inner = interior(final, sc)
        if mom is None:
            mom = Moments(inner.shape)
        mom.push(np.asarray(inner))
        if want_sf:
            sf += structure_sums(np.asarray(inner[comp]), p, H)
    return mom, sf


def sha16(a: np.ndarray) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def kelvin_helmholtz(cells, vec, gamma=1.4, ghost=2):
    """KH2D/KH3D preset initial data (presets.py:65-145) through the same
    numpy ops as iodsl/expr.py:271-316 + equations.py:132-145 (midpoint
    cell centres, grid.py:94-96)."""
    dim = len(cells)
    deltas = tuple(1.0 / n for n in cells)
    env = {}
    for axis, n in enumerate(cells):
        c = 0.0 + (np.arange(n) + 0.5) * deltas[axis]
        shape = [1] * dim
        shape[dim - 1 - axis] = n
        env["xyz"[axis]] = c.reshape(shape)
    x, y = env["x"], env["y"]
    shape = tuple(reversed(cells))
    two_pi = 2.0 * np.pi

    def iface(base, X):
        return base + 0.01 * np.sin(two_pi * (x + X))

    lo = np.less(y, iface(0.25, vec[0])).astype(float)
    hi = np.less(y, iface(0.75, vec[1])).astype(float)
    rho = np.where(lo != 0.0, 1.0, np.where(hi != 0.0, 2.0, 1.0))
    lo = np.less(y, iface(0.25, vec[2])).astype(float)
    hi = np.less(y, iface(0.75, vec[3])).astype(float)
    vx = np.where(lo != 0.0, -0.5, np.where(hi != 0.0, 0.5, -0.5))
    w = np.empty((dim + 2,) + shape)
    w[0] = np.broadcast_to(rho, shape)
    w[1] = np.broadcast_to(vx, shape)
    for k in range(1, dim):
        w[1 + k] = 0.0
    w[1 + dim] = 2.5
    u = np.empty_like(w)
    u[0] = w[0]
    kin = np.zeros_like(w[0])
    for k in range(dim):
        u[1 + k] = w[0] * w[1 + k]
        kin = kin + w[1 + k] ** 2
    u[1 + dim] = w[1 + dim] / (gamma - 1.0) + 0.5 * w[0] * kin
    sc_shape = (dim + 2,) + tuple(n + 2 * ghost for n in reversed(cells))
    out = np.zeros(sc_shape)
    out[(slice(None),) + tuple(slice(ghost, ghost + n) for n in shape)] = u
    return out


def burgers_sines(cells, vec, ghost=2):
    """Authored C5 initial data:
    u = 1.0 + 0.5 * sin(2 * pi * (x + X0)) * sin(2 * pi * (y + X1))."""
    dim = len(cells)
    deltas = tuple(1.0 / n for n in cells)
    x = (0.0 + (np.arange(cells[0]) + 0.5) * deltas[0]).reshape(1, cells[0])
    y = (0.0 + (np.arange(cells[1]) + 0.5) * deltas[1]).reshape(cells[1], 1)
    two_pi = 2.0 * np.pi
    v = 1.0 + 0.5 * np.sin(two_pi * (x + vec[0])) * np.sin(two_pi * (y + vec[1]))
    out = np.zeros((1,) + tuple(n + 2 * ghost for n in reversed(cells)))
    out[(slice(None),) + tuple(slice(ghost, ghost + n) for n in reversed(cells))] = v
    return out
