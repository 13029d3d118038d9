"""Generate golden fixtures by running the REFERENCE `conslaw` package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Writes ``tests/golden/golden.json`` (fingerprints, dt sequences, scalars) and
``tests/golden/golden.npz`` (small input/output arrays).  Nothing on the GPU
box reads /root/reference; the committed fixtures travel instead.

Inputs are built through the reference's own ``parse_config`` +
``draw_sample`` + ``eval_init``; every case records
the SHA-256 prefix of ``final.interior.tobytes()`` plus the step records.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from conslaw import presets  # noqa: E402
from conslaw import solver as rsolver  # noqa: E402
from conslaw.equations import EquationModel  # noqa: E402
from conslaw.errors import ConslawError  # noqa: E402
from conslaw.grid import BoundaryKind, GridSpec, field_from_interior, fill_boundary  # noqa: E402
from conslaw.iodsl.config import parse_config  # noqa: E402
from conslaw.iodsl.expr import eval_expr, eval_init, parse_expr, print_expr  # noqa: E402
from conslaw.numerics import FluxKind, Reconstruction, ReconstructionKind  # noqa: E402
from conslaw.solver import SchemeConfig, run_simulation, spatial_residual, wave_speed_maxima  # noqa: E402
from conslaw.uq import (FieldMoments, MlmcPlan, SamplePlan, StructureFunctionAccumulator, draw_sample,  # noqa: E402
                        run_mc, run_mlmc)

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def edit(text: str, section: str, key: str, value: str) -> str:
    """Set ``key = value`` inside ``[section]`` of a preset text."""
    lines = text.splitlines()
    out, cur, done = [], None, False
    for ln in lines:
        s = ln.strip()
        if s.startswith("["):
            if cur == section and not done:
                out.append(f"{key} = {value}")
                done = True
            cur = s[1:-1]
        elif cur == section and s.split("=")[0].strip() == key:
            out.append(f"{key} = {value}")
            done = True
            continue
        out.append(ln)
    if not done:
        if cur != section:
            out.append(f"[{section}]")
        out.append(f"{key} = {value}")
    return "\n".join(out) + "\n"


def scheme_dict(grid: GridSpec, cfg: SchemeConfig) -> dict:
    m = cfg.model
    return {
        "dim": grid.dim,
        "cells": list(grid.cells),
        "deltas": list(grid.deltas),
        "eq": m.kind,
        "gamma": m.gamma,
        "adv": list(m.advection_speed),
        "flux": cfg.flux.value,
        "recon": cfg.recon.kind.value,
        "eps": cfg.recon.epsilon,
        "rk": cfg.rk_order,
        "cfl": cfg.cfl,
        "t_end": cfg.t_end,
        "bcs": [b.value for b in cfg.bc],
        "ghost": grid.ghost_width,
    }


BURGERS_QMC = """\
[grid]
cells = 2048 2048
origin = 0 0
extent = 1 1

[scheme]
equation = burgers
flux = rusanov
reconstruction = weno2
rk_order = 3
cfl = 0.475
t_end = 0.02
boundary = periodic

[initial]
variables = scalar
u = 1.0 + 0.5 * sin(2 * pi * (x + X0)) * sin(2 * pi * (y + X1))

[uq]
method = qmc
samples = 256
stochastic_dim = 2
functionals = moments structure_function
structure_p = 2
structure_max_offset = 8
"""

# near-vacuum double rarefaction: exercises the positivity fallback
DOUBLE_RAREFACTION = """\
[grid]
cells = 200
[scheme]
equation = euler
flux = hllc
reconstruction = weno3
rk_order = 2
cfl = 0.475
t_end = 0.15
boundary = outflow
[initial]
variables = primitive
rho = 1.0
vx = x < 0.5 ? -2.0 : 2.0
p = 0.4
"""

SMOOTH_BURGERS_1D = """\
[grid]
cells = 96
[scheme]
equation = burgers
flux = rusanov
reconstruction = {recon}
rk_order = {rk}
cfl = 0.4
t_end = 0.5
boundary = {bc}
[initial]
variables = scalar
u = 0.5 + sin(2 * pi * x) + 0.25 * cos(6 * pi * x)
"""

ADVECTION_2D = """\
[grid]
cells = 24 20
extent = 1 2
[scheme]
equation = advection
advection_speed = 1.0 -0.5
flux = rusanov
reconstruction = {recon}
rk_order = {rk}
t_end = 0.3
boundary = periodic
[initial]
variables = scalar
u = exp(-20 * ((x - 0.5) ^ 2 + (y - 1) ^ 2)) + (x < 0.3 ? 1 : 0)
"""

EULER_2D_BLAST = """\
[grid]
cells = 40 32
[scheme]
equation = euler
flux = {flux}
reconstruction = {recon}
rk_order = {rk}
cfl = 0.45
t_end = 0.05
boundary = {bc}
[initial]
variables = primitive
rho = 1.0 + 0.2 * sin(2 * pi * x) * cos(2 * pi * y)
vx = 0.3 * sin(2 * pi * y)
vy = -0.2 * cos(2 * pi * x)
p = (x - 0.5) ^ 2 + (y - 0.5) ^ 2 < 0.04 ? 10.0 : 0.1
"""

EULER_3D = """\
[grid]
cells = 12 10 8
extent = 1.2 1 0.8
[scheme]
equation = euler
flux = {flux}
reconstruction = {recon}
rk_order = {rk}
t_end = 0.04
boundary = {bc}
[initial]
variables = primitive
rho = 1.0 + 0.3 * sin(2 * pi * x) * sin(2 * pi * z)
vx = 0.2
vy = -0.1 * cos(2 * pi * y)
vz = 0.15 * sin(2 * pi * (x + y))
p = 1.0 + 0.1 * cos(2 * pi * (x - z))
"""

SCALAR_3D = """\
[grid]
cells = 14 12 10
extent = 1 1.2 0.8
[scheme]
equation = {eq}
{speed}flux = rusanov
reconstruction = {recon}
rk_order = {rk}
cfl = 0.4
t_end = 0.08
boundary = {bc}
[initial]
variables = scalar
u = 0.6 + 0.5 * sin(2 * pi * x) * cos(2 * pi * y) + 0.3 * sin(2 * pi * z) + (x < 0.4 ? 0.5 : 0)
"""

EULER_3D_TILES = """\
[grid]
cells = 40 14 12
extent = 2 0.7 0.6
[scheme]
equation = euler
flux = hllc
reconstruction = weno2
rk_order = 3
t_end = 0.02
boundary = periodic
[initial]
variables = primitive
rho = 1.0 + 0.3 * sin(2 * pi * x) * sin(2 * pi * z / 0.6) + (y < 0.35 ? 0.5 : 0)
vx = 0.3 * cos(2 * pi * y / 0.7)
vy = -0.1 * cos(2 * pi * x)
vz = 0.15 * sin(2 * pi * (x + y))
p = 1.0 + 0.1 * cos(2 * pi * (x - z))
"""


def run_case(name, text, sample=0, max_steps=None, store=False, arrays=None, vec=None):
    rc = parse_config(text)
    if vec is None:
        plan = SamplePlan(rc.uq.method, rc.uq.samples, rc.uq.seed, rc.uq.stochastic_dim)
        vec = draw_sample(plan, sample)
    init = eval_init(rc.initial_exprs, rc.scheme.model, rc.grid, vec, primitive=rc.initial_primitive)
    fallbacks = [0]
    orig = rsolver._positivity_fallback

    def counting(model, sub, ax, n, g, pair):
        out = orig(model, sub, ax, n, g, pair)
        if out is not pair:
            fallbacks[0] += 1
        return out

    rsolver._positivity_fallback = counting
    try:
        final, recs = run_simulation(init, rc.scheme, max_steps=max_steps)
    finally:
        rsolver._positivity_fallback = orig
    case = {
        "name": name,
        "config": text,
        "vector": [float(v) for v in vec],
        "scheme": scheme_dict(rc.grid, rc.scheme),
        "max_steps": max_steps,
        "init_sha": sha(init.interior),
        "final_sha": sha(final.interior),
        "data_sha": sha(final.data),
        "steps": len(recs),
        "t": recs[-1].t if recs else 0.0,
        "dts": [r.dt for r in recs[:8]],
        "dt_sha": sha(np.array([r.dt for r in recs])),
        "fallback_stages": fallbacks[0],
        "sum_final": [float(s) for s in final.interior.reshape(final.ncomp, -1).sum(axis=1)],
        # the initial-data program, for the device evaluator (initdev.py)
        "init_exprs": [print_expr(e) for e in rc.initial_exprs],
        "primitive": bool(rc.initial_primitive),
        "origin": [float(o) for o in rc.grid.origin],
    }
    if store and arrays is not None:
        arrays[f"{name}__init"] = np.asarray(init.data)
        arrays[f"{name}__final"] = np.asarray(final.data)
        arrays[f"{name}__dt"] = np.array([r.dt for r in recs])
    print(f"{name}: steps={case['steps']} final={case['final_sha']} fallbacks={fallbacks[0]}")
    return case


EXPR_TEXTS = [
    "1 + 2*x", "-x^2", "(y < 0.25 + 0.01*sin(2*pi*x)) ? 2 : 1", "max(x, -y) ^ 0.5 / exp(-X0)",
    "1 < 2 == 3 >= 4", "2^3^2", "-(-x)", "x ? y ? 1 : 2 : z", ".5e-3*x - 3e2", "abs(min(1,2))",
    "x^-1 + (x - 0.5)^2 * y^0.5", "cos(x) != sin(y) ? sqrt(abs(x - y)) : -1.5e+1", "X3 * (X1 - 0.5) <= x",
    "((x))", "1 - 2 - 3 / 4 / 5 * 6",
]


def expr_cases():
    """Parser / printer fingerprints and pointwise values of the reference's
    expression language (iodsl/expr.py) on a few points."""
    xs = np.array([0.1, 0.37, 0.5, 0.81])
    env = {"x": xs, "y": xs[::-1].copy(), "z": xs * 0.5, "X0": 0.3, "X1": 0.7, "X2": 0.1, "X3": 0.9}
    out = []
    for t in EXPR_TEXTS:
        node = parse_expr(t)
        val = np.broadcast_to(np.asarray(eval_expr(node, env), dtype=float), xs.shape)
        out.append({"text": t, "print": print_expr(node), "repr": repr(node).replace("conslaw.iodsl.expr.", ""),
                    "values": [float(v) for v in val]})
    return out


def residual_cases(arrays):
    """spatial_residual / wave_speed_maxima on random physical fields."""
    rng = np.random.default_rng(1912)
    out = []
    specs = []
    for dim, cells in ((1, (37,)), (2, (13, 11)), (3, (7, 6, 5))):
        for eq in ("euler", "burgers", "advection"):
            for flux in ("rusanov", "hllc"):
                if flux == "hllc" and eq != "euler":
                    continue
                for recon in ("none", "weno2", "weno3"):
                    for bc in ("periodic", "outflow"):
                        specs.append((dim, cells, eq, flux, recon, bc))
    for i, (dim, cells, eq, flux, recon, bc) in enumerate(specs):
        adv = tuple([0.7, -1.3, 0.4][:dim]) if eq == "advection" else ()
        model = EquationModel(eq, dim, gamma=1.4, advection_speed=adv)
        recon_o = Reconstruction(ReconstructionKind(recon))
        g = max(recon_o.radius, 1)
        grid = GridSpec(dim, cells, (0.0,) * dim, tuple(1.0 + 0.1 * k for k in range(dim)), ghost_width=g)
        cfg = SchemeConfig(model, FluxKind(flux), recon_o, rk_order=2, bc=(BoundaryKind(bc),) * dim)
        shape = (model.ncomp,) + grid.interior_shape
        if eq == "euler":
            rho = 0.5 + rng.random(shape[1:])
            vel = rng.standard_normal((dim,) + shape[1:]) * 0.7
            p = 0.2 + rng.random(shape[1:])
            u = np.empty(shape)
            u[0] = rho
            kin = np.zeros_like(rho)
            for k in range(dim):
                u[1 + k] = rho * vel[k]
                kin = kin + vel[k] ** 2
            u[1 + dim] = p / 0.4 + 0.5 * rho * kin
        else:
            u = rng.standard_normal(shape)
        # some equal neighbouring states so the F(u,u) = f(u) branch is hit
        flat = u.reshape(u.shape[0], -1)
        flat[:, 3] = flat[:, 2]
        f = field_from_interior(grid, u)
        fill_boundary(f, cfg.bc)
        L = spatial_residual(f, cfg)
        mx = wave_speed_maxima(f, cfg)
        name = f"res{i:02d}_{dim}d_{eq}_{flux}_{recon}_{bc}"
        arrays[name + "__u"] = np.asarray(f.data)
        arrays[name + "__L"] = L
        arrays[name + "__max"] = mx
        out.append({
            "name": name,
            "scheme": scheme_dict(grid, cfg),
            "L_sha": sha(L),
            "max": [float(v) for v in mx],
            "filled_sha": sha(f.data),
        })
    print(f"{len(out)} residual cases")
    return out


def error_cases():
    out = []
    # unphysical initial state -> SimulationError
    txt = SMOOTH_BURGERS_1D.format(recon="none", rk=1, bc="periodic")
    rc = parse_config(txt)
    model = EquationModel("euler", 1)
    grid = GridSpec(1, (8,), (0.0,), (1.0,), ghost_width=1)
    cfg = SchemeConfig(model, FluxKind.HLLC, Reconstruction(), rk_order=1, t_end=0.1,
                       bc=(BoundaryKind.PERIODIC,))
    u = np.zeros((3, 8))
    u[0] = 1.0
    u[2] = 2.5
    u[0, 5] = -1.0
    try:
        run_simulation(field_from_interior(grid, u), cfg)
        kind, msg = None, None
    except ConslawError as e:
        kind, msg = type(e).__name__, str(e)
    out.append({"name": "unphysical_init", "kind": kind, "msg": msg})
    # static field -> StaticFieldError
    model = EquationModel("burgers", 2)
    grid = GridSpec(2, (6, 5), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = SchemeConfig(model, FluxKind.RUSANOV, Reconstruction(ReconstructionKind.WENO2), rk_order=3,
                       t_end=0.1, bc=(BoundaryKind.PERIODIC,) * 2)
    try:
        run_simulation(field_from_interior(grid, np.zeros((1, 5, 6))), cfg)
        kind, msg = None, None
    except ConslawError as e:
        kind, msg = type(e).__name__, str(e)
    out.append({"name": "static_field", "kind": kind, "msg": msg})
    # overflow to inf/nan -> SimulationError "non-finite value after step"
    model = EquationModel("burgers", 1)
    grid = GridSpec(1, (16,), (0.0,), (1.0,), ghost_width=1)
    cfg = SchemeConfig(model, FluxKind.RUSANOV, Reconstruction(), rk_order=1, t_end=1.0,
                       bc=(BoundaryKind.PERIODIC,))
    u = np.ones((1, 16))
    u[0, 9] = 1e200
    try:
        run_simulation(field_from_interior(grid, u), cfg)
        kind, msg = None, None
    except ConslawError as e:
        kind, msg = type(e).__name__, str(e)
    out.append({"name": "nonfinite", "kind": kind, "msg": msg})
    for c in out:
        print(c)
    return out


def uq_case(name, text, samples, t_end, cells):
    txt = edit(text, "grid", "cells", cells)
    txt = edit(txt, "scheme", "t_end", repr(t_end))
    txt = edit(txt, "scheme", "reconstruction", "weno2")
    txt = edit(txt, "uq", "samples", str(samples))
    rc = parse_config(txt)
    plan = SamplePlan(rc.uq.method, rc.uq.samples, rc.uq.seed, rc.uq.stochastic_dim)

    def ev(grid, vec):
        return eval_init(rc.initial_exprs, rc.scheme.model, grid, vec, primitive=rc.initial_primitive)

    fm = FieldMoments(rc.grid, rc.scheme.model.ncomp)
    sf = StructureFunctionAccumulator(rc.uq.structure_p, rc.uq.structure_max_offset,
                                      rc.uq.structure_component)
    merged = run_mc(plan, rc.grid, rc.scheme, ev, [fm, sf])
    m, s = merged
    var = m.acc.variance(ddof=1)
    case = {
        "name": name,
        "config": txt,
        "method": rc.uq.method,
        "seed": rc.uq.seed,
        "samples": samples,
        "stochastic_dim": rc.uq.stochastic_dim,
        "scheme": scheme_dict(rc.grid, rc.scheme),
        "mean_sha": sha(m.acc.mean),
        "var_sha": sha(var),
        "m2_sha": sha(m.acc.m2),
        "max_var0": float(var[0].max()),
        "sf": [float(v) for v in s.values()],
        "sf_sums": [float(v) for v in s.sums],
        "sf_p": rc.uq.structure_p,
        "sf_H": rc.uq.structure_max_offset,
        "vectors": [[float(v) for v in draw_sample(plan, k)] for k in range(samples)],
    }
    print(f"{name}: mean={case['mean_sha']} var={case['var_sha']} sf1={case['sf'][1]}")
    return case


def histogram_case():
    """run_mc with a point-PDF Histogram functional (uq.py:181-228)."""
    from conslaw.uq import Histogram

    txt = edit(edit(edit(presets.KH2D, "grid", "cells", "128 128"), "scheme", "t_end", "0.01"),
               "scheme", "reconstruction", "weno2")
    rc = parse_config(txt)
    plan = SamplePlan("mc", 8, 42, 4)

    def ev(grid, vec):
        return eval_init(rc.initial_exprs, rc.scheme.model, grid, vec, primitive=rc.initial_primitive)

    probes = ((64, 32), (10, 96), (127, 0), (64, 64))
    h = Histogram(probes, 0, 0.9, 2.1, 12)
    (res,) = run_mc(plan, rc.grid, rc.scheme, ev, [h])
    return {"probes": [list(p) for p in probes], "component": 0, "lo": 0.9, "hi": 2.1, "bins": 12,
            "counts": res.counts.tolist(), "samples": res.samples, "scheme": scheme_dict(rc.grid, rc.scheme)}


def mlmc_cases():
    """run_mlmc (uq.py:348-419): a 2-level KH2D hierarchy and the 1-level
    degenerate case (bitwise equal to run_mc)."""
    out = []
    base = edit(edit(presets.KH2D, "scheme", "reconstruction", "weno2"), "scheme", "t_end", "0.01")
    for name, cells, spl, method in (("kh2d_mlmc_2lvl", ("64 64", "128 128"), (4, 2), "mc"),
                                     ("kh2d_mlmc_1lvl", ("128 128",), (3,), "mc"),
                                     ("kh2d_mlmc_qmc_2lvl", ("64 64", "128 128"), (3, 2), "qmc")):
        rcs = [parse_config(edit(base, "grid", "cells", c)) for c in cells]
        grids = tuple(rc.grid for rc in rcs)
        plan = MlmcPlan(grids, spl, method=method, seed=42, stochastic_dim=4)
        rc0 = rcs[-1]

        def make_cfg(grid, rc0=rc0):
            return rc0.scheme

        def ev(grid, vec, rc0=rc0):
            return eval_init(rc0.initial_exprs, rc0.scheme.model, grid, vec, primitive=rc0.initial_primitive)

        res = run_mlmc(plan, make_cfg, ev)
        out.append({"name": name, "cells": [list(g.cells) for g in grids], "samples": list(spl), "method": method,
                    "seed": 42, "stochastic_dim": 4, "scheme": scheme_dict(grids[-1], rc0.scheme),
                    "mean_sha": sha(res.mean), "second_sha": sha(res.second_moment), "var_sha": sha(res.variance),
                    "mean_sum": float(res.mean.sum()), "var_sum": float(res.variance.sum())})
        print(name, out[-1]["mean_sha"], out[-1]["var_sha"])
    return out


def main():
    arrays: dict = {}
    gold: dict = {"numpy": np.__version__, "runs": [], "residuals": [], "errors": [], "uq": []}
    runs = gold["runs"]

    sod = edit(presets.SOD, "grid", "cells", "1024")
    sod = edit(sod, "scheme", "reconstruction", "none")
    sod = edit(sod, "scheme", "rk_order", "1")
    sod = edit(sod, "scheme", "cfl", "0.4")
    runs.append(run_case("sod1024_c1", sod, store=True, arrays=arrays))
    runs.append(run_case("sod400_preset", presets.SOD, store=True, arrays=arrays))
    runs.append(run_case("advection_smooth_preset", edit(presets.ADVECTION_SMOOTH, "scheme", "t_end", "0.1"),
                         store=True, arrays=arrays))
    runs.append(run_case("double_rarefaction", DOUBLE_RAREFACTION, store=True, arrays=arrays))

    kh = edit(presets.KH2D, "scheme", "reconstruction", "weno2")
    runs.append(run_case("kh2d64_weno2_50", kh, max_steps=50, store=True, arrays=arrays))
    kh32 = edit(presets.KH2D, "grid", "cells", "32 32")
    runs.append(run_case("kh2d32_weno3_20", kh32, max_steps=20, sample=3, store=True, arrays=arrays))
    kh128 = edit(presets.KH2D, "grid", "cells", "128 128")
    kh128 = edit(kh128, "scheme", "reconstruction", "weno2")
    runs.append(run_case("kh2d128_weno2_10", kh128, max_steps=10, store=False, arrays=arrays))
    kh3 = edit(presets.KH3D, "grid", "cells", "16 16 16")
    kh3 = edit(kh3, "scheme", "reconstruction", "weno2")
    runs.append(run_case("kh3d16_weno2_5", kh3, max_steps=5, store=True, arrays=arrays))
    runs.append(run_case("kh3d8_weno3_full", edit(edit(presets.KH3D, "grid", "cells", "8 8 8"),
                                                   "scheme", "t_end", "0.05"), store=True, arrays=arrays))
    bq = edit(BURGERS_QMC, "grid", "cells", "64 64")
    runs.append(run_case("burgers2d64_qmc0", bq, store=True, arrays=arrays))
    for recon in ("none", "weno2", "weno3"):
        for rk in (1, 2, 3):
            for bc in ("periodic", "outflow"):
                nm = f"burgers1d_{recon}_rk{rk}_{bc}"
                runs.append(run_case(nm, SMOOTH_BURGERS_1D.format(recon=recon, rk=rk, bc=bc),
                                     store=True, arrays=arrays))
    for recon in ("none", "weno3"):
        for rk in (2, 3):
            nm = f"advection2d_{recon}_rk{rk}"
            runs.append(run_case(nm, ADVECTION_2D.format(recon=recon, rk=rk), store=True, arrays=arrays))
    for flux in ("hllc", "rusanov"):
        for recon in ("none", "weno2", "weno3"):
            for bc in ("periodic", "outflow"):
                rk = {"none": 1, "weno2": 2, "weno3": 3}[recon]
                nm = f"euler2d_{flux}_{recon}_{bc}"
                runs.append(run_case(nm, EULER_2D_BLAST.format(flux=flux, recon=recon, rk=rk, bc=bc),
                                     store=True, arrays=arrays))
    for flux, recon, bc in (("hllc", "weno3", "periodic"), ("rusanov", "weno2", "outflow"),
                            ("hllc", "none", "outflow")):
        nm = f"euler3d_{flux}_{recon}_{bc}"
        runs.append(run_case(nm, EULER_3D.format(flux=flux, recon=recon, rk=3, bc=bc),
                             store=True, arrays=arrays))

    # 3D scalar laws and a multi-tile / multi-chunk 3D Euler domain (the 3D
    # ring kernel's one-component instantiations, tile seams, chunk seams)
    for eq, recon, rk, bc in (("burgers", "weno2", 3, "periodic"), ("burgers", "weno3", 2, "outflow"),
                              ("burgers", "none", 1, "periodic"), ("advection", "weno3", 3, "periodic"),
                              ("advection", "none", 2, "outflow")):
        nm = f"{eq}3d_{recon}_rk{rk}_{bc}"
        runs.append(run_case(nm, SCALAR_3D.format(
            eq=eq, recon=recon, rk=rk, bc=bc, speed="advection_speed = 0.7 -0.4 0.5\n" if eq == "advection" else ""), store=True, arrays=arrays))
    runs.append(run_case("euler3d_tiles_hllc_weno2", EULER_3D_TILES, store=True, arrays=arrays))

    gold["exprs"] = expr_cases()
    gold["residuals"] = residual_cases(arrays)
    gold["errors"] = error_cases()

    gold["uq"].append(uq_case("kh2d128_mc8", presets.KH2D, 8, 0.01, "128 128"))
    kq = edit(presets.KH2D, "uq", "method", "qmc")
    gold["uq"].append(uq_case("kh2d128_qmc8", kq, 8, 0.01, "128 128"))
    gold["uq"].append(uq_case("burgers128_qmc8", BURGERS_QMC, 8, 0.02, "128 128"))

    gold["mlmc"] = mlmc_cases()
    gold["histogram"] = histogram_case()

    mc = SamplePlan("mc", 8, 42, 4)
    qmc = SamplePlan("qmc", 8, 42, 4)
    gold["samples"] = {
        "mc_seed42_dim4": [[float(v) for v in draw_sample(mc, k)] for k in range(8)],
        "qmc_dim4": [[float(v) for v in draw_sample(qmc, k)] for k in range(8)],
        "mc_seed7_dim16_k1000": [float(v) for v in draw_sample(SamplePlan("mc", 2000, 7, 16), 1000)],
        "qmc_dim16_k1000": [float(v) for v in draw_sample(SamplePlan("qmc", 2000, 7, 16), 1000)],
    }
    # KH2D initial data at the bench size: pins the product's initial-data code
    rc = parse_config(edit(edit(presets.KH2D, "grid", "cells", "1024 1024"), "scheme", "reconstruction", "weno2"))
    vec = draw_sample(SamplePlan("mc", 8, 42, 4), 0)
    init = eval_init(rc.initial_exprs, rc.scheme.model, rc.grid, vec)
    gold["kh2d1024_init_sha"] = sha(init.interior)
    rc3 = parse_config(edit(edit(presets.KH3D, "grid", "cells", "64 64 64"), "scheme", "reconstruction", "weno2"))
    init3 = eval_init(rc3.initial_exprs, rc3.scheme.model, rc3.grid, vec)
    gold["kh3d64_init_sha"] = sha(init3.interior)
    rcb = parse_config(edit(BURGERS_QMC, "grid", "cells", "256 256"))
    initb = eval_init(rcb.initial_exprs, rcb.scheme.model, rcb.grid, draw_sample(SamplePlan("qmc", 256, 0, 2), 5))
    gold["burgers256_qmc5_init_sha"] = sha(initb.interior)

    (OUT / "golden.json").write_text(json.dumps(gold, indent=1))
    np.savez_compressed(OUT / "golden.npz", **arrays)
    print("arrays:", len(arrays), "bytes:", (OUT / "golden.npz").stat().st_size)


if __name__ == "__main__":
    main()
