"""install_into(conslaw): make the reference package run its hot path on the
B200 implementation.

The reference binds solver names at import time (cli.py:25, uq.py:23,
parallel.py:33-40), so each module's binding is replaced, not just
conslaw.solver's.  Results are built with the reference's own classes
(TimeStepRecord, RankRecord, functionals) and errors are raised as the
reference's exception classes.
"""

from __future__ import annotations

import importlib

from . import errors as E
from . import numerics as _num
from . import parallel as _par
from . import solver as _sol
from . import uq as _uq


def install_into(pkg) -> dict:
    """Rebind the hot-path entry points of an imported ``conslaw`` package.
    Returns {qualified name: previous object} so callers can undo."""
    mods = {name: importlib.import_module(f"{pkg.__name__}.{name}")
            for name in ("solver", "uq", "parallel", "cli", "errors", "grid", "numerics")}
    saved = {}

    def bind(mod, attr, new):
        if hasattr(mod, attr):
            saved[f"{mod.__name__}.{attr}"] = getattr(mod, attr)
            setattr(mod, attr, new)

    for m in (pkg, mods["solver"], mods["uq"], mods["cli"]):
        bind(m, "run_simulation", _sol.run_simulation)
    bind(pkg, "stable_dt", _sol.stable_dt)
    bind(mods["solver"], "stable_dt", _sol.stable_dt)
    bind(mods["solver"], "spatial_residual", _sol.spatial_residual)
    bind(mods["solver"], "ssp_rk_step", _sol.ssp_rk_step)
    bind(mods["solver"], "wave_speed_maxima", _sol.wave_speed_maxima)
    bind(mods["grid"], "fill_boundary", _sol._device_fill_boundary)
    bind(pkg, "fill_boundary", _sol._device_fill_boundary)
    for m in (mods["parallel"], mods["cli"]):
        bind(m, "run_parallel", _par.run_parallel)
    for m in (mods["uq"], mods["cli"]):
        bind(m, "run_mc", _uq.run_mc)
        bind(m, "run_mlmc", _uq.run_mlmc)
    # the numerics function API and the flux registry seam (numerics.py:64-210):
    # device implementations, keyed by the reference's own FluxKind members
    nm = mods["numerics"]
    for attr in ("weno_weights", "weno_face_value", "reconstruct_axis", "reconstruct", "rusanov_flux",
                 "hllc_flux", "numerical_flux"):
        bind(nm, attr, getattr(_num, attr))
    if hasattr(nm, "FLUX_FUNCTIONS") and hasattr(nm, "FluxKind"):
        saved[f"{nm.__name__}.FLUX_FUNCTIONS"] = dict(nm.FLUX_FUNCTIONS)
        nm.FLUX_FUNCTIONS[nm.FluxKind.RUSANOV] = _num.rusanov_flux
        nm.FLUX_FUNCTIONS[nm.FluxKind.HLLC] = _num.hllc_flux
    # result / error classes of the reference
    _sol.TYPES["TimeStepRecord"] = mods["solver"].TimeStepRecord
    _sol.TYPES["Field"] = mods["grid"].Field
    _par.RankRecord = mods["parallel"].RankRecord
    for cls in ("ConfigError", "UnphysicalStateError", "SimulationError", "StaticFieldError", "ProtocolError",
                "ConslawError", "ExprError"):
        setattr(E, cls, getattr(mods["errors"], cls))
    return saved
