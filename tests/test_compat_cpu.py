"""install_into rebinds every import-time binding of the hot path in the
reference package (CPU: no compute).  Skipped where the reference is absent
(the GPU box)."""
import importlib
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference package not present")
def test_install_into_rebinds():
    sys.path.insert(0, str(REF))
    try:
        import conslaw
        import conslaw.cli
        import conslaw.parallel
        import conslaw.solver
        import conslaw.uq

        import paper_1912_07645_b200 as fvb
        from paper_1912_07645_b200 import compat, errors, parallel, solver, uq

        names = ("ConfigError", "UnphysicalStateError", "SimulationError", "StaticFieldError", "ProtocolError",
                 "ConslawError")
        orig_errors = {n: getattr(errors, n) for n in names}
        saved = compat.install_into(conslaw)
        try:
            assert conslaw.solver.run_simulation is fvb.run_simulation
            assert conslaw.uq.run_simulation is fvb.run_simulation
            assert conslaw.cli.run_simulation is fvb.run_simulation
            assert conslaw.cli.run_parallel is parallel.run_parallel
            assert conslaw.cli.run_mc is uq.run_mc
            assert conslaw.solver.spatial_residual is solver.spatial_residual
            assert errors.SimulationError is conslaw.errors.SimulationError
            assert solver.TYPES["TimeStepRecord"] is conslaw.solver.TimeStepRecord
        finally:
            for qual, obj in saved.items():
                mod, attr = qual.rsplit(".", 1)
                setattr(importlib.import_module(mod), attr, obj)
            for n, cls in orig_errors.items():
                setattr(errors, n, cls)
            solver.TYPES["TimeStepRecord"] = solver.TimeStepRecord
            solver.TYPES["Field"] = None
    finally:
        sys.path.remove(str(REF))
        for m in [m for m in sys.modules if m == "conslaw" or m.startswith("conslaw.")]:
            del sys.modules[m]
