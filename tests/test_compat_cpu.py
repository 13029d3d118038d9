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


@pytest.mark.skipif(not REF.exists(), reason="reference package not present")
def test_uq_results_feed_reference_write_stats(tmp_path):
    """Row 24 boundary: run_mc hands back the caller's functional types, so
    the reference's write_stats (output.py:142-192, isinstance dispatch)
    consumes them unchanged.  The GPU accumulators are replaced by host
    stand-ins here (CPU test); the hand-back path is the product's."""
    import numpy as np

    sys.path.insert(0, str(REF))
    try:
        from conslaw.grid import GridSpec as RGrid
        from conslaw.iodsl.output import OutputHeader, write_stats
        from conslaw.uq import FieldMoments as RMoments
        from conslaw.uq import StructureFunctionAccumulator as RSF

        from paper_1912_07645_b200 import uq

        grid = RGrid(2, (4, 3), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
        slot_m = uq._Slot(RMoments(grid, 4), grid, 4)
        slot_s = uq._Slot(RSF(2.0, 3), grid, 4)

        class FakeMoments:
            acc = uq.MomentAccumulator((4, 3, 4))

        fm = FakeMoments()
        fm.acc.count = 3
        fm.acc.mean = np.arange(48.0).reshape(4, 3, 4)
        fm.acc.m2 = np.ones((4, 3, 4))
        slot_m.gpu = fm

        class FakeSF:
            sums = np.array([0.0, 1.0, 2.0, 3.0])
            samples = 3

        slot_s.gpu = FakeSF()
        res_m, res_s = slot_m.result(), slot_s.result()
        assert isinstance(res_m, RMoments) and isinstance(res_s, RSF)
        assert res_m.acc.count == 3 and np.array_equal(res_m.acc.variance(), np.ones((4, 3, 4)) / 2)
        assert list(res_s.values()) == [0.0, 1.0 / 3, 2.0 / 3, 1.0]
        header = OutputHeader(config_digest="0" * 64, seed=0)
        paths = write_stats([res_m, res_s], header, tmp_path)
        assert {p.name for p in paths} == {"mean.snap", "variance.snap", "structure_function.csv"}
    finally:
        sys.path.remove(str(REF))
        for m in [m for m in sys.modules if m == "conslaw" or m.startswith("conslaw.")]:
            del sys.modules[m]
