"""The reference's OWN test suite (147 tests: pkg/tests of the reference,
placed in baseline/_ref/conslaw_tests by tools/vendor_reference.sh) run
against the B200 path: compat.install_into(conslaw) rebinds the reference's
hot-path entry points (run_simulation, spatial_residual, ssp_rk_step,
stable_dt, fill_boundary, run_parallel, run_mc / run_mlmc, the numerics
functions and the FLUX_FUNCTIONS registry) before the test modules import
them, so reference-typed Fields, SchemeConfigs and functionals flow through
the CUDA kernels -- including cli.cmd_bench, the weak-scaling overhead
harness (acceptance criterion 8, test_acceptance.py:240-284), and
write_stats with the GPU run_mc's statistics."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref" / "conslaw_tests"


@pytest.mark.skipif(not SUITE.exists(), reason="baseline/_ref/conslaw_tests absent (tools/vendor_reference.sh)")
def test_reference_suite_through_the_shim(tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "baseline" / "_ref"), str(ROOT), str(SUITE),
                                        env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "tests.ref_shim_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(SUITE), "-o", "addopts="]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=tmp_path, env=env, timeout=1500)
    tail = r.stdout[-6000:]
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite.txt").write_text(r.stdout[-200000:] + "\n" + r.stderr[-20000:])
    assert r.returncode == 0, tail + r.stderr[-3000:]
    launches = re.search(r"conslaw hot path -> paper_1912_07645_b200: (\d+) kernel launches", r.stdout)
    assert launches and int(launches.group(1)) > 1000, tail  # the reference's calls ran the CUDA kernels
    m = re.search(r"(\d+) passed", tail)
    assert m and int(m.group(1)) >= 147 and "failed" not in tail, tail
