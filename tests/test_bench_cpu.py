"""bench.py reference arm on the CPU (no GPU needed): the driver's --steps K
--warmup W are honoured and the JSON line carries the contract keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_honours_steps_and_warmup():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--cells", "64",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["unit"] == "Gcell-stage/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_gpus_flag_relaunches_one_process_per_rank():
    """--gpus N without torchrun re-executes bench.py under
    torch.distributed.run with N ranks; exactly one JSON line (rank 0)
    reports n_gpus = N (the reference arm needs no GPU, so this runs here)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference", "--cells",
                          "32", "--steps", "1", "--warmup", "1"], capture_output=True, text=True, cwd=ROOT,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
