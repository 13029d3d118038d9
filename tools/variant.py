"""Build a tuning variant of libfvb200.so into build/<name>/ recompiling only
the fast-mode 2D/3D stage units with extra nvcc flags (the other objects are
reused from paper_1912_07645_b200/_lib).  Usage:
  python tools/variant.py NAME [--dims 2,3] [--modes fast,exact] -DFLAG=V ...
Then run with FVB_LIB=build/NAME/libfvb200.so."""
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1912_07645_b200 import build as B  # noqa: E402

name = sys.argv[1]
args = sys.argv[2:]
dims = ["2"]
modes = ["fast"]
while args and args[0] in ("--dims", "--modes"):
    if args[0] == "--dims":
        dims = args[1].split(",")
    else:
        modes = args[1].split(",")
    args = args[2:]
out = ROOT / "build" / name
out.mkdir(parents=True, exist_ok=True)
B.build(verbose=False)
for u in B.UNITS:
    shutil.copy(B.OUT / u[1], out / u[1])
units = [u for u in B.UNITS if u[1] in [f"fvb_{m}_d{d}.o" for d in dims for m in modes]]
import concurrent.futures as cf
with cf.ThreadPoolExecutor(len(units)) as ex:
    list(ex.map(lambda u: B._compile((u[0], u[1], u[2] + args), out), units))
cmd = [B.NVCC] + B.ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", str(out / "libfvb200.so")] + [str(out / u[1]) for u in B.UNITS]
subprocess.run(cmd, check=True)
for u in B.UNITS:  # keep only the linked library (gpurun snapshot size)
    (out / u[1]).unlink(missing_ok=True)
print(out / "libfvb200.so")
