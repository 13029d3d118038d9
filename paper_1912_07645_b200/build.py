"""Build the in-tree CUDA library ``_lib/libfvb200.so`` for sm_100a.

Translation units (paper_1912_07645_b200/csrc):
  fvb_kernels.cu  x8  -> namespace exact (-fmad=false, bitwise == reference)
                         namespace fast  (-fmad=true, algebraic rewrites),
                         one unit per dimension (-DFVB_KDIM=1,2,3) + dispatch (0)
  fvb_aux.cu          -> ghost fill, halo slabs, UQ statistics (-fmad=false)
  fvb_capi.cu         -> extern "C" ABI declared in include/fvb200.h
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib"
LIB = OUT / "libfvb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")] + ARCH

_MODES = [("exact", ["-fmad=false", "-DFVB_FAST=0", "-DFVB_NS=exact"]),
          ("fast", ["-fmad=true", "-DFVB_FAST=1", "-DFVB_NS=fast"])]
# the stage kernels: one unit per (mode, dimension) so they compile in
# parallel (FVB_KDIM = 0 is the dispatcher + wave-speed kernels)
UNITS = [("fvb_kernels.cu", f"fvb_{m}_d{d}.o", flags + [f"-DFVB_KDIM={d}"]) for d in (2, 3, 1, 0)
         for m, flags in _MODES] + [
    ("fvb_aux.cu", "fvb_aux.o", ["-fmad=false"]),
    ("fvb_capi.cu", "fvb_capi.o", ["-fmad=false"]),
]


def _sources_digest() -> str:
    h = hashlib.sha256()
    for f in sorted(CSRC.glob("*")) + [ROOT / "include" / "fvb200.h", Path(__file__)]:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()


def _compile(unit, out: Path = OUT):
    src, obj, flags = unit
    cmd = [NVCC] + COMMON + flags + ["-c", str(CSRC / src), "-o", str(out / obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True, extra=(), out_dir: Path | None = None) -> Path:
    """Compile the translation units and link libfvb200.so.  ``extra``
    adds nvcc flags (tuning experiments build variants into ``out_dir``)."""
    out = Path(out_dir) if out_dir else OUT
    out.mkdir(parents=True, exist_ok=True)
    lib = out / "libfvb200.so"
    stamp = out / "build.sha256"
    digest = _sources_digest() + "|" + " ".join(extra)
    if lib.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return lib
    units = [(src, obj, flags + list(extra)) for src, obj, flags in UNITS]
    with cf.ThreadPoolExecutor(max_workers=min(len(units), os.cpu_count() or 4)) as ex:
        list(ex.map(lambda u: _compile(u, out), units))
    cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", str(lib)] + [str(out / u[1]) for u in UNITS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    stamp.write_text(digest)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("extra", nargs="*", help="extra nvcc flags, e.g. -DFVB_STRIP_MINB=3")
    a = ap.parse_args()
    build(force=a.force, extra=a.extra, out_dir=a.out)
