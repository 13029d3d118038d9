"""Build the in-tree CUDA library ``_lib/libfvb200.so`` for sm_100a.

Translation units (paper_1912_07645_b200/csrc):
  fvb_kernels.cu  x2  -> namespace exact (-fmad=false, bitwise == reference)
                         namespace fast  (-fmad=true, algebraic rewrites)
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

UNITS = [
    ("fvb_kernels.cu", "fvb_exact.o", ["-fmad=false", "-DFVB_FAST=0", "-DFVB_NS=exact"]),
    ("fvb_kernels.cu", "fvb_fast.o", ["-fmad=true", "-DFVB_FAST=1", "-DFVB_NS=fast"]),
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
    """Compile the four translation units and link libfvb200.so.  ``extra``
    adds nvcc flags (tuning experiments build variants into ``out_dir``)."""
    out = Path(out_dir) if out_dir else OUT
    out.mkdir(parents=True, exist_ok=True)
    lib = out / "libfvb200.so"
    stamp = out / "build.sha256"
    digest = _sources_digest() + "|" + " ".join(extra)
    if lib.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return lib
    units = [(src, obj, flags + list(extra)) for src, obj, flags in UNITS]
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
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
