"""ctypes binding of the C ABI in ``include/fvb200.h`` (libfvb200.so).

This is the only door into the compute path.  There is no CPU fallback: if
the in-tree library is missing, or no CUDA device is visible, every compute
call raises ``NativeUnavailable`` loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import errors as E

LIB_PATH = Path(os.environ.get("FVB_LIB") or Path(__file__).resolve().parent / "_lib" / "libfvb200.so")

# status codes (fvb200.h)
OK, E_CONFIG, E_UNPHYSICAL, E_SIMULATION, E_STATIC, E_PROTOCOL, E_CUDA = range(7)
SUB_NONE, SUB_INIT_UNPHYS, SUB_STAGE_UNPHYS, SUB_NONFINITE, SUB_POST_UNPHYS, SUB_HLLC, SUB_SPEED_UNPHYS, SUB_REMOTE = range(8)
EQ = {"euler": 0, "burgers": 1, "advection": 2}
FLUX = {"rusanov": 0, "hllc": 1}
RECON = {"none": 0, "weno2": 1, "weno3": 2}
BC_PERIODIC, BC_OUTFLOW, BC_HALO = 0, 1, 2
MODE_T_END, MODE_FIXED, MODE_PAR_T_END = 0, 1, 2
ARITH = {"exact": 0, "fast": 1}


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing: the hot path cannot run."""


class Scheme(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("ncomp", C.c_int32), ("eq", C.c_int32), ("flux", C.c_int32),
        ("recon", C.c_int32), ("rk_order", C.c_int32), ("arith", C.c_int32), ("ghost", C.c_int32),
        ("bc", C.c_int32 * 3), ("pad", C.c_int32),
        ("cells", C.c_int64 * 3), ("deltas", C.c_double * 3),
        ("gamma", C.c_double), ("weno_eps", C.c_double), ("cfl", C.c_double), ("t_end", C.c_double),
        ("adv", C.c_double * 3),
    ]


class Layout(C.Structure):
    _fields_ = [("origin", C.c_int64), ("sy", C.c_int64), ("sz", C.c_int64), ("sc", C.c_int64),
                ("si", C.c_int64)]


class RunInfo(C.Structure):
    _fields_ = [("t", C.c_double), ("dt", C.c_double), ("steps", C.c_int64), ("err", C.c_int32),
                ("errsub", C.c_int32), ("errcell", C.c_int64)]


_lib = None
_lib_lock = threading.Lock()

_SIGS = {
    "fvb_version": ([], C.c_int),
    "fvb_ctx_create": ([C.c_int, C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "fvb_ctx_destroy": ([C.c_void_p], C.c_int),
    "fvb_ctx_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "fvb_last_error": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
    "fvb_sync": ([C.c_void_p], C.c_int),
    "fvb_fill_ghosts": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int], C.c_int),
    "fvb_wave_speed_maxima": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int,
                               C.POINTER(C.c_double)], C.c_int),
    "fvb_spatial_residual": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_void_p,
                              C.c_int], C.c_int),
    "fvb_ssp_rk_step": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_void_p,
                         C.c_void_p, C.c_int, C.c_double], C.c_int),
    "fvb_run": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.POINTER(C.c_void_p), C.c_int, C.c_int,
                 C.c_int64, C.POINTER(C.c_double), C.c_int64, C.c_int, C.POINTER(RunInfo)], C.c_int),
    "fvb_run_begin": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.POINTER(C.c_void_p), C.c_int,
                       C.c_int, C.c_int64], C.c_int),
    "fvb_run_steps": ([C.c_void_p, C.c_int64], C.c_int),
    "fvb_run_end": ([C.c_void_p, C.POINTER(RunInfo), C.POINTER(C.c_double), C.c_int64], C.c_int),
    "fvb_run_poll": ([C.c_void_p, C.POINTER(RunInfo), C.POINTER(C.c_int32)], C.c_int),
    "fvb_run_set_log": ([C.c_void_p, C.c_int64, C.c_int], C.c_int),
    "fvb_run_set_topology": ([C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
    "fvb_run_set_external_reduce": ([C.c_void_p, C.c_int], C.c_int),
    "fvb_run_stage": ([C.c_void_p, C.c_int], C.c_int),
    "fvb_run_stage_rows": ([C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int], C.c_int),
    "fvb_run_stage_box": ([C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int], C.c_int),
    "fvb_run_set_peers": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
    "fvb_run_export": ([C.c_void_p, C.c_void_p], C.c_int),
    "fvb_run_finalize": ([C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "fvb_run_read_log": ([C.c_void_p, C.POINTER(C.c_double), C.c_int64], C.c_int),
    "fvb_launch_count": ([C.c_void_p], C.c_int64),
    "fvb_moments_push": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int,
                          C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "fvb_moments_push_batch": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int, C.c_int,
                                C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "fvb_moments_merge": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                           C.c_int64, C.c_int64], C.c_int),
    "fvb_structure_push": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int, C.c_int,
                            C.c_double, C.c_int, C.c_void_p], C.c_int),
    "fvb_init_eval": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.POINTER(C.c_double), C.c_void_p,
                       C.POINTER(C.c_int32), C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                       C.c_void_p, C.c_void_p], C.c_int),
    "fvb_halo_pack": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int, C.c_int,
                       C.c_void_p], C.c_int),
    "fvb_halo_unpack": ([C.c_void_p, C.POINTER(Scheme), C.POINTER(Layout), C.c_void_p, C.c_int, C.c_int,
                         C.c_void_p], C.c_int),
    "fvb_halo_count": ([C.POINTER(Scheme), C.c_int], C.c_int64),
    "fvb_face_flux": ([C.c_void_p, C.POINTER(Scheme), C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
                      C.c_int),
    "fvb_weno": ([C.c_void_p, C.POINTER(Scheme), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                  C.c_void_p, C.c_void_p], C.c_int),
}

EXPORTS = tuple(_SIGS)


def _warn_if_stale(lib_path: Path) -> None:
    """The in-tree library records the digest of the sources it was built
    from (build.py); loading one built from other sources (e.g. a tuning
    variant left behind) would silently measure the wrong code."""
    try:
        from . import build as B

        stamp = lib_path.parent / "build.sha256"
        if stamp.exists() and stamp.read_text().split("|")[0] != B._sources_digest():
            import warnings

            warnings.warn(f"{lib_path} was built from different sources than the ones in csrc/: "
                          "rebuild with `python -m paper_1912_07645_b200.build`", RuntimeWarning)
    except Exception:
        pass


def load_library(path: Path | None = None) -> C.CDLL:
    """Load libfvb200.so (no GPU needed); raise NativeUnavailable if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -m paper_1912_07645_b200.build` "
                "(there is no CPU fallback for the finite-volume hot path)")
        if path is None and not os.environ.get("FVB_LIB"):
            _warn_if_stale(p)
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


_CUDA_OK = False


def _require_cuda():
    global _CUDA_OK
    if _CUDA_OK:  # a device stays visible once seen (is_available() queries the driver every call)
        return
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the B200 hot path cannot run (no CPU fallback)")
    _CUDA_OK = True


class Context:
    """One fvb_ctx per (device, stream).  Not re-entrant."""

    def __init__(self, device: int = 0, stream=None):
        _require_cuda()
        tune_host_malloc()
        import torch

        self.lib = load_library()
        self.device = device
        torch.cuda.set_device(device)
        # torch owns the stream; the library launches on it
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        rc = self.lib.fvb_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        self.h = h
        self.check(rc)

    def set_stream(self, stream):
        self.stream = stream
        self.check(self.lib.fvb_ctx_set_stream(self.h, C.c_void_p(stream.cuda_stream)))

    def message(self) -> str:
        buf = C.create_string_buffer(1024)
        self.lib.fvb_last_error(self.h, buf, 1024)
        return buf.value.decode(errors="replace")

    def check(self, rc: int):
        if rc == OK:
            return
        msg = self.message()
        raise status_error(rc, msg)

    def launches(self) -> int:
        return int(self.lib.fvb_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.fvb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def status_error(rc: int, msg: str) -> Exception:
    if rc == E_CONFIG:
        return E.ConfigError(msg)
    if rc == E_UNPHYSICAL:
        return E.UnphysicalStateError(msg)
    if rc == E_SIMULATION:
        return E.SimulationError(msg)
    if rc == E_STATIC:
        return E.StaticFieldError(msg)
    if rc == E_PROTOCOL:
        return E.ProtocolError(msg)
    return RuntimeError(f"CUDA failure in libfvb200: {msg}")


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()


def context(device: int | None = None) -> Context:
    """Per-thread, per-device, per-stream context (contexts are not re-entrant)."""
    import torch

    _require_cuda()
    if device is None:
        device = torch.cuda.current_device()
    stream = torch.cuda.current_stream(device)
    key = (threading.get_ident(), device, stream.cuda_stream)
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            ctx = Context(device, stream)
            _ctx_cache[key] = ctx
        return ctx


def tune_host_malloc() -> None:
    """Keep large host allocations (result fields) in the malloc heap instead
    of fresh mmaps, so repeated results reuse already-faulted pages
    (FVB_MALLOPT=1)."""
    if os.environ.get("FVB_MALLOPT", "1") != "1":
        return
    try:
        libc = C.CDLL("libc.so.6")
        libc.mallopt(-3, 1 << 30)  # M_MMAP_THRESHOLD
        libc.mallopt(-1, 1 << 31)  # M_TRIM_THRESHOLD
    except OSError:
        pass


def default_arith() -> str:
    return os.environ.get("FVB_ARITH", "exact")
