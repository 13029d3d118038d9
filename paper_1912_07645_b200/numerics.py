"""Reconstruction and two-state numerical fluxes (numerics.py of the
reference), evaluated on the GPU.

The descriptors (ReconstructionKind, FluxKind, Reconstruction,
IDEAL_WEIGHTS, FacePair) mirror numerics.py:29-61.  The function-level API
-- weno_weights / weno_face_value (numerics.py:64-87), reconstruct_axis /
reconstruct (:90-130), rusanov_flux / hllc_flux (:133-196), the
FLUX_FUNCTIONS registry seam and numerical_flux (:199-210) -- runs the same
device functions the fused stage kernels use (csrc/fvb_physics.cuh) through
the C ABI (fvb_weno, fvb_face_flux): arrays go to the GPU, come back with the
caller's shape.  In exact arithmetic (the default) every value is bitwise
equal to the reference; a degenerate HLLC wave fan raises
UnphysicalStateError as the reference does (numerics.py:166-167).

Inputs may be numpy arrays (returned as numpy) or CUDA tensors (returned as
CUDA tensors, no host round trip).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np

from . import _native as N
from . import errors as E


class ReconstructionKind(Enum):
    NONE = "none"
    WENO2 = "weno2"
    WENO3 = "weno3"


class FluxKind(Enum):
    RUSANOV = "rusanov"
    HLLC = "hllc"


@dataclass(frozen=True)
class Reconstruction:
    kind: ReconstructionKind = ReconstructionKind.NONE
    epsilon: float = 1e-6

    @property
    def radius(self) -> int:
        return 1 if self.kind is ReconstructionKind.NONE or getattr(self.kind, "value", None) == "none" else 2


IDEAL_WEIGHTS = {ReconstructionKind.WENO2: (0.5, 0.5), ReconstructionKind.WENO3: (1.0 / 3.0, 2.0 / 3.0)}


class FacePair(NamedTuple):
    """Reconstructed states on the two sides of each interface."""

    uL: object
    uR: object


def _v(x):
    return getattr(x, "value", x)


# ---------------------------------------------------------------------------
# host <-> device plumbing
# ---------------------------------------------------------------------------

def _is_tensor(a) -> bool:
    return type(a).__module__.startswith("torch")


def _dev(a):
    """Contiguous CUDA float64 tensor of ``a`` (numpy / scalar / tensor)."""
    import torch

    N._require_cuda()
    if _is_tensor(a):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to("cuda")


def _out(t, like_tensor: bool, shape):
    t = t.reshape(shape)
    return t if like_tensor else t.cpu().numpy()


def _scheme(model=None, flux=None, recon=None, eps: float = 1e-6, arith: str | None = None) -> N.Scheme:
    s = N.Scheme()
    s.arith = N.ARITH[arith or N.default_arith()]
    s.weno_eps = float(eps)
    if recon is not None:
        s.recon = N.RECON[_v(recon)]
    if model is not None:
        s.dim = int(model.dim)
        s.eq = N.EQ[model.kind]
        s.ncomp = s.dim + 2 if model.kind == "euler" else 1
        s.gamma = float(getattr(model, "gamma", 1.4))
        speeds = tuple(getattr(model, "advection_speed", ()) or ())
        for k in range(3):
            s.adv[k] = float(speeds[k]) if (model.kind == "advection" and k < len(speeds)) else 0.0
    if flux is not None:
        s.flux = N.FLUX[_v(flux)]
    return s


# ---------------------------------------------------------------------------
# WENO (numerics.py:64-87)
# ---------------------------------------------------------------------------

def _weno(um, uc, up, kind, epsilon, want):
    if _v(kind) not in ("weno2", "weno3"):
        raise E.ConfigError(f"weno_weights needs WENO2 or WENO3, got {kind}")
    tensor = any(_is_tensor(a) for a in (um, uc, up))
    if tensor:
        import torch

        a, b, c = torch.broadcast_tensors(*(_dev(x) for x in (um, uc, up)))
    else:
        a, b, c = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (um, uc, up)))
    shape = tuple(a.shape)
    a, b, c = (_dev(x).reshape(-1) for x in (a, b, c))
    n = int(a.numel())
    import torch

    outs = {k: torch.empty(n, dtype=torch.float64, device="cuda") for k in want}
    ctx = N.context()
    ptr = lambda k: N.C.c_void_p(outs[k].data_ptr()) if k in outs else None  # noqa: E731
    if n:
        ctx.check(ctx.lib.fvb_weno(ctx.h, N.C.byref(_scheme(recon=kind, eps=epsilon)),
                                   N.C.c_void_p(a.data_ptr()), N.C.c_void_p(b.data_ptr()),
                                   N.C.c_void_p(c.data_ptr()), n, ptr("w0"), ptr("w1"), ptr("face")))
    return tuple(_out(outs[k], tensor, shape) for k in want)


def weno_weights(um, uc, up, kind: ReconstructionKind, epsilon: float = 1e-6):
    """Normalised nonlinear weights (w0, w1) of the two substencils
    (numerics.py:64-78)."""
    return _weno(um, uc, up, kind, epsilon, ("w0", "w1"))


def weno_face_value(um, uc, up, kind: ReconstructionKind, epsilon: float):
    """Reconstructed value at the downwind face of the centre cell
    (numerics.py:81-87): uc + 0.5 (w0 (uc - um) + w1 (up - uc))."""
    return _weno(um, uc, up, kind, epsilon, ("face",))[0]


def _take(data, ax, lo, hi):
    s = [slice(None)] * data.ndim
    s[ax] = slice(lo, hi)
    return data[tuple(s)]


def reconstruct_axis(data, np_ax: int, n: int, g: int, recon: Reconstruction) -> FacePair:
    """Face states at the n+1 interfaces of one axis of a padded array
    (numerics.py:90-118): interface j sits between padded cells (g-1+j, g+j)."""
    if recon.radius > g:
        raise E.ConfigError(f"reconstruction radius {recon.radius} exceeds ghost width {g}")
    if _v(recon.kind) == "none":
        return FacePair(_take(data, np_ax, g - 1, g + n), _take(data, np_ax, g, g + n + 1))
    uL = weno_face_value(_take(data, np_ax, g - 2, g + n - 1), _take(data, np_ax, g - 1, g + n),
                         _take(data, np_ax, g, g + n + 1), recon.kind, recon.epsilon)
    uR = weno_face_value(_take(data, np_ax, g + 1, g + n + 2), _take(data, np_ax, g, g + n + 1),
                         _take(data, np_ax, g - 1, g + n), recon.kind, recon.epsilon)
    return FacePair(uL, uR)


def reconstruct(field, axis: int, recon: Reconstruction) -> FacePair:
    """Face states along ``axis`` for every interface of a ghost-filled field
    (numerics.py:121-130)."""
    grid = field.grid
    return reconstruct_axis(field.data, grid.dim - axis, grid.cells[axis], grid.ghost_width, recon)


# ---------------------------------------------------------------------------
# two-state fluxes (numerics.py:133-196) and the registry seam (:199-210)
# ---------------------------------------------------------------------------

def _face_flux(model, flux: str, pair, axis: int):
    uL, uR = pair
    tensor = _is_tensor(uL) or _is_tensor(uR)
    if tensor:
        import torch

        a, b = torch.broadcast_tensors(_dev(uL), _dev(uR))
    else:
        a, b = np.broadcast_arrays(np.asarray(uL, dtype=np.float64), np.asarray(uR, dtype=np.float64))
    shape = tuple(a.shape)
    nc = model.dim + 2 if model.kind == "euler" else 1
    if not shape or shape[0] != nc:
        raise E.ConfigError(f"face states need {nc} components on axis 0, got shape {shape}")
    a, b = _dev(a).reshape(nc, -1), _dev(b).reshape(nc, -1)
    n = int(a.shape[1])
    import torch

    F = torch.empty((nc, n), dtype=torch.float64, device="cuda")
    if n:
        ctx = N.context()
        rc = ctx.lib.fvb_face_flux(ctx.h, N.C.byref(_scheme(model, flux)), int(axis),
                                   N.C.c_void_p(a.data_ptr()), N.C.c_void_p(b.data_ptr()), n,
                                   N.C.c_void_p(F.data_ptr()))
        msg = ctx.message() if rc else ""
        if rc == N.E_UNPHYSICAL and msg.startswith("unphysical state: side"):
            # physical_flux's check (equations.py:77-86): first bad cell of uL, then uR
            side, flat = msg.split()[3], int(msg.split()[-1])
            u = (a if side == "L" else b)[:, flat].cpu().numpy()
            idx = tuple(int(i) for i in np.unravel_index(flat, shape[1:])) if len(shape) > 1 else (flat,)
            raise E.UnphysicalStateError(f"unphysical state at cell {idx}: u = {u}")
        ctx.check(rc)
    return _out(F, tensor, shape)


def rusanov_flux(model, pair: FacePair, axis: int):
    """Local Lax-Friedrichs flux (numerics.py:133-142)."""
    return _face_flux(model, "rusanov", pair, axis)


def hllc_flux(model, pair: FacePair, axis: int):
    """Three-wave HLLC flux with Davis wave speeds (numerics.py:145-196)."""
    if model.kind != "euler":
        raise E.ConfigError("HLLC flux is only defined for the Euler equations")
    return _face_flux(model, "hllc", pair, axis)


FLUX_FUNCTIONS = {FluxKind.RUSANOV: rusanov_flux, FluxKind.HLLC: hllc_flux}


def numerical_flux(model, kind, pair: FacePair, axis: int):
    """numerics.py:209-210: dispatch through FLUX_FUNCTIONS (accepts the
    reference's FluxKind members too)."""
    return FLUX_FUNCTIONS[FluxKind(_v(kind))](model, pair, axis)
