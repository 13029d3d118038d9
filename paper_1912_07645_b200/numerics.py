"""Reconstruction / flux descriptors (numerics.py:29-54).  The kernels live in
csrc/fvb_physics.cuh; FLUX_FUNCTIONS names the device implementations."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


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

# device flux implementations (fvb_physics.cuh: rusanov<>, hllc<>)
FLUX_FUNCTIONS = {FluxKind.RUSANOV: "fvb::rusanov", FluxKind.HLLC: "fvb::hllc"}
