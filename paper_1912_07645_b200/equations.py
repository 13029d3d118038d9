"""Equation models (equations.py:27-59).  The physics itself runs in CUDA
(csrc/fvb_physics.cuh); this module only describes the model."""

from __future__ import annotations

from dataclasses import dataclass

from . import errors as E

POSITIVITY_FLOOR = 1e-12
EULER, BURGERS, ADVECTION = "euler", "burgers", "advection"


@dataclass(frozen=True)
class EquationModel:
    kind: str
    dim: int
    gamma: float = 1.4
    advection_speed: tuple = ()

    def __post_init__(self):
        if self.kind not in (EULER, BURGERS, ADVECTION):
            raise E.ConfigError(f"unknown equation kind {self.kind!r}")
        if self.dim not in (1, 2, 3):
            raise E.ConfigError(f"dim must be 1, 2 or 3, got {self.dim}")
        if self.kind == EULER and self.gamma <= 1.0:
            raise E.ConfigError(f"gamma must be > 1, got {self.gamma}")
        if self.kind == ADVECTION:
            if len(self.advection_speed) != self.dim:
                raise E.ConfigError(
                    f"advection needs {self.dim} speed components, got {len(self.advection_speed)}")
            object.__setattr__(self, "advection_speed", tuple(float(a) for a in self.advection_speed))

    @property
    def ncomp(self) -> int:
        return self.dim + 2 if self.kind == EULER else 1

    @property
    def component_names(self) -> tuple:
        if self.kind != EULER:
            return ("u",)
        return ("rho",) + tuple("m" + "xyz"[k] for k in range(self.dim)) + ("E",)
