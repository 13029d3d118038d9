"""Initial data of the benchmark configurations (host side, boundary input).

Each function evaluates the reference preset's expression with the same
numpy operations, in the same order, as iodsl/expr.py:271-316 +
eval_init (expr.py:350-386) + primitive_to_conserved (equations.py:132-145),
so the fields are bitwise identical to the reference's ``eval_init`` on the
same random vector (pinned by tests/test_initial.py against golden SHAs).
A GPU evaluator of the DSL is SURVEY 8(f) item 1 ("next").
"""

from __future__ import annotations

import numpy as np

from .equations import EquationModel
from .grid import Field, GridSpec, make_field

TWO_PI = 2.0 * np.pi


def _centres(grid: GridSpec):
    env = {}
    for axis in range(grid.dim):
        shape = [1] * grid.dim
        shape[grid.dim - 1 - axis] = grid.cells[axis]
        env["xyz"[axis]] = grid.cell_centers(axis).reshape(shape)
    return env


def _conserved(model: EquationModel, w: np.ndarray) -> np.ndarray:
    dim = model.dim
    u = np.empty_like(w)
    u[0] = w[0]
    kin = np.zeros_like(w[0])
    for k in range(dim):
        u[1 + k] = w[0] * w[1 + k]
        kin = kin + w[1 + k] ** 2
    u[1 + dim] = w[1 + dim] / (model.gamma - 1.0) + 0.5 * w[0] * kin
    return u


def _field(grid, values) -> Field:
    f = make_field(grid, values.shape[0], 0.0) if values.size * 1.0 < 2 ** 28 else None
    if f is None:  # device-scale grids bypass the host size cap
        data = np.zeros((values.shape[0],) + grid.data_shape)
        f = Field(grid, values.shape[0], data)
    f.interior[...] = values
    return f


def kelvin_helmholtz(grid: GridSpec, vec, gamma: float = 1.4) -> Field:
    """KH2D / KH3D presets (presets.py:65-145): two shear layers at y = 1/4,
    3/4 perturbed by sin(2 pi (x + X_i)), rho in {1, 2}, vx = -/+0.5, p = 2.5."""
    env = _centres(grid)
    x, y = env["x"], env["y"]
    shape = grid.interior_shape

    def layer(base, X):
        return np.less(y, base + 0.01 * np.sin(TWO_PI * (x + X))).astype(float)

    lo, hi = layer(0.25, vec[0]), layer(0.75, vec[1])
    rho = np.where(lo != 0.0, 1.0, np.where(hi != 0.0, 2.0, 1.0))
    lo, hi = layer(0.25, vec[2]), layer(0.75, vec[3])
    vx = np.where(lo != 0.0, -0.5, np.where(hi != 0.0, 0.5, -0.5))
    model = EquationModel("euler", grid.dim, gamma=gamma)
    w = np.empty((grid.dim + 2,) + shape)
    w[0] = np.broadcast_to(rho, shape)
    w[1] = np.broadcast_to(vx, shape)
    for k in range(1, grid.dim):
        w[1 + k] = 0.0
    w[1 + grid.dim] = 2.5
    return _field(grid, _conserved(model, w))


def burgers_sines(grid: GridSpec, vec) -> Field:
    """C5 authored config:
    u = 1.0 + 0.5 * sin(2 pi (x + X0)) * sin(2 pi (y + X1))."""
    env = _centres(grid)
    v = 1.0 + 0.5 * np.sin(TWO_PI * (env["x"] + vec[0])) * np.sin(TWO_PI * (env["y"] + vec[1]))
    return _field(grid, np.broadcast_to(v, grid.interior_shape)[None].copy())


def sod(grid: GridSpec, gamma: float = 1.4) -> Field:
    """SOD preset (presets.py:8-34): rho, p = (1, 1) | (0.125, 0.1), v = 0."""
    x = _centres(grid)["x"]
    rho = np.where(np.less(x, 0.5).astype(float) != 0.0, 1.0, 0.125)
    p = np.where(np.less(x, 0.5).astype(float) != 0.0, 1.0, 0.1)
    w = np.empty((3,) + grid.interior_shape)
    w[0] = rho
    w[1] = 0.0
    w[2] = p
    return _field(grid, _conserved(EquationModel("euler", 1, gamma=gamma), w))
