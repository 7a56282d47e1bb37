"""Plain-data types of the Lagrange-flux hot path, mirroring the reference.

These are the host-side descriptions the C-ABI consumes; no compute here.

  CartesianGrid, make_grid_1d/2d   /root/reference/proj/include/lagflux/grid.hpp:17-44,
                                   src/grid.cpp:23-56
  BcKind / BoundaryCondition       grid.hpp:51-58, validate_boundary grid.cpp:65-70
  SchemeParams, TimeControls,
  StepDiagnostics, SolverState     include/lagflux/solver.hpp:39-67
  exception types                  include/lagflux/error.hpp:9-64
  conserved_from_primitive         include/lagflux/euler.hpp:87-97 (host-side ICs)

A field is a float64 numpy array of shape (4, nyt, nxt): the reference's
``CellField`` (four ghosted row-major SoA components rho, rho*u, rho*v, rho*E)
with the component index first so ``field[c]`` is one contiguous array.
"""
from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from typing import List

import numpy as np

TRANSMISSIVE, REFLECTIVE, PERIODIC = 0, 1, 2
BC_NAMES = {"transmissive": TRANSMISSIVE, "reflective": REFLECTIVE, "periodic": PERIODIC}
INT64_MAX = 2**63 - 1


class Error(RuntimeError):
    """lagflux::Error (error.hpp:9-13)."""


class InvalidStateError(Error):
    """lagflux::InvalidStateError (error.hpp:15-19)."""


class ConfigError(Error):
    """lagflux::ConfigError (error.hpp:21-25)."""


class DeterminismError(Error):
    """lagflux::DeterminismError (error.hpp:60-64)."""


class DeviceError(Error):
    """CUDA / NCCL failure below the C-ABI (no reference counterpart)."""


class PositivityError(Error):
    """lagflux::PositivityError (error.hpp:48-58): carries cell_i, cell_j, step, dt."""

    def __init__(self, what: str, cell_i: int, cell_j: int, step: int, dt: float):
        super().__init__(what)
        self.cell_i, self.cell_j, self.step, self.dt = cell_i, cell_j, step, dt


@dataclass(frozen=True)
class CartesianGrid:
    dim: int = 1
    nx: int = 1
    ny: int = 1
    dx: float = 1.0
    dy: float = 1.0
    x0: float = 0.0
    y0: float = 0.0
    gx: int = 2
    gy: int = 0

    @property
    def nxt(self) -> int:
        return self.nx + 2 * self.gx

    @property
    def nyt(self) -> int:
        return self.ny + 2 * self.gy

    def idx(self, i: int, j: int) -> int:
        return j * self.nxt + i

    def xc(self, i):
        return self.x0 + (i - self.gx + 0.5) * self.dx

    def yc(self, j):
        return self.y0 + (j - self.gy + 0.5) * self.dy

    @property
    def interior_count(self) -> int:
        return self.nx * self.ny

    def cell_volume(self) -> float:
        return self.dx * self.dy if self.dim == 2 else self.dx

    def interior(self, f: np.ndarray) -> np.ndarray:
        """View of the interior cells of a (…, nyt, nxt) array."""
        return f[..., self.gy:self.gy + self.ny, self.gx:self.gx + self.nx]


def _check_count(name: str, n: int) -> None:
    if n < 1:
        raise ConfigError(f"{name} must be >= 1, got {n}")


def _check_extent(name: str, lo: float, hi: float) -> None:
    if not hi > lo:
        raise ConfigError(f"{name} extent must be positive, got [{lo:f}, {hi:f}]")


def make_grid_1d(nx: int, x_min: float, x_max: float, ghost: int = 2) -> CartesianGrid:
    """grid.cpp:23-37"""
    _check_count("nx", nx)
    _check_extent("x", x_min, x_max)
    return CartesianGrid(1, nx, 1, (x_max - x_min) / nx, 1.0, x_min, 0.0, ghost, 0)


def make_grid_2d(nx: int, ny: int, x_min: float, x_max: float, y_min: float, y_max: float,
                 ghost: int = 2) -> CartesianGrid:
    """grid.cpp:39-56"""
    _check_count("nx", nx)
    _check_count("ny", ny)
    _check_extent("x", x_min, x_max)
    _check_extent("y", y_min, y_max)
    return CartesianGrid(2, nx, ny, (x_max - x_min) / nx, (y_max - y_min) / ny, x_min, y_min,
                         ghost, ghost)


@dataclass(frozen=True)
class BoundaryCondition:
    x_low: int = TRANSMISSIVE
    x_high: int = TRANSMISSIVE
    y_low: int = TRANSMISSIVE
    y_high: int = TRANSMISSIVE

    @staticmethod
    def uniform(kind: int) -> "BoundaryCondition":
        return BoundaryCondition(kind, kind, kind, kind)

    def as_list(self) -> List[int]:
        return [self.x_low, self.x_high, self.y_low, self.y_high]


def validate_boundary(bc: BoundaryCondition, dim: int) -> None:
    """grid.cpp:65-70"""
    if (bc.x_low == PERIODIC) != (bc.x_high == PERIODIC):
        raise ConfigError("periodic boundary in x must be set on both sides")
    if dim == 2 and (bc.y_low == PERIODIC) != (bc.y_high == PERIODIC):
        raise ConfigError("periodic boundary in y must be set on both sides")


@dataclass(frozen=True)
class SchemeParams:
    """solver.hpp:45-49 (LimiterParams folded in as ``beta``)."""
    beta: float = 1.5
    spatial_order: int = 2
    time_order: int = 2


def make_limiter(beta: float) -> float:
    """reconstruct.hpp:16-20"""
    if not (beta >= 1.0 and beta <= 2.0):
        raise ConfigError(f"limiter beta must lie in [1, 2], got {beta:f}")
    return beta


def make_eos(gamma: float) -> float:
    """euler.hpp:43-47"""
    if not (gamma > 1.0 and gamma <= 3.0):
        raise ConfigError(f"adiabatic index must lie in (1, 3], got {gamma:f}")
    return gamma


@dataclass(frozen=True)
class TimeControls:
    """solver.hpp:39-43"""
    cfl: float = 0.25
    t_final: float = 0.0
    max_steps: int = INT64_MAX


@dataclass(frozen=True)
class StepDiagnostics:
    """solver.hpp:51-57"""
    step: int
    time: float
    dt: float
    min_rho: float
    min_p: float


@dataclass
class SolverState:
    """solver.hpp:59-67; ``field`` is a (4, nyt, nxt) float64 array."""
    field: np.ndarray
    time: float = 0.0
    step: int = 0
    diagnostics: List[StepDiagnostics] = dc_field(default_factory=list)
    boundary_outflow: List[float] = dc_field(default_factory=lambda: [0.0, 0.0, 0.0, 0.0])


def new_field(g: CartesianGrid) -> np.ndarray:
    """CellField(g): zero-initialised ghosted SoA storage."""
    return np.zeros((4, g.nyt, g.nxt), dtype=np.float64)


def conserved_from_primitive(rho, u, v, p, gamma: float):
    """euler.hpp:87-97, elementwise with the reference's evaluation order.

    numpy evaluates each binary operation with one IEEE rounding (no FMA), so
    the result is bit-identical to the reference's scalar C++."""
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    if not (np.all(rho > 0.0) and np.all(p > 0.0)):
        raise InvalidStateError("non-positive density or pressure in initial data")
    mx = rho * u
    my = rho * v
    e = p / (gamma - 1.0) + (0.5 * rho) * (u * u + v * v)
    return rho, mx, my, e
