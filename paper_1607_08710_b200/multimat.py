"""Multimaterial host types (include/lagflux/multimat.hpp, src/multimat.cpp).

Partial densities rho*y_k are the conserved quantities (one array per material
in the reference's ghosted grid layout); the device path transports them with
the hydro step (csrc/material_kernels.cu).  The scalar helpers below are the
reference's free functions, used on the host by case setup and tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import grid as G

MAX_MATERIALS = 16   # multimat.cpp:10


@dataclass(frozen=True)
class MaterialSet:
    """multimat.hpp:12-16: one adiabatic index per material."""
    gammas: tuple

    def count(self) -> int:
        return len(self.gammas)


def _fmt_f(v: float) -> str:
    return "%f" % v   # std::to_string(double)


def make_material_set(gammas: Sequence[float]) -> MaterialSet:
    """multimat.cpp:7-15 (same checks, same messages)."""
    gammas = [float(g) for g in gammas]
    if not gammas:
        raise G.ConfigError("material set needs at least one material")
    if len(gammas) > MAX_MATERIALS:
        raise G.ConfigError("at most 16 materials are supported")
    for g in gammas:
        if not (g > 1.0) or not (g <= 3.0):
            raise G.ConfigError("material adiabatic index must lie in (1, 3], got " + _fmt_f(g))
    return MaterialSet(tuple(gammas))


class MaterialCells:
    """multimat.hpp:21-30: per-cell partial densities, shape (n, nyt, nxt)."""

    def __init__(self, g: G.CartesianGrid, n_materials: int, partial: np.ndarray = None):
        # owns its storage, like the reference's std::vector arrays
        self.partial = (np.zeros((n_materials, g.nyt, g.nxt)) if partial is None
                        else np.array(partial, dtype=np.float64, order="C", copy=True))

    def count(self) -> int:
        return self.partial.shape[0]

    def copy(self) -> "MaterialCells":
        m = MaterialCells.__new__(MaterialCells)
        m.partial = self.partial.copy()
        return m


def clamped_fraction(partial: float, rho: float) -> float:
    """multimat.cpp:17-23 (the CellContext of the message is not restated)."""
    y = partial / rho
    if 0.0 <= y <= 1.0:
        return y
    if y < -1e-11 or y > 1.0 + 1e-11:
        raise G.InvalidStateError("mass fraction out of [0,1] beyond round-off = " + _fmt_f(y))
    return 0.0 if y < 0.0 else 1.0


def mixed_cell_gamma(material_set: MaterialSet, fractions: Sequence[float]) -> float:
    """multimat.cpp:25-32: 1/(gamma_eff - 1) = sum_k y_k/(gamma_k - 1); pure cells exact."""
    s = 0.0
    for k, y in enumerate(fractions):
        if y == 1.0:
            return material_set.gammas[k]
        s += y / (material_set.gammas[k] - 1.0)
    return 1.0 + 1.0 / s


def mass_fraction_fluxes(mass_flux: float, y_upwind: Sequence[float]) -> List[float]:
    """multimat.cpp:34-44: the last material takes the complement."""
    n = len(y_upwind)
    out = [0.0] * n
    rest = mass_flux
    for k in range(n - 1):
        out[k] = mass_flux * y_upwind[k]
        rest -= out[k]
    out[n - 1] = rest
    return out
