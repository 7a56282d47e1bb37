"""The BASELINE.json workloads as host-side case definitions (caller side of the boundary).

The reference builds initial states in its driver (run.cpp:29-78,
``initialize_hydro``); these are the same kinds of initialisers for the five
configs BASELINE.json names, frozen as recorded in DESIGN.md "Initial conditions":

  1 sod        400x4, reflective, CFL 0.5, to t = 0.2 (riemann_x, run.cpp:43)
  2 quadrant   1024^2 four-quadrant Riemann problem, transmissive, CFL 0.45, 200 steps
               (regions, run.cpp:50-67: x >= x_min && x < x_max)
  3 sedov      4096^2, rho = 1, p = 1e-5, p_c = (gamma-1) E0 / (9 dx dy) in the 3x3
               centre cells n/2-1..n/2+1, reflective, CFL 0.4, 100 steps
  4 smooth     16384^2 seeded 8-mode Fourier flow, periodic, CFL 0.5, 50 steps
  5 smooth     32768^2 same generator, 20 steps (strong scaling); weak scaling at
               16384 x 16384*n on [0,1]x[0,n]

Sizes are parameters so tests run the same generators at reduced size.  The
Fourier generator is defined by 1D sin/cos tables (glibc libm, computed here
with ``math.sin``/``math.cos``) combined with plain IEEE products and sums, so
the device initialiser (``lf_init_fourier``) and this host version produce
identical bits.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import grid as G

SMOOTH_SEED = 1607087100
E0_SEDOV = 1.0


@dataclass(frozen=True)
class Case:
    name: str
    grid: G.CartesianGrid
    bc: G.BoundaryCondition
    gamma: float
    params: G.SchemeParams
    cfl: float
    t_final: float          # 1e300 for step-driven cases (bench.cpp:57 uses DBL_MAX)
    max_steps: int
    init: str               # "riemann_x" | "quadrant" | "sedov" | "fourier"
    seed: int = SMOOTH_SEED

    @property
    def cells(self) -> int:
        return self.grid.nx * self.grid.ny


STEP_DRIVEN_LIMIT = 1.7976931348623157e308  # std::numeric_limits<double>::max()


def sod(nx: int = 400, ny: int = 4) -> Case:
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 1.0)
    return Case("sod", g, G.BoundaryCondition.uniform(G.REFLECTIVE), 1.4, G.SchemeParams(),
                0.5, 0.2, G.INT64_MAX, "riemann_x")


def quadrant(n: int = 1024, steps: int = 200) -> Case:
    g = G.make_grid_2d(n, n, 0.0, 1.0, 0.0, 1.0)
    return Case("quadrant", g, G.BoundaryCondition.uniform(G.TRANSMISSIVE), 1.4,
                G.SchemeParams(), 0.45, STEP_DRIVEN_LIMIT, steps, "quadrant")


def sedov(n: int = 4096, steps: int = 100) -> Case:
    g = G.make_grid_2d(n, n, 0.0, 1.0, 0.0, 1.0)
    return Case("sedov", g, G.BoundaryCondition.uniform(G.REFLECTIVE), 1.4, G.SchemeParams(),
                0.4, STEP_DRIVEN_LIMIT, steps, "sedov")


def smooth(n: int = 16384, steps: int = 50, ny: Optional[int] = None, y_extent: float = 1.0,
           seed: int = SMOOTH_SEED) -> Case:
    g = G.make_grid_2d(n, ny if ny is not None else n, 0.0, 1.0, 0.0, y_extent)
    return Case("smooth", g, G.BoundaryCondition.uniform(G.PERIODIC), 1.4, G.SchemeParams(),
                0.5, STEP_DRIVEN_LIMIT, steps, "fourier", seed)


def smooth_weak(n_gpus: int, n: int = 16384, steps: int = 20) -> Case:
    """Weak scaling: 16384 x (16384 n) on [0,1] x [0,n] so dx = dy (BASELINE config 5)."""
    return smooth(n, steps, ny=n * n_gpus, y_extent=float(n_gpus))


CONFIGS = {1: sod, 2: quadrant, 3: sedov, 4: smooth, 5: lambda: smooth(32768, 20)}


# ---------------------------------------------------------------- multimaterial
@dataclass(frozen=True)
class Region:
    """RegionSpec (config.hpp): a rectangle [x_min, x_max) x [y_min, y_max) of one
    primitive state and one material (1-based, as in the case files)."""
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    rho: float
    u: float
    v: float
    p: float
    material: int = 1


@dataclass(frozen=True)
class MatCase:
    """A region-initialised multimaterial case (run.cpp:29-78, 140-190)."""
    name: str
    grid: G.CartesianGrid
    bc: G.BoundaryCondition
    gamma: float                    # the solver's eos (CaseConfig::gamma)
    material_gammas: tuple
    regions: tuple
    params: G.SchemeParams
    cfl: float
    t_final: float
    max_steps: int


def regions_field(c: MatCase):
    """initialize_hydro (run.cpp:29-78) for InitKind::regions: the ghosted field
    and the partial densities (n_mat, nyt, nxt); ghosts are zero.  Vectorised:
    every operation is the same elementwise IEEE operation as the reference's."""
    from . import multimat as MM
    g = c.grid
    f = G.new_field(g)
    n_mat = len(c.material_gammas) if c.material_gammas else 1
    mat = MM.MaterialCells(g, n_mat)
    x = g.xc(np.arange(g.gx, g.gx + g.nx))[None, :] * np.ones((g.ny, 1))
    y = g.yc(np.arange(g.gy, g.gy + g.ny))[:, None] * np.ones((1, g.nx))
    hits = np.zeros((g.ny, g.nx), dtype=np.int64)
    w = np.zeros((4, g.ny, g.nx))
    material = np.zeros((g.ny, g.nx), dtype=np.int64)
    for r in c.regions:
        m = (x >= r.x_min) & (x < r.x_max)
        if g.dim == 2:
            m &= (y >= r.y_min) & (y < r.y_max)
        hits += m
        for q, v in enumerate((r.rho, r.u, r.v, r.p)):
            w[q][m] = v
        material[m] = r.material - 1
    if np.any(hits != 1):
        jj, ii = np.argwhere(hits != 1)[0]
        raise G.ConfigError("cell center (%f,%f) is covered by %d regions; regions must "
                            "tile the domain exactly" % (x[jj, ii], y[jj, ii], hits[jj, ii]))
    if c.material_gammas:
        gamma = np.asarray(c.material_gammas, dtype=np.float64)[material]
    else:
        gamma = np.full((g.ny, g.nx), c.gamma)
    cons = G.conserved_from_primitive(w[0], w[1], w[2], w[3], gamma)
    for q in range(4):
        g.interior(f)[q] = cons[q]
    if c.material_gammas:
        for k in range(n_mat):
            g.interior(mat.partial)[k] = np.where(material == k, w[0], 0.0)
    return f, (mat if c.material_gammas else None)


def triple_point(nx: int = 256, ny: int = 110, steps: int = G.INT64_MAX) -> MatCase:
    """proj/cases/triple_point.case: three states, three materials, closed vessel."""
    g = G.make_grid_2d(nx, ny, 0.0, 7.0, 0.0, 3.0)
    regions = (Region(0.0, 1.0, 0.0, 3.0, 1.0, 0.0, 0.0, 1.0, 1),
               Region(1.0, 7.0, 1.5, 3.0, 0.125, 0.0, 0.0, 0.1, 2),
               Region(1.0, 7.0, 0.0, 1.5, 1.0, 0.0, 0.0, 0.1, 3))
    return MatCase("triple_point", g, G.BoundaryCondition.uniform(G.REFLECTIVE), 1.4,
                   (1.5, 1.4, 1.5), regions, G.SchemeParams(beta=1.5), 0.25, 3.3530, steps)


def material_contact_1d(n: int = 64, gammas=(1.4, 1.4), gamma: float = 1.4,
                        steps: int = 100) -> MatCase:
    """test_multimat.cpp:62-110 / 112-137: a density contact advected through a
    periodic box (equal or unequal gammas), CFL 0.25, no time limit."""
    g = G.make_grid_1d(n, 0.0, 1.0)
    regions = (Region(0.0, 0.5, 0.0, 1.0, 1.0, 1.0, 0.0, 1.0, 1),
               Region(0.5, 1.0, 0.0, 1.0, 0.35, 1.0, 0.0, 1.0, 2))
    bc = G.BoundaryCondition(G.PERIODIC, G.PERIODIC, G.TRANSMISSIVE, G.TRANSMISSIVE)
    return MatCase("contact_1d", g, bc, gamma, tuple(gammas), regions, G.SchemeParams(), 0.25,
                   1e30, steps)


# ---------------------------------------------------------------- generators
class _MT19937_64:
    """std::mt19937_64 with integer seeding (the oracle restates the same)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mti = 312

    def __call__(self) -> int:
        M = 0xFFFFFFFFFFFFFFFF
        UM, LM, A = 0xFFFFFFFF80000000, 0x7FFFFFFF, 0xB5026F5AA96619E9
        mt = self.mt
        if self.mti >= 312:
            for i in range(312):
                x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM)
                mt[i] = mt[(i + 156) % 312] ^ (x >> 1) ^ (A if x & 1 else 0)
            self.mti = 0
        x = mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000 & M
        x ^= (x << 37) & 0xFFF7EEE000000000 & M
        x ^= x >> 43
        return x & M


def fourier_modes(seed: int):
    """Per field k and mode m: (kx, ky, a, phi), drawn in that order."""
    two_pi = 6.283185307179586476925286766559
    rng = _MT19937_64(seed)
    modes = []
    for _k in range(4):
        row = []
        for _m in range(8):
            kx = 1 + rng() % 8
            ky = 1 + rng() % 8
            a = float(rng() >> 11) * 2.0**-53
            phi = two_pi * (float(rng() >> 11) * 2.0**-53)
            row.append((kx, ky, a, phi))
        modes.append(row)
    return modes


def fourier_tables(seed: int, g: G.CartesianGrid):
    """1D tables: tx[k,m,0/1,i] = sin/cos(2 pi kx x_i + phi), ty[k,m,0/1,j] = sin/cos(2 pi ky y_j),
    amp[k,m] = a.  Uses libm through ``math`` so values match the C oracle bit for bit."""
    two_pi = 6.283185307179586476925286766559
    modes = fourier_modes(seed)
    tx = np.empty((4, 8, 2, g.nx))
    ty = np.empty((4, 8, 2, g.ny))
    amp = np.empty((4, 8))
    xs = [g.x0 + (i + 0.5) * g.dx for i in range(g.nx)]
    ys = [g.y0 + (j + 0.5) * g.dy for j in range(g.ny)]
    sin, cos = math.sin, math.cos
    for k in range(4):
        for m in range(8):
            kx, ky, a, phi = modes[k][m]
            amp[k, m] = a
            ax = [two_pi * (kx * x) + phi for x in xs]
            tx[k, m, 0] = [sin(t) for t in ax]
            tx[k, m, 1] = [cos(t) for t in ax]
            ay = [two_pi * (ky * y) for y in ys]
            ty[k, m, 0] = [sin(t) for t in ay]
            ty[k, m, 1] = [cos(t) for t in ay]
    return tx, ty, amp


def fourier_raw(tx, ty, amp) -> np.ndarray:
    """f[k, j, i] = sum_m a (sx_i cy_j + cx_i sy_j), summed in mode order."""
    ny, nx = ty.shape[-1], tx.shape[-1]
    f = np.zeros((4, ny, nx))
    for k in range(4):
        s = np.zeros((ny, nx))
        for m in range(8):
            term = tx[k, m, 0][None, :] * ty[k, m, 1][:, None] + tx[k, m, 1][None, :] * ty[k, m, 0][:, None]
            s = s + amp[k, m] * term
        f[k] = s
    return f


def fourier_primitives(f: np.ndarray):
    """Normalise by max |f_k| and map to (rho, u, v, p) (BASELINE config 4)."""
    M = [np.max(np.abs(f[k])) for k in range(4)]
    rho = 1.0 + 0.2 * (f[0] / M[0])
    u = 0.5 * (f[1] / M[1])
    v = 0.5 * (f[2] / M[2])
    p = 1.0 + 0.2 * (f[3] / M[3])
    return rho, u, v, p


def initial_field(case: Case) -> np.ndarray:
    """Host initial state in the reference's ghosted layout (ghosts zero, run.cpp:29-78)."""
    g = case.grid
    f = G.new_field(g)
    i = np.arange(g.gx, g.gx + g.nx)
    j = np.arange(g.gy, g.gy + g.ny)
    x = g.xc(i)[None, :] * np.ones((g.ny, 1))
    y = g.yc(j)[:, None] * np.ones((1, g.nx))
    shape = (g.ny, g.nx)
    if case.init == "riemann_x":
        left = x < 0.5
        rho = np.where(left, 1.0, 0.125)
        u = np.zeros(shape)
        v = np.zeros(shape)
        p = np.where(left, 1.0, 0.1)
    elif case.init == "quadrant":
        # (rho, u, v, p) per quadrant; x >= 0.5 is "east", y >= 0.5 is "north"
        east, north = x >= 0.5, y >= 0.5
        table = {(True, True): (1.5, 0.0, 0.0, 1.5),
                 (False, True): (0.5323, 1.206, 0.0, 0.3),
                 (False, False): (0.138, 1.206, 1.206, 0.029),
                 (True, False): (0.5323, 0.0, 1.206, 0.3)}
        rho, u, v, p = (np.zeros(shape) for _ in range(4))
        for (e, n), w in table.items():
            m = (east == e) & (north == n)
            rho[m], u[m], v[m], p[m] = w
    elif case.init == "sedov":
        rho = np.ones(shape)
        u = np.zeros(shape)
        v = np.zeros(shape)
        p = np.full(shape, 1e-5)
        pc = (case.gamma - 1.0) * E0_SEDOV / (9.0 * g.dx * g.dy)
        c0x, c0y = g.nx // 2 - 1, g.ny // 2 - 1
        p[c0y:c0y + 3, c0x:c0x + 3] = pc
    elif case.init == "fourier":
        tx, ty, amp = fourier_tables(case.seed, g)
        rho, u, v, p = fourier_primitives(fourier_raw(tx, ty, amp))
    else:
        raise G.ConfigError(f"unknown init kind {case.init}")
    r, mx, my, e = G.conserved_from_primitive(rho, u, v, p, case.gamma)
    g.interior(f)[0], g.interior(f)[1], g.interior(f)[2], g.interior(f)[3] = r, mx, my, e
    return f
