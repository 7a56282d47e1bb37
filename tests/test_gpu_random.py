"""GPU: seeded randomized parity sweep against the C oracle.

Each case draws a grid (1D or 2D, including tiny and ragged sizes: fewer
columns than a warp strip, fewer rows than a chunk, slabs of exactly the 4-row
halo), boundary kinds (valid periodic pairing), the limiter beta, spatial /
time order, a random 3 x 2 tiling of piecewise-constant states with velocities,
a Heun path and 1-3 in-process y-slabs, optionally a random material table
(1-4 materials, random region materials), then requires the GPU field, partial
densities, per-step dt / time / min rho / min p and boundary outflow to equal
the oracle bit for bit (==), or the same error.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import assert_fields_equal, diag_array

pytestmark = pytest.mark.gpu

N_CASES = 120


def draw(seed):
    rng = np.random.default_rng(1_607_087_100 + seed)
    dim = 1 if rng.random() < 0.15 else 2
    nx = int(rng.choice([4, 5, 7, 13, 27, 28, 29, 33, 47, 64, 90, 121]))
    ny = 1 if dim == 1 else int(rng.choice([4, 5, 6, 9, 17, 31, 40, 63]))
    xb = int(rng.integers(0, 3))
    xb = (G.PERIODIC, G.PERIODIC) if xb == 2 else (xb, int(rng.integers(0, 2)))
    yb = int(rng.integers(0, 3))
    yb = (G.PERIODIC, G.PERIODIC) if yb == 2 else (yb, int(rng.integers(0, 2)))
    bc = G.BoundaryCondition(xb[0], xb[1], yb[0], yb[1])
    params = G.SchemeParams(beta=float(rng.uniform(1.0, 2.0)),
                            spatial_order=int(rng.choice([1, 2, 2, 2])),
                            time_order=int(rng.choice([1, 2, 2, 2])))
    g = G.make_grid_1d(nx, 0.0, 1.0) if dim == 1 else G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 0.7)
    mat = rng.random() < 0.3
    n_mat = int(rng.integers(1, 5)) if mat else 0
    gammas = tuple(float(x) for x in rng.uniform(1.1, 2.5, n_mat)) if mat else ()
    # random tiling of the domain by a 3 x 2 block of regions
    xs = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0.1, 0.9, 2)]))
    ys = np.sort(np.concatenate([[0.0, 0.7], rng.uniform(0.1, 0.6, 1)]))
    regions = []
    for a in range(3):
        for b in range(2 if dim == 2 else 1):
            y0, y1 = (ys[b], ys[b + 1]) if dim == 2 else (0.0, 1.0)
            regions.append(CS.Region(xs[a], xs[a + 1], y0, y1, float(rng.uniform(0.2, 2.0)),
                                     float(rng.uniform(-0.8, 0.8)), float(rng.uniform(-0.8, 0.8)) if dim == 2 else 0.0,
                                     float(rng.uniform(0.1, 2.0)),
                                     int(rng.integers(1, n_mat + 1)) if mat else 1))
    case = CS.MatCase(f"random_{seed}", g, bc, 1.4, gammas, tuple(regions), params,
                      float(rng.uniform(0.2, 0.45)), 1e30, int(rng.integers(2, 7)))
    path = str(rng.choice(["staged", "twopass", "fused", "auto"]))
    nslabs = 1 if dim == 1 else int(rng.choice([1, 1, 2, 3]))
    nslabs = min(nslabs, max(1, ny // 4))   # a slab holds at least the 4-row halo
    return case, path, nslabs, mat


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_case_equals_oracle(cuda, seed):
    case, path, nslabs, mat = draw(seed)
    f0, m0 = CS.regions_field(case)
    ms = MM.make_material_set(case.material_gammas) if mat else None
    # oracle
    o = O.OracleSolver(case.grid, case.bc, case.gamma, case.params, materials=ms)
    ostate = G.SolverState(field=f0.copy())
    omat = m0.copy() if mat else None
    oerr = None
    try:
        for _ in range(case.max_steps):
            o.heun_step(ostate, case.cfl, case.t_final, omat)
    except G.Error as e:
        oerr = e
    # GPU
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, materials=ms,
                      devices=(0,) * nslabs, path=path)
    state = G.SolverState(field=f0.copy())
    gmat = m0.copy() if mat else None
    gerr = None
    try:
        for _ in range(case.max_steps):
            s.heun_step(state, G.TimeControls(case.cfl, case.t_final), case.t_final, gmat)
    except G.Error as e:
        gerr = e
    s.sync_to_host(state, mat=gmat)
    what = f"seed {seed}: {case.grid.nx}x{case.grid.ny} {case.bc} {case.params} path={path} slabs={nslabs} mat={mat}"
    assert (oerr is None) == (gerr is None), what + f": {oerr!r} vs {gerr!r}"
    if oerr is not None:
        assert type(oerr) is type(gerr) and str(oerr) == str(gerr), what
    g = case.grid
    assert_fields_equal(g.interior(state.field), g.interior(ostate.field), what)
    if mat and oerr is None:
        assert_fields_equal(g.interior(gmat.partial), g.interior(omat.partial), what + " partials")
    assert np.array_equal(diag_array(state)[:, :4], diag_array(ostate)[:, :4]), what
    assert np.array_equal(np.array(state.boundary_outflow), np.array(ostate.boundary_outflow)), what


def test_slabs_thinner_than_the_halo_are_rejected(cuda):
    g = G.make_grid_2d(16, 6, 0.0, 1.0, 0.0, 1.0)
    with pytest.raises(G.ConfigError, match="at least 4 rows"):
        LagfluxSolver(g, G.BoundaryCondition(), devices=(0, 0))


def draw_stress(seed):
    """Cases built to fail: CFL far past stability and extreme contrasts, so the
    positivity / trace / primitive / fraction checks and their texts are compared."""
    case, path, nslabs, mat = draw(10_000 + seed)
    rng = np.random.default_rng(77 + seed)
    regions = tuple(CS.Region(r.x_min, r.x_max, r.y_min, r.y_max,
                              float(10 ** rng.uniform(-3, 1)), float(rng.uniform(-3, 3)),
                              float(rng.uniform(-3, 3)) if case.grid.dim == 2 else 0.0,
                              float(10 ** rng.uniform(-4, 1)), r.material)
                    for r in case.regions)
    case = CS.MatCase(case.name, case.grid, case.bc, case.gamma, case.material_gammas, regions,
                      case.params, float(rng.uniform(0.9, 3.0)), case.t_final, 8)
    return case, path, nslabs, mat


@pytest.mark.parametrize("seed", range(60))
def test_random_failing_case_equals_oracle(cuda, seed):
    case, path, nslabs, mat = draw_stress(seed)
    f0, m0 = CS.regions_field(case)
    ms = MM.make_material_set(case.material_gammas) if mat else None
    o = O.OracleSolver(case.grid, case.bc, case.gamma, case.params, materials=ms)
    ostate, omat, oerr = G.SolverState(field=f0.copy()), (m0.copy() if mat else None), None
    try:
        for _ in range(case.max_steps):
            o.heun_step(ostate, case.cfl, case.t_final, omat)
    except G.Error as e:
        oerr = e
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, materials=ms,
                      devices=(0,) * nslabs, path=path)
    state, gmat, gerr = G.SolverState(field=f0.copy()), (m0.copy() if mat else None), None
    try:
        for _ in range(case.max_steps):
            s.heun_step(state, G.TimeControls(case.cfl, case.t_final), case.t_final, gmat)
    except G.Error as e:
        gerr = e
    s.sync_to_host(state, mat=gmat)
    what = f"stress {seed}: path={path} slabs={nslabs} mat={mat} cfl={case.cfl:.2f}"
    assert type(oerr) is type(gerr), what + f": {oerr!r} vs {gerr!r}"
    assert str(oerr) == str(gerr), what
    g = case.grid
    # the corrector writes in place before it throws (solver.cpp:507): same state
    assert_fields_equal(g.interior(state.field), g.interior(ostate.field), what)
    rec = lambda st: [(d.step, d.time, d.dt, d.min_rho, d.min_p) for d in st.diagnostics]  # noqa: E731
    assert rec(state) == rec(ostate), what
