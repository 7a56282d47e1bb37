"""GPU: seeded randomized parity sweep on mid-size 2D grids, where LF_PATH_AUTO picks
between the one-kernel step with short row chunks (wide grids from 5 * 2^14 cells per
slab, fused_step.cu prefer_fused) and the two-pass kernels (narrow grids, slabs below
the limit).  Several 120-column strips, ragged last strips, every boundary pairing,
1-3 in-process y-slabs, random limiter; field, per-step dt / time / min rho / min p and
boundary outflow equal the C oracle bit for bit.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import assert_fields_equal, diag_array

pytestmark = pytest.mark.gpu

N_CASES = 16


def draw(seed):
    rng = np.random.default_rng(2_016_070_871 + seed)
    # strips hold 120 columns: full, nearly full (>= 80 %) and mostly empty last strips
    nx = int(rng.choice([360, 480, 352, 590, 600, 697, 250, 384, 460]))
    ny = int(rng.integers(180, 420))
    xb = int(rng.integers(0, 3))
    xb = (G.PERIODIC, G.PERIODIC) if xb == 2 else (xb, int(rng.integers(0, 2)))
    yb = int(rng.integers(0, 3))
    yb = (G.PERIODIC, G.PERIODIC) if yb == 2 else (yb, int(rng.integers(0, 2)))
    bc = G.BoundaryCondition(xb[0], xb[1], yb[0], yb[1])
    params = G.SchemeParams(beta=float(rng.uniform(1.0, 2.0)), spatial_order=2, time_order=2)
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 0.7)
    xs = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0.1, 0.9, 2)]))
    ys = np.sort(np.concatenate([[0.0, 0.7], rng.uniform(0.1, 0.6, 1)]))
    regions = []
    for a in range(3):
        for b in range(2):
            regions.append(CS.Region(xs[a], xs[a + 1], ys[b], ys[b + 1], float(rng.uniform(0.2, 2.0)),
                                     float(rng.uniform(-0.8, 0.8)), float(rng.uniform(-0.8, 0.8)),
                                     float(rng.uniform(0.1, 2.0)), 1))
    case = CS.MatCase(f"random_mid_{seed}", g, bc, 1.4, (), tuple(regions), params,
                      float(rng.uniform(0.2, 0.45)), 1e30, 4)
    nslabs = int(rng.choice([1, 1, 2, 3]))
    return case, nslabs


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_mid_size_case_on_auto_equals_oracle(cuda, seed):
    case, nslabs = draw(seed)
    f0, _ = CS.regions_field(case)
    o = O.OracleSolver(case.grid, case.bc, case.gamma, case.params)
    ostate = G.SolverState(field=f0.copy())
    for _ in range(case.max_steps):
        o.heun_step(ostate, case.cfl, case.t_final, None)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, devices=(0,) * nslabs, path="auto")
    state = G.SolverState(field=f0.copy())
    # two single steps, then the device-resident loop (the batched enqueue path)
    ctl = G.TimeControls(case.cfl, case.t_final)
    s.heun_step(state, ctl, case.t_final)
    s.heun_step(state, ctl, case.t_final)
    s.advance(state, ctl, case.max_steps - 2)
    resolved = s.resolved_path()
    s.sync_to_host(state)
    what = (f"seed {seed}: {case.grid.nx}x{case.grid.ny} {case.bc} beta={case.params.beta:.3f} "
            f"slabs={nslabs} resolved={resolved}")
    g = case.grid
    assert_fields_equal(g.interior(state.field), g.interior(ostate.field), what)
    assert np.array_equal(diag_array(state)[:, :4], diag_array(ostate)[:, :4]), what
    assert np.array_equal(np.array(state.boundary_outflow), np.array(ostate.boundary_outflow)), what


def test_auto_rule_on_mid_size_grids(cuda):
    """Wide grids past 5 * 2^14 cells per slab take the one-kernel step; grids whose
    last 120-column strip is mostly empty stay on the small-grid path (to 2^17 cells) or
    the two-pass kernels, as do slabs below the limit."""
    def resolved(nx, ny, nslabs=1):
        g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 1.0)
        return LagfluxSolver(g, G.BoundaryCondition(), devices=(0,) * nslabs).resolved_path()
    assert resolved(480, 400) == "fused"        # 4 full strips, 192 000 cells
    assert resolved(590, 300) == "fused"        # 4.9 strips
    assert resolved(250, 400) == "small"        # narrow and up to 2^17 cells: the small-grid path
    assert resolved(250, 600) == "twopass"      # 2.08 strips (the third nearly empty), 150 000 cells
    assert resolved(480, 400, 3) == "twopass"   # 64 000 cells per slab
