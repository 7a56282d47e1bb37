"""LF_PATH_SMALL (csrc/small_step.cu): the step loop of a small grid in one thread-block
cluster (or, beyond one cluster's worth of cells, one cooperative grid), against the
oracle bit for bit.

The golden / error / random suites already run the path (test_gpu_parity.PATHS, and
LF_PATH_AUTO picks it for the small random grids); here: the AUTO choice, every
cluster size from one block to sixteen and past them (strided cells), every boundary
pair, both orders in space and time, 1D, step limits inside a batch, and the sticky
switch to the IEEE arithmetic after a cell leaves the fast arithmetic's box.
"""
import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import assert_fields_equal, diag_array, run_oracle

pytestmark = pytest.mark.gpu


def _run(case, steps, path="small", advance=True, field=None):
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path)
    assert s.resolved_path() == path
    st = G.SolverState(field=CS.initial_field(case) if field is None else np.array(field))
    ctl = G.TimeControls(case.cfl, case.t_final, steps)
    if advance:
        s.attach(st)
        while st.step < steps and st.time < case.t_final:
            if s.advance(st, ctl, steps - st.step) == 0:
                break
    else:
        while st.step < steps and st.time < case.t_final:
            s.heun_step(st, ctl, case.t_final)
    s.sync_to_host(st)
    s.close()
    return st


def _check(case, steps, st, what):
    ref, rdiag = run_oracle(case, steps)
    g = case.grid
    assert_fields_equal(g.interior(st.field), g.interior(ref.field), what)
    assert np.array_equal(diag_array(st)[:, :4], rdiag[:, :4]), what
    assert np.array_equal(np.array(st.boundary_outflow), np.array(ref.boundary_outflow)), what


def test_auto_picks_the_small_path_where_it_is_faster(cuda):
    def resolved(case, **kw):
        s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, **kw)
        p = s.resolved_path()
        s.close()
        return p
    assert resolved(CS.sod()) == "small"                      # BASELINE config 1
    assert resolved(CS.quadrant(128, 1)) == "small"
    assert resolved(CS.quadrant(256, 1)) == "small"                # (grid mode)
    assert resolved(CS.quadrant(320, 1)) == "fused"               # (from 5 * 2^14 cells)
    assert resolved(CS.quadrant(512, 1)) == "fused"
    q512 = CS.quadrant(512, 1)
    assert resolved(CS.Case("q", q512.grid, q512.bc, 1.4, G.SchemeParams(time_order=1), 0.45, 1e300,
                            1, "quadrant")) == "twopass"           # (the fused step is Heun)
    narrow = G.make_grid_2d(130, 800, 0.0, 1.0, 0.0, 1.0)         # a mostly empty second strip
    assert resolved(CS.Case("n", narrow, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2,
                            G.INT64_MAX, "quadrant")) == "small"
    g1 = G.make_grid_1d(100_000, 0.0, 1.0)
    assert resolved(CS.Case("s", g1, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2,
                            G.INT64_MAX, "riemann_x")) == "small"
    assert resolved(CS.quadrant(64, 1), devices=(0, 0)) == "twopass"   # y-slabs
    # materials (once the partial densities are resident): up to 2^15 cells in 2D
    for (nx, ny), want in (((64, 28), "small"), ((256, 200), "twopass")):
        tp = CS.triple_point(nx, ny, 1)
        f0, m0 = CS.regions_field(tp)
        s = LagfluxSolver(tp.grid, tp.bc, tp.gamma, tp.params,
                          materials=MM.make_material_set(tp.material_gammas))
        s.heun_step(G.SolverState(field=f0.copy()), G.TimeControls(tp.cfl, tp.t_final),
                    tp.t_final, MM.MaterialCells(tp.grid, len(tp.material_gammas), m0.partial.copy()))
        assert s.resolved_path() == want, (nx, ny)
        s.close()


# cells per grid: 1 block (224 cell threads) .. 16 blocks .. beyond (strided cells)
@pytest.mark.parametrize("nx,ny", [(12, 9), (40, 13), (64, 56), (128, 32), (160, 40), (300, 37)])
def test_cluster_sizes_equal_oracle(cuda, nx, ny):
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, ny / nx)
    case = CS.Case("q", g, G.BoundaryCondition(G.REFLECTIVE, G.TRANSMISSIVE, G.TRANSMISSIVE,
                                               G.REFLECTIVE), 1.4, G.SchemeParams(), 0.45,
                   CS.STEP_DRIVEN_LIMIT, 12, "quadrant")
    st = _run(case, 12)
    _check(case, 12, st, f"{nx}x{ny}")


BCS = [(G.TRANSMISSIVE, G.TRANSMISSIVE), (G.REFLECTIVE, G.REFLECTIVE),
       (G.TRANSMISSIVE, G.REFLECTIVE), (G.PERIODIC, G.PERIODIC)]


@pytest.mark.parametrize("xb", BCS)
@pytest.mark.parametrize("yb", BCS)
def test_boundary_pairs(cuda, xb, yb):
    g = G.make_grid_2d(23, 17, 0.0, 1.0, 0.0, 0.8)
    case = CS.Case("q", g, G.BoundaryCondition(xb[0], xb[1], yb[0], yb[1]), 1.4,
                   G.SchemeParams(beta=1.5), 0.4, CS.STEP_DRIVEN_LIMIT, 10, "quadrant")
    _check(case, 10, _run(case, 10), f"{xb} {yb}")


@pytest.mark.parametrize("space,time", [(1, 1), (1, 2), (2, 1), (2, 2)])
@pytest.mark.parametrize("dim", [1, 2])
def test_orders_and_dimensions(cuda, space, time, dim):
    if dim == 1:
        g = G.make_grid_1d(333, 0.0, 1.0)
        case = CS.Case("s", g, G.BoundaryCondition(G.REFLECTIVE, G.TRANSMISSIVE), 1.4,
                       G.SchemeParams(spatial_order=space, time_order=time), 0.5, 0.2,
                       G.INT64_MAX, "riemann_x")
        steps = 10_000
    else:
        case = CS.quadrant(48, 25)
        case = CS.Case(case.name, case.grid, case.bc, case.gamma,
                       G.SchemeParams(spatial_order=space, time_order=time), case.cfl,
                       case.t_final, 25, "quadrant")
        steps = 25
    _check(case, steps, _run(case, steps), f"dim {dim} order {space}/{time}")


def test_heun_step_calls_and_limits_inside_a_batch(cuda):
    """Single heun_step calls; lf_advance batches that end at t_final mid-batch and at a
    step count -- the same records as the oracle."""
    case = CS.sod()
    _check(case, 10**6, _run(case, 10**6, advance=False), "heun_step")
    _check(case, 10**6, _run(case, 10**6, advance=True), "advance to t_final")
    _check(case, 77, _run(case, 77, advance=True), "advance 77 steps")


def test_out_of_box_cell_switches_to_ieee_and_stays_exact(cuda):
    """A region of density / pressure 1e-35 (outside the fast arithmetic's box): the first
    step flags, the stage-wise kernels re-run it, the handle continues with the IEEE
    arithmetic -- every step equal to the oracle."""
    base = CS.quadrant(48, 6)
    g = base.grid
    f = CS.initial_field(base)
    f[:, g.gy + 20:g.gy + 24, g.gx + 20:g.gx + 24] *= 1e-35
    ref, rdiag = run_oracle(base, 6, field=f)
    for advance in (False, True):
        st = _run(base, 6, advance=advance, field=f)
        assert_fields_equal(g.interior(st.field), g.interior(ref.field), f"advance={advance}")
        assert np.array_equal(diag_array(st)[:, :4], rdiag[:, :4])


@pytest.mark.parametrize("nx,ny", [(2, 2), (2, 3), (3, 2), (3, 5), (5, 3)])
@pytest.mark.parametrize("bc", [(G.REFLECTIVE, G.PERIODIC), (G.PERIODIC, G.TRANSMISSIVE),
                                (G.TRANSMISSIVE, G.REFLECTIVE)])
def test_tiny_grids_ghost_map(cuda, nx, ny, bc):
    """Grids of 2-5 cells per axis: every ghost of the first two layers maps to an
    interior cell (periodic wrap, reflective images of the far cells)."""
    xb = (bc[0], bc[0])
    yb = (bc[1], bc[1]) if bc[1] == G.PERIODIC else (bc[1], G.TRANSMISSIVE)
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 1.0)
    case = CS.Case("q", g, G.BoundaryCondition(xb[0], xb[1], yb[0], yb[1]), 1.4, G.SchemeParams(),
                   0.3, CS.STEP_DRIVEN_LIMIT, 8, "quadrant")
    _check(case, 8, _run(case, 8), f"{nx}x{ny} {bc}")


@pytest.mark.parametrize("nx", [2, 3])
@pytest.mark.parametrize("bc", [G.TRANSMISSIVE, G.REFLECTIVE, G.PERIODIC])
def test_tiny_1d_grids(cuda, nx, bc):
    g = G.make_grid_1d(nx, 0.0, 1.0)
    case = CS.Case("s", g, G.BoundaryCondition(bc, bc), 1.4, G.SchemeParams(), 0.3,
                   CS.STEP_DRIVEN_LIMIT, 8, "riemann_x")
    _check(case, 8, _run(case, 8), f"1D {nx} {bc}")


@pytest.mark.parametrize("nx,ny", [(256, 256), (1400, 2), (3, 1500), (400, 300)])
def test_grid_mode_equals_oracle(cuda, nx, ny):
    """The cooperative-grid mode: beyond one cluster's worth of cells, and for any grid
    whose boundary faces do not fit in shared memory (perimeter > 1280); its outflow is
    summed after each batch (k_small_sums / k_small_accum)."""
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 1.0)
    case = CS.Case("q", g, G.BoundaryCondition(G.REFLECTIVE, G.TRANSMISSIVE, G.TRANSMISSIVE,
                                               G.REFLECTIVE), 1.4, G.SchemeParams(), 0.4,
                   CS.STEP_DRIVEN_LIMIT, 9, "quadrant")
    _check(case, 9, _run(case, 9), f"{nx}x{ny}")


def test_grid_mode_batches_and_1d(cuda):
    """More steps than one grid-mode batch (256), and a 1D grid of 2^16 cells."""
    case = CS.quadrant(96, 300)   # (9 216 cells: grid mode)
    _check(case, 300, _run(case, 300), "300 steps")
    g = G.make_grid_1d(1 << 16, 0.0, 1.0)
    c1 = CS.Case("s", g, G.BoundaryCondition(G.REFLECTIVE, G.TRANSMISSIVE), 1.4, G.SchemeParams(),
                 0.5, 0.2, 40, "riemann_x")
    _check(c1, 40, _run(c1, 40), "1D 65536")


# ---------------------------------------------------------------- multimaterial
from test_oracle_multimat import MAT_CASES, run_oracle_mat  # noqa: E402
from test_gpu_multimat import run_gpu_mat, _many_materials_case  # noqa: E402


@pytest.mark.parametrize("name", list(MAT_CASES))
@pytest.mark.parametrize("advance", [False, True])
def test_materials_golden_cases_on_the_small_path(cuda, name, advance):
    """The multimaterial goldens (1D contacts, triple point 70x30, four-material quadrant,
    first order) on the small path: field, partials, records, outflow equal the oracle."""
    c = MAT_CASES[name]
    ref, rmat = run_oracle_mat(c)
    state, mat = run_gpu_mat(c, use_advance=advance, path="small")
    g = c.grid
    assert_fields_equal(g.interior(state.field), g.interior(ref.field), name)
    assert_fields_equal(g.interior(mat.partial), g.interior(rmat.partial), name + "/partials")
    assert np.array_equal(diag_array(state)[:, :4], diag_array(ref)[:, :4]), name
    assert np.array_equal(np.array(state.boundary_outflow), np.array(ref.boundary_outflow))


@pytest.mark.parametrize("n_mat", [2, 5, 8])
@pytest.mark.parametrize("mode", ["auto", "grid"])
def test_many_materials_on_the_small_path(cuda, n_mat, mode):
    c = _many_materials_case(n_mat)
    if mode == "grid":   # a grid larger than one cluster's worth of cells
        c = CS.MatCase(c.name, G.make_grid_2d(96, 60, 0.0, 1.0, 0.0, 0.625), c.bc, c.gamma,
                       c.material_gammas, c.regions, c.params, c.cfl, c.t_final, 6)
    ref, rmat = run_oracle_mat(c)
    state, mat = run_gpu_mat(c, use_advance=True, path="small")
    g = c.grid
    assert_fields_equal(g.interior(state.field), g.interior(ref.field), f"{n_mat} {mode}")
    assert_fields_equal(g.interior(mat.partial), g.interior(rmat.partial), f"{n_mat} {mode}")
    assert np.array_equal(diag_array(state)[:, :4], diag_array(ref)[:, :4])
    assert np.array_equal(np.array(state.boundary_outflow), np.array(ref.boundary_outflow))
