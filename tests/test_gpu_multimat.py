"""GPU: multimaterial partial-density transport (csrc/material_kernels.cu) through
the C ABI, against golden vectors from the compiled reference and the oracle.

Bar: bit equality per element (==) of the field, the partial densities, the
per-step dt / time / min rho / min p and the boundary outflow -- the same bar as
the single-material path.  The reference's own physics checks of
test_multimat.cpp:62-137 are asserted on the GPU results as well.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import assert_fields_equal, diag_array, load_golden
from test_oracle_multimat import MAT_CASES, run_oracle_mat

pytestmark = pytest.mark.gpu


def run_gpu_mat(c, devices=(0,), field=None, partial=None, steps=None, use_advance=False,
                path="auto"):
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas), devices=devices,
                      path=path)
    state = G.SolverState(field=np.array(f0 if field is None else field))
    mat = MM.MaterialCells(c.grid, len(c.material_gammas), m0.partial if partial is None else partial)
    n = c.max_steps if steps is None else steps
    controls = G.TimeControls(c.cfl, c.t_final, n)
    if use_advance:
        s.attach(state)
        while state.step < n:
            if s.advance(state, controls, n, mat) == 0:
                break
    else:
        for _ in range(n):
            s.heun_step(state, controls, c.t_final, mat)
    s.sync_to_host(state, mat=mat)
    s.close()
    return state, mat


@pytest.mark.parametrize("path", ["auto", "twopass", "staged"])
@pytest.mark.parametrize("name", list(MAT_CASES))
def test_multimaterial_golden_bitwise(cuda, name, path):
    """(auto: the small-grid path on these grids; twopass: the two-pass material kernels
    in 2D, the stage-wise kernels in 1D, where the two-pass kernels do not run)"""
    c = MAT_CASES[name]
    gold = load_golden(name)
    state, mat = run_gpu_mat(c, path=path)
    g = c.grid
    assert_fields_equal(g.interior(state.field), gold["final"], name)
    assert_fields_equal(g.interior(mat.partial), gold["final_partial"], name + "/partials")
    assert np.array_equal(diag_array(state)[:, :4], gold["diag"][:, :4])
    assert np.array_equal(np.array(state.boundary_outflow), gold["outflow"])


@pytest.mark.parametrize("name", ["mm_triple_70x30", "mm_quadrant_48x40"])
@pytest.mark.parametrize("devices", [(0, 0), (0, 0, 0)])
def test_multimaterial_slabs_equal_single(cuda, name, devices):
    c = MAT_CASES[name]
    gold = load_golden(name)
    state, mat = run_gpu_mat(c, devices=devices)
    g = c.grid
    assert_fields_equal(g.interior(state.field), gold["final"], name)
    assert_fields_equal(g.interior(mat.partial), gold["final_partial"], name + "/partials")
    assert np.array_equal(diag_array(state)[:, :4], gold["diag"][:, :4])


def test_multimaterial_advance_and_paths(cuda):
    """lf_advance and every requested path run the material step exactly."""
    c = MAT_CASES["mm_triple_70x30"]
    gold = load_golden("mm_triple_70x30")
    for kw in ({"use_advance": True}, {"path": "fused"}, {"path": "twopass"}):
        state, mat = run_gpu_mat(c, **kw)
        assert_fields_equal(c.grid.interior(state.field), gold["final"], str(kw))
        assert_fields_equal(c.grid.interior(mat.partial), gold["final_partial"], str(kw))


def test_multimaterial_clamped_fractions_vs_oracle(cuda):
    c = MAT_CASES["mm_quadrant_48x40"]
    f0, m0 = CS.regions_field(c)
    rng = np.random.default_rng(11)
    p = m0.partial * (1.0 + rng.uniform(-1e-13, 1e-13, m0.partial.shape))
    ostate, omat = run_oracle_mat(c, partial=p, steps=12)
    state, mat = run_gpu_mat(c, partial=p, steps=12)
    g = c.grid
    assert_fields_equal(g.interior(state.field), g.interior(ostate.field), "field")
    assert_fields_equal(g.interior(mat.partial), g.interior(omat.partial), "partials")
    assert np.array_equal(diag_array(state)[:, :4], diag_array(ostate)[:, :4])


def test_fraction_failure_text_matches_oracle(cuda):
    c = MAT_CASES["mm_triple_70x30"]
    f0, m0 = CS.regions_field(c)
    p = m0.partial.copy()
    p[1, c.grid.gy + 7, c.grid.gx + 33] *= -0.5
    p[0, c.grid.gy + 9, c.grid.gx + 3] *= 1.1
    with pytest.raises(G.InvalidStateError) as eo:
        run_oracle_mat(c, partial=p, steps=1)
    with pytest.raises(G.InvalidStateError) as eg:
        run_gpu_mat(c, partial=p, steps=1)
    assert str(eg.value) == str(eo.value)


def test_step_without_material_storage_is_an_error(cuda):
    c = MAT_CASES["mm_triple_70x30"]
    f0, _ = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas))
    with pytest.raises(G.ConfigError):
        s.heun_step(G.SolverState(field=f0), G.TimeControls(c.cfl, c.t_final), c.t_final)
    with pytest.raises(G.ConfigError, match="must lie in"):
        LagfluxSolver(c.grid, c.bc, materials=MM.MaterialSet((1.4, 3.5)))


def test_two_material_contact_physics(cuda):
    """test_multimat.cpp:62-110 on the GPU result: partial masses add up to rho,
    no pressure oscillation at the interface, per-material conservation."""
    c = CS.material_contact_1d(64, (1.4, 1.4), 1.4, 100)
    g = c.grid
    f0, m0 = CS.regions_field(c)
    mass0 = [g.interior(m0.partial)[k].sum() * g.dx for k in range(2)]
    state, mat = run_gpu_mat(c)
    rho = g.interior(state.field)[0][0]
    part = g.interior(mat.partial)[:, 0]
    assert np.all(np.abs(part[0] + part[1] - rho) < 1e-12 * rho)
    u = g.interior(state.field)[1][0] / rho
    p = 0.4 * (g.interior(state.field)[3][0] - 0.5 * rho * u * u)
    assert np.all(np.abs(u - 1.0) < 1e-10)
    assert np.all(np.abs(p - 1.0) < 1e-10)
    for k in range(2):
        assert abs(part[k].sum() * g.dx - mass0[k]) < 1e-12 * mass0[k]


def test_unequal_gammas_stay_positive(cuda):
    """test_multimat.cpp:112-137: positivity survives the gamma jump."""
    state, _ = run_gpu_mat(CS.material_contact_1d(64, (1.5, 1.4), 1.5, 50))
    for d in state.diagnostics:
        assert d.min_rho > 0.0 and d.min_p > 0.0


@pytest.mark.parametrize("name", ["mm_triple_70x30", "mm_quadrant_48x40", "mm_contact_unequal_64"])
@pytest.mark.parametrize("devices", [(0,), (0, 0, 0)])
def test_device_region_init_equals_host(cuda, name, devices):
    """lf_init_regions == initialize_hydro on the host (regions_field), field and
    partials, and the steps from it equal the golden run."""
    c = MAT_CASES[name]
    if c.grid.dim == 1 and len(devices) > 1:
        pytest.skip("y-slabs need a 2D grid")
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas), devices=devices)
    state = G.SolverState(field=G.new_field(c.grid))
    mat = MM.MaterialCells(c.grid, len(c.material_gammas))
    s.init_regions(state, c.regions, mat)
    s.sync_to_host(state, mat=mat)
    g = c.grid
    assert_fields_equal(g.interior(state.field), g.interior(f0), "field")
    assert_fields_equal(g.interior(mat.partial), g.interior(m0.partial), "partials")
    for _ in range(c.max_steps):
        s.heun_step(state, G.TimeControls(c.cfl, c.t_final), c.t_final, mat)
    s.sync_to_host(state, mat=mat)
    gold = load_golden(name)
    assert_fields_equal(g.interior(state.field), gold["final"], name)
    assert_fields_equal(g.interior(mat.partial), gold["final_partial"], name)


def test_device_region_init_errors(cuda):
    c = MAT_CASES["mm_triple_70x30"]
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas))
    state = G.SolverState(field=G.new_field(c.grid))
    bad = list(c.regions)
    bad[1] = CS.Region(0.5, 7.0, 1.5, 3.0, 0.125, 0.0, 0.0, 0.1, 2)   # overlaps region 1
    with pytest.raises(G.ConfigError) as e1:
        s.init_regions(state, bad)
    with pytest.raises(G.ConfigError) as e2:
        CS.regions_field(CS.MatCase(c.name, c.grid, c.bc, c.gamma, c.material_gammas, tuple(bad),
                                    c.params, c.cfl, c.t_final, c.max_steps))
    assert str(e1.value) == str(e2.value)


def _many_materials_case(n_mat, space=2, time=2):
    """n_mat materials in a 4 x 2 tiling of regions (two reuse a material when n_mat < 8),
    shearing contacts and pressure jumps -- mixed cells of up to four materials appear
    within a few steps."""
    g = G.make_grid_2d(64, 40, 0.0, 1.0, 0.0, 0.625)
    rng = np.random.default_rng(5_000 + n_mat)
    gammas = tuple(float(x) for x in rng.uniform(1.2, 2.2, n_mat))
    regions = []
    for a in range(4):
        for b in range(2):
            m = (2 * a + b) % n_mat + 1
            regions.append(CS.Region(a / 4, (a + 1) / 4, b * 0.3125, (b + 1) * 0.3125,
                                     float(rng.uniform(0.3, 2.0)), float(rng.uniform(-0.6, 0.6)),
                                     float(rng.uniform(-0.6, 0.6)), float(rng.uniform(0.2, 2.0)), m))
    return CS.MatCase(f"mm_{n_mat}mat", g, G.BoundaryCondition(G.REFLECTIVE, G.TRANSMISSIVE,
                                                                G.PERIODIC, G.PERIODIC),
                      1.4, gammas, tuple(regions), G.SchemeParams(spatial_order=space, time_order=time),
                      0.4, 1e30, 12)


@pytest.mark.parametrize("n_mat", [5, 6, 7, 8])
@pytest.mark.parametrize("devices", [(0,), (0, 0)])
def test_five_to_eight_materials_on_the_two_pass_kernels(cuda, n_mat, devices):
    """More than four materials run the two-pass material kernels (up to 8; more go
    stage-wise) with the oracle's bits."""
    c = _many_materials_case(n_mat)
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas), devices=devices,
                      path="twopass")
    st = G.SolverState(field=f0.copy())
    s.heun_step(st, G.TimeControls(c.cfl, c.t_final), c.t_final,
                MM.MaterialCells(c.grid, n_mat, m0.partial.copy()))
    assert s.resolved_path() == "twopass"   # (once the partial densities are resident)
    s.close()
    ref, rmat = run_oracle_mat(c)
    for use_advance in (False, True):
        state, mat = run_gpu_mat(c, devices=devices, use_advance=use_advance, path="twopass")
        g = c.grid
        what = f"{n_mat} materials, {len(devices)} slab(s), advance={use_advance}"
        assert_fields_equal(g.interior(state.field), g.interior(ref.field), what)
        assert_fields_equal(g.interior(mat.partial), g.interior(rmat.partial), what + "/partials")
        assert np.array_equal(diag_array(state)[:, :4], diag_array(ref)[:, :4]), what
        assert np.array_equal(np.array(state.boundary_outflow), np.array(ref.boundary_outflow))


@pytest.mark.parametrize("space,time", [(1, 2), (2, 1)])
def test_eight_materials_other_orders(cuda, space, time):
    c = _many_materials_case(8, space, time)
    ref, rmat = run_oracle_mat(c)
    state, mat = run_gpu_mat(c, use_advance=True)
    g = c.grid
    assert_fields_equal(g.interior(state.field), g.interior(ref.field), f"{space}/{time}")
    assert_fields_equal(g.interior(mat.partial), g.interior(rmat.partial), f"{space}/{time}")


def test_nine_materials_go_stage_wise(cuda):
    c = _many_materials_case(8)
    c = CS.MatCase(c.name, c.grid, c.bc, c.gamma, c.material_gammas + (1.6,), c.regions, c.params,
                   c.cfl, c.t_final, 3)
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas))
    st = G.SolverState(field=f0.copy())
    s.heun_step(st, G.TimeControls(c.cfl, c.t_final), c.t_final, MM.MaterialCells(c.grid, 9, m0.partial.copy()))
    assert s.resolved_path() == "staged"
    s.close()
