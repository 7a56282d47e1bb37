"""Multimaterial oracle pins (CPU): the C restatement against the reference's
own known answers (test_multimat.cpp:19-60), against golden vectors generated
from the compiled reference (tests/golden/make_golden.py mat), and live against
the reference where oracle/_ref is present.  Also the product's host helpers
(paper_1607_08710_b200/multimat.py) against the same answers."""
import importlib.util
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import multimat as MM
from helpers import load_golden

HERE = os.path.dirname(os.path.abspath(__file__))


def _mat_cases():
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "golden", "make_golden.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.golden_mat_cases()


MAT_CASES = _mat_cases()
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def run_oracle_mat(c, field=None, partial=None, steps=None):
    f0, m0 = CS.regions_field(c)
    f = f0 if field is None else field
    mat = MM.MaterialCells(c.grid, len(c.material_gammas), m0.partial if partial is None else partial)
    s = O.OracleSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas))
    state = G.SolverState(field=np.array(f))
    for _ in range(c.max_steps if steps is None else steps):
        s.heun_step(state, c.cfl, c.t_final, mat)
    return state, mat


# ------------------------------------------------------------ element answers
IMPLS = {"host": (MM.mass_fraction_fluxes, lambda gs, y: MM.mixed_cell_gamma(MM.MaterialSet(tuple(gs)), y)),
         "oracle": (O.oracle_mass_fraction_fluxes, O.oracle_mixed_cell_gamma)}


@pytest.mark.parametrize("impl", list(IMPLS))
def test_mass_fraction_fluxes_known_answers(impl):
    mff = IMPLS[impl][0]
    assert list(mff(3.7, [1.0])) == [3.7]
    assert list(mff(0.0, [0.3, 0.7])) == [0.0, 0.0]
    assert list(mff(2.0, [0.3, 0.7])) == [0.6, 1.4]
    rng = np.random.default_rng(0x3A7)
    for _ in range(1000):
        y0 = rng.uniform(0.0, 1.0)
        y1 = rng.uniform(0.0, 1.0 - y0)
        y = [y0, y1, 1.0 - y0 - y1]
        flux = rng.uniform(-10.0, 10.0)
        out = mff(flux, y)
        rest = flux
        for f in out:
            rest -= f
        assert rest == 0.0   # the complement makes the sequential sum exact


@pytest.mark.parametrize("impl", list(IMPLS))
def test_mixed_cell_gamma_known_answers(impl):
    mcg = IMPLS[impl][1]
    assert mcg([1.5, 1.4], [1.0, 0.0]) == 1.5
    assert mcg([1.5, 1.4], [0.0, 1.0]) == 1.4
    assert abs(mcg([1.5, 1.4], [0.5, 0.5]) - 1.4444444444444444) < 1e-15


@needs_ref
def test_element_functions_equal_reference():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 6))
        y = rng.dirichlet(np.ones(n))
        if rng.random() < 0.3:
            y = np.zeros(n)
            y[rng.integers(0, n)] = 1.0
        gs = rng.uniform(1.05, 3.0, n)
        flux = rng.uniform(-5, 5)
        assert np.array_equal(O.oracle_mass_fraction_fluxes(flux, y), O.ref_mass_fraction_fluxes(flux, y))
        assert np.array_equal(np.array(MM.mass_fraction_fluxes(flux, list(y))),
                              O.ref_mass_fraction_fluxes(flux, y))
        assert O.oracle_mixed_cell_gamma(gs, y) == O.ref_mixed_cell_gamma(gs, y)
        assert MM.mixed_cell_gamma(MM.MaterialSet(tuple(gs)), list(y)) == O.ref_mixed_cell_gamma(gs, y)
    for part, rho in [(0.5, 1.0), (1.0 + 5e-12, 1.0), (-5e-12, 1.0), (1.0 + 1e-9, 1.0), (-1e-9, 1.0)]:
        rv, rfail = O.ref_clamped_fraction(part, rho)
        ov, ofail = O.oracle_clamped_fraction(part, rho)
        assert rfail == ofail
        if not rfail:
            assert rv == ov == MM.clamped_fraction(part, rho)
        else:
            with pytest.raises(G.InvalidStateError):
                MM.clamped_fraction(part, rho)


def test_make_material_set_errors():
    with pytest.raises(G.ConfigError, match="needs at least one material"):
        MM.make_material_set([])
    with pytest.raises(G.ConfigError, match=r"must lie in \(1, 3\], got 0.900000"):
        MM.make_material_set([1.4, 0.9])
    with pytest.raises(G.ConfigError, match="at most 16"):
        MM.make_material_set([1.4] * 17)
    g = G.make_grid_2d(8, 8, 0, 1, 0, 1)
    for bad in ([], [1.4, 0.9], [1.4] * 17, [3.5]):
        with pytest.raises(G.ConfigError) as e1:
            O.OracleSolver(g, G.BoundaryCondition(), materials=MM.MaterialSet(tuple(bad)))
        if O.ref_available():
            with pytest.raises(G.ConfigError) as e2:
                O.ref_make_material_set(bad)
            assert str(e1.value) == str(e2.value)


# ------------------------------------------------------------ whole steps
@pytest.mark.parametrize("name", list(MAT_CASES))
def test_oracle_matches_multimaterial_golden(name):
    c = MAT_CASES[name]
    gold = load_golden(name)
    f0, m0 = CS.regions_field(c)
    g = c.grid
    assert np.array_equal(g.interior(f0), gold["initial"])
    assert np.array_equal(g.interior(m0.partial), gold["initial_partial"])
    state, mat = run_oracle_mat(c)
    assert np.array_equal(g.interior(state.field), gold["final"])
    assert np.array_equal(g.interior(mat.partial), gold["final_partial"])
    d = np.array([[x.dt, x.time, x.min_rho, x.min_p] for x in state.diagnostics])
    assert np.array_equal(d, gold["diag"][:, :4])
    assert np.array_equal(np.array(state.boundary_outflow), gold["outflow"])


@needs_ref
def test_oracle_matches_reference_with_clamped_fractions():
    """Partial densities perturbed by ~1e-13 relative: fractions land just
    outside [0, 1] and take the clamp (solver.cpp:108-115)."""
    c = MAT_CASES["mm_quadrant_48x40"]
    f0, m0 = CS.regions_field(c)
    rng = np.random.default_rng(11)
    p = m0.partial.copy()
    p *= 1.0 + rng.uniform(-1e-13, 1e-13, p.shape)
    state, mat = run_oracle_mat(c, partial=p, steps=8)
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas))
    r.set_state(f0)
    r.set_partials(p)
    diag = r.heun_steps(8, c.cfl, c.t_final)
    rf = r.get_state()[0]
    g = c.grid
    assert np.array_equal(g.interior(state.field), g.interior(rf))
    assert np.array_equal(g.interior(mat.partial), g.interior(r.get_partials()))
    assert np.array_equal(np.array([[x.dt, x.time, x.min_rho, x.min_p] for x in state.diagnostics]),
                          diag[:, :4])


@needs_ref
def test_fraction_failure_matches_reference():
    c = MAT_CASES["mm_triple_70x30"]
    f0, m0 = CS.regions_field(c)
    p = m0.partial.copy()
    p[1, c.grid.gy + 7, c.grid.gx + 33] *= -0.5   # a negative partial density
    p[0, c.grid.gy + 9, c.grid.gx + 3] *= 1.1     # and one above rho
    with pytest.raises(G.InvalidStateError) as eo:
        run_oracle_mat(c, partial=p, steps=1)
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas))
    r.set_state(f0)
    r.set_partials(p)
    with pytest.raises(G.InvalidStateError) as er:
        r.heun_steps(1, c.cfl, c.t_final)
    assert str(eo.value) == str(er.value)
    assert "mass fraction out of [0,1] beyond round-off at cell" in str(eo.value)
