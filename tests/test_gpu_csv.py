"""GPU: field dumps (lf_write_field_csv) byte-identical to the reference's own
field_csv (csv.cpp:26-83, compiled into oracle/_ref) for single- and
multimaterial states, 2D and 1D, and the same failure text."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
from test_oracle_multimat import MAT_CASES

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

DIGEST = 0x1607087100ABCDEF


def _ours(tmp_path, s, time, threads=0):
    p = os.path.join(tmp_path, "dump.csv")
    s.write_field_csv(p, DIGEST, time, threads)
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("threads", [1, 7, 0])
def test_field_csv_single_material(cuda, tmp_path, threads):
    case = CS.quadrant(40, 5)
    f0 = CS.initial_field(case)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params)
    state = G.SolverState(field=f0.copy())
    for _ in range(5):
        s.heun_step(state, G.TimeControls(case.cfl, case.t_final), case.t_final)
    s.sync_to_host(state)
    r = O.RefSolver(case.grid, case.bc, case.gamma, case.params)
    r.set_state(state.field)
    assert _ours(str(tmp_path), s, state.time, threads) == r.field_csv(DIGEST, state.time)


def test_field_csv_1d(cuda, tmp_path):
    g = G.make_grid_1d(100, 0.0, 1.0)
    case = CS.Case("sod1d", g, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2,
                   G.INT64_MAX, "riemann_x")
    s = LagfluxSolver(g, case.bc)
    state = G.SolverState(field=CS.initial_field(case))
    for _ in range(20):
        s.heun_step(state, G.TimeControls(0.5, 0.2), 0.2)
    s.sync_to_host(state)
    r = O.RefSolver(g, case.bc)
    r.set_state(state.field)
    assert _ours(str(tmp_path), s, state.time) == r.field_csv(DIGEST, state.time)


@pytest.mark.parametrize("name", ["mm_triple_70x30", "mm_quadrant_48x40"])
def test_field_csv_multimaterial(cuda, tmp_path, name):
    c = MAT_CASES[name]
    f0, m0 = CS.regions_field(c)
    ms = MM.make_material_set(c.material_gammas)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    state = G.SolverState(field=f0.copy())
    mat = m0.copy()
    for _ in range(10):
        s.heun_step(state, G.TimeControls(c.cfl, c.t_final), c.t_final, mat)
    s.sync_to_host(state, mat=mat)
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    r.set_state(state.field)
    r.set_partials(mat.partial)
    assert _ours(str(tmp_path), s, state.time) == r.field_csv(DIGEST, state.time)


def test_field_csv_fraction_failure(cuda, tmp_path):
    c = MAT_CASES["mm_triple_70x30"]
    f0, m0 = CS.regions_field(c)
    p = m0.partial.copy()
    p[2, c.grid.gy + 4, c.grid.gx + 50] *= 1.5
    ms = MM.make_material_set(c.material_gammas)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    state = G.SolverState(field=f0.copy())
    mat = MM.MaterialCells(c.grid, 3, p)
    s.attach(state)
    s._attach_mat(mat)
    with pytest.raises(G.InvalidStateError) as eg:
        _ours(str(tmp_path), s, 0.0)
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    r.set_state(f0)
    r.set_partials(p)
    with pytest.raises(G.InvalidStateError) as er:
        r.field_csv(DIGEST, 0.0)
    assert str(eg.value) == str(er.value)
