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


def _read(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", ["mm_triple_70x30", None])
def test_field_csv_async_snapshots_the_dump_time_state(cuda, tmp_path, name):
    """lf_write_field_csv_async: several dumps queued while stepping continues; each
    file equals the synchronous dump of the state it was queued at."""
    if name:
        c = MAT_CASES[name]
        f0, m0 = CS.regions_field(c)
        ms = MM.make_material_set(c.material_gammas)
        s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
        ref = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
        mat, mref = m0.copy(), m0.copy()
    else:
        c = CS.quadrant(48, 5)
        f0 = CS.initial_field(c)
        s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params)
        ref = LagfluxSolver(c.grid, c.bc, c.gamma, c.params)
        mat = mref = None
    tc = G.TimeControls(c.cfl, c.t_final)
    st, sr = G.SolverState(field=f0.copy()), G.SolverState(field=f0.copy())
    d = str(tmp_path)
    expect = []
    for k in range(4):
        for _ in range(3):
            s.heun_step(st, tc, c.t_final, mat)
            ref.heun_step(sr, tc, c.t_final, mref)
        pa, pb = os.path.join(d, f"a{k}.csv"), os.path.join(d, f"s{k}.csv")
        s.write_field_csv_async(pa, DIGEST + k, sr.time, threads=3)
        ref.write_field_csv(pb, DIGEST + k, sr.time)
        expect.append((pa, pb))
    for _ in range(5):   # stepping on while the dumps are written
        s.heun_step(st, tc, c.t_final, mat)
    s.wait_dumps()
    for pa, pb in expect:
        assert _read(pa) == _read(pb)
    s.wait_dumps()   # nothing pending: a no-op


def test_field_csv_async_errors_at_wait(cuda, tmp_path):
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
    good = os.path.join(str(tmp_path), "never.csv")
    s.write_field_csv_async(good, DIGEST, 0.0)   # queued; fails on the worker
    with pytest.raises(G.InvalidStateError) as eg:
        s.wait_dumps()
    assert not os.path.exists(good)
    with pytest.raises(G.InvalidStateError) as es:
        _ours(str(tmp_path), s, 0.0)
    assert str(eg.value) == str(es.value)
    # an unwritable path is reported at the wait too
    q = CS.quadrant(16, 1)
    s2 = LagfluxSolver(q.grid, q.bc)
    s2.attach(G.SolverState(field=CS.initial_field(q)))
    s2.write_field_csv_async(os.path.join(str(tmp_path), "no", "such", "dir.csv"), 1, 0.0)
    with pytest.raises(Exception, match="cannot open"):
        s2.wait_dumps()
    # destroying a solver with a pending dump waits for it
    s3 = LagfluxSolver(q.grid, q.bc)
    s3.attach(G.SolverState(field=CS.initial_field(q)))
    p3 = os.path.join(str(tmp_path), "late.csv")
    s3.write_field_csv_async(p3, 1, 0.0)
    s3.close()
    assert _read(p3).startswith(b"# config 0000000000000001 time 0\n")
