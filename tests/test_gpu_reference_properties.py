"""GPU: the reference's own property tests (proj/tests/test_solver.cpp:182-369)
restated on the CUDA path, at the reference's sizes and larger, on every Heun path.

  * a uniform field is a fixed point of both stages           (:182-201)
  * a single stage balances the boundary fluxes               (:203-223)
  * periodic runs conserve the global invariants              (:254-271)
  * pure contact advection keeps velocity and pressure        (:273-291)
  * one step commutes with a quarter turn (bit-equal dt)      (:293-344)
  * results are bitwise identical for any worker count        (:346-369):
    here, across runs, paths and y-slab counts
"""
import math

import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver

pytestmark = pytest.mark.gpu

PATHS = ["staged", "twopass", "fused"]
FREE = G.TimeControls(0.25, 1e30)   # kFreeRun (test_solver.cpp:20)
TWO_PI = 6.283185307179586476925286766559


def uniform(g, w):
    f = G.new_field(g)
    r, mx, my, e = G.conserved_from_primitive(*w, 1.4)
    for c, v in enumerate((r, mx, my, e)):
        g.interior(f)[c] = v
    return f


def sod(g):
    f = G.new_field(g)
    x = g.xc(np.arange(g.gx, g.gx + g.nx))
    left = x < 0.5
    r, mx, my, e = G.conserved_from_primitive(np.where(left, 1.0, 0.125), 0.0 * x, 0.0 * x,
                                              np.where(left, 1.0, 0.1), 1.4)
    for c, v in enumerate((r, mx, my, e)):
        g.interior(f)[c][:] = v
    return f


def interior_totals(g, f):
    """grid.cpp:123-134"""
    vol = g.dx * g.dy if g.dim == 2 else g.dx
    return [float(np.sum(g.interior(f)[c], dtype=np.float64)) * vol for c in range(4)]


def step(g, bc, f, n, path, devices=(0,), params=G.SchemeParams()):
    s = LagfluxSolver(g, bc, 1.4, params, path=path, devices=devices)
    st = G.SolverState(field=f.copy())
    for _ in range(n):
        s.heun_step(st, FREE, 1e30)
    s.sync_to_host(st)
    s.close()
    return st


@pytest.mark.parametrize("path", PATHS)
def test_uniform_field_is_a_fixed_point(cuda, path):
    g1 = G.make_grid_1d(32, 0.0, 1.0)
    f1 = uniform(g1, (1.2, 0.7, 0.0, 2.0))
    s1 = LagfluxSolver(g1, G.BoundaryCondition(), path=path)
    out = G.new_field(g1)
    s1.euler_stage(f1, 1e-3, out)
    assert np.array_equal(g1.interior(out), g1.interior(f1))
    for n in (12, 200):
        g2 = G.make_grid_2d(n, 9 if n == 12 else 150, 0.0, 1.0, 0.0, 1.0)
        f2 = uniform(g2, (1.2, 0.7, -0.4, 2.0))
        st = step(g2, G.BoundaryCondition(), f2, 1, path)
        assert np.array_equal(g2.interior(st.field), g2.interior(f2))


def test_single_stage_balances_boundary_fluxes(cuda):
    from oracle import oracle as O
    g = G.make_grid_1d(100, 0.0, 1.0)
    f = sod(g)
    s = LagfluxSolver(g, G.BoundaryCondition())
    dt = 1e-3
    out = G.new_field(g)
    s.euler_stage(f, dt, out)
    before, after = interior_totals(g, f), interior_totals(g, out)
    lib = O.oracle_lib()
    fl, fr = np.zeros(4), np.zeros(4)
    for w, dst in (((1.0, 0.0, 0.0, 1.0), fl), ((0.125, 0.0, 0.0, 0.1), fr)):
        a = np.array(w)
        lib.lfo_edge_flux(a.ctypes.data_as(O.DP), a.ctypes.data_as(O.DP), 1.0, 0.0, 1.4,
                          dst.ctypes.data_as(O.DP))
    assert math.isclose(after[0] - before[0], -dt * (fr[0] - fl[0]), rel_tol=1e-12)
    assert abs(after[1] - before[1] + dt * (fr[1] - fl[1])) < 1e-15
    assert math.isclose(after[3] - before[3], -dt * (fr[3] - fl[3]), rel_tol=1e-12)


@pytest.mark.parametrize("path", PATHS)
def test_periodic_runs_conserve_invariants(cuda, path):
    case = CS.smooth(96, 120, ny=64, y_extent=64 / 96)
    f0 = CS.initial_field(case)
    st = step(case.grid, case.bc, f0, 120, path, params=case.params)
    t0, t1 = interior_totals(case.grid, f0), interior_totals(case.grid, st.field)
    for c in (0, 3):
        assert abs(t1[c] - t0[c]) < 1e-12 * abs(t0[c])
    for c in (1, 2):   # zero-mean momenta: absolute
        assert abs(t1[c] - t0[c]) < 1e-13


@pytest.mark.parametrize("path", PATHS)
def test_pure_contact_keeps_velocity_and_pressure(cuda, path):
    for dim in (1, 2):
        g = G.make_grid_1d(64, 0.0, 1.0) if dim == 1 else G.make_grid_2d(64, 32, 0.0, 1.0, 0.0, 0.5)
        f = G.new_field(g)
        x = g.xc(np.arange(g.gx, g.gx + g.nx))[None, :] * np.ones((g.ny, 1))
        rho = np.where(x < 0.5, 1.0, 2.0)
        r, mx, my, e = G.conserved_from_primitive(rho, 1.0 + 0 * x, 0 * x, 1.0 + 0 * x, 1.4)
        for c, v in enumerate((r, mx, my, e)):
            g.interior(f)[c] = v
        bc = G.BoundaryCondition(G.PERIODIC, G.PERIODIC, G.PERIODIC if dim == 2 else G.TRANSMISSIVE,
                                 G.PERIODIC if dim == 2 else G.TRANSMISSIVE)
        st = step(g, bc, f, 100, path)
        I = g.interior(st.field)
        u = I[1] / I[0]
        p = 0.4 * (I[3] - 0.5 * (I[1] * I[1] + I[2] * I[2]) / I[0])
        assert np.all(np.abs(u - 1.0) < 1e-12)
        assert np.all(np.abs(p - 1.0) < 1e-12)


def quarter_turn(g, f):
    """cell (i, j) <- cell (j, n-1-i), (u, v) <- (-v, u)  (test_solver.cpp:313-320)"""
    n = g.nx
    I = g.interior(f)
    out = G.new_field(g)
    O_ = g.interior(out)
    src = lambda c: I[c].T[:, ::-1]   # noqa: E731  out[j, i] = in[n-1-i, j]
    O_[0] = src(0)
    O_[1] = -src(2)
    O_[2] = src(1)
    O_[3] = src(3)
    return out


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n", [16, 256])
def test_one_step_commutes_with_a_quarter_turn(cuda, path, n):
    g = G.make_grid_2d(n, n, 0.0, 1.0, 0.0, 1.0)
    bc = G.BoundaryCondition.uniform(G.PERIODIC)
    x = g.xc(np.arange(g.gx, g.gx + g.nx))[None, :] * np.ones((n, 1))
    y = g.yc(np.arange(g.gy, g.gy + g.ny))[:, None] * np.ones((1, n))
    sx, sy = np.sin(TWO_PI * x), np.sin(TWO_PI * y)
    cx, cy = np.cos(TWO_PI * x), np.cos(TWO_PI * y)
    base = G.new_field(g)
    r, mx, my, e = G.conserved_from_primitive(1.0 + 0.3 * sx * sy, 0.2 * cx, -0.3 * sy,
                                              1.0 + 0.2 * cx * cy, 1.4)
    for c, v in enumerate((r, mx, my, e)):
        g.interior(base)[c] = v
    a = step(g, bc, base, 1, path)
    b = step(g, bc, quarter_turn(g, base), 1, path)
    assert a.diagnostics[0].dt == b.diagnostics[0].dt
    ra = g.interior(quarter_turn(g, a.field))
    rb = g.interior(b.field)
    assert np.all(np.abs(rb - ra) <= 1e-13 * (1.0 + np.abs(rb)))


def test_bitwise_identical_across_runs_paths_and_slabs(cuda):
    g = G.make_grid_2d(96, 64, 0.0, 1.0, 0.0, 0.5)
    f = sod(g)
    bc = G.BoundaryCondition.uniform(G.REFLECTIVE)
    ref = step(g, bc, f, 20, "staged")
    for path in PATHS:
        for devices in ((0,), (0, 0), (0, 0, 0, 0)):
            for _ in range(2):
                st = step(g, bc, f, 20, path, devices=devices)
                assert np.array_equal(g.interior(st.field), g.interior(ref.field)), (path, devices)
                assert [d.dt for d in st.diagnostics] == [d.dt for d in ref.diagnostics]
