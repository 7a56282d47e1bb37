"""GPU, full BASELINE size: size-independent properties on config 4 (16384^2).

The CPU oracle needs 77 GB and ~10 s/step here, so full-size correctness rests
on properties that hold exactly or to round-off at any size:
  * every Heun implementation gives the same bits (two-pass, one-kernel fused,
    stage-wise = the reference's phase structure);
  * a y-slab decomposition gives the same bits as one slab;
  * periodic boundaries conserve mass, both momenta and energy
    (test_solver.cpp:254-271 uses 1e-12);
  * the device initial state equals the host generator (checked at 2048^2).
"""
import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 16384
STEPS = 8


def run(path, devices=(0,), steps=STEPS):
    case = CS.smooth(N, steps)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, devices=devices, path=path)
    state = G.SolverState(field=G.new_field(case.grid))
    s.init_fourier(state, case.seed)
    f0 = None
    if path == "twopass":
        f0 = G.new_field(case.grid)
        s.download(f0)
    s.advance(state, G.TimeControls(case.cfl, case.t_final, steps), steps)
    s.sync_to_host(state)
    s.close()
    return case, state, f0


def totals(g, f):
    return [float(np.sum(g.interior(f)[c], dtype=np.float64)) * g.cell_volume() for c in range(4)]


def test_fullsize_paths_agree_and_conserve(cuda):
    case, a, f0 = run("twopass")
    g = case.grid
    t0, t1 = totals(g, f0), totals(g, a.field)
    for c in (0, 3):
        assert abs(t1[c] - t0[c]) <= 1e-12 * abs(t0[c])
    for c in (1, 2):
        assert abs(t1[c] - t0[c]) <= 1e-12 * (abs(t0[0]) + abs(t0[3]))
    ai = g.interior(a.field).copy()
    da = [(d.dt, d.min_rho, d.min_p) for d in a.diagnostics]
    del a
    _, b, _ = run("fused")
    assert np.array_equal(g.interior(b.field) == ai, np.ones_like(ai, dtype=bool))
    assert [(d.dt, d.min_rho, d.min_p) for d in b.diagnostics] == da
    del b
    _, c, _ = run("twopass", devices=(0, 0))
    assert np.array_equal(g.interior(c.field) == ai, np.ones_like(ai, dtype=bool))
    assert [(d.dt, d.min_rho, d.min_p) for d in c.diagnostics] == da


def test_fullsize_staged_equals_fast(cuda):
    _, a, _ = run("twopass", steps=2)
    case, b, _ = run("staged", steps=2)
    g = case.grid
    assert np.array_equal(g.interior(a.field) == g.interior(b.field),
                          np.ones_like(g.interior(a.field), dtype=bool))
    assert [d.dt for d in a.diagnostics] == [d.dt for d in b.diagnostics]


def test_large_initial_state_matches_host(cuda):
    """lf_init_fourier == the host generator (cases.py) on a 2048^2 grid."""
    case = CS.smooth(2048, 1)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params)
    state = G.SolverState(field=G.new_field(case.grid))
    s.init_fourier(state, case.seed)
    s.sync_to_host(state)
    s.close()
    host = CS.initial_field(case)
    g = case.grid
    assert np.array_equal(g.interior(state.field) == g.interior(host),
                          np.ones_like(g.interior(host), dtype=bool))


def test_auto_path_by_size_and_device_memory(cuda):
    """LF_PATH_AUTO: the one-kernel step on every 2D slab past the small-grid path's range
    whose 120-column strips are at least 80 % full, the two-pass kernels on narrower ones
    below 2^23 cells per slab (2^22 in the contract arithmetic; fused_step.cu prefer_fused); at
    BASELINE config 5's 32768^2 only the one-kernel step fits one B200 (the two-pass
    scratch is 206 GB) -- periodic boundaries conserve mass and energy over its steps."""
    for n, ny, math, want in ((2048, 2048, "exact", "fused"), (4096, 4096, "exact", "fused"),
                              (1024, 1024, "contract", "fused"), (512, 512, "exact", "fused"),
                              (130, 4096, "exact", "twopass"), (130, 32768, "exact", "twopass"),
                              (130, 65536, "exact", "fused"), (130, 32768, "contract", "fused"),
                              (16384, 16384, "exact", "fused")):
        case = CS.smooth(n, 1, ny=ny)
        s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, math=math)
        s.init_fourier(G.SolverState(field=None), case.seed)
        assert s.resolved_path() == want, (n, math)
        s.close()
    case = CS.smooth(16384, 1)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path="twopass")
    assert s.resolved_path() == "twopass"
    s.close()
    case = CS.smooth(32768, 3)
    g = case.grid
    s = LagfluxSolver(g, case.bc, case.gamma, case.params)
    st = G.SolverState(field=None)
    s.init_fourier(st, case.seed)
    assert s.resolved_path() == "fused"
    t0 = s.interior_totals()
    assert s.advance(st, G.TimeControls(case.cfl, case.t_final, 3), 3) == 3
    t1 = s.interior_totals()
    s.close()
    for c in (0, 3):
        assert abs(t1[c] - t0[c]) <= 1e-12 * abs(t0[c])
    for c in (1, 2):
        assert abs(t1[c] - t0[c]) <= 1e-12 * (abs(t0[0]) + abs(t0[3]))
