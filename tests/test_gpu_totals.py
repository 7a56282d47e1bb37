"""GPU: lf_interior_totals (grid.cpp:122-133) against the oracle and the reference.

The reference's conservation audit sums each component in row-major order; the
device chain must reproduce that order exactly -- across the 1024-element chunks
of a row, across rows, across y-slabs -- so the fields span 16 decades with mixed
signs (a correctly rounded or pairwise sum differs from the ordered one).
"""
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver

pytestmark = pytest.mark.gpu


def wide_field(g, seed):
    rng = np.random.default_rng(seed)
    f = G.new_field(g)
    I = g.interior(f)
    I[...] = rng.standard_normal(I.shape) * 10.0 ** rng.uniform(-8, 8, I.shape)
    return f


GRIDS = [
    ("1d_37", lambda: G.make_grid_1d(37, 0.0, 1.0)),
    ("1d_3001", lambda: G.make_grid_1d(3001, 0.0, 1.0)),
    ("2d_5x4", lambda: G.make_grid_2d(5, 4, 0.0, 1.0, 0.0, 1.0)),
    ("2d_1023x9", lambda: G.make_grid_2d(1023, 9, 0.0, 1.0, 0.0, 0.5)),
    ("2d_1024x8", lambda: G.make_grid_2d(1024, 8, 0.0, 1.0, 0.0, 0.5)),
    ("2d_1025x12", lambda: G.make_grid_2d(1025, 12, 0.0, 1.0, 0.0, 0.5)),
    ("2d_3000x17", lambda: G.make_grid_2d(3000, 17, 0.0, 3.0, 0.0, 0.1)),
]


@pytest.mark.parametrize("name,mk", GRIDS, ids=[n for n, _ in GRIDS])
@pytest.mark.parametrize("devices", [(0,), (0, 0), (0, 0, 0)])
def test_totals_equal_oracle(cuda, name, mk, devices):
    g = mk()
    if g.dim == 1 and len(devices) > 1:
        pytest.skip("1D grids are one slab")
    if g.dim == 2 and g.ny < 4 * len(devices):
        pytest.skip("slabs need >= 4 rows")
    f = wide_field(g, hash(name) & 0xffff)
    s = LagfluxSolver(g, G.BoundaryCondition(), devices=devices)
    s.upload(f)
    got = s.interior_totals()
    s.close()
    assert got == O.oracle_interior_totals(g, f)
    if O.ref_available():
        ref = O.RefSolver(g, G.BoundaryCondition())
        ref.set_state(f)
        assert got == ref.interior_totals()


@pytest.mark.parametrize("path", ["twopass", "staged"])
def test_totals_after_steps_match_reference_audit(cuda, path):
    """acceptance.cpp:226-266 audits interior_totals before and after a run: the
    device totals of the device state equal the oracle's on the downloaded state."""
    case = CS.sedov(256, 20)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path)
    st = G.SolverState(field=CS.initial_field(case))
    t0 = None
    for k in range(20):
        s.heun_step(st, G.TimeControls(case.cfl, 1e30), 1e30)
        if k == 0:
            t0 = s.interior_totals()
    t1 = s.interior_totals()
    s.sync_to_host(st)
    s.close()
    assert t1 == O.oracle_interior_totals(case.grid, st.field)
    # reflective walls: mass and energy are conserved to round-off
    for c in (0, 3):
        assert abs(t1[c] - t0[c]) <= 1e-12 * abs(t0[c])


def test_totals_full_size(cuda):
    """BASELINE config 4 size: 16384^2, the chain over 2^28 cells per component."""
    case = CS.smooth(16384, 1)
    g = case.grid
    s = LagfluxSolver(g, case.bc, case.gamma, case.params)
    st = G.SolverState(field=None)
    s.init_fourier(st, case.seed)
    t = time.perf_counter()
    got = s.interior_totals()
    dt = time.perf_counter() - t
    f = G.new_field(g)
    s.download(f)
    s.close()
    assert got == O.oracle_interior_totals(g, f)
    print(f"interior_totals 16384^2: {dt:.3f} s")
