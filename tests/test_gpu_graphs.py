"""GPU: CUDA-graph batches of lf_advance (fused_step.cu run_batch).  A batch runs launch
by launch the first time its key is seen, is captured when the key comes back and is
replayed from then on; all three must continue one run with the bits of single
heun_step calls (which never use graphs), boundary-outflow sums included."""
import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import assert_fields_equal, diag_array

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nx,ny,path", [(480, 300, "fused"), (250, 600, "twopass")])
def test_graph_batches_continue_a_run_bit_for_bit(cuda, nx, ny, path):
    q = CS.quadrant(64, 10)   # transmissive walls: outflow sums on the side stream
    g = G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 1.0)
    case = CS.Case("quadrant_rect", g, q.bc, q.gamma, q.params, q.cfl, 1e30, 10 ** 9, q.init)
    f0 = CS.initial_field(case)
    ctl = G.TimeControls(case.cfl, 1e30)
    # reference run: single steps
    a = LagfluxSolver(g, case.bc, case.gamma, case.params)
    assert a.resolved_path() == path
    sa = G.SolverState(field=f0.copy())
    for _ in range(96):
        a.heun_step(sa, ctl, 1e30)
    a.sync_to_host(sa)
    # six batches of 16: launch by launch, captured, then replayed four times
    b = LagfluxSolver(g, case.bc, case.gamma, case.params)
    sb = G.SolverState(field=f0.copy())
    l0 = b.launch_count()
    for _ in range(6):
        assert b.advance(sb, ctl, 16) == 16
    assert b.launch_count() - l0 >= 96   # replays count their kernels
    b.sync_to_host(sb)
    assert_fields_equal(g.interior(sb.field), g.interior(sa.field), f"{nx}x{ny} {path}")
    assert np.array_equal(diag_array(sb), diag_array(sa))
    assert np.array_equal(np.array(sb.boundary_outflow), np.array(sa.boundary_outflow))
