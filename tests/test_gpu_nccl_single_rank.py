"""GPU: the distributed code path on the real NCCL (torch's libnccl.so.2), one rank.

The pool exposes one GPU and NCCL refuses two ranks on one device, so the N > 1
decomposition is covered by the thread-rank stand-in (tests/test_gpu_dist_threads.py).
A one-rank communicator still drives every NCCL call of the slab path for real: the
periodic halo exchange is a grouped send / receive to itself (on the fused path on
the comm stream, overlapped with the interior row chunks), the step reductions and
the interior_totals chain are one-rank collectives.  Bit-equal to a plain handle."""
import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver, nccl_unique_id

pytestmark = pytest.mark.gpu


def run(case, path, dist=None, steps=12):
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path, dist=dist)
    st = G.SolverState(field=CS.initial_field(case))
    s.attach(st)
    s.advance(st, G.TimeControls(case.cfl, case.t_final, case.max_steps), steps)
    tot = s.interior_totals()
    out = G.new_field(case.grid)
    s.download(out)
    s.close()
    return out, [(d.dt, d.time, d.min_rho, d.min_p) for d in st.diagnostics], \
        list(st.boundary_outflow), tot


@pytest.mark.parametrize("path", ["fused", "twopass", "staged"])
@pytest.mark.parametrize("cfg", ["smooth", "quadrant"])
def test_one_rank_real_nccl_equals_plain_handle(cuda, path, cfg):
    # (smooth: 400 rows = 6 row chunks on the fused path, so the halo exchange overlaps
    # the interior chunks on the comm stream)
    case = CS.smooth(200, 12, ny=400) if cfg == "smooth" else CS.quadrant(96, 12)
    g = case.grid
    a = run(case, path)
    b = run(case, path, dist=(0, 1, 0, nccl_unique_id()))
    inter = (slice(None), slice(g.gy, g.gy + g.ny), slice(g.gx, g.gx + g.nx))
    assert np.all(a[0][inter] == b[0][inter])
    assert a[1] == b[1] and a[2] == b[2] and a[3] == b[3]
