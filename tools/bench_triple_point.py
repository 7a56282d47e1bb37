"""Device-resident multimaterial steps (cases/triple_point.case regions, 3 materials)
at the reference resolution and at 16x the cells, CUDA-event timed.

    python tools/bench_triple_point.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

for nx, ny, steps in ((2048, 878, 100), (8192, 3512, 20)):
    c = CS.triple_point(nx, ny)
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas))
    stream = torch.cuda.current_stream()
    s.set_stream(stream.cuda_stream)
    st, mat = G.SolverState(field=f0), m0.copy()
    s.attach(st)
    ctl = G.TimeControls(c.cfl, c.t_final, 10 ** 9)
    s.advance(st, ctl, 5, mat)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    n = s.advance(st, ctl, steps, mat)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"triple point {nx}x{ny}: {ms / n * 1e3:.1f} us/step, {nx * ny * n / ms / 1e6:.2f} G cell-updates/s")
    s.close()
