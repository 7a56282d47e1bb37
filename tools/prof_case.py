"""Device-resident lf_advance over a named case, CUDA-event timed (ncu launch lists).

    python tools/prof_case.py quadrant|sedov N steps
    python tools/prof_case.py sod          # BASELINE config 1: 400x4 to t = 0.2 (353 steps)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "quadrant"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
case = CS.sod() if name == "sod" else {"quadrant": CS.quadrant, "sedov": CS.sedov}[name](n, steps)
s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params)
stream = torch.cuda.current_stream()
s.set_stream(stream.cuda_stream)
st = G.SolverState(field=CS.initial_field(case))
s.attach(st)
ctl = G.TimeControls(case.cfl, case.t_final if name == "sod" else 1e30)
if name == "sod":
    steps = 10 ** 6   # to t_final
    warm = G.SolverState(field=CS.initial_field(case))
    s.attach(warm)
    s.advance(warm, ctl, 20)   # one-time allocations
    s.attach(st)
else:
    s.advance(st, ctl, 5)   # warm-up (and the sticky exact-kernel switch, if any)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
l0 = s.launch_count()
e0.record(stream)
steps = s.advance(st, ctl, steps)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
cells = case.grid.nx * case.grid.ny
print(f"{name} {case.grid.nx}x{case.grid.ny}: {steps} steps {ms:.2f} ms, {ms / steps * 1e3:.1f} us/step, "
      f"{cells * steps / ms / 1e6:.2f} G cell-updates/s, {(s.launch_count() - l0) / steps:.1f} launches/step")
s.close()
