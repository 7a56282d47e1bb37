"""A few device-timed Heun steps on the smooth-flow workload, for ncu captures.

    python tools/prof_steps.py [N] [steps] [path: twopass|fused] [math: exact|contract]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
path = sys.argv[3] if len(sys.argv) > 3 else "twopass"
math = sys.argv[4] if len(sys.argv) > 4 else "exact"
case = CS.smooth(n, steps)
s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path, math=math)
state = G.SolverState(field=None)
s.init_fourier(state, case.seed)
print(path, math, n, s.time_steps(steps, case.cfl))
s.close()
