"""A few multimaterial steps (triple point) for ncu launch lists.

    python tools/prof_mat.py [nx ny steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

nx, ny, steps = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 878, 4)
c = CS.triple_point(nx, ny)
f0, m0 = CS.regions_field(c)
s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas))
state = G.SolverState(field=f0)
mat = m0.copy()
s.attach(state)
s.advance(state, G.TimeControls(c.cfl, c.t_final, steps), steps, mat)
print("steps", state.step)
