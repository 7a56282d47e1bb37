import sys; sys.path.insert(0,'.')
from paper_1607_08710_b200 import native as N
N.LIB_PATH = "tools/_variants/matdbg.so"
import torch
from paper_1607_08710_b200 import cases as CS, grid as G, multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
c = CS.triple_point(2048, 878)
f0, m0 = CS.regions_field(c)
s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas), path="twopass")
st = G.SolverState(field=f0.copy()); m = m0.copy()
s.advance(st, G.TimeControls(c.cfl, c.t_final, 10**9), 30, m); torch.cuda.synchronize()
print("done", st.step)
