import sys, time; sys.path.insert(0,'.')
import torch
from paper_1607_08710_b200 import cases as CS, grid as G, multimat as MM
from paper_1607_08710_b200.solver import LagfluxSolver
for (nx, ny) in ((2048, 878), (8192, 3512)):
    c = CS.triple_point(nx, ny)
    for path in ("twopass", "staged"):
        s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=MM.make_material_set(c.material_gammas), path=path)
        st = G.SolverState(field=G.new_field(c.grid)); m = MM.MaterialCells(c.grid, 3)
        s.init_regions(st, c.regions, m)
        ctl = G.TimeControls(c.cfl, c.t_final, 10**9)
        s.advance(st, ctl, 5, m); torch.cuda.synchronize()
        n0 = s.launch_count()
        t0 = time.perf_counter(); k = s.advance(st, ctl, 30, m); torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(nx, ny, path, "%.2f G/s" % (nx * ny * k / t / 1e9), "launches/step %.1f" % ((s.launch_count() - n0) / k), flush=True)
        s.close()
