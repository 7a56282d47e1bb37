"""Kernel launches per Heun step on non-smooth cases: a fast path that re-runs a
flagged step with the stage-wise kernels shows up as extra launches.

    python tools/fallback_check.py [lib.so]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_08710_b200 import native as N  # noqa: E402
if len(sys.argv) > 1:
    N.LIB_PATH = sys.argv[1]
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

def run(name, case, field, mat=None, ms=None, steps=60):
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, materials=ms, path="twopass")
    st = G.SolverState(field=field)
    ctl = G.TimeControls(case.cfl, case.t_final, 10**9)
    s.attach(st)
    s.advance(st, ctl, 5, mat)
    n0 = s.launch_count()
    t0 = time.perf_counter()
    k = s.advance(st, ctl, steps, mat)
    s.sync_to_host(st)
    t = time.perf_counter() - t0
    print(f"{name}: {k} steps, {(s.launch_count() - n0) / k:.1f} launches/step, "
          f"{case.grid.nx * case.grid.ny * k / t / 1e9:.2f} G cell-updates/s (wall)", flush=True)

for n in (2048,):
    for mk in (CS.sedov, CS.quadrant):
        c = mk(n, 60)
        run(f"{c.name} {n}", c, CS.initial_field(c))
c = CS.triple_point(2048, 878)
f0, m0 = CS.regions_field(c)
run("triple_point 2048x878", c, f0, m0.copy(), MM.make_material_set(c.material_gammas))
