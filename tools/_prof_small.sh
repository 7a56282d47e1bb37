mkdir -p gpurun_out/s5
cat > /tmp/one.py <<'PY'
import sys, time; sys.path.insert(0, '.')
from paper_1607_08710_b200 import cases as CS, grid as G
from paper_1607_08710_b200.solver import LagfluxSolver
case = CS.sod()
s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path="small")
for rep in range(3):
    st = G.SolverState(field=CS.initial_field(case)); s.attach(st)
    t0 = time.perf_counter(); n = s.advance(st, G.TimeControls(case.cfl, case.t_final, 1 << 30), 1 << 30); t1 = time.perf_counter()
    print("config1 small", n, 1e6 * (t1 - t0) / n, "us/step")
PY
python /tmp/one.py > gpurun_out/s5/one.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_small -c 1 -o gpurun_out/s5/prof_small python /tmp/one.py > gpurun_out/s5/ncu.log 2>&1
