mkdir -p gpurun_out/c2
cat > /tmp/c2.py <<'PY'
import sys, time; sys.path.insert(0, '.')
from paper_1607_08710_b200 import cases as CS, grid as G
from paper_1607_08710_b200.solver import LagfluxSolver
case = CS.quadrant(1024, 200)
s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params)
print(s.resolved_path())
for rep in range(2):
    st = G.SolverState(field=CS.initial_field(case)); s.attach(st)
    t0 = time.perf_counter(); n = s.advance(st, G.TimeControls(case.cfl, case.t_final, 200), 200); t1 = time.perf_counter()
    print("config2", n, 1e6 * (t1 - t0) / n, "us/step")
PY
python /tmp/c2.py > gpurun_out/c2/plain.log 2>&1
LF_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c2/launches.csv python /tmp/c2.py > gpurun_out/c2/ncu.log 2>&1
