"""Time a field dump (run.cpp's dump: field_csv + write) of the triple point at its
reference resolution: lf_write_field_csv (device-derived columns, threaded
formatting) against the reference's own field_csv (oracle/_ref) on the same state.

    python tools/bench_dump.py [nx ny] [out.json]
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 2 else 2048
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 878
c = CS.triple_point(nx, ny)
f0, m0 = CS.regions_field(c)
ms = MM.make_material_set(c.material_gammas)
s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
state = G.SolverState(field=f0.copy())
mat = m0.copy()
for _ in range(20):
    s.heun_step(state, G.TimeControls(c.cfl, c.t_final), c.t_final, mat)
s.sync_to_host(state, mat=mat)
d = tempfile.mkdtemp()
p = os.path.join(d, "ours.csv")
s.write_field_csv(p, 1, state.time)  # warm
t0 = time.perf_counter()
s.write_field_csv(p, 1, state.time)
ours = time.perf_counter() - t0
size = os.path.getsize(p)
# the asynchronous dump: how long the caller is held, and 20 further steps run with
# the dump in flight against the same 20 steps after a synchronous dump
tc = G.TimeControls(c.cfl, c.t_final)


def steps(n):
    for _ in range(n):
        s.heun_step(state, tc, c.t_final, mat)
    s.sync_to_host(state, mat=mat)


steps(2)
t0 = time.perf_counter()
s.write_field_csv(os.path.join(d, "seq.csv"), 1, state.time)
steps(20)
seq = time.perf_counter() - t0
pa = os.path.join(d, "async.csv")
t0 = time.perf_counter()
s.write_field_csv_async(pa, 1, state.time)
held = time.perf_counter() - t0
steps(20)
s.wait_dumps()
ovl = time.perf_counter() - t0
res = {"workload": f"triple_point {nx}x{ny}, 3 materials, after 20 steps",
       "bytes": size, "ours_s": ours, "threads": os.cpu_count(),
       "async_call_s": held, "dump_then_20_steps_s": seq, "async_dump_with_20_steps_s": ovl}
if O.ref_available():
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    r.set_state(state.field)
    r.set_partials(mat.partial)
    t0 = time.perf_counter()
    txt = r.field_csv(1, state.time)
    with open(os.path.join(d, "ref.csv"), "wb") as f:
        f.write(txt)
    ref = time.perf_counter() - t0
    res.update({"reference_s": ref, "identical": txt == open(p, "rb").read(),
                "speedup": ref / ours})
print(json.dumps(res))
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        json.dump(res, f, indent=1)
