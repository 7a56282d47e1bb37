"""BASELINE config 4 (seeded smooth flow, 16384^2 periodic, CFL 0.5, 50 steps):
bitwise parity of the GPU path against the reference compiled from its own sources
(oracle/_ref), plus the tolerance arithmetic (LF_MATH_CONTRACT) against the same
reference run.

    python tools/bench_config4.py [out.json] [n]

The reference needs ~77 GB of host memory at 16384^2 (32 doubles per cell of
scratch); on a box with less, n falls back to 8192 (same generator,
same seed) and the record says so.  The initial state comes from the device
generator (lf_init_fourier, equal to the host generator: tests/test_gpu_fullsize.py)
and is handed to both sides bit for bit.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import psutil  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

STEPS = 50
ram = psutil.virtual_memory().total
n = int(sys.argv[2]) if len(sys.argv) > 2 else (16384 if ram >= 128e9 else 8192)
case = CS.smooth(n, STEPS)
g = case.grid
rec = {"config": f"config 4 generator, {n}x{n} periodic, CFL 0.5, {STEPS} steps, seed {case.seed}",
       "full_size": n == 16384, "host_ram_GB": ram / 1e9, "host_cores": os.cpu_count()}

# initial state from the device generator, downloaded once (ghosted reference layout)
s = LagfluxSolver(g, case.bc, case.gamma, case.params)
stream = torch.cuda.current_stream()
s.set_stream(stream.cuda_stream)
st0 = G.SolverState(field=G.new_field(g))
s.init_fourier(st0, case.seed)
f0 = G.new_field(g)
s.download(f0)


def gpu_run(math):
    s.set_math(math)
    st = G.SolverState(field=f0.copy())
    s.attach(st)
    ctl = G.TimeControls(case.cfl, case.t_final, STEPS)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k = s.advance(st, ctl, STEPS)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s.sync_to_host(st)
    d = np.array([[x.dt, x.time, x.min_rho, x.min_p] for x in st.diagnostics])
    return st.field, d, {"steps": k, "gpu_ms_per_step": ms / k,
                         "gpu_cell_updates_per_s": g.nx * g.ny * k / (ms / 1e3)}


def rel_l1_chunked(a, b):
    num, den = np.zeros(4), np.zeros(4)
    for c in range(4):
        for r0 in range(0, g.ny, 1024):
            sa = a[c, g.gy + r0:g.gy + min(r0 + 1024, g.ny), g.gx:g.gx + g.nx]
            sb = b[c, g.gy + r0:g.gy + min(r0 + 1024, g.ny), g.gx:g.gx + g.nx]
            num[c] += np.abs(sa - sb).sum()
            den[c] += np.abs(sb).sum()
    return (num / np.where(den > 0, den, 1.0)).tolist()


fe, de, re_ = gpu_run("exact")
rec["exact"] = re_
fc, dc, rc_ = gpu_run("contract")
rec["contract"] = rc_
s.close()
print("gpu", json.dumps(rec), flush=True)

if O.ref_available():
    threads = os.cpu_count() or 1
    r = O.RefSolver(g, case.bc, case.gamma, case.params, threads=threads)
    r.set_state(f0)
    del f0
    t0 = time.perf_counter()
    diag = r.heun_steps(STEPS, case.cfl, case.t_final)
    wall = time.perf_counter() - t0
    rf = r.get_state()[0]
    del r
    rec["reference"] = {"threads": threads, "s_per_step": wall / STEPS,
                        "cell_updates_per_s": g.nx * g.ny * STEPS / wall}
    inter = (slice(None), slice(g.gy, g.gy + g.ny), slice(g.gx, g.gx + g.nx))
    rec["exact"]["field_equal"] = bool(np.all(fe[inter] == rf[inter]))
    rec["exact"]["diagnostics_equal"] = bool(np.array_equal(de, diag[:, :4]))
    rec["contract"]["rel_l1_per_field"] = rel_l1_chunked(fc, rf)
    rec["contract"]["dt_max_rel_diff"] = float(np.max(np.abs(dc[:, 0] - diag[:, 0]) / diag[:, 0]))
    rec["contract"]["within_tolerance"] = bool(max(rec["contract"]["rel_l1_per_field"]) <= 1e-10
                                               and rec["contract"]["dt_max_rel_diff"] <= 1e-12
                                               and dc.shape == diag[:, :4].shape)
    rec["dt_first_last"] = [float(diag[0, 0]), float(diag[-1, 0])]
print("config4", json.dumps(rec), flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(rec, f, indent=1)
