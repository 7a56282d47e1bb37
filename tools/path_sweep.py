"""Two-pass vs fused one-kernel step across grid sizes (the LF_PATH_AUTO threshold).

    python tools/path_sweep.py [out.json]

Device-resident steps through lf_advance, CUDA-event timed after an untimed warm-up
run, for BASELINE configs 2 and 3 and the smooth-flow generator at 1024^2 .. 8192^2,
each path in both arithmetics; prints G cell-updates/s per (case, path, math).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

cases = [("config2_quadrant_1024", CS.quadrant(1024, 200)),
         ("config3_sedov_4096", CS.sedov(4096, 100)),
         ("smooth_2048", CS.smooth(2048, 60)), ("smooth_4096", CS.smooth(4096, 40)),
         ("smooth_8192", CS.smooth(8192, 20))]
out = {}
for name, case in cases:
    g = case.grid
    f0 = CS.initial_field(case) if case.init != "fourier" else None
    for path in ("twopass", "fused"):
        for math in ("exact", "contract"):
            s = LagfluxSolver(g, case.bc, case.gamma, case.params, path=path, math=math)
            stream = torch.cuda.current_stream()
            s.set_stream(stream.cuda_stream)
            ctl = G.TimeControls(case.cfl, case.t_final, case.max_steps)
            best = None
            for rep in range(2):
                st = G.SolverState(field=f0.copy() if f0 is not None else G.new_field(g))
                if f0 is None:
                    s.init_fourier(st, case.seed)
                else:
                    s.attach(st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                n = s.advance(st, ctl, case.max_steps)
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                v = g.nx * g.ny * n / (ms / 1e3) / 1e9
                best = v if best is None else max(best, v)
            s.close()
            out[f"{name}/{path}/{math}"] = best
            print(name, path, math, f"{best:.3f} G cell-updates/s", flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
