"""Fused one-kernel step with shorter row chunks on mid-size grids (LF_FUSED_MIN_ROWS).

    python tools/chunk_sweep.py [out.json]

Each case runs on the two-pass kernels and on the fused step with the chunk-row floor at
64 / 32 / 16 / 8 rows; device-resident lf_advance, CUDA-event timed after a warm-up run;
the final fields are compared bit for bit with the two-pass run's.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402

cases = [("smooth_256", CS.smooth(256, 300)), ("smooth_320", CS.smooth(320, 300)),
         ("smooth_384", CS.smooth(384, 300)), ("quadrant_400", CS.quadrant(400, 300)),
         ("smooth_512", CS.smooth(512, 200)), ("quadrant_512", CS.quadrant(512, 200)),
         ("smooth_640", CS.smooth(640, 200)),
         ("smooth_768", CS.smooth(768, 200)), ("config2_quadrant_1024", CS.quadrant(1024, 200)),
         ("smooth_1024", CS.smooth(1024, 100)), ("smooth_1536", CS.smooth(1536, 80)),
         ("smooth_2048", CS.smooth(2048, 60))]
if len(sys.argv) > 2:
    cases = [c for c in cases if c[0] in sys.argv[2].split(",")]
out = {}
for name, case in cases:
    g = case.grid
    f0 = CS.initial_field(case) if case.init != "fourier" else None
    ref = None
    for path, mr in (("twopass", 0), ("small", 0), ("fused", 64), ("fused", 16), ("fused", 8), ("fused", 4), ("fused", 2)):
        for math in ("exact", "contract"):
            if mr:
                os.environ["LF_FUSED_MIN_ROWS"] = str(mr)
            if path == "small" and (math == "contract" or g.nx * g.ny > 1 << 19):
                continue
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
            same = None
            if math == "exact":
                s.sync_to_host(st)
                fin = np.array(st.field, copy=True)
                if ref is None:
                    ref = fin
                else:
                    same = bool(np.array_equal(ref, fin))
            s.close()
            key = f"{name}/{path}{mr or ''}/{math}"
            out[key] = {"gcups": best, "us_per_step": ms / n * 1e3, "equal_twopass": same}
            print(key, f"{best:.3f} G cell-updates/s", same, flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
