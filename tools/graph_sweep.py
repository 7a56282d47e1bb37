"""lf_advance with and without CUDA-graph batches (LF_GRAPHS=1/0) on mid-size grids,
LF_PATH_AUTO: quadrant (transmissive: boundary-outflow sums on the side stream) and
the periodic smooth flow, n^2 cells.

    python tools/graph_sweep.py [--json out.json]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(name, n, steps):
    import torch
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200.solver import LagfluxSolver
    case = CS.quadrant(n, steps) if name == "quadrant" else CS.smooth(n, steps)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params)
    stream = torch.cuda.current_stream()
    s.set_stream(stream.cuda_stream)
    f0 = CS.initial_field(case)
    ctl = G.TimeControls(case.cfl, 1e30)
    best = None
    for rep in range(3):
        st = G.SolverState(field=f0.copy())
        s.attach(st)
        s.advance(st, ctl, 8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = s.advance(st, ctl, steps)
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / done * 1e3
        best = us if best is None or us < best else best
    print(json.dumps({"case": name, "n": n, "path": s.resolved_path(), "us_per_step": best,
                      "graphs": os.environ.get("LF_GRAPHS", "1")}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    res = []
    for name in ("quadrant", "smooth"):
        for n in (384, 512, 640, 768, 896, 1024):
            row = {"case": name, "n": n}
            for g in ("1", "0"):
                out = subprocess.run([sys.executable, __file__, "--one", name, str(n), "256"],
                                     env=dict(os.environ, LF_GRAPHS=g), stdout=subprocess.PIPE,
                                     check=True).stdout.decode().strip().splitlines()[-1]
                r = json.loads(out)
                row["path"] = r["path"]
                row["graphs_on_us" if g == "1" else "graphs_off_us"] = round(r["us_per_step"], 2)
            print(row, flush=True)
            res.append(row)
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
