"""lf_advance with and without CUDA-graph batches (LF_GRAPHS=0/1), small BASELINE configs.

    python tools/graph_ab.py            # runs itself twice (LF_GRAPHS=1, 0) and compares
    python tools/graph_ab.py --one      # one timing pass in this process

Config 1 (Sod 400x4 to t = 0.2, 353 steps) and config 2 (quadrant 1024^2, 200 steps):
device-resident steps through lf_advance, timed with CUDA events after an untimed
run of the same length (so the graphs of every batch length are instantiated); the
final fields of the two modes must be equal bit for bit.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import hashlib
    import torch
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200.solver import LagfluxSolver
    out = {}
    for name, case, reps in (("config1_sod_400x4", CS.sod(), 5),
                             ("config2_quadrant_1024", CS.quadrant(1024, 200), 2)):
        g = case.grid
        f0 = CS.initial_field(case)
        s = LagfluxSolver(g, case.bc, case.gamma, case.params)
        stream = torch.cuda.current_stream()
        s.set_stream(stream.cuda_stream)
        ctl = G.TimeControls(case.cfl, case.t_final, case.max_steps)
        best, digest, n = None, None, 0
        for rep in range(reps + 1):
            st = G.SolverState(field=f0.copy())
            s.attach(st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            n = s.advance(st, ctl, case.max_steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if rep > 0:   # the first run instantiates the graphs
                best = ms if best is None else min(best, ms)
            s.sync_to_host(st)
            digest = hashlib.sha256(g.interior(st.field).tobytes()).hexdigest()[:16]
        s.close()
        out[name] = {"steps": n, "us_per_step": 1e3 * best / n, "digest": digest}
    print(json.dumps(out))


def main():
    res = {}
    for mode in ("1", "0"):
        env = dict(os.environ, LF_GRAPHS=mode)
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--one"], env=env,
                           capture_output=True, text=True, timeout=600)
        if p.returncode:
            print(p.stdout, p.stderr)
            sys.exit(1)
        res["graphs" if mode == "1" else "launches"] = json.loads(p.stdout.strip().splitlines()[-1])
    for k in res["graphs"]:
        a, b = res["graphs"][k], res["launches"][k]
        print(f"{k}: graphs {a['us_per_step']:.1f} us/step, launch by launch "
              f"{b['us_per_step']:.1f} us/step, same bits: {a['digest'] == b['digest']}")
    print(json.dumps(res))


if __name__ == "__main__":
    one() if "--one" in sys.argv else main()
