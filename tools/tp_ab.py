"""Two-pass path timings for an A/B of library builds (run once per build).

    python tools/tp_ab.py [label]

Config 2 (quadrant 1024^2, 200 steps), Sedov 2048^2 (50 steps), quadrant 256^2 (200
steps) on LF_PATH_TWOPASS through lf_advance (device-resident, CUDA-event timed, best
of 3 after a warm-up run), and a digest of each final field (A/B builds must agree).
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200.solver import LagfluxSolver
    out = {}
    for name, case, steps in (("config2_quadrant_1024", CS.quadrant(1024, 200), 200),
                              ("sedov_2048", CS.sedov(2048, 50), 50),
                              ("quadrant_256", CS.quadrant(256, 200), 200)):
        g = case.grid
        f0 = CS.initial_field(case)
        s = LagfluxSolver(g, case.bc, case.gamma, case.params, path="twopass")
        stream = torch.cuda.current_stream()
        s.set_stream(stream.cuda_stream)
        ctl = G.TimeControls(case.cfl, case.t_final, steps)
        best, dig = None, None
        for rep in range(4):
            st = G.SolverState(field=f0.copy())
            s.attach(st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            n = s.advance(st, ctl, steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            if rep:
                best = ms if best is None else min(best, ms)
            s.sync_to_host(st)
            dig = hashlib.sha256(g.interior(st.field).tobytes()).hexdigest()[:16]
        s.close()
        out[name] = {"us_per_step": 1e3 * best, "gcells_s": g.nx * g.ny / best / 1e6, "digest": dig}
    print(json.dumps({"label": sys.argv[1] if len(sys.argv) > 1 else "", **out}))


if __name__ == "__main__":
    main()
