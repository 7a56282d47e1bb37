"""Small grids: LF_PATH_SMALL (one persistent block) against the two-pass and stage-wise
paths, and the reference on the host cores beside them.

    python tools/small_sweep.py [--json out.json]

Each case runs to its t_final (or step count) through lf_advance -- the run.cpp step
loop with the state resident on the device -- timed on the host around the call
(records and outflow come back inside it), best of a few repetitions after a warm-up
run; the final fields of every path must be equal bit for bit, and equal to the
reference's.  The reference times heun_step calls over the same steps (1 thread and
all host threads).  The crossover sizes set SMALL_AUTO_CELLS_1D / _2D (csrc/small.h).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402


def sod1d(n):
    g = G.make_grid_1d(n, 0.0, 1.0)
    return CS.Case(f"sod1d_{n}", g, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2,
                   G.INT64_MAX, "riemann_x")


def cases():
    out = [("config1_sod_400x4", CS.sod())]
    for n in (100, 1000, 10000, 65536):
        out.append((f"sod1d_{n}", sod1d(n)))
    for n in (32, 64, 128, 256, 512):
        c = CS.quadrant(n, 200)
        out.append((f"quadrant_{n}", c))
    return out


def time_path(case, path, reps=3):
    g = case.grid
    f0 = CS.initial_field(case)
    s = LagfluxSolver(g, case.bc, case.gamma, case.params, path=path)
    if s.resolved_path() != path:
        s.close()
        return None
    ctl = G.TimeControls(case.cfl, case.t_final, case.max_steps)
    best, field, n = None, None, 0
    for rep in range(reps + 1):
        st = G.SolverState(field=f0.copy())
        s.attach(st)
        t0 = time.perf_counter()
        n = s.advance(st, ctl, min(case.max_steps, 1 << 30))
        t1 = time.perf_counter()
        if rep > 0:
            best = t1 - t0 if best is None else min(best, t1 - t0)
        s.sync_to_host(st)
        field = g.interior(st.field).copy()
    s.close()
    return {"steps": n, "us_per_step": 1e6 * best / n, "cells": g.nx * g.ny,
            "cell_updates_per_s": g.nx * g.ny * n / best}, field


def time_reference(case, steps, threads):
    from oracle import oracle as O
    g = case.grid
    r = O.RefSolver(g, case.bc, case.gamma, case.params, threads=threads)
    r.set_state(CS.initial_field(case))
    t0 = time.perf_counter()
    r.heun_steps(steps, case.cfl, case.t_final)
    t1 = time.perf_counter()
    f, _, _, _ = r.get_state()
    return {"us_per_step": 1e6 * (t1 - t0) / steps, "threads": threads}, g.interior(f).copy()


def main():
    res = {}
    for name, case in cases():
        row, ref_field = {}, None
        for path in ("small", "twopass", "staged") if "--small-only" not in sys.argv else ("small",):
            if path == "staged" and case.grid.nx * case.grid.ny > 20000:
                continue
            r = time_path(case, path)
            if r is None:
                continue
            row[path], field = r
            if ref_field is None:
                ref_field = field
            row[path]["same_bits_as_small"] = bool(np.array_equal(field, ref_field))
        steps = row["small"]["steps"]
        if "--small-only" in sys.argv:
            res[name] = row
            print(name, json.dumps(row), flush=True)
            continue
        try:
            for th in (1, os.cpu_count() or 1):
                rr, rf = time_reference(case, steps, th)
                rr["same_bits"] = bool(np.array_equal(rf, ref_field))
                row[f"reference_{th}t"] = rr
        except Exception as e:  # noqa: BLE001 (no compiled reference: say so)
            row["reference"] = f"unavailable: {e}"
        res[name] = row
        print(name, json.dumps(row), flush=True)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
