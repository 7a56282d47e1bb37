"""Multimaterial runs on the small path against the two-pass / stage-wise paths (one
B200): lf_advance, host-timed, best of 3 after a warm-up run; final fields and partial
densities bit-equal across paths.

    python tools/small_mat_sweep.py [--json out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200.solver import LagfluxSolver  # noqa: E402


def run(c, path, steps):
    f0, m0 = CS.regions_field(c)
    s = LagfluxSolver(c.grid, c.bc, c.gamma, c.params,
                      materials=MM.make_material_set(c.material_gammas), path=path)
    best, out = None, None
    for rep in range(4):
        st = G.SolverState(field=f0.copy())
        mat = MM.MaterialCells(c.grid, len(c.material_gammas), m0.partial.copy())
        s.attach(st)
        t0 = time.perf_counter()
        n = s.advance(st, G.TimeControls(c.cfl, c.t_final, steps), steps, mat)   # (uploads both)
        t1 = time.perf_counter()
        if rep == 0 and s.resolved_path() != path:
            s.close()
            return None
        if rep:
            best = (t1 - t0) / n if best is None else min(best, (t1 - t0) / n)
        s.sync_to_host(st, mat=mat)
        out = (c.grid.interior(st.field).copy(), c.grid.interior(mat.partial).copy())
    s.close()
    return {"us_per_step": 1e6 * best, "steps": n}, out


def main():
    cases = [("contact_1d_400", CS.material_contact_1d(400), 300),
             ("triple_point_70x30", CS.triple_point(70, 30), 100),
             ("triple_point_140x60", CS.triple_point(140, 60), 100),
             ("triple_point_256x110", CS.triple_point(256, 110), 100),
             ("triple_point_512x220", CS.triple_point(512, 220), 100)]
    res = {}
    for name, c, steps in cases:
        row, ref = {}, None
        for path in ("small", "twopass", "staged"):
            r = run(c, path, steps)
            if r is None:
                continue
            row[path], out = r
            if ref is None:
                ref = out
            row[path]["same_bits_as_small"] = bool(np.array_equal(out[0], ref[0]) and
                                                   np.array_equal(out[1], ref[1]))
        res[name] = row
        print(name, json.dumps(row), flush=True)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
