"""The distributed (one y-slab per rank) code path on ONE GPU: ranks are host
threads, each with its own lf_create_dist handle, talking through the thread-rank
NCCL stand-in (tests/fake_nccl, loaded via LF_NCCL_LIB).  Every run is compared
bit for bit with a single-handle run of the same case: the assembled field, every
step's dt / time / min rho / min p, the boundary outflow and interior_totals.

    python tools/dist_threads.py          # prints one line per case, exit 1 on a mismatch

No kernel waits on another rank (the stand-in orders transfers with stream
events and reduces on the host), so this is safe on one GPU.
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("LF_NCCL_LIB", os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so"))

import numpy as np  # noqa: E402

from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200 import solver as S  # noqa: E402


def run(g, bc, gamma, params, f0, steps, cfl, t_final, path, dist=None, ms=None, m0=None,
        fourier_seed=None):
    s = S.LagfluxSolver(g, bc, gamma, params, path=path, dist=dist, materials=ms)
    st = G.SolverState(field=f0.copy() if f0 is not None else G.new_field(g))
    mat = m0.copy() if m0 is not None else None
    if fourier_seed is not None:
        s.init_fourier(st, fourier_seed)
    s.advance(st, G.TimeControls(cfl, t_final), steps, mat)
    tot = s.interior_totals()
    out = G.new_field(g)
    s.download(out)
    part = None
    if mat is not None:
        s.sync_to_host(st, mat=mat)
        part = mat.partial.copy()
    y0, rows = s.local_rows()
    s.close()
    diag = [(d.dt, d.time, d.min_rho, d.min_p) for d in st.diagnostics]
    return out, diag, list(st.boundary_outflow), tot, (y0, rows), part


def dist_run(nranks, *args, **kw):
    uid = S.nccl_unique_id()
    res, errs = [None] * nranks, []

    def worker(r):
        try:
            res[r] = run(*args, dist=(r, nranks, 0, uid), **kw)
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
        if t.is_alive():
            print("HANG: a rank did not finish", flush=True)
            os._exit(3)
    if errs:
        raise RuntimeError(errs)
    return res


def compare(name, g, single, ranks):
    out, diag, outflow, tot, _, part = single
    ok = True
    gy = g.gy
    for r, (o, d, of, t, (y0, rows), p) in enumerate(ranks):
        sl = slice(gy + y0, gy + y0 + rows)
        ok &= bool(np.array_equal(o[:, sl, g.gx:g.gx + g.nx], out[:, sl, g.gx:g.gx + g.nx]))
        if part is not None:
            ok &= bool(np.array_equal(p[:, sl, g.gx:g.gx + g.nx], part[:, sl, g.gx:g.gx + g.nx]))
        ok &= d == diag
        ok &= of == outflow
        ok &= t == tot
    print(f"{name}: {'ok' if ok else 'MISMATCH'} ({len(diag)} steps, {len(ranks)} ranks)", flush=True)
    return ok


def main():
    ok = True
    smooth = CS.smooth(64, 1, ny=48, y_extent=48 / 64)
    quad = CS.quadrant(48, 1)
    sedov = CS.sedov(40, 1)
    plan = [("smooth periodic", smooth, 12, (2, 3), ("twopass", "staged", "fused")),
            ("quadrant transmissive", quad, 16, (2, 4), ("twopass", "staged")),
            ("sedov reflective", sedov, 12, (3,), ("twopass", "fused"))]
    for name, case, steps, nrs, paths in plan:
        f0 = CS.initial_field(case)
        args = (case.grid, case.bc, case.gamma, case.params, f0, steps, case.cfl, case.t_final)
        for path in paths:
            single = run(*args, path=path)
            for n in nrs:
                ok &= compare(f"{name} {path}", case.grid, single, dist_run(n, *args, path=path))
    # on-device initial state: global maxima over the ranks
    args = (smooth.grid, smooth.bc, smooth.gamma, smooth.params, None, 6, smooth.cfl, smooth.t_final)
    single = run(*args, path="twopass", fourier_seed=smooth.seed)
    ok &= compare("fourier init", smooth.grid, single, dist_run(2, *args, path="twopass",
                                                                fourier_seed=smooth.seed))
    # three materials: partial-density halos and the min-p reduction
    c = CS.triple_point(64, 28)
    f0, m0 = CS.regions_field(c)
    ms = MM.make_material_set(c.material_gammas)
    args = (c.grid, c.bc, c.gamma, c.params, f0, 10, c.cfl, c.t_final)
    single = run(*args, path="twopass", ms=ms, m0=m0)
    ok &= compare("triple point", c.grid, single, dist_run(2, *args, path="twopass", ms=ms, m0=m0))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
