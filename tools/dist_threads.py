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


def run_err(g, bc, f0, steps, cfl, t_final, path, dist=None):
    """(exception type, text) of a failing run (None if it does not fail)."""
    s = S.LagfluxSolver(g, bc, path=path, dist=dist)
    st = G.SolverState(field=f0.copy())
    try:
        for _ in range(steps):
            s.heun_step(st, G.TimeControls(cfl, t_final), t_final)
    except G.Error as e:  # noqa: PERF203
        return type(e).__name__, str(e)
    finally:
        s.close()
    return None


def errors(ok):
    """Failures in cells owned by a rank other than 0: every rank reports the
    reference's exception (type, text with the cell's values) like one handle."""
    # corrector positivity failure (CFL far beyond stability)
    g = G.make_grid_2d(24, 16, 0.0, 1.0, 0.0, 1.0)
    case = CS.Case("q", g, G.BoundaryCondition.uniform(G.TRANSMISSIVE), 1.4, G.SchemeParams(),
                   4.0, CS.STEP_DRIVEN_LIMIT, 5, "quadrant")
    f0 = CS.initial_field(case)
    # a cell with negative energy in the upper rows: "non-positive pressure = <value>"
    bad = f0.copy()
    bad[3, 2 + 13, 2 + 7] = -0.25
    plan = [("positivity", case.bc, f0, case.cfl), ("bad cell", case.bc, bad, 0.45)]
    for name, bc, f, cfl in plan:
        for path in ("twopass", "fused", "staged"):
            single = run_err(g, bc, f, 5, cfl, CS.STEP_DRIVEN_LIMIT, path)
            for n in (2, 3):
                uid = S.nccl_unique_id()
                res = [None] * n

                def worker(r):
                    res[r] = run_err(g, bc, f, 5, cfl, CS.STEP_DRIVEN_LIMIT, path,
                                     dist=(r, n, 0, uid))

                ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(n)]
                for t in ts:
                    t.start()
                for t in ts:
                    t.join(300)
                    if t.is_alive():
                        print("HANG: a rank did not finish", flush=True)
                        os._exit(3)
                good = single is not None and all(x == single for x in res)
                ok &= good
                print(f"error {name} {path}: {'ok' if good else 'MISMATCH'} ({n} ranks) "
                      f"{single} {'' if good else res}", flush=True)
    return ok


def strip5(ok, nranks=8, steps=20):
    """BASELINE config 5's generator on a 32768 x 2048 periodic strip (dy = dx), 20
    steps, as `nranks` y-slab ranks == one handle: every step's dt / time / min rho /
    min p, interior_totals and each rank's rows of the final field, on the fused and
    the two-pass kernels.  Ranks download
    only their own rows (local_host), as bench.py's ranks do."""
    n, ny = 32768, 2048
    case = CS.smooth(n, steps, ny=ny, y_extent=ny / n)
    g = case.grid

    def go(path, dist=None):
        s = S.LagfluxSolver(g, case.bc, case.gamma, case.params, path=path, dist=dist)
        st = G.SolverState(field=np.zeros((4, 1, 1)))
        s.init_fourier(st, case.seed)
        s.advance(st, G.TimeControls(case.cfl, case.t_final), steps)
        tot = s.interior_totals()
        y0, rows = s.local_rows()
        if dist is None:
            out = G.new_field(g)
            s.download(out)
            part = out[:, g.gy:g.gy + g.ny, g.gx:g.gx + g.nx]
        else:
            s.local_host = True
            out = np.empty(s.local_field_shape())
            s.download(out)
            part = out[:, g.gy:g.gy + rows, g.gx:g.gx + g.nx]
        s.close()
        diag = [(d.dt, d.time, d.min_rho, d.min_p) for d in st.diagnostics]
        return part, diag, tot, (y0, rows)

    for path in ("fused", "twopass"):
        single = go(path)
        uid = S.nccl_unique_id()
        res = [None] * nranks

        def worker(r):
            res[r] = go(path, dist=(r, nranks, 0, uid))

        ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(600)
            if t.is_alive():
                print("HANG: a rank did not finish", flush=True)
                os._exit(3)
        good = len(single[1]) == steps
        for part, diag, tot, (y0, rows) in res:
            good &= bool(np.array_equal(part, single[0][:, y0:y0 + rows]))
            good &= diag == single[1] and tot == single[2]
        ok &= good
        print(f"config5 strip {n}x{ny} {path}: {'ok' if good else 'MISMATCH'} ({steps} steps, "
              f"{nranks} ranks)", flush=True)
        del single, res
    return ok


def main():
    ok = True
    if "--errors-only" in sys.argv:
        sys.exit(0 if errors(ok) else 1)
    if "--config5-strip" in sys.argv:
        sys.exit(0 if strip5(ok) else 1)
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
    ok = errors(ok)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
