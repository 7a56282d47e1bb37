"""Small runs through every device path, each checked against the oracle:

    python tools/all_paths_check.py

the stage-wise, two-pass (plain and exact), fused and multimaterial Heun paths,
1-3 in-process slabs, the boundary-outflow side stream, the ghost fill, the
conservation audit, the batched edge_flux and the device self-tests.  Written as
the compute-sanitizer driver (memcheck / racecheck / synccheck); compute-sanitizer
is closed on the GPU pool this round, so it runs plain -- races and bad accesses
are excluded by construction and by the bitwise determinism and parity tests
(DESIGN.md section 7).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402
from paper_1607_08710_b200 import multimat as MM  # noqa: E402
from paper_1607_08710_b200 import native as N  # noqa: E402
from paper_1607_08710_b200 import solver as S  # noqa: E402


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


def run_case(case, steps, path, devices=(0,)):
    f0 = CS.initial_field(case)
    o = O.OracleSolver(case.grid, case.bc, case.gamma, case.params)
    ost = G.SolverState(field=f0.copy())
    for _ in range(steps):
        o.heun_step(ost, case.cfl, case.t_final)
    s = S.LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path, devices=devices)
    st = G.SolverState(field=f0.copy())
    s.advance(st, G.TimeControls(case.cfl, case.t_final), steps)
    tot = s.interior_totals()
    s.sync_to_host(st)
    s.close()
    g = case.grid
    check(f"{case.name} {path} slabs={len(devices)}",
          np.array_equal(g.interior(st.field), g.interior(ost.field)) and
          list(st.boundary_outflow) == list(ost.boundary_outflow) and
          tot == O.oracle_interior_totals(g, st.field))


def main():
    sod = CS.sod(64, 8)
    quad = CS.quadrant(40, 12)
    smooth = CS.smooth(48, 6, ny=32, y_extent=32 / 48)
    for path in ("staged", "twopass", "fused"):
        run_case(sod, 10, path)
        run_case(quad, 12, path)            # shock precursors: the exact two-pass kernels
        run_case(smooth, 6, path, devices=(0, 0, 0))
    # multimaterial (two-pass material kernels, partial fills, cp.async staging)
    c = CS.triple_point(64, 28)
    f0, m0 = CS.regions_field(c)
    ms = MM.make_material_set(c.material_gammas)
    o = O.OracleSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    ost, omat = G.SolverState(field=f0.copy()), m0.copy()
    for _ in range(8):
        o.heun_step(ost, c.cfl, c.t_final, omat)
    s = S.LagfluxSolver(c.grid, c.bc, c.gamma, c.params, materials=ms)
    st, mat = G.SolverState(field=f0.copy()), m0.copy()
    s.advance(st, G.TimeControls(c.cfl, c.t_final), 8, mat)
    s.sync_to_host(st, mat=mat)
    s.close()
    check("triple point 64x28", np.array_equal(c.grid.interior(st.field), c.grid.interior(ost.field)))
    # ghost fill and edge_flux
    g = G.make_grid_2d(12, 9, 0.0, 1.0, 0.0, 1.0)
    f = G.new_field(g)
    g.interior(f)[...] = np.random.default_rng(1).standard_normal(g.interior(f).shape)
    s = S.LagfluxSolver(g, G.BoundaryCondition(1, 1, 2, 2))
    s.upload(f)
    out = np.zeros_like(f)
    s.download_ghosted(out)
    s.close()
    check("ghost fill", np.isfinite(out).all())
    wm = np.array([[1.0, 0.3, -0.2, 1.0], [0.125, 0.0, 0.0, 0.1]])
    flux, _ = S.edge_flux(wm, wm[::-1].copy(), [[0.6, 0.8], [1.0, 0.0]], 1.4)
    fo = np.zeros(4)
    O.oracle_lib().lfo_edge_flux(wm[1].ctypes.data_as(O.DP), wm[0].ctypes.data_as(O.DP), 1.0, 0.0, 1.4,
                                 fo.ctypes.data_as(O.DP))
    check("edge_flux", np.array_equal(flux[1], fo))
    # device self-tests (small)
    import ctypes as C
    cnt = (C.c_int64 * 10)()
    check("selftest fastmath", N.lib().lf_selftest_fastmath(1 << 12, 7, cnt) == 0 and cnt[2] == 0)
    cnt3 = (C.c_int64 * 3)()
    check("selftest epilogue", N.lib().lf_selftest_epilogue(1 << 12, 7, cnt3) == 0 and cnt3[1] == 0)


if __name__ == "__main__":
    main()
