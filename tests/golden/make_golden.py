"""Generate the golden vectors in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference solver (/root/reference/proj/src/solver.cpp +
grid.cpp, compiled by oracle/Makefile into oracle/_ref/libref_lagflux.so) on
small seeded cases and stores inputs and outputs.  Only runs where the
reference was built (this container); the .npz files are committed so the
tests (and the GPU box, which has no /root/reference) use them as fixtures.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1607_08710_b200 import cases as CS  # noqa: E402
from paper_1607_08710_b200 import grid as G  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def golden_cases():
    """name -> (Case, steps).  Small versions of the BASELINE configs plus variants."""
    one_d = CS.Case("sod1d", G.make_grid_1d(100, 0.0, 1.0), G.BoundaryCondition(), 1.4,
                    G.SchemeParams(), 0.5, 0.2, G.INT64_MAX, "riemann_x")
    mixed = CS.Case("mixed", G.make_grid_2d(40, 24, 0.0, 2.0, 0.0, 1.0),
                    G.BoundaryCondition(G.PERIODIC, G.PERIODIC, G.REFLECTIVE, G.TRANSMISSIVE),
                    1.4, G.SchemeParams(beta=1.0), 0.45, CS.STEP_DRIVEN_LIMIT, 25, "fourier")
    first = CS.Case("first_order", G.make_grid_2d(32, 32, 0.0, 1.0, 0.0, 1.0),
                    G.BoundaryCondition.uniform(G.TRANSMISSIVE), 1.4,
                    G.SchemeParams(spatial_order=1, time_order=1), 0.45, CS.STEP_DRIVEN_LIMIT,
                    30, "quadrant")
    return {
        "sod_400x4": (CS.sod(), 353),
        "quadrant_32": (CS.quadrant(32, 40), 40),
        "sedov_48": (CS.sedov(48, 30), 30),
        "smooth_32": (CS.smooth(32, 20), 20),
        "sod1d_100": (one_d, 200),
        "mixed_40x24": (mixed, 25),
        "first_order_32": (first, 30),
    }


def golden_mat_cases():
    """name -> MatCase (steps in max_steps): the reference's multimaterial cases
    (test_multimat.cpp:62-137, cases/triple_point.case) at small sizes, plus a
    2D four-material quadrant whose contacts shear and mix."""
    quad_regions = (CS.Region(0.5, 1.0, 0.5, 1.0, 1.5, 0.0, 0.0, 1.5, 1),
                    CS.Region(0.0, 0.5, 0.5, 1.0, 0.5323, 1.206, 0.0, 0.3, 2),
                    CS.Region(0.0, 0.5, 0.0, 0.5, 0.138, 1.206, 1.206, 0.029, 3),
                    CS.Region(0.5, 1.0, 0.0, 0.5, 0.5323, 0.0, 1.206, 0.3, 4))
    quad = CS.MatCase("mm_quadrant", G.make_grid_2d(48, 40, 0.0, 1.0, 0.0, 1.0),
                      G.BoundaryCondition(G.TRANSMISSIVE, G.TRANSMISSIVE, G.PERIODIC, G.PERIODIC),
                      1.4, (1.4, 1.67, 1.3, 1.5), quad_regions, G.SchemeParams(beta=1.3), 0.4,
                      1e30, 30)
    first = CS.MatCase("mm_first_order", G.make_grid_2d(40, 20, 0.0, 7.0, 0.0, 3.0),
                       G.BoundaryCondition.uniform(G.REFLECTIVE), 1.4, (1.5, 1.4, 1.5),
                       CS.triple_point().regions,
                       G.SchemeParams(beta=1.5, spatial_order=1, time_order=1), 0.25, 1e30, 30)
    return {
        "mm_contact_equal_64": CS.material_contact_1d(64, (1.4, 1.4), 1.4, 100),
        "mm_contact_unequal_64": CS.material_contact_1d(64, (1.5, 1.4), 1.5, 50),
        "mm_triple_70x30": CS.triple_point(70, 30, 40),
        "mm_quadrant_48x40": quad,
        "mm_first_order_40x20": first,
    }


def run_reference_mat(c):
    from paper_1607_08710_b200 import multimat as MM
    f0, mat0 = CS.regions_field(c)
    r = O.RefSolver(c.grid, c.bc, c.gamma, c.params, threads=1,
                    materials=MM.make_material_set(c.material_gammas))
    r.set_state(f0)
    r.set_partials(mat0.partial)
    diag = r.heun_steps(c.max_steps, c.cfl, c.t_final)
    f, t, s, acc = r.get_state()
    return f0, mat0.partial, diag, f, r.get_partials(), np.array(acc)


def run_reference(case, steps):
    f0 = CS.initial_field(case)
    r = O.RefSolver(case.grid, case.bc, case.gamma, case.params, threads=1)
    r.set_state(f0)
    if case.t_final < CS.STEP_DRIVEN_LIMIT:
        # time-driven (run.cpp:180): step until the clipped last step reaches t_final
        rows = []
        t = 0.0
        while t < case.t_final and len(rows) < steps:
            rows.append(r.heun_steps(1, case.cfl, case.t_final)[0])
            t = rows[-1][1]
        diag = np.array(rows)
    else:
        diag = r.heun_steps(steps, case.cfl, case.t_final)
    f, t, s, acc = r.get_state()
    return f0, diag, f, np.array(acc)


def main_mat(force=False):
    for name, c in golden_mat_cases().items():
        path = os.path.join(OUT, f"{name}.npz")
        if os.path.exists(path) and not force:
            continue
        f0, p0, diag, f, p, acc = run_reference_mat(c)
        g = c.grid
        np.savez_compressed(path, initial=g.interior(f0), initial_partial=g.interior(p0),
                            final=g.interior(f), final_partial=g.interior(p), diag=diag,
                            outflow=acc)
        print(name, c.max_steps, diag[0, 0], diag[-1, 0], diag[-1, 1], diag[-1, 3])


def main():
    for name, (case, steps) in golden_cases().items():
        f0, diag, f, acc = run_reference(case, steps)
        g = case.grid
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"),
                            initial=g.interior(f0), final=g.interior(f), diag=diag, outflow=acc)
        print(name, steps, diag[0, 0], diag[-1, 0], diag[-1, 1])
    # euler_stage straight-line case of test_solver.cpp:225-252 (Sod 50 cells, dt 8e-4)
    g = G.make_grid_1d(50, 0.0, 1.0)
    case = CS.Case("sod_stage", g, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2,
                   G.INT64_MAX, "riemann_x")
    out = {}
    for beta in (1.0, 1.5):
        r = O.RefSolver(g, case.bc, 1.4, G.SchemeParams(beta=beta))
        f0 = CS.initial_field(case)
        r.set_state(f0)
        out[f"beta_{beta}"] = g.interior(r.euler_stage(8e-4))
    np.savez_compressed(os.path.join(OUT, "euler_stage_sod50.npz"), initial=g.interior(f0), **out)
    # element known answers
    lib = O.ref_lib()
    D = O.DP
    rng = np.random.default_rng(0xF1)
    wl = np.column_stack([np.exp(rng.uniform(np.log(0.1), np.log(10), 200)),
                          rng.uniform(-5, 5, 200), rng.uniform(-5, 5, 200),
                          np.exp(rng.uniform(np.log(0.01), np.log(10), 200))])
    wr = np.column_stack([np.exp(rng.uniform(np.log(0.1), np.log(10), 200)),
                          rng.uniform(-5, 5, 200), rng.uniform(-5, 5, 200),
                          np.exp(rng.uniform(np.log(0.01), np.log(10), 200))])
    flux = np.zeros((2, 200, 4))
    hll = np.zeros((2, 200, 2))
    for ax, (nx_, ny_) in enumerate(((1.0, 0.0), (0.0, 1.0))):
        for k in range(200):
            a, b = np.ascontiguousarray(wl[k]), np.ascontiguousarray(wr[k])
            f = np.zeros(4)
            lib.lfr_edge_flux(a.ctypes.data_as(D), b.ctypes.data_as(D), nx_, ny_, 1.4,
                              f.ctypes.data_as(D))
            flux[ax, k] = f
            ps, us = np.zeros(1), np.zeros(1)
            lib.lfr_lagrangian_hll(a.ctypes.data_as(D), b.ctypes.data_as(D), nx_, ny_, 1.4,
                                   ps.ctypes.data_as(D), us.ctypes.data_as(D))
            hll[ax, k] = (ps[0], us[0])
    ab = rng.uniform(-10, 10, (2000, 2))
    betas = rng.uniform(1.0, 2.0, 2000)
    sw = np.array([lib.lfr_sweby(a, b, be) for (a, b), be in zip(ab, betas)])
    np.savez_compressed(os.path.join(OUT, "elements.npz"), wl=wl, wr=wr, flux=flux, hll=hll,
                        ab=ab, betas=betas, sweby=sw)
    print("elements ok")


if __name__ == "__main__":
    if "mat" in sys.argv[1:]:
        main_mat(force="--force" in sys.argv)
    else:
        main()
