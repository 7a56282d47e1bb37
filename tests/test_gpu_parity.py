"""GPU parity: the CUDA path through the C ABI against the oracle and the golden vectors.

Bar (north star): bit equality per element (==) with the reference CPU build;
the tolerance the north star allows (relative L1 <= 1e-10, dt to 1e-12) is
asserted as well, but every case here is expected -- and required -- to be exact.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver
from helpers import (assert_fields_equal, diag_array, golden_cases, load_golden, rel_l1,
                     run_oracle)

pytestmark = pytest.mark.gpu

GOLDEN = list(golden_cases().items())
PATHS = ["staged", "twopass", "fused", "small"]


def run_gpu(case, steps, path="auto", devices=(0,), field=None, use_advance=False):
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, devices=devices, path=path)
    state = G.SolverState(field=CS.initial_field(case) if field is None else np.array(field))
    controls = G.TimeControls(case.cfl, case.t_final, steps)
    if use_advance:
        s.attach(state)
        while state.step < steps and state.time < case.t_final:
            if s.advance(state, controls, steps) == 0:
                break
    else:
        while state.step < steps and state.time < case.t_final:
            s.heun_step(state, controls, case.t_final)
    s.sync_to_host(state)
    s.close()
    return state


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name,spec", GOLDEN, ids=[n for n, _ in GOLDEN])
def test_golden_bitwise(cuda, name, spec, path):
    case, steps = spec
    gold = load_golden(name)
    state = run_gpu(case, steps, path)
    got = case.grid.interior(state.field)
    assert_fields_equal(got, gold["final"], f"{name}/{path}")
    d = diag_array(state)
    assert np.array_equal(d[:, :4], gold["diag"][:, :4]), "dt / time / min_rho / min_p"
    assert np.array_equal(np.array(state.boundary_outflow), gold["outflow"])
    assert rel_l1(got, gold["final"]).max() <= 1e-10


@pytest.mark.parametrize("name", ["quadrant_32", "smooth_32", "sod_400x4", "mixed_40x24"])
def test_device_resident_advance(cuda, name):
    """lf_advance (dt/time kept on the device, no per-step sync) == golden."""
    case, steps = dict(GOLDEN)[name]
    gold = load_golden(name)
    state = run_gpu(case, steps, "auto", use_advance=True)
    assert_fields_equal(case.grid.interior(state.field), gold["final"], name)
    assert np.array_equal(diag_array(state)[:, :4], gold["diag"][:, :4])


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cfg", ["quadrant", "sedov", "smooth"])
def test_larger_grids_vs_oracle(cuda, cfg, path):
    case = {"quadrant": CS.quadrant(256, 30), "sedov": CS.sedov(192, 30),
            "smooth": CS.smooth(200, 30, ny=136, y_extent=0.68)}[cfg]
    ref, rdiag = run_oracle(case, case.max_steps)
    state = run_gpu(case, case.max_steps, path)
    assert_fields_equal(case.grid.interior(state.field), case.grid.interior(ref.field), cfg)
    assert np.array_equal(diag_array(state)[:, :4], rdiag[:, :4])
    assert np.array_equal(np.array(state.boundary_outflow), np.array(ref.boundary_outflow))


@pytest.mark.parametrize("nslabs", [2, 3, 5])
@pytest.mark.parametrize("cfg", ["smooth", "sedov", "quadrant"])
def test_in_process_slabs_equal_single(cuda, cfg, nslabs):
    """y-slab decomposition (halo rows + combined dt) is bit-identical to one slab."""
    case = {"quadrant": CS.quadrant(64, 20), "sedov": CS.sedov(64, 20),
            "smooth": CS.smooth(64, 20, ny=45, y_extent=45 / 64)}[cfg]
    one = run_gpu(case, 20, "auto")
    many = run_gpu(case, 20, "auto", devices=[0] * nslabs)
    assert_fields_equal(case.grid.interior(many.field), case.grid.interior(one.field), cfg)
    assert np.array_equal(diag_array(many), diag_array(one))
    assert np.array_equal(np.array(many.boundary_outflow), np.array(one.boundary_outflow))


def test_euler_stage_golden(cuda):
    gold = load_golden("euler_stage_sod50")
    g = G.make_grid_1d(50, 0.0, 1.0)
    case = CS.Case("s", g, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5, 0.2, G.INT64_MAX,
                   "riemann_x")
    for beta in (1.0, 1.5):
        s = LagfluxSolver(g, case.bc, 1.4, G.SchemeParams(beta=beta))
        out = G.new_field(g)
        s.euler_stage(CS.initial_field(case), 8e-4, out)
        assert_fields_equal(g.interior(out), gold[f"beta_{beta}"], f"beta {beta}")


def test_compute_dt_known_answers(cuda):
    """test_solver.cpp:161-180."""
    import math
    g = G.make_grid_1d(100, 0.0, 1.0)
    f = G.new_field(g)
    r, mx, my, e = G.conserved_from_primitive(np.ones(100), np.zeros(100), np.zeros(100), np.ones(100), 1.4)
    g.interior(f)[:] = np.stack([r, mx, my, e])[:, None, :]
    s = LagfluxSolver(g, G.BoundaryCondition())
    dt = s.compute_dt(f, G.TimeControls(0.25, 10.0, 1000), 0.0, 10.0)
    assert dt == pytest.approx(0.25 * 0.01 / math.sqrt(1.4), rel=1e-15)
    assert dt == O.OracleSolver(g, G.BoundaryCondition()).compute_dt(f, 0.25, 0.0, 10.0)
    assert s.compute_dt(f, G.TimeControls(0.25, 10.0, 1000), 9.9999, 10.0) == 10.0 - 9.9999
    with pytest.raises(G.Error, match="non-positive time step"):
        s.compute_dt(f, G.TimeControls(0.25, 10.0, 1000), 10.0, 10.0)


def _sod1d(n=50):
    g = G.make_grid_1d(n, 0.0, 1.0)
    return g, CS.initial_field(CS.Case("s", g, G.BoundaryCondition(), 1.4, G.SchemeParams(), 0.5,
                                       0.2, G.INT64_MAX, "riemann_x"))


def test_errors_match_oracle_text(cuda):
    """PositivityError / InvalidStateError carry the reference's text and fields."""
    g, f = _sod1d()
    o = O.OracleSolver(g, G.BoundaryCondition())
    s = LagfluxSolver(g, G.BoundaryCondition())
    with pytest.raises(G.PositivityError) as eo:
        o.euler_stage(f.copy(), 10.0, G.new_field(g), 7)
    with pytest.raises(G.PositivityError) as eg:
        s.euler_stage(f.copy(), 10.0, G.new_field(g), 7)
    assert str(eg.value) == str(eo.value)
    assert (eg.value.cell_i, eg.value.cell_j, eg.value.step, eg.value.dt) == \
        (eo.value.cell_i, eo.value.cell_j, eo.value.step, eo.value.dt)
    bad = f.copy()
    bad[3, 0, 2 + 13] = -1.0
    with pytest.raises(G.InvalidStateError) as eo2:
        o.euler_stage(bad.copy(), 1e-4, G.new_field(g), 3)
    with pytest.raises(G.InvalidStateError) as eg2:
        s.euler_stage(bad.copy(), 1e-4, G.new_field(g), 3)
    assert str(eg2.value) == str(eo2.value)
    # compute_dt sees the bad cell first in a full step
    state = G.SolverState(field=bad.copy())
    with pytest.raises(G.InvalidStateError) as eg3:
        s.heun_step(state, G.TimeControls(0.5, 1.0), 1.0)
    ostate = G.SolverState(field=bad.copy())
    with pytest.raises(G.InvalidStateError) as eo3:
        o.heun_step(ostate, 0.5, 1.0)
    assert str(eg3.value) == str(eo3.value)


def test_trace_failure_text(cuda):
    from test_oracle_cpu import trace_failure_case
    g, f, params = trace_failure_case()
    o = O.OracleSolver(g, G.BoundaryCondition(), params=params)
    s = LagfluxSolver(g, G.BoundaryCondition(), params=params)
    with pytest.raises(G.InvalidStateError) as eo:
        o.euler_stage(f.copy(), 1e-4, G.new_field(g), 5)
    with pytest.raises(G.InvalidStateError) as eg:
        s.euler_stage(f.copy(), 1e-4, G.new_field(g), 5)
    assert str(eg.value) == str(eo.value)
    for path in PATHS:
        state = G.SolverState(field=f.copy())
        s2 = LagfluxSolver(g, G.BoundaryCondition(), params=params, path=path)
        with pytest.raises(G.InvalidStateError) as eg2:
            s2.heun_step(state, G.TimeControls(0.5, 1.0), 1.0)
        ostate = G.SolverState(field=f.copy())
        with pytest.raises(G.InvalidStateError) as eo2:
            o.heun_step(ostate, 0.5, 1.0)
        assert str(eg2.value) == str(eo2.value)


def test_corrector_positivity_failure_matches(cuda):
    """A step whose corrector loses positivity: same error, same (in-place) state."""
    g = G.make_grid_2d(24, 16, 0.0, 1.0, 0.0, 1.0)
    case = CS.Case("q", g, G.BoundaryCondition.uniform(G.TRANSMISSIVE), 1.4, G.SchemeParams(),
                   4.0, CS.STEP_DRIVEN_LIMIT, 5, "quadrant")   # CFL far beyond stability
    f0 = CS.initial_field(case)
    o = O.OracleSolver(g, case.bc)
    ostate = G.SolverState(field=f0.copy())
    with pytest.raises(G.Error) as eo:
        for _ in range(5):
            o.heun_step(ostate, case.cfl, case.t_final)
    for path in PATHS:
        s = LagfluxSolver(g, case.bc, path=path)
        state = G.SolverState(field=f0.copy())
        with pytest.raises(G.Error) as eg:
            for _ in range(5):
                s.heun_step(state, G.TimeControls(case.cfl, case.t_final), case.t_final)
        assert type(eg.value) is type(eo.value)
        assert str(eg.value) == str(eo.value)
        s.sync_to_host(state)
        assert_fields_equal(g.interior(state.field), g.interior(ostate.field), path)


def test_fourier_device_init_equals_host(cuda):
    case = CS.smooth(96, ny=80, y_extent=80 / 96)
    host = CS.initial_field(case)
    for devices in ((0,), (0, 0, 0)):
        s = LagfluxSolver(case.grid, case.bc, devices=devices)
        state = G.SolverState(field=G.new_field(case.grid))
        s.init_fourier(state, case.seed)
        s.sync_to_host(state)
        assert_fields_equal(case.grid.interior(state.field), case.grid.interior(host), str(devices))


def test_download_fill_ghosts_matches_reference_fill(cuda):
    case = CS.smooth(20, ny=12, y_extent=0.6)
    g = case.grid
    f = CS.initial_field(case)
    for bcs in ((0, 0, 0, 0), (1, 1, 1, 1), (2, 2, 2, 2), (2, 2, 1, 0)):
        bc = G.BoundaryCondition(*bcs)
        s = LagfluxSolver(g, bc)
        s.upload(f)
        out = G.new_field(g)
        s.download(out, fill_ghosts=True)
        ref = f.copy()
        lib = O.oracle_lib()
        for c, parity in enumerate((0, 1, 2, 0)):
            arr = np.ascontiguousarray(ref[c])
            lib.lfo_fill_ghosts(O.C.byref(O._cgrid(g)), (O.C.c_int * 4)(*bcs), parity,
                                arr.ctypes.data_as(O.DP))
            ref[c] = arr
        assert_fields_equal(out, ref, str(bcs))


@pytest.mark.parametrize("shape,devices", [((20, 12), (0,)), ((4, 4), (0,)), ((33, 17), (0, 0)),
                                          ((29, 24), (0, 0, 0)), ((37, 1), (0,)), ((3, 9), (0,))])
def test_device_ghost_fill_matches_reference(cuda, shape, devices):
    """The kernels' ghost fill (x and y sides in one launch when nx, ny >= 4; the
    two-kernel fill otherwise), corners included, against apply_boundary
    (grid.cpp:79-120) of the reference (the oracle's restatement without oracle/_ref)."""
    nx, ny = shape
    g = G.make_grid_1d(nx, 0.0, 1.0) if ny == 1 else G.make_grid_2d(nx, ny, 0.0, 1.0, 0.0, 0.7)
    rng = np.random.default_rng(nx * 100 + ny)
    f = G.new_field(g)
    g.interior(f)[...] = rng.standard_normal(g.interior(f).shape)
    g.interior(f)[1][..., 0] = 0.0                       # signed zeros through the flips
    fill = O.ref_lib().lfr_fill_ghosts if O.ref_available() else O.oracle_lib().lfo_fill_ghosts
    combos = [(a, b, c, d) for a in range(3) for b in range(3) for c in range(3) for d in range(3)
              if (a == 2) == (b == 2) and (c == 2) == (d == 2)]
    for bcs in combos:
        if g.dim == 1 and bcs[2:] != (0, 0):
            continue
        if len(devices) > 1 and (bcs[2] == 2) != (bcs[3] == 2):
            continue
        s = LagfluxSolver(g, G.BoundaryCondition(*bcs), devices=devices)
        s.upload(f)
        out = np.full_like(f, np.nan)
        s.download_ghosted(out)
        s.close()
        ref = f.copy()
        for c, parity in enumerate((0, 1, 2, 0)):
            arr = np.ascontiguousarray(ref[c])
            fill(O.C.byref(O._cgrid(g)), (O.C.c_int * 4)(*bcs), parity, arr.ctypes.data_as(O.DP))
            ref[c] = arr
        assert np.array_equal(out, ref), (bcs, devices)
        assert np.array_equal(np.signbit(out), np.signbit(ref)), (bcs, devices)


def _box_cases():
    """States outside the fast kernels' cell box (face_fast.cuh): each must take
    the stage-wise IEEE re-run and still equal the oracle."""
    base = CS.quadrant(48, 4)
    f = CS.initial_field(base)
    g = base.grid
    tiny_u = f.copy()
    tiny_u[1][g.gy + 10, g.gx + 5:g.gx + 9] = 1e-200 * tiny_u[0][g.gy + 10, g.gx + 5:g.gx + 9]
    light = f.copy()
    light[:, g.gy + 20:g.gy + 24, g.gx + 20:g.gx + 24] *= 1e-35   # rho, p ~ 1e-35 < 2^-100
    near_iso = CS.Case("q", g, base.bc, 1.00001, base.params, base.cfl, base.t_final, 4,
                       "quadrant")                                 # gamma - 1 < 2^-14
    return {"tiny_velocity": (base, tiny_u), "light_region": (base, light),
            "gamma_near_one": (near_iso, f)}


@pytest.mark.parametrize("path", ["twopass", "fused"])
def test_tiny_velocities_stay_on_the_fast_path(cuda, path):
    """Velocities down to the subnormals (numerical precursors ahead of shocks):
    the plain two-pass kernels flag the step, it is re-run by the exact two-pass
    kernels (div_exact) -- never by the stage-wise ones -- with the oracle's bits."""
    case, field = _box_cases()["tiny_velocity"]
    field = field.copy()
    g = case.grid
    field[2][g.gy + 20, g.gx + 3:g.gx + 7] = 5e-324 * field[0][g.gy + 20, g.gx + 3:g.gx + 7]
    ref, rdiag = run_oracle(case, 4, field=field)

    def run(fld):
        s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path)
        st = G.SolverState(field=np.array(fld))
        n0 = s.launch_count()
        for _ in range(4):
            s.heun_step(st, G.TimeControls(case.cfl, case.t_final), case.t_final)
        s.sync_to_host(st)
        n = s.launch_count() - n0
        s.close()
        return st, n

    state, n_tiny = run(field)
    assert_fields_equal(g.interior(state.field), g.interior(ref.field), "tiny")
    assert np.array_equal(diag_array(state)[:, :4], rdiag[:, :4])
    _, n_plain = run(CS.initial_field(CS.quadrant(48, 4)))
    if path == "twopass":
        assert n_tiny <= n_plain + 12  # one flagged two-pass attempt (7 launches + re-seed)
    else:
        assert n_tiny == n_plain       # the fused kernel always takes the exact quotient


@pytest.mark.parametrize("cfg", ["sedov", "quadrant"])
def test_shock_precursors_need_no_stagewise_rerun(cuda, cfg):
    """Shocks into quiescent regions create arbitrarily small velocities ahead of
    the front; the two-pass path switches to its exact kernels once (one flagged
    attempt) and never falls back to the stage-wise kernels; bits as the oracle."""
    case = CS.sedov(128, 40) if cfg == "sedov" else CS.quadrant(128, 40)
    f0 = CS.initial_field(case)
    ref, rdiag = run_oracle(case, 40, field=f0)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path="twopass")
    st = G.SolverState(field=f0.copy())
    counts = []
    for _ in range(40):
        n0 = s.launch_count()
        s.heun_step(st, G.TimeControls(case.cfl, case.t_final), case.t_final)
        counts.append(s.launch_count() - n0)
    s.sync_to_host(st)
    assert_fields_equal(case.grid.interior(st.field), case.grid.interior(ref.field), cfg)
    assert np.array_equal(diag_array(st)[:, :4], rdiag[:, :4])
    base = counts[-1]                                     # one step: 7 launches, +1 outflow sums
    assert max(counts[-20:]) == min(counts[-20:]) == base <= 8, counts
    assert max(counts) <= 2 * base + 3, counts            # no stage-wise re-run (29+)
    assert sum(c > base + 3 for c in counts) <= 1, counts  # at most one flagged step (the
    # first step also seeds the control record: rate, reset, accumulators)


@pytest.mark.parametrize("path", ["twopass", "fused"])
@pytest.mark.parametrize("which", ["light_region", "gamma_near_one"])
def test_out_of_box_states_rerun_exactly(cuda, which, path):
    case, field = _box_cases()[which]
    ref, rdiag = run_oracle(case, 4, field=field)

    def run(cs, fld):
        s = LagfluxSolver(cs.grid, cs.bc, cs.gamma, cs.params, path=path)
        state = G.SolverState(field=np.array(fld))
        n0 = s.launch_count()   # process-wide counter
        for _ in range(4):
            s.heun_step(state, G.TimeControls(cs.cfl, cs.t_final), cs.t_final)
        s.sync_to_host(state)
        n = s.launch_count() - n0
        s.close()
        return state, n

    state, n_out = run(case, field)
    assert_fields_equal(case.grid.interior(state.field), case.grid.interior(ref.field), which)
    assert np.array_equal(diag_array(state)[:, :4], rdiag[:, :4])
    # the fast kernel flagged every step and the stage-wise kernels recomputed it
    inbox = CS.quadrant(48, 4)
    _, n_in = run(inbox, CS.initial_field(inbox))
    assert n_out > n_in


@pytest.mark.parametrize("spatial_order", [1, 2])
@pytest.mark.parametrize("cfg", ["sod", "quadrant", "smooth"])
def test_time_order_1_on_the_two_pass_kernels(cuda, cfg, spatial_order):
    """time_order 1 (solver.cpp:510-514: one forward-Euler stage, F alone in the
    update and the outflow) runs as one corrector-kernel pass -- not stage-wise --
    and equals the oracle bit for bit."""
    import dataclasses
    base = {"sod": CS.sod(96, 8), "quadrant": CS.quadrant(80, 30),
            "smooth": CS.smooth(64, 30, ny=40, y_extent=40 / 64)}[cfg]
    case = dataclasses.replace(base, params=G.SchemeParams(spatial_order=spatial_order, time_order=1))
    ref, rdiag = run_oracle(case, 30)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path="twopass")
    st = G.SolverState(field=CS.initial_field(case))
    s.advance(st, G.TimeControls(case.cfl, case.t_final), 3)
    n0 = s.launch_count()
    s.advance(st, G.TimeControls(case.cfl, case.t_final), 27)
    per_step = (s.launch_count() - n0) / 27
    s.sync_to_host(st)
    s.close()
    assert_fields_equal(case.grid.interior(st.field), case.grid.interior(ref.field), cfg)
    assert np.array_equal(diag_array(st)[:, :4], rdiag[:, :4])
    assert list(st.boundary_outflow) == list(ref.boundary_outflow)
    assert per_step <= 5, per_step     # fill, pass, finalize (+ outflow sums): not stage-wise


@pytest.mark.parametrize("path", ["twopass", "fused", "staged"])
def test_foreign_field_between_steps_keeps_the_resident_state(cuda, path):
    """A diagnostic compute_dt / euler_stage of another field between heun_steps must
    not rewind the device-resident state (the mirror saves it into its host field
    before replacing it, solver.py _evict); results as the oracle's uninterrupted run."""
    case = CS.quadrant(48, 12)
    f0 = CS.initial_field(case)
    ref, rdiag = run_oracle(case, 12, field=f0)
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, path=path)
    st = G.SolverState(field=f0.copy())
    ctl = G.TimeControls(case.cfl, case.t_final, case.max_steps)
    other = CS.initial_field(CS.quadrant(48, 1))
    for k in range(12):
        s.heun_step(st, ctl, case.t_final)
        if k == 3:
            s.compute_dt(other, ctl, 0.0, 1e30)
        if k == 7:
            s.euler_stage(other.copy(), 1e-5, G.new_field(case.grid))
    s.sync_to_host(st)
    assert_fields_equal(case.grid.interior(st.field), case.grid.interior(ref.field), path)
    assert np.array_equal(diag_array(st)[:, :4], rdiag[:, :4])


def test_beta_below_one_runs_the_reference_limiter(cuda):
    """LimiterParams beta < 1 (accepted by LagfluxSolver, outside make_limiter's range):
    the fast kernels' limiter form holds for beta >= 1 only, so the handle runs the
    stage-wise kernels (or, on a small grid, the one-block path, whose IEEE arithmetic is
    the stage-wise kernels') -- bit-equal to the oracle, which evaluates sweby as written."""
    case = CS.quadrant(40, 10)
    params = G.SchemeParams(beta=0.5)
    f0 = CS.initial_field(case)
    o = O.OracleSolver(case.grid, case.bc, case.gamma, params)
    ref = G.SolverState(field=f0.copy())
    for _ in range(10):
        o.heun_step(ref, case.cfl, case.t_final)
    for path in ("auto", "fused", "twopass", "small"):
        s = LagfluxSolver(case.grid, case.bc, case.gamma, params, path=path)
        want = {"small": ("small",), "auto": ("small", "staged")}.get(path, ("staged",))
        assert s.resolved_path() in want, path
        st = G.SolverState(field=f0.copy())
        for _ in range(10):
            s.heun_step(st, G.TimeControls(case.cfl, case.t_final), case.t_final)
        s.sync_to_host(st)
        assert_fields_equal(case.grid.interior(st.field), case.grid.interior(ref.field), path)
