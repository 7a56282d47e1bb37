"""GPU: the LF_MATH_CONTRACT arithmetic (FMA contraction, reciprocal products) of the
two-pass kernels, held to the north star's tolerance instead of bit equality:

    relative L1 <= 1e-10 per conserved field after the case's steps,
    dt sequence equal to 1e-12 (relative, step by step, same step count).

Small cases compare with the reference's golden vectors (tests/golden, made by the
compiled reference); BASELINE configs 1-3 at full size and a 4096^2 strip of the
config-4 generator compare with the exact GPU path, which the parity tests prove
bit-identical to the reference (test_gpu_parity.py, profiles/r01_configs_1_2_3.json).
"""
import numpy as np
import pytest

from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200.solver import LagfluxSolver

from helpers import diag_array, golden_cases, load_golden, rel_l1

pytestmark = pytest.mark.gpu

TOL_FIELD = 1e-10   # north star: relative L1 per conserved field
TOL_DT = 1e-12      # north star: dt sequences

GOLDEN_2D = [(n, s) for n, s in golden_cases().items() if s[0].grid.dim == 2]


def run(case, steps, math, use_advance=True, seed_state=False, path="twopass"):
    s = LagfluxSolver(case.grid, case.bc, case.gamma, case.params, devices=(0,), path=path,
                      math=math)
    controls = G.TimeControls(case.cfl, case.t_final, steps)
    if seed_state:
        state = G.SolverState(field=G.new_field(case.grid))
        s.init_fourier(state, case.seed)
    else:
        state = G.SolverState(field=CS.initial_field(case))
        s.attach(state)
    while state.step < steps and state.time < case.t_final:
        if use_advance:
            if s.advance(state, controls, steps) == 0:
                break
        else:
            s.heun_step(state, controls, case.t_final)
    s.sync_to_host(state)
    s.close()
    return state


def assert_within_tolerance(got_state, ref_field, ref_dt, grid, what):
    got = grid.interior(got_state.field)
    err = rel_l1(got, ref_field)
    assert err.max() <= TOL_FIELD, f"{what}: relative L1 per field {err.tolist()}"
    dt = diag_array(got_state)[:, 0]
    assert dt.shape == ref_dt.shape, f"{what}: {dt.shape[0]} steps vs {ref_dt.shape[0]}"
    rel = np.abs(dt - ref_dt) / np.abs(ref_dt)
    assert rel.max() <= TOL_DT, f"{what}: dt relative difference {rel.max():.3e}"
    return err, rel.max()


@pytest.mark.parametrize("name,spec", GOLDEN_2D, ids=[n for n, _ in GOLDEN_2D])
@pytest.mark.parametrize("stepwise", [False, True], ids=["advance", "heun_step"])
@pytest.mark.parametrize("path", ["twopass", "fused"])
def test_contract_golden_within_tolerance(cuda, name, spec, stepwise, path):
    case, steps = spec
    gold = load_golden(name)
    state = run(case, steps, "contract", use_advance=not stepwise, path=path)
    assert_within_tolerance(state, gold["final"], gold["diag"][:, 0], case.grid, name)


@pytest.mark.parametrize("path", ["twopass", "fused"])
def test_contract_kernels_are_the_ones_running(cuda, path):
    """The contract handle really computes differently (else the test above proves nothing)."""
    case = CS.smooth(256, 10)
    a = run(case, 10, "exact", seed_state=True, path=path)
    b = run(case, 10, "contract", seed_state=True, path=path)
    g = case.grid
    assert not np.array_equal(g.interior(a.field), g.interior(b.field))
    err = rel_l1(g.interior(b.field), g.interior(a.field))
    assert 0 < err.max() <= TOL_FIELD


FULL = [
    ("config1_sod_400x4", CS.sod(), 10 ** 6),
    ("config2_quadrant_1024", CS.quadrant(1024, 200), 200),
    ("config3_sedov_4096", CS.sedov(4096, 100), 100),
]


@pytest.mark.slow
@pytest.mark.parametrize("path", ["twopass", "fused"])
@pytest.mark.parametrize("name,case,steps", FULL, ids=[f[0] for f in FULL])
def test_contract_baseline_configs_full_size(cuda, name, case, steps, path):
    ref = run(case, steps, "exact")
    got = run(case, steps, "contract", path=path)
    err, dterr = assert_within_tolerance(got, case.grid.interior(ref.field), diag_array(ref)[:, 0],
                                         case.grid, name)
    print(f"{name}: relative L1 {err.tolist()}, dt {dterr:.2e}")


@pytest.mark.slow
@pytest.mark.parametrize("path", ["twopass", "fused"])
def test_contract_smooth_4096(cuda, path):
    """The headline generator (config 4) at 4096^2, 50 steps."""
    case = CS.smooth(4096, 50)
    ref = run(case, 50, "exact", seed_state=True)
    got = run(case, 50, "contract", seed_state=True, path=path)
    assert_within_tolerance(got, case.grid.interior(ref.field), diag_array(ref)[:, 0], case.grid,
                            "smooth_4096")
