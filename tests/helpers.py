"""Shared helpers for the parity tests (test infrastructure)."""
import os

import numpy as np

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLDEN, "make_golden.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.golden_cases()


def run_oracle(case, steps, field=None):
    """Drive the C restatement like run.cpp:180-210 (stop at t_final or after `steps`)."""
    s = O.OracleSolver(case.grid, case.bc, case.gamma, case.params)
    state = G.SolverState(field=CS.initial_field(case) if field is None else np.array(field))
    while state.step < steps and state.time < case.t_final:
        s.heun_step(state, case.cfl, case.t_final)
    diag = np.array([[d.dt, d.time, d.min_rho, d.min_p, d.step] for d in state.diagnostics])
    return state, diag


def diag_array(state):
    return np.array([[d.dt, d.time, d.min_rho, d.min_p, d.step] for d in state.diagnostics])


def assert_fields_equal(a, b, what=""):
    """Value equality per element (== treats -0.0 and +0.0 as equal)."""
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    bad = ~(a == b)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} of {a.size} values differ; first at {idx.tolist()}: "
                             f"{a[tuple(idx[0])]!r} vs {b[tuple(idx[0])]!r}")


def rel_l1(a, b):
    """Per-component relative L1 (absolute when the reference norm is 0)."""
    out = []
    for c in range(4):
        num = np.abs(a[c] - b[c]).sum()
        den = np.abs(b[c]).sum()
        out.append(num / den if den > 0 else num)
    return np.array(out)
