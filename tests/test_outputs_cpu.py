"""CPU: the host-side output formatting (paper_1607_08710_b200/outputs.py) against the
reference's own diagnostics_csv (csv.cpp:104-114, compiled into oracle/_ref)."""
import os

import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import outputs as OUT
from helpers import run_oracle

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

EDGE = [G.StepDiagnostics(0, 0.0, 0.0, 0.0, 0.0),
        G.StepDiagnostics(1, 1e-300, 5e-324, -0.0, 1.7976931348623157e308),
        G.StepDiagnostics(2**62, 0.1, 1.0 / 3.0, 2.5e-16, -1e-17),
        G.StepDiagnostics(-3, float("inf"), float("-inf"), 123456789.125, 1e22)]


def _oracle_diags(steps=40):
    case = CS.sod(100, 4)
    state, _ = run_oracle(case, steps)
    return state.diagnostics


@needs_ref
@pytest.mark.parametrize("which", ["empty", "edge", "sod"])
def test_diagnostics_csv_matches_reference(which):
    diags = {"empty": [], "edge": EDGE, "sod": None}[which]
    if diags is None:
        diags = _oracle_diags()
        assert len(diags) == 40
    assert OUT.diagnostics_csv(diags).encode() == O.ref_diagnostics_csv(diags)


def test_diagnostics_csv_layout(tmp_path):
    diags = _oracle_diags(3)
    p = os.path.join(str(tmp_path), "run_diag.csv")
    OUT.write_diagnostics_csv(p, diags)
    lines = open(p).read().splitlines()
    assert lines[0] == "step,time,dt,min_rho,min_p"
    assert [int(l.split(",")[0]) for l in lines[1:]] == [1, 2, 3]
    for l, d in zip(lines[1:], diags):
        assert [float(x) for x in l.split(",")[1:]] == [d.time, d.dt, d.min_rho, d.min_p]
    assert OUT.format_g17(0.1) == "0.10000000000000001"
