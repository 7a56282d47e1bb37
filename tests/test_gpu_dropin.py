"""GPU: the C++ drop-in (include/lagflux_b200.hpp) against the reference's own
LagfluxSolver, both driven through the reference's C++ types (tools/dropin_check.cpp,
built with the reference sources into oracle/_ref/ by oracle/Makefile)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference(cuda):
    assert os.path.exists(EXE), "oracle/_ref/dropin_check not built (make -C oracle dropin)"
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK (0 mismatches)" in out.stdout


DRIVER = os.path.join(ROOT, "oracle", "_ref", "driver_check")
CASES = os.path.join(ROOT, "oracle", "_ref", "cases")


def test_cpp_driver_loop_matches_reference(cuda, tmp_path):
    """lagflux::b200::run_hydro_case (include/lagflux_b200_run.hpp) next to the
    reference's run_hydro_case (run.cpp:132-227) on the same CaseConfigs
    (tools/driver_check.cpp): scheduled dumps, a max_steps truncation, three materials,
    a run failing at once and one failing after five steps -- the same HydroRun, the same
    exception, byte-identical dumps and diagnostics files."""
    assert os.path.exists(DRIVER), "oracle/_ref/driver_check not built (make -C oracle driver)"
    out = subprocess.run([DRIVER], cwd=tmp_path, env=dict(os.environ, LAGFLUX_CASE_DIR=CASES),
                         capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK (0 mismatches)" in out.stdout
    assert "sod2d-failing-late: " in out.stdout and "step 5" in out.stdout
