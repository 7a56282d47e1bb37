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
