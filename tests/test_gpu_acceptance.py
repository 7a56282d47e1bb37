"""GPU: the reference's own acceptance program (tests/acceptance.cpp, its 12 SPEC
criteria) and driver loop (run.cpp run_hydro_case, bench.cpp run_steps) running on the
B200 path.  oracle/Makefile compiles those reference sources where they lie with
oracle/dropin_swap.hpp force-included, so their three `LagfluxSolver solver(...)`
constructions build lagflux::b200::LagfluxSolver (include/lagflux_b200.hpp); the same
program without the swap is the CPU reference.  Both run here side by side: every
criterion line must read the same (verdict and every reported number: errors, orders,
minima, drifts, step counts) apart from wall-clock figures, and every dump the driver
writes (field_csv through run.cpp's dump lambda) must be byte-identical.

Criteria 10 and 11 FAIL for the unmodified reference too (#10 compares
dumps whose header digest covers the worker count, #11 is the out-of-scope advection
solver); the swapped program must fail them in the same way, not differently."""
import filecmp
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
B200 = os.path.join(REF_DIR, "acceptance_b200")
RESIDENT = os.path.join(REF_DIR, "acceptance_b200_resident")
REF = os.path.join(REF_DIR, "acceptance_ref")
CASES = os.path.join(REF_DIR, "cases")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def runs(cuda, tmp_path_factory):
    """{exe: (cwd, returncode, stdout, stderr)}: the three programs run side by side
    (two on the GPU, the CPU reference on the host cores), once per session."""
    for p in (B200, RESIDENT, REF, CASES):
        assert os.path.exists(p), f"{p} not built (make -C oracle acceptance)"
    env = dict(os.environ, LAGFLUX_CASE_DIR=CASES)
    # criterion 1 also asks each Sod run for < 5 s of wall clock, and the program's first
    # run pays the process's CUDA start-up: page the driver and the library in first
    # (a fresh box loads them from a cold image), so that the timing sees a warm start
    warm = os.path.join(REF_DIR, "dropin_check")
    if os.path.exists(warm):
        subprocess.run([warm], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=900)
    procs = {}
    for exe in (B200, RESIDENT, REF):
        cwd = tmp_path_factory.mktemp(os.path.basename(exe))
        procs[exe] = (cwd, subprocess.Popen([exe], cwd=cwd, env=env, stdout=subprocess.PIPE,
                                            stderr=subprocess.PIPE, text=True))
    res = {}
    for exe, (cwd, p) in procs.items():
        try:
            out, err = p.communicate(timeout=1500)
        except subprocess.TimeoutExpired:
            p.kill()
            out, err = p.communicate()
        res[exe] = (cwd, p.returncode, out, err)
    return res


def _criteria(stdout):
    """{n: (verdict, text without wall-clock figures)}"""
    res = {}
    for line in stdout.splitlines():
        m = re.match(r"\[\s*(\d+)/12\]\s+(PASS|FAIL)\s+(.*)", line)
        if not m:
            continue
        text = m.group(3)
        text = re.sub(r", runtimes .*", "", text)            # criterion 1
        text = re.sub(r"MCUPs/speedup: .*", "", text)        # criterion 10
        res[int(m.group(1))] = (m.group(2), text)
    return res


@pytest.mark.parametrize("exe", [B200, RESIDENT], ids=["solver_swapped", "driver_swapped"])
def test_reference_acceptance_program_on_the_gpu_path(cuda, runs, exe):
    """solver_swapped: the reference's run.cpp loop stepping the GPU solver (state.field
    copied both ways every step).  driver_swapped: acceptance.cpp's run_hydro_case calls
    also go to lagflux::b200::run_hydro_case (include/lagflux_b200_run.hpp): the state
    stays on the device between dump events and the dumps are written from it."""
    db, rc_b, out_b, err_b = runs[exe]
    dr, rc_r, out_r, err_r = runs[REF]
    print(out_b)
    cb, cr = _criteria(out_b), _criteria(out_r)
    assert sorted(cb) == list(range(1, 13)), out_b + err_b
    assert sorted(cr) == list(range(1, 13)), out_r + err_r
    # the hot path's criteria pass on the GPU
    for n in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12):
        assert cb[n][0] == "PASS", cb[n]
    # and every line reads as the reference's does, number for number
    for n in range(1, 13):
        assert cb[n] == cr[n], (n, cb[n], cr[n])
    assert rc_b == rc_r
    # every dump and diagnostics file the driver wrote: byte-identical
    fb = sorted(os.listdir(db / "acceptance_out"))
    fr = sorted(os.listdir(dr / "acceptance_out"))
    assert fb == fr and fb
    for f in fb:
        assert filecmp.cmp(db / "acceptance_out" / f, dr / "acceptance_out" / f, shallow=False), f
