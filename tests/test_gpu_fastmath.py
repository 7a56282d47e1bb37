"""GPU: fastmath.cuh (the compiler's fast paths with shared reciprocals and deferred
range checks) equals the IEEE operators / the reference limiter wherever it
claims validity, on 2^28 random operand pairs over the whole finite range."""
import ctypes as C

import pytest

from paper_1607_08710_b200 import native as N

pytestmark = pytest.mark.gpu


def test_fast_division_sqrt_limiter_exact(cuda):
    counts = (C.c_int64 * 10)()
    n = 1 << 28
    assert N.lib().lf_selftest_fastmath(n, 0x1607087100, counts) == 0
    tested, div_ok, div_bad, shared_bad, sqrt_ok, sqrt_bad, lim_bad, tiny, tiny_bad, tiny_oor = list(counts)
    assert tested == n
    assert div_bad == 0 and shared_bad == 0 and sqrt_bad == 0 and lim_bad == 0
    # div_exact (tiny dividends, subnormal quotients, constructed rounding ties)
    assert tiny == n and tiny_bad == 0 and tiny_oor == 0
    # the fast paths must cover the physical range (half the draws) and more
    assert div_ok > 0.5 * n and sqrt_ok > 0.5 * n


def test_cell_box_implies_fast_path_validity(cuda):
    """The kernels test one box per cell instead of range-checking every
    division (face_fast.cuh): faces built from in-box cells -- box edges,
    one-ulp neighbours and zero velocities over-represented -- never fail a
    fast-path range check."""
    counts = (C.c_int64 * 2)()
    n = 1 << 26
    assert N.lib().lf_selftest_box(n, 0x1607087101, counts) == 0
    solved, failed = list(counts)
    assert solved > n // 4
    assert failed == 0


def test_epilogue_box_implies_fast_path_validity(cuda):
    """The corrector's epilogue box (cell_epilogue_box): wherever it accepts an
    updated cell, the per-operation checks pass and rate / e_int are identical."""
    counts = (C.c_int64 * 3)()
    n = 1 << 26
    assert N.lib().lf_selftest_epilogue(n, 0x1607087102, counts) == 0
    accepted, check_failed, differ = list(counts)
    assert accepted > n // 8
    assert check_failed == 0
    assert differ == 0


def test_fp64_peak_measurement(cuda):
    """lf_fp64_peak (the fp64 roof bench.py reports against): DFMA, DMUL and DADD
    thread-instruction rates, burst and sustained, positive and consistent with one
    fp64 instruction per lane per cycle on 64 lanes per SM (B200: ~18.5 T/s)."""
    out = (C.c_double * 6)()
    assert N.lib().lf_fp64_peak(0, 20.0, 100.0, out) == 0
    rates = list(out)
    assert all(r > 1e12 for r in rates), rates
    assert max(rates) / min(rates) < 1.2, rates
    assert N.lib().lf_fp64_peak(0, 0.0, 0.0, out) == N.LF_ERR_ARGUMENT
