"""GPU: fastmath.cuh (the compiler's fast paths with shared reciprocals and deferred
range checks) equals the IEEE operators / the reference limiter wherever it
claims validity, on 2^28 random operand pairs over the whole finite range."""
import ctypes as C

import pytest

from paper_1607_08710_b200 import native as N

pytestmark = pytest.mark.gpu


def test_fast_division_sqrt_limiter_exact(cuda):
    counts = (C.c_int64 * 7)()
    n = 1 << 28
    assert N.lib().lf_selftest_fastmath(n, 0x1607087100, counts) == 0
    tested, div_ok, div_bad, shared_bad, sqrt_ok, sqrt_bad, lim_bad = list(counts)
    assert tested == n
    assert div_bad == 0 and shared_bad == 0 and sqrt_bad == 0 and lim_bad == 0
    # the fast paths must cover the physical range (half the draws) and more
    assert div_ok > 0.5 * n and sqrt_ok > 0.5 * n
