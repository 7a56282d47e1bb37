"""GPU: lf_edge_flux -- the reference's free edge_flux (solver.cpp:45-53) on the
device -- bit for bit against the reference compiled from its sources (signed
zeros included), over general normals, mixed gammas, the u* == 0 mean branch and
sound_speed's failure message (euler.hpp:99-104)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import solver as S

pytestmark = pytest.mark.gpu


def faces(n, seed):
    rng = np.random.default_rng(seed)
    w = lambda: np.stack([10.0 ** rng.uniform(-3, 3, n), rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 2, n),  # noqa: E731
                          rng.standard_normal(n), 10.0 ** rng.uniform(-3, 3, n)], axis=1)
    wm, wp = w(), w()
    th = rng.uniform(0, 2 * math.pi, n)
    nr = np.stack([np.cos(th), np.sin(th)], axis=1)
    nr[: n // 4] = (1.0, 0.0)
    nr[n // 4: n // 2] = (0.0, 1.0)
    wp[-n // 8:] = wm[-n // 8:]          # u* == 0 with a symmetric state and zero velocity
    wp[-n // 8:, 1:3] = wm[-n // 8:, 1:3] = 0.0
    wm[: n // 16, 1] = -0.0             # signed zeros through the normal products
    gm = rng.uniform(1.1, 3.0, n)
    gp = np.where(rng.random(n) < 0.5, gm, rng.uniform(1.1, 3.0, n))
    return wm, wp, nr, gm, gp


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_edge_flux_bitwise_vs_reference(cuda):
    n = 4096
    wm, wp, nr, gm, gp = faces(n, 7)
    flux, contact = S.edge_flux(wm, wp, nr, gm, gp)
    lib = O.ref_lib()
    rf, rc = np.zeros(4), np.zeros(2)
    msg = O.C.create_string_buffer(320)
    mean = 0
    for i in range(n):
        assert lib.lfr_edge_flux2(wm[i].ctypes.data_as(O.DP), wp[i].ctypes.data_as(O.DP), nr[i, 0], nr[i, 1],
                                  gm[i], gp[i], rf.ctypes.data_as(O.DP), rc.ctypes.data_as(O.DP), msg, 320) == 0
        assert np.array_equal(flux[i], rf) and np.array_equal(np.signbit(flux[i]), np.signbit(rf)), i
        assert np.array_equal(contact[i], rc), i
        mean += rc[1] == 0.0
    assert mean >= n // 8


def test_edge_flux_error_is_sound_speeds(cuda):
    wm, wp, nr, gm, gp = faces(64, 9)
    wp[40, 3] = -2.5       # right pressure of face 40
    wm[41, 0] = 0.0        # left density of face 41
    with pytest.raises(G.InvalidStateError) as e:
        S.edge_flux(wm, wp, nr, gm, gp)
    assert str(e.value) == "non-positive pressure = -2.500000"
    wm[12, 0] = -1.0
    wm[12, 3] = -1.0       # both checks fail: the density is reported first
    with pytest.raises(G.InvalidStateError) as e:
        S.edge_flux(wm, wp, nr, gm, gp)
    assert str(e.value) == "non-positive density = -1.000000"
    if O.ref_available():
        msg = O.C.create_string_buffer(320)
        f, c = np.zeros(4), np.zeros(2)
        assert O.ref_lib().lfr_edge_flux2(wm[12].ctypes.data_as(O.DP), wp[12].ctypes.data_as(O.DP), 1.0, 0.0,
                                          1.4, 1.4, f.ctypes.data_as(O.DP), c.ctypes.data_as(O.DP), msg, 320) == 1
        assert msg.value.decode() == "non-positive density = -1.000000"


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_free_compute_dt_equals_reference(cuda):
    """The free compute_dt (solver.cpp:55-59) on the device equals the reference's."""
    from paper_1607_08710_b200 import cases as CS
    case = CS.quadrant(96, 1)
    f = CS.initial_field(case)
    ctl = G.TimeControls(0.45, 1e30)
    for t, limit in ((0.0, 1e30), (0.25, 0.25 + 1e-6)):
        r = O.RefSolver(case.grid, G.BoundaryCondition(), 1.4)
        r.set_state(f)
        assert S.compute_dt(case.grid, f, 1.4, ctl, t, limit) == r.compute_dt(0.45, t, limit)
