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


def test_known_answers_on_the_device(cuda):
    """test_solver.cpp:114-137 and test_riemann.cpp:19-43, through lf_edge_flux."""
    wm = np.array([[1.0, 2.0, 0.0, 1.0], [1.0, 1.0, 0.0, 1.0], [1.0, 1.0, 0.0, 1.0],
                   [1.0, 0.0, 0.0, 1.0], [0.7, 1.3, 0.0, 2.1]])
    wp = np.array([[1.0, 2.0, 0.0, 1.0], [1.0, -1.0, 0.0, 1.0], [0.5, 0.8, 0.0, 0.9],
                   [0.125, 0.0, 0.0, 0.1], [0.7, 1.3, 0.0, 2.1]])
    f, c = S.edge_flux(wm, wp, [1.0, 0.0], 1.4)
    assert f[0, 0] == pytest.approx(2.0, rel=1e-14) and f[0, 1] == pytest.approx(5.0, rel=1e-14)
    assert f[0, 2] == 0.0 and f[0, 3] == pytest.approx(11.0, rel=1e-14)
    assert f[1, 0] == 0.0 and f[1, 3] == 0.0 and f[1, 1] == pytest.approx(1.0 + math.sqrt(1.4), rel=1e-14)
    assert c[2, 1] > 0.0 and f[2, 0] == 1.0 * c[2, 1]
    assert c[3, 0] == pytest.approx(0.2, rel=1e-14) and c[3, 1] == pytest.approx(0.8 / math.sqrt(1.4), rel=1e-14)
    assert c[4, 0] == pytest.approx(2.1, rel=1e-15) and c[4, 1] == pytest.approx(1.3, rel=1e-15)


def _state_gen(n, seed):
    """testing::StateGen (test_util.hpp:12-36): log-uniform rho in [0.1, 10], p in
    [0.01, 10], u, v uniform in [-5, 5]."""
    rng = np.random.default_rng(seed)
    rho = np.exp(rng.uniform(np.log(0.1), np.log(10.0), n))
    p = np.exp(rng.uniform(np.log(0.01), np.log(10.0), n))
    return np.stack([rho, rng.uniform(-5, 5, n), rng.uniform(-5, 5, n), p], axis=1)


def test_flux_consistency_and_symmetries_on_the_device(cuda):
    """test_solver.cpp:139-159 (consistency: equal traces give the exact Euler flux
    F(U).n, 4 normals, 1e-14) and test_riemann.cpp:45-67 (mirror symmetry of the
    contact solution), 1000 states each, on lf_edge_flux."""
    n = 1000
    w = _state_gen(n, 0xF1)
    g = 1.4
    for nrm in ((1.0, 0.0), (0.0, 1.0), (-1.0, 0.0), (0.6, 0.8)):
        f, c = S.edge_flux(w, w, nrm, g)
        rho, u, v, p = w.T
        un = u * nrm[0] + v * nrm[1]
        E = p / (g - 1.0) + 0.5 * rho * (u * u + v * v)
        exact = np.stack([rho * un, rho * u * un + p * nrm[0], rho * v * un + p * nrm[1], (E + p) * un], axis=1)
        scale = 1.0 + np.abs(exact)
        assert np.all(np.abs(f - exact) <= 1e-14 * scale * 8), nrm
        assert np.allclose(c[:, 0], p, rtol=1e-14) and np.allclose(c[:, 1], un, rtol=1e-14, atol=1e-14)
    # mirror: swapping the sides and flipping the normal velocity mirrors (p*, u*)
    wl, wr = _state_gen(n, 0x411), _state_gen(n, 0x412)
    ml, mr = wr.copy(), wl.copy()
    ml[:, 1] *= -1.0
    mr[:, 1] *= -1.0
    _, c1 = S.edge_flux(wl, wr, (1.0, 0.0), g)
    _, c2 = S.edge_flux(ml, mr, (1.0, 0.0), g)
    assert np.allclose(c1[:, 0], c2[:, 0], rtol=1e-13) and np.allclose(c1[:, 1], -c2[:, 1], rtol=1e-13, atol=1e-13)
