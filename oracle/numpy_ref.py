"""Vectorised numpy restatement of the stage-wise Heun step on a y-slab.  TEST INFRASTRUCTURE.

Same algorithm and operation order as oracle/lagflux_oracle.c (which cites the
reference file:line for every piece), written on arrays so that a slab with
explicit halo rows can be stepped: tests/test_slab_gloo.py runs it on two gloo
ranks with the library's slab partition, the NCCL path's halo protocol and its
reductions, and checks the result against the single-domain C oracle bit for
bit.  numpy evaluates each binary operation with one IEEE rounding (no FMA) and
np.sqrt is correctly rounded, so the values match the C build exactly.

Slab arrays have shape (4, rows + 4, nx + 4): two ghost / halo rows below and
above, two ghost columns left and right (the reference's ghost width).
"""
from __future__ import annotations

import numpy as np

G = 2  # ghost width (grid.cpp:53-54)


def fill_x(f, bc_lo, bc_hi):
    """grid.cpp:81-96 on the interior rows of every component."""
    nx = f.shape[2] - 2 * G
    for c in range(4):
        sx = -1.0 if c == 1 else 1.0
        a = f[c, G:-G]
        for l in range(1, G + 1):
            lo, hi = G - l, G + nx - 1 + l
            if bc_lo == 0:
                a[:, lo] = a[:, G]
            elif bc_lo == 1:
                a[:, lo] = sx * a[:, G + l - 1]
            else:
                a[:, lo] = a[:, G + ((nx - l) % nx + nx) % nx]
            if bc_hi == 0:
                a[:, hi] = a[:, G + nx - 1]
            elif bc_hi == 1:
                a[:, hi] = sx * a[:, G + nx - l]
            else:
                a[:, hi] = a[:, G + (l - 1) % nx]


def fill_y(f, bc_lo, bc_hi, do_lo=True, do_hi=True):
    """grid.cpp:98-113 over every column (corners pick up the x ghosts)."""
    ny = f.shape[1] - 2 * G
    for c in range(4):
        sy = -1.0 if c == 2 else 1.0
        a = f[c]
        for l in range(1, G + 1):
            lo, hi = G - l, G + ny - 1 + l
            if do_lo:
                if bc_lo == 0:
                    a[lo] = a[G]
                elif bc_lo == 1:
                    a[lo] = sy * a[G + l - 1]
                else:
                    a[lo] = a[G + ((ny - l) % ny + ny) % ny]
            if do_hi:
                if bc_hi == 0:
                    a[hi] = a[G + ny - 1]
                elif bc_hi == 1:
                    a[hi] = sy * a[G + ny - l]
                else:
                    a[hi] = a[G + (l - 1) % ny]


def primitives(f, gm1):
    """solver.cpp:153-157 (all cells; callers use physical data)."""
    r, mx, my, e = f
    inv = 1.0 / r
    return np.stack([r, mx * inv, my * inv, gm1 * (e - 0.5 * (mx * mx + my * my) * inv)])


def _min(a, b):
    return np.where(b < a, b, a)


def _max(a, b):
    return np.where(a < b, b, a)


def sweby(a, b, beta):
    """reconstruct.hpp:24-30"""
    with np.errstate(invalid="ignore", over="ignore"):
        aa, bb = np.abs(a), np.abs(b)
        m = _max(_min(aa, beta * bb), _min(beta * aa, bb))
        return np.where(a * b > 0.0, np.where(a > 0.0, m, -m), 0.0)


def conserved(w, gm1):
    """euler.hpp:91-95 (gamma - 1 recomputed inline in the reference: same value)."""
    r, u, v, p = w
    return np.stack([r, r * u, r * v, p / gm1 + 0.5 * r * (u * u + v * v)])


def face_flux(wm, wp, axis, gamma, gm1):
    """riemann_hll.hpp:29-39 + solver.cpp:26-43 with n = e_axis."""
    nx_, ny_ = (1.0, 0.0) if axis == 0 else (0.0, 1.0)
    ul = wm[1] * nx_ + wm[2] * ny_
    ur = wp[1] * nx_ + wp[2] * ny_
    cl = np.sqrt(gamma * wm[3] / wm[0])
    cr = np.sqrt(gamma * wp[3] / wp[0])
    cmax = _max(cl, cr)
    rs = wm[0] + wp[0]
    ps = (wp[0] * wm[3] + wm[0] * wp[3]) / rs - (wm[0] * wp[0] / rs) * cmax * (ur - ul)
    us = (wm[0] * ul + wp[0] * ur) / rs - (wp[3] - wm[3]) / (cmax * rs)
    um, up = conserved(wm, gm1), conserved(wp, gm1)
    ua = np.where(us > 0.0, um, np.where(us < 0.0, up, 0.5 * (um + up)))
    return np.stack([ua[0] * us, ua[1] * us + ps * nx_, ua[2] * us + ps * ny_, ua[3] * us + ps * us])


def traces(q, axis, beta):
    """minus / plus traces of every face along `axis` (reconstruct.hpp:44-49).

    x: faces between columns i-1 and i for i in [G, G+nx] (rows G..G+rows-1);
    y: faces between rows j-1 and j for j in [G, G+rows] (cols G..G+nx-1)."""
    if axis == 0:
        q = q[:, G:-G, :]
        q0, q1, q2, q3 = q[..., 0:-3], q[..., 1:-2], q[..., 2:-1], q[..., 3:]
    else:
        q = q[:, :, G:-G]
        q0, q1, q2, q3 = q[:, 0:-3], q[:, 1:-2], q[:, 2:-1], q[:, 3:]
    s1 = sweby(q2 - q1, q1 - q0, beta)
    s2 = sweby(q3 - q2, q2 - q1, beta)
    return q1 + 0.5 * s1, q2 - 0.5 * s2


def stage_fluxes(f, gamma, beta):
    gm1 = gamma - 1.0
    w = primitives(f, gm1)
    fx = face_flux(*traces(w, 0, beta), 0, gamma, gm1)   # (4, rows, nx+1)
    fy = face_flux(*traces(w, 1, beta), 1, gamma, gm1)   # (4, rows+1, nx)
    return fx, fy


def apply_update(base, fa, fb, dt, dx, dy):
    """solver.cpp:272-308; fb None: one flux set.  Returns interior values, min rho, min e_int."""
    lam_x, lam_y = dt / dx, dt / dy
    fxa, fya = fa
    if fb is None:
        fxl, fxr, fyb, fyt = fxa[..., :-1], fxa[..., 1:], fya[:, :-1], fya[:, 1:]
    else:
        fxb, fyb_ = fb
        fxl = 0.5 * (fxa[..., :-1] + fxb[..., :-1])
        fxr = 0.5 * (fxa[..., 1:] + fxb[..., 1:])
        fyb = 0.5 * (fya[:, :-1] + fyb_[:, :-1])
        fyt = 0.5 * (fya[:, 1:] + fyb_[:, 1:])
    val = base[:, G:-G, G:-G] - lam_x * (fxr - fxl)
    val = val - lam_y * (fyt - fyb)
    eint = val[3] - 0.5 * (val[1] * val[1] + val[2] * val[2]) / val[0]
    assert np.all(val[0] > 0.0) and np.all(eint > 0.0), "test data must stay physical"
    return val, val[0].min(), eint.min()


def local_rate(f, gamma, dx, dy):
    """max over the slab's interior of the CFL rate (solver.cpp:457-469)."""
    r, mx, my, e = f[:, G:-G, G:-G]
    inv = 1.0 / r
    u, v = mx * inv, my * inv
    p = (gamma - 1.0) * (e - 0.5 * (mx * mx + my * my) * inv)
    c = np.sqrt(gamma * p * inv)
    rr = (np.abs(u) + c) / dx + (np.abs(v) + c) / dy
    return rr.max()


def boundary_faces(fa, fb):
    """Heun-averaged faces on the domain boundary (solver.cpp:410-411)."""
    fxa, fya = fa
    fxb, fyb = fb
    fx = 0.5 * (fxa + fxb)
    fy = 0.5 * (fya + fyb)
    return fx[..., 0], fx[..., -1], fy[:, 0, :], fy[:, -1, :]


def ordered_outflow(acc, left, right, bot, top, dt, dx, dy):
    """solver.cpp:412-430 (serial, fixed order)."""
    ax, ay = dt * dy, dt * dx
    out = list(acc)
    for c in range(4):
        s = 0.0
        for j in range(left.shape[1]):
            s += right[c, j] - left[c, j]
        out[c] += ax * s
    for c in range(4):
        s = 0.0
        for i in range(bot.shape[1]):
            s += top[c, i] - bot[c, i]
        out[c] += ay * s
    return out
