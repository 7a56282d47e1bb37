"""ctypes loaders for the two CPU parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module; the product (paper_1607_08710_b200) never does.

  OracleSolver  -> oracle/_build/liboracle.so   C restatement (lagflux_oracle.c)
  RefSolver     -> oracle/_ref/libref_lagflux.so the unmodified reference solver
                   (/root/reference/proj/src/solver.cpp + grid.cpp, via ref_shim.cpp)

Both take the same plain descriptors as the product (grid.py types) and work on
(4, nyt, nxt) float64 fields in the reference's ghosted layout.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Tuple

import numpy as np

from paper_1607_08710_b200 import grid as G

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_lagflux.so")

# error kinds (lagflux_oracle.h)
ERR_CONFIG, ERR_DT_STATE, ERR_DT_NONPOS, ERR_PRIMITIVE, ERR_TRACE, ERR_POSITIVITY = 1, 2, 3, 4, 5, 6
ERR_FRACTION = 9


class lfo_grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("gx", C.c_int),
                ("gy", C.c_int), ("dx", C.c_double), ("dy", C.c_double), ("x0", C.c_double),
                ("y0", C.c_double)]


class lfo_scheme(C.Structure):
    _fields_ = [("gamma", C.c_double), ("beta", C.c_double), ("spatial_order", C.c_int),
                ("time_order", C.c_int), ("bc", C.c_int * 4)]


class lfo_error(C.Structure):
    _fields_ = [("kind", C.c_int), ("axis", C.c_int), ("i", C.c_int64), ("j", C.c_int64),
                ("step", C.c_int64), ("dt", C.c_double), ("value", C.c_double),
                ("value2", C.c_double), ("message", C.c_char * 320)]


class lfo_step_out(C.Structure):
    _fields_ = [("dt", C.c_double), ("hits_limit", C.c_int), ("time", C.c_double),
                ("step", C.c_int64), ("min_rho", C.c_double), ("min_p", C.c_double),
                ("boundary_outflow", C.c_double * 4)]


P4 = C.POINTER(C.c_double) * 4
DP = C.POINTER(C.c_double)


def _ptrs(field: np.ndarray):
    assert field.dtype == np.float64 and field.flags.c_contiguous and field.shape[0] == 4
    return P4(*[field[c].ctypes.data_as(DP) for c in range(4)])


def _kptrs(partial: np.ndarray):
    """(n, nyt, nxt) partial densities -> double*[n]."""
    assert partial.dtype == np.float64 and partial.flags.c_contiguous
    return (DP * partial.shape[0])(*[partial[k].ctypes.data_as(DP) for k in range(partial.shape[0])])


def _cgrid(g: G.CartesianGrid) -> lfo_grid:
    return lfo_grid(g.dim, g.nx, g.ny, g.gx, g.gy, g.dx, g.dy, g.x0, g.y0)


def _cscheme(gamma: float, params: G.SchemeParams, bc: G.BoundaryCondition) -> lfo_scheme:
    return lfo_scheme(gamma, params.beta, params.spatial_order, params.time_order,
                      (C.c_int * 4)(*bc.as_list()))


def raise_error(e: lfo_error):
    """Map an error record to the reference's exception types."""
    msg = e.message.decode()
    if e.kind == ERR_POSITIVITY:
        raise G.PositivityError(msg, e.i, e.j, e.step, e.dt)
    if e.kind == ERR_CONFIG:
        raise G.ConfigError(msg)
    if e.kind in (ERR_DT_STATE, ERR_PRIMITIVE, ERR_TRACE, ERR_FRACTION):
        raise G.InvalidStateError(msg)
    raise G.Error(msg)


_lib_cache = {}


def _load(path: str):
    if path not in _lib_cache:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        _lib_cache[path] = C.CDLL(path)
    return _lib_cache[path]


def oracle_lib():
    lib = _load(ORACLE_SO)
    lib.lfo_create.restype = C.c_void_p
    lib.lfo_create.argtypes = [C.POINTER(lfo_grid), C.POINTER(lfo_scheme), C.POINTER(lfo_error)]
    lib.lfo_destroy.argtypes = [C.c_void_p]
    lib.lfo_compute_dt.argtypes = [C.c_void_p, P4, C.c_double, C.c_double, C.c_double, DP,
                                   C.POINTER(lfo_error)]
    lib.lfo_euler_stage.argtypes = [C.c_void_p, P4, C.c_double, P4, C.c_int64, C.POINTER(lfo_error)]
    lib.lfo_heun_step.argtypes = [C.c_void_p, P4, C.c_double, C.c_double, DP,
                                  C.POINTER(C.c_int64), DP, C.POINTER(lfo_step_out),
                                  C.POINTER(lfo_error)]
    lib.lfo_set_materials.argtypes = [C.c_void_p, C.c_int, DP, C.POINTER(lfo_error)]
    lib.lfo_heun_step_mat.argtypes = [C.c_void_p, P4, C.c_void_p, C.c_double, C.c_double, DP,
                                      C.POINTER(C.c_int64), DP, C.POINTER(lfo_step_out),
                                      C.POINTER(lfo_error)]
    lib.lfo_clamped_fraction.argtypes = [C.c_double, C.c_double, DP]
    lib.lfo_mixed_cell_gamma.restype = C.c_double
    lib.lfo_mixed_cell_gamma.argtypes = [C.c_int, DP, DP]
    lib.lfo_mass_fraction_fluxes.argtypes = [C.c_double, C.c_int, DP, DP]
    lib.lfo_fill_ghosts.argtypes = [C.POINTER(lfo_grid), C.c_int * 4, C.c_int, DP]
    lib.lfo_sweby.restype = C.c_double
    lib.lfo_sweby.argtypes = [C.c_double, C.c_double, C.c_double]
    lib.lfo_lagrangian_hll.argtypes = [DP, DP, C.c_double, C.c_double, C.c_double, C.c_double,
                                       DP, DP]
    lib.lfo_edge_flux.argtypes = [DP, DP, C.c_double, C.c_double, C.c_double, DP]
    lib.lfo_interior_totals.argtypes = [C.POINTER(lfo_grid), P4, DP]
    lib.lfo_fourier_tables.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_double, DP, DP, DP]
    lib.lfo_init_fourier.argtypes = [C.c_uint64, C.POINTER(lfo_grid), C.c_double, P4, C.c_int]
    return lib


def ref_lib():
    lib = _load(REF_SO)
    lib.lfr_create.restype = C.c_void_p
    lib.lfr_create.argtypes = [C.POINTER(lfo_grid), C.POINTER(lfo_scheme), C.c_int,
                               C.POINTER(lfo_error)]
    lib.lfr_destroy.argtypes = [C.c_void_p]
    lib.lfr_set_state.argtypes = [C.c_void_p, P4, C.c_double, C.c_int64]
    lib.lfr_get_state.argtypes = [C.c_void_p, P4, DP, C.POINTER(C.c_int64), DP]
    lib.lfr_heun_steps.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, DP, DP,
                                   C.POINTER(C.c_int), C.POINTER(lfo_error)]
    lib.lfr_compute_dt.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, DP,
                                   C.POINTER(lfo_error)]
    lib.lfr_euler_stage.argtypes = [C.c_void_p, C.c_double, C.c_int64, P4, C.POINTER(lfo_error)]
    lib.lfr_fill_ghosts.argtypes = [C.POINTER(lfo_grid), C.c_int * 4, C.c_int, DP]
    lib.lfr_sweby.restype = C.c_double
    lib.lfr_sweby.argtypes = [C.c_double, C.c_double, C.c_double]
    lib.lfr_lagrangian_hll.argtypes = [DP, DP, C.c_double, C.c_double, C.c_double, DP, DP]
    lib.lfr_edge_flux.argtypes = [DP, DP, C.c_double, C.c_double, C.c_double, DP]
    lib.lfr_omp_max_threads.restype = C.c_int
    lib.lfr_create_mat.restype = C.c_void_p
    lib.lfr_create_mat.argtypes = [C.POINTER(lfo_grid), C.POINTER(lfo_scheme), C.c_int, C.c_int,
                                   DP, C.POINTER(lfo_error)]
    lib.lfr_make_material_set.argtypes = [C.c_int, DP, C.POINTER(lfo_error)]
    lib.lfr_set_partials.argtypes = [C.c_void_p, C.c_void_p]
    lib.lfr_get_partials.argtypes = [C.c_void_p, C.c_void_p]
    lib.lfr_clamped_fraction.restype = C.c_double
    lib.lfr_clamped_fraction.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int)]
    lib.lfr_mixed_cell_gamma.restype = C.c_double
    lib.lfr_mixed_cell_gamma.argtypes = [C.c_int, DP, DP]
    lib.lfr_mass_fraction_fluxes.argtypes = [C.c_double, C.c_int, DP, DP]
    lib.lfr_interior_totals.argtypes = [C.c_void_p, DP]
    lib.lfr_edge_flux2.argtypes = [DP, DP, C.c_double, C.c_double, C.c_double, C.c_double, DP, DP,
                                   C.c_char_p, C.c_int]
    lib.lfr_diagnostics_csv.restype = C.c_int64
    lib.lfr_diagnostics_csv.argtypes = [C.c_int, DP, C.c_char_p, C.c_int64]
    lib.lfr_field_csv.restype = C.c_int64
    lib.lfr_field_csv.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_char_p, C.c_int64,
                                  C.POINTER(lfo_error)]
    return lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_diagnostics_csv(diags) -> bytes:
    """The reference's diagnostics_csv (csv.cpp:104-114) of StepDiagnostics records."""
    lib = ref_lib()
    rec = np.array([[d.step, d.time, d.dt, d.min_rho, d.min_p] for d in diags],
                   dtype=np.float64).reshape(-1)
    n = lib.lfr_diagnostics_csv(len(diags), rec.ctypes.data_as(DP), None, 0)
    buf = C.create_string_buffer(max(n, 1))
    lib.lfr_diagnostics_csv(len(diags), rec.ctypes.data_as(DP), buf, n)
    return buf.raw[:n]


class OracleSolver:
    """The C restatement behind the LagfluxSolver API (solver.hpp:78-131)."""

    def __init__(self, g: G.CartesianGrid, bc: G.BoundaryCondition, gamma: float = 1.4,
                 params: G.SchemeParams = G.SchemeParams(), materials=None):
        self.lib = oracle_lib()
        self.g, self.bc, self.gamma, self.params = g, bc, gamma, params
        err = lfo_error()
        self.h = self.lib.lfo_create(C.byref(_cgrid(g)), C.byref(_cscheme(gamma, params, bc)),
                                     C.byref(err))
        if not self.h:
            raise_error(err)
        self.materials = materials
        if materials is not None:
            gs = np.array(materials.gammas, dtype=np.float64)
            if self.lib.lfo_set_materials(self.h, len(gs), gs.ctypes.data_as(DP), C.byref(err)):
                raise_error(err)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.lfo_destroy(self.h)
            self.h = None

    def compute_dt(self, field: np.ndarray, cfl: float, time: float, limit: float) -> float:
        err, dt = lfo_error(), C.c_double()
        if self.lib.lfo_compute_dt(self.h, _ptrs(field), cfl, time, limit, C.byref(dt), C.byref(err)):
            raise_error(err)
        return dt.value

    def euler_stage(self, field: np.ndarray, dt: float, out: np.ndarray, step: int = -1) -> None:
        err = lfo_error()
        if self.lib.lfo_euler_stage(self.h, _ptrs(field), dt, _ptrs(out), step, C.byref(err)):
            raise_error(err)

    def heun_step(self, state: G.SolverState, cfl: float, limit_time: float, mat=None) -> float:
        """heun_step(state, controls, limit_time, mat) -- mat: multimat.MaterialCells."""
        err, out = lfo_error(), lfo_step_out()
        t, s = C.c_double(state.time), C.c_int64(state.step)
        acc = (C.c_double * 4)(*state.boundary_outflow)
        parts = _kptrs(mat.partial) if mat is not None else None
        rc = self.lib.lfo_heun_step_mat(self.h, _ptrs(state.field), parts, cfl, limit_time,
                                        C.byref(t), C.byref(s), C.cast(acc, DP), C.byref(out),
                                        C.byref(err))
        if rc:
            raise_error(err)
        state.time, state.step = t.value, s.value
        state.boundary_outflow = list(acc)
        state.diagnostics.append(G.StepDiagnostics(s.value, t.value, out.dt, out.min_rho, out.min_p))
        return out.dt


class RefSolver:
    """The reference's own LagfluxSolver (compiled from /root/reference sources)."""

    def __init__(self, g: G.CartesianGrid, bc: G.BoundaryCondition, gamma: float = 1.4,
                 params: G.SchemeParams = G.SchemeParams(), threads: int = 1, materials=None):
        self.lib = ref_lib()
        self.g, self.bc, self.gamma, self.params = g, bc, gamma, params
        err = lfo_error()
        gs = np.array(materials.gammas if materials is not None else [0.0], dtype=np.float64)
        self.n_mat = len(materials.gammas) if materials is not None else 0
        self.h = self.lib.lfr_create_mat(C.byref(_cgrid(g)), C.byref(_cscheme(gamma, params, bc)),
                                         threads, self.n_mat, gs.ctypes.data_as(DP), C.byref(err))
        if not self.h:
            raise_error(err)

    def field_csv(self, digest: int, time: float) -> bytes:
        """The reference's field_csv (csv.cpp:26-83) of the current state."""
        err = lfo_error()
        n = self.lib.lfr_field_csv(self.h, digest, time, None, 0, C.byref(err))
        if n < 0:
            raise_error(err)
        buf = C.create_string_buffer(n)
        self.lib.lfr_field_csv(self.h, digest, time, buf, n, C.byref(err))
        return buf.raw[:n]

    def set_partials(self, partial: np.ndarray) -> None:
        self.lib.lfr_set_partials(self.h, _kptrs(np.ascontiguousarray(partial)))

    def get_partials(self) -> np.ndarray:
        out = np.zeros((self.n_mat, self.g.nyt, self.g.nxt))
        self.lib.lfr_get_partials(self.h, _kptrs(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.lfr_destroy(self.h)
            self.h = None

    def set_state(self, field: np.ndarray, time: float = 0.0, step: int = 0) -> None:
        self.lib.lfr_set_state(self.h, _ptrs(np.ascontiguousarray(field)), time, step)

    def get_state(self) -> Tuple[np.ndarray, float, int, List[float]]:
        f = G.new_field(self.g)
        t, s = C.c_double(), C.c_int64()
        acc = (C.c_double * 4)()
        self.lib.lfr_get_state(self.h, _ptrs(f), C.byref(t), C.byref(s), C.cast(acc, DP))
        return f, t.value, s.value, list(acc)

    def interior_totals(self) -> List[float]:
        """lagflux::interior_totals of the current state (grid.cpp:122-133)."""
        t = np.zeros(4)
        self.lib.lfr_interior_totals(self.h, t.ctypes.data_as(DP))
        return [float(x) for x in t]

    def heun_steps(self, n: int, cfl: float, limit_time: float) -> np.ndarray:
        """n heun_step calls; returns (n, 5) rows {dt, time, min_rho, min_p, step}."""
        diag = np.zeros((max(n, 1), 5))
        err, done = lfo_error(), C.c_int()
        rc = self.lib.lfr_heun_steps(self.h, n, cfl, limit_time, None,
                                     diag.ctypes.data_as(DP), C.byref(done), C.byref(err))
        if rc:
            raise_error(err)
        return diag[:n]

    def compute_dt(self, cfl: float, time: float, limit: float) -> float:
        err, dt = lfo_error(), C.c_double()
        if self.lib.lfr_compute_dt(self.h, cfl, time, limit, C.byref(dt), C.byref(err)):
            raise_error(err)
        return dt.value

    def euler_stage(self, dt: float, step: int = -1) -> np.ndarray:
        out = G.new_field(self.g)
        err = lfo_error()
        if self.lib.lfr_euler_stage(self.h, dt, step, _ptrs(out), C.byref(err)):
            raise_error(err)
        return out


def oracle_run(g, bc, gamma, params, field, cfl, steps: int, limit: float = 1e300,
               stop_at_limit: bool = False):
    """Drive OracleSolver.heun_step like bench.cpp:70-75 / run.cpp:180-210.

    Returns (final field, list of StepDiagnostics, boundary_outflow)."""
    s = OracleSolver(g, bc, gamma, params)
    state = G.SolverState(field=np.array(field, copy=True))
    for _ in range(steps):
        if stop_at_limit and state.time >= limit:
            break
        s.heun_step(state, cfl, limit)
    return state.field, state.diagnostics, state.boundary_outflow


def oracle_interior_totals(g: G.CartesianGrid, field: np.ndarray) -> List[float]:
    """The oracle's restatement of interior_totals (grid.cpp:122-133)."""
    f = np.ascontiguousarray(field)
    t = np.zeros(4)
    oracle_lib().lfo_interior_totals(C.byref(_cgrid(g)), _ptrs(f), t.ctypes.data_as(DP))
    return [float(x) for x in t]


def fourier_tables_oracle(seed: int, g: G.CartesianGrid):
    lib = oracle_lib()
    tx = np.zeros(4 * 8 * 2 * g.nx)
    ty = np.zeros(4 * 8 * 2 * g.ny)
    amp = np.zeros(32)
    lib.lfo_fourier_tables(seed, g.nx, g.ny, g.x0, g.y0, g.dx, g.dy, tx.ctypes.data_as(DP),
                           ty.ctypes.data_as(DP), amp.ctypes.data_as(DP))
    return tx.reshape(4, 8, 2, g.nx), ty.reshape(4, 8, 2, g.ny), amp.reshape(4, 8)


def oracle_init_fourier(case, threads: int = 0) -> np.ndarray:
    """The seeded smooth-flow initial field (cases.initial_field for "fourier") from
    the C restatement, rows over `threads` OpenMP threads (0: all cores): the reference
    arm's 16384^2 input without the Python generator's minutes."""
    g = case.grid
    f = G.new_field(g)
    oracle_lib().lfo_init_fourier(case.seed, C.byref(_cgrid(g)), case.gamma, _ptrs(f),
                                  threads or (os.cpu_count() or 1))
    return f


# ---- multimat.cpp element functions (known-answer tests) -------------------
def ref_make_material_set(gammas):
    err = lfo_error()
    gs = np.array(list(gammas) or [0.0], dtype=np.float64)
    if ref_lib().lfr_make_material_set(len(gammas), gs.ctypes.data_as(DP), C.byref(err)):
        raise_error(err)


def ref_clamped_fraction(partial: float, rho: float):
    """(value, failed)"""
    failed = C.c_int()
    v = ref_lib().lfr_clamped_fraction(partial, rho, C.byref(failed))
    return v, bool(failed.value)


def oracle_clamped_fraction(partial: float, rho: float):
    y = C.c_double()
    rc = oracle_lib().lfo_clamped_fraction(partial, rho, C.byref(y))
    return y.value, rc != 0


def _mixed(lib_fn, gammas, fractions):
    gs = np.array(gammas, dtype=np.float64)
    fs = np.array(fractions, dtype=np.float64)
    return lib_fn(len(gs), gs.ctypes.data_as(DP), fs.ctypes.data_as(DP))


def ref_mixed_cell_gamma(gammas, fractions):
    return _mixed(ref_lib().lfr_mixed_cell_gamma, gammas, fractions)


def oracle_mixed_cell_gamma(gammas, fractions):
    return _mixed(oracle_lib().lfo_mixed_cell_gamma, gammas, fractions)


def _mff(lib_fn, mass_flux, y):
    ys = np.array(y, dtype=np.float64)
    out = np.zeros(len(ys))
    lib_fn(mass_flux, len(ys), ys.ctypes.data_as(DP), out.ctypes.data_as(DP))
    return out


def ref_mass_fraction_fluxes(mass_flux, y):
    return _mff(ref_lib().lfr_mass_fraction_fluxes, mass_flux, y)


def oracle_mass_fraction_fluxes(mass_flux, y):
    return _mff(oracle_lib().lfo_mass_fraction_fluxes, mass_flux, y)
