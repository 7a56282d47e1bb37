"""LagfluxSolver: the reference's solver interface over the CUDA C ABI.

Mirrors lagflux::LagfluxSolver (/root/reference/proj/include/lagflux/solver.hpp:78-131)
-- same method names, argument meaning and exception types -- so the parity
tests read like the reference's own (proj/tests/test_solver.cpp).  The field
lives on the GPU between steps: a SolverState is uploaded on its first step
and ``sync_to_host(state)`` copies it back (dumps, end of run), the one-line
addition a run.cpp-style driver needs.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import grid as G
from . import native as N


def _raise(e: N.lf_error):
    msg = e.message.decode(errors="replace")
    if e.kind == N.LF_ERR_POSITIVITY:
        raise G.PositivityError(msg, e.i, e.j, e.step, e.dt)
    if e.kind == N.LF_ERR_CONFIG:
        raise G.ConfigError(msg)
    if e.kind in (N.LF_ERR_DT_STATE, N.LF_ERR_PRIMITIVE, N.LF_ERR_TRACE, N.LF_ERR_FRACTION):
        raise G.InvalidStateError(msg)
    if e.kind == N.LF_ERR_DT_NONPOS:
        raise G.Error(msg)
    if e.kind == N.LF_ERR_ARGUMENT:
        raise ValueError(msg)
    raise G.DeviceError(msg or f"lagflux_b200 error kind {e.kind}")


def make_desc(g: G.CartesianGrid, bc: G.BoundaryCondition, gamma: float,
              params: G.SchemeParams) -> N.lf_desc:
    return N.lf_desc(g.dim, g.nx, g.ny, g.dx, g.dy, g.x0, g.y0, gamma, params.beta,
                     params.spatial_order, params.time_order, (C.c_int * 4)(*bc.as_list()))


class LagfluxSolver:
    """CUDA-backed drop-in for lagflux::LagfluxSolver.

    devices: one entry per y-slab driven from this process (repeats allowed).
    dist:    (rank, nranks, device, nccl_id_bytes) for one-process-per-GPU slabs.
    path:    "auto" | "twopass" | "fused" | "staged" | "small" (Heun step
             implementation; all produce identical results).
    materials: a multimat.MaterialSet (the constructor's `const MaterialSet*`,
             solver.cpp:61-88); heun_step then takes the MaterialCells."""

    def __init__(self, g: G.CartesianGrid, bc: G.BoundaryCondition, gamma: float = 1.4,
                 params: G.SchemeParams = G.SchemeParams(), threads: int = 1,
                 materials=None, devices: Sequence[int] = (0,), path: str = "auto", dist=None,
                 math: str = "exact"):
        # constructor checks of solver.cpp:66-69
        if g.nx < 1 or g.ny < 1:
            raise G.ConfigError("grid has no interior cells")
        if g.gx < 2 or (g.dim == 2 and g.gy < 2):
            raise G.ConfigError("MUSCL stencils need at least two ghost layers")
        G.validate_boundary(bc, g.dim)
        self._lib = N.lib()
        self._grid, self.bc, self.gamma, self.params = g, bc, gamma, params
        self._threads = max(1, threads)
        self._desc = make_desc(g, bc, gamma, params)
        h = C.c_void_p()
        if dist is None:
            devs = (C.c_int * len(devices))(*devices)
            rc = self._lib.lf_create(C.byref(self._desc), devs, len(devices), C.byref(h))
        else:
            rank, nranks, device, nccl_id = dist
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            rc = self._lib.lf_create_dist(C.byref(self._desc), device, rank, nranks, idbuf,
                                          C.byref(h))
        self._h = h
        if rc:
            err = self._error()
            self.close()
            _raise(err)
        self.set_path(path)
        self.set_math(math)
        self._resident = None  # SolverState whose field is on the device
        # host fields hold only this rank's rows (distributed handles): see
        # local_field_shape(); the ABI takes pointers biased by -y0 * ld
        self.local_host = False
        self._resident_mat = None  # MaterialCells whose partials are on the device
        self.materials = materials
        if materials is not None:
            gs = (C.c_double * materials.count())(*materials.gammas)
            self._check(self._lib.lf_set_materials(self._h, materials.count(), gs))

    # ------------------------------------------------------------ plumbing
    def _error(self) -> N.lf_error:
        e = N.lf_error()
        if self._h:
            self._lib.lf_last_error(self._h, C.byref(e))
        return e

    def _check(self, rc: int):
        if rc:
            _raise(self._error())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lf_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def grid(self) -> G.CartesianGrid:
        return self._grid

    def threads(self) -> int:
        return self._threads

    @property
    def handle(self):
        return self._h

    def set_path(self, path: str):
        code = {"auto": N.LF_PATH_AUTO, "fused": N.LF_PATH_FUSED, "staged": N.LF_PATH_STAGED,
                "twopass": N.LF_PATH_TWOPASS, "small": N.LF_PATH_SMALL}[path]
        self._check(self._lib.lf_set_path(self._h, code))

    def set_math(self, math: str):
        """'exact' (default): bit-identical to the reference.  'contract': the two-pass
        kernels with FMA contraction and reciprocal products, within the north star's
        tolerance (relative L1 <= 1e-10 per field, dt to 1e-12), not bit-identical."""
        code = {"exact": N.LF_MATH_EXACT, "contract": N.LF_MATH_CONTRACT}[math]
        self._check(self._lib.lf_set_math(self._h, code))
        self.math = math

    def resolved_path(self) -> str:
        """The path the next step takes ('twopass', 'fused', 'staged' or 'small')."""
        p = C.c_int()
        self._check(self._lib.lf_resolved_path(self._h, C.byref(p)))
        return {N.LF_PATH_TWOPASS: "twopass", N.LF_PATH_FUSED: "fused",
                N.LF_PATH_STAGED: "staged", N.LF_PATH_SMALL: "small"}[p.value]

    def set_stream(self, stream_ptr: Optional[int]):
        self._check(self._lib.lf_set_stream(self._h, stream_ptr))

    def local_rows(self):
        r0, n = C.c_int(), C.c_int()
        self._check(self._lib.lf_local_rows(self._h, C.byref(r0), C.byref(n)))
        return r0.value, n.value

    def local_field_shape(self):
        """(4, rows + 2 gy, nxt): a host field holding this rank's slab rows and
        their two ghost rows each side (total rows y0 .. y0 + rows + 2 gy - 1)."""
        _, n = self.local_rows()
        return (4, n + 2 * self._grid.gy, self._grid.nxt)

    def _ptrs(self, field):
        if not self.local_host:
            g = self._grid
            if field.shape != (4, g.nyt, g.nxt):
                raise ValueError(f"field shape {field.shape} is not the grid's ghosted layout "
                                 f"{(4, g.nyt, g.nxt)}")
            return N.field_ptrs(field)
        assert field.shape == self.local_field_shape(), (field.shape, self.local_field_shape())
        return N.biased_field_ptrs(field, self.local_rows()[0])

    def device_bytes(self) -> int:
        b = C.c_int64()
        self._check(self._lib.lf_device_bytes(self._h, C.byref(b)))
        return b.value

    # ------------------------------------------------------------ state transfer
    def upload(self, field: np.ndarray):
        self._evict(field)
        self._check(self._lib.lf_upload(self._h, self._ptrs(field), self._grid.nxt))
        self._resident = None

    def _evict(self, field: np.ndarray):
        """The device copy of the resident state is about to be replaced by `field`
        (compute_dt / euler_stage of another field, or another state): it is the only
        current copy, so save it into the resident state's host field first; the
        next heun_step of that state re-attaches from there.  A device-only state
        (host field of another shape, e.g. after init_fourier for a benchmark) cannot
        be saved: it is dropped, and stepping it again fails on the shape check."""
        r = self._resident
        if r is None or r.field is field:
            return
        try:
            self._ptrs(r.field)
        except (ValueError, AssertionError):
            self._resident = None
            return
        self.download(r.field)
        self._resident = None

    def download(self, field: np.ndarray, fill_ghosts: bool = False):
        if fill_ghosts and self.local_host:
            raise ValueError("fill_ghosts needs the whole grid on the host")
        self._check(self._lib.lf_download(self._h, self._ptrs(field), self._grid.nxt,
                                          1 if fill_ghosts else 0))

    def download_ghosted(self, field: np.ndarray):
        """The device kernels' own ghost fill of the current state, two layers
        (corners included), into `field` (test hook: lf_download_ghosted)."""
        self._check(self._lib.lf_download_ghosted(self._h, self._ptrs(field), self._grid.nxt))

    def attach(self, state: G.SolverState):
        """Make `state` the device-resident state (uploads its field)."""
        self.upload(state.field)
        self._resident = state

    def sync_to_host(self, state: G.SolverState, fill_ghosts: bool = False, mat=None):
        """Copy the device-resident state (and the MaterialCells' interior) back."""
        if self._resident is not state:
            raise G.Error("state is not resident on this solver")
        self.download(state.field, fill_ghosts)
        if mat is not None:
            if self._resident_mat is not mat:
                raise G.Error("material cells are not resident on this solver")
            self._check(self._lib.lf_download_partials(self._h, N.partial_ptrs(mat.partial),
                                                       self._grid.nxt))

    def _attach_mat(self, mat):
        if self.materials is None:
            return
        if mat is None:
            raise G.ConfigError("multimaterial step needs material storage")
        if self._resident_mat is not mat:
            self._check(self._lib.lf_upload_partials(self._h, N.partial_ptrs(mat.partial),
                                                     self._grid.nxt))
            self._resident_mat = mat

    def write_field_csv(self, path: str, digest: int, time: float, threads: int = 0):
        """run.cpp's dump: field_csv (csv.cpp:26-83) of the resident state (and its
        material fractions) to `path`, formatted on `threads` host threads."""
        self._check(self._lib.lf_write_field_csv(self._h, path.encode(), digest, time, threads))

    def write_field_csv_async(self, path: str, digest: int, time: float, threads: int = 0):
        """write_field_csv of the current resident state without waiting: the columns
        are snapshotted on the device in stream order and a host thread copies,
        formats and writes them while stepping continues.  The dump's own errors
        (fraction, I/O) come from wait_dumps()."""
        self._check(self._lib.lf_write_field_csv_async(self._h, path.encode(), digest, time,
                                                       threads))

    def wait_dumps(self):
        """Join every pending write_field_csv_async of this solver (first error raised)."""
        self._check(self._lib.lf_wait_dumps(self._h))

    def init_regions(self, state: G.SolverState, regions, mat=None):
        """Device-side initialize_hydro for region cases (cases.Region list); with a
        material set, `mat` becomes the resident MaterialCells (download with
        sync_to_host(state, mat=mat))."""
        flat = []
        for r in regions:
            flat += [r.x_min, r.x_max, r.y_min, r.y_max, r.rho, r.u, r.v, r.p, float(r.material)]
        arr = (C.c_double * len(flat))(*flat)
        self._check(self._lib.lf_init_regions(self._h, arr, len(regions)))
        self._resident = state
        if self.materials is not None:
            self._resident_mat = mat

    def init_fourier(self, state: G.SolverState, seed: int):
        """Device-side seeded smooth-flow initial state (cases.fourier_*)."""
        self._check(self._lib.lf_init_fourier(self._h, seed))
        self._resident = state

    # ------------------------------------------------------------ the reference API
    def compute_dt(self, field: np.ndarray, controls: G.TimeControls, time: float,
                   limit_time: float) -> float:
        """LagfluxSolver::compute_dt (solver.cpp:434-480) of a host field."""
        self.upload(field)
        dt = C.c_double()
        self._check(self._lib.lf_compute_dt(self._h, controls.cfl, time, limit_time, C.byref(dt)))
        return dt.value

    def euler_stage(self, field_in: np.ndarray, dt: float, field_out: np.ndarray,
                    step: int = -1) -> None:
        """LagfluxSolver::euler_stage (solver.cpp:482-487): out's interior receives the stage."""
        self.upload(field_in)
        self._check(self._lib.lf_euler_stage(self._h, dt, step))
        self.download(field_out)

    def heun_step(self, state: G.SolverState, controls: G.TimeControls,
                  limit_time: float, mat=None) -> float:
        """LagfluxSolver::heun_step (solver.cpp:489-546) on the device-resident state;
        with a material set, `mat` (multimat.MaterialCells) is advected too and stays
        resident like the field (sync_to_host(state, mat=mat) copies it back)."""
        if self._resident is not state:
            self.attach(state)
        self._attach_mat(mat)
        out = N.lf_step_out()
        acc = (C.c_double * 4)(*state.boundary_outflow)
        rc = self._lib.lf_heun_step(self._h, controls.cfl, state.time, limit_time, state.step,
                                    C.cast(acc, N.DP), C.byref(out))
        if rc:
            # on a corrector PositivityError the device state already holds the
            # corrector output, as state.field does in the reference
            _raise(self._error())
        state.boundary_outflow = list(acc)
        state.time, state.step = out.time, out.step
        state.diagnostics.append(G.StepDiagnostics(out.step, out.time, out.dt, out.min_rho,
                                                   out.min_p))
        return out.dt

    def advance(self, state: G.SolverState, controls: G.TimeControls, nsteps: int,
                mat=None) -> int:
        """Up to nsteps heun_steps while time < t_final, with dt on the device (run.cpp:180-210)."""
        if self._resident is not state:
            self.attach(state)
        self._attach_mat(mat)
        n = int(min(nsteps, max(0, controls.max_steps - state.step)))
        done = 0
        # records come back in bounded chunks (nsteps may be far more than the
        # steps to t_final)
        rec = (N.lf_step_out * min(max(n, 1), 4096))()
        while done < n:
            chunk = min(n - done, len(rec))
            t, s = C.c_double(state.time), C.c_int64(state.step)
            acc = (C.c_double * 4)(*state.boundary_outflow)
            taken = C.c_int()
            rc = self._lib.lf_advance(self._h, chunk, controls.cfl, controls.t_final, C.byref(t),
                                      C.byref(s), C.cast(acc, N.DP), rec, C.byref(taken))
            for k in range(taken.value):
                o = rec[k]
                state.diagnostics.append(G.StepDiagnostics(o.step, o.time, o.dt, o.min_rho, o.min_p))
            state.time, state.step = t.value, s.value
            state.boundary_outflow = list(acc)
            done += taken.value
            if rc:
                _raise(self._error())
            if taken.value < chunk:
                break
        return done

    def time_steps(self, nsteps: int, cfl: float):
        """Device-timed steps: (summed kernel ms, loop ms, kernel launches)."""
        k, s, n = C.c_double(), C.c_double(), C.c_int()
        self._check(self._lib.lf_time_steps(self._h, nsteps, cfl, C.byref(k), C.byref(s),
                                            C.byref(n)))
        return k.value, s.value, n.value

    def launch_count(self) -> int:
        n = C.c_int64()
        self._check(self._lib.lf_launch_count(self._h, C.byref(n)))
        return n.value

    def interior_totals(self) -> List[float]:
        """interior_totals(grid, state.field) (grid.cpp:122-133) of the device-resident
        state, bit-equal to the reference's ordered sums."""
        t = (C.c_double * 4)()
        self._check(self._lib.lf_interior_totals(self._h, C.cast(t, C.POINTER(C.c_double))))
        return list(t)

    def max_rate(self) -> float:
        r = C.c_double()
        self._check(self._lib.lf_max_rate(self._h, C.byref(r)))
        return r.value


def edge_flux(w_minus, w_plus, normals, gamma_minus, gamma_plus=None, device: int = 0):
    """The reference's free edge_flux (solver.cpp:45-53) for a batch of faces on the
    device: w_* (n, 4) primitive traces {rho, u, v, p}, normals (n, 2), one gamma
    per side (scalars or (n,) arrays).  Returns (flux (n, 4), contact (n, 2) =
    lagrangian_hll's {p*, u*}); a non-physical trace raises InvalidStateError with
    sound_speed's message for the smallest such face."""
    wm = np.ascontiguousarray(w_minus, dtype=np.float64).reshape(-1, 4)
    wp = np.ascontiguousarray(w_plus, dtype=np.float64).reshape(-1, 4)
    n = wm.shape[0]
    nr = np.ascontiguousarray(np.broadcast_to(np.asarray(normals, dtype=np.float64), (n, 2)))
    gm = np.ascontiguousarray(np.broadcast_to(np.asarray(gamma_minus, dtype=np.float64), (n,)))
    gp = np.ascontiguousarray(np.broadcast_to(np.asarray(
        gamma_minus if gamma_plus is None else gamma_plus, dtype=np.float64), (n,)))
    flux = np.empty((n, 4))
    contact = np.empty((n, 2))
    err = N.lf_error()
    p = lambda a: a.ctypes.data_as(N.DP)  # noqa: E731
    rc = N.lib().lf_edge_flux(n, p(wm), p(wp), p(nr), p(gm), p(gp), p(flux), p(contact), device,
                              C.byref(err))
    if rc:
        _raise(err)
    return flux, contact


def compute_dt(g: G.CartesianGrid, field: np.ndarray, gamma: float, controls: G.TimeControls,
               time: float, limit_time: float, device: int = 0) -> float:
    """The free compute_dt (solver.cpp:55-59): default boundaries and scheme
    parameters, evaluated on the device."""
    s = LagfluxSolver(g, G.BoundaryCondition(), gamma, G.SchemeParams(), devices=(device,))
    try:
        return s.compute_dt(field, controls, time, limit_time)
    finally:
        s.close()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = N.lib().lf_nccl_unique_id(buf)
    if rc:
        raise G.DeviceError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return buf.raw


def run_case(case, solver: Optional[LagfluxSolver] = None, field: Optional[np.ndarray] = None,
             batch: int = 64, **kw) -> G.SolverState:
    """run_hydro_case's step loop (run.cpp:178-210) without dumps: to t_final or max_steps."""
    from . import cases as CS
    s = solver or LagfluxSolver(case.grid, case.bc, case.gamma, case.params, **kw)
    state = G.SolverState(field=CS.initial_field(case) if field is None else field)
    controls = G.TimeControls(case.cfl, case.t_final, case.max_steps)
    s.attach(state)
    while state.time < case.t_final and state.step < case.max_steps:
        if s.advance(state, controls, batch) == 0:
            break
    s.sync_to_host(state)
    return state
