"""ctypes binding of the C ABI in include/lagflux_b200.h (liblagflux_b200.so).

The product's only compute path: if the shared library is missing this module
raises on import -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblagflux_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "lagflux_b200.h")

LF_OK, LF_ERR_CONFIG, LF_ERR_DT_STATE, LF_ERR_DT_NONPOS = 0, 1, 2, 3
LF_ERR_PRIMITIVE, LF_ERR_TRACE, LF_ERR_POSITIVITY, LF_ERR_DEVICE, LF_ERR_ARGUMENT = 4, 5, 6, 7, 8
LF_ERR_FRACTION = 9
LF_PATH_AUTO, LF_PATH_FUSED, LF_PATH_STAGED, LF_PATH_TWOPASS, LF_PATH_SMALL = 0, 1, 2, 3, 4
LF_MATH_EXACT, LF_MATH_CONTRACT = 0, 1


class lf_desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("dx", C.c_double),
                ("dy", C.c_double), ("x0", C.c_double), ("y0", C.c_double),
                ("gamma", C.c_double), ("beta", C.c_double), ("spatial_order", C.c_int),
                ("time_order", C.c_int), ("bc", C.c_int * 4)]


class lf_error(C.Structure):
    _fields_ = [("kind", C.c_int), ("axis", C.c_int), ("i", C.c_int64), ("j", C.c_int64),
                ("step", C.c_int64), ("dt", C.c_double), ("value", C.c_double),
                ("value2", C.c_double), ("message", C.c_char * 320)]


class lf_step_out(C.Structure):
    _fields_ = [("dt", C.c_double), ("hits_limit", C.c_int), ("time", C.c_double),
                ("step", C.c_int64), ("min_rho", C.c_double), ("min_p", C.c_double)]


DP = C.POINTER(C.c_double)
P4 = DP * 4
H = C.c_void_p

# (name, restype, argtypes) -- the full exported surface of lagflux_b200.h
SIGNATURES = [
    ("lf_abi_version", C.c_int, []),
    ("lf_create", C.c_int, [C.POINTER(lf_desc), C.POINTER(C.c_int), C.c_int, C.POINTER(H)]),
    ("lf_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("lf_create_dist", C.c_int, [C.POINTER(lf_desc), C.c_int, C.c_int, C.c_int, C.c_void_p,
                                 C.POINTER(H)]),
    ("lf_destroy", None, [H]),
    ("lf_local_rows", C.c_int, [H, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("lf_upload", C.c_int, [H, P4, C.c_int64]),
    ("lf_download", C.c_int, [H, P4, C.c_int64, C.c_int]),
    ("lf_set_materials", C.c_int, [H, C.c_int, C.POINTER(C.c_double)]),
    ("lf_write_field_csv", C.c_int, [H, C.c_char_p, C.c_uint64, C.c_double, C.c_int]),
    ("lf_write_field_csv_async", C.c_int, [H, C.c_char_p, C.c_uint64, C.c_double, C.c_int]),
    ("lf_wait_dumps", C.c_int, [H]),
    ("lf_init_regions", C.c_int, [H, C.POINTER(C.c_double), C.c_int]),
    ("lf_upload_partials", C.c_int, [H, C.c_void_p, C.c_int64]),
    ("lf_download_partials", C.c_int, [H, C.c_void_p, C.c_int64]),
    ("lf_init_fourier", C.c_int, [H, C.c_uint64]),
    ("lf_compute_dt", C.c_int, [H, C.c_double, C.c_double, C.c_double, DP]),
    ("lf_euler_stage", C.c_int, [H, C.c_double, C.c_int64]),
    ("lf_heun_step", C.c_int, [H, C.c_double, C.c_double, C.c_double, C.c_int64, DP,
                               C.POINTER(lf_step_out)]),
    ("lf_advance", C.c_int, [H, C.c_int, C.c_double, C.c_double, DP, C.POINTER(C.c_int64), DP,
                             C.POINTER(lf_step_out), C.POINTER(C.c_int)]),
    ("lf_last_error", C.c_int, [H, C.POINTER(lf_error)]),
    ("lf_set_stream", C.c_int, [H, C.c_void_p]),
    ("lf_set_path", C.c_int, [H, C.c_int]),
    ("lf_set_math", C.c_int, [H, C.c_int]),
    ("lf_resolved_path", C.c_int, [H, C.POINTER(C.c_int)]),
    ("lf_time_steps", C.c_int, [H, C.c_int, C.c_double, DP, DP, C.POINTER(C.c_int)]),
    ("lf_device_bytes", C.c_int, [H, C.POINTER(C.c_int64)]),
    ("lf_max_rate", C.c_int, [H, DP]),
    ("lf_interior_totals", C.c_int, [H, DP]),
    ("lf_edge_flux", C.c_int, [C.c_int64, DP, DP, DP, DP, DP, DP, DP, C.c_int, C.POINTER(lf_error)]),
    ("lf_download_ghosted", C.c_int, [H, P4, C.c_int64]),
    ("lf_launch_count", C.c_int, [H, C.POINTER(C.c_int64)]),
    ("lf_slab_partition", C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("lf_selftest_fastmath", C.c_int, [C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]),
    ("lf_selftest_box", C.c_int, [C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]),
    ("lf_selftest_epilogue", C.c_int, [C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]),
    ("lf_fp64_peak", C.c_int, [C.c_int, C.c_double, C.c_double, DP]),
]

_lib = None


def lib():
    """Load liblagflux_b200.so (built by __graft_entry__.build() / csrc/Makefile)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built: the CUDA path is the only implementation "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        l = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        if l.lf_abi_version() != 1:
            raise ImportError("liblagflux_b200.so ABI version mismatch")
        _lib = l
    return _lib


def partial_ptrs(partial):
    """double*[n] of the n contiguous (nyt, nxt) arrays of a partial-density stack."""
    assert partial.dtype == np.float64 and partial.flags.c_contiguous and partial.ndim == 3
    DPT = C.POINTER(C.c_double)
    return (DPT * partial.shape[0])(*[partial[k].ctypes.data_as(DPT) for k in range(partial.shape[0])])


def biased_field_ptrs(field, row_bias: int):
    """P4 of a field that holds only the total rows row_bias .. row_bias + nyt_local - 1
    of the global ghosted layout: each pointer is biased by -row_bias * ld so the
    library's global row addressing (lf_upload / lf_download of a distributed
    handle) lands inside the local buffer."""
    base = field_ptrs(field)
    if not row_bias:
        return base
    off = row_bias * field.shape[2] * 8
    return P4(*[C.cast(C.c_void_p(C.cast(base[c], C.c_void_p).value - off), DP) for c in range(4)])


def field_ptrs(field):
    """P4 of the four contiguous component arrays of a (4, nyt, nxt) float64 field."""
    assert field.dtype.name == "float64" and field.flags.c_contiguous and field.shape[0] == 4
    return P4(*[field[c].ctypes.data_as(DP) for c in range(4)])
