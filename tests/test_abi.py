"""CPU: the C-ABI library loads and exports exactly what include/lagflux_b200.h declares.

No compute calls are made (this container has no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1607_08710_b200 import native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(N.HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lf_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_reference_replacements():
    syms = declared_symbols()
    for name in ["lf_create", "lf_destroy", "lf_upload", "lf_download", "lf_compute_dt",
                 "lf_euler_stage", "lf_heun_step", "lf_last_error", "lf_create_dist",
                 "lf_advance"]:
        assert name in syms


def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (lf_\w+)", out))
    assert exported == set(declared_symbols())


def test_python_binding_covers_the_header():
    bound = {name for name, _, _ in N.SIGNATURES}
    assert bound == set(declared_symbols())
    assert N.lib().lf_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    """sizeof/offsetof from the C compiler == the ctypes mirrors."""
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "lagflux_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(lf_desc), sizeof(lf_error),'
                   ' sizeof(lf_step_out), offsetof(lf_desc, bc), offsetof(lf_error, message));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(N.lf_desc), ctypes.sizeof(N.lf_error), ctypes.sizeof(N.lf_step_out),
                   N.lf_desc.bc.offset, N.lf_error.message.offset]


def test_sm100a_cubin_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_partial_pointer_marshalling():
    """n_mat partial-density arrays -> double*[n] (host only)."""
    import ctypes as C
    import numpy as np
    from paper_1607_08710_b200 import native as N
    p = np.arange(3 * 4 * 5, dtype=np.float64).reshape(3, 4, 5)
    ptrs = N.partial_ptrs(p)
    assert len(ptrs) == 3
    for k in range(3):
        assert C.cast(ptrs[k], C.c_void_p).value == p[k].ctypes.data
        assert ptrs[k][7] == p[k].ravel()[7]


def test_biased_field_pointers_address_the_local_rows():
    """A distributed rank's host buffer holds total rows y0 .. y0 + rows + 3 only; the
    library addresses row y0 + 2 + r of the global layout through biased pointers
    (lf_upload / lf_download of a distributed handle, include/lagflux_b200.h)."""
    import numpy as np
    y0, rows, nxt = 37, 5, 11
    local = np.zeros((4, rows + 4, nxt))
    p = N.biased_field_ptrs(local, y0)
    for c in range(4):
        addr = ctypes.cast(p[c], ctypes.c_void_p).value
        # global interior row r of this slab -> local buffer row 2 + r
        for r in (0, rows - 1):
            assert addr + ((y0 + 2 + r) * nxt + 2) * 8 == local[c, 2 + r, 2:].ctypes.data
    assert N.biased_field_ptrs(local, 0)[1][0] == N.field_ptrs(local)[1][0]


def test_cpp_adapter_headers_compile_against_the_reference_headers(tmp_path):
    """include/lagflux_b200.hpp and include/lagflux_b200_run.hpp are compiled inside the
    reference's build: they must parse against its headers (only where the reference
    tree is present: this container, not the GPU box)."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference tree absent")
    src = tmp_path / "use.cpp"
    src.write_text('#include "lagflux_b200_run.hpp"\n'
                   "lagflux::HydroRun go(const lagflux::CaseConfig& c) {\n"
                   "  return lagflux::b200::run_hydro_case(c, false);\n}\n")
    subprocess.run(["/usr/bin/g++", "-std=gnu++20", "-fsyntax-only", "-Wall", "-Wextra", "-I", ref_inc,
                    "-I", os.path.join(ROOT, "include"), str(src)], check=True)
