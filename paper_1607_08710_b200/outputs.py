"""Host-side output formatting around the dumps (csv.cpp).

field_csv itself is on the device (LagfluxSolver.write_field_csv /
write_field_csv_async, lf_write_field_csv[_async]); the step diagnostics are a few
numbers per step that lf_advance already returns to the host, so their file is
formatted here, with the reference's spelling.
"""
from typing import Iterable

from . import grid as G


def format_g17(v: float) -> str:
    """format_g17 (csv.cpp:8-12): snprintf "%.17g"."""
    return "%.17g" % v


def diagnostics_csv(diags: Iterable[G.StepDiagnostics]) -> str:
    """diagnostics_csv (csv.cpp:104-114): "step,time,dt,min_rho,min_p" then one row per
    StepDiagnostics record (step as std::to_string, the rest %.17g)."""
    out = ["step,time,dt,min_rho,min_p\n"]
    for d in diags:
        out.append("%d,%s,%s,%s,%s\n" % (int(d.step), format_g17(d.time), format_g17(d.dt),
                                         format_g17(d.min_rho), format_g17(d.min_p)))
    return "".join(out)


def write_diagnostics_csv(path: str, diags: Iterable[G.StepDiagnostics]) -> None:
    """run.cpp:170-174 flush_diagnostics: write_text_file(path, diagnostics_csv(...))."""
    with open(path, "wb") as f:
        f.write(diagnostics_csv(diags).encode())
