"""CPU: the bench's host-side logic (no GPU): the reference arm's workload sizing,
the fp64-roofline inputs and the JSON contract pieces that do not need a device."""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_reference_arm_runs_the_full_config4_grid_when_it_fits(bench, monkeypatch):
    from paper_1607_08710_b200 import cases as CS
    monkeypatch.setattr(bench, "host_ram_bytes", lambda: 211e9)   # the GPU box
    case, what = bench.reference_case(CS, 1, "weak")
    assert (case.grid.nx, case.grid.ny) == (16384, 16384) and "full grid" in what
    assert case.grid.dx == case.grid.dy and case.seed == CS.SMOOTH_SEED
    # strong scaling (config 5): 32768 columns on as many rows as fit the host
    case, what = bench.reference_case(CS, 8, "strong")
    assert case.grid.nx == 32768 and case.grid.ny == 16384 and "strip" in what
    assert case.grid.dx == case.grid.dy


def test_reference_arm_shrinks_to_a_strip_on_a_small_host(bench, monkeypatch):
    from paper_1607_08710_b200 import cases as CS
    monkeypatch.setattr(bench, "host_ram_bytes", lambda: 62e9)    # this container
    case, what = bench.reference_case(CS, 1, "weak")
    assert case.grid.nx == 16384 and case.grid.ny == 8192 and "strip" in what
    assert 300.0 * case.grid.nx * case.grid.ny <= 0.8 * 62e9


def test_fp64_ops_profile_is_well_formed(bench):
    p = os.path.join(ROOT, "profiles", "fp64_ops.json")
    if not os.path.exists(p):
        pytest.skip("no fp64 op-count capture committed yet")
    d = json.load(open(p))
    for key, v in d.items():
        path, math = key.split("/")
        assert path in ("fused", "twopass") and math in ("exact", "contract")
        assert 300 < v["fp64_ops_per_cell_update"] < 2000
        assert bench.ncu_fp64_ops(key) == v


def test_cpu_model_and_omp_binding(bench):
    assert isinstance(bench.cpu_model(), str) and bench.cpu_model()
    assert set(bench.omp_binding()) == {"OMP_PLACES", "OMP_PROC_BIND", "OMP_NUM_THREADS"}
