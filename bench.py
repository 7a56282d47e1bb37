"""Benchmark: cell-updates/s of the full second-order Lagrange-flux step on B200.

Workload (BASELINE.json configs[3]/[4]): the seeded smooth-perturbation flow,
periodic, fp64, 16384 x 16384 cells per GPU -- config 4 at N = 1 and the weak
scaling of config 5 (16384 x 16384 N on [0,1] x [0,N], one y-slab per rank) at
N > 1.  A step is one LagfluxSolver::heun_step (both stages + dt, solver.cpp:489-546);
one cell-update advances one interior cell by one step (bench.cpp:104,107).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong]

ours:       value = cells x K / device time of K device-resident steps (CUDA events on
            the launching stream, barrier + synchronize around, max over ranks).
            e2e   = the same through the public API with HOST buffers: upload of the
            initial state from pinned memory, K steps, download of the final state,
            all inside the timed region.
            --scaling strong: config 5's 32768^2 grid split over the N ranks (total
            work fixed), with a final-state digest checked against one handle
            holding the whole grid (the reference's scaling_sweep determinism check,
            bench.cpp:96-99,113-135).
reference:  the reference's own LagfluxSolver (oracle/_ref, compiled from its sources)
            on all host cores on the same 16384^2 config-4 grid, with the same
            --steps / --warmup, timed like bench.cpp:70-76.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BYTES_PER_CELL_UPDATE = 160  # read U^n, write U*, read U^n + U*, write U^{n+1}
FALLBACK_HBM_GBS = 6650.0    # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
METRIC = "cell-updates/sec (fp64, full 2nd-order step)"
UNIT = "cell-updates/s"
CPU_SAMPLE_ROWS = 4096       # cpu_baseline leg of our arm: 16384 x 4096 strip of config 4


# stdout carries exactly the one JSON line: everything else any library prints there
# (NCCL's version banner, say) goes to stderr (main() moves fd 1 onto fd 2)
_JSON_FD = None


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    sys.stdout.flush()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(path):
    """DRAM bytes per step of the path's dominant kernel(s) from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[path]
    except Exception:
        return None


def ncu_compute_bound(path, math="exact"):
    """The path's kernels' real bound from the committed ncu --set full capture of the
    current build (profiles/r02_ncu_16k.json; the two-pass kernels from round 1's
    profiles/r01_ncu_16k.json): fp64-pipe and issue utilisation per kernel."""
    for fn, key in (("r02_ncu_16k.json", f"{path}/{math}"), ("r01_ncu_16k.json", path)):
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                ks = json.load(f)[key]["kernels"]
        except Exception:
            continue
        return {"bound": "fp64 pipe / issue latency (not HBM)",
                "kernels": {k["kernel"].split("(")[0].split("::")[-1]:
                            {"fp64_pipe_pct": round(k["fp64_pipe_pct"], 1),
                             "issue_active_pct": round(k["issue_active_pct"], 1),
                             "top_stall": max(k["top_stalls_pct"], key=k["top_stalls_pct"].get)}
                            for k in ks},
                "source": f"profiles/{fn} (ncu --set full, 16384^2)"}
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows
                                                         if r[2].replace(".", "").isdigit())}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # LF_BENCH_DIST=1 with one process: the distributed machinery (process group, a
    # one-rank distributed handle on the real NCCL) on a one-GPU box -- a check of
    # the N > 1 code path where only one GPU is available
    multi = world > 1 or os.environ.get("LF_BENCH_DIST") == "1"
    if multi:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return torch, dist, world, rank, local, multi


def cpu_sample_case(cases, rows=CPU_SAMPLE_ROWS, n=16384):
    """A bounded strip of the config-4 workload: 16384 x rows cells, same dx = dy, periodic."""
    return cases.smooth(n, 1, ny=rows, y_extent=rows / n)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_ram_bytes():
    try:
        import psutil
        return psutil.virtual_memory().total
    except Exception:
        return 0


def omp_binding():
    return {k: os.environ.get(k) for k in ("OMP_PLACES", "OMP_PROC_BIND", "OMP_NUM_THREADS")}


def time_reference_cpu(case, steps, warmup, threads):
    """The reference's LagfluxSolver::heun_step on host cores (bench.cpp:70-76 timing:
    steady_clock around the step loop after the warm-up steps).  The initial state
    comes from the oracle's C generator (bit-identical to cases.initial_field)."""
    from oracle import oracle as O
    f0 = O.oracle_init_fourier(case, threads)
    r = O.RefSolver(case.grid, case.bc, case.gamma, case.params, threads=threads)
    r.set_state(f0)
    del f0
    if warmup:
        r.heun_steps(warmup, case.cfl, case.t_final)
    t0 = time.perf_counter()
    r.heun_steps(steps, case.cfl, case.t_final)
    wall = time.perf_counter() - t0
    del r
    return case.cells * steps / wall, wall


def reference_case(cases, world, scaling):
    """The grid the reference arm times: our arm's N = 1 workload (config 4, 16384^2)
    when it fits the host (the reference holds 288 B/cell, 77 GB), else the largest
    strip of the same generator that does; for --scaling strong the config-5 columns
    (32768) on as many rows as fit (the whole 32768^2 grid needs 309 GB)."""
    ram = host_ram_bytes()
    n = 32768 if scaling == "strong" else 16384
    rows = n
    while rows > 512 and 300.0 * n * rows > 0.8 * ram:
        rows //= 2
    case = cases.smooth(n, 1, ny=rows, y_extent=rows / n)
    if rows == n:
        what = f"config{5 if n == 32768 else 4}-smooth {n}x{n} periodic (the full grid)"
    else:
        what = (f"config{5 if n == 32768 else 4} generator, {n}x{rows} periodic strip (dx = dy; "
                f"the full {n}^2 grid needs {288 * n * n / 1e9:.0f} GB of host memory, "
                f"this box has {ram / 1e9:.0f} GB)")
    return case, what


def run_reference(args):
    """--impl reference: the reference CPU implementation on this box's host cores."""
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    if rank != 0:
        return 0
    from paper_1607_08710_b200 import cases as CS
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    if not O.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libref_lagflux.so not built"})
        return 0
    case, what = reference_case(CS, world, args.scaling)
    value, wall = time_reference_cpu(case, args.steps, args.warmup, threads)
    sample = (f"{case.grid.nx}x{case.grid.ny} periodic, seed {case.seed}: {args.steps} timed "
              f"heun_step calls after {args.warmup} warm-up ({wall:.1f} s), OpenMP {threads} "
              f"threads on {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": what, "nx": case.grid.nx, "ny": case.grid.ny,
                       "boundary": "periodic", "cfl": case.cfl, "seed": case.seed,
                       "per_rank_share": world > 1 and args.scaling == "weak",
                       "cpu_model": cpu_model(), "cores": threads, "omp": omp_binding()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def fp64_roof(lib, device):
    """lf_fp64_peak: measured fp64 thread-instruction rates of this GPU (burst and
    sustained, DFMA / DMUL / DADD; csrc/fp64_peak.cu)."""
    import ctypes as C
    out = (C.c_double * 6)()
    if lib.lf_fp64_peak(device, 60.0, 1000.0, out) != 0:
        return None
    keys = ["dfma_burst", "dfma_sustained", "dmul_burst", "dmul_sustained", "dadd_burst",
            "dadd_sustained"]
    return {k: out[i] for i, k in enumerate(keys)}


def ncu_fp64_ops(kernel_key):
    """fp64 arithmetic instructions (DADD + DMUL + DFMA, thread level) per cell-update of
    the dominant kernel, from the committed ncu capture of the current build."""
    p = os.path.join(ROOT, "profiles", "fp64_ops.json")
    try:
        with open(p) as f:
            return json.load(f)[kernel_key]
    except Exception:
        return None


def run_ours(args):
    torch, dist, world, rank, local, multi = dist_setup(args)
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200 import native as N
    from paper_1607_08710_b200.solver import LagfluxSolver, nccl_unique_id

    n = args.n
    strong = args.scaling == "strong"
    if strong:
        case = CS.smooth(32768 if args.n == 16384 else args.n, args.steps)   # config 5
    else:
        case = CS.smooth(n, args.steps) if world == 1 else CS.smooth_weak(world, n, args.steps)
    g = case.grid
    dist_arg = None
    nid = None
    if multi:
        nid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        dist_arg = (rank, world, local, nid[0])
    solver = LagfluxSolver(g, case.bc, case.gamma, case.params, devices=(local,), path=args.path,
                           dist=dist_arg, math=args.math)
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)
    state = G.SolverState(field=np.zeros((4, 1, 1)))  # device-resident; host copy not needed
    solver.init_fourier(state, case.seed)
    controls = G.TimeControls(case.cfl, case.t_final, G.INT64_MAX)

    def barrier():
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        torch.cuda.synchronize()

    resolved = solver.resolved_path()   # auto: the fused one-kernel step on this grid
    # warm-up
    solver.advance(state, controls, args.warmup)
    barrier()
    launches0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        taken = solver.advance(state, controls, args.steps)
        ev1.record(stream)
        barrier()
    launches = solver.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if multi:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    cells_total = g.nx * g.ny
    value = cells_total * taken / (ms_max / 1e3)
    clock_summary = clocks.summary()

    # final-state digest (all ranks; interior_totals is the reference's ordered sums,
    # chained over the ranks, so it is bit-identical for any slab count)
    digest = {"interior_totals": [float(x).hex() for x in solver.interior_totals()],
              "time": float(state.time).hex(), "steps": state.step}
    if strong and multi:
        # the reference's scaling_sweep check (bench.cpp:96-99,124-128): the N-rank
        # run must equal one handle holding the whole grid, bit for bit
        single = None
        if rank == 0:
            s1 = LagfluxSolver(g, case.bc, case.gamma, case.params, devices=(local,), path=args.path,
                               math=args.math)
            st1 = G.SolverState(field=np.zeros((4, 1, 1)))
            s1.init_fourier(st1, case.seed)
            s1.advance(st1, controls, args.warmup)
            s1.advance(st1, controls, args.steps)
            single = {"interior_totals": [float(x).hex() for x in s1.interior_totals()],
                      "time": float(st1.time).hex(), "steps": st1.step}
            s1.close()
            del st1
        barrier()
        digest["single_handle"] = single
        digest["equal"] = single == {k: digest[k] for k in ("interior_totals", "time", "steps")} \
            if rank == 0 else None
        if rank == 0 and not digest["equal"]:
            print(json.dumps({"error": "DeterminismError: the N-rank final state differs from "
                                       "one handle", "digest": digest}), file=sys.stderr)

    # dominant kernel: per-launch CUDA events around the fused step kernel
    try:
        kernel_ms, loop_ms, k_launches = solver.time_steps(max(5, min(args.steps, 20)), case.cfl)
        kernel_name = ("one-kernel Heun step (lfb::k_fused_step)" if resolved == "fused" else
                       "two-pass Heun step (lfb::k_pass predictor + corrector, one launch pair)")
    except ValueError:  # stage-wise path: no single dominant kernel, use the whole step
        kernel_ms, loop_ms, k_launches = ms_max, ms_max, max(taken, 1)
        kernel_name = "whole stage-wise step (no fused kernel on this path)"
    per_launch_ms = kernel_ms / max(k_launches, 1)
    cells_local = g.nx * solver.local_rows()[1]
    hbm, hbm_src = measured_hbm()
    achieved = BYTES_PER_CELL_UPDATE * cells_local / (per_launch_ms / 1e3) / 1e9
    traffic = ncu_traffic(resolved)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": hbm_src,
                "algorithmic_bytes_per_cell_update": BYTES_PER_CELL_UPDATE,
                "kernel": kernel_name,
                "kernel_ms_per_launch": per_launch_ms,
                "kernel_share_of_step": kernel_ms / loop_ms if loop_ms > 0 else None,
                "frac_of_nominal_8TBs": achieved / 8000.0,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_source": traffic.get("source") if traffic else None,
                "compute": ncu_compute_bound(resolved, args.math)}
    # the roof that binds: fp64 (measured on this GPU now, lf_fp64_peak), with the
    # kernel's fp64 instructions per cell-update from the current build's ncu capture
    roof = fp64_roof(N.lib(), local) if rank == 0 else None
    ops = ncu_fp64_ops(f"{resolved}/{args.math}")
    if roof is not None:
        peak_ops = roof["dfma_sustained"]
        f64 = {"bound": "fp64", "unit": "G fp64 instr/s",
               "peak": peak_ops / 1e9,
               "peak_source": "measured now: lf_fp64_peak, DFMA back to back for ~1 s "
                              "(csrc/fp64_peak.cu); thread instructions, a DFMA counts once",
               "peaks_measured_G": {k: v / 1e9 for k, v in roof.items()}}
        if ops is not None:
            opc = ops["fp64_ops_per_cell_update"]
            ach = opc * cells_local / (per_launch_ms / 1e3)
            f64.update({"achieved": ach / 1e9, "frac": ach / peak_ops,
                        "ops_per_cell_update": opc, "ops_source": ops.get("source"),
                        "fp64_pipe_pct_ncu": ops.get("fp64_pipe_pct"),
                        "issue_active_pct_ncu": ops.get("issue_active_pct"),
                        "ceiling_cell_updates_per_s": peak_ops / opc,
                        "ceiling_hbm_frac": peak_ops / opc * BYTES_PER_CELL_UPDATE / (hbm * 1e9)})
        roofline["fp64"] = f64
        roofline["binding"] = ("fp64 / issue: the fp64 ceiling (fp64.ceiling_hbm_frac) is "
                               "below the HBM roof; frac is read against it")

    # the same workload in the tolerance arithmetic (LF_MATH_CONTRACT), device-resident
    contract = None
    if args.math == "exact" and not args.no_contract and resolved != "staged":
        solver.set_math("contract")
        cstate = G.SolverState(field=np.zeros((4, 1, 1)))
        solver.init_fourier(cstate, case.seed)
        solver.advance(cstate, controls, args.warmup)
        barrier()
        with ClockSampler(local) as cclocks:
            ev0.record(stream)
            ctaken = solver.advance(cstate, controls, args.steps)
            ev1.record(stream)
            barrier()
        t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        cvalue = cells_total * ctaken / (float(t.item()) / 1e3)
        ck_ms, _, ck_n = solver.time_steps(max(5, min(args.steps, 20)), case.cfl)
        ck_per = ck_ms / max(ck_n, 1)
        cach = BYTES_PER_CELL_UPDATE * cells_local / (ck_per / 1e3) / 1e9
        contract = {"value": cvalue, "unit": UNIT, "ms_per_step": float(t.item()) / max(ctaken, 1),
                    "roofline_frac": cach / hbm, "kernel_ms_per_launch": ck_per,
                    "clocks": cclocks.summary(),
                    "what": "the same steps with lf_set_math(LF_MATH_CONTRACT): FMA contraction and "
                            "reciprocal products in the same kernels; within the north-star "
                            "tolerance of the reference (relative L1 <= 1e-10 per field, dt to "
                            "1e-12; tests/test_gpu_contract.py, tests/test_gpu_baseline_configs.py), "
                            "not bit-identical"}
        cops = ncu_fp64_ops(f"{resolved}/contract")
        if roof is not None and cops is not None:
            opc = cops["fp64_ops_per_cell_update"]
            ach = opc * cells_local / (ck_per / 1e3)
            contract["fp64_frac"] = ach / roof["dfma_sustained"]
            contract["fp64_ops_per_cell_update"] = opc
        solver.set_math("exact")
        solver.init_fourier(state, case.seed)   # the e2e leg below starts from a fresh state

    # e2e through the public API with host buffers (rank-local slab)
    e2e = None
    if not args.no_e2e:
        row0, rows = solver.local_rows()
        # this rank's rows only (weak scaling: the global grid is N x 8.6 GB)
        solver.local_host = True
        host = torch.empty(solver.local_field_shape(), dtype=torch.float64, pin_memory=True)
        hf = host.numpy()
        solver.download(hf)  # the current state as this step's input (untimed)
        barrier()
        with_state = G.SolverState(field=hf)
        t0 = time.perf_counter()
        ev0.record(stream)
        solver.attach(with_state)                  # H2D from pinned host memory
        k2 = solver.advance(with_state, controls, args.steps)
        solver.sync_to_host(with_state)            # D2H of the result
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        # on the device (the copies and steps are on this stream), max over ranks; the
        # host wall clock of the same region is a cross-check
        e_ms = ev0.elapsed_time(ev1)
        barrier()
        t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        state_bytes = 4 * 8 * g.nx * rows
        e2e = {"value": cells_total * k2 / (float(t.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": state_bytes / max(k2, 1),
               "d2h_bytes_per_step": (state_bytes + 48 * k2) / max(k2, 1),
               "steps_amortised": k2, "host_wall_ms": wall * 1e3,
               "what": f"upload of the state from pinned host memory, {k2} steps "
                       f"(dt/diagnostics back to the host), download of the final state; the "
                       f"{state_bytes / 1e9:.1f} GB each way over PCIe are amortised over {k2} "
                       f"steps, so e2e approaches value as the run gets longer"}
        del host

    cpu_baseline = None
    if world == 1 and rank == 0 and not args.no_cpu:
        from oracle import oracle as O
        if O.ref_available():
            threads = os.cpu_count() or 1
            cs = cpu_sample_case(CS)
            steps = 5
            v, wall = time_reference_cpu(cs, steps, 1, threads)
            cpu_baseline = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{cs.grid.nx}x{cs.grid.ny} periodic strip of the config-4 "
                                      f"generator, {steps} heun_step calls after 1 warm-up "
                                      f"({wall:.1f} s), OpenMP {threads} threads on {cpu_model()}; "
                                      f"bench.py --impl reference times the full grid"}

    if rank == 0:
        if strong:
            workload = f"config5-smooth {g.nx}x{g.ny} periodic strong, y-slabs={world}"
        else:
            workload = (f"config{4 if world == 1 and g.nx < 32768 else 5}-smooth "
                        f"{g.nx}x{g.ny} periodic{' weak' if world > 1 else ''}, y-slabs={world}")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": taken, "warmup": args.warmup, "ms_per_step": ms_max / max(taken, 1),
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded 8-mode Fourier flow, BASELINE config 4/5)",
                "config": {"workload": workload,
                           "nx": g.nx, "ny": g.ny, "cfl": case.cfl, "seed": case.seed,
                           "parallelism": f"y-slab x{world}", "path": args.path, "resolved_path": resolved,
                           "math": args.math,
                           "l2": "inputs larger than L2 (state %.1f GB per GPU)" % (
                               4 * 8 * g.nx * solver.local_rows()[1] / 1e9)},
                "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
                "gpu_launches": launches, "clocks": clock_summary, "digest": digest}
        if contract is not None:
            line["math_contract"] = contract
        emit(line)
    solver.close()
    if multi:
        dist.destroy_process_group()
    if strong and multi and rank == 0 and not digest.get("equal"):
        return 3
    return 0


def run_ours_mat(args):
    """--workload triple_point: the multimaterial partial-density transport (SURVEY.md
    §8f row 1) on cases/triple_point.case at its reference resolution, one GPU."""
    torch, dist, world, rank, local, _ = dist_setup(args)
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200 import multimat as MM
    from paper_1607_08710_b200.solver import LagfluxSolver

    c = CS.triple_point(2048, 878)
    g = c.grid
    n_mat = len(c.material_gammas)
    ms = MM.make_material_set(c.material_gammas)
    f0, m0 = CS.regions_field(c)
    solver = LagfluxSolver(g, c.bc, c.gamma, c.params, materials=ms, devices=(local,))
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)
    state = G.SolverState(field=f0.copy())
    mat = m0.copy()
    controls = G.TimeControls(c.cfl, c.t_final, G.INT64_MAX)
    solver.advance(state, controls, args.warmup, mat)
    torch.cuda.synchronize()
    launches0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        taken = solver.advance(state, controls, args.steps, mat)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / max(taken, 1)
    launches = solver.launch_count() - launches0
    value = g.nx * g.ny / (ms_step / 1e3)
    bytes_per = BYTES_PER_CELL_UPDATE + 40 * n_mat   # + read P^n twice, write P*, read P*, write P^{n+1}
    hbm, hbm_src = measured_hbm()
    achieved = bytes_per * g.nx * g.ny / (ms_step / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": hbm_src,
                "algorithmic_bytes_per_cell_update": bytes_per,
                "kernel": "whole multimaterial step (two-pass material kernels lfb::k_pass_mat "
                          "+ ghost fills + finalize)",
                "kernel_ms_per_launch": ms_step, "kernel_share_of_step": 1.0, "traffic": None}

    e2e = None
    if not args.no_e2e:
        hf = torch.empty((4, g.nyt, g.nxt), dtype=torch.float64, pin_memory=True).numpy()
        hp = torch.empty((n_mat, g.nyt, g.nxt), dtype=torch.float64, pin_memory=True).numpy()
        hf[...] = f0
        hp[...] = m0.partial
        st2 = G.SolverState(field=hf)
        mat2 = MM.MaterialCells.__new__(MM.MaterialCells)
        mat2.partial = hp
        s2 = LagfluxSolver(g, c.bc, c.gamma, c.params, materials=ms, devices=(local,))
        s2.set_stream(stream.cuda_stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2.attach(st2)
        k2 = s2.advance(st2, controls, args.steps, mat2)
        s2.sync_to_host(st2, mat=mat2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        nbytes = (4 + n_mat) * 8 * g.nx * g.ny
        e2e = {"value": g.nx * g.ny * k2 / wall, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / max(k2, 1),
               "d2h_bytes_per_step": (nbytes + 48 * k2) / max(k2, 1),
               "what": f"upload of field + {n_mat} partial densities from pinned memory, {k2} "
                       f"steps (records to the host), download of both"}
        s2.close()

    cpu_baseline = None
    if not args.no_cpu:
        from oracle import oracle as O
        if O.ref_available():
            threads = os.cpu_count() or 1
            r = O.RefSolver(g, c.bc, c.gamma, c.params, threads=threads, materials=ms)
            r.set_state(f0)
            r.set_partials(m0.partial)
            r.heun_steps(1, c.cfl, c.t_final)
            nsteps = 5
            t0 = time.perf_counter()
            r.heun_steps(nsteps, c.cfl, c.t_final)
            wall = time.perf_counter() - t0
            cpu_baseline = {"value": g.nx * g.ny * nsteps / wall, "unit": UNIT, "cores": threads,
                            "kind": "reference",
                            "sample": f"the same triple point {g.nx}x{g.ny}, {nsteps} heun_step "
                                      f"calls with MaterialCells after 1 warm-up ({wall:.1f} s), "
                                      f"OpenMP {threads} threads"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": taken,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (cases/triple_point.case regions)",
            "config": {"workload": f"triple_point {g.nx}x{g.ny}, {n_mat} materials "
                                   f"(gammas {list(c.material_gammas)}), reflective",
                       "nx": g.nx, "ny": g.ny, "cfl": c.cfl,
                       "path": "two-pass material kernels (csrc/twopass_mat_kernel.cu)",
                       "l2": "state %.2f GB (field + partials)" % ((4 + n_mat) * 8 * g.nx * g.ny / 1e9)},
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks.summary()}
    emit(line)
    solver.close()
    return 0


def run_ours_sod(args):
    """--workload sod: BASELINE config 1 (Sod 400x4, reflective, CFL 0.5, to t = 0.2: 353
    steps) -- launch / latency bound, on the LF_PATH_AUTO choice (the small-grid cluster
    path, csrc/small_step.cu): whole runs of lf_advance, timed on the device."""
    torch, dist, world, rank, local, _ = dist_setup(args)
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200.solver import LagfluxSolver

    c = CS.sod()
    g = c.grid
    f0 = CS.initial_field(c)
    solver = LagfluxSolver(g, c.bc, c.gamma, c.params, devices=(local,),
                           path=args.path)
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)
    controls = G.TimeControls(c.cfl, c.t_final, G.INT64_MAX)
    big = 1 << 30
    for _ in range(max(args.warmup, 1)):   # whole runs to t_final
        st = G.SolverState(field=f0.copy())
        solver.attach(st)
        solver.advance(st, controls, big)
    torch.cuda.synchronize()
    launches0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs, taken, ms = max(1, args.steps // 50), 0, 0.0
    with ClockSampler(local) as clocks:
        for _ in range(runs):
            st = G.SolverState(field=f0.copy())
            solver.attach(st)
            torch.cuda.synchronize()
            ev0.record(stream)
            taken += solver.advance(st, controls, big)
            ev1.record(stream)
            torch.cuda.synchronize()
            ms += ev0.elapsed_time(ev1)
    ms_step = ms / taken
    launches = solver.launch_count() - launches0
    value = g.nx * g.ny / (ms_step / 1e3)
    solver.sync_to_host(st)
    e2e = None
    if not args.no_e2e:
        hf = torch.empty((4, g.nyt, g.nxt), dtype=torch.float64, pin_memory=True).numpy()
        hf[...] = f0
        s2 = LagfluxSolver(g, c.bc, c.gamma, c.params, devices=(local,))
        s2.set_stream(stream.cuda_stream)
        st2 = G.SolverState(field=hf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2.attach(st2)
        k2 = s2.advance(st2, controls, big)
        s2.sync_to_host(st2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        nbytes = 4 * 8 * g.nx * g.ny
        e2e = {"value": g.nx * g.ny * k2 / wall, "unit": UNIT, "h2d_bytes_per_step": nbytes / k2,
               "d2h_bytes_per_step": (nbytes + 48 * k2) / k2, "steps_amortised": k2,
               "what": f"upload from pinned memory, the {k2} steps to t = 0.2 (records to the "
                       f"host), download of the final state"}
        s2.close()
    cpu_baseline = None
    if not args.no_cpu:
        from oracle import oracle as O
        if O.ref_available():
            threads = os.cpu_count() or 1
            best = {}
            for th in sorted({1, threads}):
                r = O.RefSolver(g, c.bc, c.gamma, c.params, threads=th)
                r.set_state(f0)
                t0 = time.perf_counter()
                n = len(r.heun_steps(taken // runs, c.cfl, c.t_final))
                best[th] = g.nx * g.ny * n / (time.perf_counter() - t0)
            th = max(best, key=best.get)
            cpu_baseline = {"value": best[th], "unit": UNIT, "cores": th, "kind": "reference",
                            "sample": f"the whole config-1 run ({taken // runs} heun_step calls), "
                                      f"OpenMP on {th} thread(s) (the faster of 1 and {threads}: "
                                      + ", ".join(f"{k}: {v / 1e6:.1f} M/s" for k, v in best.items())
                                      + ")"}
    path = solver.resolved_path()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": taken,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 1 initial state)",
            "config": {"workload": "config1-sod 400x4 reflective, CFL 0.5, to t = 0.2",
                       "nx": g.nx, "ny": g.ny, "cfl": c.cfl, "path": path,
                       "runs": runs, "l2": "state 51 KB: L2 / L1 resident; latency-bound"},
            "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": None,
                         "frac": None, "traffic": None,
                         "note": "1 600 cells: neither HBM nor fp64 binds; the step is two "
                                 "dependent stage chains and two cluster barriers "
                                 "(DESIGN.md §4, Small grids)",
                         "us_per_step": 1e3 * ms_step},
            "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary()}
    emit(line)
    solver.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384, help="cells per side per GPU")
    ap.add_argument("--path", choices=["auto", "twopass", "fused", "staged", "small"], default="auto")
    ap.add_argument("--math", choices=["exact", "contract"], default="exact",
                    help="exact: bit-identical to the reference; contract: FMA contraction and "
                         "reciprocal products in the two-pass kernels (north-star tolerance)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-contract", action="store_true",
                    help="skip the extra LF_MATH_CONTRACT measurement of the headline workload")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N > 1: weak = 16384 x 16384 per GPU (config 5's weak mode); strong = "
                         "config 5's 32768^2 split over the N GPUs, with the single-handle "
                         "determinism digest")
    ap.add_argument("--workload", choices=["smooth", "triple_point", "sod"], default="smooth",
                    help="smooth: BASELINE config 4/5 (the headline); triple_point: the "
                         "multimaterial transport (one GPU); sod: BASELINE config 1 (one GPU)")
    args = ap.parse_args()
    global _JSON_FD
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    # OpenMP binding of the reference CPU path (bench.cpp-style timing on all cores),
    # before any library that loads libgomp (oracle/_ref, the oracle, torch)
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_PROC_BIND", "close")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "triple_point":
        return run_ours_mat(args)
    if args.workload == "sod":
        return run_ours_sod(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
