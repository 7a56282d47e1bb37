"""CPU, world size 2 (gloo): the y-slab decomposition of the multi-GPU path.

Each rank owns the rows the LIBRARY assigns it (lf_slab_partition, the same
function lf_create_dist uses) and steps its slab with the numpy restatement
(oracle/numpy_ref.py), exchanging halo rows with the two-phase protocol of
csrc/nccl_comm.cpp (phase A: bottom rows down / top halo from above; phase B:
top rows up / bottom halo from below -- unambiguous even when both neighbours
are the same rank on a periodic ring) and combining the CFL rate, min rho and
min e_int with all-reduces, the boundary faces with a gather + the ordered sum.
The gathered result must equal the single-domain C oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numpy_ref as NR
from oracle import oracle as O
from paper_1607_08710_b200 import cases as CS
from paper_1607_08710_b200 import grid as G
from paper_1607_08710_b200 import native as N

W = 2
STEPS = 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def partition(ny, nranks, rank):
    import ctypes as C
    r0, n = C.c_int(), C.c_int()
    assert N.lib().lf_slab_partition(ny, nranks, rank, C.byref(r0), C.byref(n)) == 0
    return r0.value, n.value


def neighbours(rank, nranks, periodic):
    lo = rank - 1 if rank > 0 else (nranks - 1 if periodic else -1)
    hi = rank + 1 if rank < nranks - 1 else (0 if periodic else -1)
    return lo, hi


def exchange(f, rank, nranks, periodic):
    """csrc/nccl_comm.cpp nccl_exchange_halos, 2 ghost rows, over gloo."""
    g = NR.G
    lo, hi = neighbours(rank, nranks, periodic)
    rows = f.shape[1] - 2 * g
    reqs = []
    bufs = []
    # phase A: bottom rows down, top halo from above
    if lo >= 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(f[:, g:2 * g])), lo))
    if hi >= 0:
        b = torch.empty((4, g, f.shape[2]), dtype=torch.float64)
        reqs.append(dist.irecv(b, hi))
        bufs.append((b, slice(g + rows, 2 * g + rows)))
    for r in reqs:
        r.wait()
    reqs = []
    # phase B: top rows up, bottom halo from below
    if hi >= 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(f[:, rows:rows + g])), hi))
    if lo >= 0:
        b = torch.empty((4, g, f.shape[2]), dtype=torch.float64)
        reqs.append(dist.irecv(b, lo))
        bufs.append((b, slice(0, g)))
    for r in reqs:
        r.wait()
    for b, sl in bufs:
        f[:, sl] = b.numpy()


def ghosts(f, bc, rank, nranks):
    NR.fill_x(f, bc[0], bc[1])
    periodic = bc[2] == G.PERIODIC
    exchange(f, rank, nranks, periodic)
    NR.fill_y(f, bc[2], bc[3], do_lo=(not periodic and rank == 0) or nranks == 1,
              do_hi=(not periodic and rank == nranks - 1) or nranks == 1)


def allreduce(x, op):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=op)
    return float(t.item())


def rank_main(rank, port, cfg, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=W)
    case = cfg_case(cfg)
    g = case.grid
    y0, rows = partition(g.ny, W, rank)
    full = CS.initial_field(case)
    f = np.zeros((4, rows + 4, g.nx + 4))
    f[:, 2:2 + rows, 2:2 + g.nx] = g.interior(full)[:, y0:y0 + rows]
    gm1 = case.gamma - 1.0
    time, acc, diag = 0.0, [0.0] * 4, []
    for _ in range(STEPS):
        ghosts(f, case.bc.as_list(), rank, W)
        rate = allreduce(NR.local_rate(f, case.gamma, g.dx, g.dy), dist.ReduceOp.MAX)
        dt = case.cfl / rate
        if time + dt > case.t_final:
            dt = case.t_final - time
        fa = NR.stage_fluxes(f, case.gamma, case.params.beta)
        us = f.copy()
        us[:, 2:-2, 2:-2], _, _ = NR.apply_update(f, fa, None, dt, g.dx, g.dy)
        ghosts(us, case.bc.as_list(), rank, W)
        fb = NR.stage_fluxes(us, case.gamma, case.params.beta)
        new, mr, me = NR.apply_update(f, fa, fb, dt, g.dx, g.dy)
        mr = allreduce(mr, dist.ReduceOp.MIN)
        me = allreduce(me, dist.ReduceOp.MIN)
        left, right, bot, top = NR.boundary_faces(fa, fb)
        parts = [None] * W
        dist.all_gather_object(parts, (y0, left, right, bot, top))
        parts.sort(key=lambda p: p[0])
        L = np.concatenate([p[1] for p in parts], axis=1)
        R = np.concatenate([p[2] for p in parts], axis=1)
        acc = NR.ordered_outflow(acc, L, R, parts[0][3], parts[-1][4], dt, g.dx, g.dy)
        f[:, 2:-2, 2:-2] = new
        time = time + dt
        diag.append((dt, time, mr, gm1 * me))
    parts = [None] * W
    dist.all_gather_object(parts, (y0, f[:, 2:-2, 2:-2].copy()))
    if rank == 0:
        parts.sort(key=lambda p: p[0])
        out.put((np.concatenate([p[1] for p in parts], axis=1), diag, acc))
    dist.barrier()
    dist.destroy_process_group()


def cfg_case(cfg):
    if cfg == "smooth":
        return CS.smooth(24, STEPS, ny=18, y_extent=0.75)
    if cfg == "sedov":
        return CS.sedov(24, STEPS)
    return CS.quadrant(20, STEPS)


@pytest.mark.parametrize("cfg", ["smooth", "sedov", "quadrant"])
def test_two_rank_slabs_equal_single_domain(cfg):
    case = cfg_case(cfg)
    # the numpy restatement itself is pinned to the C oracle on one slab
    ref_state, ref_diag = None, None
    s = O.OracleSolver(case.grid, case.bc, case.gamma, case.params)
    state = G.SolverState(field=CS.initial_field(case))
    for _ in range(STEPS):
        s.heun_step(state, case.cfl, case.t_final)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=rank_main, args=(r, port, cfg, q)) for r in range(W)]
    for p in procs:
        p.start()
    got, diag, acc = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = case.grid.interior(state.field)
    assert np.array_equal(got == ref, np.ones_like(ref, dtype=bool)), "slab result differs"
    assert [d[0] for d in diag] == [d.dt for d in state.diagnostics]
    assert [d[2] for d in diag] == [d.min_rho for d in state.diagnostics]
    assert [d[3] for d in diag] == [d.min_p for d in state.diagnostics]
    assert acc == list(state.boundary_outflow)


def test_partition_matches_python_rule():
    """lf_slab_partition: contiguous, covering, remainder to the first slabs."""
    for ny in (1, 7, 16, 33, 32768):
        for n in (1, 2, 3, 8):
            if n > ny:
                continue
            rows = [partition(ny, n, r) for r in range(n)]
            assert rows[0][0] == 0
            assert sum(r[1] for r in rows) == ny
            for a, b in zip(rows, rows[1:]):
                assert a[0] + a[1] == b[0]
            assert max(r[1] for r in rows) - min(r[1] for r in rows) <= 1
