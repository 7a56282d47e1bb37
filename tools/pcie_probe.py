"""Host<->device copy rates of the e2e leg's shapes (one B200): the C ABI's 2D copies
(lf_upload / lf_download, pitched rows of the reference's ghosted layout) against
plain 1D copies of the same bytes, pinned host memory throughout.

    python tools/pcie_probe.py [n]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import grid as G
    from paper_1607_08710_b200 import native as N
    from paper_1607_08710_b200.solver import LagfluxSolver
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    case = CS.smooth(n, 1)
    g = case.grid
    s = LagfluxSolver(g, case.bc, case.gamma, case.params)
    host = torch.empty((4, g.nyt, g.nxt), dtype=torch.float64, pin_memory=True)
    host.fill_(1.0)
    f = host.numpy()
    out = {}
    nbytes = 4 * 8 * g.nx * g.ny
    lib, h = s._lib, s._h
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert lib.lf_upload(h, N.field_ptrs(f), g.nxt) == 0
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        assert lib.lf_download(h, N.field_ptrs(f), g.nxt, 0) == 0
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out.setdefault("abi_upload_GBs", []).append(nbytes / (t1 - t0) / 1e9)
        out.setdefault("abi_download_GBs", []).append(nbytes / (t2 - t1) / 1e9)
    dev = torch.empty(host.numel(), dtype=torch.float64, device="cuda")
    flat = host.view(-1)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(flat, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        flat.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out.setdefault("flat_h2d_GBs", []).append(host.numel() * 8 / (t1 - t0) / 1e9)
        out.setdefault("flat_d2h_GBs", []).append(host.numel() * 8 / (t2 - t1) / 1e9)
    s.close()
    print(json.dumps({k: max(v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
