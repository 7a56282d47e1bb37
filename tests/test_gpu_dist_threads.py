"""GPU: the distributed y-slab path (lf_create_dist + NCCL) on one GPU, ranks as
host threads over the thread-rank NCCL stand-in (tests/fake_nccl), bit for bit
against single-handle runs: periodic / transmissive / reflective y, 2-4 ranks,
the two-pass, stage-wise and fused paths, the exact-kernel switch, the on-device
initial state and three materials (tools/dist_threads.py).  A subprocess, so the
stand-in is the process's first NCCL."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so")


def test_distributed_slabs_equal_single_handle(cuda):
    assert os.path.exists(FAKE), "tests/fake_nccl not built (make -C tests/fake_nccl)"
    env = dict(os.environ, LF_NCCL_LIB=FAKE)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dist_threads.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "MISMATCH" not in p.stdout
    assert p.stdout.count(": ok") >= 14 + 12   # + the 12 rank-owned error cases


@pytest.mark.slow
def test_config5_strip_eight_ranks_equal_single_handle(cuda):
    """BASELINE config 5's generator on a 32768 x 2048 periodic strip, 20 steps, as
    8 y-slab ranks (the 8-GPU decomposition) == one handle, on the fused step and on
    the two-pass kernels (tools/dist_threads.py --config5-strip)."""
    assert os.path.exists(FAKE), "tests/fake_nccl not built (make -C tests/fake_nccl)"
    env = dict(os.environ, LF_NCCL_LIB=FAKE)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dist_threads.py"),
                        "--config5-strip"], env=env, capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count(": ok") == 2
