"""Build and time compile-time variants of the fused step kernel side by side.

    python tools/variants.py build            # here (no GPU): nvcc every variant
    python tools/variants.py run [N] [steps]  # on the GPU box: time + bitwise check

Each variant is a full liblagflux_b200 built with extra -D flags into
tools/_variants/<name>.so (git-ignored, travels with gpurun).  `run` times
lf_time_steps on the N^2 periodic smooth-flow workload (BASELINE config 4
generator) and checks that every variant's final state equals the first one's
bit for bit (all variants must compute identical results).
"""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "_variants")
CSRC = os.path.join(ROOT, "paper_1607_08710_b200", "csrc")

# name -> (extra nvcc flags, LF_PATH_*); "base_*" variants build the same path
# from the committed sources (git HEAD) for an A/B against the working tree
# (a third element selects LF_MATH_*: 1 = contract; bit equality is checked
# against the first variant of the same arithmetic)
VARIANTS = {
    "f": ("", 1),
    "f_intmm": ("-DLF_INTMINMAX=1", 1),
}


def _head_tree():
    tmp = "/tmp/lf_variants_head"
    subprocess.run(["rm", "-rf", tmp], check=True)
    os.makedirs(tmp)
    arch = subprocess.run(["git", "-C", ROOT, "archive", "HEAD", "paper_1607_08710_b200/csrc", "include"],
                          check=True, stdout=subprocess.PIPE).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=arch, check=True)
    return os.path.join(tmp, "paper_1607_08710_b200", "csrc")


def build(names=None):
    os.makedirs(OUT, exist_ok=True)
    # only the current variants travel to the GPU box (the snapshot is size-capped)
    for fn in os.listdir(OUT):
        if fn.split(".")[0] not in VARIANTS:
            os.unlink(os.path.join(OUT, fn))
    head = None
    procs = []
    for name, (flags, _path, *_m) in VARIANTS.items():
        if names and name not in names:
            continue
        src = CSRC
        if name.startswith("base_"):
            head = head or _head_tree()
            src = head
        so = os.path.join(OUT, f"{name}.so")
        cmd = ["make", "-s", "-C", src, f"OUT={so}", f"EXTRA_NVFLAGS={flags}", so]
        procs.append((name, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for name, p in procs:
        out = p.communicate()[0].decode()
        spill = [l for l in out.splitlines() if "spill" in l]
        print(name, "rc", p.returncode, spill[:1])


def run(n=8192, steps=10):
    import numpy as np
    from paper_1607_08710_b200 import cases as CS
    from paper_1607_08710_b200 import native as N
    from paper_1607_08710_b200.solver import make_desc
    case = CS.smooth(n, steps)
    g = case.grid
    refs = {}
    results = {}
    names = list(VARIANTS) * 2   # two rounds, interleaved: the better of each variant counts
    for name in names:
        so = os.path.join(OUT, f"{name}.so")
        if not os.path.exists(so):
            continue
        lib = C.CDLL(so)
        for fn, res, args in N.SIGNATURES:
            getattr(lib, fn).restype = res
            getattr(lib, fn).argtypes = args
        desc = make_desc(g, case.bc, case.gamma, case.params)
        h = C.c_void_p()
        assert lib.lf_create(C.byref(desc), (C.c_int * 1)(0), 1, C.byref(h)) == 0
        assert lib.lf_set_path(h, VARIANTS[name][1]) == 0
        math = VARIANTS[name][2] if len(VARIANTS[name]) > 2 else 0
        assert lib.lf_set_math(h, math) == 0
        assert lib.lf_init_fourier(h, case.seed) == 0
        km, lm, nl = C.c_double(), C.c_double(), C.c_int()
        assert lib.lf_time_steps(h, 3, case.cfl, C.byref(km), C.byref(lm), C.byref(nl)) == 0
        assert lib.lf_time_steps(h, steps, case.cfl, C.byref(km), C.byref(lm), C.byref(nl)) == 0
        f = np.zeros((4, g.nyt, g.nxt))
        assert lib.lf_download(h, N.field_ptrs(f), g.nxt, 0) == 0
        lib.lf_destroy(h)
        per = km.value / nl.value
        same = None
        ref = refs.get(math)
        if ref is None:
            refs[math] = f
        else:
            same = bool(np.array_equal(g.interior(f) == g.interior(ref), np.ones_like(g.interior(f), bool)))
        prev = results.get(name)
        if prev is not None and prev["kernel_ms"] < per:
            per = prev["kernel_ms"]
        results[name] = {"kernel_ms": per, "gcells_s": g.nx * g.ny / per / 1e6, "same_as_first": same}
        print(name, json.dumps(results[name]), flush=True)
    return results


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:] or None)
    else:
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
        s = int(sys.argv[3]) if len(sys.argv) > 3 else 10
        run(n, s)
