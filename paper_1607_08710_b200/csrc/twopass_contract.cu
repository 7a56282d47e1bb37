// twopass_contract.cu -- the two-pass Heun kernels (twopass_kernel.cu) in the
// tolerance arithmetic of LF_MATH_CONTRACT: compiled with --fmad=true (products
// and sums contract into DFMA) and with quotients as products by a refined
// reciprocal (fastmath.cuh, LF_CONTRACT).  Same data flow, same failure flags
// (a flagged step is recomputed by the stage-wise IEEE kernels); results are
// not bit-identical to the reference but within the north star's tolerance:
// relative L1 <= 1e-10 per conserved field, dt sequence to 1e-12
// (tests/test_gpu_contract.py).  Selected per handle with lf_set_math.
#define LF_CONTRACT 1
#include "twopass_kernel.cu"
