// fused_contract.cu -- the one-kernel Heun step (fused_kernel.cu) in the tolerance
// arithmetic of LF_MATH_CONTRACT (see twopass_contract.cu): --fmad=true and
// quotients as products by a refined reciprocal (fastmath.cuh, LF_CONTRACT).
#define LF_CONTRACT 1
#include "fused_kernel.cu"
