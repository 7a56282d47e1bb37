// reduce.cuh -- block-level reductions for the stage-wise kernels' scalars.
//
// Min / max are exact and order independent, so a warp -> block -> one atomic
// per block tree gives the same value as the reference's OpenMP reductions while
// keeping same-address atomics to one per block (per-warp atomics on the three
// step scalars serialised the update kernel at L2).
#pragma once

#include <cstdint>

namespace lfb {

#ifdef __CUDACC__

template <class T, class Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Every thread of the block must call it; returns the block result in thread 0
// (others: unspecified).  blockDim.x * blockDim.y * blockDim.z <= 1024.
template <class T, class Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T identity) {
  __shared__ T part[32];
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  v = warp_reduce(v, op);
  __syncthreads();  // part[] may still be read by a previous call
  if ((tid & 31) == 0) part[tid >> 5] = v;
  __syncthreads();
  if (tid < 32) {
    v = tid < (nthreads + 31) / 32 ? part[tid] : identity;
    v = warp_reduce(v, op);
  }
  return v;
}

struct MinOp {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return b < a ? b : a; }
};
struct MaxOp {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? b : a; }
};

#endif  // __CUDACC__

}  // namespace lfb
