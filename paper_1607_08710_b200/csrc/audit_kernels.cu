// audit_kernels.cu -- lagflux::interior_totals (grid.cpp:122-133) on the device.
//
// The reference sums each component over the interior in row-major order with
// one rounding per addition, then scales by the cell volume.  A bit-equal sum
// is one dependent fp64 add chain per component, so this is a latency-bound
// audit, not a bandwidth kernel: one warp per component streams its rows with
// coalesced loads (the next chunk in flight in registers while the current one
// is summed) and runs the chain lane-uniformly from shared memory.  A slab
// starts from the running sums of the slab below (`s_in`), so slabs -- and
// ranks, over NCCL -- chain in the reference's row order.
#include <cuda_runtime.h>

#include "kernels.h"

namespace lfb {

namespace {

constexpr int TOT_PER_LANE = 32;
constexpr int TOT_CHUNK = 32 * TOT_PER_LANE;  // elements per chunk (8 KB)

__global__ void __launch_bounds__(32)
    k_interior_sums(const double* __restrict__ u, int64_t fstride, int pitch, int nx, int ny,
                    const double* __restrict__ s_in, double* __restrict__ s_out) {
  __shared__ __align__(16) double buf[TOT_CHUNK];
  const int c = blockIdx.x, lane = threadIdx.x;
  const double* f = u + c * fstride;
  double s = s_in ? s_in[c] : 0.0;
  const int per_row = (nx + TOT_CHUNK - 1) / TOT_CHUNK;
  const int64_t nch = (int64_t)per_row * ny;
  double r[TOT_PER_LANE];
  auto load = [&](int64_t k) {
    const int j = (int)(k / per_row), i0 = (int)(k % per_row) * TOT_CHUNK;
    const double* p = f + (int64_t)j * pitch + i0;
#pragma unroll
    for (int q = 0; q < TOT_PER_LANE; ++q) {
      const int i = lane + 32 * q;
      r[q] = i0 + i < nx ? __ldcs(p + i) : 0.0;
    }
  };
  if (nch > 0) load(0);
  for (int64_t k = 0; k < nch; ++k) {
    __syncwarp();  // every lane is done reading the previous chunk
#pragma unroll
    for (int q = 0; q < TOT_PER_LANE; ++q) buf[lane + 32 * q] = r[q];
    __syncwarp();
    if (k + 1 < nch) load(k + 1);
    const int m = nx - (int)(k % per_row) * TOT_CHUNK;
    if (m >= TOT_CHUNK) {
#pragma unroll 64
      for (int e = 0; e < TOT_CHUNK; ++e) s += buf[e];
    } else {
      for (int e = 0; e < m; ++e) s += buf[e];
    }
  }
  if (lane == 0) s_out[c] = s;
}

}  // namespace

void launch_interior_sums(const double* u, int64_t fstride, int pitch, int nx, int ny,
                          const double* s_in, double* s_out, cudaStream_t st) {
  count_launch();
  k_interior_sums<<<4, 32, 0, st>>>(u, fstride, pitch, nx, ny, s_in, s_out);
}

}  // namespace lfb
