// selftest.cu -- device self-check of fastmath.cuh against the IEEE operators.
//
// lf_selftest_fastmath draws n operand pairs (splitmix64 bit patterns over the
// whole finite range, half of them concentrated in the physical range) and
// counts, for the division (with and without a shared reciprocal), the square
// root and the Sweby limiter, how often the fast path claims validity and how
// often a valid fast result differs from the IEEE / reference result.
// tests/test_gpu_fastmath.py requires zero differences.
#include <cuda_runtime.h>

#include "../../include/lagflux_b200.h"
#include "face_fast.cuh"
#include "fastmath.cuh"
#include "kernels.h"
#include "lagflux_device.cuh"

namespace lfb {

namespace {

__device__ __forceinline__ unsigned long long splitmix(unsigned long long& s) {
  unsigned long long z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// finite double: either any exponent (raw bits) or a physical-range magnitude
__device__ __forceinline__ double draw(unsigned long long& s, bool wide) {
  const unsigned long long r = splitmix(s);
  if (wide) {
    unsigned long long b = r;
    const unsigned long long e = (b >> 52) & 0x7ff;
    if (e == 0x7ff) b ^= 0x4000000000000000ull;  // no inf / nan
    return __longlong_as_double((long long)b);
  }
  // mantissa random, exponent in [-40, 40]
  const unsigned long long mant = r & 0x000fffffffffffffull;
  const long long e = (long long)((r >> 52) % 81) - 40 + 1023;
  const unsigned long long sign = r & 0x8000000000000000ull;
  return __longlong_as_double((long long)(sign | ((unsigned long long)e << 52) | mant));
}

__device__ __forceinline__ bool same(double x, double y) {
  return x == y || (x != x && y != y);
}

__global__ void k_selftest(long long n, unsigned long long seed, unsigned long long* out) {
  unsigned long long c[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long s = seed ^ (unsigned long long)i * 0x632be59bd9b4e019ull;
    const bool wide = (i & 1) != 0;
    const double a = draw(s, wide);
    double b = draw(s, wide);
    if (b == 0.0) b = 1.0;
    const double a2 = draw(s, false);
    c[0] += 1;
    // division a / b, and a second quotient a2 / b through the same reciprocal
    bool ok = true;
    const Recip r = recip_of(b);
    const double q = div_fast(a, r, ok);
    if (ok) {
      c[1] += 1;
      if (!same(q, a / b)) c[2] += 1;
    }
    bool ok2 = true;
    const double q2 = div_fast(a2, r, ok2);
    if (ok2 && !same(q2, a2 / b)) c[3] += 1;
    // square root of |a|
    const double x = fabs(a);
    bool oks = true;
    const double sq = sqrt_fast(x, oks);
    if (oks) {
      c[4] += 1;
      if (!same(sq, sqrt(x))) c[5] += 1;
    }
    // limiter against the reference formula (reconstruct.hpp:24-30)
    const double beta = 1.0 + (double)(splitmix(s) >> 11) * 0x1.0p-53;
    const double la = draw(s, false), lb = draw(s, false);
    if (!same(sweby_fast(la, lb, beta), sweby(la, lb, beta))) c[6] += 1;
    // div_exact: dividends down to the subnormals (scales 2^-1074 .. 2^-700,
    // subnormal quotients included) and constructed near-ties of the subnormal
    // rounding (b (m + 1/2) 2^-1074 +- 1 ulp) over physical-range divisors
    {
      const unsigned long long rr = splitmix(s);
      double tiny, bd = fabs(draw(s, false));
      if (bd == 0.0) bd = 1.0;
      if (rr & 1) {
        const int e = (int)((rr >> 1) % 375);
        const unsigned long long mant = splitmix(s) >> (12 + (int)((rr >> 9) % 40));
        tiny = ldexp((double)mant * 0x1p-537 * 0x1p-537, e);
      } else {
        const double mm = (double)(splitmix(s) >> 20) + 0.5;
        tiny = (bd * mm) * 0x1p-537 * 0x1p-537;
        const unsigned long long t2 = splitmix(s);
        if ((t2 & 2) && tiny > 0.0)  // one ulp off the tie (never below +0)
          tiny = __longlong_as_double(__double_as_longlong(tiny) + ((t2 & 4) ? 1 : -1));
      }
      if (splitmix(s) & 1) tiny = -tiny;
      bool ok = true;
      const double q = div_exact(tiny, recip_of(bd), ok);
      c[7] += 1;
      if (ok && !same(q, tiny / bd) && !(q == 0.0 && tiny / bd == 0.0)) c[8] += 1;
      if (!ok) c[9] += 1;
    }
  }
  for (int k = 0; k < 10; ++k) atomicAdd(&out[k], c[k]);
}

// ---- the cell box (face_fast.cuh) --------------------------------------
// A value of the box drawn with its extremes over-represented: exponent at
// either end of the range, all-zero or all-one mantissas, and (through
// `near`) neighbours one ulp apart, the worst case of the cancellation bounds.
__device__ __forceinline__ double box_mag(unsigned long long& s, int emin, int emax) {
  const unsigned long long r = splitmix(s);
  int e;
  switch (r & 3) {
    case 0: e = emin; break;
    case 1: e = emax - 1; break;
    default: e = emin + (int)((r >> 2) % (unsigned long long)(emax - emin));
  }
  unsigned long long mant = (r >> 12) & 0x000fffffffffffffull;
  if (((r >> 8) & 7) == 0) mant = 0;
  if (((r >> 8) & 7) == 1) mant = 0x000fffffffffffffull;
  return __longlong_as_double((long long)(((unsigned long long)(e + 1023) << 52) | mant));
}
__device__ __forceinline__ double nudge(unsigned long long& s, double x) {
  const unsigned long long r = splitmix(s);
  const long long b = __double_as_longlong(x);
  switch (r & 3) {
    case 0: return __longlong_as_double(b + 1);
    case 1: return __longlong_as_double(b - 1);
    default: return x;
  }
}
__device__ __forceinline__ void box_cell(unsigned long long& s, const double* prev, double w[4]) {
  const unsigned long long r = splitmix(s);
  const bool near = prev && (r & 1);
  w[0] = near ? nudge(s, prev[0]) : box_mag(s, -100, 100);
  w[3] = near ? nudge(s, prev[3]) : box_mag(s, -100, 100);
  for (int q = 1; q <= 2; ++q) {
    const unsigned long long k = splitmix(s);
    if (near && (k & 1)) {
      w[q] = prev[q] == 0.0 ? 0.0 : nudge(s, prev[q]);
    } else if ((k & 7) == 2) {
      w[q] = 0.0;
    } else if ((k & 7) == 3) {
      // precursor-sized velocities: 2^-1074 .. 2^-600, subnormals included
      const double m = ldexp((double)(splitmix(s) >> (12 + (int)(k >> 8) % 50)) * 0x1p-537 * 0x1p-537,
                             (int)((k >> 16) % 470));
      w[q] = (k & 8) ? -m : m;
    } else {
      const double m = box_mag(s, -500, 100);
      w[q] = (k & 8) ? -m : m;
    }
  }
  // a nudge can step out of the box at its edges; the kernels would flag it
  if (!cell_in_box(w)) {
    w[0] = 1.0;
    w[1] = 0.0;
    w[2] = 0.0;
    w[3] = 1.0;
  }
}

// counts: {faces solved, faces with a failed range check}
__global__ void k_selftest_box(long long n, unsigned long long seed, unsigned long long* out) {
  unsigned long long c[2] = {0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long s = seed ^ (unsigned long long)i * 0x9e3779b97f4a7c15ull;
    const double gm1 = box_mag(s, -14, 6);
    const double gamma = 1.0 + gm1;
    if (!const_in_box(gamma, gm1)) continue;
    const double beta = 1.0 + (double)(splitmix(s) >> 11) * 0x1.0p-53;
    const FK C = make_fk(gamma, gm1, beta, 1.0, 1.0);
    // four cells along the face normal: i-1, i | i+1, i+2
    double w[4][4];
    for (int k = 0; k < 4; ++k) box_cell(s, k ? w[k - 1] : nullptr, w[k]);
    double mh[4], pl[4];
    for (int q = 0; q < 4; ++q) {
      double lo, hi;
      cell_traces<true>(w[0][q], w[1][q], w[2][q], beta, lo, hi);
      mh[q] = hi;
      cell_traces<true>(w[1][q], w[2][q], w[3][q], beta, lo, hi);
      pl[q] = lo;
    }
    if (!traces_ok(mh[0], mh[3], pl[0], pl[3])) continue;  // the reference's own failure
    bool ok0 = true, ok1 = true;
    double f[4], ps, us;
    face_fast<0>(mh[0], mh[1], mh[2], mh[3], pl[0], pl[1], pl[2], pl[3], C, f, ok0, ps, us);
    face_mean<0>(mh[0], mh[1], mh[2], mh[3], pl[0], pl[1], pl[2], pl[3], ps, us, C, f, ok0);
    face_fast<1>(mh[0], mh[1], mh[2], mh[3], pl[0], pl[1], pl[2], pl[3], C, f, ok1, ps, us);
    face_mean<1>(mh[0], mh[1], mh[2], mh[3], pl[0], pl[1], pl[2], pl[3], ps, us, C, f, ok1);
    bool okp = true;
    double wp[4];
    prim_fast(w[1][0], w[1][0] * w[1][1], w[1][0] * w[1][2], 1.0, gm1, wp, okp);
    c[0] += 1;
    if (!ok0 || !ok1 || !okp) c[1] += 1;
  }
  for (int k = 0; k < 2; ++k) atomicAdd(&out[k], c[k]);
}

// cell_epilogue_box against cell_epilogue on updated cells drawn at the box
// edges: counts {cells the box accepts, of those failing a per-operation check,
// of those with a different rate or e_int}.
__global__ void k_selftest_epilogue(long long n, unsigned long long seed, unsigned long long* out) {
  unsigned long long c[3] = {0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long s = seed ^ (unsigned long long)i * 0xd1b54a32d192ed03ull;
    const double gm1 = box_mag(s, -14, 6);
    const double gamma = 1.0 + gm1;
    if (!const_in_box(gamma, gm1)) continue;
    const double dx = box_mag(s, -100, 100), dy = box_mag(s, -100, 100);
    const FK C = make_fk(gamma, gm1, 1.5, dx, dy);
    double v[4];
    v[0] = box_mag(s, -101, 101);
    for (int q = 1; q <= 2; ++q) {
      const unsigned long long k = splitmix(s);
      double m = (k & 7) == 0 ? 0.0 : box_mag(s, (k & 8) ? -1074 + 60 : -300, 101);
      if ((k & 7) == 1) m = __longlong_as_double((long long)(splitmix(s) & 0xfffffffffffffull));  // subnormal
      v[q] = (k & 16) ? -m : m;
    }
    // E from a target pressure near the p box edges (the recomputed p differs by rounding)
    const double pt = box_mag(s, -402, 402);
    const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
    v[3] = pt / gm1 + kin / v[0];
    if (splitmix(s) & 1) v[3] = nudge(s, v[3]);
    const bool dxy_box = pos_in_box(dx) && pos_in_box(dy);
    double e1, r1, e2, r2;
    bool oke1 = true, okr1 = true, rok1, oke2 = true, okr2 = true, rok2;
    cell_epilogue(v, C, e1, oke1, r1, rok1, okr1);
    cell_epilogue_box(v, C, dxy_box, e2, oke2, r2, rok2, okr2);
    if (!(rok2 && okr2)) continue;
    c[0] += 1;
    if (!rok1 || !okr1) c[1] += 1;
    if (!same(r1, r2) || !same(e1, e2) || oke1 != oke2) c[2] += 1;
  }
  for (int k = 0; k < 3; ++k) atomicAdd(&out[k], c[k]);
}

}  // namespace

}  // namespace lfb

extern "C" int lf_selftest_epilogue(int64_t n, uint64_t seed, int64_t* counts) {
  if (!counts || n < 0) return LF_ERR_ARGUMENT;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 4 * sizeof(unsigned long long)) != cudaSuccess) return LF_ERR_DEVICE;
  cudaMemset(d, 0, 4 * sizeof(unsigned long long));
  lfb::count_launch();
  lfb::k_selftest_epilogue<<<148 * 8, 256>>>((long long)n, (unsigned long long)seed, d);
  unsigned long long h[4];
  const cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return LF_ERR_DEVICE;
  for (int k = 0; k < 3; ++k) counts[k] = (int64_t)h[k];
  return LF_OK;
}

extern "C" int lf_selftest_box(int64_t n, uint64_t seed, int64_t* counts) {
  if (!counts || n < 0) return LF_ERR_ARGUMENT;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 4 * sizeof(unsigned long long)) != cudaSuccess) return LF_ERR_DEVICE;
  cudaMemset(d, 0, 4 * sizeof(unsigned long long));
  lfb::count_launch();
  lfb::k_selftest_box<<<148 * 8, 256>>>((long long)n, (unsigned long long)seed, d);
  unsigned long long h[4];
  const cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return LF_ERR_DEVICE;
  for (int k = 0; k < 2; ++k) counts[k] = (int64_t)h[k];
  return LF_OK;
}

extern "C" int lf_selftest_fastmath(int64_t n, uint64_t seed, int64_t* counts) {
  if (!counts || n < 0) return LF_ERR_ARGUMENT;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 10 * sizeof(unsigned long long)) != cudaSuccess) return LF_ERR_DEVICE;
  cudaMemset(d, 0, 10 * sizeof(unsigned long long));
  lfb::count_launch();
  lfb::k_selftest<<<148 * 8, 256>>>((long long)n, (unsigned long long)seed, d);
  unsigned long long h[10];
  const cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return LF_ERR_DEVICE;
  for (int k = 0; k < 10; ++k) counts[k] = (int64_t)h[k];
  return LF_OK;
}
