// stage_kernels.cu -- the stage-wise kernels: one per reference loop.
//
// These mirror LagfluxSolver's phase structure exactly (solver.cpp:131-329)
// so they also reproduce its failure semantics (smallest failing index per
// check, checks in the reference order).  They serve euler_stage,
// time_order = 1, the per-stage diagnosis of a failed fused step, and the
// stage-wise Heun path.  The fast Heun step is fused_step.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>

#include "kernels.h"
#include "pdl.cuh"
#include "reduce.cuh"

namespace lfb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ long long warp_min_i64(long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    long long w = __shfl_xor_sync(FULL, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// ---------------------------------------------------------------- ghost fill
// grid.cpp:81-96: x sides over interior rows; each thread owns one
// (component, row) and runs the reference's sequential l loop (l = 1..NG, the
// first two layers are exactly the reference's, layers 3-4 extend the rule).
__global__ void k_fill_x(Field f, int nx, int ny, int bc_lo, int bc_hi, int odd_x) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (j >= ny) return;
  const double sx = c == odd_x ? -1.0 : 1.0;
  double* row = f.comp(c) + (int64_t)j * f.pitch;
  for (int l = 1; l <= NG; ++l) {
    const int lo = -l;
    const int hi = nx - 1 + l;
    switch (bc_lo) {
      case 0: row[lo] = row[0]; break;
      case 1: row[lo] = sx * row[l - 1]; break;
      default: row[lo] = row[((nx - l) % nx + nx) % nx]; break;
    }
    switch (bc_hi) {
      case 0: row[hi] = row[nx - 1]; break;
      case 1: row[hi] = sx * row[nx - l]; break;
      default: row[hi] = row[(l - 1) % nx]; break;
    }
  }
}

// grid.cpp:98-113: y sides over every column (corners pick up the x ghosts).
__global__ void k_fill_y(Field f, int nx, int ny, int bc_lo, int bc_hi, int do_lo, int do_hi,
                         int odd_y) {
  const int i = (int)(blockIdx.x * blockDim.x + threadIdx.x) - NG;
  const int c = blockIdx.y;
  if (i >= nx + NG) return;
  const double sy = c == odd_y ? -1.0 : 1.0;
  double* col = f.comp(c) + i;
  const int64_t P = f.pitch;
  for (int l = 1; l <= NG; ++l) {
    const int lo = -l;
    const int hi = ny - 1 + l;
    if (do_lo) {
      switch (bc_lo) {
        case 0: col[lo * P] = col[0]; break;
        case 1: col[lo * P] = sy * col[(int64_t)(l - 1) * P]; break;
        default: col[lo * P] = col[(int64_t)(((ny - l) % ny + ny) % ny) * P]; break;
      }
    }
    if (do_hi) {
      switch (bc_hi) {
        case 0: col[(int64_t)hi * P] = col[(int64_t)(ny - 1) * P]; break;
        case 1: col[(int64_t)hi * P] = sy * col[(int64_t)(ny - l) * P]; break;
        default: col[(int64_t)hi * P] = col[(int64_t)((l - 1) % ny) * P]; break;
      }
    }
  }
}

// Both sides in one launch (nx >= NG and, in 2D, ny >= NG: every source is an
// interior cell).  x ghosts of the interior rows as k_fill_x; the y ghost rows
// as k_fill_y, where a corner -- k_fill_y's copy of an x ghost -- is recomposed
// from the interior cell both rules point at, with the same multiplications
// (a reflective side multiplies by +-1: exact, so the composition is the
// sequential x-then-y fill bit for bit).  Threads own disjoint ghost cells and
// read interior cells only.
// Components c >= n1 are those of a second field f2 (the partial densities,
// even parity), so a multimaterial state fills in one launch.
__global__ void k_fill_xy(Field f, Field f2, int n1, int nx, int ny, int bx_lo, int bx_hi,
                          int by_lo, int by_hi, int do_lo, int do_hi, int odd_x, int odd_y) {
  pdl_wait();
  const int c = blockIdx.y;
  const double sx = c == odd_x ? -1.0 : 1.0, sy = c == odd_y ? -1.0 : 1.0;
  double* base = c < n1 ? f.comp(c) : f2.comp(c - n1);
  const int64_t P = f.pitch;
  const int t = (int)(blockIdx.x * blockDim.x + threadIdx.x);
  // column i of a row after the x fill
  auto xval = [&](const double* row, int i) -> double {
    if (i >= 0 && i < nx) return row[i];
    const bool lo = i < 0;
    const int l = lo ? -i : i - nx + 1;
    switch (lo ? bx_lo : bx_hi) {
      case 0: return row[lo ? 0 : nx - 1];
      case 1: return sx * row[lo ? l - 1 : nx - l];
      default: return row[lo ? ((nx - l) % nx + nx) % nx : (l - 1) % nx];
    }
  };
  if (t < 2 * ny) {  // x sides: (row, side)
    double* row = base + (int64_t)(t >> 1) * P;
    const bool lo = (t & 1) == 0;
    for (int l = 1; l <= NG; ++l) {
      const int i = lo ? -l : nx - 1 + l;
      row[i] = xval(row, i);
    }
    return;
  }
  const int u = t - 2 * ny;  // y sides: (column incl. x ghosts, side)
  if (u >= 2 * (nx + 2 * NG)) return;
  const int i = (u >> 1) - NG;
  const bool lo = (u & 1) == 0;
  if (lo ? !do_lo : !do_hi) return;
  const int b = lo ? by_lo : by_hi;
  for (int l = 1; l <= NG; ++l) {
    const int jd = lo ? -l : ny - 1 + l;
    int js;
    switch (b) {
      case 0: js = lo ? 0 : ny - 1; break;
      case 1: js = lo ? l - 1 : ny - l; break;
      default: js = lo ? ((ny - l) % ny + ny) % ny : (l - 1) % ny;
    }
    const double v = xval(base + (int64_t)js * P, i);
    base[(int64_t)jd * P + i] = b == 1 ? sy * v : v;
  }
}

// ---------------------------------------------------------------- CFL rate
// solver.cpp:449-470: max over interior cells, exact (order independent).
template <bool DIM2>
__global__ void k_rate(Field u, int nx, int ny, int y0, Consts k, Scalars* s) {
  unsigned long long best = 0ull;  // bits of +0.0 == the reference's initial rate
  long long fail = LLONG_MAX;
  const int64_t n = (int64_t)nx * ny;
  for (int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < n;
       cc += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(cc % nx), j = (int)(cc / nx);
    const int64_t o = (int64_t)j * u.pitch + i;
    double rr;
    if (cfl_rate<DIM2>(u.p[o], u.p[u.fstride + o], u.p[2 * u.fstride + o],
                       u.p[3 * u.fstride + o], k, rr)) {
      // std::max(rate, rr) ignores a NaN rr; rr >= 0 otherwise
      if (rr == rr) {
        const unsigned long long b = pos_bits(rr);
        best = b > best ? b : best;
      }
    } else {
      const long long g = (long long)(j + y0) * nx + i;
      fail = g < fail ? g : fail;
    }
  }
  best = block_reduce(best, MaxOp(), 0ull);
  fail = block_reduce(fail, MinOp(), (long long)LLONG_MAX);
  if (threadIdx.x == 0) {
    if (best) atomicMax(&s->rate_bits, best);
    if (fail != LLONG_MAX) atomicMin(&s->fail_dt, fail);
  }
}

// ---------------------------------------------------------------- primitives
// solver.cpp:145-163 over the reference's ghosted cells (gx = 2, gy = 2 in 2D,
// 0 in 1D).  The failure index is the reference's ghosted linear index.
__global__ void k_prims(Field u, Field w, int nx, int ny, int gy_ref, Slab sl, double gm1,
                        Scalars* s) {
  const int i = (int)(blockIdx.x * blockDim.x + threadIdx.x) - 2;
  const int j = (int)(blockIdx.y * blockDim.y + threadIdx.y) - gy_ref;
  long long fail = LLONG_MAX;
  if (i < nx + 2 && j < ny + gy_ref) {
    const int64_t o = (int64_t)j * u.pitch + i;
    const double r = u.p[o];
    double uu = 0.0, vv = 0.0, pp = 0.0, rr = 0.0;
    bool bad;
    if (!(r > 0.0)) {
      bad = true;
    } else {
      rr = r;
      primitive(r, u.p[u.fstride + o], u.p[2 * u.fstride + o], u.p[3 * u.fstride + o], gm1, uu,
                vv, pp);
      bad = !(pp > 0.0);
    }
    w.p[o] = rr;
    w.p[w.fstride + o] = uu;
    w.p[2 * w.fstride + o] = vv;
    w.p[3 * w.fstride + o] = pp;
    // rows outside [0, ny) belong to a neighbouring slab unless this slab is
    // the domain edge there
    const bool owned = (j >= 0 || sl.fill_lo) && (j < ny || sl.fill_hi);
    if (bad && owned) {
      const int nxt = nx + 4;
      fail = (long long)(j + sl.y0 + gy_ref) * nxt + (i + 2);
    }
  }
  fail = warp_min_i64(fail);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && fail != LLONG_MAX)
    atomicMin(&s->fail_prim, fail);
}

// ---------------------------------------------------------------- face fluxes
// solver.cpp:196-239, one thread per face.  AXIS 0: face (a, b) between cells
// (a-1, b) and (a, b), a in [0, nx], b in [0, ny).  AXIS 1: face between
// (a, b-1) and (a, b), a in [0, nx), b in [0, ny].
template <int AXIS, bool MUSCL>
__global__ void k_flux(Field w, FluxArr fo, int nx, int ny, Slab sl, Consts k, Scalars* s) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y * blockDim.y + threadIdx.y;
  const int na = AXIS == 0 ? nx + 1 : nx;
  const int nb = AXIS == 0 ? ny : ny + 1;
  long long fail = LLONG_MAX;
  if (a < na && b < nb) {
    const int64_t st = AXIS == 0 ? 1 : w.pitch;
    const int64_t hi = (int64_t)b * w.pitch + a;
    const int64_t lo = hi - st;
    double wm[4], wp[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* q = w.p + c * w.fstride;
      if (MUSCL) {
        const double q0 = q[lo - st], q1 = q[lo], q2 = q[hi], q3 = q[hi + st];
        const double s1 = slope3(q0, q1, q2, k.beta);
        const double s2 = slope3(q1, q2, q3, k.beta);
        wm[c] = q1 + 0.5 * s1;
        wp[c] = q2 - 0.5 * s2;
      } else {
        wm[c] = q[lo];
        wp[c] = q[hi];
      }
    }
    double f[4] = {0.0, 0.0, 0.0, 0.0};
    if (traces_ok(wm[0], wm[3], wp[0], wp[3])) {
      face_flux<AXIS>(wm[0], wm[1], wm[2], wm[3], wp[0], wp[1], wp[2], wp[3], k, f);
    } else {
      const long long nex = (long long)(nx + 1) * sl.ny_global;
      fail = AXIS == 0 ? (long long)(b + sl.y0) * (nx + 1) + a
                       : nex + (long long)(b + sl.y0) * nx + a;
    }
    const int64_t fo_off = (int64_t)b * fo.pitch + a;
#pragma unroll
    for (int c = 0; c < 4; ++c) fo.p[c * fo.fstride + fo_off] = f[c];
  }
  fail = warp_min_i64(fail);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && fail != LLONG_MAX)
    atomicMin(&s->fail_trace, fail);
}

// ---------------------------------------------------------------- update
// solver.cpp:272-308.  TWO: Heun corrector with F = 0.5*(Fa + Fb).
template <bool TWO, bool DIM2>
__global__ void k_update(Field base, FluxArr fxa, FluxArr fya, FluxArr fxb, FluxArr fyb,
                         Field out, int nx, int ny, int y0, double lam_x, double lam_y,
                         Scalars* s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  long long fail = LLONG_MAX;
  unsigned long long mr = ~0ull, me = ~0ull;
  for (int j = blockIdx.y * blockDim.y + threadIdx.y; i < nx && j < ny;
       j += gridDim.y * blockDim.y) {
    const int64_t o = (int64_t)j * base.pitch + i;
    const int64_t ex = (int64_t)j * fxa.pitch + i;
    const int64_t ey = (int64_t)j * fya.pitch + i;
    double vals[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* ax = fxa.p + c * fxa.fstride;
      double fxl, fxr;
      if (TWO) {
        const double* bx = fxb.p + c * fxb.fstride;
        fxl = 0.5 * (ax[ex] + bx[ex]);
        fxr = 0.5 * (ax[ex + 1] + bx[ex + 1]);
      } else {
        fxl = ax[ex];
        fxr = ax[ex + 1];
      }
      double val = base.p[c * base.fstride + o] - lam_x * (fxr - fxl);
      if (DIM2) {
        const double* ay = fya.p + c * fya.fstride;
        double fyb_, fyt_;
        if (TWO) {
          const double* by = fyb.p + c * fyb.fstride;
          fyb_ = 0.5 * (ay[ey] + by[ey]);
          fyt_ = 0.5 * (ay[ey + fya.pitch] + by[ey + fyb.pitch]);
        } else {
          fyb_ = ay[ey];
          fyt_ = ay[ey + fya.pitch];
        }
        val -= lam_y * (fyt_ - fyb_);
      }
      vals[c] = val;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) out.p[c * out.fstride + o] = vals[c];
    const double eint = internal_energy(vals[0], vals[1], vals[2], vals[3]);
    if (!(vals[0] > 0.0) || !(eint > 0.0)) {
      const long long g = (long long)(j + y0) * nx + i;
      fail = g < fail ? g : fail;
    } else {
      const unsigned long long r = pos_bits(vals[0]), e = pos_bits(eint);
      mr = r < mr ? r : mr;
      me = e < me ? e : me;
    }
  }
  fail = block_reduce(fail, MinOp(), (long long)LLONG_MAX);
  mr = block_reduce(mr, MinOp(), ~0ull);
  me = block_reduce(me, MinOp(), ~0ull);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    if (fail != LLONG_MAX) atomicMin(&s->fail_update, fail);
    if (mr != ~0ull) atomicMin(&s->min_rho_bits, mr);
    if (me != ~0ull) atomicMin(&s->min_eint_bits, me);
  }
}

__global__ void k_gather_boundary(FluxArr fxa, FluxArr fya, FluxArr fxb, FluxArr fyb, int nx,
                                  int ny, int two, double* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (t < ny) {
    const int64_t l = c * fxa.fstride + (int64_t)t * fxa.pitch, r = l + nx;
    const int64_t lb = c * fxb.fstride + (int64_t)t * fxb.pitch, rb = lb + nx;
    out[(int64_t)c * ny + t] = two ? 0.5 * (fxa.p[l] + fxb.p[lb]) : fxa.p[l];
    out[4 * (int64_t)ny + (int64_t)c * ny + t] = two ? 0.5 * (fxa.p[r] + fxb.p[rb]) : fxa.p[r];
  }
  if (t < nx) {
    const int64_t b = c * fya.fstride + t, tp = b + (int64_t)ny * fya.pitch;
    const int64_t bb = c * fyb.fstride + t, tb = bb + (int64_t)ny * fyb.pitch;
    out[8 * (int64_t)ny + (int64_t)c * nx + t] = two ? 0.5 * (fya.p[b] + fyb.p[bb]) : fya.p[b];
    out[8 * (int64_t)ny + 4 * (int64_t)nx + (int64_t)c * nx + t] =
        two ? 0.5 * (fya.p[tp] + fyb.p[tb]) : fya.p[tp];
  }
}

__global__ void k_reset(Scalars* s) {
  s->rate_bits = 0ull;
  s->fail_dt = LLONG_MAX;
  s->fail_prim = LLONG_MAX;
  s->fail_trace = LLONG_MAX;
  s->fail_update = LLONG_MAX;
  s->min_rho_bits = 0x7ff0000000000000ull;   // +inf
  s->min_eint_bits = 0x7ff0000000000000ull;
  s->status = 0;
  s->fail_frac = LLONG_MAX;
  s->min_p_key = ~0ull;
}

// ---------------------------------------------------------------- Fourier IC
__global__ void k_fourier_raw(Field f, int nx, int ny, const double* __restrict__ tx,
                              const double* __restrict__ ty, const double* __restrict__ amp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  for (int k = 0; k < 4; ++k) {
    double s = 0.0;
    for (int m = 0; m < 8; ++m) {
      const double* x = tx + (int64_t)((k * 8 + m) * 2) * nx;
      const double* y = ty + (int64_t)((k * 8 + m) * 2) * ny;
      const double term = x[i] * y[ny + j] + x[nx + i] * y[j];
      s = s + amp[k * 8 + m] * term;
    }
    f.at(k, i, j) = s;
  }
}

__global__ void k_absmax(Field f, int nx, int ny, unsigned long long* out4) {
  const int c = blockIdx.y;
  unsigned long long best = 0ull;
  const int64_t n = (int64_t)nx * ny;
  for (int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < n;
       cc += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(f.at(c, (int)(cc % nx), (int)(cc / nx)));
    const unsigned long long b = pos_bits(v);
    best = b > best ? b : best;
  }
  best = warp_max_u64(best);
  if ((threadIdx.x & 31) == 0) atomicMax(&out4[c], best);
}

__global__ void k_fourier_finish(Field f, int nx, int ny, const unsigned long long* max4,
                                 double gamma) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const double M0 = __longlong_as_double((long long)max4[0]);
  const double M1 = __longlong_as_double((long long)max4[1]);
  const double M2 = __longlong_as_double((long long)max4[2]);
  const double M3 = __longlong_as_double((long long)max4[3]);
  const double rho = 1.0 + 0.2 * (f.at(0, i, j) / M0);
  const double u = 0.5 * (f.at(1, i, j) / M1);
  const double v = 0.5 * (f.at(2, i, j) / M2);
  const double p = 1.0 + 0.2 * (f.at(3, i, j) / M3);
  f.at(0, i, j) = rho;
  f.at(1, i, j) = rho * u;
  f.at(2, i, j) = rho * v;
  f.at(3, i, j) = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
long long launch_count() { return g_launches.load(); }

void reset_scalars(Scalars* s, cudaStream_t st) {
  count_launch(), k_reset<<<1, 1, 0, st>>>(s);
}

void launch_fill_x(const Field& f, const Layout& L, const int bc[4], cudaStream_t st, int ncomp,
                   int odd_x) {
  count_launch(), k_fill_x<<<dim3(cdiv(L.ny, 128), ncomp), 128, 0, st>>>(f, L.nx, L.ny, bc[0], bc[1], odd_x);
}

void launch_fill_xy(const Field& f, const Layout& L, const int bc[4], const Slab& sl, bool dim2,
                    cudaStream_t st, int ncomp, int odd_x, int odd_y, const Field* f2, int ncomp2) {
  const int threads = 2 * L.ny + 2 * (L.nx + 2 * NG);
  count_launch();
  launch_chain(k_fill_xy, dim3(cdiv(threads, 128), ncomp + (f2 ? ncomp2 : 0)), dim3(128), 0, st,
               f, f2 ? *f2 : f, ncomp, L.nx, L.ny, bc[0], bc[1], bc[2], bc[3],
               (int)(dim2 && sl.fill_lo), (int)(dim2 && sl.fill_hi), odd_x, odd_y);
}

void launch_fill_y_only(const Field& f, const Layout& L, const int bc[4], const Slab& sl,
                        cudaStream_t st, int ncomp, int odd_y) {
  count_launch(), k_fill_y<<<dim3(cdiv(L.nx + 2 * NG, 128), ncomp), 128, 0, st>>>(
      f, L.nx, L.ny, bc[2], bc[3], sl.fill_lo, sl.fill_hi, odd_y);
}

void launch_gather_boundary(const FluxArr& fxa, const FluxArr& fya, const FluxArr& fxb,
                            const FluxArr& fyb, const Layout& L, bool two, double* out,
                            cudaStream_t st) {
  const int n = std::max(L.nx, L.ny);
  count_launch(), k_gather_boundary<<<dim3(cdiv(n, 128), 4), 128, 0, st>>>(fxa, fya, fxb, fyb, L.nx, L.ny,
                                                           two ? 1 : 0, out);
}

void launch_rate(const Field& u, const Layout& L, const Slab& sl, const Consts& k, int dim2,
                 Scalars* s, cudaStream_t st) {
  const int64_t n = (int64_t)L.nx * L.ny;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  if (dim2)
    count_launch(), k_rate<true><<<blocks, 256, 0, st>>>(u, L.nx, L.ny, sl.y0, k, s);
  else
    count_launch(), k_rate<false><<<blocks, 256, 0, st>>>(u, L.nx, L.ny, sl.y0, k, s);
}

void launch_prims(const Field& u, const Field& w, const Layout& L, const Slab& sl, double gm1,
                  int dim2, Scalars* s, cudaStream_t st) {
  const int gy = dim2 ? 2 : 0;
  dim3 blk(32, 8);
  dim3 grd(cdiv(L.nx + 4, 32), cdiv(L.ny + 2 * gy, 8));
  count_launch(), k_prims<<<grd, blk, 0, st>>>(u, w, L.nx, L.ny, gy, sl, gm1, s);
}

void launch_fluxes(const Field& w, const FluxArr& fx, const FluxArr& fy, const Layout& L,
                   const Slab& sl, const Consts& k, int muscl, int dim2, Scalars* s,
                   cudaStream_t st) {
  dim3 blk(32, 4);
  dim3 gx(cdiv(L.nx + 1, 32), cdiv(L.ny, 4));
  if (muscl)
    count_launch(), k_flux<0, true><<<gx, blk, 0, st>>>(w, fx, L.nx, L.ny, sl, k, s);
  else
    count_launch(), k_flux<0, false><<<gx, blk, 0, st>>>(w, fx, L.nx, L.ny, sl, k, s);
  if (!dim2) return;
  dim3 gy(cdiv(L.nx, 32), cdiv(L.ny + 1, 4));
  if (muscl)
    count_launch(), k_flux<1, true><<<gy, blk, 0, st>>>(w, fy, L.nx, L.ny, sl, k, s);
  else
    count_launch(), k_flux<1, false><<<gy, blk, 0, st>>>(w, fy, L.nx, L.ny, sl, k, s);
}

void launch_update(const Field& base, const FluxArr& fxa, const FluxArr& fya,
                   const FluxArr* fxb, const FluxArr* fyb, const Field& out, const Layout& L,
                   const Slab& sl, double dt, double dx, double dy, int dim2, Scalars* s,
                   cudaStream_t st) {
  const double lam_x = dt / dx;  // solver.cpp:262-263 (divisions, not reciprocals)
  const double lam_y = dt / dy;
  dim3 blk(32, 8);
  // a few blocks per SM, each looping over rows (one atomic per block per scalar)
  const unsigned gx = cdiv(L.nx, 32);
  dim3 grd(gx, std::max(1u, std::min(cdiv(L.ny, 8), cdiv(148 * 8, gx))));
  const FluxArr xb = fxb ? *fxb : fxa, yb = fyb ? *fyb : fya;
  if (fxb) {
    if (dim2)
      count_launch(), k_update<true, true><<<grd, blk, 0, st>>>(base, fxa, fya, xb, yb, out, L.nx, L.ny, sl.y0, lam_x, lam_y, s);
    else
      count_launch(), k_update<true, false><<<grd, blk, 0, st>>>(base, fxa, fya, xb, yb, out, L.nx, L.ny, sl.y0, lam_x, lam_y, s);
  } else {
    if (dim2)
      count_launch(), k_update<false, true><<<grd, blk, 0, st>>>(base, fxa, fya, xb, yb, out, L.nx, L.ny, sl.y0, lam_x, lam_y, s);
    else
      count_launch(), k_update<false, false><<<grd, blk, 0, st>>>(base, fxa, fya, xb, yb, out, L.nx, L.ny, sl.y0, lam_x, lam_y, s);
  }
}

void launch_fourier_raw(const Field& f, const Layout& L, const double* tx, const double* ty,
                        const double* amp, cudaStream_t st) {
  dim3 blk(32, 8);
  count_launch(), k_fourier_raw<<<dim3(cdiv(L.nx, 32), cdiv(L.ny, 8)), blk, 0, st>>>(f, L.nx, L.ny, tx, ty, amp);
}

void launch_absmax(const Field& f, const Layout& L, unsigned long long* out4, cudaStream_t st) {
  const int64_t n = (int64_t)L.nx * L.ny;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  count_launch(), k_absmax<<<dim3(blocks, 4), 256, 0, st>>>(f, L.nx, L.ny, out4);
}

void launch_fourier_finish(const Field& f, const Layout& L, const unsigned long long* max4,
                           double gamma, cudaStream_t st) {
  dim3 blk(32, 8);
  count_launch(), k_fourier_finish<<<dim3(cdiv(L.nx, 32), cdiv(L.ny, 8)), blk, 0, st>>>(f, L.nx, L.ny, max4, gamma);
}

}  // namespace lfb
