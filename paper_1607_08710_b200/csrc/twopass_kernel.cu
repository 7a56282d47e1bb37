// twopass_kernel.cu -- the Heun step as two warp-independent streaming passes.
//
//   predictor  U^n (ghost-filled) -> U*, F^n x-faces, F^n y-faces
//   corrector  U*  (ghost-filled), U^n, F^n -> U^{n+1}, min rho / min e_int,
//              CFL rate of U^{n+1}, boundary-face fluxes, failure flags
//
// This is the reference's own stage structure (solver.cpp:496-509: ghost fill,
// build_primitives, compute_fluxes, apply_update, twice) with each stage fused
// into one kernel.  Every warp owns a strip of 32 columns (28 output columns and
// a 2-column halo each side) and marches down a chunk of rows on its own: the
// y-direction stencil lives in a rolling 3-row register window of the lane that
// owns the column (slopes shared by the two y-faces of a cell), x-neighbours
// come from warp shuffles.  There is no block-level synchronisation at all, so
// the scheduler is free to interleave warps; the U^n / U* row of the next
// iteration is loaded one iteration ahead.
//
// Compared with the one-kernel step (fused_kernel.cu) this moves 288 B per
// cell-update instead of 64 B, whose HBM ceiling (22.7 G cell-updates/s at the
// measured 6.5 TB/s) is far above the fp64 issue rate either design achieves;
// it wins because it keeps every SM issuing instead of waiting at barriers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/lagflux_b200.h"
#include "face_fast.cuh"
#include "fused_common.cuh"
#include "kernels.h"
#include "twopass.h"
#include "pdl.cuh"

#if LF_CONTRACT
#define k_pass k_pass_contract   // distinct kernel names in launch lists and ncu filters
#endif

namespace lfb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LANES = 32;
constexpr int TXW = LANES - 4;  // output columns per warp strip

__device__ __forceinline__ double key_to_double(unsigned long long b) {
  return __longlong_as_double((long long)b);
}

template <int N>
__device__ __forceinline__ void shfl_up4(const double (&v)[N], double (&o)[N], int d) {
#pragma unroll
  for (int q = 0; q < N; ++q) o[q] = __shfl_up_sync(FULL, v[q], d);
}
template <int N>
__device__ __forceinline__ void shfl_down4(const double (&v)[N], double (&o)[N], int d) {
#pragma unroll
  for (int q = 0; q < N; ++q) o[q] = __shfl_down_sync(FULL, v[q], d);
}

// Build-time tuning knobs (tools/variants.py sweeps them):
//   LF_TP_MINBLOCKS  resident blocks per SM requested from ptxas (register budget)
//   (measured and dropped: update operands loaded after the face solves; the row
//   loop unrolled twice, -15 %; operands staged one row ahead in shared memory with
//   cp.async, -1 % here -- the loads are covered at 12 warps/SM -- but +20-32 % in
//   the 8-warp material kernel, which keeps it)
#ifndef LF_TP_MINBLOCKS
#define LF_TP_MINBLOCKS 3
#endif
#ifndef LF_EPI_BOX
#define LF_EPI_BOX 1
#endif
#ifndef LF_TP_EDGE1
#define LF_TP_EDGE1 1
#endif

// EXACT = false: the plain fast path; a warp whose stencil rows hold a velocity
// in (0, 2^-500) (shock precursors) does not compute with it but raises the
// "needs exact" flag (StepAcc::fail = 2) and the host re-runs the step with
// EXACT = true, which takes the exact u* quotient in such warps.
template <bool CORR, bool MUSCL, bool EXACT>
__global__ void __launch_bounds__(TP_THREADS, LF_TP_MINBLOCKS) k_pass(PassArgs a) {
  pdl_wait();  // the previous kernel of the step chain (pdl.cuh)
  const StepCtl ctl = *a.ctl;
  if (ctl.done) return;
  if (ctl.dtfail) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  // dt exactly as compute_dt (solver.cpp:476-477) and apply_update (:262-263)
  const double rate = key_to_double(ctl.rate_bits);
  double dt = a.cfl / rate;
  if (ctl.time + dt > a.limit) dt = a.limit - ctl.time;
  if (!(dt > 0.0)) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  const double lam_x = dt / a.dx;
  const double lam_y = dt / a.dy;
  const FK C = make_fk(a.gamma, a.gm1, a.beta, a.dx, a.dy);
#if LF_EPI_BOX
  const bool dxy_box = pos_in_box(a.dx) && pos_in_box(a.dy);
#endif

  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * (TP_THREADS / 32) + (threadIdx.x >> 5);
  const int strip = warp % a.strips;
  const int chunk = warp / a.strips;
  const int y0 = chunk * a.rows_per_chunk;
  if (y0 >= a.ny) return;  // whole warp
  const int y1 = min(y0 + a.rows_per_chunk, a.ny);
  const int x0 = strip * TXW;
  const int c = x0 - 2 + lane;
  const bool col_in_mem = c >= -NG && c < a.nx + NG;
  const bool col_interior = c >= 0 && c < a.nx;
  const bool upd = lane >= 2 && lane <= LANES - 3 && col_interior;   // owns an output cell
  // x-face (lane-1 | lane) is stored by lanes 2..29 (faces x0 .. x0+27), plus
  // the domain's last face nx by whichever lane holds column nx
  const bool store_fx = (lane >= 2 && lane <= LANES - 3 && c <= a.nx) || (lane == LANES - 2 && c == a.nx);
  const int nit = (y1 - y0) + 4;
#if LF_TP_EDGE1
  // this warp's strip holds the domain's first or last column
  const bool x_edge_warp = x0 - 2 <= 0 || x0 - 2 + LANES > a.nx - 1;
#endif

  unsigned fail = const_in_box(a.gamma, a.gm1) ? 0u : 1u;
  unsigned need_exact = 0;
  unsigned long long rate_key = 0ull, nmin_r = NINF_KEY, nmin_e = NINF_KEY;
  unsigned dtfail = 0;

  // element offsets of (row, column c) from the origin pointers fit in 32 bits
  // (launch_pass checks); one running offset serves every array
  const int P = (int)a.pitch;
  int o_in = (y0 - 2) * P + c;   // offset of this iteration's input row r
  double nxt[4] = {1.0, 0.0, 0.0, 1.0};
  if (col_in_mem) {
#pragma unroll
    for (int q = 0; q < 4; ++q) nxt[q] = __ldg(a.x + q * a.fstride + o_in);
  }
  double wm2[4] = {1.0, 0.0, 0.0, 1.0}, wm1[4] = {1.0, 0.0, 0.0, 1.0};
  double hiprev[4] = {1.0, 0.0, 0.0, 1.0}, fyprev[4] = {0.0, 0.0, 0.0, 0.0};
  // rows r-3 .. r-1 of this lane with a velocity in (0, 2^-500), one bit per row
  unsigned tiny_rows = 0;

  for (int it = 0; it < nit; ++it) {
    const int r = y0 - 2 + it;   // input row
    const int row = r - 2;       // row updated this iteration (when it >= 4)
    double cur[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    const int o_row = o_in - 2 * P;   // row r-2 (updated this iteration)
    o_in += P;                        // row r+1
    if (it + 1 < nit && col_in_mem) {
#pragma unroll
      for (int q = 0; q < 4; ++q) nxt[q] = __ldg(a.x + q * a.fstride + o_in);
    }
    // operands of this iteration's update (issued early unless LF_TP_LATELOAD)
    double base[4] = {0.0, 0.0, 0.0, 0.0}, fnx[4] = {0.0, 0.0, 0.0, 0.0}, fny[4] = {0.0, 0.0, 0.0, 0.0};
    auto load_operands = [&]() {
    if (it >= 4 && col_in_mem) {
#pragma unroll
      for (int q = 0; q < 4; ++q) base[q] = __ldg(a.base + q * a.fstride + o_row);
      if (CORR && a.heun && c >= 0 && c <= a.nx) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fnx[q] = __ldg(a.fx + q * a.fx_stride + o_row);
      }
    }
    if (CORR && a.heun && it >= 3 && col_interior) {
      // face (row | row+1); at it == 3 this is the chunk's first face (y0-1 | y0)
#pragma unroll
      for (int q = 0; q < 4; ++q) fny[q] = __ldg(a.fy + q * a.fy_stride + (o_row + P));
    }
    };
    load_operands();
    // -- W(r) (solver.cpp:145-163)
    double w[4] = {1.0, 0.0, 0.0, 1.0};
    if (col_in_mem) {
      bool okw = true;  // implied by the box
      prim_fast(cur[0], cur[1], cur[2], cur[3], a.gm1, w, okw);
      if (!cell_in_box(w) && col_interior && r >= 0 && r < a.ny) fail = 1;
    }
    // the faces of this iteration read W rows r-3 .. r of lanes l-2 .. l+1: the
    // exact kernels keep that window per warp; the plain ones only note any
    // precursor velocity at all and flag the step once, at the end
    bool tiny = false;
    if (EXACT) {
      tiny_rows = ((tiny_rows << 1) | (unsigned)(vel_tiny(w[1]) || vel_tiny(w[2]))) & 0xfu;
      tiny = __any_sync(FULL, tiny_rows != 0u);
    } else {
      // the contract arithmetic multiplies by reciprocals: tiny dividends need nothing
      if (!LF_CONTRACT) need_exact |= (unsigned)(vel_tiny(w[1]) || vel_tiny(w[2]));
    }
    // -- y: traces of row r-1, face (r-2 | r-1); x: traces of row r-2 (shuffles)
    double ylo[4], yhi[4], xlo[4], xhi[4], xp[4], da[4], db[4];
    shfl_down4(wm2, xp, 1);
#pragma unroll
    for (int q = 0; q < 4; ++q) da[q] = xp[q] - wm2[q];  // q(t+1) - q(t)
    shfl_up4(da, db, 1);                                 // q(t) - q(t-1), lane t-1's a
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cell_traces<MUSCL>(wm2[q], wm1[q], w[q], a.beta, ylo[q], yhi[q]);
      traces_ab<MUSCL>(da[q], db[q], wm2[q], a.beta, xlo[q], xhi[q]);
    }
    double xmh[4];
    shfl_up4(xhi, xmh, 1);  // minus-side trace of x-face (lane-1 | lane)
    double fx[4], fy[4];
    bool okx = true, oky = true;  // implied by the cell box (face_fast.cuh): unused
    const bool need_x = it >= 4 && lane >= 2 && lane <= LANES - 2 && c <= a.nx;
    const bool need_y = it >= 3 && lane >= 2 && lane <= LANES - 3 && col_interior;
    double psx, usx, psy, usy;
    if (EXACT && tiny) {
      // a velocity in (0, 2^-500) in this warp's stencil rows (numerical
      // precursors ahead of a shock): the exact u* quotient (div_exact)
      face_fast<0, true>(xmh[0], xmh[1], xmh[2], xmh[3], xlo[0], xlo[1], xlo[2], xlo[3], C, fx,
                         okx, psx, usx);
      face_fast<1, true>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2],
                         ylo[3], C, fy, oky, psy, usy);
      if ((need_x && !okx) || (need_y && !oky)) fail = 1;  // div_exact out of range
    } else {
      face_fast<0, false>(xmh[0], xmh[1], xmh[2], xmh[3], xlo[0], xlo[1], xlo[2], xlo[3], C, fx,
                          okx, psx, usx);
      face_fast<1, false>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2],
                          ylo[3], C, fy, oky, psy, usy);
    }
    if (needs_mean(usx))
      face_mean<0>(xmh[0], xmh[1], xmh[2], xmh[3], xlo[0], xlo[1], xlo[2], xlo[3], psx, usx, C,
                   fx, okx);
    if (needs_mean(usy))
      face_mean<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2], ylo[3],
                   psy, usy, C, fy, oky);
    if (need_x && !traces_ok(xmh[0], xmh[3], xlo[0], xlo[3]) && c >= 0 && row >= 0 && row < a.ny)
      fail = 1;
    if (need_y && !traces_ok(hiprev[0], hiprev[3], ylo[0], ylo[3]) && r - 1 >= 0 && r - 1 <= a.ny)
      fail = 1;
    if (CORR && a.heun) {
      // Heun average 0.5 (F^n + F*) per face (solver.cpp:284-289)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fx[q] = 0.5 * (fnx[q] + fx[q]);
        fy[q] = 0.5 * (fny[q] + fy[q]);
      }
    }
    double fxr[4];
    shfl_down4(fx, fxr, 1);  // x-face (lane | lane+1)
    if (it >= 4) {
      if (!CORR) {
        // F^n faces for the corrector
        if (store_fx)
#pragma unroll
          for (int q = 0; q < 4; ++q) a.fxo[q * a.fx_stride + o_row] = fx[q];
        if (upd)
#pragma unroll
          for (int q = 0; q < 4; ++q) a.fyo[q * a.fy_stride + (o_row + P)] = fy[q];
      }
      if (upd) {
        // solver.cpp:283-291
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double val = base[q] - lam_x * (fxr[q] - fx[q]);
          val -= lam_y * (fy[q] - fyprev[q]);
          v[q] = val;
          a.out[q * a.fstride + o_row] = val;
        }
        if (!CORR) {
          // e_int > 0 without the division (conservative, see fused_kernel.cu)
          const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
          const double lhs = v[3] * v[0];
          if (!(v[0] > 0.0) || !(lhs > kin * (1.0 + 0x1p-48)) || !(lhs >= 0x1p-960)) fail = 1;
        } else {
          bool ok = true, okr = true, rate_ok;
          double eint, rr;
#if LF_EPI_BOX
          cell_epilogue_box<EXACT>(v, C, dxy_box, eint, ok, rr, rate_ok, okr);
#else
          cell_epilogue(v, C, eint, ok, rr, rate_ok, okr);
#endif
          if (!(v[0] > 0.0) || !(eint > 0.0) || !ok) {
            fail = 1;
          } else {
            const unsigned long long kr = ~pos_bits(v[0]), ke = ~pos_bits(eint);
            nmin_r = kr > nmin_r ? kr : nmin_r;
            nmin_e = ke > nmin_e ? ke : nmin_e;
          }
          if (rate_ok) {
            if (rr == rr) {
              const unsigned long long b = pos_bits(rr);
              rate_key = b > rate_key ? b : rate_key;
            }
            if (!okr) fail = 1;
          } else {
            dtfail = 1;
          }
          // domain-boundary faces for accumulate_boundary_outflow (solver.cpp:406-432);
          // one warp-uniform test skips all four in the interior of the domain
          const int jg = row + a.y0g;
#if LF_TP_EDGE1
          if (x_edge_warp || jg == 0 || jg == a.nyg - 1) {
#endif
          if (c == 0)
            for (int q = 0; q < 4; ++q) a.bnd[(int64_t)q * a.nyg + jg] = fx[q];
          if (c == a.nx - 1)
            for (int q = 0; q < 4; ++q) a.bnd[4 * (int64_t)a.nyg + (int64_t)q * a.nyg + jg] = fxr[q];
          if (jg == 0)
            for (int q = 0; q < 4; ++q) a.bnd[8 * (int64_t)a.nyg + (int64_t)q * a.nx + c] = fyprev[q];
          if (jg == a.nyg - 1)
            for (int q = 0; q < 4; ++q)
              a.bnd[8 * (int64_t)a.nyg + 4 * (int64_t)a.nx + (int64_t)q * a.nx + c] = fy[q];
#if LF_TP_EDGE1
          }
#endif
        }
      }
    } else if (!CORR && it == 3 && y0 == 0 && upd) {
      // the domain's first y-face (-1 | 0) belongs to no updated row of a chunk
      // other than the bottom one
#pragma unroll
      for (int q = 0; q < 4; ++q) a.fyo[q * a.fy_stride + c] = fy[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      fyprev[q] = fy[q];
      hiprev[q] = yhi[q];
      wm2[q] = wm1[q];
      wm1[q] = w[q];
    }
  }
  // warp reductions, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long r2 = __shfl_xor_sync(FULL, rate_key, o);
    const unsigned long long a2 = __shfl_xor_sync(FULL, nmin_r, o);
    const unsigned long long b2 = __shfl_xor_sync(FULL, nmin_e, o);
    rate_key = r2 > rate_key ? r2 : rate_key;
    nmin_r = a2 > nmin_r ? a2 : nmin_r;
    nmin_e = b2 > nmin_e ? b2 : nmin_e;
  }
  const unsigned anyfail = __any_sync(FULL, fail);
  dtfail = __any_sync(FULL, dtfail);
  need_exact = __any_sync(FULL, need_exact);
  if (lane == 0) {
    if (anyfail) atomicMax(&a.acc->fail, 1ull);
    if (need_exact) atomicMax(&a.acc->fail, 2ull);   // dominates: the exact re-run decides
    if (CORR) {
      if (rate_key) atomicMax(&a.acc->rate_next, rate_key);
      if (nmin_r != NINF_KEY) atomicMax(&a.acc->nmin_rho, nmin_r);
      if (nmin_e != NINF_KEY) atomicMax(&a.acc->nmin_eint, nmin_e);
      if (dtfail) atomicMax(&a.acc->dtfail_next, 1ull);
    }
  }
}

}  // namespace

#if LF_CONTRACT
// twopass_contract.cu: the same kernels in the tolerance arithmetic (fastmath.cuh)
void launch_pass_contract(const PassArgs& a, bool corr, bool muscl, cudaStream_t st) {
  const int warps = a.strips * ((a.ny + a.rows_per_chunk - 1) / a.rows_per_chunk);
  const unsigned blocks = (unsigned)((warps + TP_THREADS / 32 - 1) / (TP_THREADS / 32));
  count_launch();
  if (corr) {
    if (muscl)
      launch_chain(k_pass<true, true, false>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
    else
      launch_chain(k_pass<true, false, false>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
  } else {
    if (muscl)
      launch_chain(k_pass<false, true, false>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
    else
      launch_chain(k_pass<false, false, false>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
  }
}
#else
int tp_strips(int nx) { return (nx + TXW - 1) / TXW; }

int tp_resident_warps(int nmat) {
  if (nmat > 0) return tp_resident_warps_mat(nmat);
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pass<true, true, false>, TP_THREADS, 0) !=
          cudaSuccess ||
      b < 1)
    b = LF_TP_MINBLOCKS;
  return b * (TP_THREADS / 32);
}

// Each warp marches one strip over one chunk of rows (plus ~4 rows of stencil
// fill); the warps are independent, so the cost is about (waves) x (rows + fill)
// where a wave is one warp per resident slot.  Chunk counts are chosen so the
// warps fill whole waves (measured: 16384^2 at 13 chunks = 4.3 waves runs 4 %
// slower than 12 chunks = 3.96 waves; 1024^2 at 22 rows = 0.98 wave 7.1 G/s,
// 20 rows = 1.08 waves 5.5 G/s).  Four waves when the marches stay long (the
// tail of a wave is the last warps' finish), else the cheapest of 1-3 waves.
int tp_choose_rows(int nx, int ny, int sms, int warps_per_sm) {
  const int64_t strips = tp_strips(nx), cap = (int64_t)sms * warps_per_sm;
  auto rows_for = [&](int64_t k) {
    const int64_t chunks = std::max<int64_t>(1, k * cap / strips);
    return (int)std::max<int64_t>((ny + chunks - 1) / chunks, 16);
  };
  const int r4 = rows_for(4);
  if (r4 >= 64) return r4;
  int best = r4;
  int64_t best_cost = INT64_MAX;
  for (int k = 1; k <= 4; ++k) {
    const int r = rows_for(k);
    const int64_t warps = strips * ((ny + r - 1) / r);
    const int64_t cost = ((warps + cap - 1) / cap) * (r + 8);
    if (cost < best_cost) {
      best_cost = cost;
      best = r;
    }
  }
  return best;
}

bool tp_fits(int64_t pitch, int ny) {
  // k_pass addresses (row, column) with 32-bit element offsets, rows -NG .. ny+NG
  return pitch * (int64_t)(ny + NG + 1) < (int64_t)1 << 31;
}

template <bool EXACT>
static void launch_k(const PassArgs& a, bool corr, bool muscl, unsigned blocks, cudaStream_t st) {
  if (corr) {
    if (muscl)
      launch_chain(k_pass<true, true, EXACT>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
    else
      launch_chain(k_pass<true, false, EXACT>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
  } else {
    if (muscl)
      launch_chain(k_pass<false, true, EXACT>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
    else
      launch_chain(k_pass<false, false, EXACT>, dim3(blocks), dim3(TP_THREADS), 0, st, a);
  }
}

void launch_pass(const PassArgs& a, bool corr, bool muscl, bool exact, cudaStream_t st) {
  const int warps = a.strips * ((a.ny + a.rows_per_chunk - 1) / a.rows_per_chunk);
  const unsigned blocks = (unsigned)((warps + TP_THREADS / 32 - 1) / (TP_THREADS / 32));
  count_launch();
  if (exact)
    launch_k<true>(a, corr, muscl, blocks, st);
  else
    launch_k<false>(a, corr, muscl, blocks, st);
}
#endif  // LF_CONTRACT

}  // namespace lfb
