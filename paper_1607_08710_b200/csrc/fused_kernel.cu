// fused_kernel.cu -- one kernel per Heun time step (LagfluxSolver::heun_step, solver.cpp:489-546).
//
// Design ("Fused one-kernel"):
//  * A block owns a strip of NC = 128 columns (TXO = 120 output columns plus a
//    4-column halo each side) and marches down a chunk of rows.  The whole step
//    -- primitives, MUSCL traces, Lagrangian HLL, upwind fluxes, predictor U*,
//    corrector U^{n+1}, positivity checks, min rho / min e_int and the CFL rate
//    of U^{n+1} for the next dt -- happens in one pass: U^n is read from HBM
//    about once (plus ~7% halo re-reads, mostly L2 hits) and U^{n+1} written once,
//    64 B/cell-update of compulsory traffic instead of the stage-wise 288 B.
//  * Warp specialisation: warps 0-3 ("P") run stage 1 on input row r (U^n ->
//    F^n faces -> U*(r-2)); warps 4-7 ("C") run stage 2 three rows behind
//    (U*(a) -> F* faces -> U^{n+1}(a-2)).  P and C exchange rows through small
//    shared-memory rings; each group synchronises internally on its own named
//    barrier and both meet once per row iteration.
//  * y-direction stencil data of a column lives in the registers of the thread
//    owning that column (rolling 3-row window, slopes shared between the two
//    faces of a cell); x-direction neighbours go through shared memory.  Each
//    thread solves its x-face and its y-face Riemann problems in one straight
//    line of code, so the two dependency chains overlap.
//  * Round 2: the row loop runs a guarded
//    body for the pipeline fill / drain and the domain's y edges and a guard-free
//    steady body in between (the same source, a compile-time flag); the corrector
//    takes the x slopes of W*(j) straight from the P -> C ring (LF_FUSED_CRING,
//    exact build); the step constants arrive as launch parameters; the four P warps
//    share the TMA issue.  The kernel is fp64 / issue bound: 1566 instructions per
//    cell-update, 645 of them fp64, 4 warps per scheduler at 128 registers.
//  * fp64 arithmetic keeps the reference's evaluation order (--fmad=false);
//    divisions and square roots use fastmath.cuh (the compiler's own IEEE fast
//    path with shared reciprocals and one deferred range check per face), so
//    results are bit-identical to the reference.
//  * Failure checks are detection only: any flag makes the host re-run that
//    step with the stage-wise kernels, which reproduce the reference's exact
//    error (kind, smallest index, text) and state semantics.
#include <cuda_runtime.h>

#include <type_traits>

#include "../../include/lagflux_b200.h"
#include "fastmath.cuh"
#include "fused_common.cuh"
#include "pdl.cuh"
#include "kernels.h"
#include "face_fast.cuh"
#include "lagflux_device.cuh"

// Build-time tuning knobs (tools/variants.py sweeps them):
//   LF_MINBLOCKS  resident blocks per SM requested from ptxas (register budget)

#if LF_CONTRACT
#define k_fused_step k_fused_step_contract   // distinct kernel names for ncu filters
#define k_make_fk k_make_fk_contract
#endif

namespace lfb {

namespace {

constexpr int NC = FUSED_NC;
constexpr int TXO = FUSED_TXO;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ void bar_named(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NC) : "memory");
}

__device__ __forceinline__ double key_to_double(unsigned long long b) {
  return __longlong_as_double((long long)b);
}

// ---------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LF_WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// one contiguous row segment global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes,
                                        unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

constexpr int URING = 8;   // U^n rows resident in shared memory (r-5 .. r+2)
constexpr int PREFETCH = 2;

// LF_FUSED_EPI_BOX 1/2: the corrector epilogue's rate checks proved by the cell box
// (face_fast.cuh), the e_int quotient inline (1) or out of line (2)
// (measured at 16384^2: box 1 +2.2 % in the exact arithmetic, -1.2 % in the contract one)
#ifndef LF_FUSED_EPI_BOX
#if LF_CONTRACT
#define LF_FUSED_EPI_BOX 0
#else
#define LF_FUSED_EPI_BOX 1
#endif
#endif
// LF_FUSED_DONTCARE_P: the same for the predictor's x-face operands (measured at
// 16384^2: +0.6 % exact, -1.2 % contract)
#ifndef LF_FUSED_DONTCARE_P
#if LF_CONTRACT
#define LF_FUSED_DONTCARE_P 0
#else
#define LF_FUSED_DONTCARE_P 1
#endif
#endif
#ifndef LF_MINBLOCKS
#define LF_MINBLOCKS (256 / FUSED_NC)
#endif
// LF_FUSED_TMA_SPREAD 1: the four component rows of each U^n row are copied by the
// four P warps (one each) instead of all by warp 0
// (measured: +1.1 % exact; in the contract build -1.5 % with the maxima in registers,
// +2.8 % with LF_FUSED_KEYSMEM)
#ifndef LF_FUSED_TMA_SPREAD
#define LF_FUSED_TMA_SPREAD 1
#endif
// LF_FUSED_CRING 1: C takes the x slopes of W*(j) straight from the P -> C ring (each
// lane's image column) instead of exchanging its W*(j) row through shared memory and a
// barrier.  Measured at 16384^2 (tools/variants.py): +5.5 % exact, -6 % in the contract
// build (register pressure: spills), which keeps the exchange.  (Also measured and
// dropped: the same for P's W rows, a 4-row ring: +-0.5 % exact, -23 % contract, whose
// shared memory then admits one block per SM; the y windows read back from the rings
// instead of rotated in registers: -4 %; the steady loop unrolled twice: -12 %,
// instruction cache.)
#ifndef LF_FUSED_CRING
#if LF_CONTRACT
#define LF_FUSED_CRING 0
#else
#define LF_FUSED_CRING 1
#endif
#endif
constexpr int WC_ROWS = LF_FUSED_CRING ? 0 : 1;

// LF_FUSED_KEYSMEM 1: the corrector's running maxima (CFL rate, ~min rho, ~min e_int)
// in per-thread shared-memory slots instead of six registers: the contract build's
// spills shrink (48 -> 20 B), +3.4 % there (with TMA_SPREAD, which then pays: 18.1 G
// cell-updates/s); -6 % in the exact build, which does not spill
#ifndef LF_FUSED_KEYSMEM
#if LF_CONTRACT
#define LF_FUSED_KEYSMEM 1
#else
#define LF_FUSED_KEYSMEM 0
#endif
#endif
template <bool MUSCL>
__global__ void __launch_bounds__(FUSED_THREADS, LF_MINBLOCKS) k_fused_step(FusedArgs a) {
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;                   // [URING][4][NC] U^n rows (TMA destination)
  double* sWr = sU + URING * 4 * NC;   // [4][NC]     P: W(r-2) for x slopes
  double* sTx = sWr + 4 * NC;          // [4][NC]     P: x hi-traces
  double* sFnx = sTx + 4 * NC;         // [4][4][NC]  ring: F^n x-faces of a row
  double* sFny = sFnx + 16 * NC;       // [4][4][NC]  ring: F^n y-faces
  double* sWs = sFny + 16 * NC;        // [4][4][NC]  ring: W* rows (P -> C: y window, x slopes)
  double* sWc = sWs + 16 * NC;         // [4][NC]     C: W*(j) for x slopes (without LF_FUSED_CRING)
  double* sTc = sWc + WC_ROWS * 4 * NC;  // [4][NC]   C: x hi-traces
  double* sFc = sTc + 4 * NC;          // [4][NC]     C: 0.5 (F^n + F*) x-faces
  double* sStash = sFc + 4 * NC;       // [4][NC]     C: top-edge ghost image
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sStash + 4 * NC);  // [URING]
#if LF_FUSED_KEYSMEM
  unsigned long long* sKey = mbar + URING;   // [3][NC] corrector maxima
#endif

  const StepCtl ctl = *a.ctl;
  if (ctl.done) return;
  if (ctl.dtfail) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  // dt exactly as compute_dt (solver.cpp:476-477) and apply_update (:262-263)
  const double rate = key_to_double(ctl.rate_bits);
  double dt = a.cfl / rate;
  if (ctl.time + dt > a.limit) dt = a.limit - ctl.time;
  if (!(dt > 0.0)) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) atomicMax(&a.acc->fail, 1ull);
    return;
  }
  const double lam_x = dt / a.dx;
  const double lam_y = dt / a.dy;

  // (from the launch parameters: the compiler may reread them from the constant bank
  // instead of holding them in registers)
  FK C;
  C.gamma = a.fk.gamma;
  C.gm1 = a.fk.gm1;
  C.beta = a.fk.beta;
  C.rgm1 = Recip{a.fk.rgm1_b, a.fk.rgm1_y};
  C.rdx = Recip{a.fk.rdx_b, a.fk.rdx_y};
  C.rdy = Recip{a.fk.rdy_b, a.fk.rdy_y};

  const int t = threadIdx.x & (NC - 1);
  const bool is_p = threadIdx.x < NC;
  const int x0 = blockIdx.x * TXO;
  const int c = x0 - 4 + t;                      // this thread's column
  const int y0 = (a.chunk0 + (int)blockIdx.y * a.chunk_step) * a.rows_per_chunk;  // rows [y0, y1)
  const int y1 = min(y0 + a.rows_per_chunk, a.ny);
  const int nit = (y1 - y0) + 9;
  const int klastp = (y1 - y0) + 7;              // last P iteration (input row y1+3)
  const bool col_in_mem = c >= -NG && c < a.nx + NG;
  const bool col_interior = c >= 0 && c < a.nx;
  const bool bottom_edge = a.bottom_edge && y0 == 0;
  const bool top_edge = a.top_edge && y1 == a.ny;
  // row rho (relative to y0-4) of component q starts at src_row(rho) + q*fstride
  const double* src0 = a.u + (int64_t)(y0 - 4) * a.pitch + (x0 - 4);
  const uint32_t row_bytes = NC * sizeof(double);

  if (threadIdx.x == 0) {
    for (int s = 0; s < URING; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < PREFETCH; ++k) {
      mbar_expect_tx(&mbar[k], 4 * row_bytes);
      for (int q = 0; q < 4; ++q)
        tma_row(sU + (k * 4 + q) * NC, src0 + (int64_t)k * a.pitch + q * a.fstride, row_bytes, &mbar[k]);
    }
  }
  __syncthreads();

  unsigned fail = const_in_box(a.gamma, a.gm1) ? 0u : 1u;

  // Row iterations k = 0 .. nit-1 run in three ranges.  The first KS and the last
  // few (k > ksteady) see the chunk's pipeline fill / drain, the domain's y edges
  // (ghost-row images, rows outside the slab) and the bottom / top boundary faces;
  // they take the guarded body (G = true).  In between every guard is true, so the
  // steady body (G = false) drops them: no default states, no row-range tests in
  // the failure checks, no per-row predicates -- the same values, fewer instructions.
  constexpr int KS = 10;
  const int ksteady = (y1 - y0) + 3;   // last steady iteration (input row y1 - 1)

  if (is_p) {
    // ================================================================ stage 1 (P)
    double wm2[4] = {1.0, 0.0, 0.0, 1.0}, wm1[4] = {1.0, 0.0, 0.0, 1.0};
    double fyprev[4] = {0.0, 0.0, 0.0, 0.0};
    double hiprev[4] = {1.0, 0.0, 0.0, 1.0};
    // this thread owns x-face (t-1 | t), needed for U* up to column nx+1
    const bool dox = t >= 2 && t <= NC - 2 && c <= a.nx + 2;
    const bool xchk = dox && c >= 0 && c <= a.nx;          // kept x-face of the grid
    const bool upd = t >= 2 && t <= NC - 3;                // lanes with a kept U* column
    const int tl = t > 0 ? t - 1 : t, tr = t < NC - 1 ? t + 1 : t;   // clamped x neighbours
    auto iter = [&](const int k, auto guard) {
      constexpr bool G = decltype(guard)::value;
      const int r = y0 - 4 + k;
      const bool p_active = !G || k <= klastp;
#if LF_FUSED_TMA_SPREAD
      // lane 0 of P warp q copies component q of row k+PREFETCH (the four warps share
      // the issue cost, so none lags at the next barrier); warp 0 also posts the
      // expected bytes -- the transaction count may run negative until it does, and
      // the phase cannot complete before its arrival
      if ((threadIdx.x & 31) == 0 && (!G || k + PREFETCH <= klastp)) {
        // the slot's previous row (k+PREFETCH-URING) was last read before the
        // previous iteration's __syncthreads
        const int kn = k + PREFETCH, s = kn & (URING - 1), q = threadIdx.x >> 5;
        if (q < 4) {   // (NC = 256: eight predictor warps, four components)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (q == 0) mbar_expect_tx(&mbar[s], 4 * row_bytes);
          tma_row(sU + (s * 4 + q) * NC, src0 + (int64_t)kn * a.pitch + q * a.fstride, row_bytes,
                  &mbar[s]);
        }
      }
#else
      if (threadIdx.x == 0 && (!G || k + PREFETCH <= klastp)) {
        // the slot's previous row (k+PREFETCH-URING) was last read before the
        // previous iteration's __syncthreads
        const int kn = k + PREFETCH, s = kn & (URING - 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[s], 4 * row_bytes);
        for (int q = 0; q < 4; ++q)
          tma_row(sU + (s * 4 + q) * NC, src0 + (int64_t)kn * a.pitch + q * a.fstride, row_bytes,
                  &mbar[s]);
      }
#endif
      double w[4], ylo[4], yhi[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = ylo[q] = yhi[q] = (q == 0 || q == 3) ? 1.0 : 0.0;
      }
      if (p_active) {
        // -- U^n(r) -> W(r) (solver.cpp:145-163); lanes past the grid's ghost columns
        //    (last strip) compute on don't-care values no kept result depends on
        mbar_wait(&mbar[k & (URING - 1)], (k / URING) & 1);
        if (!G || col_in_mem) {
          const double* u = sU + (k & (URING - 1)) * 4 * NC + t;
          const double r0 = u[0], m1 = u[NC], m2 = u[2 * NC], e3 = u[3 * NC];
          bool okw = true;  // implied by the box
          prim_fast(r0, m1, m2, e3, a.gm1, w, okw);
          if (!cell_in_box(w) && col_interior && (!G || (r >= 0 && r < a.ny))) fail = 1;
        }
        if (!G || k >= 2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            sWr[q * NC + t] = wm2[q];  // row r-2 for the x direction
            cell_traces<MUSCL>(wm2[q], wm1[q], w[q], a.beta, ylo[q], yhi[q]);  // row r-1
          }
        }
      }
      bar_named(1);
      double xlo[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) xlo[q] = (q == 0 || q == 3) ? 1.0 : 0.0;
      }
      if (G ? (p_active && k >= 2 && t >= 1 && t <= NC - 2) : true) {
        // (steady: the edge lanes use a clamped neighbour; their traces are unused)
        const int il = G ? t - 1 : tl, ir = G ? t + 1 : tr;
        const double* wr = sWr;   // W(r-2)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double hi;
          cell_traces<MUSCL>(wr[q * NC + il], wr[q * NC + t], wr[q * NC + ir], a.beta, xlo[q], hi);
          sTx[q * NC + t] = hi;
        }
      }
      bar_named(1);
      double fy[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fy[q] = 0.0;
      }
      if (!G || (p_active && k >= 2)) {
        // x-face (t-1 | t) of row r-2 and y-face (r-2 | r-1)
#if LF_FUSED_DONTCARE_P
        const int tm = tl;   // lanes without a kept x-face: unused
#else
        const int tm = dox ? t - 1 : t;
#endif
        double mx[4];
#pragma unroll
#if LF_FUSED_DONTCARE_P
        for (int q = 0; q < 4; ++q) mx[q] = sTx[q * NC + tm];
#else
        for (int q = 0; q < 4; ++q) mx[q] = dox ? sTx[q * NC + tm] : xlo[q];
#endif
        double fx[4];
        bool okx = true, oky = true;  // implied by the cell box (face_fast.cuh): unused
        double psx, usx, psy, usy;
        face_fast<0>(mx[0], mx[1], mx[2], mx[3], xlo[0], xlo[1], xlo[2], xlo[3], C, fx, okx, psx,
                     usx);
        face_fast<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2], ylo[3],
                     C, fy, oky, psy, usy);
        if (needs_mean(usx))
          face_mean<0>(mx[0], mx[1], mx[2], mx[3], xlo[0], xlo[1], xlo[2], xlo[3], psx, usx, C,
                       fx, okx);
        if (needs_mean(usy))
          face_mean<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2],
                       ylo[3], psy, usy, C, fy, oky);
        // a trace-positivity failure on a consumed face hands the step to the
        // stage-wise IEEE kernels (halo lanes and columns past the grid hold
        // dummy states and never count)
        if (G ? (xchk && r - 2 >= 0 && r - 2 < a.ny) : xchk) {
          if (!traces_ok(mx[0], mx[3], xlo[0], xlo[3])) fail = 1;
        }
        if (!G || dox) {
          // (steady: every lane stores; faces outside dox are never read for a kept value)
#pragma unroll
          for (int q = 0; q < 4; ++q) sFnx[((k & 3) * 4 + q) * NC + t] = fx[q];
        }
        if (!G || k >= 3) {
          if (!traces_ok(hiprev[0], hiprev[3], ylo[0], ylo[3]) && col_interior &&
              (!G || (r - 1 >= 0 && r - 1 <= a.ny)))
            fail = 1;
#pragma unroll
          for (int q = 0; q < 4; ++q) sFny[((k & 3) * 4 + q) * NC + t] = fy[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) hiprev[q] = yhi[q];
      }
      bar_named(1);
      // -- predictor U*(r-2) (solver.cpp:283-291 with one flux set), then its
      //    primitives W*(r-2) (build_primitives of predictor_, solver.cpp:505);
      //    steady: every lane (edge lanes read neighbouring smem, their W* is unused)
      if (G ? (p_active && k >= 4 && upd && col_in_mem) : true) {
        const int row = r - 2;
        const double* ub = sU + ((k - 2) & (URING - 1)) * 4 * NC + t;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double fxl = sFnx[((k & 3) * 4 + q) * NC + t];
          const double fxr = sFnx[((k & 3) * 4 + q) * NC + t + 1];
          double val = ub[q * NC] - lam_x * (fxr - fxl);
          val -= lam_y * (fy[q] - fyprev[q]);
          v[q] = val;
        }
        double ws[4];
        bool okw = true;
        prim_fast(v[0], v[1], v[2], v[3], a.gm1, ws, okw);
#pragma unroll
        for (int q = 0; q < 4; ++q) sWs[((k & 3) * 4 + q) * NC + t] = ws[q];
        if (upd && col_interior && (!G || (row >= 0 && row < a.ny))) {
          // e_int = v3 - (0.5 (v1^2 + v2^2)) / v0 > 0 (solver.cpp:300-302), tested
          // without the division: v3 v0 > K (1 + 2^-48) implies it; else flag
          // (conservative: the stage-wise re-run decides exactly)
          const double kin = 0.5 * (v[1] * v[1] + v[2] * v[2]);
          const double lhs = v[3] * v[0];
          if (!(v[0] > 0.0) || !(lhs > kin * (1.0 + 0x1p-48)) || !(lhs >= 0x1p-960)) fail = 1;
          if (!cell_in_box(ws)) fail = 1;
        }
      }
      if (!G || (p_active && k >= 3)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fyprev[q] = fy[q];
      }
      if (p_active) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wm2[q] = wm1[q];
          wm1[q] = w[q];
        }
      }
      __syncthreads();
    };
    int k = 0;
    for (; k < KS && k < nit; ++k) iter(k, std::true_type{});
    for (; k <= ksteady; ++k) iter(k, std::false_type{});
    for (; k < nit; ++k) iter(k, std::true_type{});
  } else {
    // ================================================================ stage 2 (C)
    double vm2[4] = {1.0, 0.0, 0.0, 1.0}, vm1[4] = {1.0, 0.0, 0.0, 1.0};
    double hiprev[4] = {1.0, 0.0, 0.0, 1.0}, fcprev[4] = {0.0, 0.0, 0.0, 0.0};
#if LF_FUSED_KEYSMEM
    sKey[t] = 0ull;
    sKey[NC + t] = NINF_KEY;
    sKey[2 * NC + t] = NINF_KEY;
#else
    unsigned long long rate_key = 0ull, nmin_r = NINF_KEY, nmin_e = NINF_KEY;
#endif
    unsigned dtfail = 0;
    // source column of this thread's W* value (ghost columns at non-periodic x edges)
    int src_t = t;
    bool flip_u = false;
    if (c < 0 && a.bc_xlo != LF_PERIODIC) {
      const int sc = a.bc_xlo == LF_REFLECTIVE ? -c - 1 : 0;
      src_t = t + (sc - c);
      flip_u = a.bc_xlo == LF_REFLECTIVE;
    } else if (c >= a.nx && a.bc_xhi != LF_PERIODIC) {
      const int sc = a.bc_xhi == LF_REFLECTIVE ? 2 * a.nx - 1 - c : a.nx - 1;
      src_t = t + (sc - c);
      flip_u = a.bc_xhi == LF_REFLECTIVE;
    }
    // lanes without a W* column (t < 2, t > NC-3) feed no face or cell that is kept:
    // they read a clamped column instead of selecting a default state
    const int src_c = min(max(src_t, 2), NC - 3);
    const unsigned long long flip_bits = flip_u ? 0x8000000000000000ull : 0ull;
    // the same for the x neighbours (lanes tl, tr): the x slopes of W*(j) are read
    // straight from the P -> C ring, with each lane's image mapping
    auto src_of = [&](int u, unsigned long long& fb) {
      const int cu = x0 - 4 + u;
      int su = u;
      bool fu = false;
      if (cu < 0 && a.bc_xlo != LF_PERIODIC) {
        su = u + ((a.bc_xlo == LF_REFLECTIVE ? -cu - 1 : 0) - cu);
        fu = a.bc_xlo == LF_REFLECTIVE;
      } else if (cu >= a.nx && a.bc_xhi != LF_PERIODIC) {
        su = u + ((a.bc_xhi == LF_REFLECTIVE ? 2 * a.nx - 1 - cu : a.nx - 1) - cu);
        fu = a.bc_xhi == LF_REFLECTIVE;
      }
      fb = fu ? 0x8000000000000000ull : 0ull;
      return min(max(su, 2), NC - 3);
    };
    const bool dox = t >= 4 && t <= NC - 4 && c <= a.nx;  // x-faces of output cells
    const bool xchk = dox && c >= 0;
    const bool upd = t >= 4 && t <= NC - 5 && col_interior;   // output cells
    const int tl = t > 0 ? t - 1 : t, tr = t < NC - 1 ? t + 1 : t;   // clamped x neighbours
    // a block holding ghost columns of a non-periodic x side (block-uniform): its lanes
    // map to image columns; elsewhere every lane reads its own column
    const bool x_img_blk = (x0 - 4 < 0 && a.bc_xlo != LF_PERIODIC) ||
                           (x0 - 4 + NC > a.nx && a.bc_xhi != LF_PERIODIC);
    const bool x_edge_blk = x0 - 4 <= 0 || x0 - 4 + NC > a.nx - 1;   // holds column 0 or nx-1
    const bool dxy_box = pos_in_box(a.dx) && pos_in_box(a.dy);
    // positivity (solver.cpp:300-307) and the diagnostics minima and the CFL rate of
    // U^{n+1} for the next step's dt (solver.cpp:457-469), of one updated cell
    auto epilogue = [&](const double (&v)[4]) {
      bool ok = true, okr = true, rate_ok;
      double eint, rr;
#if LF_FUSED_EPI_BOX
      cell_epilogue_box<LF_FUSED_EPI_BOX == 2>(v, C, dxy_box, eint, ok, rr, rate_ok, okr);
#else
      cell_epilogue(v, C, eint, ok, rr, rate_ok, okr);
#endif
      if (!(v[0] > 0.0) || !(eint > 0.0) || !ok) {
        fail = 1;
      } else {
        const unsigned long long kr = ~pos_bits(v[0]), ke = ~pos_bits(eint);
#if LF_FUSED_KEYSMEM
        const unsigned long long nr = sKey[NC + t], ne = sKey[2 * NC + t];
        sKey[NC + t] = kr > nr ? kr : nr;
        sKey[2 * NC + t] = ke > ne ? ke : ne;
#else
        nmin_r = kr > nmin_r ? kr : nmin_r;
        nmin_e = ke > nmin_e ? ke : nmin_e;
#endif
      }
      if (rate_ok) {
        if (rr == rr) {
          const unsigned long long b = pos_bits(rr);
#if LF_FUSED_KEYSMEM
          const unsigned long long rk = sKey[t];
          sKey[t] = b > rk ? b : rk;
#else
          rate_key = b > rate_key ? b : rate_key;
#endif
        }
        if (!okr) fail = 1;
      } else {
        dtfail = 1;
      }
    };
    auto iter = [&](const int k, auto guard) {
      constexpr bool G = decltype(guard)::value;
      const int aa = y0 - 7 + k;   // W* row consumed this iteration
      const int j = aa - 2;        // U^{n+1} row finished this iteration
      const bool c_active = !G || k >= 5;
      double w[4], ylo[4], yhi[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = ylo[q] = yhi[q] = (q == 0 || q == 3) ? 1.0 : 0.0;
      }
      if (c_active) {
        // -- W*(aa) with the boundary images of the reference's ghost fill of
        //    predictor_ (grid.cpp:72-114); a reflective image negates the normal
        //    velocity exactly as it negates the normal momentum
        {
          const double* ws = sWs + ((k - 1) & 3) * 4 * NC + src_c;
          w[0] = ws[0];
          w[1] = __longlong_as_double(__double_as_longlong(ws[NC]) ^ flip_bits);
          w[2] = ws[2 * NC];
          w[3] = ws[3 * NC];
        }
        // the ghost-row images below are block-uniform and rare (guarded iterations only)
        if (G && ((bottom_edge && aa <= 1) || (top_edge && aa >= a.ny))) {
          if (bottom_edge && aa == 0) {
            // W*(-1) = image of W*(0)
#pragma unroll
            for (int q = 0; q < 4; ++q) vm1[q] = w[q];
            if (a.bc_ylo == LF_REFLECTIVE) vm1[2] = -vm1[2];
          }
          if (bottom_edge && aa == 1) {
            // hi trace of ghost row -1 from W*(-2) = image(W*(1) or W*(0)), W*(-1), W*(0)
            double g2[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) g2[q] = a.bc_ylo == LF_REFLECTIVE ? w[q] : vm1[q];
            if (a.bc_ylo == LF_REFLECTIVE) g2[2] = -g2[2];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              double lo;
              cell_traces<MUSCL>(g2[q], vm2[q], vm1[q], a.beta, lo, hiprev[q]);
            }
          }
          if (top_edge && aa == a.ny) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              w[q] = vm1[q];
              sStash[q * NC + t] = a.bc_yhi == LF_REFLECTIVE ? vm2[q] : vm1[q];
            }
            if (a.bc_yhi == LF_REFLECTIVE) {
              w[2] = -w[2];
              sStash[2 * NC + t] = -sStash[2 * NC + t];
            }
          } else if (top_edge && aa == a.ny + 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = sStash[q * NC + t];
          }
        }
        if (!G || k >= 7) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
#if !LF_FUSED_CRING
            sWc[q * NC + t] = vm2[q];  // row j = aa-2 for the x direction
#endif
            cell_traces<MUSCL>(vm2[q], vm1[q], w[q], a.beta, ylo[q], yhi[q]);  // row aa-1
          }
        }
      }
#if !LF_FUSED_CRING
      bar_named(2);
#endif
      double xlo[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) xlo[q] = (q == 0 || q == 3) ? 1.0 : 0.0;
      }
      if (G ? (c_active && k >= 9 && t >= 3 && t <= NC - 4) : true) {
        // (steady: the edge lanes use a clamped neighbour; their traces are unused)
        // W*(j) = W*(aa-2), written by P three iterations ago (j is an interior row
        // here), at each lane's image column: the x slopes without an exchange barrier
        const double* wj = sWs + ((k - 3) & 3) * 4 * NC;
        double wl[4], w0[4], wr_[4];
        if (!LF_FUSED_CRING) {
          // (the exchanged W*(j) row: images applied by the lanes that stored it)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            wl[q] = sWc[q * NC + (G ? t - 1 : tl)];
            w0[q] = sWc[q * NC + t];
            wr_[q] = sWc[q * NC + (G ? t + 1 : tr)];
          }
        } else if (!x_img_blk) {
          // (lanes outside [3, NC-4] read don't-care columns; their traces are unused)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            wl[q] = wj[q * NC + tl];
            w0[q] = wj[q * NC + t];
            wr_[q] = wj[q * NC + tr];
          }
        } else {
          unsigned long long flip_l, flip_r;
          const int src_l = src_of(tl, flip_l), src_r = src_of(tr, flip_r);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            wl[q] = wj[q * NC + src_l];
            w0[q] = wj[q * NC + src_c];
            wr_[q] = wj[q * NC + src_r];
          }
          wl[1] = __longlong_as_double(__double_as_longlong(wl[1]) ^ flip_l);
          w0[1] = __longlong_as_double(__double_as_longlong(w0[1]) ^ flip_bits);
          wr_[1] = __longlong_as_double(__double_as_longlong(wr_[1]) ^ flip_r);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double hi;
          cell_traces<MUSCL>(wl[q], w0[q], wr_[q], a.beta, xlo[q], hi);
          sTc[q * NC + t] = hi;
        }
      }
      bar_named(2);
      double fc[4];
      if (G) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fc[q] = 0.0;
      }
      if (!G || (c_active && k >= 7)) {
        const bool dx_ = dox && (!G || k >= 9);
        // a lane without a kept x-face reads its left neighbour's trace anyway (unused)
        double mx[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = sTc[q * NC + tl];
        double fx[4], fs[4];
        bool okx = true, oky = true;  // implied by the cell box (face_fast.cuh): unused
        double psx, usx, psy, usy;
        face_fast<0>(mx[0], mx[1], mx[2], mx[3], xlo[0], xlo[1], xlo[2], xlo[3], C, fx, okx, psx,
                     usx);
        face_fast<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2], ylo[3],
                     C, fs, oky, psy, usy);
        if (needs_mean(usx))
          face_mean<0>(mx[0], mx[1], mx[2], mx[3], xlo[0], xlo[1], xlo[2], xlo[3], psx, usx, C,
                       fx, okx);
        if (needs_mean(usy))
          face_mean<1>(hiprev[0], hiprev[1], hiprev[2], hiprev[3], ylo[0], ylo[1], ylo[2],
                       ylo[3], psy, usy, C, fs, oky);
        if (G ? (dx_ && c >= 0 && j >= 0 && j < a.ny) : xchk) {
          if (!traces_ok(mx[0], mx[3], xlo[0], xlo[3])) fail = 1;
        }
        if (!G || dx_) {
          // (steady: every lane stores; the update reads the faces of dox lanes only)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            sFc[q * NC + t] = 0.5 * (sFnx[(((k + 1) & 3) * 4 + q) * NC + t] + fx[q]);
        }
        if (!G || k >= 8) {
          if (!traces_ok(hiprev[0], hiprev[3], ylo[0], ylo[3]) && col_interior &&
              (!G || (aa - 1 >= 0 && aa - 1 <= a.ny)))
            fail = 1;
#pragma unroll
          for (int q = 0; q < 4; ++q) fc[q] = 0.5 * (sFny[(((k + 1) & 3) * 4 + q) * NC + t] + fs[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) hiprev[q] = yhi[q];
      }
      bar_named(2);
      // -- corrector U^{n+1}(j) (solver.cpp:283-291, two flux sets) + epilogue
      if (upd && (!G || (c_active && k >= 9))) {
        const double* ub = sU + ((k - 5) & (URING - 1)) * 4 * NC + t;
        const int64_t o = (int64_t)j * a.pitch + c;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double val = ub[q * NC] - lam_x * (sFc[q * NC + t + 1] - sFc[q * NC + t]);
          val -= lam_y * (fc[q] - fcprev[q]);
          v[q] = val;
          a.un[q * a.fstride + o] = val;
        }
        epilogue(v);
        // domain-boundary faces for accumulate_boundary_outflow (solver.cpp:406-432);
        // one block-uniform test skips all four in the interior of the domain (the
        // bottom / top rows only occur in guarded iterations)
        const int jg = j + a.y0g;
        if (x_edge_blk || (G && (jg == 0 || jg == a.nyg - 1))) {
          if (c == 0)
            for (int q = 0; q < 4; ++q) a.bnd[(int64_t)q * a.nyg + jg] = sFc[q * NC + t];
          if (c == a.nx - 1)
            for (int q = 0; q < 4; ++q)
              a.bnd[4 * (int64_t)a.nyg + (int64_t)q * a.nyg + jg] = sFc[q * NC + t + 1];
          if (G && jg == 0)
            for (int q = 0; q < 4; ++q) a.bnd[8 * (int64_t)a.nyg + (int64_t)q * a.nx + c] = fcprev[q];
          if (G && jg == a.nyg - 1)
            for (int q = 0; q < 4; ++q)
              a.bnd[8 * (int64_t)a.nyg + 4 * (int64_t)a.nx + (int64_t)q * a.nx + c] = fc[q];
        }
      }
      if (!G || (c_active && k >= 8)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fcprev[q] = fc[q];
      }
      if (c_active) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          vm2[q] = vm1[q];
          vm1[q] = w[q];
        }
      }
      __syncthreads();
    };
    int k = 0;
    for (; k < KS && k < nit; ++k) iter(k, std::true_type{});
    for (; k <= ksteady; ++k) iter(k, std::false_type{});
    for (; k < nit; ++k) iter(k, std::true_type{});
    // block-level reductions (warp shuffles, then one atomic per warp)
#if LF_FUSED_KEYSMEM
    unsigned long long rate_key = sKey[t], nmin_r = sKey[NC + t], nmin_e = sKey[2 * NC + t];
#endif
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long r2 = __shfl_xor_sync(FULL, rate_key, o);
      const unsigned long long a2 = __shfl_xor_sync(FULL, nmin_r, o);
      const unsigned long long b2 = __shfl_xor_sync(FULL, nmin_e, o);
      rate_key = r2 > rate_key ? r2 : rate_key;
      nmin_r = a2 > nmin_r ? a2 : nmin_r;
      nmin_e = b2 > nmin_e ? b2 : nmin_e;
    }
    dtfail = __any_sync(FULL, dtfail);
    if ((threadIdx.x & 31) == 0) {
      if (rate_key) atomicMax(&a.acc->rate_next, rate_key);
      if (nmin_r != NINF_KEY) atomicMax(&a.acc->nmin_rho, nmin_r);
      if (nmin_e != NINF_KEY) atomicMax(&a.acc->nmin_eint, nmin_e);
      if (dtfail) atomicMax(&a.acc->dtfail_next, 1ull);
    }
  }
  if (__any_sync(FULL, fail) && (threadIdx.x & 31) == 0) atomicMax(&a.acc->fail, 1ull);
}

#if !LF_CONTRACT
// After the step's kernel (and the cross-rank all-reduce of acc): dt / time
// bookkeeping (solver.cpp:494,542-544), the ordered boundary-outflow sums
// (solver.cpp:406-432, one thread per component and direction) and the
// control record of the next step.
__global__ void k_finalize(const StepCtl* __restrict__ ctl, StepAcc* acc, StepCtl* nxt,
                           StepRec* rec, double* outflow, bool outflow_zero, double dx, double dy,
                           double cfl, double limit, double t_final) {
  pdl_wait();
  const StepCtl c = *ctl;
  const bool skip = c.done != 0;
  double dt = 0.0;
  if (!skip) {
    const double rate = __longlong_as_double((long long)c.rate_bits);
    dt = cfl / rate;
    if (c.time + dt > limit) dt = limit - c.time;
  }
  const bool failed = !skip && (acc->fail != 0 || c.dtfail || !(dt > 0.0));
  StepRec r;
  r.dt = dt;
  r.hits = 0;
  r.time = c.time;
  r.min_rho = 0.0;
  r.min_eint = 0.0;
  r.min_p_mat = __longlong_as_double(0x7ff0000000000000ll);
  StepCtl n;
  n.rate_bits = acc->rate_next;
  n.dtfail = acc->dtfail_next != 0;
  if (skip) {
    r.status = 2;
    n = c;
    n.done = 1;
  } else if (failed) {
    r.status = acc->fail == 2ull ? 3 : 1;   // 3: only the exact two-pass kernels are needed
    n = c;
    n.done = 1;
  } else {
    r.status = 0;
    r.hits = c.time + dt >= limit;
    r.time = r.hits ? limit : c.time + dt;
    r.min_rho = __longlong_as_double((long long)~acc->nmin_rho);
    r.min_eint = __longlong_as_double((long long)~acc->nmin_eint);
    r.min_p_mat = __longlong_as_double((long long)~acc->nmin_p);
    if (outflow_zero) {
      // every axis periodic: both face sums are +0.0 (k_outflow's comment)
      const double ax = dt * dy, ay = dt * dx;
      for (int q = 0; q < 4; ++q) {
        outflow[q] += ax * 0.0;
        outflow[q] += ay * 0.0;
      }
    }
    n.time = r.time;
    n.done = !(r.time < t_final);
  }
  *rec = r;
  *nxt = n;
  // reset this step's accumulators for the step after next
  acc->rate_next = 0ull;
  acc->fail = 0ull;
  acc->nmin_rho = NINF_KEY;
  acc->nmin_eint = NINF_KEY;
  acc->dtfail_next = 0ull;
  acc->nmin_p = NINF_KEY;
}

// accumulate_boundary_outflow (solver.cpp:406-432) of a completed step: per
// component, s += (right - left) over the rows in order, then s += (top -
// bottom) over the columns in order, outflow += dt*dy*s_x, += dt*dx*s_y.  Only
// the accumulation is sequential (lanes 0-7 of warp 0, one chain per component
// and axis); the other warps stage the next tile of differences meanwhile.  A
// periodic axis skips its sums: both of its boundary faces are the same face,
// solved from the same inputs by the same code, so every difference is +0.0 and
// so is their ordered sum.  Runs on a side stream, off the step's critical path.
__global__ void __launch_bounds__(256)
    k_outflow(const StepRec* __restrict__ rec, const double* __restrict__ bnd, double* outflow,
              int nx, int nyg, bool sum_x, bool sum_y, double dx, double dy) {
  constexpr int TILE = 256;
  __shared__ double dif[2][TILE][9];  // [buffer][element][chain]; 9: conflict-free rows
  const StepRec r = *rec;
  if (r.status != 0) return;
  const int tid = threadIdx.x;
  const int ex = sum_x ? nyg : 0, ey = sum_y ? nx : 0;
  const int ntiles = ((ex > ey ? ex : ey) + TILE - 1) / TILE;
  auto stage = [&](int t, int buf) {
    for (int k = tid - 32; k < 8 * TILE; k += blockDim.x - 32) {
      const int ch = k / TILE, e = t * TILE + k % TILE, q = ch & 3;
      double d = 0.0;
      if (ch < 4 && e < ex)
        d = bnd[4 * (int64_t)nyg + (int64_t)q * nyg + e] - bnd[(int64_t)q * nyg + e];
      else if (ch >= 4 && e < ey)
        d = bnd[8 * (int64_t)nyg + 4 * (int64_t)nx + (int64_t)q * nx + e] -
            bnd[8 * (int64_t)nyg + (int64_t)q * nx + e];
      dif[buf][k % TILE][ch] = d;
    }
  };
  double s = 0.0;
  if (tid >= 32 && ntiles > 0) stage(0, 0);
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    if (tid >= 32) {
      if (t + 1 < ntiles) stage(t + 1, (t + 1) & 1);
    } else if (tid < 8) {
      const int n = (tid < 4 ? ex : ey) - t * TILE;
      const double(*d)[9] = dif[t & 1];
      if (n >= TILE) {
#pragma unroll 32
        for (int e = 0; e < TILE; ++e) s += d[e][tid];
      } else {
        for (int e = 0; e < n; ++e) s += d[e][tid];
      }
    }
    __syncthreads();
  }
  __shared__ double sums[8];
  if (tid < 8) sums[tid] = s;
  __syncthreads();
  if (tid != 0) return;
  const double ax = r.dt * dy, ay = r.dt * dx;
  for (int q = 0; q < 4; ++q) {
    outflow[q] += ax * sums[q];
    outflow[q] += ay * sums[4 + q];
  }
}

__global__ void k_acc_init(StepAcc* acc) {
  for (int i = 0; i < 2; ++i) {
    acc[i].rate_next = 0ull;
    acc[i].fail = 0ull;
    acc[i].nmin_rho = NINF_KEY;
    acc[i].nmin_eint = NINF_KEY;
    acc[i].dtfail_next = 0ull;
    acc[i].nmin_p = NINF_KEY;
  }
}

#endif  // !LF_CONTRACT

__global__ void k_make_fk(double gamma, double gm1, double beta, double dx, double dy,
                          FKBits* out) {
  const FK c = make_fk(gamma, gm1, beta, dx, dy);
  FKBits b;
  b.gamma = c.gamma;
  b.gm1 = c.gm1;
  b.beta = c.beta;
  b.rgm1_b = c.rgm1.b;
  b.rgm1_y = c.rgm1.y;
  b.rdx_b = c.rdx.b;
  b.rdx_y = c.rdx.y;
  b.rdy_b = c.rdy.b;
  b.rdy_y = c.rdy.y;
  *out = b;
}

FKBits make_fk_host(double gamma, double gm1, double beta, double dx, double dy) {
  FKBits* d = nullptr;
  FKBits h{};
  if (cudaMalloc(&d, sizeof(FKBits)) != cudaSuccess) return h;
  count_launch();
  k_make_fk<<<1, 1>>>(gamma, gm1, beta, dx, dy, d);
  cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

constexpr size_t SMEM_BYTES =
    (size_t)(URING * 4 + 4 + 4 + 16 + 16 + 16 + WC_ROWS * 4 + 4 + 4 + 4) * NC *
        sizeof(double) +
    URING * sizeof(unsigned long long) + (LF_FUSED_KEYSMEM ? 3 * NC * sizeof(unsigned long long) : 0);
// two blocks per SM (228 KB, 1 KB reserved per block): one block per SM halves the
// resident warps of this latency-bound kernel
static_assert(LF_MINBLOCKS * (SMEM_BYTES + 1024) <= 228 * 1024, "fused step: two blocks per SM");

}  // namespace

#if LF_CONTRACT
FKBits fused_make_fk_contract(double gamma, double gm1, double beta, double dx, double dy) {
  return make_fk_host(gamma, gm1, beta, dx, dy);
}

// fused_contract.cu: the one-kernel step in the tolerance arithmetic (LF_MATH_CONTRACT)
void fused_configure_contract() {
  cudaFuncSetAttribute(k_fused_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SMEM_BYTES);
  cudaFuncSetAttribute(k_fused_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SMEM_BYTES);
}

void launch_fused_step_contract(const FusedArgs& a, bool muscl, dim3 grid, cudaStream_t st) {
  count_launch();
  if (muscl)
    k_fused_step<true><<<grid, FUSED_THREADS, SMEM_BYTES, st>>>(a);
  else
    k_fused_step<false><<<grid, FUSED_THREADS, SMEM_BYTES, st>>>(a);
}
#else
FKBits fused_make_fk(double gamma, double gm1, double beta, double dx, double dy) {
  return make_fk_host(gamma, gm1, beta, dx, dy);
}

size_t fused_smem_bytes() { return SMEM_BYTES; }

int fused_blocks_per_sm() {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused_step<true>, FUSED_THREADS,
                                                    SMEM_BYTES) != cudaSuccess || b < 1)
    b = LF_MINBLOCKS;
  return b;
}

void fused_configure() {
  cudaFuncSetAttribute(k_fused_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SMEM_BYTES);
  cudaFuncSetAttribute(k_fused_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SMEM_BYTES);
}

void launch_fused_step(const FusedArgs& a, bool muscl, dim3 grid, cudaStream_t st) {
  count_launch();
  if (muscl)
    k_fused_step<true><<<grid, FUSED_THREADS, SMEM_BYTES, st>>>(a);
  else
    k_fused_step<false><<<grid, FUSED_THREADS, SMEM_BYTES, st>>>(a);
}

void launch_finalize(const StepCtl* ctl, StepAcc* acc, StepCtl* nxt, StepRec* rec,
                     double* outflow, bool outflow_zero, double dx, double dy, double cfl,
                     double limit, double t_final, cudaStream_t st) {
  count_launch();
  launch_chain(k_finalize, dim3(1), dim3(1), 0, st, ctl, acc, nxt, rec, outflow, outflow_zero, dx,
               dy, cfl, limit, t_final);
}

void launch_outflow(const StepRec* rec, const double* bnd, double* outflow, int nx, int nyg,
                    bool sum_x, bool sum_y, double dx, double dy, cudaStream_t st) {
  count_launch();
  k_outflow<<<1, 256, 0, st>>>(rec, bnd, outflow, nx, nyg, sum_x, sum_y, dx, dy);
}

void launch_acc_init(StepAcc* acc, cudaStream_t st) {
  count_launch();
  k_acc_init<<<1, 1, 0, st>>>(acc);
}
#endif  // LF_CONTRACT

}  // namespace lfb
