// small_step.cu -- LF_PATH_SMALL: the whole step loop of a small grid in one
// persistent thread-block cluster (1D grids and small 2D grids, one material), or --
// beyond one cluster's worth of cells -- one persistent cooperative grid.
//
// A grid of a few thousand cells cannot fill a B200: the stage-wise step is a
// dozen launches and three host round trips (~110 us), the two-pass step five
// launches (~34 us in a CUDA graph, BASELINE config 1), against 80-190 us of CPU
// work per step.  Here one cluster of up to 16 blocks (one per SM, SMALL_THREADS
// threads each) runs a batch of up to thousands of heun_step calls in one launch.
// Each thread owns cells; a cell's stage is one straight computation: the
// primitives of its cross stencil (ghosts read through an index map of the
// reference's fill, so no fill phase), its four faces and its update (a face is
// solved by both of its cells, the same bits twice; the lower one stores it for
// the Heun average and the outflow).  A Heun step is two cluster barriers: the
// blocks' partial reductions are broadcast to every block by plain shared::cluster
// stores (no remote atomics) and every block derives the next dt / time itself; the
// lead block writes the step records and runs the ordered boundary-outflow sums;
// the state ping-pongs between U and U2, and data
// another block wrote is read through L2 (ld.global.cg after the barrier's
// release / acquire).
//
// Arithmetic: the fast kernels' exact arithmetic (face_fast.cuh: shared
// reciprocals, sweby_fast, the cell box) where its proofs hold (beta >= 1, gamma - 1
// in the constant box), else the stage-wise kernels' IEEE expressions
// (lagflux_device.cuh) -- the reference's bits either way.  A failed check or a
// cell outside the box ends the batch at that step with its input state intact;
// the host re-runs it with the stage-wise kernels, which report the reference's
// exact error (a box failure whose re-run succeeds switches the handle to the IEEE
// arithmetic until the next upload).
//
// Grid mode (more than 16 x 224 cells, or a perimeter whose boundary faces do not fit
// in shared memory): a cooperative launch of up to one block per SM, grid barriers
// instead of cluster barriers, the block partials through global memory (every block
// combines them), and every step's boundary faces into a history buffer whose ordered
// outflow sums run after the batch (k_small_sums, then k_small_accum in step order).
//
// Reference: solver.cpp:489-546 (heun_step), 482-487 (time_order 1 stage),
// 131-329 (the phases), 406-432 (outflow), 434-480 (dt); grid.cpp:72-114 (fill).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "face_fast.cuh"
#include "fused.h"
#include "fused_common.cuh"
#include "handle.h"
#include "reduce.cuh"
#include "small.h"
#include "trace.h"

namespace lfb {

namespace {

#ifndef LF_SMALL_THREADS
#define LF_SMALL_THREADS 224   // + one outflow warp: 8 warps, 2 per scheduler
#endif
constexpr int SMALL_THREADS = LF_SMALL_THREADS;

struct SmallArgs {
  double* u;    // U^n (Field origin pointers; ping-pong with u2)
  double* u2;
  double* us;   // U* (Heun predictor)
  int64_t pitch, fstride;
  double* fx[2];   // face fluxes of the two stages (FluxArr layout: [c][b][a])
  double* fy[2];
  int ob;          // doubles per boundary-face block (outflow sums; see k_small_run)
  int64_t fx_stride, fy_stride;
  int nx, ny;
  int heun;
  int bc[4];
  Consts k;
  double cfl, limit, t_final;
  StepCtl* ctl;      // in: the state's control record; out: the last state's
  StepRec* rec;      // [nsteps]
  double* outflow;   // [4], accumulated in place
  int nsteps;
  // multimaterial (MAT kernels): partial densities (Layout of the field, nmat components)
  // of U^n, U* and U^{n+1}, the stage-1 closure's fractions of every interior cell and
  // the stage-1 faces' u* (the corrector's stage-a material fluxes are rebuilt from them)
  int nmat;
  double gam[8];
  double* p;
  double* p2;
  double* ps;
  double* y0;
  double* usx0;
  double* usy0;
  // grid mode (a cooperative grid of up to one block per SM, beyond one cluster):
  unsigned long long* gpart;   // [2 parities][6 fields][SMALL_MAX_GRID] block partials
  double* bhist;               // [nsteps][ob] every step's boundary faces (summed after
                               // the kernel, k_small_sums / k_small_accum)
};

constexpr int SMALL_MAX_CTAS = 16;     // one cluster (non-portable maximum)
constexpr int SMALL_MAX_GRID = 1024;   // grid mode: blocks (one per SM in practice)
constexpr int SMALL_MAX_MAT = 8;       // materials on this path (more: the stage-wise kernels)
constexpr int SMALL_NPART = 6;         // reduced fields: rate, min rho, min e, fail, dtfail, min p

// Per block: its own partial reductions; in the lead block (rank 0) also the
// control record and every block's partials (written there by plain
// shared::cluster stores -- no remote atomics), and the outflow staging tile.
struct SmallShared {
  StepCtl ctl;                             // this block's copy (every block computes it)
  unsigned long long rate, min_r, min_e, min_pk;   // this block's partials
  int fail, dtfail, stop;
  unsigned long long g_rate, g_min_r, g_min_e, g_min_pk;   // grid mode: the combined partials
  int g_fail, g_dtfail;
  // every block's partials, in every block, by step parity (a fast block's next step
  // must not overwrite a slot a slow block has not read)
  unsigned long long p_rate[2][SMALL_MAX_CTAS], p_min_r[2][SMALL_MAX_CTAS],
      p_min_e[2][SMALL_MAX_CTAS], p_min_pk[2][SMALL_MAX_CTAS];
  int p_fail[2][SMALL_MAX_CTAS], p_dtfail[2][SMALL_MAX_CTAS];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// the same shared-memory variable in block `rank` of the cluster
__device__ __forceinline__ uint32_t remote(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_remote(uint32_t a, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void st_remote_d(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_remote(uint32_t a, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <class Op>
__device__ __forceinline__ unsigned long long wred(unsigned long long v, Op op) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// build_primitives (solver.cpp:145-170) of cell (i, j) of the ghosted grid, read
// through the ghost map; bad |= the reference's check
template <bool DIM2, bool FAST>
__device__ __forceinline__ void cell_prims(const SmallArgs& a, const double* f, int i, int j,
                                           double w[4], bool& bad) {
  bool fx, fy = false;
  // (the ghost fill as an index map, layout.cuh: no fill phase)
  const int is = ghost_src(i, a.nx, a.bc[0], a.bc[1], fx);
  const int js = DIM2 ? ghost_src(j, a.ny, a.bc[2], a.bc[3], fy) : 0;
  const int64_t o = (int64_t)js * a.pitch + is;
  const double r = __ldcg(f + o);
  double mx = __ldcg(f + a.fstride + o), my = __ldcg(f + 2 * a.fstride + o);
  const double e = __ldcg(f + 3 * a.fstride + o);
  if (fx) mx = -1.0 * mx;   // sx * row[...] (grid.cpp:86-94)
  if (fy) my = -1.0 * my;
  if constexpr (FAST) {
    // the fast reciprocal; the cell box implies the reference's checks and proves
    // every division / square root of the faces this cell feeds (face_fast.cuh)
    bool dead = true;
    prim_fast(r, mx, my, e, a.k.gm1, w, dead);
    if (!cell_in_box(w)) bad = true;
  } else {
    w[0] = 0.0;
    w[1] = w[2] = w[3] = 0.0;
    if (!(r > 0.0)) {
      bad = true;
    } else {
      w[0] = r;
      primitive(r, mx, my, e, a.k.gm1, w[1], w[2], w[3]);
      bad = bad || !(w[3] > 0.0);
    }
  }
}

// the two faces of a cell along one axis (compute_fluxes, solver.cpp:196-239):
// s[0..4] = the cells c-2 .. c+2; lo face (c-1 | c) and hi face (c | c+1)
template <int AXIS, bool MUSCL, bool FAST>
__device__ __forceinline__ void cell_faces(const SmallArgs& a, const FK& fk,
                                           const double (&s)[5][4], double flo[4], double fhi[4],
                                           bool& bad) {
  double m_lo[4], p_lo[4], m_hi[4], p_hi[4];
  if constexpr (FAST) {
    // the fast kernels' traces (sweby_fast: beta >= 1) and face solves (face_fast.cuh)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double lo;
      cell_traces<MUSCL>(s[0][c], s[1][c], s[2][c], fk.beta, lo, m_lo[c]);
      cell_traces<MUSCL>(s[1][c], s[2][c], s[3][c], fk.beta, p_lo[c], m_hi[c]);
      double hi;
      cell_traces<MUSCL>(s[2][c], s[3][c], s[4][c], fk.beta, p_hi[c], hi);
    }
    if (!traces_ok(m_lo[0], m_lo[3], p_lo[0], p_lo[3]) ||
        !traces_ok(m_hi[0], m_hi[3], p_hi[0], p_hi[3]))
      bad = true;
    bool dead = true;
    double ps0, us0, ps1, us1;
    face_fast<AXIS>(m_lo[0], m_lo[1], m_lo[2], m_lo[3], p_lo[0], p_lo[1], p_lo[2], p_lo[3], fk, flo,
                    dead, ps0, us0);
    face_fast<AXIS>(m_hi[0], m_hi[1], m_hi[2], m_hi[3], p_hi[0], p_hi[1], p_hi[2], p_hi[3], fk, fhi,
                    dead, ps1, us1);
    if (needs_mean(us0))
      face_mean<AXIS>(m_lo[0], m_lo[1], m_lo[2], m_lo[3], p_lo[0], p_lo[1], p_lo[2], p_lo[3], ps0,
                      us0, fk, flo, dead);
    if (needs_mean(us1))
      face_mean<AXIS>(m_hi[0], m_hi[1], m_hi[2], m_hi[3], p_hi[0], p_hi[1], p_hi[2], p_hi[3], ps1,
                      us1, fk, fhi, dead);
  } else {
  #pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (MUSCL) {
        // muscl_face_trace (reconstruct.hpp:44-49): each cell's limited slope serves
        // both of its faces
        const double s1 = slope3(s[0][c], s[1][c], s[2][c], a.k.beta);
        const double s2 = slope3(s[1][c], s[2][c], s[3][c], a.k.beta);
        const double s3 = slope3(s[2][c], s[3][c], s[4][c], a.k.beta);
        m_lo[c] = s[1][c] + 0.5 * s1;
        p_lo[c] = s[2][c] - 0.5 * s2;
        m_hi[c] = s[2][c] + 0.5 * s2;
        p_hi[c] = s[3][c] - 0.5 * s3;
      } else {
        m_lo[c] = s[1][c];
        p_lo[c] = s[2][c];
        m_hi[c] = s[2][c];
        p_hi[c] = s[3][c];
      }
      flo[c] = fhi[c] = 0.0;
    }
    if (traces_ok(m_lo[0], m_lo[3], p_lo[0], p_lo[3]))
      face_flux<AXIS>(m_lo[0], m_lo[1], m_lo[2], m_lo[3], p_lo[0], p_lo[1], p_lo[2], p_lo[3], a.k, flo);
    else
      bad = true;
    if (traces_ok(m_hi[0], m_hi[3], p_hi[0], p_hi[3]))
      face_flux<AXIS>(m_hi[0], m_hi[1], m_hi[2], m_hi[3], p_hi[0], p_hi[1], p_hi[2], p_hi[3], a.k, fhi);
    else
      bad = true;
  }
}

// One stage for interior cell (i, j): primitives of its cross stencil, its four
// faces, apply_update (solver.cpp:272-308).  Stage 1 (!TWO) stores its faces (a
// cell owns its low faces, the last cell of a row / column the high one too);
// stage 2 stores its own and reads stage 1's for F = 0.5 (F^n + F*).
template <bool DIM2, bool MUSCL, bool FAST, bool TWO>
__device__ __forceinline__ void cell_stage(const SmallArgs& a, const FK& fk, const double* in,
                                           const double* base, int i, int j, uint32_t rb,
                                           double* gb, double lam_x, double lam_y, double vals[4],
                                           bool& bad) {
  // the step's domain-boundary faces (Heun-averaged as k_gather_boundary) into its
  // boundary block [left 4 ny | right 4 ny | bottom 4 nx | top 4 nx]: the lead block's
  // shared memory (cluster) or the step's slot of the history (grid)
  auto put = [&](int idx, double v) {
    if (rb)
      st_remote_d(rb + 8u * idx, v);
    else
      __stcg(gb + idx, v);
  };
  const int64_t o = (int64_t)j * a.pitch + i;   // (cells and low faces share offsets)
  // the operands that do not depend on this stage's faces, loaded first
  double u0[4], fnl[4], fnr[4], fnb[4], fnt[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    u0[c] = __ldcg(base + c * a.fstride + o);
    if (TWO) {
      const double* fa = a.fx[0] + c * a.fx_stride;
      fnl[c] = __ldcg(fa + o);
      fnr[c] = __ldcg(fa + o + 1);
      if (DIM2) {
        const double* fb = a.fy[0] + c * a.fy_stride;
        fnb[c] = __ldcg(fb + o);
        fnt[c] = __ldcg(fb + o + a.pitch);
      }
    }
  }
  double fxl[4], fxr[4], fyb[4], fyt[4];
  {
    double s[5][4];
#pragma unroll
    for (int d = 0; d < 5; ++d) cell_prims<DIM2, FAST>(a, in, i - 2 + d, j, s[d], bad);
    cell_faces<0, MUSCL, FAST>(a, fk, s, fxl, fxr, bad);
  }
  if (DIM2) {
    double s[5][4];
#pragma unroll
    for (int d = 0; d < 5; ++d) cell_prims<DIM2, FAST>(a, in, i, j - 2 + d, s[d], bad);
    cell_faces<1, MUSCL, FAST>(a, fk, s, fyb, fyt, bad);
  }
  const int k = TWO ? 1 : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double* fx = a.fx[k] + c * a.fx_stride;
    __stcg(fx + o, fxl[c]);
    if (i == a.nx - 1) __stcg(fx + o + 1, fxr[c]);
    if (DIM2) {
      double* fy = a.fy[k] + c * a.fy_stride;
      __stcg(fy + o, fyb[c]);
      if (j == a.ny - 1) __stcg(fy + o + a.pitch, fyt[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double l = fxl[c], r = fxr[c];
    if (TWO) {
      l = 0.5 * (fnl[c] + l);
      r = 0.5 * (fnr[c] + r);
    }
    double val = u0[c] - lam_x * (r - l);
    if (DIM2) {
      double b = fyb[c], t = fyt[c];
      if (TWO) {
        b = 0.5 * (fnb[c] + b);
        t = 0.5 * (fnt[c] + t);
      }
      val -= lam_y * (t - b);
      if (rb || gb) {
        if (j == 0) put(8 * a.ny + c * a.nx + i, b);
        if (j == a.ny - 1) put(8 * a.ny + 4 * a.nx + c * a.nx + i, t);
      }
    }
    if (rb || gb) {
      if (i == 0) put(c * a.ny + j, l);
      if (i == a.nx - 1) put(4 * a.ny + c * a.ny + j, r);
    }
    vals[c] = val;
  }
}

// ---------------------------------------------------------------- multimaterial
// (MAT kernels; the stage-wise kernels' IEEE expressions, material_kernels.cu)

// order-preserving key of a non-NaN double (unsigned compare == IEEE compare)
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// fill_all_ghosts' closure (solver.cpp:100-121): the clamped fractions of a cell's
// partials and its mixed-cell gamma; bad: a fraction beyond round-off
template <int KM>
__device__ __forceinline__ double closure(const SmallArgs& a, const double* pk, int64_t o, double r,
                                          double y[KM], bool& bad) {
  double ysum = 0.0, gp = 0.0;
  int pure = -1;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= a.nmat) break;
    const double raw = __ldcg(pk + k * a.fstride + o) / r;
    double yk = raw;
    if (yk < 0.0 || yk > 1.0) {
      if (raw < -1e-11 || raw > 1.0 + 1e-11) {
        bad = true;
        yk = 0.0;
      } else {
        yk = raw < 0.0 ? 0.0 : 1.0;
      }
    }
    y[k] = yk;
    if (yk == 1.0) pure = k;
    ysum += yk / (a.gam[k] - 1.0);
  }
#pragma unroll
  for (int k = 0; k < KM; ++k)
    if (k < a.nmat && pure == k) gp = a.gam[k];
  return pure >= 0 ? gp : 1.0 + 1.0 / ysum;
}

// a stencil cell (i, j) read through the ghost map (partials: even parity): its closure
// and its primitives with that gamma (build_primitives, solver.cpp:145-163)
template <bool DIM2, int KM>
__device__ __forceinline__ void mat_cell(const SmallArgs& a, const double* f, const double* pk,
                                         int i, int j, double w[4], double& g, double y[KM],
                                         bool& bad) {
  bool fx, fy = false;
  const int is = ghost_src(i, a.nx, a.bc[0], a.bc[1], fx);
  const int js = DIM2 ? ghost_src(j, a.ny, a.bc[2], a.bc[3], fy) : 0;
  const int64_t o = (int64_t)js * a.pitch + is;
  const double r = __ldcg(f + o);
  double mx = __ldcg(f + a.fstride + o), my = __ldcg(f + 2 * a.fstride + o);
  const double e = __ldcg(f + 3 * a.fstride + o);
  if (fx) mx = -1.0 * mx;
  if (fy) my = -1.0 * my;
  g = closure<KM>(a, pk, o, r, y, bad);
  w[0] = w[1] = w[2] = w[3] = 0.0;
  if (!(r > 0.0)) {
    bad = true;
  } else {
    w[0] = r;
    primitive(r, mx, my, e, g - 1.0, w[1], w[2], w[3]);
    if (!(w[3] > 0.0)) bad = true;
  }
}

// the fractions a stage-1 closure stored for cell (i, j) (ghosts: the source cell's)
template <bool DIM2, int KM>
__device__ __forceinline__ void stored_fractions(const SmallArgs& a, int i, int j, double y[KM]) {
  bool f;
  const int is = ghost_src(i, a.nx, a.bc[0], a.bc[1], f);
  const int js = DIM2 ? ghost_src(j, a.ny, a.bc[2], a.bc[3], f) : 0;
  const int64_t o = (int64_t)js * a.pitch + is;
#pragma unroll
  for (int k = 0; k < KM; ++k)
    if (k < a.nmat) y[k] = __ldcg(a.y0 + k * a.fstride + o);
}

// lagrangian_hll + contact_flux with each side's own EOS (solver.cpp:228-238)
template <int AXIS>
__device__ __forceinline__ void face_g(const double wm[4], const double wp[4], double el,
                                       double er, double f[4], double& us) {
  const double ul = AXIS == 0 ? wm[1] : wm[2];
  const double ur = AXIS == 0 ? wp[1] : wp[2];
  const double cl = sqrt(el * wm[3] / wm[0]);
  const double cr = sqrt(er * wp[3] / wp[0]);
  const double cmax = smax(cl, cr);
  const double rho_sum = wm[0] + wp[0];
  const double ps =
      (wp[0] * wm[3] + wm[0] * wp[3]) / rho_sum - (wm[0] * wp[0] / rho_sum) * cmax * (ur - ul);
  us = (wm[0] * ul + wp[0] * ur) / rho_sum - (wp[3] - wm[3]) / (cmax * rho_sum);
  double a0, a1, a2, a3;
  if (us > 0.0) {
    a0 = wm[0];
    a1 = wm[0] * wm[1];
    a2 = wm[0] * wm[2];
    a3 = wm[3] / (el - 1.0) + 0.5 * wm[0] * (wm[1] * wm[1] + wm[2] * wm[2]);
  } else if (us < 0.0) {
    a0 = wp[0];
    a1 = wp[0] * wp[1];
    a2 = wp[0] * wp[2];
    a3 = wp[3] / (er - 1.0) + 0.5 * wp[0] * (wp[1] * wp[1] + wp[2] * wp[2]);
  } else {
    const double m1 = wm[0] * wm[1], m2 = wm[0] * wm[2];
    const double m3 = wm[3] / (el - 1.0) + 0.5 * wm[0] * (wm[1] * wm[1] + wm[2] * wm[2]);
    const double p1 = wp[0] * wp[1], p2 = wp[0] * wp[2];
    const double p3 = wp[3] / (er - 1.0) + 0.5 * wp[0] * (wp[1] * wp[1] + wp[2] * wp[2]);
    a0 = 0.5 * (wm[0] + wp[0]);
    a1 = 0.5 * (m1 + p1);
    a2 = 0.5 * (m2 + p2);
    a3 = 0.5 * (m3 + p3);
  }
  f[0] = a0 * us;
  f[1] = AXIS == 0 ? a1 * us + ps : a1 * us;
  f[2] = AXIS == 1 ? a2 * us + ps : a2 * us;
  f[3] = a3 * us + ps * us;
}

// edge_material_flux (solver.cpp:345-357) added to acc as gather does (acc += w t)
template <int KM>
__device__ __forceinline__ void add_mat_flux(const SmallArgs& a, double mass, double us,
                                             const double ylo[KM], const double yhi[KM], double w,
                                             double acc[KM]) {
  double rest = mass;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= a.nmat) break;
    double fk;
    if (k < a.nmat - 1) {
      fk = us == 0.0 ? 0.0 : mass * (us > 0.0 ? ylo[k] : yhi[k]);
      rest -= fk;
    } else {
      fk = us == 0.0 ? 0.0 : rest;
    }
    acc[k] += w * fk;
  }
}

// The two faces of a cell along one axis with the cells' own EOS; traces as cell_faces
template <int AXIS, bool MUSCL>
__device__ __forceinline__ void mat_faces(const SmallArgs& a, const double (&s)[5][4],
                                          const double (&g)[5], double flo[4], double fhi[4],
                                          double& uslo, double& ushi, bool& bad) {
  double m_lo[4], p_lo[4], m_hi[4], p_hi[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (MUSCL) {
      const double s1 = slope3(s[0][c], s[1][c], s[2][c], a.k.beta);
      const double s2 = slope3(s[1][c], s[2][c], s[3][c], a.k.beta);
      const double s3 = slope3(s[2][c], s[3][c], s[4][c], a.k.beta);
      m_lo[c] = s[1][c] + 0.5 * s1;
      p_lo[c] = s[2][c] - 0.5 * s2;
      m_hi[c] = s[2][c] + 0.5 * s2;
      p_hi[c] = s[3][c] - 0.5 * s3;
    } else {
      m_lo[c] = s[1][c];
      p_lo[c] = s[2][c];
      m_hi[c] = s[2][c];
      p_hi[c] = s[3][c];
    }
    flo[c] = fhi[c] = 0.0;
  }
  uslo = ushi = 0.0;
  if (traces_ok(m_lo[0], m_lo[3], p_lo[0], p_lo[3]))
    face_g<AXIS>(m_lo, p_lo, g[1], g[2], flo, uslo);
  else
    bad = true;
  if (traces_ok(m_hi[0], m_hi[3], p_hi[0], p_hi[3]))
    face_g<AXIS>(m_hi, p_hi, g[2], g[3], fhi, ushi);
  else
    bad = true;
}

// One multimaterial stage for interior cell (i, j): closures and primitives of the cross
// stencil, the four faces with per-side EOS, apply_update (solver.cpp:272-308) and
// update_partials (solver.cpp:331-404).  Stage 1 (!TWO) stores its faces, their u* and
// this cell's fractions (the corrector's stage-a material fluxes); stage 2 rebuilds
// those and accumulates as gather does: (0 + 0.5 a) + 0.5 b.
template <bool DIM2, bool MUSCL, bool TWO, int KM>
__device__ __forceinline__ void cell_stage_mat(const SmallArgs& a, const double* in,
                                               const double* pin, const double* base,
                                               const double* pbase, int i, int j, uint32_t rb,
                                               double* gb, double lam_x, double lam_y,
                                               double vals[4], double pv[KM],
                                               bool& bad) {
  auto put = [&](int idx, double v) {
    if (rb)
      st_remote_d(rb + 8u * idx, v);
    else
      __stcg(gb + idx, v);
  };
  const int64_t o = (int64_t)j * a.pitch + i;
  double u0[4], fnl[4], fnr[4], fnb[4], fnt[4];
  double usl0 = 0.0, usr0 = 0.0, usb0 = 0.0, ust0 = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    u0[c] = __ldcg(base + c * a.fstride + o);
    if (TWO) {
      const double* fa = a.fx[0] + c * a.fx_stride;
      fnl[c] = __ldcg(fa + o);
      fnr[c] = __ldcg(fa + o + 1);
      if (DIM2) {
        const double* fb = a.fy[0] + c * a.fy_stride;
        fnb[c] = __ldcg(fb + o);
        fnt[c] = __ldcg(fb + o + a.pitch);
      }
    }
  }
  if (TWO) {
    usl0 = __ldcg(a.usx0 + o);
    usr0 = __ldcg(a.usx0 + o + 1);
    if (DIM2) {
      usb0 = __ldcg(a.usy0 + o);
      ust0 = __ldcg(a.usy0 + o + a.pitch);
    }
  }
  // partial-flux accumulators of the four faces
  double ml[KM], mr[KM], mb[KM], mt[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) ml[k] = mr[k] = mb[k] = mt[k] = 0.0;
  const double w = TWO ? 0.5 : 1.0;
  double ymid[KM];   // this cell's fractions (this stage's closure)
  double fxl[4], fxr[4], fyb[4], fyt[4], usl, usr, usb = 0.0, ust = 0.0;
  {
    double s[5][4], g[5], yl[KM], yr[KM], yd[KM];
    mat_cell<DIM2, KM>(a, in, pin, i - 2, j, s[0], g[0], yd, bad);
    mat_cell<DIM2, KM>(a, in, pin, i - 1, j, s[1], g[1], yl, bad);
    mat_cell<DIM2, KM>(a, in, pin, i, j, s[2], g[2], ymid, bad);
    mat_cell<DIM2, KM>(a, in, pin, i + 1, j, s[3], g[3], yr, bad);
    mat_cell<DIM2, KM>(a, in, pin, i + 2, j, s[4], g[4], yd, bad);
    mat_faces<0, MUSCL>(a, s, g, fxl, fxr, usl, usr, bad);
    if (TWO) {   // stage a: the stage-1 faces with the stage-1 fractions
      double y0l[KM], y0m[KM], y0r[KM];
      stored_fractions<DIM2, KM>(a, i - 1, j, y0l);
      stored_fractions<DIM2, KM>(a, i, j, y0m);
      stored_fractions<DIM2, KM>(a, i + 1, j, y0r);
      add_mat_flux<KM>(a, fnl[0], usl0, y0l, y0m, w, ml);
      add_mat_flux<KM>(a, fnr[0], usr0, y0m, y0r, w, mr);
    }
    add_mat_flux<KM>(a, fxl[0], usl, yl, ymid, w, ml);
    add_mat_flux<KM>(a, fxr[0], usr, ymid, yr, w, mr);
  }
  if (DIM2) {
    double s[5][4], g[5], yb[KM], yt[KM], yd[KM];
    mat_cell<DIM2, KM>(a, in, pin, i, j - 2, s[0], g[0], yd, bad);
    mat_cell<DIM2, KM>(a, in, pin, i, j - 1, s[1], g[1], yb, bad);
    mat_cell<DIM2, KM>(a, in, pin, i, j, s[2], g[2], yd, bad);
    mat_cell<DIM2, KM>(a, in, pin, i, j + 1, s[3], g[3], yt, bad);
    mat_cell<DIM2, KM>(a, in, pin, i, j + 2, s[4], g[4], yd, bad);
    mat_faces<1, MUSCL>(a, s, g, fyb, fyt, usb, ust, bad);
    if (TWO) {
      double y0b[KM], y0m[KM], y0t[KM];
      stored_fractions<DIM2, KM>(a, i, j - 1, y0b);
      stored_fractions<DIM2, KM>(a, i, j, y0m);
      stored_fractions<DIM2, KM>(a, i, j + 1, y0t);
      add_mat_flux<KM>(a, fnb[0], usb0, y0b, y0m, w, mb);
      add_mat_flux<KM>(a, fnt[0], ust0, y0m, y0t, w, mt);
    }
    add_mat_flux<KM>(a, fyb[0], usb, yb, ymid, w, mb);
    add_mat_flux<KM>(a, fyt[0], ust, ymid, yt, w, mt);
  }
  const int k = TWO ? 1 : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double* fx = a.fx[k] + c * a.fx_stride;
    __stcg(fx + o, fxl[c]);
    if (i == a.nx - 1) __stcg(fx + o + 1, fxr[c]);
    if (DIM2) {
      double* fy = a.fy[k] + c * a.fy_stride;
      __stcg(fy + o, fyb[c]);
      if (j == a.ny - 1) __stcg(fy + o + a.pitch, fyt[c]);
    }
  }
  if (!TWO) {   // the corrector's stage-a inputs: u* of the faces, this cell's fractions
    __stcg(a.usx0 + o, usl);
    if (i == a.nx - 1) __stcg(a.usx0 + o + 1, usr);
    if (DIM2) {
      __stcg(a.usy0 + o, usb);
      if (j == a.ny - 1) __stcg(a.usy0 + o + a.pitch, ust);
    }
#pragma unroll
    for (int kk = 0; kk < KM; ++kk)
      if (kk < a.nmat) __stcg(a.y0 + kk * a.fstride + o, ymid[kk]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double l = fxl[c], r = fxr[c];
    if (TWO) {
      l = 0.5 * (fnl[c] + l);
      r = 0.5 * (fnr[c] + r);
    }
    double val = u0[c] - lam_x * (r - l);
    if (DIM2) {
      double b = fyb[c], t = fyt[c];
      if (TWO) {
        b = 0.5 * (fnb[c] + b);
        t = 0.5 * (fnt[c] + t);
      }
      val -= lam_y * (t - b);
      if (rb || gb) {
        if (j == 0) put(8 * a.ny + c * a.nx + i, b);
        if (j == a.ny - 1) put(8 * a.ny + 4 * a.nx + c * a.nx + i, t);
      }
    }
    if (rb || gb) {
      if (i == 0) put(c * a.ny + j, l);
      if (i == a.nx - 1) put(4 * a.ny + c * a.ny + j, r);
    }
    vals[c] = val;
  }
#pragma unroll
  for (int kk = 0; kk < KM; ++kk) {
    if (kk >= a.nmat) break;
    double val = __ldcg(pbase + kk * a.fstride + o) - lam_x * (mr[kk] - ml[kk]);
    if (DIM2) val -= lam_y * (mt[kk] - mb[kk]);
    pv[kk] = val;
  }
}

// accumulate_boundary_outflow (solver.cpp:406-432) of a completed step, by lanes 0-3
// (x: s += right - left over the rows in order) and 4-7 (y: s += top - bottom over the
// columns) of one warp, from the step's boundary block in shared memory; then
// outflow += dt dy s_x, += dt dx s_y.
template <bool DIM2>
__device__ void outflow_sums(const SmallArgs& a, const double* sb, double dt) {
  const int lane = threadIdx.x & 31;
  if (lane < 8) {
    const int q = lane & 3;
    double s = 0.0;
    if (lane < 4) {
      const double* L = sb + q * a.ny;
      const double* R = L + 4 * a.ny;
#pragma unroll 8
      for (int j = 0; j < a.ny; ++j) s += R[j] - L[j];
    } else if (DIM2) {
      const double* B = sb + 8 * a.ny + q * a.nx;
      const double* T = B + 4 * a.nx;
#pragma unroll 8
      for (int i = 0; i < a.nx; ++i) s += T[i] - B[i];
    }
    const double ax = dt * (DIM2 ? a.k.dy : 1.0), ay = dt * a.k.dx;
    if (lane < 4) a.outflow[q] += ax * s;
    __syncwarp(0xffu);
    if (DIM2 && lane >= 4) a.outflow[q] += ay * s;
  }
  __syncwarp();
}

template <bool DIM2, bool MUSCL, bool FAST, bool GRID, int KM>
__global__ void __launch_bounds__(SMALL_THREADS + 32, 1) k_small_run(SmallArgs a) {
  // KM: 0 one material; else the material kernels' array bound (nmat <= KM)
  constexpr bool MAT = KM > 0;
  constexpr int KA = KM > 0 ? KM : 1;
  namespace cg = cooperative_groups;
  __shared__ SmallShared sh;
  // GRID: a cooperative grid (one block per SM) synchronised by grid barriers; else one
  // cluster synchronised by barrier.cluster (both release / acquire the global stores)
  auto sync_all = [&]() {
    if constexpr (GRID)
      cg::this_grid().sync();
    else
      cg::this_cluster().sync();
  };
  // two boundary blocks (step parity): a step's boundary faces, stored by the cells
  // that own them in its last stage, summed by the lead's outflow warp during the
  // next step's first stage
  extern __shared__ double sbnd[];
  const int tid = threadIdx.x;
  const bool cellw = tid < SMALL_THREADS;   // cell warps; the last warp sums the outflow
  const uint32_t rank = GRID ? blockIdx.x : cg::this_cluster().block_rank();
  const uint32_t nblk = GRID ? gridDim.x : cg::this_cluster().num_blocks();
  const bool lead = rank == 0;
  const int gtid = (int)rank * SMALL_THREADS + tid;
  const int gthreads = (int)nblk * SMALL_THREADS;
  if (tid == 0) sh.ctl = *a.ctl;
  const FK fk = make_fk(a.k.gamma, a.k.gm1, a.k.beta, a.k.dx, a.k.dy);
  double* u = a.u;
  double* u2 = a.u2;
  double* pk = a.p;     // (MAT) partial densities of U^n / U^{n+1}
  double* pk2 = a.p2;
  const MaxOp mx;
  const MinOp mn;
  const int ncell = a.nx * a.ny;
  int pend = -1, pend_par = 0;   // (lead outflow warp) a completed step whose sums are due
  double pend_dt = 0.0;
  int n = 0;
  for (; n < a.nsteps; ++n) {
    if (tid == 0) {
      sh.rate = 0ull;
      sh.min_r = sh.min_e = 0x7ff0000000000000ull;
      sh.fail = sh.dtfail = 0;
      sh.min_pk = ~0ull;
      sh.g_rate = 0ull;
      sh.g_min_r = sh.g_min_e = 0x7ff0000000000000ull;
      sh.g_min_pk = ~0ull;
      sh.g_fail = sh.g_dtfail = 0;
    }
    __syncthreads();   // (this block's control record of the step, the resets)
    const StepCtl c = sh.ctl;
    if (c.done) break;
    // compute_dt's tail (solver.cpp:471-479) from the rate of the input state
    const double rate = __longlong_as_double((long long)c.rate_bits);
    double dt = a.cfl / rate;
    if (c.time + dt > a.limit) dt = a.limit - c.time;
    if (c.dtfail || !(dt > 0.0)) break;
    const double lam_x = dt / a.k.dx;  // solver.cpp:262-263
    const double lam_y = dt / a.k.dy;
    const int par = n & 1;
    const uint32_t rb = GRID ? 0u : remote(sbnd + par * a.ob, 0);
    double* const gb = GRID ? a.bhist + (int64_t)n * a.ob : nullptr;
    bool bad = false, dtbad = false;
    unsigned long long mr = 0x7ff0000000000000ull, me = 0x7ff0000000000000ull, rk = 0ull;
    unsigned long long mpk = ~0ull;   // (MAT) min p (order key)
    // the last stage's cell: positivity (solver.cpp:300-307), minima, and the next
    // step's CFL rate (solver.cpp:449-470) of the new value
    auto finish = [&](const double v[4]) {
      const double eint = internal_energy(v[0], v[1], v[2], v[3]);
      if (!(v[0] > 0.0) || !(eint > 0.0)) {
        bad = true;
      } else {
        const unsigned long long r = pos_bits(v[0]), e = pos_bits(eint);
        mr = r < mr ? r : mr;
        me = e < me ? e : me;
      }
      double rr;
      if (cfl_rate<DIM2>(v[0], v[1], v[2], v[3], a.k, rr)) {
        if (rr == rr) {
          const unsigned long long b = pos_bits(rr);
          rk = b > rk ? b : rk;
        }
      } else {
        dtbad = true;
      }
    };
    // (MAT) the last stage's cell: positivity and min rho as above; min p from the fresh
    // partials (solver.cpp:522-538); the next step's CFL rate with the mixed-cell gamma of
    // the next fill's closure (solver.cpp:449-470 with gamma_[0]; a fraction beyond
    // round-off there fails the next step)
    auto finish_mat = [&](const double v[4], const double pv[KA]) {
      const double eint = internal_energy(v[0], v[1], v[2], v[3]);
      if (!(v[0] > 0.0) || !(eint > 0.0)) {
        bad = true;
      } else {
        const unsigned long long r = pos_bits(v[0]), e = pos_bits(eint);
        mr = r < mr ? r : mr;
        me = e < me ? e : me;
      }
      const double r = v[0];
      double sm = 0.0, ysum = 0.0, gp = 0.0;
      int pure = -1;
      bool fbad = false;
#pragma unroll
      for (int k = 0; k < KA; ++k) {
        if (k >= a.nmat) break;
        sm += (pv[k] / r) / (a.gam[k] - 1.0);
        const double raw = pv[k] / r;
        double yk = raw;
        if (yk < 0.0 || yk > 1.0) {
          if (raw < -1e-11 || raw > 1.0 + 1e-11) {
            fbad = true;
            yk = 0.0;
          } else {
            yk = raw < 0.0 ? 0.0 : 1.0;
          }
        }
        if (yk == 1.0) pure = k;
        ysum += yk / (a.gam[k] - 1.0);
      }
      const double x = (v[3] - 0.5 * (v[1] * v[1] + v[2] * v[2]) / r) / sm;
      if (x == x) {
        const unsigned long long key = order_key(x);
        mpk = key < mpk ? key : mpk;
      }
#pragma unroll
      for (int k = 0; k < KA; ++k)
        if (k < a.nmat && pure == k) gp = a.gam[k];
      const double g = pure >= 0 ? gp : 1.0 + 1.0 / ysum;
      bool ok = !fbad && r > 0.0;
      if (ok) {
        const double inv = 1.0 / r;
        const double uu = v[1] * inv, vv = v[2] * inv;
        const double p = (g - 1.0) * (v[3] - 0.5 * (v[1] * v[1] + v[2] * v[2]) * inv);
        ok = p > 0.0;
        if (ok) {
          const double cs = sqrt(g * p * inv);
          double rr = (fabs(uu) + cs) / a.k.dx;
          if (DIM2) rr += (fabs(vv) + cs) / a.k.dy;
          if (rr == rr) {
            const unsigned long long b = pos_bits(rr);
            rk = b > rk ? b : rk;
          }
        }
      }
      if (!ok) dtbad = true;
    };
    if (MAT && cellw) {
      // stage 1: (U^n, P^n) -> (U*, P*) (or the next state when time_order = 1)
      for (int t = gtid; t < ncell; t += gthreads) {
        const int i = t % a.nx, j = t / a.nx;
        double v[4], pv[KA];
        cell_stage_mat<DIM2, MUSCL, false, KA>(a, u, pk, u, pk, i, j, a.heun ? 0u : rb,
                                           a.heun ? nullptr : gb, lam_x, lam_y, v, pv, bad);
        const int64_t o = (int64_t)j * a.pitch + i;
        double* out = a.heun ? a.us : u2;
        double* pout = a.heun ? a.ps : pk2;
#pragma unroll
        for (int q = 0; q < 4; ++q) __stcg(out + q * a.fstride + o, v[q]);
#pragma unroll
        for (int q = 0; q < KA; ++q)
          if (q < a.nmat) __stcg(pout + q * a.fstride + o, pv[q]);
        if (a.heun) {
          const double eint = internal_energy(v[0], v[1], v[2], v[3]);
          if (!(v[0] > 0.0) || !(eint > 0.0)) bad = true;
        } else {
          finish_mat(v, pv);
        }
      }
    } else if (cellw) {
      // stage 1: U^n -> U* (or U^{n+1} when time_order = 1)
      for (int t = gtid; t < ncell; t += gthreads) {
        const int i = t % a.nx, j = t / a.nx;
        double v[4];
        cell_stage<DIM2, MUSCL, FAST, false>(a, fk, u, u, i, j, a.heun ? 0u : rb,
                                             a.heun ? nullptr : gb, lam_x, lam_y, v, bad);
        const int64_t o = (int64_t)j * a.pitch + i;
        double* out = a.heun ? a.us : u2;
#pragma unroll
        for (int q = 0; q < 4; ++q) __stcg(out + q * a.fstride + o, v[q]);
        if (a.heun) {
          const double eint = internal_energy(v[0], v[1], v[2], v[3]);
          if (!(v[0] > 0.0) || !(eint > 0.0)) bad = true;
        } else {
          finish(v);
        }
      }
    } else if (!GRID && lead && pend >= 0) {
      // the previous step's outflow sums, off the critical path
      outflow_sums<DIM2>(a, sbnd + pend_par * a.ob, pend_dt);
      pend = -1;
    }
    if (a.heun) {
      // (releases U* and the stage-1 faces)
      sync_all();
      // stage 2: U* -> U^{n+1} from U^n with 0.5 (F^n + F*)
      if (MAT && cellw) {
        for (int t = gtid; t < ncell; t += gthreads) {
          const int i = t % a.nx, j = t / a.nx;
          double v[4], pv[KA];
          cell_stage_mat<DIM2, MUSCL, true, KA>(a, a.us, a.ps, u, pk, i, j, rb, gb, lam_x, lam_y, v,
                                            pv, bad);
          const int64_t o = (int64_t)j * a.pitch + i;
#pragma unroll
          for (int q = 0; q < 4; ++q) __stcg(u2 + q * a.fstride + o, v[q]);
#pragma unroll
          for (int q = 0; q < KA; ++q)
            if (q < a.nmat) __stcg(pk2 + q * a.fstride + o, pv[q]);
          finish_mat(v, pv);
        }
      } else if (cellw) {
        for (int t = gtid; t < ncell; t += gthreads) {
          const int i = t % a.nx, j = t / a.nx;
          double v[4];
          cell_stage<DIM2, MUSCL, FAST, true>(a, fk, a.us, u, i, j, rb, gb, lam_x, lam_y, v, bad);
          const int64_t o = (int64_t)j * a.pitch + i;
#pragma unroll
          for (int q = 0; q < 4; ++q) __stcg(u2 + q * a.fstride + o, v[q]);
          finish(v);
        }
      }
    }
    // block partials (warp shuffles, then the block's own shared atomics), broadcast by
    // plain shared::cluster stores into every block's slot for this block: after one
    // barrier every block reduces them itself (no second barrier for a control record)
    rk = wred(rk, mx);
    mr = wred(mr, mn);
    me = wred(me, mn);
    if (MAT) mpk = wred(mpk, mn);
    const bool wbad = __any_sync(0xffffffffu, bad), wdt = __any_sync(0xffffffffu, dtbad);
    if ((tid & 31) == 0) {
      if (rk) atomicMax(&sh.rate, rk);
      if (mr != 0x7ff0000000000000ull) atomicMin(&sh.min_r, mr);
      if (me != 0x7ff0000000000000ull) atomicMin(&sh.min_e, me);
      if (MAT && mpk != ~0ull) atomicMin(&sh.min_pk, mpk);
      if (wbad) sh.fail = 1;
      if (wdt) sh.dtfail = 1;
    }
    __syncthreads();
    unsigned long long* const gp = GRID ? a.gpart + par * SMALL_NPART * SMALL_MAX_GRID : nullptr;
    if constexpr (GRID) {
      if (tid == 0) {
        __stcg(gp + rank, sh.rate);
        __stcg(gp + SMALL_MAX_GRID + rank, sh.min_r);
        __stcg(gp + 2 * SMALL_MAX_GRID + rank, sh.min_e);
        __stcg(gp + 3 * SMALL_MAX_GRID + rank, (unsigned long long)sh.fail);
        __stcg(gp + 4 * SMALL_MAX_GRID + rank, (unsigned long long)sh.dtfail);
        __stcg(gp + 5 * SMALL_MAX_GRID + rank, sh.min_pk);
      }
    } else if (tid < nblk) {   // one thread per destination block
      st_remote(remote(&sh.p_rate[par][rank], tid), sh.rate);
      st_remote(remote(&sh.p_min_r[par][rank], tid), sh.min_r);
      st_remote(remote(&sh.p_min_e[par][rank], tid), sh.min_e);
      st_remote(remote(&sh.p_fail[par][rank], tid), sh.fail);
      st_remote(remote(&sh.p_dtfail[par][rank], tid), sh.dtfail);
      st_remote(remote(&sh.p_min_pk[par][rank], tid), sh.min_pk);
    }
    // (releases U^{n+1}, the boundary faces and the partials)
    sync_all();
    if constexpr (GRID) {
      // every block combines all blocks' partials (one slot per thread, then warps)
      unsigned long long vr = 0ull, vm = 0x7ff0000000000000ull, ve = 0x7ff0000000000000ull;
      unsigned long long vp = ~0ull;
      int vf = 0, vd = 0;
      for (uint32_t b = tid; b < nblk; b += blockDim.x) {
        const unsigned long long r_ = __ldcg(gp + b), m_ = __ldcg(gp + SMALL_MAX_GRID + b);
        const unsigned long long e_ = __ldcg(gp + 2 * SMALL_MAX_GRID + b);
        vr = r_ > vr ? r_ : vr;
        vm = m_ < vm ? m_ : vm;
        ve = e_ < ve ? e_ : ve;
        vf |= (int)__ldcg(gp + 3 * SMALL_MAX_GRID + b);
        vd |= (int)__ldcg(gp + 4 * SMALL_MAX_GRID + b);
        const unsigned long long p_ = __ldcg(gp + 5 * SMALL_MAX_GRID + b);
        vp = p_ < vp ? p_ : vp;
      }
      vp = wred(vp, mn);
      vr = wred(vr, mx);
      vm = wred(vm, mn);
      ve = wred(ve, mn);
      vf = __any_sync(0xffffffffu, vf);
      vd = __any_sync(0xffffffffu, vd);
      if ((tid & 31) == 0) {
        if (vr) atomicMax(&sh.g_rate, vr);
        if (vm != 0x7ff0000000000000ull) atomicMin(&sh.g_min_r, vm);
        if (ve != 0x7ff0000000000000ull) atomicMin(&sh.g_min_e, ve);
        if (vp != ~0ull) atomicMin(&sh.g_min_pk, vp);
        if (vf) sh.g_fail = 1;
        if (vd) sh.g_dtfail = 1;
      }
      __syncthreads();
    }
    if (tid == 0) {
      unsigned long long rt = 0ull, m_r = 0x7ff0000000000000ull, m_e = 0x7ff0000000000000ull;
      unsigned long long m_p = ~0ull;
      int fail = 0, dtf = 0;
      if constexpr (GRID) {
        rt = sh.g_rate;
        m_r = sh.g_min_r;
        m_e = sh.g_min_e;
        m_p = sh.g_min_pk;
        fail = sh.g_fail;
        dtf = sh.g_dtfail;
      } else {
        for (uint32_t b = 0; b < nblk; ++b) {
          rt = sh.p_rate[par][b] > rt ? sh.p_rate[par][b] : rt;
          m_r = sh.p_min_r[par][b] < m_r ? sh.p_min_r[par][b] : m_r;
          m_e = sh.p_min_e[par][b] < m_e ? sh.p_min_e[par][b] : m_e;
          m_p = sh.p_min_pk[par][b] < m_p ? sh.p_min_pk[par][b] : m_p;
          fail |= sh.p_fail[par][b];
          dtf |= sh.p_dtfail[par][b];
        }
      }
      sh.stop = fail;
      if (!fail) {
        StepRec r;
        r.dt = dt;
        r.hits = c.time + dt >= a.limit;
        r.time = r.hits ? a.limit : c.time + dt;
        r.min_rho = __longlong_as_double((long long)m_r);
        r.min_eint = __longlong_as_double((long long)m_e);
        // (MAT) min p decoded from its order key; +inf (min_p's initial value) if none
        r.min_p_mat = m_p == ~0ull ? __longlong_as_double(0x7ff0000000000000ll)
                      : __longlong_as_double(
                            (long long)((m_p >> 63) ? (m_p & 0x7fffffffffffffffull) : ~m_p));
        r.status = 0;
        if (lead) a.rec[n] = r;
        StepCtl nx_;
        nx_.time = r.time;
        nx_.rate_bits = rt;
        nx_.dtfail = dtf;
        nx_.done = !(r.time < a.t_final);
        sh.ctl = nx_;
      }
    }
    __syncthreads();
    if (sh.stop) break;   // the host re-runs this step stage-wise
    pend = n;
    pend_par = par;
    pend_dt = dt;
    double* t = u;
    u = u2;
    u2 = t;
    t = pk;
    pk = pk2;
    pk2 = t;
  }
  if (!GRID && lead && !cellw && pend >= 0) outflow_sums<DIM2>(a, sbnd + pend_par * a.ob, pend_dt);
  // the step that stopped the batch: 1 failed (the host re-runs it stage-wise),
  // 2 skipped (limit reached); later steps skipped
  if (lead && tid == 0) {
    for (int k = n; k < a.nsteps; ++k) {
      StepRec r{};
      r.status = (k == n && !sh.ctl.done) ? 1 : 2;
      r.time = sh.ctl.time;
      a.rec[k] = r;
    }
    *a.ctl = sh.ctl;
  }
  if constexpr (!GRID)
    cg::this_cluster().sync();   // no block leaves while another may still address its shared memory
}

// Grid mode's outflow (solver.cpp:406-432), after the kernel: k_small_sums forms each
// completed step's ordered sums (one thread per step and chain: lanes of chains 0-3 sum
// right - left over the rows in order, 4-7 top - bottom over the columns), k_small_accum
// adds them to the outflow step by step in order (acc += dt dy s_x, += dt dx s_y).
__global__ void k_small_sums(const StepRec* __restrict__ rec, const double* __restrict__ bhist,
                             int nsteps, int ob, int nx, int ny, int dim2, double* sums) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = t >> 3, ch = t & 7;
  if (n >= nsteps || rec[n].status != 0) return;
  const double* sb = bhist + (int64_t)n * ob;
  const int q = ch & 3;
  double s = 0.0;
  if (ch < 4) {
    const double* L = sb + q * ny;
    const double* R = L + 4 * ny;
#pragma unroll 8
    for (int j = 0; j < ny; ++j) s += R[j] - L[j];
  } else if (dim2) {
    const double* B = sb + 8 * ny + q * nx;
    const double* T = B + 4 * nx;
#pragma unroll 8
    for (int i = 0; i < nx; ++i) s += T[i] - B[i];
  }
  sums[t] = s;
}

__global__ void k_small_accum(const StepRec* __restrict__ rec, const double* __restrict__ sums,
                              int nsteps, int dim2, double dx, double dy, double* outflow) {
  const int q = threadIdx.x;
  if (q >= 4) return;
  double acc = outflow[q];
  for (int n = 0; n < nsteps && rec[n].status == 0; ++n) {
    const double ax = rec[n].dt * (dim2 ? dy : 1.0), ay = rec[n].dt * dx;
    acc += ax * sums[8 * n + q];
    if (dim2) acc += ay * sums[8 * n + 4 + q];
  }
  outflow[q] = acc;
}

// LF_SMALL_FAST=0 in the environment: the IEEE expressions throughout (A/B)
bool small_fast_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LF_SMALL_FAST");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One cluster of up to 16 blocks (the non-portable maximum; fewer where the device
// cannot co-schedule them), each block on its own SM -- or, in grid mode, a cooperative
// grid of up to one block per SM (every block co-resident, grid barriers).
template <bool DIM2, bool MUSCL>
cudaError_t launch_small(const SmallArgs& a, int want, bool fast, bool grid, bool mat,
                         cudaStream_t st) {
  // (the material kernels: the IEEE arithmetic only)
  // (array bounds of 4 or 8 materials: registers for the common 2-4)
  auto pick = [&](bool g) {
    if (mat && a.nmat <= 4)
      return g ? k_small_run<DIM2, MUSCL, false, true, 4>
               : k_small_run<DIM2, MUSCL, false, false, 4>;
    if (mat)
      return g ? k_small_run<DIM2, MUSCL, false, true, 8>
               : k_small_run<DIM2, MUSCL, false, false, 8>;
    if (fast)
      return g ? k_small_run<DIM2, MUSCL, true, true, 0>
               : k_small_run<DIM2, MUSCL, true, false, 0>;
    return g ? k_small_run<DIM2, MUSCL, false, true, 0>
             : k_small_run<DIM2, MUSCL, false, false, 0>;
  };
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(SMALL_THREADS + 32);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (grid) {
    auto kern = pick(true);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, SMALL_THREADS + 32, 0);
    if (e != cudaSuccess) return e;
    const int nb = std::max(1, std::min({want, sms * std::max(per, 1), SMALL_MAX_GRID}));
    cfg.gridDim = dim3(nb);
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  }
  auto kern = pick(false);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  const size_t smem = 2 * (size_t)a.ob * sizeof(double);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  int ncta = std::max(1, std::min(want, SMALL_MAX_CTAS));
  cfg.gridDim = dim3(ncta);
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  int maxc = 0;
  if (cudaOccupancyMaxPotentialClusterSize(&maxc, kern, &cfg) == cudaSuccess && maxc >= 1 &&
      ncta > maxc) {
    ncta = maxc;
    cfg.gridDim = dim3(ncta);
    at[0].val.clusterDim.x = ncta;
  }
  // (a device shared with other work may not co-schedule the whole cluster at launch
  // time: halve it until it fits -- the kernel strides its cells over any block count)
  for (;;) {
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if ((e != cudaErrorInvalidClusterSize && e != cudaErrorLaunchOutOfResources) || ncta == 1)
      return e;
    (void)cudaGetLastError();
    ncta = (ncta + 1) / 2;
    cfg.gridDim = dim3(ncta);
    at[0].val.clusterDim.x = ncta;
  }
}

// grid mode beyond one cluster's worth of cells, and whenever the boundary faces of two
// steps do not fit in the lead block's shared memory (LF_SMALL_GRID=0 / 1 in the
// environment: never / always where possible, for A/B)
bool use_grid_mode(const lf_handle* h) {
  static const int force = [] {
    const char* e = std::getenv("LF_SMALL_GRID");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  if (h->dim2 && h->d.nx + h->d.ny > SMALL_MAX_PERIMETER) return true;
  if (force >= 0) return force == 1;
  return (int64_t)h->d.nx * h->d.ny > (int64_t)SMALL_MAX_CTAS * SMALL_THREADS;
}

}  // namespace

// ================================================================= host driver

struct SmallState {
  StepCtl* ctl = nullptr;        // device [1]
  StepCtl* ctl_host = nullptr;   // pinned [1]
  StepRec* rec = nullptr;        // device [cap]
  StepRec* rec_host = nullptr;   // pinned [cap]
  double* outflow = nullptr;     // device [4]
  double* outflow_host = nullptr;
  int cap = 0;
  bool valid = false;            // ctl holds the rate of the current U
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // grid mode: block partials, the boundary-face history and per-step sums of a batch
  unsigned long long* gpart = nullptr;   // device [2][5][SMALL_MAX_GRID]
  double* bhist = nullptr;               // device [SMALL_GRID_BATCH][ob]
  double* sums = nullptr;                // device [SMALL_GRID_BATCH][8]
};

namespace {

struct SmallFail : std::runtime_error {
  explicit SmallFail(const std::string& w) : std::runtime_error(w) {}
};
#define SK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) throw SmallFail(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

SmallState* sstate(lf_handle* h) { return reinterpret_cast<SmallState*>(h->small); }

void small_alloc(lf_handle* h, int steps) {
  SlabState& s = h->slabs[0];
  SK(cudaSetDevice(s.device));
  alloc_staged_public(h);
  SmallState* m = sstate(h);
  if (!m) {
    m = new SmallState;
    h->small = m;
    SK(cudaMalloc(&m->ctl, sizeof(StepCtl)));
    SK(cudaHostAlloc(&m->ctl_host, sizeof(StepCtl), cudaHostAllocDefault));
    SK(cudaMalloc(&m->outflow, 4 * sizeof(double)));
    SK(cudaHostAlloc(&m->outflow_host, 4 * sizeof(double), cudaHostAllocDefault));
    SK(cudaEventCreate(&m->e0));
    SK(cudaEventCreate(&m->e1));
  }
  if (!m->gpart && use_grid_mode(h)) {
    const int64_t ob = 8 * (int64_t)s.L.ny + (h->dim2 ? 8 * (int64_t)s.L.nx : 0);
    SK(cudaMalloc(&m->gpart, 2 * SMALL_NPART * SMALL_MAX_GRID * sizeof(unsigned long long)));
    SK(cudaMalloc(&m->bhist, (size_t)SMALL_GRID_BATCH * ob * sizeof(double)));
    SK(cudaMalloc(&m->sums, (size_t)SMALL_GRID_BATCH * 8 * sizeof(double)));
  }
  if (steps > m->cap) {
    cudaFree(m->rec);
    cudaFreeHost(m->rec_host);
    m->cap = std::max(steps, 256);
    SK(cudaMalloc(&m->rec, (size_t)m->cap * sizeof(StepRec)));
    SK(cudaHostAlloc(&m->rec_host, (size_t)m->cap * sizeof(StepRec), cudaHostAllocDefault));
  }
}

// Run up to n steps from `time` in one launch; returns the completed count and
// the index of a failed step (-1 if none).  U holds the state after them.
int run_small(lf_handle* h, int n, double cfl, double limit, double t_final, double time,
              double* outflow, int* failed_at, float* ms) {
  LF_TRACE("small-grid step batch");
  SmallState* m = sstate(h);
  SlabState& s = h->slabs[0];
  if (!m->valid) {
    const Scalars sc = rate_of_current(h);
    m->ctl_host->rate_bits = sc.rate_bits;
    m->ctl_host->dtfail = sc.fail_dt != LLONG_MAX || sc.fail_frac != LLONG_MAX;
    m->valid = true;
  } else {
    SK(cudaMemcpyAsync(m->ctl_host, m->ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost, s.stream));
    SK(cudaStreamSynchronize(s.stream));
  }
  m->ctl_host->time = time;
  m->ctl_host->done = 0;
  SK(cudaMemcpyAsync(m->ctl, m->ctl_host, sizeof(StepCtl), cudaMemcpyHostToDevice, s.stream));
  double o[4] = {0, 0, 0, 0};
  if (outflow) std::memcpy(o, outflow, sizeof o);
  std::memcpy(m->outflow_host, o, sizeof o);
  SK(cudaMemcpyAsync(m->outflow, m->outflow_host, sizeof o, cudaMemcpyHostToDevice, s.stream));
  SmallArgs a;
  a.u = s.U + s.L.origin();
  a.u2 = s.U2 + s.L.origin();
  a.us = s.Us + s.L.origin();
  a.pitch = s.L.pitch;
  a.fstride = s.L.fstride;
  for (int k = 0; k < 2; ++k) {
    a.fx[k] = s.FX[k];
    a.fy[k] = s.FY[k];
  }
  a.fx_stride = s.fx_stride;
  a.fy_stride = s.fy_stride;
  a.nx = s.L.nx;
  a.ny = s.L.ny;
  a.ob = 8 * a.ny + (h->dim2 ? 8 * a.nx : 0);
  a.heun = h->d.time_order >= 2;
  for (int q = 0; q < 4; ++q) a.bc[q] = h->d.bc[q];
  a.k = h->k;
  a.cfl = cfl;
  a.limit = limit;
  a.t_final = t_final;
  a.ctl = m->ctl;
  a.rec = m->rec;
  a.outflow = m->outflow;
  a.nsteps = n;
  const bool grid = use_grid_mode(h);
  a.gpart = m->gpart;
  a.bhist = m->bhist;
  const bool mat = h->mc.n > 0;
  a.nmat = h->mc.n;
  for (int k = 0; k < 8; ++k) a.gam[k] = k < h->mc.n ? h->mc.gamma[k] : 1.5;
  a.p = mat ? s.P + s.L.origin() : nullptr;
  a.p2 = mat ? s.P2 + s.L.origin() : nullptr;
  a.ps = mat ? s.Ps + s.L.origin() : nullptr;
  a.y0 = mat ? s.Y[0] + s.L.origin() : nullptr;
  a.usx0 = mat ? s.USX[0] : nullptr;
  a.usy0 = mat ? s.USY[0] : nullptr;
  const bool muscl = h->d.spatial_order >= 2;
  if (ms) SK(cudaEventRecord(m->e0, s.stream));
  count_launch();
  const int64_t cells = (int64_t)a.nx * a.ny;
  const int want = (int)std::min<int64_t>((cells + SMALL_THREADS - 1) / SMALL_THREADS, SMALL_MAX_GRID);
  cudaError_t le;
  // the fast exact arithmetic where its proofs hold (beta >= 1 for sweby_fast, gamma - 1
  // in the constant box); a cell outside the cell box flags the step (stage-wise re-run)
  const bool fast = !mat && small_fast_enabled() && !h->small_ieee && h->d.beta >= 1.0 && h->k.gm1 >= 0x1p-14 &&
                    h->k.gm1 < 0x1p6 && h->k.gamma < 0x1p7;
  if (h->dim2)
    le = muscl ? launch_small<true, true>(a, want, fast, grid, mat, s.stream)
               : launch_small<true, false>(a, want, fast, grid, mat, s.stream);
  else
    le = muscl ? launch_small<false, true>(a, want, fast, grid, mat, s.stream)
               : launch_small<false, false>(a, want, fast, grid, mat, s.stream);
  SK(le);
  if (grid) {   // the batch's boundary-outflow sums, in step order
    count_launch(2);
    k_small_sums<<<(8 * n + 255) / 256, 256, 0, s.stream>>>(m->rec, m->bhist, n, a.ob, a.nx,
                                                           a.ny, h->dim2, m->sums);
    k_small_accum<<<1, 32, 0, s.stream>>>(m->rec, m->sums, n, h->dim2, h->d.dx, h->d.dy,
                                          m->outflow);
    SK(cudaGetLastError());
  }
  SK(cudaGetLastError());
  if (ms) SK(cudaEventRecord(m->e1, s.stream));
  SK(cudaMemcpyAsync(m->rec_host, m->rec, (size_t)n * sizeof(StepRec), cudaMemcpyDeviceToHost,
                     s.stream));
  SK(cudaMemcpyAsync(m->outflow_host, m->outflow, 4 * sizeof(double), cudaMemcpyDeviceToHost,
                     s.stream));
  SK(cudaStreamSynchronize(s.stream));
  if (ms) SK(cudaEventElapsedTime(ms, m->e0, m->e1));
  int done = 0;
  *failed_at = -1;
  for (int i = 0; i < n; ++i) {
    if (m->rec_host[i].status == 0) {
      ++done;
      continue;
    }
    if (m->rec_host[i].status == 1) *failed_at = i;
    break;
  }
  if (done & 1) {   // the kernel ping-pongs U and U2 (and the partials) once per step
    std::swap(s.U, s.U2);
    if (mat) std::swap(s.P, s.P2);
  }
  fused_invalidate(h);   // (also clears m->valid)
  m->valid = *failed_at < 0;
  h->rate_valid = false;
  if (outflow) std::memcpy(outflow, m->outflow_host, 4 * sizeof(double));
  return done;
}

void to_out(const StepRec& r, int64_t step, double gm1, lf_step_out* o, bool mat) {
  o->dt = r.dt;
  o->hits_limit = r.hits;
  o->time = r.time;
  o->step = step;
  o->min_rho = r.min_rho;
  o->min_p = mat ? r.min_p_mat : gm1 * r.min_eint;
}

}  // namespace

// LF_PATH_SMALL: up to 8 materials (partials resident), one slab on one device (no
// NCCL), up to SMALL_MAX_CELLS cells (AUTO: the crossovers in small.h, measured by
// tools/small_sweep.py and tools/small_mat_sweep.py).
bool small_supported(lf_handle* h) {
  if (h->mc.n > SMALL_MAX_MAT || (h->mc.n > 0 && !h->partials_ready) || h->slabs.size() != 1 ||
      h->nccl)
    return false;
  // (the kernel reads ghosts through an index map whose sources are interior cells)
  if (h->d.nx < 2 || (h->dim2 && h->d.ny < 2)) return false;
  return (int64_t)h->d.nx * h->d.ny <= SMALL_MAX_CELLS;
}

bool prefer_small(lf_handle* h) {
  const int64_t lim = !h->dim2        ? SMALL_AUTO_CELLS_1D
                      : h->mc.n > 0 ? SMALL_AUTO_CELLS_2D_MAT
                                    : SMALL_AUTO_CELLS_2D;
  if (!(h->path == LF_PATH_AUTO && small_supported(h) && (int64_t)h->d.nx * h->d.ny <= lim))
    return false;
  // the top of the 2D range (5 * 2^14 .. 2^17 cells) goes to the one-kernel step where
  // that applies (fused.h FUSED_AUTO_MIN_CELLS); narrow grids stay here
  return !(prefer_fused(h) && fused_supported(h));
}

void small_invalidate(lf_handle* h) {
  if (SmallState* m = sstate(h)) m->valid = false;
}

void small_release(lf_handle* h) {
  SmallState* m = sstate(h);
  if (!m) return;
  cudaFree(m->ctl);
  cudaFreeHost(m->ctl_host);
  cudaFree(m->rec);
  cudaFreeHost(m->rec_host);
  cudaFree(m->outflow);
  cudaFreeHost(m->outflow_host);
  if (m->e0) cudaEventDestroy(m->e0);
  if (m->e1) cudaEventDestroy(m->e1);
  cudaFree(m->gpart);
  cudaFree(m->bhist);
  cudaFree(m->sums);
  delete m;
  h->small = nullptr;
}

int small_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
               double* outflow, lf_step_out* out) {
  small_alloc(h, 1);
  int failed_at;
  double acc[4] = {0, 0, 0, 0};
  if (outflow) std::memcpy(acc, outflow, sizeof acc);
  if (run_small(h, 1, cfl, limit, limit, time, acc, &failed_at, nullptr) == 1) {
    if (outflow) std::memcpy(outflow, acc, sizeof acc);
    if (out) to_out(sstate(h)->rec_host[0], step + 1, h->d.gamma - 1.0, out, h->mc.n > 0);
    return 0;
  }
  // a check failed: the stage-wise kernels reproduce the reference's error
  small_invalidate(h);
  fused_invalidate(h);
  const int rc = staged_heun_public(h, cfl, time, limit, step, outflow, out);
  if (rc == 0) h->small_ieee = 1;   // the fast arithmetic's box failed, not the step
  return rc;
}

int small_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
                  int64_t* step, double* outflow, lf_step_out* per_step, int* taken) {
  if (taken) *taken = 0;
  int k = 0;
  while (k < nsteps && *time < t_final) {
    const int batch = std::min(nsteps - k, use_grid_mode(h) ? SMALL_GRID_BATCH : SMALL_BATCH);
    small_alloc(h, batch);
    SmallState* m = sstate(h);
    int failed_at;
    const int done = run_small(h, batch, cfl, t_final, t_final, *time, outflow, &failed_at, nullptr);
    for (int i = 0; i < done; ++i) {
      *step += 1;
      if (per_step) to_out(m->rec_host[i], *step, h->d.gamma - 1.0, &per_step[k + i], h->mc.n > 0);
      *time = m->rec_host[i].time;
    }
    k += done;
    if (taken) *taken = k;
    if (failed_at >= 0) {
      small_invalidate(h);
      fused_invalidate(h);
      lf_step_out o;
      const int rc = staged_heun_public(h, cfl, *time, t_final, *step, outflow, &o);
      if (rc) return rc;
      h->small_ieee = 1;   // the fast arithmetic's box failed, not the step
      *step = o.step;
      *time = o.time;
      if (per_step) per_step[k] = o;
      ++k;
      if (taken) *taken = k;
      continue;
    }
    if (done < batch) break;  // reached t_final
  }
  return 0;
}

int small_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                     int* launches) {
  const int per = use_grid_mode(h) ? SMALL_GRID_BATCH : SMALL_BATCH;
  small_alloc(h, std::min(nsteps, per));
  SmallState* m = sstate(h);
  double t0 = 0.0;
  if (m->valid) {
    SK(cudaMemcpy(m->ctl_host, m->ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost));
    t0 = m->ctl_host->time;
  }
  const double big = 1.7976931348623157e308;
  double total = 0.0;
  int k = 0, nl = 0;
  while (k < nsteps) {
    int failed_at;
    float ms = 0.f;
    const int n = std::min(nsteps - k, per);
    const int done = run_small(h, n, cfl, big, big, t0, nullptr, &failed_at, &ms);
    total += ms;
    ++nl;
    if (failed_at >= 0) return LF_ERR_DEVICE;
    t0 = m->rec_host[done - 1].time;
    k += done;
  }
  *kernel_ms = total;
  *step_ms = total;
  *launches = nl;
  return 0;
}

}  // namespace lfb
