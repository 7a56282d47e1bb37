// fused_step.cu -- host driver of the device-resident Heun step: the two-pass
// kernels (twopass_kernel.cu / twopass_mat_kernel.cu, the default) or the
// one-kernel step (fused_kernel.cu).
//
// Per step, on the slab stream: ghost fill of U^n (one launch, then halo rows)
// -> predictor -> fill of U* -> corrector (or k_fused_step) -> [NCCL max of the
// step accumulators and sum of the boundary faces across ranks] -> k_finalize
// (dt, time, diagnostics, next step's control record); the chain is launched
// with programmatic dependent launch (pdl.cuh).  The ordered boundary-outflow
// sums (k_outflow) run on a low-priority side stream.  dt and time stay on the
// device, so lf_advance enqueues whole batches of steps without a host round
// trip; records come back once per batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "fused.h"
#include "fused_common.cuh"
#include "twopass.h"
#include "nccl_comm.h"
#include "small.h"
#include "trace.h"

namespace lfb {

namespace {

struct DevFail : std::runtime_error {
  explicit DevFail(const std::string& w) : std::runtime_error(w) {}
};

#define FK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) throw DevFail(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

// Fused-path state of a handle (one per handle; all slabs on one device).
struct FusedState {
  StepCtl* ctl = nullptr;          // device [2]
  StepAcc* acc = nullptr;          // device [2]
  StepRec* rec = nullptr;          // device [cap]
  StepRec* rec_host = nullptr;     // pinned [cap]
  int cap = 0;
  double* bnd = nullptr;           // device [2][8 nyg + 8 nx]
  double* outflow = nullptr;       // device [4]
  double* outflow_host = nullptr;  // pinned [4]
  StepCtl* ctl_host = nullptr;     // pinned [2]
  int cur = 0;                     // ctl slot of the current state
  bool valid = false;              // ctl[cur].rate_bits is the rate of the current U
  int rows_per_chunk = 0;          // fused kernel
  int tp_rows = 0;                 // two-pass kernels
  int tp_rows_nmat = -1;           // the material count tp_rows was sized for
  int sms = 148;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // boundary-outflow sums run on a low-priority side stream: ev_fin[b] = the
  // finalize of a step using bnd slot b, ev_out[b] = its sums (slot b is
  // rewritten two steps later, after ev_out[b])
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fin[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  // distributed fused step: halo exchange and the slab's edge row chunks on `comm`,
  // overlapped with the interior chunks on the slab stream
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_fill = nullptr, ev_edge = nullptr;
  FKBits fk_exact{}, fk_contract{};   // launch-parameter constants of the fused kernels
  bool fk_ok = false;                 // (computed on the first fused step)
  // CUDA graphs of whole step batches (lf_advance, single-slab handles without NCCL):
  // a batch's launches are captured once per key and replayed; the key holds every
  // value the captured launches bake in (batch length, the control-record slot, every
  // state and scratch buffer as the batch starts -- euler_stage swaps U with U*, so
  // U alone does not identify them --, the step parameters, the path).  Capturing and
  // instantiating costs ~8 us per kernel node against ~1 us saved per replayed node
  // (tools/graph_sweep.py; quadrant 1024^2, 200 steps from cold: 31.9 ms with every
  // batch captured at first sight, 25.6 ms launch by launch), so a batch runs launch by
  // launch the first time its key is seen and is captured when the key comes back --
  // only runs long enough to repeat a batch pay for graphs, and only they build them
  using GraphKey = std::tuple<int, int, const double*, const double*, const double*,
                              const double*, const double*, const double*, double, double,
                              double, int, int, int>;
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int launches = 0;   // kernels per replay (lf_launch_count)
  };
  std::map<GraphKey, Graph> graphs;
  std::set<GraphKey> seen;   // keys that ran launch by launch once
  bool capturing = false;
};

// LF_GRAPHS in the environment: 0 = enqueue every batch launch by launch (A/B),
// 2 = capture a batch the first time its key is seen, 1 / unset = the second time
static int graphs_mode() {
  static const int mode = [] {
    const char* e = std::getenv("LF_GRAPHS");
    return e && e[0] == '0' ? 0 : (e && e[0] == '2' ? 2 : 1);
  }();
  return mode;
}

static void drop_graphs(FusedState* f) {
  for (auto& kv : f->graphs) cudaGraphExecDestroy(kv.second.exec);
  f->graphs.clear();
  f->seen.clear();
}

static FusedState* fstate(lf_handle* h) { return reinterpret_cast<FusedState*>(h->fused); }

static size_t bnd_words(lf_handle* h) { return 8 * (size_t)h->d.ny + 8 * (size_t)h->d.nx; }

static bool use_twopass(lf_handle* h);

bool fused_supported(lf_handle* h) {
  if (!h->dim2) return false;
  // time_order 1 runs on the two-pass kernels only (the fused step is Heun)
  if (h->d.time_order < 2 && !use_twopass(h)) return false;
  if (h->d.nx < 4) return false;
  for (auto& s : h->slabs) {
    if (s.L.ny < 4) return false;
    if (s.device != h->slabs[0].device) return false;  // shared step records need one device
  }
  return true;
}

// LF_PATH_AUTO, one material, Heun: the one-kernel step on every 2D slab past the
// small-grid path's range.  From 2^23 cells per slab (2^22 in the contract arithmetic)
// it is clearly the faster one (tools/path_sweep.py, round 2: Sedov 4096^2 11.7 vs 10.9
// G cell-updates/s, smooth 8192^2 13.7 vs 12.1, 16384^2 14.7 vs ~12): it moves 64 B per
// cell-update instead of 290 and stays at the full clock where the two-pass step meets
// the board's power cap.  Below that, with row chunks as short as the cost model in
// fused_alloc likes (a 1024^2 step is one wave of 288 blocks of 32 rows), it is ahead
// of or level with the two-pass kernels down to 320^2 (tools/chunk_sweep.py,
// profiles/r02_chunk_sweep.json: 512^2 4.3 vs 3.0 G/s, 768^2 6.2 vs 5.5, quadrant
// 1024^2 8.1 vs 7.8, smooth 1024^2 7.9 vs 8.3, 2048^2 10.5 vs 10.6; in the contract
// arithmetic ahead everywhere), and it needs no U* / F^n scratch.  Narrow grids, whose
// last 120-column strip would be mostly empty, stay on the two-pass kernels' 28-column
// warp strips.
bool prefer_fused(lf_handle* h) {
  if (h->path != LF_PATH_AUTO || !h->dim2 || h->d.time_order < 2 || h->mc.n > 0) return false;
  if (!(h->d.beta >= 1.0)) return false;   // (stage-wise: api.cu use_fused)
  const int64_t big = (int64_t)1 << (h->math == LF_MATH_CONTRACT ? 22 : 23);
  const int strips = (h->d.nx + FUSED_TXO - 1) / FUSED_TXO;
  const bool wide = 5 * (int64_t)h->d.nx >= 4 * (int64_t)strips * FUSED_TXO;   // >= 80 % full
  for (auto& s : h->slabs) {
    const int64_t cells = (int64_t)s.L.nx * s.L.ny;
    if (cells >= big) continue;
    if (!(wide && cells > FUSED_AUTO_MIN_CELLS)) return false;
  }
  return true;
}

static bool use_twopass(lf_handle* h) {
  if (h->path == LF_PATH_FUSED) return false;
  for (auto& s : h->slabs)
    if (!tp_fits(s.L.pitch, s.L.ny)) return false;
  if (prefer_fused(h)) return false;
  if (h->path == LF_PATH_AUTO && h->tp_mem_ok < 0) {
    // the two passes need U*, W and two F face sets beside U^n / U^{n+1}: six more
    // state-sized arrays (32768^2: 206 GB in all).  Decided once, before they are
    // allocated; a slab that does not fit runs the one-kernel step (two states).
    h->tp_mem_ok = 1;
    for (auto& s : h->slabs) {
      double need = 0.0;   // all slabs of this device (in-process slabs share one)
      for (auto& o : h->slabs)
        if (o.device == s.device && !o.Us)
          need += 8.0 * ((double)o.L.alloc * 2 +
                         2.0 * 4 * ((double)o.L.pitch * o.L.ny * 2 + o.L.pitch));
      size_t free_b = 0, total_b = 0;
      FK(cudaSetDevice(s.device));
      FK(cudaMemGetInfo(&free_b, &total_b));
      // (scratch already allocated, e.g. by the material path: nothing to veto)
      if (need > 0.0 && need + (double)(1ull << 30) > (double)free_b) h->tp_mem_ok = 0;
    }
  }
  return h->path != LF_PATH_AUTO || h->tp_mem_ok != 0;
}

bool twopass_selected(lf_handle* h) { return use_twopass(h); }

static void fused_alloc(lf_handle* h, int steps) {
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  FK(cudaSetDevice(s0.device));
  if (use_twopass(h)) alloc_staged_public(h);  // U*, F^n faces of the two passes
  if (!f) {
    f = new FusedState;
    h->fused = f;
    FK(cudaMalloc(&f->ctl, 2 * sizeof(StepCtl)));
    FK(cudaMalloc(&f->acc, 2 * sizeof(StepAcc)));
    FK(cudaHostAlloc(&f->ctl_host, 2 * sizeof(StepCtl), cudaHostAllocDefault));
    FK(cudaMalloc(&f->bnd, 2 * bnd_words(h) * sizeof(double)));
    FK(cudaMemsetAsync(f->bnd, 0, 2 * bnd_words(h) * sizeof(double), s0.stream));
    FK(cudaMalloc(&f->outflow, 4 * sizeof(double)));
    FK(cudaHostAlloc(&f->outflow_host, 4 * sizeof(double), cudaHostAllocDefault));
    FK(cudaEventCreate(&f->e0));
    FK(cudaEventCreate(&f->e1));
    int lo = 0, hi = 0;
    FK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FK(cudaStreamCreateWithPriority(&f->side, cudaStreamNonBlocking, lo));
    for (int b = 0; b < 2; ++b) {
      FK(cudaEventCreateWithFlags(&f->ev_fin[b], cudaEventDisableTiming));
      FK(cudaEventCreateWithFlags(&f->ev_out[b], cudaEventDisableTiming));
    }
    if (h->nccl) {
      FK(cudaStreamCreateWithPriority(&f->comm, cudaStreamNonBlocking, hi));
      FK(cudaEventCreateWithFlags(&f->ev_fill, cudaEventDisableTiming));
      FK(cudaEventCreateWithFlags(&f->ev_edge, cudaEventDisableTiming));
    }
    launch_acc_init(f->acc, s0.stream);
    fused_configure();
    fused_configure_contract();
    // chunk rows: the blocks are independent and equally long, so a step costs about
    // (waves) x (rows + 9 rows of pipeline fill); pick the chunk count that minimises
    // it (16384^2: 15 chunks = 6.94 waves instead of 13 = 6.02, i.e. 7 waves either way;
    // 32768^2: 14 chunks = 12.96 waves instead of 7 = 6.48)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s0.device);
    const int strips = (h->d.nx + FUSED_TXO - 1) / FUSED_TXO;
    int ny_local = 0;
    for (auto& s : h->slabs) ny_local = std::max(ny_local, s.L.ny);
    const int64_t cap = (int64_t)sms * fused_blocks_per_sm();
    const int64_t nslab = (int64_t)h->slabs.size();   // in-process slabs share the device
    int best_rows = std::max(ny_local, 1);
    int64_t best_cost = INT64_MAX;
    int min_rows = 4;
    if (const char* e = getenv("LF_FUSED_MIN_ROWS")) min_rows = std::max(1, atoi(e));
    for (int chunks = 1; chunks <= 512; ++chunks) {
      const int rows = (ny_local + chunks - 1) / chunks;
      if (rows < min_rows && chunks > 1) break;
      const int64_t blocks = nslab * strips * ((ny_local + rows - 1) / rows);
      const int64_t cost = ((blocks + cap - 1) / cap) * (rows + 9);
      if (cost < best_cost) {
        best_cost = cost;
        best_rows = rows;
      }
    }
    f->rows_per_chunk = best_rows;
    f->sms = sms;
  }
  // two-pass chunking follows the resident warps of the kernel in use
  const int nmat = std::min(h->mc.n, TP_MAX_MATERIALS);
  if (f->tp_rows_nmat != nmat) {
    int ny_local = 0;
    for (auto& s : h->slabs) ny_local = std::max(ny_local, s.L.ny);
    f->tp_rows = tp_choose_rows(h->d.nx, ny_local, f->sms, tp_resident_warps(nmat));
    f->tp_rows_nmat = nmat;
  }
  if (steps > f->cap) {
    drop_graphs(f);   // captured finalize launches point into the old records
    cudaFree(f->rec);
    cudaFreeHost(f->rec_host);
    f->cap = std::max(steps, 64);
    FK(cudaMalloc(&f->rec, (size_t)f->cap * sizeof(StepRec)));
    FK(cudaHostAlloc(&f->rec_host, (size_t)f->cap * sizeof(StepRec), cudaHostAllocDefault));
  }
}

void fused_release(lf_handle* h) {
  FusedState* f = fstate(h);
  if (!f) return;
  cudaFree(f->ctl);
  cudaFree(f->acc);
  cudaFree(f->rec);
  cudaFreeHost(f->rec_host);
  cudaFree(f->bnd);
  cudaFree(f->outflow);
  cudaFreeHost(f->outflow_host);
  cudaFreeHost(f->ctl_host);
  if (f->e0) cudaEventDestroy(f->e0);
  if (f->e1) cudaEventDestroy(f->e1);
  if (f->side) {
    cudaStreamSynchronize(f->side);
    cudaStreamDestroy(f->side);
  }
  for (int b = 0; b < 2; ++b) {
    if (f->ev_fin[b]) cudaEventDestroy(f->ev_fin[b]);
    if (f->ev_out[b]) cudaEventDestroy(f->ev_out[b]);
  }
  if (f->comm) {
    cudaStreamSynchronize(f->comm);
    cudaStreamDestroy(f->comm);
  }
  if (f->ev_fill) cudaEventDestroy(f->ev_fill);
  if (f->ev_edge) cudaEventDestroy(f->ev_edge);
  drop_graphs(f);
  delete f;
  h->fused = nullptr;
}

int64_t fused_bytes(lf_handle* h) {
  FusedState* f = fstate(h);
  if (!f) return 0;
  return (int64_t)(2 * bnd_words(h)) * 8 + (int64_t)f->cap * (int64_t)sizeof(StepRec);
}

void fused_invalidate(lf_handle* h) {
  if (FusedState* f = fstate(h)) f->valid = false;
  small_invalidate(h);   // every path's cached control record
}

// The control record of the current state: its CFL rate (the compute_dt of
// the next step) and the caller's time.
static void seed_ctl(lf_handle* h, double time) {
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  if (!f->valid) {
    const Scalars sc = rate_of_current(h);
    StepCtl c{};
    c.time = time;
    c.rate_bits = sc.rate_bits;
    c.done = 0;
    c.dtfail = sc.fail_dt != LLONG_MAX || sc.fail_frac != LLONG_MAX;
    f->ctl_host[0] = c;
    FK(cudaMemcpyAsync(&f->ctl[f->cur], &f->ctl_host[0], sizeof(StepCtl), cudaMemcpyHostToDevice,
                       s0.stream));
    f->valid = true;
  } else {
    FK(cudaMemcpyAsync(&f->ctl_host[0], &f->ctl[f->cur], sizeof(StepCtl), cudaMemcpyDeviceToHost,
                       s0.stream));
    FK(cudaStreamSynchronize(s0.stream));
    f->ctl_host[0].time = time;
    f->ctl_host[0].done = 0;
    FK(cudaMemcpyAsync(&f->ctl[f->cur], &f->ctl_host[0], sizeof(StepCtl), cudaMemcpyHostToDevice,
                       s0.stream));
  }
}

// The fused kernels' launch-parameter constants (one-time, synchronous: never inside
// a graph capture).
static void ensure_fk(lf_handle* h) {
  FusedState* f = fstate(h);
  if (f->fk_ok) return;
  f->fk_exact = fused_make_fk(h->k.gamma, h->k.gm1, h->k.beta, h->d.dx, h->d.dy);
  f->fk_contract = fused_make_fk_contract(h->k.gamma, h->k.gm1, h->k.beta, h->d.dx, h->d.dy);
  FK(cudaGetLastError());
  f->fk_ok = true;
}

// Enqueue one fused step on every slab.
static void enqueue_step(lf_handle* h, int n_in_batch, double cfl, double limit, double t_final,
                         cudaEvent_t k0, cudaEvent_t k1) {
  LF_TRACE("enqueue heun step");
  FusedState* f = fstate(h);
  const int cur = f->cur, nxt = cur ^ 1;
  SlabState& s0 = h->slabs[0];
  // bnd slot `cur` is free once the outflow sums of two steps ago have read it (the
  // first two steps of a captured batch: waited for before the capture began)
  const bool mat = h->mc.n > 0;   // (materials run on the two-pass kernels only)
  const bool twopass = use_twopass(h);
  // the outflow sums of a periodic axis are +0.0 without reading the faces
  // (k_outflow), so their faces are neither cleared nor summed across ranks
  const bool sum_x = !(h->d.bc[0] == LF_PERIODIC && h->d.bc[1] == LF_PERIODIC);
  const bool sum_y = !(h->d.bc[2] == LF_PERIODIC && h->d.bc[3] == LF_PERIODIC);
  if ((sum_x || sum_y) && (!f->capturing || n_in_batch >= 2))
    FK(cudaStreamWaitEvent(s0.stream, f->ev_out[cur], 0));
  double* bnd = f->bnd + (size_t)cur * bnd_words(h);
  // distributed one-kernel step: the halo rows travel on the comm stream while the
  // slab's interior row chunks (which read no halo row) run on the slab stream; the
  // two edge chunks follow the exchange on the comm stream
  const bool overlap = h->nccl && !twopass && !mat && f->comm &&
                       fill_local_public(h, &SlabState::U);
  if (!overlap) {
    if (mat)
      fill_state_public(h, &SlabState::U, &SlabState::P);
    else
      fill_all_public(h, &SlabState::U);
  }
  if (h->nccl && (sum_x || sum_y))
    FK(cudaMemsetAsync(bnd, 0, bnd_words(h) * sizeof(double), s0.stream));
  if (overlap) {
    FK(cudaEventRecord(f->ev_fill, s0.stream));
    FK(cudaStreamWaitEvent(f->comm, f->ev_fill, 0));
    nccl_exchange_halos(h, &SlabState::U, 4, f->comm);
  }
  if (k0) FK(cudaEventRecord(k0, s0.stream));
  if (twopass) {
    // two passes: predictor U^n -> U*, F^n; ghosts / halos of U*; corrector.
    // time_order 1: one pass, the corrector kernels as the single forward-Euler
    // stage (input and base U^n, no Heun average; solver.cpp:510-514)
    const bool heun = h->d.time_order >= 2;
    for (int pass = heun ? 0 : 1; pass < 2; ++pass) {
      if (pass == 1 && heun) {
        if (mat)
          fill_state_public(h, &SlabState::Us, &SlabState::Ps);
        else
          fill_all_public(h, &SlabState::Us);
      }
      for (auto& s : h->slabs) {
        PassArgs a;
        a.x = (pass == 0 || !heun ? s.U : s.Us) + s.L.origin();
        a.base = s.U + s.L.origin();
        a.out = (pass == 0 ? s.Us : s.U2) + s.L.origin();
        a.fx = s.FX[0];
        a.fy = s.FY[0];
        a.fxo = s.FX[0];
        a.fyo = s.FY[0];
        a.pitch = s.L.pitch;
        a.fstride = s.L.fstride;
        a.fx_stride = s.fx_stride;
        a.fy_stride = s.fy_stride;
        a.nx = s.L.nx;
        a.ny = s.L.ny;
        a.y0g = s.sl.y0;
        a.nyg = h->d.ny;
        a.strips = tp_strips(s.L.nx);
        a.rows_per_chunk = f->tp_rows;
        a.gamma = h->k.gamma;
        a.gm1 = h->k.gm1;
        a.beta = h->k.beta;
        a.dx = h->d.dx;
        a.dy = h->d.dy;
        a.cfl = cfl;
        a.limit = limit;
        a.ctl = f->ctl + cur;
        a.acc = f->acc + cur;
        a.bnd = bnd;
        a.heun = heun ? 1 : 0;
        if (mat) {
          MatPassArgs m;
          m.px = (pass == 0 || !heun ? s.P : s.Ps) + s.L.origin();
          m.pbase = s.P + s.L.origin();
          m.pout = (pass == 0 ? s.Ps : s.P2) + s.L.origin();
          m.mfx = s.MFX;
          m.mfy = s.MFY;
          m.mfxo = s.MFX;
          m.mfyo = s.MFY;
          m.mfx_stride = s.fx_stride;
          m.mfy_stride = s.fy_stride;
          launch_pass_mat(a, m, h->mc, pass == 1, h->d.spatial_order >= 2, s.stream);
        } else {
          if (h->math == LF_MATH_CONTRACT)
            launch_pass_contract(a, pass == 1, h->d.spatial_order >= 2, s.stream);
          else
            launch_pass(a, pass == 1, h->d.spatial_order >= 2, h->tp_exact != 0, s.stream);
        }
      }
    }
  }
  for (auto& s : h->slabs) {
    if (twopass) break;
    FusedArgs a;
    a.u = s.U + s.L.origin();
    a.un = s.U2 + s.L.origin();
    a.pitch = s.L.pitch;
    a.fstride = s.L.fstride;
    a.nx = s.L.nx;
    a.ny = s.L.ny;
    a.y0g = s.sl.y0;
    a.nyg = h->d.ny;
    a.rows_per_chunk = f->rows_per_chunk;
    a.chunk0 = 0;
    a.chunk_step = 1;
    a.gamma = h->k.gamma;
    a.gm1 = h->k.gm1;
    a.beta = h->k.beta;
    a.dx = h->d.dx;
    a.dy = h->d.dy;
    a.cfl = cfl;
    a.limit = limit;
    a.bc_xlo = h->d.bc[0];
    a.bc_xhi = h->d.bc[1];
    a.bc_ylo = h->d.bc[2];
    a.bc_yhi = h->d.bc[3];
    a.bottom_edge = s.sl.fill_lo && h->d.bc[2] != LF_PERIODIC;
    a.top_edge = s.sl.fill_hi && h->d.bc[3] != LF_PERIODIC;
    a.ctl = f->ctl + cur;
    a.acc = f->acc + cur;
    a.bnd = bnd;
    const int strips = (h->d.nx + FUSED_TXO - 1) / FUSED_TXO;
    const int chunks = (s.L.ny + f->rows_per_chunk - 1) / f->rows_per_chunk;
    const bool contract = h->math == LF_MATH_CONTRACT;
    const bool muscl = h->d.spatial_order >= 2;
    ensure_fk(h);
    a.fk = contract ? f->fk_contract : f->fk_exact;
    auto launch = [&](int c0, int step, int n, cudaStream_t st) {
      if (n <= 0) return;
      a.chunk0 = c0;
      a.chunk_step = step;
      if (contract)
        launch_fused_step_contract(a, muscl, dim3(strips, n), st);
      else
        launch_fused_step(a, muscl, dim3(strips, n), st);
    };
    if (overlap && chunks >= 3) {
      launch(1, 1, chunks - 2, s.stream);                 // interior chunks
      launch(0, chunks - 1, 2, f->comm);                  // first and last, after the halos
      FK(cudaEventRecord(f->ev_edge, f->comm));
      FK(cudaStreamWaitEvent(s.stream, f->ev_edge, 0));
    } else {
      if (overlap) {
        FK(cudaEventRecord(f->ev_edge, f->comm));
        FK(cudaStreamWaitEvent(s.stream, f->ev_edge, 0));
      }
      launch(0, 1, chunks, s.stream);
    }
  }
  if (k1) FK(cudaEventRecord(k1, s0.stream));
  FK(cudaGetLastError());
  if (h->nccl)
    nccl_reduce_step(h, f->acc + cur, STEP_ACC_WORDS, bnd, sum_x ? 8 * (size_t)h->d.ny : 0,
                     bnd + 8 * (size_t)h->d.ny, sum_y ? 8 * (size_t)h->d.nx : 0);
  launch_finalize(f->ctl + cur, f->acc + cur, f->ctl + nxt, f->rec + n_in_batch, f->outflow,
                  !sum_x && !sum_y, h->d.dx, h->d.dy, cfl, limit, t_final, s0.stream);
  if (sum_x || sum_y) {
    FK(cudaEventRecord(f->ev_fin[cur], s0.stream));
    FK(cudaStreamWaitEvent(f->side, f->ev_fin[cur], 0));
    launch_outflow(f->rec + n_in_batch, bnd, f->outflow, h->d.nx, h->d.ny, sum_x, sum_y, h->d.dx,
                   h->d.dy, f->side);
    FK(cudaEventRecord(f->ev_out[cur], f->side));
  }
  FK(cudaGetLastError());
  for (auto& s : h->slabs) {
    std::swap(s.U, s.U2);
    if (mat) std::swap(s.P, s.P2);
  }
  f->cur = nxt;
}

// Run n fused steps from `time`; returns the number that completed (records
// in f->rec_host) and the index of a failed step (-1 if none).
static int run_batch(lf_handle* h, int n, double cfl, double limit, double t_final, double time,
                     const double* outflow_in, int* failed_at, bool timing, double* kernel_ms) {
  LF_TRACE("step batch");
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  seed_ctl(h, time);
  double o[4] = {0, 0, 0, 0};
  if (outflow_in) std::memcpy(o, outflow_in, sizeof o);
  std::memcpy(f->outflow_host, o, sizeof o);
  FK(cudaMemcpyAsync(f->outflow, f->outflow_host, sizeof o, cudaMemcpyHostToDevice, s0.stream));
  std::vector<cudaEvent_t> evs;
  if (timing) {
    evs.resize(2 * (size_t)n);
    for (auto& e : evs) FK(cudaEventCreate(&e));
  }
  const bool outsums = !(h->d.bc[0] == LF_PERIODIC && h->d.bc[1] == LF_PERIODIC) ||
                       !(h->d.bc[2] == LF_PERIODIC && h->d.bc[3] == LF_PERIODIC);
  // CUDA graphs pay where launch latency dominates the step: small single-material
  // grids (tools/graph_ab.py: Sod 400x4 38 -> 33 us per step, quadrant 1024^2 125 ->
  // 122); on the triple point (1.8M cells, 3 materials) the replay measured 9 % slower
  // than the stream launches (the side stream's low priority is not part of a graph)
  const bool small = (int64_t)h->d.nx * h->d.ny <= ((int64_t)1 << 20) && h->mc.n == 0;
  bool graph = !timing && n >= 8 && small && graphs_mode() != 0 && h->slabs.size() == 1 && !h->nccl;
  FusedState::GraphKey key{};
  if (graph) {
    key = FusedState::GraphKey{n,        f->cur,  s0.U,  s0.U2,   s0.Us,   s0.P,     s0.P2,
                               s0.Ps,    cfl,     limit, t_final, h->math, use_twopass(h) ? 1 : 0,
                               h->tp_exact};
    if (graphs_mode() == 1 && !f->graphs.count(key) && !f->seen.count(key)) {
      if (f->seen.size() >= 64) f->seen.clear();
      f->seen.insert(key);   // first sight: launch by launch
      graph = false;
    }
  }
  if (graph) {
    // CUDA graph of the whole batch (lf_advance batches; a single heun_step, whose
    // limit time may change from call to call, stays launch by launch): decide
    // everything that allocates or synchronises first, then capture once per key and
    // replay
    const bool twopass = use_twopass(h);
    if (!twopass) ensure_fk(h);
    if (outsums)  // the first two steps' bnd slots: the previous batch's sums
      for (int b = 0; b < 2; ++b) FK(cudaStreamWaitEvent(s0.stream, f->ev_out[b], 0));
    auto it = f->graphs.find(key);
    if (it == f->graphs.end()) {
      const long long l0 = launch_count();
      FK(cudaStreamBeginCapture(s0.stream, cudaStreamCaptureModeThreadLocal));
      f->capturing = true;
      try {
        for (int i = 0; i < n; ++i) enqueue_step(h, i, cfl, limit, t_final, nullptr, nullptr);
        if (outsums) FK(cudaStreamWaitEvent(s0.stream, f->ev_out[f->cur ^ 1], 0));
      } catch (...) {
        f->capturing = false;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(s0.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      f->capturing = false;
      cudaGraph_t g = nullptr;
      FK(cudaStreamEndCapture(s0.stream, &g));
      FusedState::Graph gr;
      const cudaError_t e = cudaGraphInstantiate(&gr.exec, g, 0);
      cudaGraphDestroy(g);
      FK(e);
      gr.launches = (int)(launch_count() - l0);
      count_launch(-gr.launches);   // counted when they run
      if (f->graphs.size() >= 16) drop_graphs(f);
      it = f->graphs.emplace(key, gr).first;
    } else {
      // what the captured enqueue_step calls did to the handle's host state
      for (int i = 0; i < n; ++i) {
        std::swap(s0.U, s0.U2);
        if (h->mc.n > 0) std::swap(s0.P, s0.P2);
        f->cur ^= 1;
      }
    }
    FK(cudaGraphLaunch(it->second.exec, s0.stream));
    count_launch(it->second.launches);
    // events recorded inside a capture belong to it: record them again, after the
    // replay (which joins the side stream), for the next launch-by-launch batch
    for (int b = 0; b < 2; ++b) {
      FK(cudaEventRecord(f->ev_fin[b], s0.stream));
      FK(cudaEventRecord(f->ev_out[b], s0.stream));
    }
  } else {
    for (int i = 0; i < n; ++i)
      enqueue_step(h, i, cfl, limit, t_final, timing ? evs[2 * i] : nullptr,
                   timing ? evs[2 * i + 1] : nullptr);
    // the side stream's last outflow sums (in-order) before the outflow comes back
    if (outsums) FK(cudaStreamWaitEvent(s0.stream, f->ev_out[f->cur ^ 1], 0));
  }
  FK(cudaMemcpyAsync(f->rec_host, f->rec, (size_t)n * sizeof(StepRec), cudaMemcpyDeviceToHost,
                     s0.stream));
  FK(cudaMemcpyAsync(f->outflow_host, f->outflow, 4 * sizeof(double), cudaMemcpyDeviceToHost,
                     s0.stream));
  for (auto& s : h->slabs) {
    FK(cudaSetDevice(s.device));
    FK(cudaStreamSynchronize(s.stream));
  }
  if (timing) {
    double ms = 0.0;
    for (int i = 0; i < n; ++i) {
      float x = 0.f;
      FK(cudaEventElapsedTime(&x, evs[2 * i], evs[2 * i + 1]));
      ms += x;
    }
    *kernel_ms = ms;
    for (auto& e : evs) cudaEventDestroy(e);
  }
  int done = 0;
  *failed_at = -1;
  for (int i = 0; i < n; ++i) {
    if (f->rec_host[i].status == 0) {
      ++done;
      continue;
    }
    if (f->rec_host[i].status == 1 || f->rec_host[i].status == 3) *failed_at = i;
    break;
  }
  // U/U2 were swapped once per enqueued step; the state after `done` steps is
  // the output of step done-1 (a failed or skipped step leaves its input intact)
  const int undo = n - done;
  if (undo & 1)
    for (auto& s : h->slabs) {
      std::swap(s.U, s.U2);
      if (h->mc.n) std::swap(s.P, s.P2);
    }
  f->cur = (f->cur + undo) & 1;
  f->valid = *failed_at < 0;
  return done;
}

static void to_out(const StepRec& r, int64_t step, double gm1, lf_step_out* o, bool mat = false) {
  o->dt = r.dt;
  o->hits_limit = r.hits;
  o->time = r.time;
  o->step = step;
  o->min_rho = r.min_rho;
  o->min_p = mat ? r.min_p_mat : gm1 * r.min_eint;
}

// A step flagged "needs exact" (status 3) by the plain two-pass kernels: switch
// the handle to the exact kernels (sticky) and report that it should be re-run.
static bool needs_exact(lf_handle* h, int i) {
  FusedState* f = fstate(h);
  if (f->rec_host[i].status != 3 || h->tp_exact) return false;
  h->tp_exact = 1;
  fused_invalidate(h);
  return true;
}

int fused_heun(lf_handle* h, double cfl, double time, double limit, int64_t step,
               double* outflow, lf_step_out* out) {
  fused_alloc(h, 1);
  int failed_at;
  int done = run_batch(h, 1, cfl, limit, limit, time, outflow, &failed_at, false, nullptr);
  if (done == 0 && failed_at == 0 && needs_exact(h, 0)) {
    done = run_batch(h, 1, cfl, limit, limit, time, outflow, &failed_at, false, nullptr);
  }
  if (done == 1) {
    if (outflow) std::memcpy(outflow, fstate(h)->outflow_host, 4 * sizeof(double));
    if (out) to_out(fstate(h)->rec_host[0], step + 1, h->d.gamma - 1.0, out, h->mc.n > 0);
    return 0;
  }
  // a flag was raised: the stage-wise kernels reproduce the exact error / state
  fused_invalidate(h);
  return staged_heun_public(h, cfl, time, limit, step, outflow, out);
}

int fused_advance(lf_handle* h, int nsteps, double cfl, double t_final, double* time,
                  int64_t* step, double* outflow, lf_step_out* per_step, int* taken) {
  if (taken) *taken = 0;
  int k = 0;
  // batches grow 16 -> 256: a flag early in a run (a shock precursor on the
  // plain kernels) discards at most a short batch of enqueued steps
  int cap = 16;
  while (k < nsteps && *time < t_final) {
    const int batch = std::min(nsteps - k, cap);
    cap = std::min(2 * cap, 256);
    fused_alloc(h, batch);
    FusedState* f = fstate(h);
    int failed_at;
    const int done = run_batch(h, batch, cfl, t_final, t_final, *time, outflow, &failed_at,
                               false, nullptr);
    for (int i = 0; i < done; ++i) {
      *step += 1;
      if (per_step) to_out(f->rec_host[i], *step, h->d.gamma - 1.0, &per_step[k + i], h->mc.n > 0);
      *time = f->rec_host[i].time;
    }
    k += done;
    if (taken) *taken = k;
    // the device outflow covers exactly the completed steps (finalize skips others)
    if (outflow) std::memcpy(outflow, f->outflow_host, 4 * sizeof(double));
    if (failed_at >= 0 && needs_exact(h, failed_at)) continue;  // the batch resumes, exact kernels
    if (failed_at >= 0) {
      fused_invalidate(h);
      lf_step_out o;
      const int rc = staged_heun_public(h, cfl, *time, t_final, *step, outflow, &o);
      if (rc) return rc;
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

int fused_time_steps(lf_handle* h, int nsteps, double cfl, double* kernel_ms, double* step_ms,
                     int* launches) {
  fused_alloc(h, nsteps);
  FusedState* f = fstate(h);
  SlabState& s0 = h->slabs[0];
  const double big = 1.7976931348623157e308;
  double t0 = 0.0;
  if (f->valid) {
    FK(cudaMemcpy(&f->ctl_host[1], &f->ctl[f->cur], sizeof(StepCtl), cudaMemcpyDeviceToHost));
    t0 = f->ctl_host[1].time;
  }
  FK(cudaEventRecord(f->e0, s0.stream));
  int failed_at;
  double kms = 0.0;
  int done = run_batch(h, nsteps, cfl, big, big, t0, nullptr, &failed_at, true, &kms);
  if (failed_at >= 0 && needs_exact(h, failed_at)) {
    // precursor velocities: time the exact kernels from the last completed step
    if (f->valid) {
      FK(cudaMemcpy(&f->ctl_host[1], &f->ctl[f->cur], sizeof(StepCtl), cudaMemcpyDeviceToHost));
      t0 = f->ctl_host[1].time;
    }
    FK(cudaEventRecord(f->e0, s0.stream));
    done = run_batch(h, nsteps, cfl, big, big, t0, nullptr, &failed_at, true, &kms);
  }
  FK(cudaEventRecord(f->e1, s0.stream));
  FK(cudaEventSynchronize(f->e1));
  float loop = 0.f;
  FK(cudaEventElapsedTime(&loop, f->e0, f->e1));
  *kernel_ms = kms;
  *step_ms = loop;
  *launches = done * (int)h->slabs.size();
  return failed_at >= 0 ? LF_ERR_DEVICE : 0;
}

}  // namespace lfb
