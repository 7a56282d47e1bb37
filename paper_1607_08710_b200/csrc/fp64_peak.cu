// fp64_peak.cu -- measured fp64 throughput of this GPU (the fp64 roof of bench.py).
//
// The Heun step is bound by the fp64 pipe and issue, not by HBM (DESIGN.md
// "Roofline"), and MEASURED_PEAKS.json holds no fp64 figure, so the bench
// measures one: every thread runs ILP independent chains of one fp64 operation
// (DFMA, DMUL or DADD, each one SASS instruction per thread per iteration), in
// enough warps per SM scheduler to hide the pipe latency.  Rates are thread
// instructions per second (a DFMA counts once; x2 for FLOP/s).
//
//   burst:     one launch of ~`ms` milliseconds after a warm-up launch
//   sustained: back-to-back launches for ~`sustain_ms` milliseconds
#include <cuda_runtime.h>

#include "../../include/lagflux_b200.h"
#include "kernels.h"

namespace lfb {
namespace {

constexpr int PK_THREADS = 256;
constexpr int PK_ILP = 8;

// op 0: DFMA, 1: DMUL, 2: DADD.  m = 1.0 and add = 0.0 arrive as kernel
// arguments (the compiler cannot fold them), so the chains keep their values;
// the result is stored only if an impossible condition holds.
template <int OP>
__global__ void __launch_bounds__(PK_THREADS) k_fp64_peak(long long iters, double m, double add,
                                                          double* sink) {
  double x[PK_ILP];
#pragma unroll
  for (int i = 0; i < PK_ILP; ++i) x[i] = 1.0 + 0x1p-30 * (i + threadIdx.x);
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int i = 0; i < PK_ILP; ++i) {
        if (OP == 0) x[i] = fma(x[i], m, add);
        else if (OP == 1) x[i] = x[i] * m;
        else x[i] = x[i] + add;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < PK_ILP; ++i) s += x[i];
  if (s == 1234.5678) sink[threadIdx.x] = s;
}

template <int OP>
double run_one(long long iters, int blocks, double* sink, cudaEvent_t e0, cudaEvent_t e1,
               float* ms_out, int reps) {
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) {
    count_launch();
    k_fp64_peak<OP><<<blocks, PK_THREADS>>>(iters, 1.0, 0.0, sink);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms;
  const double ops = (double)blocks * PK_THREADS * (double)iters * 4.0 * PK_ILP * reps;
  return ops / (ms * 1e-3);
}

template <int OP>
void measure(int blocks, double* sink, cudaEvent_t e0, cudaEvent_t e1, double burst_ms,
             double sustain_ms, double* burst, double* sustained) {
  // calibrate: a short launch, then scale the iteration count to ~burst_ms
  float ms = 0.f;
  long long iters = 4096;
  run_one<OP>(iters, blocks, sink, e0, e1, &ms, 1);   // warm-up
  run_one<OP>(iters, blocks, sink, e0, e1, &ms, 1);
  if (ms > 0.f) iters = (long long)(iters * (burst_ms / ms));
  if (iters < 1024) iters = 1024;
  *burst = run_one<OP>(iters, blocks, sink, e0, e1, &ms, 1);
  int reps = ms > 0.f ? (int)(sustain_ms / ms) : 1;
  if (reps < 1) reps = 1;
  *sustained = sustain_ms > 0 ? run_one<OP>(iters, blocks, sink, e0, e1, &ms, reps) : *burst;
}

}  // namespace
}  // namespace lfb

// out[6] = {DFMA burst, DFMA sustained, DMUL burst, DMUL sustained, DADD burst,
// DADD sustained}, fp64 thread instructions per second on `device`.
extern "C" int lf_fp64_peak(int device, double burst_ms, double sustain_ms, double* out) {
  if (!out || burst_ms <= 0.0 || sustain_ms < 0.0) return LF_ERR_ARGUMENT;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return LF_ERR_DEVICE;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // 8 blocks x 8 warps per SM = 16 warps per scheduler, 8 independent chains each
  const int blocks = sms * 8;
  double* sink = nullptr;
  if (cudaMalloc(&sink, lfb::PK_THREADS * sizeof(double)) != cudaSuccess) return LF_ERR_DEVICE;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  lfb::measure<0>(blocks, sink, e0, e1, burst_ms, sustain_ms, &out[0], &out[1]);
  lfb::measure<1>(blocks, sink, e0, e1, burst_ms, sustain_ms, &out[2], &out[3]);
  lfb::measure<2>(blocks, sink, e0, e1, burst_ms, sustain_ms, &out[4], &out[5]);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const bool ok = cudaGetLastError() == cudaSuccess;
  cudaSetDevice(prev);   // the caller's current device is left as it was
  return ok ? LF_OK : LF_ERR_DEVICE;
}
