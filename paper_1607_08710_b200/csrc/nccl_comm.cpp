// nccl_comm.cpp -- NCCL plumbing for one-process-per-GPU y-slabs.
#include "nccl_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace lfb {

namespace {

struct Api {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Api g_api;

struct NcclFail : std::runtime_error {
  explicit NcclFail(const std::string& w) : std::runtime_error(w), what_(w) {}
  std::string what_;
};

bool load_api() {
  if (g_api.lib) return true;
  // LF_NCCL_LIB: another implementation of the same entry points (the tests'
  // thread-rank stand-in, tests/fake_nccl)
  const char* over = std::getenv("LF_NCCL_LIB");
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  if (over && over[0]) g_api.lib = dlopen(over, RTLD_NOW | RTLD_LOCAL);
  for (const char* n : names) {
    if (g_api.lib) break;
    g_api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!g_api.lib) return false;
#define SYM(field, name) g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(g_api.lib, name))
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(AllReduce, "ncclAllReduce");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  return g_api.GetUniqueId && g_api.CommInitRank && g_api.AllReduce && g_api.Send && g_api.Recv;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw NcclFail(std::string(what) + ": " +
                   (g_api.GetErrorString ? g_api.GetErrorString(r) : "nccl error"));
}

void cck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw NcclFail(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

struct Nccl {
  ncclComm_t comm = nullptr;
  unsigned long long* dbuf = nullptr;  // device staging for small reductions
  double* dbnd = nullptr;              // device staging for boundary faces
  size_t dbnd_n = 0;
};

int nccl_unique_id(void* id128) {
  if (!load_api()) return LF_ERR_DEVICE;
  ncclUniqueId id;
  if (g_api.GetUniqueId(&id) != ncclSuccess) return LF_ERR_DEVICE;
  std::memcpy(id128, &id, sizeof id);
  return 0;
}

int nccl_init(lf_handle* h, const void* id128) {
  if (!load_api()) {
    h->err.kind = LF_ERR_DEVICE;
    std::snprintf(h->err.message, sizeof h->err.message, "libnccl.so.2 could not be loaded");
    return LF_ERR_DEVICE;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  auto* n = new Nccl;
  try {
    cck(cudaSetDevice(h->slabs[0].device), "cudaSetDevice");
    nck(g_api.CommInitRank(&n->comm, h->nranks, id, h->rank), "ncclCommInitRank");
    cck(cudaMalloc(&n->dbuf, 16 * sizeof(unsigned long long)), "cudaMalloc");
  } catch (const NcclFail& f) {
    delete n;
    h->err.kind = LF_ERR_DEVICE;
    std::snprintf(h->err.message, sizeof h->err.message, "%s", f.what());
    return LF_ERR_DEVICE;
  }
  h->nccl = n;
  return 0;
}

void nccl_destroy(lf_handle* h) {
  if (!h->nccl) return;
  if (h->nccl->comm && g_api.CommDestroy) g_api.CommDestroy(h->nccl->comm);
  cudaFree(h->nccl->dbuf);
  cudaFree(h->nccl->dbnd);
  delete h->nccl;
  h->nccl = nullptr;
}

// Two phases so that matching is unambiguous even for 2 ranks on a periodic
// ring (both neighbours are the same peer): A sends the bottom NG rows down and
// receives the top halo from above; B sends the top rows up and receives the
// bottom halo from below.  Rows are whole padded rows (x ghosts included).
void nccl_exchange_halos(lf_handle* h, double* SlabState::*buf, int ncomp, cudaStream_t st) {
  SlabState& s = h->slabs[0];
  if (!st) st = s.stream;
  const bool periodic = h->d.bc[2] == LF_PERIODIC;
  const int R = h->nranks, r = h->rank;
  const int lo = r > 0 ? r - 1 : (periodic ? R - 1 : -1);
  const int hi = r < R - 1 ? r + 1 : (periodic ? 0 : -1);
  const size_t n = (size_t)NG * s.L.pitch;
  double* base = (s.*buf) + s.L.origin() - XPAD;  // row 0, allocation column 0
  auto rows = [&](int c, int row) { return base + c * s.L.fstride + (int64_t)row * s.L.pitch; };
  nck(g_api.GroupStart(), "ncclGroupStart");
  for (int c = 0; c < ncomp; ++c) {  // phase A
    if (lo >= 0) nck(g_api.Send(rows(c, 0), n, ncclFloat64, lo, h->nccl->comm, st), "ncclSend");
    if (hi >= 0) nck(g_api.Recv(rows(c, s.L.ny), n, ncclFloat64, hi, h->nccl->comm, st), "ncclRecv");
  }
  for (int c = 0; c < ncomp; ++c) {  // phase B
    if (hi >= 0)
      nck(g_api.Send(rows(c, s.L.ny - NG), n, ncclFloat64, hi, h->nccl->comm, st), "ncclSend");
    if (lo >= 0) nck(g_api.Recv(rows(c, -NG), n, ncclFloat64, lo, h->nccl->comm, st), "ncclRecv");
  }
  nck(g_api.GroupEnd(), "ncclGroupEnd");
}

void nccl_combine_scalars(lf_handle* h, Scalars* sc) {
  SlabState& s = h->slabs[0];
  unsigned long long v[9] = {~sc->rate_bits,
                             (unsigned long long)sc->fail_dt,
                             (unsigned long long)sc->fail_prim,
                             (unsigned long long)sc->fail_trace,
                             (unsigned long long)sc->fail_update,
                             sc->min_rho_bits,
                             sc->min_eint_bits,
                             (unsigned long long)sc->fail_frac,
                             sc->min_p_key};
  cck(cudaMemcpyAsync(h->nccl->dbuf, v, sizeof v, cudaMemcpyHostToDevice, s.stream), "copy");
  nck(g_api.AllReduce(h->nccl->dbuf, h->nccl->dbuf, 9, ncclUint64, ncclMin, h->nccl->comm, s.stream),
      "ncclAllReduce");
  cck(cudaMemcpyAsync(v, h->nccl->dbuf, sizeof v, cudaMemcpyDeviceToHost, s.stream), "copy");
  cck(cudaStreamSynchronize(s.stream), "sync");
  sc->rate_bits = ~v[0];
  sc->fail_dt = (long long)v[1];
  sc->fail_prim = (long long)v[2];
  sc->fail_trace = (long long)v[3];
  sc->fail_update = (long long)v[4];
  sc->min_rho_bits = v[5];
  sc->min_eint_bits = v[6];
  sc->fail_frac = (long long)v[7];
  sc->min_p_key = v[8];
}

void nccl_max_u64(lf_handle* h, unsigned long long* v, int n) {
  SlabState& s = h->slabs[0];
  cck(cudaMemcpyAsync(h->nccl->dbuf, v, n * sizeof(*v), cudaMemcpyHostToDevice, s.stream), "copy");
  nck(g_api.AllReduce(h->nccl->dbuf, h->nccl->dbuf, (size_t)n, ncclUint64, ncclMax, h->nccl->comm,
                      s.stream),
      "ncclAllReduce");
  cck(cudaMemcpyAsync(v, h->nccl->dbuf, n * sizeof(*v), cudaMemcpyDeviceToHost, s.stream), "copy");
  cck(cudaStreamSynchronize(s.stream), "sync");
}

void nccl_recv_prev(lf_handle* h, double* d, int n) {
  if (h->rank == 0) return;
  nck(g_api.Recv(d, (size_t)n, ncclFloat64, h->rank - 1, h->nccl->comm, h->slabs[0].stream),
      "ncclRecv");
}

void nccl_send_next(lf_handle* h, const double* d, int n) {
  if (h->rank == h->nranks - 1) return;
  nck(g_api.Send(d, (size_t)n, ncclFloat64, h->rank + 1, h->nccl->comm, h->slabs[0].stream),
      "ncclSend");
}

void nccl_sum_f64(lf_handle* h, double* d, int n) {
  nck(g_api.AllReduce(d, d, (size_t)n, ncclFloat64, ncclSum, h->nccl->comm, h->slabs[0].stream),
      "ncclAllReduce");
}

void nccl_gather_boundary(lf_handle* h, double* left, double* right, double* bot, double* top) {
  SlabState& s = h->slabs[0];
  const size_t ny = (size_t)h->d.ny, nx = (size_t)h->d.nx;
  const size_t total = 8 * ny + 8 * nx;
  Nccl* n = h->nccl;
  if (n->dbnd_n < total) {
    cudaFree(n->dbnd);
    cck(cudaMalloc(&n->dbnd, total * sizeof(double)), "cudaMalloc");
    n->dbnd_n = total;
  }
  std::vector<double> host(total);
  // each rank owns disjoint entries and zero elsewhere: the sum is exact
  std::memcpy(&host[0], left, 4 * ny * sizeof(double));
  std::memcpy(&host[4 * ny], right, 4 * ny * sizeof(double));
  std::memcpy(&host[8 * ny], bot, 4 * nx * sizeof(double));
  std::memcpy(&host[8 * ny + 4 * nx], top, 4 * nx * sizeof(double));
  cck(cudaMemcpyAsync(n->dbnd, host.data(), total * sizeof(double), cudaMemcpyHostToDevice, s.stream),
      "copy");
  nck(g_api.AllReduce(n->dbnd, n->dbnd, total, ncclFloat64, ncclSum, n->comm, s.stream),
      "ncclAllReduce");
  cck(cudaMemcpyAsync(host.data(), n->dbnd, total * sizeof(double), cudaMemcpyDeviceToHost, s.stream),
      "copy");
  cck(cudaStreamSynchronize(s.stream), "sync");
  std::memcpy(left, &host[0], 4 * ny * sizeof(double));
  std::memcpy(right, &host[4 * ny], 4 * ny * sizeof(double));
  std::memcpy(bot, &host[8 * ny], 4 * nx * sizeof(double));
  std::memcpy(top, &host[8 * ny + 4 * nx], 4 * nx * sizeof(double));
}

}  // namespace lfb

namespace lfb {

void nccl_reduce_step(lf_handle* h, void* acc_u64, int n, double* bnd_x, size_t nbnd_x,
                      double* bnd_y, size_t nbnd_y) {
  SlabState& s = h->slabs[0];
  nck(g_api.GroupStart(), "ncclGroupStart");
  nck(g_api.AllReduce(acc_u64, acc_u64, (size_t)n, ncclUint64, ncclMax, h->nccl->comm, s.stream),
      "ncclAllReduce(step)");
  if (nbnd_x)
    nck(g_api.AllReduce(bnd_x, bnd_x, nbnd_x, ncclFloat64, ncclSum, h->nccl->comm, s.stream),
        "ncclAllReduce(boundary x)");
  if (nbnd_y)
    nck(g_api.AllReduce(bnd_y, bnd_y, nbnd_y, ncclFloat64, ncclSum, h->nccl->comm, s.stream),
        "ncclAllReduce(boundary y)");
  nck(g_api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace lfb
