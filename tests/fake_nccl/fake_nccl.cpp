// fake_nccl.cpp -- test infrastructure: the subset of NCCL the library uses
// (nccl_comm.cpp), for ranks that are host threads of one process, so the
// distributed code path (lf_create_dist: halos, step reductions, boundary sums,
// the interior_totals chain) runs on one GPU.  Loaded through LF_NCCL_LIB.
//
// Nothing here makes a kernel wait on another rank: point-to-point transfers
// are stream-ordered copies (the receiver's stream waits on an event the sender
// recorded when it posted the send, the sender's stream then waits on the
// receiver's copy), and all-reduces are done on the host after every rank's
// stream has been synchronised.  The host threads rendezvous; the GPU only sees
// ordinary stream dependencies.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace {

struct Post {  // a posted send
  const void* buf;
  size_t bytes;
  cudaEvent_t ready;   // recorded on the sender's stream at post time
  cudaEvent_t done;    // recorded by the receiver after its copy
  bool copied = false;
};

struct Group {
  int nranks = 0;
  int joined = 0;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<Post*>> mail;   // (src, dst) -> posted sends
  // all-reduce rounds
  long round = 0;
  int arrived = 0;
  std::vector<std::vector<unsigned char>> snap;
};

std::mutex g_reg_m;
std::map<std::string, Group*> g_reg;
std::atomic<unsigned long long> g_id{1};

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

struct Op {
  enum Kind { SEND, RECV, ALLREDUCE } kind;
  const void* sbuf;
  void* rbuf;
  size_t count;
  ncclDataType_t type;
  ncclRedOp_t red;
  int peer;
  cudaStream_t st;
};

thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

}  // namespace

struct ncclComm {
  Group* g;
  int rank;
};

namespace {

void barrier(Group* g) {
  std::unique_lock<std::mutex> lk(g->m);
  const long r = g->round;
  if (++g->arrived == g->nranks) {
    g->arrived = 0;
    ++g->round;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->round != r; });
  }
}

template <class T>
void reduce_into(std::vector<unsigned char>& acc, const std::vector<unsigned char>& x, size_t n,
                 ncclRedOp_t op) {
  T* a = reinterpret_cast<T*>(acc.data());
  const T* b = reinterpret_cast<const T*>(x.data());
  for (size_t i = 0; i < n; ++i) {
    switch (op) {
      case ncclSum: a[i] = a[i] + b[i]; break;
      case ncclMax: a[i] = std::max(a[i], b[i]); break;
      case ncclMin: a[i] = std::min(a[i], b[i]); break;
      default: break;
    }
  }
}

void allreduce(ncclComm* c, const Op& o) {
  Group* g = c->g;
  const size_t bytes = o.count * type_size(o.type);
  cudaStreamSynchronize(o.st);
  std::vector<unsigned char> mine(bytes);
  cudaMemcpy(mine.data(), o.sbuf, bytes, cudaMemcpyDeviceToHost);
  {
    std::lock_guard<std::mutex> lk(g->m);
    if (g->snap.size() != (size_t)g->nranks) g->snap.assign(g->nranks, {});
    g->snap[c->rank] = mine;
  }
  barrier(g);   // every rank's input snapshotted
  std::vector<unsigned char> acc;
  {
    std::lock_guard<std::mutex> lk(g->m);
    acc = g->snap[0];   // ranks combined in rank order (sums: +0.0 terms only here)
    for (int r = 1; r < g->nranks; ++r) {
      if (o.type == ncclFloat64) reduce_into<double>(acc, g->snap[r], o.count, o.red);
      else if (o.type == ncclUint64) reduce_into<unsigned long long>(acc, g->snap[r], o.count, o.red);
      else if (o.type == ncclInt64) reduce_into<long long>(acc, g->snap[r], o.count, o.red);
    }
  }
  barrier(g);   // everyone has read the snapshots
  cudaMemcpy(o.rbuf, acc.data(), bytes, cudaMemcpyHostToDevice);
}

void run_ops(ncclComm* c, std::vector<Op>& ops) {
  Group* g = c->g;
  std::vector<Post*> mine;
  // 1. post every send
  for (const Op& o : ops)
    if (o.kind == Op::SEND) {
      Post* p = new Post{o.sbuf, o.count * type_size(o.type), nullptr, nullptr};
      cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming);
      cudaEventRecord(p->ready, o.st);
      std::lock_guard<std::mutex> lk(g->m);
      g->mail[{c->rank, o.peer}].push_back(p);
      mine.push_back(p);
      g->cv.notify_all();
    }
  // 2. all-reduces, in order
  for (const Op& o : ops)
    if (o.kind == Op::ALLREDUCE) allreduce(c, o);
  // 3. receives: the k-th receive from a peer takes its k-th send to this rank
  for (const Op& o : ops)
    if (o.kind == Op::RECV) {
      Post* p = nullptr;
      {
        std::unique_lock<std::mutex> lk(g->m);
        auto& q = g->mail[{o.peer, c->rank}];
        g->cv.wait(lk, [&] { return !q.empty(); });
        p = q.front();
        q.pop_front();
      }
      cudaStreamWaitEvent(o.st, p->ready, 0);
      cudaMemcpyAsync(o.rbuf, p->buf, std::min(p->bytes, o.count * type_size(o.type)),
                      cudaMemcpyDeviceToDevice, o.st);
      cudaEventRecord(p->done, o.st);
      std::lock_guard<std::mutex> lk(g->m);
      p->copied = true;
      g->cv.notify_all();
    }
  // 4. a send completes when its receiver has copied it
  for (Post* p : mine) {
    {
      std::unique_lock<std::mutex> lk(g->m);
      g->cv.wait(lk, [&] { return p->copied; });
    }
    cudaStream_t st = nullptr;
    for (const Op& o : ops)
      if (o.kind == Op::SEND && o.sbuf == p->buf) st = o.st;
    cudaStreamWaitEvent(st, p->done, 0);
    cudaEventDestroy(p->ready);
    cudaEventDestroy(p->done);
    delete p;
  }
}

ncclResult_t submit(const Op& o, ncclComm* c) {
  if (t_depth > 0) {
    t_ops.push_back(o);
    return ncclSuccess;
  }
  std::vector<Op> one{o};
  run_ops(c, one);
  return ncclSuccess;
}

thread_local ncclComm* t_group_comm = nullptr;

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof *id);
  const unsigned long long v = g_id++;
  std::memcpy(id->internal, "fakenccl", 8);
  std::memcpy(id->internal + 8, &v, sizeof v);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  const std::string key(id.internal, 16);
  Group* g;
  {
    std::lock_guard<std::mutex> lk(g_reg_m);
    auto it = g_reg.find(key);
    if (it == g_reg.end()) {
      g = new Group;
      g->nranks = nranks;
      g_reg[key] = g;
    } else {
      g = it->second;
    }
  }
  {
    std::unique_lock<std::mutex> lk(g->m);
    ++g->joined;
    g->cv.notify_all();
    g->cv.wait(lk, [&] { return g->joined >= g->nranks; });
  }
  *comm = new ncclComm{g, rank};
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;   // (the group stays registered: ids are never reused)
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* s, void* r, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  t_group_comm = comm;
  return submit(Op{Op::ALLREDUCE, s, r, count, t, op, -1, st}, comm);
}

ncclResult_t ncclSend(const void* s, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t st) {
  t_group_comm = comm;
  return submit(Op{Op::SEND, s, nullptr, count, t, ncclSum, peer, st}, comm);
}

ncclResult_t ncclRecv(void* r, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t st) {
  t_group_comm = comm;
  return submit(Op{Op::RECV, nullptr, r, count, t, ncclSum, peer, st}, comm);
}

ncclResult_t ncclGroupStart() {
  ++t_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--t_depth == 0 && !t_ops.empty()) {
    std::vector<Op> ops;
    ops.swap(t_ops);
    run_ops(t_group_comm, ops);
  }
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t) { return "fake nccl error"; }

}  // extern "C"
