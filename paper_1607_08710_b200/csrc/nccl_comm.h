// nccl_comm.h -- inter-rank exchange for one-process-per-GPU y-slabs.
//
// NCCL is loaded with dlopen on first use (the torch-bundled libnccl.so.2 when
// torch is already in the process), so single-GPU use has no NCCL dependency.
// Per stage: NG halo rows to/from each y-neighbour (grouped send/recv, ring
// when y is periodic); per step: one all-reduce(min) over the packed scalars
// (the CFL rate max travels as ~bits, so max and min share one collective).
#pragma once

#include "handle.h"

namespace lfb {

int nccl_unique_id(void* id128);
int nccl_init(lf_handle* h, const void* id128);
void nccl_destroy(lf_handle* h);
// halo rows of `buf` with the y-neighbours, on `st` (default: the slab stream)
void nccl_exchange_halos(lf_handle* h, double* SlabState::*buf, int ncomp = 4,
                         cudaStream_t st = nullptr);
void nccl_combine_scalars(lf_handle* h, Scalars* s);
void nccl_max_u64(lf_handle* h, unsigned long long* v, int n);
// fused step: max-reduce n u64 step accumulators and sum-reduce the boundary
// faces (nbnd doubles, each rank owns disjoint entries, zero elsewhere) in place
// the step accumulators (max over ranks) and the boundary-face segments the outflow
// sums need (disjoint per rank, so a sum; nbnd_x / nbnd_y = 0 skips a segment)
void nccl_reduce_step(lf_handle* h, void* acc_u64, int n, double* bnd_x, size_t nbnd_x,
                      double* bnd_y, size_t nbnd_y);
// ordered chains over the ranks (interior totals): rank r-1 -> rank r, n doubles
void nccl_recv_prev(lf_handle* h, double* d, int n);
void nccl_send_next(lf_handle* h, const double* d, int n);
// in-place sum of n device doubles over the ranks
void nccl_sum_f64(lf_handle* h, double* d, int n);
// sum-combine the boundary-face arrays (each rank owns disjoint entries)
void nccl_gather_boundary(lf_handle* h, double* left, double* right, double* bot, double* top);

}  // namespace lfb
