#pragma once
#include "rcg_internal.cuh"

namespace rcg {
int comm_ranks(const Ctx* c);
// in-place fp64 sum over all ranks on the ctx stream (no-op on 1 rank)
int allreduce_sum(Ctx* c, double* buf, size_t count);
// pack src[send_idx] and exchange with every peer; received ghosts land at
// dst_col + n_local + recv_off[q] (no-op without a communicator)
int halo_exchange(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, double* dst_col);
// solve-loop variant with fixed addresses (CUDA-graph capturable with NCCL):
// pack src.at(j), receive into the ctx staging buffer, unpack into
// dst.at(j)[n_local + ...] with j read from st on the device
// allocate the ctx staging buffer for H's ghosts (outside any graph capture)
int halo_prepare(Ctx* c, const rcg_halo* H);
// solve-loop exchange: column selectors and the state pointer are read from device memory (graph-replayable)
int halo_exchange_dev(Ctx* c, const rcg_halo* H, const ColSel* src_d, const SolveState* const* st_d,
                      const ColSel* dst_d);
// whether solve-loop batches of a sharded solve may be captured in a graph
bool comm_graphable(const Ctx* c);
bool halo_active(const Ctx* c, const rcg_halo* H);   // the exchange really moves data (peers, or a forced self exchange)
void comm_free(Ctx* c);
}  // namespace rcg
