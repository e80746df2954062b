#pragma once
#include "rcg_internal.cuh"

namespace rcg {
int comm_ranks(const Ctx* c);
// in-place fp64 sum over all ranks on the ctx stream (no-op on 1 rank)
int allreduce_sum(Ctx* c, double* buf, size_t count);
// pack src[send_idx] and exchange with every peer; received ghosts land at
// dst_col + n_local + recv_off[q] (no-op without a communicator)
int halo_exchange(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, double* dst_col);
void comm_free(Ctx* c);
}  // namespace rcg
