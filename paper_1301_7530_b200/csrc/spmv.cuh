#pragma once
#include "rcg_internal.cuh"

namespace rcg {
// device-resident SpMV arguments (mode 1: y = A x + (x, y)) for graph replay
struct SpmvArgs {
  int64_t n;
  const void* ro;
  const int32_t* ci;
  const double* va;
  const int32_t* bro;
  const int32_t* bci;
  const double* bval;
  int32_t dia_nd, dia_block;
  const int64_t* dia_offsets;
  const double* dia_values;
  ColSel xs, ys;
  const SolveState* st;
  double* part;
  unsigned int* counter;
  double* out;
  unsigned int* claim;   // 3x3 block-DIA: tile claim counter (zero between launches; claim[1]: mode-0
                         // arrivals; claim[2]: arrivals of the ghost-column remainder kernel)
  int32_t rem_rows;      // row slab with a DIA copy: ghost-column remainder (rcg.h rcg_csr.rem_*)
  int32_t rem_width;
  const int32_t* rem_ids;
  const int32_t* rem_ci;
  const double* rem_va;
  double* rem_part;      // its block partials (after the main kernel's slots)
};
int launch_spmv_ind(Ctx* c, const rcg_csr* A, const SpmvArgs* dargs);
// a slab with a ghost-column remainder: the local part (reads local x only) and the ghost part
int launch_spmv_ind_main(Ctx* c, const rcg_csr* A, const SpmvArgs* dargs);
int launch_spmv_ind_rem(Ctx* c, const rcg_csr* A, const SpmvArgs* dargs);
bool spmv_has_rem(const rcg_csr* A);
void spmv_args_fill(const rcg_csr* A, SpmvArgs* s);
// mode 0: y = A x; 1: y = A x + (x,y) -> out[0]; 2: y = b - A x + (y,y),(b,b) -> out[0..1]
int launch_spmv(Ctx* c, const rcg_csr* A, int mode, ColSel xs, ColSel ys, const double* b,
                const SolveState* st, double* part, unsigned int* counter, double* out,
                unsigned int* claim = nullptr);
int spmv_partials(Ctx* c, const rcg_csr* A);
int spmv_main_partials(Ctx* c, const rcg_csr* A);
int spmv_width(const rcg_csr* A);  // number of partial slots per value
int elementwise_grid(Ctx* c, int64_t n);
}  // namespace rcg
