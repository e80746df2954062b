#pragma once
#include "rcg_internal.cuh"

namespace rcg {
int gemm_tn(Ctx* c, int64_t n, int64_t a, int64_t b, const double* X, int64_t ldx, const double* Y,
            int64_t ldy, double* G, int symmetrize);
int gemm_nn(Ctx* c, int64_t n, int64_t m, int64_t s, const double* X, int64_t ldx, const double* Q,
            int64_t ldq, double* Y, int64_t ldy);
int cholesky(Ctx* c, const double* G, int64_t n, double pivot_rtol, double* L, double* Ginv,
             int64_t* bad_col);
}  // namespace rcg
