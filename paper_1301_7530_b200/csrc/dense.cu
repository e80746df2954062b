// Small/skinny dense fp64 kernels: X^T Y (coarse matrix C^T A C,
// solver.py:113-114), X Q (Ritz vectors V Q, ritz.py:100), guarded Cholesky
// (core.py:195-243) + explicit coarse inverse, column norms / scaling (TRKS,
// recycle.py:127-140).
//
// These are bandwidth- or latency-bound at the shapes of the hot path
// (n_c <= ~100, s <= ~100 selected Ritz vectors), so they are plain
// smem-tiled CUDA-core fp64 kernels; tensor cores are not used (fp64 DMMA
// would not change the bound).  Every reduction is fixed-order.
#include "rcg_internal.cuh"
#include "dense.cuh"
#include "comm.cuh"

#include <cmath>
#include <vector>

namespace rcg {

// ---------------------------------------------------------------------------
// G = X^T Y, split over rows (grid.z) into fixed-order partials

constexpr int TN_T = 32;  // output tile edge

__global__ void __launch_bounds__(256)
gemm_tn_partial(int64_t n, int64_t a, int64_t b, const double* __restrict__ X, int64_t ldx,
                const double* __restrict__ Y, int64_t ldy, int64_t chunk, double* __restrict__ P) {
  __shared__ double Xs[32][TN_T + 1];
  __shared__ double Ys[32][TN_T + 1];
  const int t = threadIdx.x;
  const int ia = t & 31;
  const int ib0 = (t >> 5) * 4;
  const int64_t a0 = (int64_t)blockIdx.x * TN_T, b0 = (int64_t)blockIdx.y * TN_T;
  const int64_t r_begin = (int64_t)blockIdx.z * chunk;
  const int64_t r_end = min(n, r_begin + chunk);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 32) {
    // load 32 rows x 32 cols of X and Y (row index fastest -> coalesced)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rr = t & 31, cc = (t >> 5) + 8 * q;
      const int64_t row = r0 + rr;
      Xs[rr][cc] = (row < r_end && a0 + cc < a) ? X[(a0 + cc) * ldx + row] : 0.0;
      Ys[rr][cc] = (row < r_end && b0 + cc < b) ? Y[(b0 + cc) * ldy + row] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double xv = Xs[rr][ia];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += xv * Ys[rr][ib0 + q];
    }
    __syncthreads();
  }
  double* Pz = P + (size_t)blockIdx.z * a * b;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = a0 + ia, jj = b0 + ib0 + q;
    if (i < a && jj < b) Pz[jj * a + i] = acc[q];
  }
}

__global__ void gemm_tn_reduce(int64_t a, int64_t b, int S, const double* __restrict__ P, double* G,
                               int symmetrize) {
  const int64_t total = a * b;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % a, jj = idx / a;
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += P[(size_t)z * total + idx];
    if (symmetrize) {
      double s2 = 0.0;
      const int64_t tidx = i * a + jj;  // (jj, i)
      for (int z = 0; z < S; ++z) s2 += P[(size_t)z * total + tidx];
      s = 0.5 * (s + s2);
    }
    G[idx] = s;
  }
}

int gemm_tn(Ctx* c, int64_t n, int64_t a, int64_t b, const double* X, int64_t ldx, const double* Y,
            int64_t ldy, double* G, int symmetrize) {
  if (a == 0 || b == 0) return RCG_OK;
  const int64_t ta = ceil_div(a, TN_T), tb = ceil_div(b, TN_T);
  int64_t S = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 1024), (2 * c->num_sms) / (ta * tb)));
  if (S > 65535) S = 65535;
  int64_t chunk = ceil_div(ceil_div(n, S), 32) * 32;
  if (chunk == 0) chunk = 32;
  S = std::max<int64_t>(1, ceil_div(n, chunk));
  double* P = nullptr;
  int rc = scratch(c, sizeof(double) * (size_t)S * a * b, (void**)&P);
  if (rc) return rc;
  dim3 grid((unsigned)ta, (unsigned)tb, (unsigned)S);
  gemm_tn_partial<<<grid, 256, 0, c->stream>>>(n, a, b, X, ldx, Y, ldy, chunk, P);
  RCG_LAUNCH_CHECK(c);
  const int g = (int)std::min<int64_t>(ceil_div(a * b, 256), c->num_sms * 4);
  gemm_tn_reduce<<<g, 256, 0, c->stream>>>(a, b, (int)S, P, G, symmetrize);
  RCG_LAUNCH_CHECK(c);
  return RCG_OK;
}

// ---------------------------------------------------------------------------
// Y = X Q  (n x m) (m x s), tile 64 rows x 64 cols (4x4 per thread), k-slab
// 32: for s <= 64 selected Ritz vectors the history X is streamed once.

__global__ void __launch_bounds__(256)
gemm_nn_kernel(int64_t n, int64_t m, int64_t s, const double* __restrict__ X, int64_t ldx,
               const double* __restrict__ Q, int64_t ldq, double* __restrict__ Y, int64_t ldy) {
  __shared__ double Xs[32][64 + 1];
  __shared__ double Qs[32][64 + 1];
  const int t = threadIdx.x;
  const int tr = t & 15, tc = t >> 4;          // 16 x 16 threads
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int64_t col0 = (int64_t)blockIdx.y * 64;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  for (int64_t k0 = 0; k0 < m; k0 += 32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {             // 32 x 64 slab of X, rows contiguous
      const int e = t + 256 * q;
      const int kk = e >> 6, r = e & 63;
      const int64_t row = row0 + r;
      Xs[kk][r] = (row < n && k0 + kk < m) ? __ldcs(X + (k0 + kk) * ldx + row) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {             // 32 x 64 slab of Q
      const int e = t + 256 * q;
      const int kk = e & 31, cc = e >> 5;
      Qs[kk][cc] = (k0 + kk < m && col0 + cc < s) ? Q[(col0 + cc) * ldq + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      double xv[4], qv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = Xs[kk][tr + 16 * i];
#pragma unroll
      for (int q = 0; q < 4; ++q) qv[q] = Qs[kk][tc + 16 * q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] += xv[i] * qv[q];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = row0 + tr + 16 * i;
    if (row >= n) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t col = col0 + tc + 16 * q;
      if (col < s) Y[col * ldy + row] = acc[i][q];
    }
  }
}

int gemm_nn(Ctx* c, int64_t n, int64_t m, int64_t s, const double* X, int64_t ldx, const double* Q,
            int64_t ldq, double* Y, int64_t ldy) {
  if (n == 0 || s == 0) return RCG_OK;
  dim3 grid((unsigned)ceil_div(n, 64), (unsigned)ceil_div(s, 64));
  gemm_nn_kernel<<<grid, 256, 0, c->stream>>>(n, m, s, X, ldx, Q, ldq, Y, ldy);
  RCG_LAUNCH_CHECK(c);
  return RCG_OK;
}

// ---------------------------------------------------------------------------
// guarded Cholesky.  Pivot rule of core.py:233-243 (and the LAPACK branch
// core.py:226-232, which applies the same test to diag(L)^2):
//   d_j <= pivot_rtol * max(d_0..d_{j-1})  or  d_j <= 0  or  !isfinite(d_j)
//   -> RankDeficient(j) for the FIRST such j.

constexpr int CHOL_SMEM_MAX = 128;

// single CTA, whole matrix in shared memory (n <= 128), right-looking
__global__ void __launch_bounds__(1024)
chol_smem_kernel(int n, const double* __restrict__ G, double pivot_rtol, double* L, long long* bad) {
  extern __shared__ double A[];  // n x n, column-major
  __shared__ double s_piv;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  for (int idx = t; idx < n * n; idx += nt) A[idx] = G[idx];
  if (t == 0) {
    s_piv = 0.0;
    s_bad = -1;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double d = A[j * n + j];
    const double top = s_piv;
    if (d <= top * pivot_rtol || d <= 0.0 || !isfinite(d)) {
      if (t == 0) s_bad = j;
      break;  // uniform: every thread evaluates the same test
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (t == 0) s_piv = fmax(top, d);
    for (int i = j + 1 + t; i < n; i += nt) A[j * n + i] /= ljj;
    __syncthreads();
    if (t == 0) A[j * n + j] = ljj;
    // trailing update of the lower triangle
    const int m = n - j - 1;
    for (int idx = t; idx < m * m; idx += nt) {
      const int kk = j + 1 + idx / m, i = j + 1 + idx % m;
      if (i >= kk) A[kk * n + i] -= A[j * n + i] * A[j * n + kk];
    }
    __syncthreads();
  }
  __syncthreads();
  for (int idx = t; idx < n * n; idx += nt) {
    const int i = idx % n, kk = idx / n;
    L[idx] = (i >= kk) ? A[idx] : 0.0;
  }
  if (t == 0) *bad = s_bad;
}

// global-memory left-looking column step for large n: column j of L
// (launched once per column).  All blocks evaluate d_j identically.
__global__ void __launch_bounds__(256)
chol_col_kernel(int64_t n, int64_t j, const double* __restrict__ G, double* L, double* pivmax,
                double pivot_rtol, long long* bad) {
  if (*bad >= 0) return;
  __shared__ double sm[8];
  // d_j = G_jj - sum_k L_jk^2 (fixed-order block tree)
  double part = 0.0;
  for (int64_t k = threadIdx.x; k < j; k += blockDim.x) {
    const double v = L[k * n + j];
    part += v * v;
  }
  const double sumsq = block_sum<256>(part, sm);
  const double d = G[j * n + j] - sumsq;
  const double top = pivmax[j];
  if (d <= top * pivot_rtol || d <= 0.0 || !isfinite(d)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *bad = j;
    return;
  }
  const double ljj = sqrt(d);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    L[j * n + j] = ljj;
    pivmax[j + 1] = fmax(top, d);
  }
  for (int64_t i = j + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = G[j * n + i];
    for (int64_t k = 0; k < j; ++k) s -= L[k * n + i] * L[k * n + j];
    L[j * n + i] = s / ljj;
  }
}

// Blocked guarded Cholesky for n > 128 (TRKS bases reach n_c ~ 1.6 k):
// panels of CHOL_NB columns, three launches per panel -
//   (1) chol_update_kernel: A[p0:, p0:p0+nb] -= L[p0:, :p0] L[p0:p0+nb, :p0]^T
//       (left-looking GEMM, 64 x 64 tiles, fixed k order);
//   (2) chol_diag_kernel: one CTA factors the nb x nb diagonal block in smem
//       with the pivot rule (running max of the pivots in pivmax[0]);
//   (3) chol_trsm_kernel: L21 = A21 L11^-T, one thread per row, L11 in smem.
// L holds the working matrix (lower triangle of G copied in first).  A failed
// pivot sets *bad and every later launch returns at entry.
constexpr int CHOL_NB = 64;

__global__ void __launch_bounds__(256)
chol_update_kernel(int64_t n, int64_t p0, int nb, double* L, const long long* bad) {
  if (*bad >= 0) return;
  __shared__ double As[32][64 + 1];   // [k][row]
  __shared__ double Bs[32][64 + 1];   // [k][panel column]
  const int t = threadIdx.x, tr = t & 15, tc = t >> 4;
  const int64_t i0 = p0 + (int64_t)blockIdx.x * 64;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < p0; k0 += 32) {
    for (int idx = t; idx < 32 * 64; idx += 256) {
      const int kk = idx >> 6, rr = idx & 63;
      const int64_t k = k0 + kk, i = i0 + rr, c = p0 + rr;
      As[kk][rr] = (k < p0 && i < n) ? L[k * n + i] : 0.0;
      Bs[kk][rr] = (k < p0 && rr < nb) ? L[k * n + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][tr + 16 * u];
        b[u] = Bs[kk][tc + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = i0 + tr + 16 * u;
      const int c = tc + 16 * v;
      if (i < n && c < nb && i >= p0 + c) L[(p0 + c) * n + i] -= acc[u][v];
    }
}

__global__ void __launch_bounds__(1024)
chol_diag_kernel(int64_t n, int64_t p0, int nb, double* L, double* pivmax, double pivot_rtol, long long* bad) {
  if (*bad >= 0) return;
  __shared__ double A[CHOL_NB * CHOL_NB];   // nb x nb, column-major
  __shared__ double s_piv;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  for (int idx = t; idx < nb * nb; idx += nt) {
    const int i = idx % nb, c = idx / nb;
    A[idx] = i >= c ? L[(p0 + c) * n + p0 + i] : 0.0;
  }
  if (t == 0) {
    s_piv = *pivmax;
    s_bad = -1;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = A[j * nb + j];
    const double top = s_piv;
    if (d <= top * pivot_rtol || d <= 0.0 || !isfinite(d)) {
      if (t == 0) s_bad = j;
      break;  // uniform
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (t == 0) s_piv = fmax(top, d);
    for (int i = j + 1 + t; i < nb; i += nt) A[j * nb + i] /= ljj;
    __syncthreads();
    if (t == 0) A[j * nb + j] = ljj;
    const int m = nb - j - 1;
    for (int idx = t; idx < m * m; idx += nt) {
      const int kk = j + 1 + idx / m, i = j + 1 + idx % m;
      if (i >= kk) A[kk * nb + i] -= A[j * nb + i] * A[j * nb + kk];
    }
    __syncthreads();
  }
  __syncthreads();
  for (int idx = t; idx < nb * nb; idx += nt) {
    const int i = idx % nb, c = idx / nb;
    if (i >= c) L[(p0 + c) * n + p0 + i] = A[idx];
  }
  if (t == 0) {
    *pivmax = s_piv;
    if (s_bad >= 0) *bad = p0 + s_bad;
  }
}

constexpr int CHOL_TRSM_ROWS = 128;

__global__ void __launch_bounds__(CHOL_TRSM_ROWS)
chol_trsm_kernel(int64_t n, int64_t p0, int nb, double* L, const long long* bad) {
  if (*bad >= 0) return;
  extern __shared__ double trsm_sm[];
  double* L11 = trsm_sm;                                // nb x nb, column-major
  double* X = trsm_sm + CHOL_NB * CHOL_NB;              // [c][thread]
  const int t = threadIdx.x;
  for (int idx = t; idx < nb * nb; idx += CHOL_TRSM_ROWS) {
    const int i = idx % nb, c = idx / nb;
    L11[idx] = i >= c ? L[(p0 + c) * n + p0 + i] : 0.0;
  }
  const int64_t i = p0 + nb + (int64_t)blockIdx.x * CHOL_TRSM_ROWS + t;
  for (int c = 0; c < nb; ++c) X[c * CHOL_TRSM_ROWS + t] = i < n ? L[(p0 + c) * n + i] : 0.0;
  __syncthreads();
  if (i >= n) return;
  for (int c = 0; c < nb; ++c) {           // x_c = (a_c - sum_{k<c} x_k L11[c, k]) / L11[c, c]
    double s = X[c * CHOL_TRSM_ROWS + t];
    for (int k = 0; k < c; ++k) s -= X[k * CHOL_TRSM_ROWS + t] * L11[k * nb + c];
    X[c * CHOL_TRSM_ROWS + t] = s / L11[c * nb + c];
  }
  for (int c = 0; c < nb; ++c) L[(p0 + c) * n + i] = X[c * CHOL_TRSM_ROWS + t];
}

__global__ void copy_lower_kernel(int64_t n, const double* __restrict__ G, double* L) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, c = idx / n;
    L[idx] = i >= c ? G[idx] : 0.0;
  }
}

// Lt = L^T (so row i of L is contiguous for the warp-per-column inverse)
__global__ void transpose_kernel(int64_t n, const double* __restrict__ L, double* Lt) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = bx + threadIdx.x, c = by + r;
    tile[r][threadIdx.x] = (i < n && c < n) ? L[c * n + i] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t c = by + threadIdx.x, i = bx + r;
    if (i < n && c < n) Lt[i * n + c] = tile[threadIdx.x][r];
  }
}

// Linv = L^{-1}, one warp per column c: Linv[i, c] = (delta_ic - sum_{c<=k<i}
// L[i, k] Linv[k, c]) / L[i, i], the sum split over the lanes (contiguous
// rows of Lt) and warp-reduced in a fixed order
__global__ void __launch_bounds__(256)
trtri_warp_kernel(int64_t n, const double* __restrict__ Lt, double* Linv) {
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n) return;
  double* col = Linv + c * n;
  for (int64_t i = lane; i < c; i += 32) col[i] = 0.0;
  for (int64_t i = c; i < n; ++i) {
    const double* row = Lt + i * n;
    double p = 0.0;
    for (int64_t k = c + lane; k < i; k += 32) p += row[k] * col[k];
    p = warp_sum(p);
    if (lane == 0) col[i] = ((i == c ? 1.0 : 0.0) - p) / row[i];
    __syncwarp();
  }
}

// Linv = L^{-1} (lower), one thread per column, forward substitution
__global__ void trtri_lower_kernel(int64_t n, const double* __restrict__ L, double* Linv) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int64_t i = 0; i < c; ++i) Linv[c * n + i] = 0.0;
  for (int64_t i = c; i < n; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
    for (int64_t k = c; k < i; ++k) s -= L[k * n + i] * Linv[c * n + k];
    Linv[c * n + i] = s / L[i * n + i];
  }
}

int cholesky(Ctx* c, const double* G, int64_t n, double pivot_rtol, double* L, double* Ginv,
             int64_t* bad_col) {
  *bad_col = -1;
  if (n == 0) return RCG_OK;
  // scratch layout: [bad (8 B) | pad | pivmax (n+1)]
  const size_t need = 256 + sizeof(double) * (size_t)(n + 1);
  char* base = nullptr;
  int rc = scratch(c, need, (void**)&base);
  if (rc) return rc;
  long long* bad = (long long*)base;
  double* pivmax = (double*)(base + 256);
  if (n <= CHOL_SMEM_MAX) {
    const size_t smem = sizeof(double) * (size_t)n * n;
    RCG_CUDA(c, cudaFuncSetAttribute(chol_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 48 * 1024)));
    chol_smem_kernel<<<1, 1024, smem, c->stream>>>((int)n, G, pivot_rtol, L, bad);
    RCG_LAUNCH_CHECK(c);
  } else if (getenv("RCG_CHOL_COLUMNS")) {   // the per-column left-looking kernel (A/B reference)
    RCG_CUDA(c, cudaMemsetAsync(L, 0, sizeof(double) * (size_t)n * n, c->stream));
    RCG_CUDA(c, cudaMemsetAsync(pivmax, 0, sizeof(double) * (size_t)(n + 1), c->stream));
    RCG_CUDA(c, cudaMemsetAsync(bad, 0xff, sizeof(long long), c->stream));  // -1
    for (int64_t j = 0; j < n; ++j) {
      const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n - j, 256), c->num_sms));
      chol_col_kernel<<<g, 256, 0, c->stream>>>(n, j, G, L, pivmax, pivot_rtol, bad);
      RCG_LAUNCH_CHECK(c);
    }
  } else {
    RCG_CUDA(c, cudaMemsetAsync(pivmax, 0, sizeof(double), c->stream));
    RCG_CUDA(c, cudaMemsetAsync(bad, 0xff, sizeof(long long), c->stream));  // -1
    copy_lower_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * n, 256), 8 * c->num_sms), 256, 0, c->stream>>>(
        n, G, L);
    RCG_LAUNCH_CHECK(c);
    for (int64_t p0 = 0; p0 < n; p0 += CHOL_NB) {
      const int nb = (int)std::min<int64_t>(CHOL_NB, n - p0);
      if (p0 > 0) {
        chol_update_kernel<<<(unsigned)ceil_div(n - p0, (int64_t)64), 256, 0, c->stream>>>(n, p0, nb, L, bad);
        RCG_LAUNCH_CHECK(c);
      }
      chol_diag_kernel<<<1, 1024, 0, c->stream>>>(n, p0, nb, L, pivmax, pivot_rtol, bad);
      RCG_LAUNCH_CHECK(c);
      if (p0 + nb < n) {
        const int trsm_smem = (int)(sizeof(double) * CHOL_NB * (CHOL_NB + CHOL_TRSM_ROWS));
        RCG_CUDA(c, cudaFuncSetAttribute(chol_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem));
        chol_trsm_kernel<<<(unsigned)ceil_div(n - p0 - nb, (int64_t)CHOL_TRSM_ROWS), CHOL_TRSM_ROWS, trsm_smem,
                           c->stream>>>(n, p0, nb, L, bad);
        RCG_LAUNCH_CHECK(c);
      }
    }
  }
  long long hbad = -1;
  RCG_CUDA(c, cudaMemcpyAsync(&hbad, bad, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));
  if (hbad >= 0) {
    *bad_col = hbad;
    return set_error(c, RCG_ERR_RANK_DEFICIENT, "non-positive pivot at column %lld", hbad);
  }
  if (Ginv) {
    // Linv lives outside the ctx scratch because gemm_tn reuses the scratch
    double* Linv = nullptr;
    RCG_CUDA(c, cudaMallocAsync((void**)&Linv, sizeof(double) * (size_t)n * n, c->stream));
    if (n <= CHOL_SMEM_MAX) {
      trtri_lower_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, c->stream>>>(n, L, Linv);
      RCG_LAUNCH_CHECK(c);
    } else {
      double* Lt = nullptr;
      RCG_CUDA(c, cudaMallocAsync((void**)&Lt, sizeof(double) * (size_t)n * n, c->stream));
      transpose_kernel<<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32)), dim3(32, 8), 0, c->stream>>>(
          n, L, Lt);
      RCG_LAUNCH_CHECK(c);
      trtri_warp_kernel<<<(unsigned)ceil_div(n * 32, (int64_t)256), 256, 0, c->stream>>>(n, Lt, Linv);
      RCG_LAUNCH_CHECK(c);
      cudaFreeAsync(Lt, c->stream);
    }
    rc = gemm_tn(c, n, n, n, Linv, n, Linv, n, Ginv, 1);   // Ginv = Linv^T Linv
    cudaFreeAsync(Linv, c->stream);
    if (rc) return rc;
  }
  return RCG_OK;
}

// ---------------------------------------------------------------------------
// column norms / scaling (update_basis_trks, recycle.py:127-140)

__global__ void __launch_bounds__(256)
colnorm_kernel(int64_t n, const double* __restrict__ X, int64_t ldx, double* norms, int squared) {
  __shared__ double sm[8];
  const double* x = X + (int64_t)blockIdx.x * ldx;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
  s = block_sum<256>(s, sm);
  if (threadIdx.x == 0) norms[blockIdx.x] = squared ? s : sqrt(s);
}

__global__ void sqrt_kernel(int64_t k, double* v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = sqrt(v[i]);
}

__global__ void scalecol_kernel(int64_t n, int64_t k, const double* __restrict__ X, int64_t ldx,
                                const double* __restrict__ sdiv, double* Y, int64_t ldy) {
  const int64_t col = blockIdx.y;
  const double d = sdiv[col];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Y[col * ldy + i] = X[col * ldx + i] / d;
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_gemm_tn(rcg_ctx* ctx, int64_t n, int64_t a, int64_t b, const double* X, int64_t ldx,
                           const double* Y, int64_t ldy, double* G, int32_t symmetrize) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (symmetrize && a != b) return set_error(ctx, RCG_ERR_CONTRACT, "symmetrize needs a square result");
  return gemm_tn(ctx, n, a, b, X, ldx, Y, ldy, G, symmetrize);
}

extern "C" int rcg_gemm_nn(rcg_ctx* ctx, int64_t n, int64_t m, int64_t s, const double* X, int64_t ldx,
                           const double* Q, int64_t ldq, double* Y, int64_t ldy) {
  if (!ctx) return RCG_ERR_CONTRACT;
  return gemm_nn(ctx, n, m, s, X, ldx, Q, ldq, Y, ldy);
}

extern "C" int rcg_dense_cholesky(rcg_ctx* ctx, const double* G, int64_t n, double pivot_rtol, double* L,
                                  double* Ginv, int64_t* bad_col_host) {
  if (!ctx) return RCG_ERR_CONTRACT;
  int64_t bad = -1;
  int rc = cholesky(ctx, G, n, pivot_rtol, L, Ginv, &bad);
  if (bad_col_host) *bad_col_host = bad;
  return rc;
}

extern "C" int rcg_column_norms(rcg_ctx* ctx, int64_t n, int64_t k, const double* X, int64_t ldx,
                                double* norms) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (k == 0) return RCG_OK;
  colnorm_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(n, X, ldx, norms, 0);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}

extern "C" int rcg_column_norms_sharded(rcg_ctx* ctx, int64_t n, int64_t k, const double* X, int64_t ldx,
                                        double* norms) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (k == 0) return RCG_OK;
  colnorm_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(n, X, ldx, norms, 1);   // local sums of squares
  RCG_LAUNCH_CHECK(ctx);
  int rc = allreduce_sum(ctx, norms, (size_t)k);                                 // over the row slabs
  if (rc) return rc;
  sqrt_kernel<<<(unsigned)std::min<int64_t>(ceil_div(k, 256), 64), 256, 0, ctx->stream>>>(k, norms);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}

extern "C" int rcg_scale_columns(rcg_ctx* ctx, int64_t n, int64_t k, const double* X, int64_t ldx,
                                 const double* s, double* Y, int64_t ldy) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (k == 0 || n == 0) return RCG_OK;
  dim3 grid((unsigned)std::min<int64_t>(ceil_div(n, 256), 64), (unsigned)k);
  scalecol_kernel<<<grid, 256, 0, ctx->stream>>>(n, k, X, ldx, s, Y, ldy);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}
