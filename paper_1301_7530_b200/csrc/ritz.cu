// Ritz extraction and stagnation selection on device — the between-solve part
// of the hot path: select_spectrum (/root/reference/pkg/src/recycg/recycle.py:
// 157-175) -> lanczos_from_trace / ritz_pairs (ritz.py:61-100) -> tridiag_eig
// (core.py:169-177, LAPACK dstevd in the reference) -> select_converged
// (ritz.py:103-138), and the SRKS block Y_sel / sqrt|theta| (recycle.py:151).
//
// Design: the north star's single-CTA Jacobi only covers
// m <= 256 and needs m^2 doubles of shared memory, but config-1 solves already
// reach m = 390 and elasticity solves reach thousands.  Instead:
//   * eigenvalues of H_m and H_{m-1}: Sturm-sequence bisection, one thread per
//     eigenvalue (O(m) per step, ~60-70 steps), parallel over all 2m-1 values;
//   * eigenvectors only for the requested (selected) values: inverse
//     iteration on the tridiagonal (partially pivoted LU, perturbed pivots)
//     with modified Gram-Schmidt inside clusters of near-equal values — the
//     published dstein algorithm, restated;
//   * Ritz vectors only for the selected columns: Y_sel = Z Qtilde, one skinny
//     fp64 GEMM over the device-resident z history (O(n m s), not O(n m^2)).
#include "rcg_internal.cuh"
#include "dense.cuh"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <vector>

namespace rcg {

// ---------------------------------------------------------------------------
// Lanczos tridiagonal (ritz.py:61-78)

__global__ void lanczos_kernel(const double* __restrict__ alphas, const double* __restrict__ betas, int64_t m,
                               double* d, double* e, int* neg) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    if (j == 0) {
      d[0] = 1.0 / alphas[0];
    } else {
      const double bj = betas[j - 1];
      if (bj < 0.0) atomicExch(neg, 1);
      d[j] = 1.0 / alphas[j] + bj / alphas[j - 1];
      e[j - 1] = sqrt(bj) / alphas[j - 1];
    }
  }
}

// ---------------------------------------------------------------------------
// Sturm bisection

struct TriBounds {
  double gl, gu, pivmin, onenrm;
};

__global__ void __launch_bounds__(256) bounds_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                     int64_t m, TriBounds* out) {
  __shared__ double s_lo[256], s_hi[256], s_e2[256], s_nrm[256];
  double lo = INFINITY, hi = -INFINITY, e2max = 0.0, nrm = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double el = i > 0 ? fabs(e[i - 1]) : 0.0;
    const double er = i + 1 < m ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - el - er);
    hi = fmax(hi, d[i] + el + er);
    nrm = fmax(nrm, fabs(d[i]) + el + er);
    if (i + 1 < m) e2max = fmax(e2max, e[i] * e[i]);
  }
  s_lo[threadIdx.x] = lo;
  s_hi[threadIdx.x] = hi;
  s_e2[threadIdx.x] = e2max;
  s_nrm[threadIdx.x] = nrm;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_lo[threadIdx.x] = fmin(s_lo[threadIdx.x], s_lo[threadIdx.x + s]);
      s_hi[threadIdx.x] = fmax(s_hi[threadIdx.x], s_hi[threadIdx.x + s]);
      s_e2[threadIdx.x] = fmax(s_e2[threadIdx.x], s_e2[threadIdx.x + s]);
      s_nrm[threadIdx.x] = fmax(s_nrm[threadIdx.x], s_nrm[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double pivmin = DBL_MIN * fmax(1.0, s_e2[0]);
    const double tnorm = fmax(fabs(s_lo[0]), fabs(s_hi[0]));
    const double ulp = DBL_EPSILON;
    const double fudge = 2.1 * tnorm * ulp * (double)m + 2.1 * 2.0 * pivmin;
    out->gl = s_lo[0] - fudge;
    out->gu = s_hi[0] + fudge;
    out->pivmin = pivmin;
    out->onenrm = s_nrm[0];
  }
}

// number of eigenvalues <= x (LDL^T inertia of T - x I)
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int64_t m,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q <= 0.0;
  for (int64_t i = 1; i < m; ++i) {
    q = d[i] - e2[i - 1] / q - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q <= 0.0;
  }
  return cnt;
}

__global__ void e2_kernel(const double* __restrict__ e, int64_t m1, double* e2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m1; i += (int64_t)gridDim.x * blockDim.x)
    e2[i] = e[i] * e[i];
}

// warp k -> k-th largest eigenvalue (descending order, as core.py:163-166):
// multisection — the 32 lanes evaluate Sturm counts at 31 interior points of
// the current bracket at once, so the bracket shrinks 32x per step (~11 steps
// to full precision instead of ~64 bisection steps).  The result is the same
// bracket-midpoint rule as bisection: the last bracket [lo, hi] has adjacent
// or equal floating-point ends.
__global__ void __launch_bounds__(128) bisect_kernel(const double* __restrict__ d, const double* __restrict__ e2,
                                                     int64_t m, const TriBounds* __restrict__ bnd,
                                                     double* values_desc) {
  const int lane = threadIdx.x & 31;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t target = m - k;  // smallest x with count(x) >= target is lambda_asc[m-1-k]
  double lo = bnd->gl, hi = bnd->gu;
  const double pivmin = bnd->pivmin;
  for (int it = 0; it < 64; ++it) {
    // lane q < 31 probes lo + (q+1)/32 (hi - lo)
    const double w = hi - lo;
    const double x = lo + w * ((double)(lane + 1) * (1.0 / 32.0));
    const bool valid = lane < 31 && x > lo && x < hi;
    const int cnt = valid ? sturm_count(d, e2, m, x, pivmin) : 0;
    const unsigned ge = __ballot_sync(0xffffffffu, valid && cnt >= target);
    const unsigned any_valid = __ballot_sync(0xffffffffu, valid);
    if (!any_valid) break;                      // bracket cannot be split further
    // new bracket: [last probe with count < target, first probe with count >= target]
    const int first = ge ? __ffs(ge) - 1 : 31;  // probes are increasing in x
    const double nlo_cand = __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0);
    const double nhi_cand = __shfl_sync(0xffffffffu, x, first < 31 ? first : 0);
    const double nlo = first > 0 ? nlo_cand : lo;
    const double nhi = (first < 31 && ((ge >> first) & 1u)) ? nhi_cand : hi;
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) values_desc[k] = lo + 0.5 * (hi - lo);
}

// ---------------------------------------------------------------------------
// stagnation selection (ritz.py:103-138), sequential semantics in one thread

__global__ void select_kernel(const double* __restrict__ cur, const double* __restrict__ prev, int64_t m,
                              double eps, uint8_t* mask) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double gap = 1e-12;  // DEGENERATE_GAP (ritz.py:23)
  for (int64_t j = 0; j < m; ++j) mask[j] = 0;
  if (m < 2) return;
  for (int64_t j = 0; j < m - 1; ++j) {
    if (fabs(cur[j] - prev[j]) <= eps * fabs(cur[j])) mask[j] = 1;
    if (fabs(cur[j + 1] - prev[j]) <= eps * fabs(cur[j + 1])) mask[j + 1] = 1;
  }
  for (int64_t j = 1; j < m; ++j) {
    const double denom = fmax(fabs(cur[j - 1]), fabs(cur[j]));
    if (denom > 0.0 && fabs(cur[j - 1] - cur[j]) < gap * denom) {
      if (mask[j]) {
        int64_t first = j - 1;
        while (first > 0 && fabs(cur[first - 1] - cur[first]) < gap * fmax(fabs(cur[first - 1]), fabs(cur[first])))
          --first;
        mask[first] = 1;
        mask[j] = 0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// inverse iteration (dstein restated).  One warp per task; a task is a run of
// ascending indices [start, start+count) of one cluster, processed in order.

struct EigTask {
  int64_t start;   // first ascending index
  int64_t count;
  int64_t out_col; // first output column in Qall
};

__device__ __forceinline__ double hash_uniform(uint64_t a, uint64_t b) {
  uint64_t x = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull);
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return ((double)(x >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;  // (-1, 1)
}

__global__ void __launch_bounds__(128)
eigvec_kernel(const double* __restrict__ d, const double* __restrict__ e, int64_t m,
              const double* __restrict__ vals_asc, const TriBounds* __restrict__ bnd, const EigTask* __restrict__ tasks,
              int ntasks, double* Qall, double* lu /* 5*m per warp */) {
  const int lane = threadIdx.x & 31;
  const int64_t wglob = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wglob >= ntasks) return;
  const EigTask t = tasks[wglob];
  double* u0 = lu + (size_t)wglob * 5 * m;
  double* u1 = u0 + m;
  double* u2 = u1 + m;
  double* lm = u2 + m;
  double* sw = lm + m;  // swap flags as doubles
  const double onenrm = bnd->onenrm;
  const double eps = DBL_EPSILON * 0.5;
  const double tol = eps * onenrm;  // pivot perturbation floor (dlagts job = -1)
  const double dtpcrt = sqrt(0.1 / (double)m);
  double xjm = 0.0;
  for (int64_t q = 0; q < t.count; ++q) {
    const int64_t ia = t.start + q;
    double xj = vals_asc[ia];
    if (q > 0) {
      const double pertol = 10.0 * fabs(eps * xj);
      if (xj - xjm < pertol) xj = xjm + pertol;
    }
    double* x = Qall + (size_t)(t.out_col + q) * m;
    // LU of T - xj I with partial pivoting (lane 0, sequential)
    if (lane == 0) {
      double cu = d[0] - xj, cv = m > 1 ? e[0] : 0.0;  // carry row (cols k, k+1)
      for (int64_t k = 0; k + 1 < m; ++k) {
        const double ek = e[k];
        const double dn = d[k + 1] - xj;
        const double en = k + 2 < m ? e[k + 1] : 0.0;
        if (fabs(ek) > fabs(cu)) {  // swap: pivot = original row k+1
          const double l = cu / ek;
          u0[k] = ek;
          u1[k] = dn;
          u2[k] = en;
          lm[k] = l;
          sw[k] = 1.0;
          const double ncu = cv - l * dn;
          const double ncv = -l * en;
          cu = ncu;
          cv = ncv;
        } else {
          double piv = cu;
          if (fabs(piv) < tol) piv = piv >= 0.0 ? tol : -tol;
          const double l = ek / piv;
          u0[k] = piv;
          u1[k] = cv;
          u2[k] = 0.0;
          lm[k] = l;
          sw[k] = 0.0;
          cu = dn - l * cv;
          cv = en;
        }
      }
      double piv = cu;
      if (fabs(piv) < tol) piv = piv >= 0.0 ? tol : -tol;
      u0[m - 1] = piv;
      for (int64_t k = 0; k + 1 < m; ++k)
        if (fabs(u0[k]) < tol) u0[k] = u0[k] >= 0.0 ? tol : -tol;
    }
    // random start vector
    for (int64_t i = lane; i < m; i += 32) x[i] = hash_uniform((uint64_t)ia + 1, (uint64_t)i);
    __syncwarp();
    int nrmchk = 0;
    for (int its = 0; its < 8; ++its) {
      // scale rhs: max entry -> m * onenrm * max(eps, |u_last|)
      double amax = 0.0;
      for (int64_t i = lane; i < m; i += 32) amax = fmax(amax, fabs(x[i]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      const double scl = (double)m * onenrm * fmax(eps, fabs(u0[m - 1])) / (amax > 0.0 ? amax : 1.0);
      for (int64_t i = lane; i < m; i += 32) x[i] *= scl;
      __syncwarp();
      // solve (forward with the recorded pivoting, then back substitution)
      if (lane == 0) {
        double carry = x[0];
        for (int64_t k = 0; k + 1 < m; ++k) {
          const double yk1 = x[k + 1];
          if (sw[k] != 0.0) {
            x[k] = yk1;
            carry = carry - lm[k] * yk1;
          } else {
            x[k] = carry;
            carry = yk1 - lm[k] * carry;
          }
        }
        x[m - 1] = carry;
        x[m - 1] = x[m - 1] / u0[m - 1];
        if (m > 1) x[m - 2] = (x[m - 2] - u1[m - 2] * x[m - 1]) / u0[m - 2];
        for (int64_t k = m - 3; k >= 0; --k) x[k] = (x[k] - u1[k] * x[k + 1] - u2[k] * x[k + 2]) / u0[k];
      }
      __syncwarp();
      // MGS against the earlier members of this cluster (normalized)
      for (int64_t p = 0; p < q; ++p) {
        const double* v = Qall + (size_t)(t.out_col + p) * m;
        double dot = 0.0;
        for (int64_t i = lane; i < m; i += 32) dot += x[i] * v[i];
        dot = warp_sum(dot);
        for (int64_t i = lane; i < m; i += 32) x[i] -= dot * v[i];
        __syncwarp();
      }
      double nrm = 0.0;
      for (int64_t i = lane; i < m; i += 32) nrm = fmax(nrm, fabs(x[i]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
      if (nrm < dtpcrt) continue;
      if (++nrmchk >= 3) break;  // EXTRA = 2 further iterations
    }
    // normalize, largest component positive
    double ss = 0.0, amax = 0.0, sgnv = 0.0;
    int64_t imax = 0;
    for (int64_t i = lane; i < m; i += 32) {
      ss += x[i] * x[i];
      if (fabs(x[i]) > amax) {
        amax = fabs(x[i]);
        imax = i;
      }
    }
    ss = warp_sum(ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, amax, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, (long long)imax, o);
      if (oa > amax || (oa == amax && oi < imax)) {
        amax = oa;
        imax = oi;
      }
    }
    sgnv = x[imax];
    double scl = 1.0 / sqrt(ss);
    if (sgnv < 0.0) scl = -scl;
    __syncwarp();
    for (int64_t i = lane; i < m; i += 32) x[i] *= scl;
    __syncwarp();
    xjm = xj;
  }
}

// Q[:, k] = Qall[:, col_of[k]]
__global__ void gather_cols_kernel(int64_t m, int64_t k, const double* __restrict__ Qall,
                                   const int64_t* __restrict__ col_of, double* Q, int64_t ldq) {
  const int64_t c = blockIdx.y;
  if (c >= k) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    Q[c * ldq + i] = Qall[(size_t)col_of[c] * m + i];
}

// Qtilde[i, c] = (-1)^i / sqrt(rz_i) * Q[i, c]  (/ sqrt|theta_c|)   (ritz.py:91-93, recycle.py:151)
__global__ void qtilde_kernel(int64_t m, int64_t k, const double* __restrict__ rz, const double* __restrict__ Q,
                              const double* __restrict__ theta_desc, const int64_t* __restrict__ idx, int scale,
                              double* Qt) {
  const int64_t c = blockIdx.y;
  double f = 1.0;
  if (scale) f = 1.0 / sqrt(fabs(theta_desc[idx[c]]));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double sgn = (i & 1) ? -1.0 : 1.0;
    Qt[c * m + i] = (sgn / sqrt(rz[i])) * Q[c * m + i] * f;
  }
}

int eigvals(Ctx* c, const double* d, const double* e, int64_t m, double* out, TriBounds* bnd, double* e2) {
  bounds_kernel<<<1, 256, 0, c->stream>>>(d, e, m, bnd);
  RCG_LAUNCH_CHECK(c);
  if (m > 1) {
    e2_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 64)), 256, 0, c->stream>>>(e, m - 1, e2);
    RCG_LAUNCH_CHECK(c);
  }
  bisect_kernel<<<(unsigned)ceil_div(m * 32, 128), 128, 0, c->stream>>>(d, e2, m, bnd, out);
  RCG_LAUNCH_CHECK(c);
  return RCG_OK;
}

struct Work {
  TriBounds* bnd = nullptr;
  double* e2 = nullptr;
};

int get_work(Ctx* c, int64_t m, Work* w) {
  char* base = nullptr;
  int rc = scratch(c, 512 + sizeof(double) * (size_t)(m + 1), (void**)&base);
  if (rc) return rc;
  w->bnd = (TriBounds*)base;
  w->e2 = (double*)(base + 512);
  return RCG_OK;
}

int eigvecs(Ctx* c, const double* d, const double* e, int64_t m, const double* values_desc, const int64_t* idx,
            int64_t k, double* Q, int64_t ldq) {
  if (k == 0 || m == 0) return RCG_OK;
  // host planning: clusters of near-equal values (gap <= 1e-6 ||T||_1) that
  // contain requested indices; every member of such a cluster is computed
  std::vector<double> vdesc(m);
  std::vector<int64_t> hidx(k);
  RCG_CUDA(c, cudaMemcpyAsync(vdesc.data(), values_desc, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA(c, cudaMemcpyAsync(hidx.data(), idx, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, c->stream));
  Work w;
  int rc = get_work(c, m, &w);
  if (rc) return rc;
  bounds_kernel<<<1, 256, 0, c->stream>>>(d, e, m, w.bnd);
  RCG_LAUNCH_CHECK(c);
  TriBounds hb;
  RCG_CUDA(c, cudaMemcpyAsync(&hb, w.bnd, sizeof(hb), cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));
  std::vector<double> asc(m);
  for (int64_t i = 0; i < m; ++i) asc[i] = vdesc[m - 1 - i];
  const double ortol = 1e-6 * hb.onenrm;
  std::vector<int64_t> cl_start(m), cl_end(m);
  {
    int64_t s = 0;
    for (int64_t i = 0; i < m; ++i) {
      if (i > 0 && fabs(asc[i] - asc[i - 1]) > ortol) s = i;
      cl_start[i] = s;
    }
    int64_t en = m - 1;
    for (int64_t i = m - 1; i >= 0; --i) {
      if (i < m - 1 && cl_start[i + 1] != cl_start[i]) en = i;
      cl_end[i] = en;
    }
  }
  std::vector<EigTask> tasks;
  std::vector<int64_t> col_of(k);
  std::vector<int64_t> task_of_start(m, -1);
  int64_t ncols = 0;
  for (int64_t q = 0; q < k; ++q) {
    const int64_t ia = m - 1 - hidx[q];
    if (hidx[q] < 0 || hidx[q] >= m) return set_error(c, RCG_ERR_CONTRACT, "eigenvector index out of range");
    const int64_t s = cl_start[ia];
    if (task_of_start[s] < 0) {
      task_of_start[s] = (int64_t)tasks.size();
      EigTask t;
      t.start = s;
      t.count = cl_end[ia] - s + 1;
      t.out_col = ncols;
      ncols += t.count;
      tasks.push_back(t);
    }
    const EigTask& t = tasks[task_of_start[s]];
    col_of[q] = t.out_col + (ia - t.start);
  }
  const int ntasks = (int)tasks.size();
  // device buffers: asc values, tasks, col_of, Qall, lu scratch
  const size_t bytes = sizeof(double) * m + sizeof(EigTask) * ntasks + sizeof(int64_t) * k +
                       sizeof(double) * (size_t)ncols * m + sizeof(double) * 5 * (size_t)m * ntasks + 1024;
  char* buf = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&buf, bytes, c->stream));
  double* d_asc = (double*)buf;
  EigTask* d_tasks = (EigTask*)(d_asc + m);
  int64_t* d_col = (int64_t*)(d_tasks + ntasks);
  double* d_Qall = (double*)(((uintptr_t)(d_col + k) + 255) & ~(uintptr_t)255);
  double* d_lu = d_Qall + (size_t)ncols * m;
  RCG_CUDA(c, cudaMemcpyAsync(d_asc, asc.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  RCG_CUDA(c, cudaMemcpyAsync(d_tasks, tasks.data(), sizeof(EigTask) * ntasks, cudaMemcpyHostToDevice, c->stream));
  RCG_CUDA(c, cudaMemcpyAsync(d_col, col_of.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, c->stream));
  eigvec_kernel<<<(unsigned)ceil_div((int64_t)ntasks * 32, 128), 128, 0, c->stream>>>(d, e, m, d_asc, w.bnd, d_tasks,
                                                                                     ntasks, d_Qall, d_lu);
  RCG_LAUNCH_CHECK(c);
  dim3 g((unsigned)std::min<int64_t>(ceil_div(m, 256), 32), (unsigned)k);
  gather_cols_kernel<<<g, 256, 0, c->stream>>>(m, k, d_Qall, d_col, Q, ldq);
  RCG_LAUNCH_CHECK(c);
  cudaFreeAsync(buf, c->stream);
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));  // host vectors above must outlive the copies
  return RCG_OK;
}


// ---------------------------------------------------------------------------
// cluster filter (ritz.py:141-183): the best three-segment constant fit of the
// m-1 gaps between consecutive Ritz values.  Every admissible split (a, b)
// (cluster = gaps [a, b), at least min_cluster-1 of them) is scored by its
// own thread; the per-CTA winners are then reduced in one CTA.  Scores use the
// reference's arithmetic exactly (sequential prefix sums, explicitly rounded
// products and quotients), so the winning split is the reference's, including
// its tie order (error, larger cluster, smaller gap level, smaller start).

struct ClusterBest {
  double err;
  double level;
  int64_t size;
  int64_t a;
};

__device__ __forceinline__ bool cluster_better(const ClusterBest& x, const ClusterBest& y) {
  if (x.err != y.err) return x.err < y.err;
  if (x.size != y.size) return x.size > y.size;
  if (x.level != y.level) return x.level < y.level;
  return x.a < y.a;
}

// one thread: sequential running sums of the gaps and squared gaps
// (numpy cumsum order), p[0] = 0
__global__ void cluster_prefix_kernel(const double* __restrict__ v, int64_t m, double* p1, double* p2) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s1 = 0.0, s2 = 0.0;
  p1[0] = 0.0;
  p2[0] = 0.0;
  for (int64_t i = 0; i + 1 < m; ++i) {
    const double g = fabs(__dsub_rn(v[i + 1], v[i]));
    s1 = __dadd_rn(s1, g);
    s2 = __dadd_rn(s2, __dmul_rn(g, g));
    p1[i + 1] = s1;
    p2[i + 1] = s2;
  }
}

__device__ __forceinline__ double seg_sse(const double* p1, const double* p2, int64_t i, int64_t j) {
  if (j <= i) return 0.0;
  const double s = __dsub_rn(p1[j], p1[i]);
  const double q = __dsub_rn(p2[j], p2[i]);
  return __dsub_rn(q, __ddiv_rn(__dmul_rn(s, s), (double)(j - i)));
}

template <int T>
__device__ void cluster_block_argmin(ClusterBest mine, ClusterBest* out) {
  __shared__ ClusterBest sb[T];
  sb[threadIdx.x] = mine;
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s && cluster_better(sb[threadIdx.x + s], sb[threadIdx.x])) sb[threadIdx.x] = sb[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sb[0];
}

// CTA q scores the splits whose cluster starts at a = q, q + G, ...; threads
// sweep the cluster end b
template <int T>
__global__ void __launch_bounds__(T) cluster_search_kernel(const double* __restrict__ p1, const double* __restrict__ p2,
                                                           int64_t ng, int64_t span, ClusterBest* part) {
  ClusterBest best{INFINITY, INFINITY, -1, INT64_MAX};
  for (int64_t a = blockIdx.x; a + span <= ng; a += gridDim.x) {
    const double head = seg_sse(p1, p2, 0, a);
    for (int64_t b = a + span + threadIdx.x; b <= ng; b += T) {
      const double err = __dadd_rn(__dadd_rn(head, seg_sse(p1, p2, a, b)), seg_sse(p1, p2, b, ng));
      const double level = b > a ? __ddiv_rn(__dsub_rn(p1[b], p1[a]), (double)(b - a)) : 0.0;
      const ClusterBest cand{err, level, b - a, a};
      if (cluster_better(cand, best)) best = cand;
    }
  }
  cluster_block_argmin<T>(best, part + blockIdx.x);
}

template <int T>
__global__ void __launch_bounds__(T) cluster_final_kernel(const ClusterBest* __restrict__ part, int n, ClusterBest* out) {
  ClusterBest best{INFINITY, INFINITY, -1, INT64_MAX};
  for (int i = threadIdx.x; i < n; i += T)
    if (cluster_better(part[i], best)) best = part[i];
  cluster_block_argmin<T>(best, out);
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_lanczos_tridiag(rcg_ctx* ctx, const double* alphas, const double* betas, int64_t m, double* d,
                                   double* e) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (m < 1) return set_error(ctx, RCG_ERR_CONTRACT, "need at least one iteration");
  int* neg = nullptr;
  int rc = scratch(ctx, 256, (void**)&neg);
  if (rc) return rc;
  RCG_CUDA(ctx, cudaMemsetAsync(neg, 0, sizeof(int), ctx->stream));
  lanczos_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 64)), 256, 0, ctx->stream>>>(
      alphas, betas, m, d, e, neg);
  RCG_LAUNCH_CHECK(ctx);
  int h = 0;
  RCG_CUDA(ctx, cudaMemcpyAsync(&h, neg, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RCG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (h) return set_error(ctx, RCG_ERR_NUMERICAL, "negative beta coefficient: operator not SPD");
  return RCG_OK;
}

extern "C" int rcg_tridiag_eigvals(rcg_ctx* ctx, const double* d, const double* e, int64_t m, double* values_desc) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (m < 1) return set_error(ctx, RCG_ERR_CONTRACT, "need |diag| >= 1");
  Work w;
  int rc = get_work(ctx, m, &w);
  if (rc) return rc;
  return eigvals(ctx, d, e, m, values_desc, w.bnd, w.e2);
}

extern "C" int rcg_tridiag_eigvecs(rcg_ctx* ctx, const double* d, const double* e, int64_t m,
                                   const double* values_desc, const int64_t* idx, int64_t k, double* Q) {
  if (!ctx) return RCG_ERR_CONTRACT;
  return eigvecs(ctx, d, e, m, values_desc, idx, k, Q, m);
}

extern "C" int rcg_select_converged(rcg_ctx* ctx, const double* cur, const double* prev, int64_t m, double epsilon,
                                    uint8_t* mask) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (!(epsilon > 0.0)) return set_error(ctx, RCG_ERR_CONTRACT, "epsilon must be positive");
  select_kernel<<<1, 32, 0, ctx->stream>>>(cur, prev, m, epsilon, mask);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}

extern "C" int rcg_ritz_select(rcg_ctx* ctx, const double* alphas, const double* betas, int64_t m, double epsilon,
                               double* d_work, double* e_work, double* values, double* prev, uint8_t* mask) {
  if (!ctx) return RCG_ERR_CONTRACT;
  int rc = rcg_lanczos_tridiag(ctx, alphas, betas, m, d_work, e_work);
  if (rc) return rc;
  Work w;
  if ((rc = get_work(ctx, m, &w))) return rc;
  if ((rc = eigvals(ctx, d_work, e_work, m, values, w.bnd, w.e2))) return rc;
  if (m >= 2) {
    // H_{m-1} is the leading principal block: same d/e pointers, m-1
    // (separate bounds so the two launches do not share scratch)
    TriBounds* b2 = w.bnd + 1;
    double* e2b = w.e2;  // e2 of the leading block is a prefix: recomputed identically
    if ((rc = eigvals(ctx, d_work, e_work, m - 1, prev, b2, e2b))) return rc;
  }
  if ((rc = rcg_select_converged(ctx, values, prev, m, epsilon, mask))) return rc;
  RCG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return RCG_OK;
}

extern "C" int rcg_ritz_vectors(rcg_ctx* ctx, const double* alphas, const double* betas, const double* rz, int64_t m,
                                const double* Z, int64_t ldz, int64_t n, const double* values_desc, const int64_t* idx,
                                int64_t k, int32_t scale_by_theta, double* Y, int64_t ldy) {
  if (!ctx) return RCG_ERR_CONTRACT;
  if (k == 0) return RCG_OK;
  Ctx* c = ctx;
  // d, e, Q, Qtilde
  char* buf = nullptr;
  const size_t bytes = sizeof(double) * (2 * (size_t)m + 2 * (size_t)m * k) + 1024;
  RCG_CUDA(c, cudaMallocAsync((void**)&buf, bytes, c->stream));
  double* d = (double*)buf;
  double* e = d + m;
  double* Q = e + m;
  double* Qt = Q + (size_t)m * k;
  int rc = rcg_lanczos_tridiag(ctx, alphas, betas, m, d, e);
  if (!rc) rc = eigvecs(c, d, e, m, values_desc, idx, k, Q, m);
  if (!rc) {
    dim3 g((unsigned)std::min<int64_t>(ceil_div(m, 256), 32), (unsigned)k);
    qtilde_kernel<<<g, 256, 0, c->stream>>>(m, k, rz, Q, values_desc, idx, scale_by_theta, Qt);
    c->launches++;
    rc = gemm_nn(c, n, m, k, Z, ldz, Qt, m, Y, ldy);       // Y = Z Qtilde
  }
  cudaFreeAsync(buf, c->stream);
  return rc;
}

extern "C" int rcg_cluster_filter(rcg_ctx* ctx, const double* values, int64_t m, int64_t min_cluster,
                                  int64_t* range_host) {
  if (!ctx || !range_host) return RCG_ERR_CONTRACT;
  if (min_cluster < 1) return set_error(ctx, RCG_ERR_CONTRACT, "min_cluster must be >= 1");
  if (m < min_cluster || m < 2) {  // no cluster: every value is kept (ritz.py:158-159)
    range_host[0] = m;
    range_host[1] = m - 1;
    return RCG_OK;
  }
  Ctx* c = ctx;
  const int64_t ng = m - 1, span = min_cluster - 1;
  const int G = (int)std::min<int64_t>(ng - span + 1, 4 * (int64_t)c->num_sms);
  constexpr int T = 256;
  char* buf = nullptr;
  const size_t bytes = sizeof(double) * 2 * (size_t)m + sizeof(ClusterBest) * (size_t)(G + 1) + 256;
  RCG_CUDA(c, cudaMallocAsync((void**)&buf, bytes, c->stream));
  double* p1 = (double*)buf;
  double* p2 = p1 + m;
  ClusterBest* part = (ClusterBest*)(((uintptr_t)(p2 + m) + 63) & ~(uintptr_t)63);
  ClusterBest* fin = part + G;
  cluster_prefix_kernel<<<1, 32, 0, c->stream>>>(values, m, p1, p2);
  cluster_search_kernel<T><<<G, T, 0, c->stream>>>(p1, p2, ng, span, part);
  cluster_final_kernel<T><<<1, T, 0, c->stream>>>(part, G, fin);
  c->launches += 3;
  ClusterBest h{};
  cudaError_t e = cudaMemcpyAsync(&h, fin, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
  cudaFreeAsync(buf, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_error(c, RCG_ERR_CUDA, "cluster filter: %s", cudaGetErrorString(e));
  // cluster = value indices a .. a + size (ritz.py:182-183)
  range_host[0] = h.a;
  range_host[1] = h.a + h.size;
  return RCG_OK;
}
