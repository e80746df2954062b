// Layout microbenchmark with the real reorth access patterns:
//  precond-like: per tile (R rows) warps own 8-column groups, 2 vectors (z, w), 128-bit loads
//  wupdate-like: thread-per-row (4 rows / thread), loop over all columns, coefficients in smem
// layouts: 0 = column-major (col k at base + k*ld)
//          1 = column-block panels: (k/8, tile) panel of 8 x R doubles contiguous
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 2048, CG = 8;
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int L>
__device__ __forceinline__ const double* colp(const double* M, long long ld, long long ntile, long long t, int k) {
  return L == 0 ? M + k * ld + t * R : M + (((long long)(k / CG) * ntile + t) * CG + (k % CG)) * R;
}
template <int L>
__global__ void __launch_bounds__(256) pre(const double* __restrict__ M, long long n, long long ld, long long ntile,
                                           int J, const double* __restrict__ z, double* out) {
  __shared__ double zt[R], wt[R];
  const long long t = blockIdx.x;
  for (int i = threadIdx.x; i < R; i += 256) { zt[i] = z[t * R + i]; wt[i] = z[t * R + i] * 0.5; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double tot = 0.0;
  for (int g = wid; g * CG < J; g += 8) {
    double a[CG] = {0}, b[CG] = {0};
#pragma unroll 2
    for (int p = lane; p < R / 2; p += 32) {
      const double2 x = *reinterpret_cast<const double2*>(zt + 2 * p);
      const double2 y = *reinterpret_cast<const double2*>(wt + 2 * p);
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(colp<L>(M, ld, ntile, t, g * CG + c)) + p);
        a[c] += v.x * x.x + v.y * x.y;
        b[c] += v.x * y.x + v.y * y.y;
      }
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) tot += warp_sum(a[c]) + warp_sum(b[c]);
  }
  if (lane == 0) out[blockIdx.x * 8 + wid] = tot;
}
template <int L>
__global__ void __launch_bounds__(256) wu(const double* __restrict__ M, long long n, long long ld, long long ntile,
                                          int J, double* out) {
  __shared__ double cp[4096];
  for (int k = threadIdx.x; k < J; k += 256) cp[k] = 1e-3 * k;
  __syncthreads();
  // block covers R rows = 256 threads x 8 rows
  const long long t = blockIdx.x;
  double acc[8] = {0};
#pragma unroll 4
  for (int k = 0; k < J; ++k) {
    const double* col = colp<L>(M, ld, ntile, t, k) + threadIdx.x;
    const double ck = cp[k];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] += col[q * 256] * ck;
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += acc[q];
  out[t * 256 + threadIdx.x] = s;
}
int main() {
  const long long n = 811200, ntile = (n + R - 1) / R, ld = ntile * R;
  const int J = 600;
  double *M, *z, *out;
  cudaMalloc(&M, sizeof(double) * ld * J);
  cudaMalloc(&z, sizeof(double) * ld);
  cudaMalloc(&out, sizeof(double) * ld);
  cudaMemset(M, 0, sizeof(double) * ld * J);
  cudaMemset(z, 0, sizeof(double) * ld);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    return 8.0 * ld * J / (best * 1e-3) / 1e9;
  };
  printf("precond-like column-major %.0f GB/s\n", timeit([&] { pre<0><<<(unsigned)ntile, 256>>>(M, n, ld, ntile, J, z, out); }));
  printf("precond-like panels       %.0f GB/s\n", timeit([&] { pre<1><<<(unsigned)ntile, 256>>>(M, n, ld, ntile, J, z, out); }));
  printf("wupdate-like column-major %.0f GB/s\n", timeit([&] { wu<0><<<(unsigned)ntile, 256>>>(M, n, ld, ntile, J, out); }));
  printf("wupdate-like panels       %.0f GB/s\n", timeit([&] { wu<1><<<(unsigned)ntile, 256>>>(M, n, ld, ntile, J, out); }));
  return 0;
}
