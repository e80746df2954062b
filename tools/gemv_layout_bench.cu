// Microbenchmark: does the reorth GEMV-T lose bandwidth to DRAM page locality?
// Compares AW^T [z w] over an n x J fp64 history stored (a) column-major
// (current) and (b) row-tiled ("panels": rows of one tile of all columns are
// contiguous).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// /tmp/glb tools/gemv_layout_bench.cu ; run on a B200.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 2816;    // rows per tile (= precond tile at config 2)
constexpr int CG = 8;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// layout 0: column k at base + k*ld; layout 1: tile t, column k at base + (t*J + k)*R
template <int LAYOUT>
__global__ void __launch_bounds__(256) gemvt(const double* __restrict__ M, long long n, long long ld, int J,
                                             const double* __restrict__ z, double* out) {
  __shared__ double zt[R];
  const long long t = blockIdx.x, r0 = t * R;
  const int len = (int)min((long long)R, n - r0);
  for (int i = threadIdx.x; i < len; i += 256) zt[i] = z[r0 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double tot = 0.0;
  for (int g = wid; g * CG < J; g += 8) {
    double a[CG] = {0};
    for (int p = lane; p < len / 2; p += 32) {
      const double2 x = *reinterpret_cast<const double2*>(zt + 2 * p);
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        const int k = g * CG + c;
        const double* col = LAYOUT == 0 ? M + k * ld + r0 : M + (t * J + k) * (long long)R;
        const double2 v = __ldcs(reinterpret_cast<const double2*>(col) + p);
        a[c] += v.x * x.x + v.y * x.y;
      }
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) tot += warp_sum(a[c]);
  }
  if (lane == 0) out[blockIdx.x * 8 + wid] = tot;
}

int main() {
  const long long n = 811200;
  const long long ntile = (n + R - 1) / R;
  const long long ld = ntile * R;
  const int J = 600;
  double *M, *z, *out;
  cudaMalloc(&M, sizeof(double) * ld * J);
  cudaMalloc(&z, sizeof(double) * ld);
  cudaMalloc(&out, sizeof(double) * ntile * 8);
  cudaMemset(M, 0, sizeof(double) * ld * J);
  cudaMemset(z, 0, sizeof(double) * ld);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int layout = 0; layout < 2; ++layout) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (layout == 0) gemvt<0><<<(unsigned)ntile, 256>>>(M, n, ld, J, z, out);
      else gemvt<1><<<(unsigned)ntile, 256>>>(M, n, ld, J, z, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    const double bytes = 8.0 * n * J;
    printf("layout %s: %.1f us  %.0f GB/s\n", layout ? "row-tiled panels" : "column-major", best * 1e3,
           bytes / (best * 1e-3) / 1e9);
  }
  // sequential copy reference
  double* M2;
  cudaMalloc(&M2, sizeof(double) * ld * J / 2);
  float best = 1e9;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(M2, M, sizeof(double) * ld * J / 2, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  printf("cudaMemcpy D2D: %.0f GB/s (read+write)\n", 2.0 * 8.0 * ld * J / 2 / (best * 1e-3) / 1e9);
  return 0;
}
