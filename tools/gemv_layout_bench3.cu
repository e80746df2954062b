// GEMV-T (precond reorth) access-pattern microbenchmark, column-major history,
// n = 811200, J = 600, tile R = 2816 rows per CTA, CG = 8 columns, 2 vectors:
//  cur : warp w owns column groups w, w+8, ...; walks the whole tile (64 short runs / CTA)
//  blk : all 8 warps on the same column group; warp w covers rows [w R/8, (w+1) R/8)
//  ilv : all 8 warps on the same column group; 16-byte chunks interleaved over warps
//  wu  : thread-per-row W c GEMV (wupdate pattern) for reference
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/glb3 tools/gemv_layout_bench3.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 2816, CG = 8;
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 ld_l2_256(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// MODE 3: cur + L2::256B fetch hint; MODE 4/5: cur + bulk L2 prefetch PF steps ahead
template <int MODE, int PF = 4, int WIN = 4>
__global__ void __launch_bounds__(256) pre(const double* __restrict__ M, long long ld, int J,
                                           const double* __restrict__ z, double* out) {
  __shared__ double zt[R], wt[R];
  const long long t = blockIdx.x, r0 = t * R;
  for (int i = threadIdx.x; i < R; i += 256) {
    zt[i] = z[r0 + i];
    wt[i] = z[r0 + i] * 0.5;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double tot = 0.0;
  const int g0 = (MODE == 0 || MODE >= 3) ? wid : 0, gs = (MODE == 0 || MODE >= 3) ? 8 : 1;
  for (int g = g0; g * CG < J; g += gs) {
    double a[CG] = {0}, b[CG] = {0};
    int p0, pstep, pend;
    if (MODE == 0 || MODE >= 3) {
      p0 = lane;
      pstep = 32;
      pend = R / 2;
    } else if (MODE == 1) {
      p0 = wid * (R / 16) + lane;
      pstep = 32;
      pend = (wid + 1) * (R / 16);
    } else {
      p0 = threadIdx.x;
      pstep = 256;
      pend = R / 2;
    }
    if (MODE >= 4 && lane < CG) {  // prime: first PF steps of each column
      const double* cp0 = M + (long long)(g * CG + lane) * ld + r0;
      bulk_prefetch_l2(cp0, 512u * PF);
    }
#pragma unroll 2
    for (int p = p0; p < pend; p += pstep) {
      if (MODE >= 4 && lane < CG && ((p - lane) & (32 * WIN - 1)) == 0) {
        // every WIN steps: prefetch the WIN steps (WIN x 512 B) that lie PF steps ahead
        const long long ahead = (long long)(p - lane) + 32 * PF;
        if (ahead < pend) {
          const unsigned bytes = (unsigned)min(512LL * WIN, 16LL * (pend - ahead));
          bulk_prefetch_l2(M + (long long)(g * CG + lane) * ld + r0 + 2 * ahead, bytes);
        }
      }
      const double2 x = *reinterpret_cast<const double2*>(zt + 2 * p);
      const double2 y = *reinterpret_cast<const double2*>(wt + 2 * p);
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        const double2* src = reinterpret_cast<const double2*>(M + (long long)(g * CG + c) * ld + r0) + p;
        const double2 v = MODE == 3 ? ld_l2_256(src) : __ldcs(src);
        a[c] += v.x * x.x + v.y * x.y;
        b[c] += v.x * y.x + v.y * y.y;
      }
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) tot += warp_sum(a[c]) + warp_sum(b[c]);
  }
  if (lane == 0) out[blockIdx.x * 8 + wid] = tot;
}
template <int RPT, int UNR>
__global__ void __launch_bounds__(256) wu(const double* __restrict__ M, long long ld, int J, double* out) {
  __shared__ double cp[4096];
  for (int k = threadIdx.x; k < J; k += 256) cp[k] = 1e-3 * k;
  __syncthreads();
  const long long r0 = (long long)blockIdx.x * 256 * RPT;
  double acc[RPT] = {0};
#pragma unroll UNR
  for (int k = 0; k < J; ++k) {
    const double* col = M + (long long)k * ld + r0 + threadIdx.x;
    const double ck = cp[k];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] += col[q * 256] * ck;
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < RPT; ++q) s += acc[q];
  out[r0 + threadIdx.x] = s;
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
    for (int rep = 0; rep < 8; ++rep) {
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
  printf("copy  %.0f GB/s (read+write)\n", 2.0 * 8.0 * ld * J / 2 / (best * 1e-3) / 1e9);
  printf("cur   %.0f GB/s\n", timeit([&] { pre<0><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
  printf("blk   %.0f GB/s\n", timeit([&] { pre<1><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
  printf("ilv   %.0f GB/s\n", timeit([&] { pre<2><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
  printf("l2hint %.0f GB/s\n", timeit([&] { pre<3><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
#define PFV(PF, WIN) printf("pf dist=%2d win=%d  %.0f GB/s\n", PF, WIN, \
    timeit([&] { pre<4, PF, WIN><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
  printf("cur   %.0f GB/s\n", timeit([&] { pre<0><<<(unsigned)ntile, 256>>>(M, ld, J, z, out); }));
  PFV(1, 2) PFV(1, 4) PFV(2, 2) PFV(2, 4) PFV(2, 8) PFV(1, 8) PFV(3, 8) PFV(2, 2) PFV(2, 4)
#define WU(RPT, UNR) printf("wu rpt=%2d unroll=%d  %.0f GB/s\n", RPT, UNR, \
    timeit([&] { wu<RPT, UNR><<<(unsigned)(ld / (256 * RPT)), 256>>>(M, ld, J, out); }));
  WU(4, 4) WU(4, 8) WU(8, 2) WU(8, 4) WU(16, 1) WU(16, 2) WU(11, 4)
  return 0;
}
