// K3 reorth GEMV-T (out[k] = AW[:,k]^T z, AW[:,k]^T w for k < J) access-pattern
// microbenchmark at BASELINE config-3 size (n = 2,709,792, J = 1000 columns of
// a column-major history, 21.7 GB), against the K5 (W c, GEMV-N) pattern.
//   cur  : production K3 - warp w owns column groups w, w+8, ... of CG=8 and walks
//          the CTA's whole row tile (2 tiles per SM)
//   blk  : all 8 warps on one column group; warp w covers rows [w R/8, (w+1) R/8)
//   trow : K5-like - thread owns RPT rows (stride 256) of a 256*RPT row block,
//          the CTA sweeps CG-column chunks; per chunk the 2*CG partials are
//          warp-reduced (shuffles) and written as per-warp partial rows
//   wu   : the K5 GEMV-N pattern (upper bound for the same bytes)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k3lb tools/k3_layout_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int CG, int MODE>
__global__ void __launch_bounds__(256, 2) pre(const double* __restrict__ M, long long ld, long long n, int J, int R,
                                              const double* __restrict__ z, const double* __restrict__ w,
                                              double* __restrict__ out) {
  extern __shared__ double sm[];
  double* zt = sm;
  double* wt = sm + R;
  const long long r0 = (long long)blockIdx.x * R;
  const int len = (int)min((long long)R, n - r0);
  for (int i = threadIdx.x; i < len; i += 256) {
    zt[i] = z[r0 + i];
    wt[i] = w[r0 + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pairs = len >> 1;
  const int ng = (J + CG - 1) / CG;
  const int g0 = MODE == 0 ? wid : 0, gs = MODE == 0 ? 8 : 1;
  int p0 = lane, pend = pairs;
  if (MODE == 1) {
    const int per = (pairs + 7) / 8;
    p0 = wid * per + lane;
    pend = min(pairs, (wid + 1) * per);
  }
  for (int g = g0; g < ng; g += gs) {
    double a[CG], b[CG];
#pragma unroll
    for (int c = 0; c < CG; ++c) a[c] = b[c] = 0.0;
    const double* cols = M + (long long)g * CG * ld + r0;
#pragma unroll 2
    for (int p = p0; p < pend; p += 32) {
      const double2 x = reinterpret_cast<const double2*>(zt)[p];
      const double2 y = reinterpret_cast<const double2*>(wt)[p];
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + p);
        a[c] += v.x * x.x + v.y * x.y;
        b[c] += v.x * y.x + v.y * y.y;
      }
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) {
      a[c] = warp_sum(a[c]);
      b[c] = warp_sum(b[c]);
    }
    if (lane == 0) {
      double* o = out + ((size_t)blockIdx.x * 8 + (MODE == 1 ? wid : 0)) * 2 * J + 2 * g * CG;
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        o[2 * c] = a[c];
        o[2 * c + 1] = b[c];
      }
    }
  }
}

// thread-rows: block of 256*RPT rows; z/w of the thread's rows in registers
template <int RPT, int CG, int MINB>
__global__ void __launch_bounds__(256, MINB) trow(const double* __restrict__ M, long long ld, long long n, int J,
                                                  const double* __restrict__ z, const double* __restrict__ w,
                                                  double* __restrict__ out) {
  const long long r0 = (long long)blockIdx.x * 256 * RPT + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double zr[RPT], wr[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const long long i = r0 + q * 256;
    zr[q] = i < n ? z[i] : 0.0;
    wr[q] = i < n ? w[i] : 0.0;
  }
  double* o = out + ((size_t)blockIdx.x * 8 + wid) * 2 * J;
  for (int k0 = 0; k0 < J; k0 += CG) {
    double a[CG], b[CG];
#pragma unroll
    for (int c = 0; c < CG; ++c) {
      const double* col = M + (long long)(k0 + c) * ld + r0;
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const double v = __ldcs(col + q * 256);
        sa += v * zr[q];
        sb += v * wr[q];
      }
      a[c] = sa;
      b[c] = sb;
    }
    // 2*CG warp sums: butterfly over the pairs (lane-parallel transpose)
#pragma unroll
    for (int c = 0; c < CG; ++c) {
      a[c] = warp_sum(a[c]);
      b[c] = warp_sum(b[c]);
    }
    if (lane < 2 * CG) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        if (lane == 2 * c) v = a[c];
        if (lane == 2 * c + 1) v = b[c];
      }
      o[2 * k0 + lane] = v;
    }
  }
}

template <int RPT, int UNR>
__global__ void __launch_bounds__(256) wu(const double* __restrict__ M, long long ld, long long n, int J,
                                          double* out) {
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
    for (int q = 0; q < RPT; ++q) acc[q] += __ldcs(col + q * 256) * ck;
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < RPT; ++q) s += acc[q];
  if (r0 + threadIdx.x < n) out[r0 + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 2709792;
  const int J = argc > 2 ? atoi(argv[2]) : 1000;
  const long long ld = (n + 31) / 32 * 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *M, *z, *w, *out;
  if (cudaMalloc(&M, sizeof(double) * ld * (J + 16)) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMalloc(&z, sizeof(double) * ld);
  cudaMalloc(&w, sizeof(double) * ld);
  const size_t outsz = sizeof(double) * (size_t)(n / 256 + 64) * 8 * 2 * (J + 16);
  cudaMalloc(&out, outsz);
  cudaMemset(M, 0, sizeof(double) * ld * J);
  cudaMemset(z, 0, sizeof(double) * ld);
  cudaMemset(w, 0, sizeof(double) * ld);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 8.0 * n * J;
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
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
    return bytes / (best * 1e-3) / 1e9;
  };
  printf("n=%lld J=%d  %.1f GB per pass\n", n, J, bytes / 1e9);
  for (int tps : {2, 3, 4}) {
    const int R = (int)(((n + (long long)tps * sms - 1) / ((long long)tps * sms) + 63) / 64 * 64);
    const int nt = (int)((n + R - 1) / R);
    const size_t smem = sizeof(double) * 2 * R;
    cudaFuncSetAttribute(pre<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem > 227 * 1024) continue;
    printf("tiles/SM=%d R=%d: cur %.0f  blk %.0f  blk4 %.0f GB/s\n", tps, R,
           timeit([&] { pre<8, 0><<<nt, 256, smem>>>(M, ld, n, J, R, z, w, out); }),
           timeit([&] { pre<8, 1><<<nt, 256, smem>>>(M, ld, n, J, R, z, w, out); }),
           timeit([&] { pre<4, 1><<<nt, 256, smem>>>(M, ld, n, J, R, z, w, out); }));
  }
#define TROW(RPT, CG, MINB)                                                                                  \
  printf("trow rpt=%2d cg=%d minb=%d  %.0f GB/s\n", RPT, CG, MINB, timeit([&] {                             \
           trow<RPT, CG, MINB><<<(unsigned)((n + 256 * RPT - 1) / (256 * RPT)), 256>>>(M, ld, n, J, z, w, out); \
         }));
  TROW(4, 8, 2) TROW(4, 8, 3) TROW(4, 8, 4) TROW(8, 4, 2) TROW(8, 4, 3) TROW(8, 8, 2) TROW(2, 8, 4) TROW(2, 16, 2)
  TROW(4, 4, 4) TROW(16, 2, 2)
#define WU(RPT, UNR) printf("wu rpt=%2d unroll=%d  %.0f GB/s\n", RPT, UNR, \
    timeit([&] { wu<RPT, UNR><<<(unsigned)((n + 256 * RPT - 1) / (256 * RPT)), 256>>>(M, ld, n, J, out); }));
  WU(8, 4) WU(4, 4) WU(8, 2)
  return 0;
}
