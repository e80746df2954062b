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
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k3lb tools/k3_layout_bench.cu -lcuda
// Run:   tools/k3lb [n] [J] [vmm chunk MB, 0 = cudaMalloc]
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

// the production histories' allocation: one VA range, physical chunks of
// `chunk` bytes mapped behind it (csrc/vmm.cu)
static double* vmm_alloc(size_t bytes, size_t chunk) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  size_t g = 0;
  cuMemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  chunk = (chunk + g - 1) / g * g;
  const size_t total = (bytes + chunk - 1) / chunk * chunk;
  CUdeviceptr base = 0;
  if (cuMemAddressReserve(&base, total, 0, 0, 0) != CUDA_SUCCESS) return nullptr;
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t off = 0; off < total; off += chunk) {
    CUmemGenericAllocationHandle h;
    if (cuMemCreate(&h, chunk, &prop, 0) != CUDA_SUCCESS) return nullptr;
    cuMemMap(base + off, chunk, 0, h, 0);
    cuMemSetAccess(base + off, chunk, &acc, 1);
  }
  printf("vmm: %.1f GB in chunks of %zu MB (granularity %zu KB)\n", total / 1e9, chunk >> 20, g >> 10);
  return (double*)base;
}

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
  const int g0 = MODE != 1 ? wid : 0, gs = MODE != 1 ? 8 : 1;
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
    if (MODE == 2) {
      // explicit batch: the CG loads of two consecutive steps, then the FMAs
      int p = p0;
      for (; p + 32 < pend; p += 64) {
        double2 v0[CG], v1[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) v0[c] = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + p);
#pragma unroll
        for (int c = 0; c < CG; ++c) v1[c] = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + p + 32);
        const double2 x0 = reinterpret_cast<const double2*>(zt)[p];
        const double2 y0 = reinterpret_cast<const double2*>(wt)[p];
        const double2 x1 = reinterpret_cast<const double2*>(zt)[p + 32];
        const double2 y1 = reinterpret_cast<const double2*>(wt)[p + 32];
#pragma unroll
        for (int c = 0; c < CG; ++c) {
          a[c] += v0[c].x * x0.x + v0[c].y * x0.y;
          b[c] += v0[c].x * y0.x + v0[c].y * y0.y;
          a[c] += v1[c].x * x1.x + v1[c].y * x1.y;
          b[c] += v1[c].x * y1.x + v1[c].y * y1.y;
        }
      }
      for (; p < pend; p += 32) {
        const double2 x = reinterpret_cast<const double2*>(zt)[p];
        const double2 y = reinterpret_cast<const double2*>(wt)[p];
#pragma unroll
        for (int c = 0; c < CG; ++c) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + p);
          a[c] += v.x * x.x + v.y * x.y;
          b[c] += v.x * y.x + v.y * y.y;
        }
      }
    } else
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

// K5 variants at the production occupancy (3 CTAs/SM): 64-bit loads (as
// production), 128-bit row pairs, and 128-bit with an explicit 4-column batch
template <int RPT, int UNR>
__global__ void __launch_bounds__(256, 3) wu3(const double* __restrict__ M, long long ld, long long n, int J,
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
template <int PPT, int KB>
__global__ void __launch_bounds__(256, 3) wu128(const double* __restrict__ M, long long ld, long long n, int J,
                                                double* out) {
  __shared__ double cp[4096];
  for (int k = threadIdx.x; k < J; k += 256) cp[k] = 1e-3 * k;
  __syncthreads();
  // thread owns row pairs p0 + q*256, q < PPT (2*PPT rows)
  const long long p0 = (long long)blockIdx.x * 256 * PPT + threadIdx.x;
  double2 acc[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) acc[q] = make_double2(0.0, 0.0);
  int k = 0;
  for (; k + KB <= J; k += KB) {
    double2 v[KB][PPT];
#pragma unroll
    for (int u = 0; u < KB; ++u)
#pragma unroll
      for (int q = 0; q < PPT; ++q) v[u][q] = __ldcs(reinterpret_cast<const double2*>(M + (long long)(k + u) * ld) + p0 + q * 256);
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      const double ck = cp[k + u];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        acc[q].x = fma(v[u][q].x, ck, acc[q].x);
        acc[q].y = fma(v[u][q].y, ck, acc[q].y);
      }
    }
  }
  for (; k < J; ++k) {
    const double ck = cp[k];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(M + (long long)k * ld) + p0 + q * 256);
      acc[q].x = fma(v.x, ck, acc[q].x);
      acc[q].y = fma(v.y, ck, acc[q].y);
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) s += acc[q].x + acc[q].y;
  if (2 * p0 < n) out[p0] = s;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 2709792;
  const int J = argc > 2 ? atoi(argv[2]) : 1000;
  const long long ld = (n + 31) / 32 * 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *M, *z, *w, *out;
  const long long vmm_chunk = argc > 3 ? atoll(argv[3]) : 0;   // MB; 0: cudaMalloc
  if (vmm_chunk > 0) {
    cuInit(0);
    M = vmm_alloc(sizeof(double) * ld * (J + 16), (size_t)vmm_chunk << 20);
    if (!M) {
      printf("vmm alloc failed\n");
      return 1;
    }
  } else if (cudaMalloc(&M, sizeof(double) * ld * (J + 16)) != cudaSuccess) {
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
  for (int tps : {2, 3, 4, 6, 8, 12, 16}) {
    const int R = (int)(((n + (long long)tps * sms - 1) / ((long long)tps * sms) + 63) / 64 * 64);
    const int nt = (int)((n + R - 1) / R);
    const size_t smem = sizeof(double) * 2 * R;
    cudaFuncSetAttribute(pre<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pre<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem > 227 * 1024) continue;
    printf("tiles/SM=%d R=%d: batch8 %.0f batch4 %.0f\n", tps, R,
           timeit([&] { pre<8, 2><<<nt, 256, smem>>>(M, ld, n, J, R, z, w, out); }),
           timeit([&] { pre<4, 2><<<nt, 256, smem>>>(M, ld, n, J, R, z, w, out); }));
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
#define WU3(RPT, UNR) printf("wu3 rpt=%2d unroll=%d  %.0f GB/s\n", RPT, UNR, \
    timeit([&] { wu3<RPT, UNR><<<(unsigned)((n + 256 * RPT - 1) / (256 * RPT)), 256>>>(M, ld, n, J, out); }));
  WU3(8, 4) WU3(8, 2) WU3(4, 4)
#define WU128(PPT, KB) printf("wu128 pairs/thread=%d kbatch=%d  %.0f GB/s\n", PPT, KB, \
    timeit([&] { wu128<PPT, KB><<<(unsigned)((n / 2 + 256 * PPT - 1) / (256 * PPT)), 256>>>(M, ld, n, J, out); }));
  WU128(4, 2) WU128(4, 4) WU128(2, 4) WU128(2, 8) WU128(8, 2) WU128(4, 3)
  return 0;
}
