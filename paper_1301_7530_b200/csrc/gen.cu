// Device-side assembly of the BASELINE operators:
// the structured finite-difference diffusion operator (reference
// `_assemble_diffusion`, /root/reference/pkg/src/recycg/problems.py:115-156)
// and the Q1 hex elasticity operator (new; host twin
// paper_1301_7530_b200/problems.py:elasticity_q1).  At 12-17 M rows the host
// assemblers spend minutes and tens of GB of host RAM on numpy temporaries;
// here only the random coefficient field crosses PCIe and the CSR is written
// straight into HBM.
//
// Both assemblers reproduce the host bytes exactly: every value is formed
// with the same operations in the same order as the numpy code (explicit
// __dmul_rn / __ddiv_rn / __dadd_rn, no FMA contraction), entries are
// emitted in ascending column order, and the explicit zeros of the host
// pattern are kept.  tests/test_gpu_generators.py checks bitwise equality.
//
// Two passes: per-row entry counts -> in-place inclusive scan (tiles of 4096
// rows, a single-CTA scan of the tile sums, then the tile-local scans) ->
// fill, each row writing from its offset.
#include "rcg_internal.cuh"

namespace rcg {

namespace {

constexpr int SCAN_TILE = 4096;   // rows per scan tile (256 threads x 16)

// ---- diffusion ------------------------------------------------------------
// cells are row-major over (g0, g1, g2) (1-D/2-D grids use leading 1s); only
// axes with g >= 2 couple (problems.py:131-133).

struct Grid3 {
  int64_t g[3];
  int64_t s[3];   // strides
};

__device__ __forceinline__ void cell_coords(const Grid3& G, int64_t i, int64_t c[3]) {
  c[2] = i % G.g[2];
  const int64_t t = i / G.g[2];
  c[1] = t % G.g[1];
  c[0] = t / G.g[1];
}

__global__ void diff_count_kernel(Grid3 G, int64_t n, int64_t* __restrict__ ro) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    cell_coords(G, i, c);
    int64_t k = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (G.g[a] >= 2) k += (c[a] > 0) + (c[a] < G.g[a] - 1);
    ro[i + 1] = k;
    if (i == 0) ro[0] = 0;
  }
}

// 2 c_lo c_hi / (c_lo + c_hi), evaluated left to right like numpy
__device__ __forceinline__ double face_weight(double lo, double hi) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, lo), hi), __dadd_rn(lo, hi));
}

__global__ void diff_fill_kernel(Grid3 G, int64_t n, const double* __restrict__ coeff,
                                 const int64_t* __restrict__ ro, int32_t* __restrict__ ro32,
                                 int32_t* __restrict__ ci, double* __restrict__ va) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    cell_coords(G, i, c);
    const double ci_ = coeff[i];
    double lo_w[3] = {0.0, 0.0, 0.0}, hi_w[3] = {0.0, 0.0, 0.0};
    // diagonal: per axis, face to +s, face to -s, then the Dirichlet ends
    // (problems.py:140-151 order)
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (G.g[a] < 2) continue;
      if (c[a] < G.g[a] - 1) {
        hi_w[a] = face_weight(ci_, coeff[i + G.s[a]]);
        d = __dadd_rn(d, hi_w[a]);
      }
      if (c[a] > 0) {
        lo_w[a] = face_weight(coeff[i - G.s[a]], ci_);
        d = __dadd_rn(d, lo_w[a]);
      }
      if (c[a] == 0) d = __dadd_rn(d, ci_);
      if (c[a] == G.g[a] - 1) d = __dadd_rn(d, ci_);
    }
    int64_t p = ro[i];
    if (ro32) ro32[i + 1] = (int32_t)ro[i + 1];
    if (ro32 && i == 0) ro32[0] = 0;
    // ascending columns: -s0, -s1, -s2, centre, +s2, +s1, +s0
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (G.g[a] >= 2 && c[a] > 0) {
        ci[p] = (int32_t)(i - G.s[a]);
        va[p++] = -lo_w[a];
      }
    ci[p] = (int32_t)i;
    va[p++] = d;
#pragma unroll
    for (int a = 2; a >= 0; --a)
      if (G.g[a] >= 2 && c[a] < G.g[a] - 1) {
        ci[p] = (int32_t)(i + G.s[a]);
        va[p++] = -hi_w[a];
      }
  }
}

// ---- Q1 elasticity -------------------------------------------------------------
// free nodes (gx, gy, gz) on NX x NY x NZ = N x (N+1) x (N+1), gx = ix - 1;
// node id (gx NY + gy) NZ + gz; dof 3 id + comp.  Neighbour slot
// s = 9 (dx+1) + 3 (dy+1) + (dz+1).  Local corner (a, b, c) has index
// 4a + 2b + c.

struct Q1Grid {
  int64_t N, NX, NY, NZ;
};

__device__ __forceinline__ unsigned q1_slot_mask(const Q1Grid& G, int64_t p, int64_t& gx, int64_t& gy, int64_t& gz) {
  gz = p % G.NZ;
  const int64_t t = p / G.NZ;
  gy = t % G.NY;
  gx = t / G.NY;
  unsigned m = 0;
  for (int s = 0; s < 27; ++s) {
    const int64_t qx = gx + s / 9 - 1, qy = gy + (s / 3) % 3 - 1, qz = gz + s % 3 - 1;
    if (qx >= 0 && qx < G.NX && qy >= 0 && qy < G.NY && qz >= 0 && qz < G.NZ) m |= 1u << s;
  }
  return m;
}

__global__ void q1_count_kernel(Q1Grid G, int64_t nn, int64_t* __restrict__ ro) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nn; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t gx, gy, gz;
    const int64_t k = 3 * __popc(q1_slot_mask(G, p, gx, gy, gz));
    ro[3 * p + 1] = k;
    ro[3 * p + 2] = k;
    ro[3 * p + 3] = k;
    if (p == 0) ro[0] = 0;
  }
}

// Warp per free node: the node's three rows share one column pattern; lane
// t covers entries t, t + 32, t + 64 of each row (coalesced stores).  Entry
// value (i, slot, jj) = sum over the node's local corners lp in DEcreasing
// order of E_e * Ke[3 ip + i, 3 iq + jj], e = p - lp, lq = lp + d(slot): the
// element order of problems.py:elasticity_q1 (so (p,q) and (q,p) match too).
__global__ void __launch_bounds__(256) q1_fill_kernel(Q1Grid G, int64_t nn, const double* __restrict__ Ke,
                                                      const double* __restrict__ E,
                                                      const int64_t* __restrict__ ro,
                                                      int32_t* __restrict__ ro32, int32_t* __restrict__ ci,
                                                      double* __restrict__ va) {
  __shared__ double ke[576];
  for (int t = threadIdx.x; t < 576; t += blockDim.x) ke[t] = Ke[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < nn; p += nw) {
    int64_t gx, gy, gz;
    const unsigned mask = q1_slot_mask(G, p, gx, gy, gz);
    const int nv = __popc(mask);
    const int64_t ix = gx + 1, iy = gy, iz = gz;
    if (ro32 && lane < 3) ro32[3 * p + lane + 1] = (int32_t)ro[3 * p + lane + 1];
    if (ro32 && p == 0 && lane == 0) ro32[0] = 0;
    for (int t = lane; t < 3 * nv; t += 32) {
      const int k = t / 3, jj = t % 3;
      // k-th set bit of mask
      unsigned m = mask;
      for (int u = 0; u < k; ++u) m &= m - 1;
      const int s = __ffs(m) - 1;
      const int dx = s / 9 - 1, dy = (s / 3) % 3 - 1, dz = s % 3 - 1;
      const int64_t q = ((gx + dx) * G.NY + (gy + dy)) * G.NZ + (gz + dz);
      double acc[3] = {0.0, 0.0, 0.0};
      for (int lp = 7; lp >= 0; --lp) {
        const int a = lp >> 2, b = (lp >> 1) & 1, c = lp & 1;
        const int qa = a + dx, qb = b + dy, qc = c + dz;
        if (qa < 0 || qa > 1 || qb < 0 || qb > 1 || qc < 0 || qc > 1) continue;
        const int64_t ex = ix - a, ey = iy - b, ez = iz - c;
        if (ex < 0 || ex >= G.N || ey < 0 || ey >= G.N || ez < 0 || ez >= G.N) continue;
        const double Ee = E ? E[(ex * G.N + ey) * G.N + ez] : 1.0;
        const int iq = 4 * qa + 2 * qb + qc;
#pragma unroll
        for (int i = 0; i < 3; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(Ee, ke[(3 * lp + i) * 24 + 3 * iq + jj]));
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int64_t o = ro[3 * p + i] + t;
        ci[o] = (int32_t)(3 * q + jj);
        va[o] = acc[i];
      }
    }
  }
}

// ---- in-place inclusive scan of ro[1..n] (int64) -------------------------------

__global__ void __launch_bounds__(256) scan_tile_sums_kernel(const int64_t* __restrict__ v, int64_t n,
                                                             int64_t* __restrict__ sums) {
  __shared__ int64_t sm[8];
  const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
  for (int64_t i = t0 + threadIdx.x; i < min(n, t0 + SCAN_TILE); i += blockDim.x) s += v[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < 8; ++w) t += sm[w];
    sums[blockIdx.x] = t;
  }
}

// exclusive scan of the tile sums by one CTA (chunks of 1024 sequentially)
__global__ void __launch_bounds__(1024) scan_sums_kernel(int64_t* sums, int64_t ntiles, int64_t* total) {
  __shared__ int64_t sm[1024];
  int64_t carry = 0;
  for (int64_t b = 0; b < ntiles; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const int64_t v = i < ntiles ? sums[i] : 0;
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t u = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
      __syncthreads();
      sm[threadIdx.x] += u;
      __syncthreads();
    }
    if (i < ntiles) sums[i] = carry + sm[threadIdx.x] - v;
    const int64_t last = sm[1023];
    __syncthreads();
    carry += last;
  }
  if (threadIdx.x == 0) *total = carry;
}

// tile-local inclusive scan (16 consecutive values per thread) + tile offset
__global__ void __launch_bounds__(256) scan_apply_kernel(int64_t* __restrict__ v, int64_t n,
                                                         const int64_t* __restrict__ offs) {
  __shared__ int64_t sm[256];
  const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE + 16 * threadIdx.x;
  int64_t loc[16];
  int64_t s = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    loc[u] = t0 + u < n ? v[t0 + u] : 0;
    s += loc[u];
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int64_t w = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
    __syncthreads();
    sm[threadIdx.x] += w;
    __syncthreads();
  }
  int64_t run = offs[blockIdx.x] + sm[threadIdx.x] - s;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    run += loc[u];
    if (t0 + u < n) v[t0 + u] = run;
  }
}

int inclusive_scan(Ctx* c, int64_t* v, int64_t n, int64_t* total_host) {
  const int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  int64_t* sums = nullptr;
  int rc = scratch(c, (size_t)(ntiles + 1) * sizeof(int64_t) + 256, (void**)&sums);
  if (rc) return rc;
  if (ntiles > 0) {
    scan_tile_sums_kernel<<<(unsigned)ntiles, 256, 0, c->stream>>>(v, n, sums);
    RCG_LAUNCH_CHECK(c);
  }
  scan_sums_kernel<<<1, 1024, 0, c->stream>>>(sums, ntiles, sums + ntiles);
  RCG_LAUNCH_CHECK(c);
  if (ntiles > 0) {
    scan_apply_kernel<<<(unsigned)ntiles, 256, 0, c->stream>>>(v, n, sums);
    RCG_LAUNCH_CHECK(c);
  }
  RCG_CUDA(c, cudaMemcpyAsync(total_host, sums + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));
  return RCG_OK;
}

int gen_grid(Ctx* c, int64_t items) {
  int64_t g = (items + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)c->num_sms * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

bool diff_grid(const int64_t* dims, int ndim, Grid3& G, int64_t& n) {
  if (ndim < 1 || ndim > 3) return false;
  G.g[0] = G.g[1] = G.g[2] = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return false;
    G.g[3 - ndim + a] = dims[a];
  }
  G.s[2] = 1;
  G.s[1] = G.g[2];
  G.s[0] = G.g[1] * G.g[2];
  n = G.g[0] * G.s[0];
  return n < ((int64_t)1 << 31) - 1;
}

bool q1_grid(int64_t N, Q1Grid& G, int64_t& nn) {
  if (N < 1) return false;
  G.N = N;
  G.NX = N;
  G.NY = G.NZ = N + 1;
  nn = G.NX * G.NY * G.NZ;
  return 3 * nn < ((int64_t)1 << 31) - 1;
}

}  // namespace

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_gen_diffusion_rows(rcg_ctx* ctx, const int64_t* dims, int32_t ndim, int64_t* ro64,
                                      int64_t* nnz_host) {
  if (!ctx || !dims || !ro64 || !nnz_host) return RCG_ERR_CONTRACT;
  Grid3 G;
  int64_t n;
  if (!diff_grid(dims, ndim, G, n)) return set_error(ctx, RCG_ERR_CONTRACT, "rcg_gen_diffusion_rows: bad grid");
  diff_count_kernel<<<gen_grid(ctx, n), kThreads, 0, ctx->stream>>>(G, n, ro64);
  RCG_LAUNCH_CHECK(ctx);
  return inclusive_scan(ctx, ro64 + 1, n, nnz_host);
}

extern "C" int rcg_gen_diffusion_fill(rcg_ctx* ctx, const int64_t* dims, int32_t ndim, const double* coeff,
                                      const int64_t* ro64, int32_t* ro32, int32_t* ci, double* va) {
  if (!ctx || !dims || !coeff || !ro64 || !ci || !va) return RCG_ERR_CONTRACT;
  Grid3 G;
  int64_t n;
  if (!diff_grid(dims, ndim, G, n)) return set_error(ctx, RCG_ERR_CONTRACT, "rcg_gen_diffusion_fill: bad grid");
  diff_fill_kernel<<<gen_grid(ctx, n), kThreads, 0, ctx->stream>>>(G, n, coeff, ro64, ro32, ci, va);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}

extern "C" int rcg_gen_elasticity_rows(rcg_ctx* ctx, int64_t nelem, int64_t* ro64, int64_t* nnz_host) {
  if (!ctx || !ro64 || !nnz_host) return RCG_ERR_CONTRACT;
  Q1Grid G;
  int64_t nn;
  if (!q1_grid(nelem, G, nn)) return set_error(ctx, RCG_ERR_CONTRACT, "rcg_gen_elasticity_rows: bad nelem");
  q1_count_kernel<<<gen_grid(ctx, nn), kThreads, 0, ctx->stream>>>(G, nn, ro64);
  RCG_LAUNCH_CHECK(ctx);
  return inclusive_scan(ctx, ro64 + 1, 3 * nn, nnz_host);
}

extern "C" int rcg_gen_elasticity_fill(rcg_ctx* ctx, int64_t nelem, const double* Ke, const double* E,
                                       const int64_t* ro64, int32_t* ro32, int32_t* ci, double* va) {
  if (!ctx || !Ke || !ro64 || !ci || !va) return RCG_ERR_CONTRACT;
  Q1Grid G;
  int64_t nn;
  if (!q1_grid(nelem, G, nn)) return set_error(ctx, RCG_ERR_CONTRACT, "rcg_gen_elasticity_fill: bad nelem");
  const int64_t warps = nn;
  int64_t g = (warps + 7) / 8;
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  g = g < 1 ? 1 : (g > cap ? cap : g);
  q1_fill_kernel<<<(unsigned)g, 256, 0, ctx->stream>>>(G, nn, Ke, E, ro64, ro32, ci, va);
  RCG_LAUNCH_CHECK(ctx);
  return RCG_OK;
}
