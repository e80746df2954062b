// Augmented (deflated) preconditioned CG for sm_100a — the iteration of
// apcg_solve (/root/reference/pkg/src/recycg/solver.py:193-290) as five
// fused, bandwidth-bound fp64 kernels per iteration:
//
//   K1 spmv      Aw_j = A w_j  (written straight into AW[:, j]) + (w_j, Aw_j)     :242-243
//   K2 update    alpha = rz/wAw; x += alpha w; r -= alpha Aw; ||r||^2;
//                AC^T (M^{-1} r) block partials (the projector's GEMV-T)          :246-258, :84-91
//   K3 precond   ||r|| test (device flag); s = G^{-1} AC^T y; z = M^{-1} r - C s
//                (written into Z[:, j+1]); (r, z); reorth partials AW^T z, AW^T w_j  :273-278
//   K4 colreduce fixed-order reduction of the reorth partials (reorth only)
//   K5 wupdate   beta = rz'/rz; w_{j+1} = z + beta w_j - W ((AW^T w)/diag)            :281-287
//
// Every kernel reads the iteration index j and a `done` flag from a device-
// resident SolveState, so iterations are queued in batches with identical
// launch parameters and the host polls convergence once per batch; kernels
// queued past convergence / failure are no-ops.  The stopping iteration is
// therefore exactly the reference's.  Elementwise updates use
// explicitly non-fused multiply/add to match numpy's rounding; every reduction
// is a fixed-order two-stage tree (bitwise reproducible run to run).
#include "rcg_internal.cuh"
#include "spmv.cuh"
#include "dense.cuh"
#include "comm.cuh"
#include "vmm.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <vector>

namespace rcg {

#ifndef RCG_CG_SYNC
#define RCG_CG_SYNC 0
#endif
#ifndef RCG_PRE_MINB
#define RCG_PRE_MINB 2
#endif
#ifndef RCG_GEMV_UNROLL
#define RCG_GEMV_UNROLL 2
#endif
constexpr int kGemvUnroll = RCG_GEMV_UNROLL;
#ifndef RCG_PRE_FENCE
#define RCG_PRE_FENCE 1   // A/B r02m: K3 6.60 -> 6.73 TB/s in-solve (config 3)
#endif
#ifndef RCG_WU_KB
#define RCG_WU_KB 2     // K5 columns per explicit load batch (x RPT/2 128-bit loads)
#endif
// no-reorth K3 (z pass only): CTAs/SM and rows per thread per step.  At the
// former 4 CTAs/SM (64 registers) the body spilled 168 B of stack; 2 CTAs/SM
// with 8 rows (16 loads) in flight per thread has no spills: config 4
// (7-point 256^3) 4,220 -> 4,690 GB/s; 3 CTAs x 4 rows 3,990, 3 x 8 2,530
// (spills), 2 x 4 4,090.  Same rows per thread in the same order: same bits.
#ifndef RCG_PRE_LEAN_MINB
#define RCG_PRE_LEAN_MINB 2
#endif
#ifndef RCG_PRE_ZB_LEAN
#define RCG_PRE_ZB_LEAN 8
#endif
#ifndef RCG_ACTR_PIPE
#define RCG_ACTR_PIPE 1
#endif
constexpr int CP_CHUNK = 4096;   // reorth coefficients staged per smem chunk
constexpr int WU_RPT = 4;        // rows per thread in K5
constexpr int NC_INLINE = 64;    // coarse solve recomputed per CTA up to this n_c

struct IterArgs {
  int64_t n;
  const double* inv_diag;  // nullptr: identity preconditioner
  // deflation
  int64_t n_c;
  const double* C;
  int64_t ldc;
  const double* AC;
  int64_t ldac;
  const double* Ginv;
  double* s_ext;           // coarse solution when n_c > NC_INLINE
  // vectors / histories
  double* x;
  double* r;
  ColSel W, AW, Z, R;      // R.base == nullptr: no r history
  double* waw_diag;
  double* alphas;
  double* betas;
  double* rz_hist;
  double* rnorms;
  // reductions: sums[0] wAw | [1] rr | [2..2+n_c) AC^T y | [rz_off] rz | [rz_off+1+2k] AW_k^T z, [+1] AW_k^T w
  double* sums;
  int64_t rz_off;
  double* part_upd;        // nb x (1 + n_c)
  double* part_z;          // nb
  double* part_reo;        // nb x reo_stride
  int64_t reo_stride;
  unsigned int* counters;  // [0] spmv [1] update [2] precond [3..] misc ([5], [6]: 3x3 DIA tile claims)
  SolveState* st;
  int reorth;
  int rows_per_block;      // K3 row tile
  int s_smem;              // K3 stages the coarse solution s in smem (0: reads s_ext, n_c too large)
  int rows_per_block_upd;  // K2 row tile (smaller: its AC^T y GEMV-T has few columns)
  int rows_per_block_actr; // K2b row tile (long: ~4 CTAs/SM over all column groups)
  int nb_pre;              // K3 row tiles (partial rows in part_reo / part_z)
  int nb_upd;              // K2 row tiles
  int nb_wu;               // K5 row blocks
  double* part_wu;         // K5 column-split partial sums [S][n] (small n)
  SpmvArgs spmv;           // K1 arguments (device-resident, graph-replayable)
};

// Tile GEMV-T: partial dots of `ncols` columns (column k at base + k*ld, the
// tile's first row already applied) with NV smem vectors of length len.
// Work items are (group of CG consecutive columns) x (row slice); when there
// are fewer column groups than warps the rows are split so every warp
// streams.  Lanes read 2 consecutive rows with one 128-bit load per column
// (base, ld and the tile start are 16-B aligned), so a lane keeps CG
// LDG.128 in flight per step and reuses each smem vector element for CG
// columns.  Slice partials are combined in smem in a fixed order.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// With `pf`, lanes 0..CG-1 keep the bulk-copy engine PF_DIST steps (x 512 B)
// ahead of the warp's own loads: every PF_WIN steps each issues one
// cp.async.bulk.prefetch.L2 of PF_WIN x 512 B of its column.  The register-
// limited K3 (2 CTAs/SM) gets HBM requests in flight without holding
// registers: 5.86 -> 6.4 TB/s in tools/gemv_layout_bench3.cu.  In the full
// solve loop of the current build it no longer pays (config 2: K3 6.45 TB/s
// with, 6.56 without, K5 also slightly faster): off unless RCG_PF=1.
constexpr int PF_DIST = 2, PF_WIN = 4;

// GEMV-T of one row tile: out[k*NV + v] = sum_rows M[:, k] v_v for k < ncols.
// Items are (column group, row slice) pairs taken round-robin by the warps;
// the slice count S is uniform per round.  Whole rounds run one group per
// warp (S = 1); the r < kWarps leftover groups then run split kWarps ways
// (one group per round), so no warp idles at the CTA's final barrier through
// a whole extra item (j ~ 600: 75 groups = 9 rounds + 3/8).  With few groups
// (< kWarps) S is the power of two that gives every warp an item.  The S
// slices of a group are consecutive warps of one round and are combined in
// smem in slice order (deterministic).
template <int CG, int NV, bool PF = false>
__device__ __forceinline__ void gemv_t_tile(const double* __restrict__ base, int64_t ld, int64_t ncols, int64_t len,
                                            const double* __restrict__ v0, const double* __restrict__ v1,
                                            double* __restrict__ out, double* __restrict__ red /* smem kWarps*CG*NV */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t ngroups = (ncols + CG - 1) / CG;
  const int64_t pairs = len >> 1;  // full row pairs
  int S0 = 1;
  while (S0 < kWarps && ngroups * S0 < kWarps) S0 *= 2;
  const int64_t main_rounds = ngroups >= kWarps ? ngroups / kWarps : (ngroups * S0 + kWarps - 1) / kWarps;
  const int64_t tail_groups = ngroups >= kWarps ? ngroups - main_rounds * kWarps : 0;
  const int64_t rounds = main_rounds + tail_groups;
  for (int64_t rnd = 0; rnd < rounds; ++rnd) {
    const bool tail = rnd >= main_rounds;
    const int S = tail ? kWarps : S0;
    const int64_t item = tail ? (main_rounds * kWarps + (rnd - main_rounds) * kWarps + wid)
                              : rnd * kWarps + wid;  // tail: group main_groups + (rnd - main_rounds)
    const int64_t nitems = tail ? (main_rounds * kWarps + tail_groups * kWarps) : ngroups * S0;
    const int64_t per = (pairs + S - 1) / S;
    double a0[CG], a1[CG];
#pragma unroll
    for (int c = 0; c < CG; ++c) a0[c] = a1[c] = 0.0;
    int64_t g = -1;
    int sl = 0;
    if (item < nitems) {
      g = tail ? main_rounds * kWarps + (rnd - main_rounds) : item / S;
      sl = tail ? wid : (int)(item % S);
      const int64_t k0 = g * CG;
      const int kc = (int)min((int64_t)CG, ncols - k0);
      const double* __restrict__ cols = base + k0 * ld;
      const int64_t p_begin = sl * per, p_end = min(pairs, p_begin + per);
      if (kc == CG && !PF) {
        // explicit batch: the CG 128-bit loads of two consecutive steps are
        // issued before any FMA (the compiler, at the 128-register budget,
        // otherwise interleaves them with the FMAs and keeps only ~4 loads in
        // flight: tools/k3_layout_bench.cu, 6.96 -> 7.12 TB/s at config 3).
        // Accumulation order per column is unchanged (step p, then p + 32).
        // warp-uniform trip count (the scheduling fence below needs every
        // lane): full double steps while 64 pairs remain, then single steps
        int64_t base = p_begin;
        for (; base + 64 <= p_end; base += 64) {
          const int64_t pi = base + lane;
          double2 va[CG], vb[CG];
#pragma unroll
          for (int c = 0; c < CG; ++c) va[c] = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + pi);
#pragma unroll
          for (int c = 0; c < CG; ++c) vb[c] = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + pi + 32);
#if RCG_PRE_FENCE
          __syncwarp();   // scheduling fence: all 2 CG loads issue before the first FMA
#endif
          const double2 x0a = *reinterpret_cast<const double2*>(v0 + 2 * pi);
          const double2 x0b = *reinterpret_cast<const double2*>(v0 + 2 * (pi + 32));
          double2 x1a = make_double2(0.0, 0.0), x1b = make_double2(0.0, 0.0);
          if (NV == 2) {
            x1a = *reinterpret_cast<const double2*>(v1 + 2 * pi);
            x1b = *reinterpret_cast<const double2*>(v1 + 2 * (pi + 32));
          }
#pragma unroll
          for (int c = 0; c < CG; ++c) {
            a0[c] = fma(va[c].y, x0a.y, fma(va[c].x, x0a.x, a0[c]));
            if (NV == 2) a1[c] = fma(va[c].y, x1a.y, fma(va[c].x, x1a.x, a1[c]));
            a0[c] = fma(vb[c].y, x0b.y, fma(vb[c].x, x0b.x, a0[c]));
            if (NV == 2) a1[c] = fma(vb[c].y, x1b.y, fma(vb[c].x, x1b.x, a1[c]));
          }
        }
        for (int64_t pi = base + lane; pi < p_end; pi += 32) {
          const double2 x0 = *reinterpret_cast<const double2*>(v0 + 2 * pi);
          double2 x1 = make_double2(0.0, 0.0);
          if (NV == 2) x1 = *reinterpret_cast<const double2*>(v1 + 2 * pi);
#pragma unroll
          for (int c = 0; c < CG; ++c) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + pi);
            a0[c] = fma(v.y, x0.y, fma(v.x, x0.x, a0[c]));
            if (NV == 2) a1[c] = fma(v.y, x1.y, fma(v.x, x1.x, a1[c]));
          }
        }
      } else if (kc == CG) {
        if (PF && lane < CG && p_begin < p_end)
          bulk_prefetch_l2(cols + lane * ld + 2 * p_begin,
                           (unsigned)(16 * min((int64_t)32 * PF_DIST, p_end - p_begin)));
#pragma unroll(kGemvUnroll)
        for (int64_t pi = p_begin + lane; pi < p_end; pi += 32) {
          if (PF && lane < CG) {
            const int64_t step0 = pi - lane - p_begin;  // multiple of 32
            if ((step0 & (32 * PF_WIN - 1)) == 0) {
              const int64_t ahead = p_begin + step0 + 32 * PF_DIST;
              if (ahead < p_end)
                bulk_prefetch_l2(cols + lane * ld + 2 * ahead,
                                 (unsigned)(16 * min((int64_t)32 * PF_WIN, p_end - ahead)));
            }
          }
          const double2 x0 = *reinterpret_cast<const double2*>(v0 + 2 * pi);
          double2 x1 = make_double2(0.0, 0.0);
          if (NV == 2) x1 = *reinterpret_cast<const double2*>(v1 + 2 * pi);
#pragma unroll
          for (int c = 0; c < CG; ++c) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + pi);
            a0[c] += v.x * x0.x + v.y * x0.y;
            if (NV == 2) a1[c] += v.x * x1.x + v.y * x1.y;
          }
        }
      } else {
        for (int64_t pi = p_begin + lane; pi < p_end; pi += 32) {
          const double2 x0 = *reinterpret_cast<const double2*>(v0 + 2 * pi);
          double2 x1 = make_double2(0.0, 0.0);
          if (NV == 2) x1 = *reinterpret_cast<const double2*>(v1 + 2 * pi);
#pragma unroll
          for (int c = 0; c < CG; ++c)
            if (c < kc) {
              const double2 v = __ldcs(reinterpret_cast<const double2*>(cols + c * ld) + pi);
              a0[c] += v.x * x0.x + v.y * x0.y;
              if (NV == 2) a1[c] += v.x * x1.x + v.y * x1.y;
            }
        }
      }
      // odd tail row (len odd) belongs to the last slice
      if ((len & 1) && sl == S - 1 && lane == 0) {
        const int64_t i = len - 1;
#pragma unroll
        for (int c = 0; c < CG; ++c)
          if (c < kc) {
            const double v = cols[c * ld + i];
            a0[c] += v * v0[i];
            if (NV == 2) a1[c] += v * v1[i];
          }
      }
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        a0[c] = warp_sum(a0[c]);
        if (NV == 2) a1[c] = warp_sum(a1[c]);
      }
    }
    if (S == 1) {
      if (g >= 0 && lane == 0) {
        const int64_t k0 = g * CG;
#pragma unroll
        for (int c = 0; c < CG; ++c)
          if (k0 + c < ncols) {
            out[(k0 + c) * NV] = a0[c];
            if (NV == 2) out[(k0 + c) * NV + 1] = a1[c];
          }
      }
    } else {
      // combine the S slices of each group in slice order (deterministic)
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < CG; ++c) {
          red[(wid * CG + c) * NV] = a0[c];
          if (NV == 2) red[(wid * CG + c) * NV + 1] = a1[c];
        }
      }
      __syncthreads();
      if (g >= 0 && sl == 0 && lane == 0) {
        const int64_t k0 = g * CG;
        for (int c = 0; c < CG; ++c) {
          if (k0 + c >= ncols) break;
          double s0 = 0.0, s1 = 0.0;
          for (int q = 0; q < S; ++q) {
            s0 += red[((wid + q) * CG + c) * NV];
            if (NV == 2) s1 += red[((wid + q) * CG + c) * NV + 1];
          }
          out[(k0 + c) * NV] = s0;
          if (NV == 2) out[(k0 + c) * NV + 1] = s1;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// K2: alpha, x/r update, ||r||^2, AC^T y partials.  init != 0: no update
// (initial residual: only ||r||^2 and AC^T y).

__global__ void __launch_bounds__(kThreads)
update_kernel(const IterArgs* __restrict__ ap, int init) {
  pdl_wait();
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  if (st->done) return;
  const long long j = st->j;
  double alpha = 0.0;
  if (!init) {
    const double wAw = a.sums[0];
    const double rz = st->rz;
    if (wAw <= 0.0) {                                       // solver.py:244-245
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->failure = RCG_FAIL_WAW;
        st->done = 1;
      }
      return;
    }
    alpha = rz / wAw;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.alphas[j] = alpha;
      a.rz_hist[j] = rz;
      if (a.waw_diag) a.waw_diag[j] = wAw;
    }
  }
  __shared__ double sm[kWarps];
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_block_upd;
  const int64_t r1 = min(a.n, r0 + a.rows_per_block_upd);
  const double* w = a.W.at(j);
  const double* aw = a.AW.at(j);
  double* rh = a.R.base ? a.R.at(j) : nullptr;
  double rr = 0.0;
  // row pairs with 128-bit accesses (tiles start at multiples of 256 rows and
  // every vector / history column is 16-B aligned), then an odd last row
  const int64_t p0 = r0 >> 1, p1 = r1 >> 1;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(a.x);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(a.r);
#pragma unroll 2
  for (int64_t pi = p0 + threadIdx.x; pi < p1; pi += kThreads) {
    double2 rv = r2[pi];
    if (!init) {
      if (rh) reinterpret_cast<double2*>(rh)[pi] = rv;
      const double2 wv = reinterpret_cast<const double2*>(w)[pi];
      const double2 av = reinterpret_cast<const double2*>(aw)[pi];
      double2 xv = x2[pi];
      xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, wv.x));      // x = x + alpha w
      xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, wv.y));
      rv.x = __dsub_rn(rv.x, __dmul_rn(alpha, av.x));      // r = r - alpha Aw
      rv.y = __dsub_rn(rv.y, __dmul_rn(alpha, av.y));
      x2[pi] = xv;
      r2[pi] = rv;
    }
    rr += rv.x * rv.x + rv.y * rv.y;
  }
  if ((r1 & 1) && threadIdx.x == 0) {
    const int64_t i = r1 - 1;
    double ri = a.r[i];
    if (!init) {
      if (rh) rh[i] = ri;
      a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, w[i]));
      ri = __dsub_rn(ri, __dmul_rn(alpha, aw[i]));
      a.r[i] = ri;
    }
    rr += ri * ri;
  }
  // ||r||^2 partial in column 0 of the [tile][1 + n_c] partial rows; the
  // AC^T y columns come from actr_kernel (same tiles)
  const int64_t K = 1 + a.n_c;
  const double rrb = block_sum<kThreads>(rr, sm);
  if (threadIdx.x == 0) a.part_upd[(size_t)blockIdx.x * K] = rrb;
  if (arrive_last(a.counters + 1)) reduce_partials_strided<kThreads>(a.part_upd, gridDim.x, (int)K, 1, a.sums + 1);
}

// AC^T (M^{-1} r) for the projector (solver.py:84-91): grid (row tiles, groups
// of 8 columns).  The 8 warps split the tile's rows; lanes read 2 rows per
// column with one 128-bit load; y = inv_diag * r is recomputed exactly as in
// the reference (one rounding).  Partials go to columns 1..n_c of the
// [tile][1 + n_c] rows; the last CTA reduces them in a fixed order.
__global__ void __launch_bounds__(kThreads)
actr_kernel(const IterArgs* __restrict__ ap) {
  pdl_wait();
  const IterArgs& a = *ap;
  if (a.st->done) return;
  constexpr int CG = 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x, k0 = (int64_t)blockIdx.y * CG;
  const int kc = (int)min((int64_t)CG, a.n_c - k0);
  const int64_t r0 = tile * a.rows_per_block_actr;
  const int64_t len = min(a.n, r0 + a.rows_per_block_actr) - r0;
  const int64_t pairs = len >> 1, per = (pairs + kWarps - 1) / kWarps;
  const int64_t pb = wid * per, pe = min(pairs, pb + per);
  const double* __restrict__ cols = a.AC + k0 * a.ldac + r0;
  const double* __restrict__ rr = a.r + r0;
  const double* __restrict__ inv = a.inv_diag ? a.inv_diag + r0 : nullptr;
  double acc[CG];
#pragma unroll
  for (int c = 0; c < CG; ++c) acc[c] = 0.0;
  // all CG column loads of a row pair are issued unconditionally (a short
  // last group re-reads its last column from L1) before any arithmetic, so
  // each lane keeps CG + 2 LDG.128 in flight
  const double2* __restrict__ c2 = reinterpret_cast<const double2*>(cols);
  const int64_t ld2 = a.ldac >> 1;
#if RCG_ACTR_PIPE
  // software pipeline: the next row pair's CG + 2 loads are issued before
  // this pair's FMAs, so a warp never waits a full round trip per step
  double2 v[CG], y = make_double2(0.0, 0.0), d = make_double2(1.0, 1.0);
  int64_t pi = pb + lane;
  if (pi < pe) {
#pragma unroll
    for (int c = 0; c < CG; ++c) v[c] = __ldcs(c2 + (c < kc ? c : kc - 1) * ld2 + pi);
    y = *reinterpret_cast<const double2*>(rr + 2 * pi);
    if (inv) d = *reinterpret_cast<const double2*>(inv + 2 * pi);
  }
  for (; pi < pe; pi += 32) {
    const int64_t pn = pi + 32;
    double2 vn[CG], yn = make_double2(0.0, 0.0), dn = make_double2(1.0, 1.0);
    if (pn < pe) {
#pragma unroll
      for (int c = 0; c < CG; ++c) vn[c] = __ldcs(c2 + (c < kc ? c : kc - 1) * ld2 + pn);
      yn = *reinterpret_cast<const double2*>(rr + 2 * pn);
      if (inv) dn = *reinterpret_cast<const double2*>(inv + 2 * pn);
    }
    if (inv) {
      y.x = __dmul_rn(d.x, y.x);
      y.y = __dmul_rn(d.y, y.y);
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) acc[c] += v[c].x * y.x + v[c].y * y.y;
#pragma unroll
    for (int c = 0; c < CG; ++c) v[c] = vn[c];
    y = yn;
    d = dn;
  }
#else
#pragma unroll 1
  for (int64_t pi = pb + lane; pi < pe; pi += 32) {
    double2 v[CG];
#pragma unroll
    for (int c = 0; c < CG; ++c) v[c] = __ldcs(c2 + (c < kc ? c : kc - 1) * ld2 + pi);
    double2 y = *reinterpret_cast<const double2*>(rr + 2 * pi);
    if (inv) {
      const double2 d = *reinterpret_cast<const double2*>(inv + 2 * pi);
      y.x = __dmul_rn(d.x, y.x);
      y.y = __dmul_rn(d.y, y.y);
    }
#pragma unroll
    for (int c = 0; c < CG; ++c) acc[c] += v[c].x * y.x + v[c].y * y.y;
  }
#endif
  if ((len & 1) && wid == kWarps - 1 && lane == 0) {
    const int64_t i = len - 1;
    const double y = inv ? __dmul_rn(inv[i], rr[i]) : rr[i];
#pragma unroll
    for (int c = 0; c < CG; ++c)
      if (c < kc) acc[c] += cols[c * a.ldac + i] * y;
  }
  __shared__ double red[kWarps][CG];
#pragma unroll
  for (int c = 0; c < CG; ++c) {
    const double s = warp_sum(acc[c]);
    if (lane == 0) red[wid][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < kc) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += red[q][threadIdx.x];   // warp order: fixed
    a.part_upd[(size_t)tile * (1 + a.n_c) + 1 + k0 + threadIdx.x] = s;
  }
  // last CTA of the 2-D grid reduces the AC^T y columns over the tiles
  __shared__ bool last;
  __syncthreads();  // + thread-0 fence (cumulative), see arrive_last
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(a.counters + 3, 1u);
    last = (prev == gridDim.x * gridDim.y - 1);
    if (last) a.counters[3] = 0u;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    reduce_partials_strided<kThreads>(a.part_upd + 1, (int)gridDim.x, (int)(1 + a.n_c), (int)a.n_c, a.sums + 2);
  }
}

// coarse solve s = G^{-1} (AC^T y) for n_c > NC_INLINE: one warp per row of
// Ginv, grid-stride over rows (fixed grid: graph-replayable for any n_c)
__global__ void __launch_bounds__(kThreads)
coarse_kernel(const IterArgs* __restrict__ ap, int check_done) {
  pdl_wait();
  const IterArgs& a = *ap;
  if (check_done && a.st->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* u = a.sums + 2;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < a.n_c; row += nw) {
    const double* g = a.Ginv + row * a.n_c;   // symmetric: row == column
    double s = 0.0;
    for (int64_t k = lane; k < a.n_c; k += 32) s += g[k] * u[k];
    s = warp_sum(s);
    if (lane == 0) a.s_ext[row] = s;
  }
}

// ---------------------------------------------------------------------------
// K3: convergence test, z = M^{-1} r - C s, (r, z), reorth partials

// REO = false: the lean no-reorth variant (no GEMV code): RCG_PRE_LEAN_MINB
// CTAs/SM with RCG_PRE_ZB_LEAN rows in flight per thread for the z pass
template <int CG, bool PF, bool REO>
__global__ void __launch_bounds__(kThreads, REO ? RCG_PRE_MINB : RCG_PRE_LEAN_MINB)
precond_kernel(const IterArgs* __restrict__ ap, int init) {
  pdl_wait();
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  if (st->done) return;
  const long long j = st->j;
  if (!init) {
    const double rnorm = sqrt(a.sums[1]);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) a.rnorms[j + 1] = rnorm;
    if (rnorm <= st->tol_abs) {                              // solver.py:273
      if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        st->converged = 1;
        st->iterations = j + 1;
        st->done = 1;
      }
      return;
    }
  }
  extern __shared__ double dyn[];
  __shared__ double sm[kWarps];
  const int R = a.rows_per_block;
  const int RT = a.reorth ? R : 0;
  double* ztile = dyn;            // R (reorth only)
  double* wtile = dyn + RT;       // R (reorth only)
  double* s = a.s_smem ? dyn + 2 * RT : a.s_ext;   // n_c (global when it does not fit in smem)
  if (a.n_c && a.s_smem) {
    if (a.n_c <= NC_INLINE) {
      // s_i = sum_k Ginv[i,k] u_k, fixed order (every CTA computes the same s)
      const double* u = a.sums + 2;
      for (int64_t i = threadIdx.x; i < a.n_c; i += kThreads) {
        const double* g = a.Ginv + i * a.n_c;
        double acc = 0.0;
        for (int64_t k = 0; k < a.n_c; ++k) acc += g[k] * u[k];
        s[i] = acc;
      }
    } else {
      for (int64_t i = threadIdx.x; i < a.n_c; i += kThreads) s[i] = a.s_ext[i];
    }
    __syncthreads();
  }
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int64_t r1 = min(a.n, r0 + R);
  double* z = init ? a.Z.at(j) : a.Z.at(j + 1);
  double* w0 = init ? a.W.at(j) : nullptr;
  const double* wj = a.W.at(j);
  const bool reo = REO && a.reorth && !init;
  // column splits (small n): split 0 owns the z / (r, z) outputs, every split
  // rebuilds the z tile and streams its share of the AW columns
  const int split = blockIdx.y, S = gridDim.y;
  const bool lead = split == 0;
  double rz = 0.0;
  // ZB rows per thread per step, every load of the step issued before the
  // step's stores (z may alias r / W for the compiler, which would otherwise
  // serialize one HBM round trip per row); rows i, i + 256, ... keep the
  // per-thread (r, z) summation order of a plain row loop
  constexpr int ZB = RCG_PRE_ZB_LEAN > 0 && !REO ? RCG_PRE_ZB_LEAN : 4;
  for (int64_t ib = r0 + threadIdx.x; ib < r1; ib += ZB * kThreads) {
    double rv[ZB], zv[ZB], wv[ZB];
#pragma unroll
    for (int u = 0; u < ZB; ++u) {
      const int64_t i = ib + u * kThreads;
      rv[u] = i < r1 ? a.r[i] : 0.0;
      zv[u] = (i < r1 && a.inv_diag) ? a.inv_diag[i] : 1.0;
      wv[u] = (reo && i < r1) ? wj[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < ZB; ++u) {
      const int64_t i = ib + u * kThreads;
      double zi = a.inv_diag ? __dmul_rn(zv[u], rv[u]) : rv[u];
      if (a.n_c && i < r1) {
        double cs = 0.0;
        for (int64_t c = 0; c < a.n_c; ++c) cs += a.C[c * a.ldc + i] * s[c];
        zi = __dsub_rn(zi, cs);                             // y - C s  (solver.py:91)
      }
      zv[u] = zi;
    }
#pragma unroll
    for (int u = 0; u < ZB; ++u) {
      const int64_t i = ib + u * kThreads;
      if (i >= r1) break;
      const double zi = zv[u];
      if (lead) {
        z[i] = zi;
        if (w0) w0[i] = zi;                                 // w_0 = z_0 (solver.py:231)
      }
      rz += rv[u] * zi;
      if (reo) {
        ztile[i - r0] = zi;
        wtile[i - r0] = wv[u];
      }
    }
  }
  const double rzb = block_sum<kThreads>(rz, sm);
  if (lead && threadIdx.x == 0) a.part_z[blockIdx.x] = rzb;
  if (REO && reo) {
    __syncthreads();
    // AW is fully stored when reorthogonalizing (mod 0): column k at base + k*ld
    __shared__ double red[kWarps * CG * 2];
    const long long kb = (j + 1) * split / S, ke = (j + 1) * (split + 1) / S;
    gemv_t_tile<CG, 2, PF>(a.AW.base + kb * a.AW.ld + r0, a.AW.ld, ke - kb, r1 - r0, ztile, wtile,
                          a.part_reo + (size_t)blockIdx.x * a.reo_stride + 2 * kb, red);
  }
  if (lead && arrive_last(a.counters + 2)) reduce_partials<kThreads>(a.part_z, gridDim.x, 1, a.sums + a.rz_off);
}

// K4: sums[rz_off+1+q] = sum_b part_reo[b][q], q < 2(j+1).  8 q per CTA step
// x 32 tile slices: each thread adds ~nb/32 tile partials (loads batched 4 at
// a time), then the 32 slice sums of each q are added in slice order (fixed
// order: bitwise reproducible).  Grid-stride over q with a fixed grid so the
// launch is graph-replayable.
__global__ void __launch_bounds__(256)
colreduce_kernel(const IterArgs* __restrict__ ap) {
  pdl_wait();
  const IterArgs& a = *ap;
  if (a.st->done) return;
  const long long j = a.st->j;
  const int nb = a.nb_pre;
  const int64_t Q = 2 * (j + 1);
  const int tq = threadIdx.x & 7, ts = threadIdx.x >> 3;   // q in step, tile slice (0..31)
  __shared__ double sm[32][9];
  for (int64_t q0 = (int64_t)blockIdx.x * 8; q0 < Q; q0 += (int64_t)gridDim.x * 8) {
    const int64_t q = q0 + tq;
    double s = 0.0;
    if (q < Q) {
      const double* __restrict__ pc = a.part_reo + q;
      int b = ts;
      for (; b + 96 < nb; b += 128) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(pc + (size_t)(b + 32 * u) * a.reo_stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) s += v[u];
      }
      for (; b < nb; b += 32) s += __ldcg(pc + (size_t)b * a.reo_stride);
    }
    sm[ts][tq] = s;
    __syncthreads();
    if (threadIdx.x < 8 && q0 + threadIdx.x < Q) {
      double t = 0.0;
#pragma unroll 8
      for (int g = 0; g < 32; ++g) t += sm[g][threadIdx.x];
      a.sums[a.rz_off + 1 + q0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
  // zero the slots past 2(j+1) up to the history capacity: a sharded batch
  // allreduces the whole capacity (one width per captured graph)
  for (int64_t q = Q + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.reo_stride;
       q += (int64_t)gridDim.x * blockDim.x)
    a.sums[a.rz_off + 1 + q] = 0.0;
}

// ---------------------------------------------------------------------------
// Persistent solve loop for small operators (n = 16,384 is
// L2-resident and each iteration is 3-4 dependent reductions, so six kernel
// launches and their last-block tails dominate).  One cooperative grid of one
// CTA per SM runs up to B iterations; block b owns the contiguous rows
// [b R, (b+1) R).  Five grid-wide barriers per iteration replace the launch
// boundaries; every block re-derives alpha, ||r||, beta and the convergence /
// failure decisions from the same partial rows in the same fixed order, so
// all blocks take identical branches and write identical bits (block 0 writes
// the trace).  Same arithmetic as K1-K5 (CSR SpMV with sequential row sums,
// explicitly rounded updates, r history and capped z history as K2/K3); used
// when n <= RCG_SMALL_N, n_c <= 64 and not sharded.
//   sp row b: [0] (w, Aw)  [1] ||r||^2  [2, 2+n_c) AC^T y  [2+n_c] (r, z)

constexpr int SMALL_ROWS = 512;   // max rows per block (n <= 148 * 512)

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& gen) {
#if RCG_CG_SYNC
  (void)bar;
  (void)gen;
  cooperative_groups::this_grid().sync();
  return;
#endif
  // sense-free generation barrier over gridDim.x co-resident blocks
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    const unsigned int target = gen * gridDim.x;
    atomicAdd(bar, 1u);
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if ((int)(v - target) >= 0) break;
    }
  }
  __syncthreads();
}

// fixed-order sum over the G block rows of column `col` (stride `ld`), same
// bits in every block: lanes stride the rows, then a fixed shuffle tree
__device__ __forceinline__ double grid_sum_col(const double* part, int ld, int col, int G) {
  return warp_sum(lane_strided_sum(part + col, G, ld, threadIdx.x & 31));
}

__global__ void __launch_bounds__(kThreads, 1)
small_solve_kernel(const IterArgs* __restrict__ ap, double* sp, int sps, unsigned int* bar, long long B) {
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n = a.n, R = (n + G - 1) / G;
  const int64_t r0 = min(n, (int64_t)blockIdx.x * R), r1 = min(n, r0 + R);
  const int64_t len = r1 - r0;
  const int32_t* __restrict__ ci = a.spmv.ci;
  const double* __restrict__ va = a.spmv.va;
  __shared__ double ys[SMALL_ROWS], zs[SMALL_ROWS], wsh[SMALL_ROWS];
  __shared__ double ssh[NC_INLINE];
  __shared__ double cp[CP_CHUNK];
  __shared__ double red[kWarps];
  __shared__ double bc[4];
  unsigned int gen = 0;
  if (threadIdx.x == 0) gen = __ldcg(bar) / G;   // barrier generations already completed
  const int ncs = (int)a.n_c;
  for (long long it = 0; it < B; ++it) {
    if (__ldcg(&st->done)) return;
    const long long j = __ldcg(&st->j);
    const double rz = __ldcg(&st->rz);
    const double* __restrict__ w = a.W.at(j);
    double* __restrict__ aw = a.AW.at(j);
    // ---- K1: Aw_j = A w_j (thread per row, CSR, sequential row sum); (w, Aw)
    double d0 = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
      const int64_t ks = ((const int32_t*)a.spmv.ro)[i], ke = ((const int32_t*)a.spmv.ro)[i + 1];
      double acc = 0.0;
      for (int64_t k = ks; k < ke; ++k) acc += va[k] * __ldcg(w + ci[k]);
      aw[i] = acc;
      d0 += __ldcg(w + i) * acc;
    }
    d0 = block_sum<kThreads>(d0, red);
    if (threadIdx.x == 0) sp[(size_t)blockIdx.x * sps] = d0;
    grid_barrier(bar, gen);
    // ---- K2: alpha; x += alpha w; r -= alpha Aw; ||r||^2; AC^T y (own rows)
    if (wid == 0) {
      const double t = grid_sum_col(sp, sps, 0, G);
      if (lane == 0) bc[0] = t;
    }
    __syncthreads();
    const double wAw = bc[0];
    if (wAw <= 0.0) {                                        // solver.py:244-245
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->failure = RCG_FAIL_WAW;
        st->done = 1;
      }
      return;
    }
    const double alpha = rz / wAw;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.alphas[j] = alpha;
      a.rz_hist[j] = rz;
      if (a.waw_diag) a.waw_diag[j] = wAw;
    }
    double rr = 0.0;
    double* __restrict__ rh = a.R.base ? a.R.at(j) : nullptr;      // r history (TRKS)
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
      const double rold = a.r[i];
      if (rh) rh[i] = rold;
      const double xi = __dadd_rn(a.x[i], __dmul_rn(alpha, w[i]));     // x = x + alpha w
      const double ri = __dsub_rn(rold, __dmul_rn(alpha, __ldcg(aw + i)));   // r = r - alpha Aw
      a.x[i] = xi;
      a.r[i] = ri;
      rr += ri * ri;
      ys[i - r0] = a.inv_diag ? __dmul_rn(a.inv_diag[i], ri) : ri;
      wsh[i - r0] = w[i];
    }
    rr = block_sum<kThreads>(rr, red);
    if (threadIdx.x == 0) sp[(size_t)blockIdx.x * sps + 1] = rr;
    for (int c = wid; c < ncs; c += kWarps) {                // AC^T y over the block's rows
      const double* col = a.AC + (int64_t)c * a.ldac;
      double t = 0.0;
      for (int64_t q = lane; q < len; q += 32) t += col[r0 + q] * ys[q];
      t = warp_sum(t);
      if (lane == 0) sp[(size_t)blockIdx.x * sps + 2 + c] = t;
    }
    grid_barrier(bar, gen);
    // ---- K3: ||r|| test; s = G^{-1} u; z = M^{-1} r - C s; (r, z); reorth partials
    if (wid == 0) {
      const double t = grid_sum_col(sp, sps, 1, G);
      if (lane == 0) bc[1] = t;
    }
    for (int c = wid; c < ncs; c += kWarps) {
      const double t = grid_sum_col(sp, sps, 2 + c, G);
      if (lane == 0) cp[c] = t;                               // u = AC^T y
    }
    __syncthreads();
    const double rnorm = sqrt(bc[1]);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.rnorms[j + 1] = rnorm;
    if (rnorm <= st->tol_abs) {                               // solver.py:273
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->converged = 1;
        st->iterations = j + 1;
        st->done = 1;
      }
      return;
    }
    for (int i = threadIdx.x; i < ncs; i += kThreads) {      // s = Ginv u, fixed order
      const double* g = a.Ginv + (int64_t)i * ncs;
      double acc = 0.0;
      for (int k = 0; k < ncs; ++k) acc += g[k] * cp[k];
      ssh[i] = acc;
    }
    __syncthreads();
    double* __restrict__ z = a.Z.at(j + 1);
    double rzp = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
      const double ri = a.r[i];
      double zi = a.inv_diag ? __dmul_rn(a.inv_diag[i], ri) : ri;
      if (ncs) {
        double cs = 0.0;
        for (int c = 0; c < ncs; ++c) cs += a.C[(int64_t)c * a.ldc + i] * ssh[c];
        zi = __dsub_rn(zi, cs);                               // y - C s  (solver.py:91)
      }
      z[i] = zi;
      zs[i - r0] = zi;
      rzp += ri * zi;
    }
    rzp = block_sum<kThreads>(rzp, red);
    if (threadIdx.x == 0) sp[(size_t)blockIdx.x * sps + 2 + ncs] = rzp;
    if (a.reorth) {                                           // AW^T z, AW^T w_j over own rows
      // warp per group of 8 columns, lanes over the block's rows: 8 loads in
      // flight per lane and row step, one shuffle tree per column
      constexpr int SG = 8;
      double* pr = a.part_reo + (size_t)blockIdx.x * a.reo_stride;
      for (long long k0 = (long long)wid * SG; k0 <= j; k0 += (long long)kWarps * SG) {
        double t0[SG], t1[SG];
#pragma unroll
        for (int u = 0; u < SG; ++u) t0[u] = t1[u] = 0.0;
        const double* col = a.AW.base + (k0 + a.AW.shift) * a.AW.ld + r0;
        for (int64_t q = lane; q < len; q += 32) {
          const double zq = zs[q], wq = wsh[q];
          double v[SG];
#pragma unroll
          for (int u = 0; u < SG; ++u) v[u] = k0 + u <= j ? __ldcg(col + u * a.AW.ld + q) : 0.0;
#pragma unroll
          for (int u = 0; u < SG; ++u) {
            t0[u] += v[u] * zq;
            t1[u] += v[u] * wq;
          }
        }
#pragma unroll
        for (int u = 0; u < SG; ++u) {
          t0[u] = warp_sum(t0[u]);
          t1[u] = warp_sum(t1[u]);
          if (lane == 0 && k0 + u <= j) {
            pr[2 * (k0 + u)] = t0[u];
            pr[2 * (k0 + u) + 1] = t1[u];
          }
        }
      }
    }
    grid_barrier(bar, gen);
    // ---- K4: (r, z); reorth coefficients, column q reduced by block q mod G
    if (wid == 0) {
      const double t = grid_sum_col(sp, sps, 2 + ncs, G);
      if (lane == 0) bc[2] = t;
    }
    if (a.reorth) {
      const long long Q = 2 * (j + 1);
      for (long long q = (long long)blockIdx.x * kWarps + wid; q < Q; q += (long long)G * kWarps) {
        const double t = grid_sum_col(a.part_reo, (int)a.reo_stride, (int)q, G);
        if (lane == 0) a.sums[a.rz_off + 1 + q] = t;
      }
    }
    __syncthreads();
    const double rz_new = bc[2];
    if (rz_new <= 0.0) {                                      // solver.py:279-280
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->failure = RCG_FAIL_RZ;
        st->done = 1;
      }
      return;
    }
    const double beta = rz_new / rz;
    if (a.reorth) grid_barrier(bar, gen);
    // ---- K5: w_{j+1} = z + beta w_j - W ((AW^T (z + beta w)) / diag)
    double* __restrict__ wn = a.W.at(j + 1);
    const double* red2 = a.sums + a.rz_off + 1;
    double acc[2] = {0.0, 0.0};
    if (a.reorth) {
      for (long long k0 = 0; k0 <= j; k0 += CP_CHUNK) {
        const long long kn = min((long long)CP_CHUNK, j + 1 - k0);
        __syncthreads();
        for (long long k = threadIdx.x; k < kn; k += kThreads) {
          const long long kk = k0 + k;
          cp[k] = (__ldcg(red2 + 2 * kk) + beta * __ldcg(red2 + 2 * kk + 1)) / __ldcg(a.waw_diag + kk);
        }
        __syncthreads();
        // 8 columns per step, all 16 loads issued before the FMAs (in-order
        // issue would otherwise pay one L2 round trip per column)
        const double* colb = a.W.base + (k0 + a.W.shift) * a.W.ld;
        long long k = 0;
        for (; k + 8 <= kn; k += 8) {
          double v[8][2];
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int64_t i = r0 + threadIdx.x + q * kThreads;
              v[u][q] = i < r1 ? __ldcg(colb + (k + u) * a.W.ld + i) : 0.0;
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int q = 0; q < 2; ++q) acc[q] += v[u][q] * cp[k + u];
        }
        for (; k < kn; ++k) {
          const double ck = cp[k];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int64_t i = r0 + threadIdx.x + q * kThreads;
            if (i < r1) acc[q] += __ldcg(colb + k * a.W.ld + i) * ck;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t i = r0 + threadIdx.x + q * kThreads;
      if (i < r1) {
        double v = __dadd_rn(zs[i - r0], __dmul_rn(beta, wsh[i - r0]));   // w = z + beta w
        if (a.reorth) v = __dsub_rn(v, acc[q]);                          // w -= W c'
        wn[i] = v;
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.betas[j] = beta;
      st->rz = rz_new;
      st->j = j + 1;
      st->iterations = j + 1;
    }
    grid_barrier(bar, gen);
  }
}

// ---------------------------------------------------------------------------
// K5: beta, w_{j+1} = z + beta w_j  (- W c' with c' = (AW^T w)/diag)

// K5 without reorth: w_{j+1} = z + beta w_j, a pure stream.  A fixed grid of
// one wave of resident CTAs walks row blocks of RPT rows per thread (all 2 RPT
// loads of a block issued before its stores), so at 16.7 M rows 592 CTAs
// instead of 4,096 arrive on the iteration counter.
template <int RPT>
__global__ void __launch_bounds__(kThreads)
wupdate_plain_kernel(const IterArgs* __restrict__ ap) {
  pdl_wait();
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  if (st->done) return;
  const long long j = st->j;
  const double rz_new = a.sums[a.rz_off];
  const double rz_old = st->rz;
  if (rz_new <= 0.0) {                                       // solver.py:279-280
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->failure = RCG_FAIL_RZ;
      st->done = 1;
    }
    return;
  }
  const double beta = rz_new / rz_old;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.betas[j] = beta;
  const double* __restrict__ z = a.Z.at(j + 1);
  const double* __restrict__ wo = a.W.at(j);
  double* __restrict__ wn = a.W.at(j + 1);
  for (int64_t r0 = (int64_t)blockIdx.x * (kThreads * RPT); r0 < a.n; r0 += (int64_t)gridDim.x * (kThreads * RPT)) {
    double zq[RPT], wq[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t i = r0 + threadIdx.x + q * kThreads;
      zq[q] = i < a.n ? z[i] : 0.0;
      wq[q] = i < a.n ? wo[i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t i = r0 + threadIdx.x + q * kThreads;
      if (i < a.n) wn[i] = __dadd_rn(zq[q], __dmul_rn(beta, wq[q]));   // w = z + beta w
    }
  }
  // the grid's last block advances the iteration (all blocks arrive once)
  __shared__ bool g_last;
  __syncthreads();  // + thread-0 fence (cumulative), see arrive_last
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(a.counters + 4, 1u);
    g_last = (prev == gridDim.x - 1);
    if (g_last) a.counters[4] = 0u;
  }
  __syncthreads();
  if (g_last && threadIdx.x == 0) {
    __threadfence();
    st->rz = rz_new;
    st->j = j + 1;
    st->iterations = j + 1;
  }
}

// Rows of a block: thread t owns the row pairs (r0 + 2 (t + q kThreads), +1),
// q < RPT / 2, so every W load is one 128-bit access; acc[2q + e] is row
// r0 + 2 (t + q kThreads) + e.  Each row's W c sum keeps the reference's
// column order (k ascending, one rounding per FMA).
template <int RPT>
__device__ __forceinline__ int64_t wu_row(int64_t r0, int q2) {
  return r0 + 2 * ((int64_t)threadIdx.x + (q2 >> 1) * kThreads) + (q2 & 1);
}

template <int RPT>
__global__ void __launch_bounds__(kThreads, 3)
wupdate_kernel(const IterArgs* __restrict__ ap) {
  pdl_wait();
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  if (st->done) return;
  const long long j = st->j;
  const double rz_new = a.sums[a.rz_off];
  const double rz_old = st->rz;
  if (rz_new <= 0.0) {                                       // solver.py:279-280
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      st->failure = RCG_FAIL_RZ;
      st->done = 1;
    }
    return;
  }
  const double beta = rz_new / rz_old;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) a.betas[j] = beta;
  __shared__ double cp[CP_CHUNK];
  __shared__ bool s_last;
  const int S = gridDim.y;           // column splits (small n: rows alone do not fill the GPU)
  const int split = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * (kThreads * RPT);
  double acc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) acc[q] = 0.0;
  if (a.reorth) {
    const long long kb = (j + 1) * split / S, ke = (j + 1) * (split + 1) / S;
    const double* red = a.sums + a.rz_off + 1;
    for (long long k0 = kb; k0 < ke; k0 += CP_CHUNK) {
      const long long kn = min((long long)CP_CHUNK, ke - k0);
      __syncthreads();
      for (long long k = threadIdx.x; k < kn; k += kThreads) {
        const long long kk = k0 + k;
        // (AW^T (z + beta w))_k / (w_k, A w_k)   (solver.py:287)
        cp[k] = (red[2 * kk] + beta * red[2 * kk + 1]) / a.waw_diag[kk];
      }
      __syncthreads();
      // reorth implies a stored W history (ColSel mod == 0): column k at base + k ld
      const double* col0 = a.W.base + (k0 + a.W.shift) * a.W.ld + r0;
      const int64_t ldw = a.W.ld;
      constexpr int PPT = RPT / 2, KB = RCG_WU_KB;
      if (r0 + (int64_t)kThreads * RPT <= a.n) {
        // full row block: the 128-bit loads of KB columns x PPT row pairs are
        // issued before their FMAs (at the 80-register budget the compiler
        // otherwise interleaves them and keeps ~7 loads in flight)
        long long k = 0;
        for (; k + KB <= kn; k += KB) {
          double2 v[KB][PPT];
#pragma unroll
          for (int u = 0; u < KB; ++u)
#pragma unroll
            for (int q = 0; q < PPT; ++q)
              v[u][q] = __ldcs(reinterpret_cast<const double2*>(col0 + (k + u) * ldw) + threadIdx.x + q * kThreads);
          __syncwarp();   // scheduling fence: every load of the batch issues before the first FMA
#pragma unroll
          for (int u = 0; u < KB; ++u) {
            const double ck = cp[k + u];
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
              acc[2 * q] = fma(v[u][q].x, ck, acc[2 * q]);
              acc[2 * q + 1] = fma(v[u][q].y, ck, acc[2 * q + 1]);
            }
          }
        }
        for (; k < kn; ++k) {
          const double ck = cp[k];
#pragma unroll
          for (int q = 0; q < PPT; ++q) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(col0 + k * ldw) + threadIdx.x + q * kThreads);
            acc[2 * q] = fma(v.x, ck, acc[2 * q]);
            acc[2 * q + 1] = fma(v.y, ck, acc[2 * q + 1]);
          }
        }
      } else {
#pragma unroll 4
        for (long long k = 0; k < kn; ++k) {
          const double* col = col0 + k * ldw;
          const double ck = cp[k];
#pragma unroll
          for (int q2 = 0; q2 < RPT; ++q2) {
            const int64_t i = wu_row<RPT>(r0, q2);
            if (i < a.n) acc[q2] = fma(col[i - r0], ck, acc[q2]);
          }
        }
      }
    }
  }
  bool finisher = true;
  if (S > 1) {
    // park this split's partial sums; the last split of the row block adds
    // them in split order (deterministic) and finishes the rows
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t i = wu_row<RPT>(r0, q);
      if (i < a.n) a.part_wu[(int64_t)split * a.n + i] = acc[q];
    }
    __syncthreads();  // + thread-0 fence (cumulative), see arrive_last
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned int* cnt = a.counters + 16 + blockIdx.x;
      const unsigned int prev = atomicAdd(cnt, 1u);
      s_last = (prev == (unsigned)S - 1);
      if (s_last) *cnt = 0u;
    }
    __syncthreads();
    finisher = s_last;
    if (finisher) {
      __threadfence();
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int64_t i = wu_row<RPT>(r0, q);
        double t = 0.0;
        if (i < a.n)
          for (int sp = 0; sp < S; ++sp) t += __ldcg(a.part_wu + (int64_t)sp * a.n + i);
        acc[q] = t;
      }
    }
  }
  if (finisher) {
    const double* z = a.Z.at(j + 1);
    const double* wo = a.W.at(j);
    double* wn = a.W.at(j + 1);
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t i = wu_row<RPT>(r0, q);
      if (i < a.n) {
        double v = __dadd_rn(z[i], __dmul_rn(beta, wo[i]));   // w = z + beta w
        if (a.reorth) v = __dsub_rn(v, acc[q]);                // w -= W c'
        wn[i] = v;
      }
    }
  }
  // the grid's last block advances the iteration (all blocks arrive once)
  __shared__ bool g_last;
  __syncthreads();  // + thread-0 fence (cumulative), see arrive_last
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(a.counters + 4, 1u);
    g_last = (prev == gridDim.x * gridDim.y - 1);
    if (g_last) a.counters[4] = 0u;
  }
  __syncthreads();
  if (g_last && threadIdx.x == 0) {
    __threadfence();
    st->rz = rz_new;
    st->j = j + 1;
    st->iterations = j + 1;
  }
}

// initial (r0, z0) guard: rz <= 0 -> NumericalFailure before the loop (solver.py:229-230)
__global__ void init_finish_kernel(const IterArgs* __restrict__ ap) {
  const IterArgs& a = *ap;
  SolveState* st = a.st;
  if (st->done) return;
  const double rz = a.sums[a.rz_off];
  if (rz <= 0.0) {
    st->failure = RCG_FAIL_RZ;
    st->done = 1;
  } else {
    st->rz = rz;
  }
}

// ---------------------------------------------------------------------------
// generic GEMV-T (out[c] = X[:,c]^T v) with last-block reduction, and the
// coarse combination out = base - sign * X (Ginv u)  (project / initial_guess)

__global__ void __launch_bounds__(kThreads)
gemv_t_kernel(int64_t n, int64_t k, const double* __restrict__ X, int64_t ldx, const double* __restrict__ v,
              int rows_per_block, double* part, unsigned int* counter, double* out) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t len = min(n, r0 + rows_per_block) - r0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t c = wid; c < k; c += kWarps) {
    const double* col = X + c * ldx + r0;
    double p = 0.0;
    for (int64_t i = lane; i < len; i += 32) p += col[i] * v[r0 + i];
    p = warp_sum(p);
    if (lane == 0) part[(size_t)blockIdx.x * k + c] = p;
  }
  if (arrive_last(counter)) reduce_partials<kThreads>(part, gridDim.x, (int)k, out);
}

// s = G^{-1} u, one thread per row with a sequential (fixed-order) sum
__global__ void __launch_bounds__(kThreads)
coarse_s_kernel(int64_t n_c, const double* __restrict__ Ginv, const double* __restrict__ u, double* s) {
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= n_c) return;
  const double* g = Ginv + i * n_c;
  double acc = 0.0;
  for (int64_t kk = 0; kk < n_c; ++kk) acc += g[kk] * u[kk];
  s[i] = acc;
}

// out = base - X s (or X s): s staged in smem when it fits, else read from
// global memory (L2-resident, uniform across the warp)
__global__ void __launch_bounds__(kThreads)
coarse_combine_kernel(int64_t n, int64_t n_c, const double* __restrict__ X, int64_t ldx,
                      const double* __restrict__ s_glob, int stage, const double* __restrict__ base, double* out) {
  extern __shared__ double s_sm[];
  if (stage) {
    for (int64_t i = threadIdx.x; i < n_c; i += kThreads) s_sm[i] = s_glob[i];
    __syncthreads();
  }
  const double* s = stage ? s_sm : s_glob;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    double cs = 0.0;
    for (int64_t c = 0; c < n_c; ++c) cs += X[c * ldx + i] * s[c];
    out[i] = base ? __dsub_rn(base[i], cs) : cs;
  }
}

__global__ void copy_norms_kernel(int64_t n, const double* __restrict__ b, double* r, double* x,
                                  double* part, unsigned int* counter, double* out) {
  __shared__ double sm[kWarps];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const double bv = b[i];
    r[i] = bv;
    x[i] = 0.0;
    s += bv * bv;
  }
  s = block_sum<kThreads>(s, sm);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = s;
  }
  if (arrive_last(counter)) reduce_partials<kThreads>(part, gridDim.x, 2, out);
}

// ---------------------------------------------------------------------------
// host side

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int rows_per_block_for(const Ctx* c, int64_t n, int tiles_per_sm);

static int rows_per_block_for(const Ctx* c, int64_t n) {
  static const int tiles_per_sm = env_int("RCG_TILES_PER_SM", 2);
  return rows_per_block_for(c, n, tiles_per_sm);
}

static int rows_per_block_for(const Ctx* c, int64_t n, int tiles_per_sm) {
  // ~4 row tiles per SM: the tile kernels run 3-4 CTAs/SM (45 KB smem, <= 64 regs)
  const int64_t wave_rows = (int64_t)kThreads * tiles_per_sm * c->num_sms;   // one wave at 1 row/thread
  int64_t rpt = ceil_div(n, wave_rows);
  if (rpt > 16) {
    // the tile is capped (smem: 2 x 16 x 256 doubles); size it so the tiles
    // fill whole waves of resident CTAs instead of leaving a short last wave
    // (config 3, n = 2.7 M: 662 tiles = 2.24 waves -> 883 tiles = 2.98 waves)
    const int64_t waves = ceil_div(rpt, (int64_t)16);
    rpt = ceil_div(n, wave_rows * waves);
  }
  rpt = std::max<int64_t>(1, std::min<int64_t>(rpt, 16));
  return (int)(rpt * kThreads);
}

int gemv_t(Ctx* c, int64_t n, int64_t k, const double* X, int64_t ldx, const double* v, double* out) {
  if (k == 0) return RCG_OK;
  const int R = rows_per_block_for(c, n);
  const int nb = (int)std::max<int64_t>(1, ceil_div(n, R));
  char* base = nullptr;
  int rc = scratch(c, 256 + sizeof(double) * (size_t)nb * k, (void**)&base);
  if (rc) return rc;
  gemv_t_kernel<<<nb, kThreads, 0, c->stream>>>(n, k, X, ldx, v, R, (double*)(base + 256), c->counters + 8,
                                               out);
  RCG_LAUNCH_CHECK(c);
  return RCG_OK;
}

int coarse_combine(Ctx* c, const rcg_deflation* D, const double* u, const double* base, double* out) {
  const int64_t n_c = std::max<int64_t>(D->n_c, 1);
  double* sv = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&sv, sizeof(double) * (size_t)n_c, c->stream));
  coarse_s_kernel<<<(unsigned)ceil_div(n_c, (int64_t)kThreads), kThreads, 0, c->stream>>>(D->n_c, D->Ginv, u, sv);
  cudaError_t e = cudaGetLastError();
  const size_t smem = sizeof(double) * (size_t)n_c;
  const int stage = smem <= 48 * 1024 ? 1 : 0;
  if (e == cudaSuccess) {
    coarse_combine_kernel<<<elementwise_grid(c, D->n), kThreads, stage ? smem : 0, c->stream>>>(
        D->n, D->n_c, D->C, D->ldc, sv, stage, base, out);
    e = cudaGetLastError();
  }
  c->launches += 2;
  cudaFreeAsync(sv, c->stream);
  if (e != cudaSuccess) return set_error(c, RCG_ERR_CUDA, "coarse combine: %s", cudaGetErrorString(e));
  return RCG_OK;
}

}  // namespace rcg

using namespace rcg;

// ---------------------------------------------------------------------------
// trace object (owns the device histories of one solve)

struct rcg_trace {
  rcg_trace_view view{};
  std::vector<std::pair<void*, size_t>> allocs;   // returned to the pool on free
  std::vector<rcg::VmmBuf> vbufs;                  // Krylov histories (VA ranges)
  std::shared_ptr<rcg::VmmPool> vpool;
  std::shared_ptr<rcg::Pool> pool;
  cudaStream_t stream = nullptr;
  int device = 0;
};

extern "C" int rcg_trace_get_view(const rcg_trace* t, rcg_trace_view* out) {
  if (!t || !out) return RCG_ERR_CONTRACT;
  *out = t->view;
  return RCG_OK;
}

extern "C" void rcg_trace_free(rcg_trace* t) {
  if (!t) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  cudaStreamSynchronize(t->stream);
  for (auto& pb : t->allocs)
    if (pb.first) t->pool->put(pb.first, pb.second);
  for (auto& vb : t->vbufs) {
    if (t->vpool) t->vpool->give(vb);
    else vb.release();
  }
  cudaSetDevice(prev);
  delete t;
}

namespace {

struct Grow {
  // a column-major history buffer that grows geometrically (pooled blocks)
  double* ptr = nullptr;
  int64_t cols = 0;
  size_t bytes = 0;
};


// Krylov history on a growable VA range: the pointer never moves, growth
// maps more physical chunks (no copy, no peak)
struct Hist {
  VmmBuf v;
  double* ptr = nullptr;
  int64_t cols = 0;
};

int hist_init(Ctx* c, Hist& h, int64_t max_cols, int64_t init_cols, int64_t ld) {
  size_t total = 0, free_b = 0;
  cudaMemGetInfo(&free_b, &total);
  const size_t col_bytes = sizeof(double) * (size_t)ld;
  size_t max_bytes = std::min((size_t)std::max<int64_t>(max_cols, 1) * col_bytes, total);
  const size_t chunk = std::min<size_t>(std::max<size_t>(64 * col_bytes, (size_t)2 << 20), (size_t)512 << 20);
  const size_t g = vmm_granularity(c->device);
  const size_t chunk_r = std::max(g, ((chunk + g - 1) / g) * g);
  const size_t reserved = ((std::max<size_t>(max_bytes, 1) + chunk_r - 1) / chunk_r) * chunk_r;
  if (!c->vpool->take(chunk_r, reserved, &h.v) && !h.v.reserve(c->chunks, c->device, max_bytes, chunk))
    return set_error(c, RCG_ERR_OOM, "cannot reserve %.2f GB of device address space", max_bytes / 1e9);
  h.ptr = h.v.ptr();
  const size_t want = std::min(max_bytes, (size_t)init_cols * col_bytes);
  if (!h.v.ensure(want)) {
    c->vpool->clear();  // idle histories of earlier solves, then retry once
    c->chunks->trim();
    if (!h.v.ensure(want))
      return set_error(c, RCG_ERR_OOM, "out of device memory for a Krylov history (%lld columns, %.2f GB)",
                       (long long)init_cols, init_cols * col_bytes / 1e9);
  }
  h.cols = (int64_t)(h.v.mapped / col_bytes);
  return RCG_OK;
}

int hist_grow(Ctx* c, Hist& h, int64_t need_cols, int64_t ld) {
  if (need_cols <= h.cols) return RCG_OK;
  const size_t col_bytes = sizeof(double) * (size_t)ld;
  const size_t want = (size_t)std::max<int64_t>(need_cols, h.cols + h.cols / 4) * col_bytes;
  if (!h.v.ensure(std::min(want, h.v.reserved)) && !h.v.ensure((size_t)need_cols * col_bytes)) {
    c->vpool->clear();
    c->chunks->trim();
    if (!h.v.ensure((size_t)need_cols * col_bytes))
      return set_error(c, RCG_ERR_OOM, "out of device memory growing a Krylov history to %lld columns (%.2f GB)",
                       (long long)need_cols, need_cols * col_bytes / 1e9);
  }
  h.cols = (int64_t)(h.v.mapped / col_bytes);
  return RCG_OK;
}

}  // namespace

// collectives only for sharded calls (a context may own a communicator and
// still run unsharded solves)
static inline int allreduce_h(const rcg_halo* H, Ctx* c, double* buf, size_t count) {
  return H ? allreduce_sum(c, buf, count) : RCG_OK;
}

static int solve_impl(rcg_ctx* ctx, const rcg_csr* A, const double* inv_diag, const rcg_deflation* D,
                      const double* b, double* x, const rcg_solve_cfg* cfg, const rcg_halo* H,
                      rcg_trace** trace_out) {
  if (!ctx || !A || !cfg || !trace_out) return RCG_ERR_CONTRACT;
  *trace_out = nullptr;
  Ctx* c = ctx;
  const int64_t n = A->n;
  if (D && D->n != n) return set_error(c, RCG_ERR_CONTRACT, "deflation operator dimension mismatch");
  if (!(cfg->tol > 0.0 && cfg->tol < 1.0)) return set_error(c, RCG_ERR_CONTRACT, "tol must be in (0, 1)");
  if (cfg->max_iters < 1) return set_error(c, RCG_ERR_CONTRACT, "max_iters must be >= 1");
  const int64_t n_c = D ? D->n_c : 0;
  if (H && H->n_local != n) return set_error(ctx, RCG_ERR_CONTRACT, "halo n_local does not match the local rows");
  const int64_t n_ghost = H ? H->n_ghost : 0;
  // columns that feed the SpMV carry the ghost entries after the owned ones
  const int64_t ld = pad_ld(std::max<int64_t>(n + n_ghost, 1));
  const bool reorth = cfg->reorthogonalize != 0;
  const bool store = cfg->store_directions != 0;
  const bool capture = cfg->trace_capture != 0;
  const int64_t max_it = cfg->max_iters;

  rcg_trace* T = new rcg_trace();
  T->stream = c->stream;
  T->device = c->device;
  T->pool = c->pool;
  T->vpool = c->vpool;
  Grow gPR, gSum;
  Hist gW, gAW, gZ, gR;
  auto fail = [&](int rc) {
    for (Grow* g : {&gPR, &gSum})
      if (g->ptr) c->pool->put(g->ptr, g->bytes);
    for (Hist* h : {&gW, &gAW, &gZ, &gR}) c->vpool->give(h->v);
    rcg_trace_free(T);
    return rc;
  };
  // after this point every error path returns the solve's pooled buffers,
  // histories and trace (fail) instead of leaking them
#define RCG_CUDA_F(call)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(set_error(c, RCG_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__)); \
  } while (0)
#define RCG_LAUNCH_CHECK_F()                                                              \
  do {                                                                                    \
    c->launches++;                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail(set_error(c, RCG_ERR_CUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__)); \
  } while (0)

  auto alloc = [&](size_t bytes, void** p) -> int {
    bytes = std::max<size_t>(bytes, 256);
    *p = c->pool->get(bytes);
    if (!*p) return set_error(c, RCG_ERR_OOM, "device allocation of %zu bytes failed", bytes);
    T->allocs.emplace_back(*p, bytes);
    return RCG_OK;
  };

  // row tiles: K3 needs 2 smem tiles only when reorthogonalizing and K2 one
  // only with an augmentation basis; otherwise tiles grow so the grid stays
  // at <= 8 CTAs/SM (few last-block arrivals even at n = 16.7 M)
  auto big_tile = [&](int R0, int per_sm) {
    const int64_t rmin = ceil_div(ceil_div(n, (int64_t)per_sm * c->num_sms), kThreads) * kThreads;
    return (int)std::max<int64_t>(R0, rmin);
  };
  // without reorth K3 is the lean 4-CTA/SM variant: at most one wave of tiles
  // with reorth, K3 tiles (2 x R doubles of smem each) come in whole waves of
  // resident CTAs (RCG_PRE_MINB per SM): tiles = resident x waves, R a
  // multiple of 64 rows <= 4096; RCG_PRE_WAVES raises the wave count
  // (smaller tiles: CTAs drift apart, so one CTA's z pass and reduction tail
  // overlap other CTAs' AW streams)
  auto pre_tile = [&]() -> int {
    static const int min_waves = env_int("RCG_PRE_WAVES", 1);
    const int64_t resident = (int64_t)RCG_PRE_MINB * c->num_sms;
    if (n <= resident * 1024) return rows_per_block_for(c, n);
    const int64_t waves = std::max<int64_t>(min_waves, ceil_div(n, resident * 4096));
    const int64_t Rr = ceil_div(ceil_div(n, resident * waves), (int64_t)64) * 64;
    return (int)std::max<int64_t>(64, std::min<int64_t>(Rr, 4096));
  };
  const int R = reorth ? pre_tile() : big_tile(rows_per_block_for(c, n), 4);
  const int nb = (int)std::max<int64_t>(1, ceil_div(n, R));
  static const int upd_tiles = env_int("RCG_UPD_TILES_PER_SM", 4);
  const int Ru = n_c ? rows_per_block_for(c, n, upd_tiles) : big_tile(rows_per_block_for(c, n, upd_tiles), 8);
  const int nbu = (int)std::max<int64_t>(1, ceil_div(n, Ru));
  // K2b: exactly one wave of resident CTAs over all (tile, 8-column group)
  // pairs (a 1.3-wave grid ran its tail at a third of the SMs: 3.4 TB/s), so
  // each warp streams long runs (at most nbu tiles: the partial rows are K2's)
  static const int actr_occ = [] {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, actr_kernel, kThreads, 0) != cudaSuccess || occ < 1)
      occ = 2;
    return occ * env_int("RCG_ACTR_WAVES", 1);
  }();
  const int64_t ngr = std::max<int64_t>(1, ceil_div(n_c, 8));
  const int64_t nta0 = std::max<int64_t>(1, std::min<int64_t>(nbu, (int64_t)actr_occ * c->num_sms / ngr));
  const int Ra = (int)(ceil_div(ceil_div(n, nta0), (int64_t)2) * 2);
  const int nta = (int)std::max<int64_t>(1, ceil_div(n, Ra));
  const int nbs = spmv_partials(c, A);
  // K3 column splits for small n (the AW GEMV-T otherwise runs on nb CTAs only)
  const int pre_split = reorth ? (int)std::max<int64_t>(1, std::min<int64_t>(8, (2 * c->num_sms) / nb)) : 1;
  // K5 rows per thread: 4, or 16 when that keeps the grid below 8 CTAs/SM
  // (n ~ 1e7: fewer last-block arrivals on one counter)
  // (without reorth only: the 16-row variant is slow on the W GEMV)
  // rows per thread: 8 with reorth (8 rows x 4 unrolled columns = 32 loads in
  // flight per thread: 0.96 of copy bandwidth vs 0.78 for 4 rows,
  // tools/gemv_layout_bench3.cu); RCG_WU_RPT=4 restores the old shape
  static const int wu_rpt_env = env_int("RCG_WU_RPT", 8) == 4 ? 4 : 8;
  const int wu_rpt = (!reorth && ceil_div(n, (int64_t)kThreads * WU_RPT) > 8 * c->num_sms) ? 16
                     : (reorth ? wu_rpt_env : WU_RPT);
  const int wu_grid = (int)std::max<int64_t>(1, ceil_div(n, (int64_t)kThreads * wu_rpt));
  static const int wu_plain_occ = [] {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wupdate_plain_kernel<8>, kThreads, 0) != cudaSuccess ||
        occ < 1)
      occ = 4;
    return occ;
  }();
  const int wu_plain_grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(n, (int64_t)kThreads * 8), (int64_t)wu_plain_occ * c->num_sms));
  // launch grids: the tile kernels grid-stride, capped at a few CTAs per SM
  const int cap_grid = 8 * c->num_sms;
  const int nb_l = nb, nbu_l = nbu, wu_l = std::min(wu_grid, cap_grid);
  // K5 column splits when the row blocks alone cannot fill the SMs (small n)
  const int wu_split = reorth ? (int)std::max<int64_t>(1, std::min<int64_t>(16, (2 * c->num_sms) / wu_grid)) : 1;

  // fixed-size device allocations
  SolveState* st = nullptr;
  double *hist = nullptr, *r = nullptr, *part_upd = nullptr, *part_z = nullptr;
  double* part_spmv = nullptr;
  double* s_ext = nullptr;
  unsigned int* counters = nullptr;
  const int64_t nh = max_it + 2;
  int rc;
  if ((rc = alloc(sizeof(SolveState), (void**)&st))) return fail(rc);
  if ((rc = alloc(sizeof(double) * 5 * nh, (void**)&hist))) return fail(rc);
  if ((rc = alloc(sizeof(double) * ld, (void**)&r))) return fail(rc);
  if ((rc = alloc(sizeof(double) * nbu * (1 + n_c), (void**)&part_upd))) return fail(rc);
  // part_spmv holds 2 partials per CTA of the SpMV (mode 2) AND of copy_norms
  // (n_c = 0 initial residual), whose grids differ (BSR3 SpMV: 4 CTAs/SM)
  const int nps = std::max(nbs, elementwise_grid(c, n));
  if ((rc = alloc(sizeof(double) * (nb + 2 * nps + 64), (void**)&part_z))) return fail(rc);
  part_spmv = part_z + nb + 32;
  if ((rc = alloc(sizeof(double) * (n_c + 1), (void**)&s_ext))) return fail(rc);
  const size_t n_counters = 16 + (size_t)wu_grid;
  if ((rc = alloc(sizeof(unsigned int) * n_counters, (void**)&counters))) return fail(rc);
  RCG_CUDA_F(cudaMemsetAsync(counters, 0, sizeof(unsigned int) * n_counters, c->stream));
  double* part_wu = nullptr;
  if (wu_split > 1 && (rc = alloc(sizeof(double) * (size_t)wu_split * n, (void**)&part_wu))) return fail(rc);
  RCG_CUDA_F(cudaMemsetAsync(hist, 0, sizeof(double) * 5 * nh, c->stream));
  double* alphas = hist;
  double* betas = hist + nh;
  double* rzh = hist + 2 * nh;
  double* rnorms = hist + 3 * nh;
  double* wawd = hist + 4 * nh;

  // growable histories
  const bool storeW = reorth || store;
  // initial capacity from the previous solve of this size (sequences repeat)
  int64_t hint = 64;
  {
    auto h = c->m_hint.find(n);
    if (h != c->m_hint.end()) hint = std::max<int64_t>(64, h->second + h->second / 8 + 16);
  }
  const int64_t init_cols = std::min<int64_t>(max_it + 2, hint);
  const int64_t full_cols = max_it + 2;
  // capped z history: columns 0..cap-1 kept, column cap is the scratch column
  const int64_t zcap = (capture && cfg->krylov_cap > 0 && cfg->krylov_cap < max_it + 1) ? cfg->krylov_cap : 0;
  if ((rc = hist_init(c, gW, storeW ? full_cols : 2, storeW ? init_cols : 2, ld))) return fail(rc);
  if ((rc = hist_init(c, gAW, reorth ? full_cols : 1, reorth ? init_cols : 1, ld))) return fail(rc);
  if ((rc = hist_init(c, gZ, capture ? (zcap ? zcap + 1 : full_cols) : 2,
                      capture ? (zcap ? zcap + 1 : init_cols) : 2, ld)))
    return fail(rc);
  if (store && (rc = hist_init(c, gR, full_cols, init_cols, ld))) return fail(rc);

  auto reo_cols = [&]() { return gAW.cols; };
  // persistent cooperative solve loop for small operators (small_solve_kernel)
  // crossover (tools/small_threshold.py, 3-system sequences): persistent 26.7 vs 38.5 ms
  // at n = 16 k, 51 vs 60 ms at 33 k, 129 vs 121 ms at 65 k
  const int64_t small_n = env_int("RCG_SMALL_N", 49152);   // read per solve (tests switch paths)
  const bool small = !H && n <= small_n && n <= (int64_t)c->num_sms * SMALL_ROWS && n_c <= NC_INLINE &&
                     !A->row_offsets_64 && n > 0;
  // one CTA per SM, or fewer when RCG_SMALL_G says so (rows per CTA <= SMALL_ROWS)
  const int small_G = !small ? 0 : (int)std::min<int64_t>(c->num_sms, std::max<int64_t>(
      ceil_div(n, (int64_t)SMALL_ROWS), env_int("RCG_SMALL_G", c->num_sms)));
  auto ensure_sums = [&](void) -> int {
    const int64_t need = 8 + n_c + 1 + 2 * reo_cols() + 8;
    if (gSum.cols < need) {
      double* p = (double*)c->pool->get(sizeof(double) * need);
      if (!p) return set_error(c, RCG_ERR_OOM, "sums alloc");
      RCG_CUDA(c, cudaMemsetAsync(p, 0, sizeof(double) * need, c->stream));
      if (gSum.ptr) {
        RCG_CUDA(c, cudaMemcpyAsync(p, gSum.ptr, sizeof(double) * gSum.cols, cudaMemcpyDeviceToDevice, c->stream));
        RCG_CUDA(c, cudaStreamSynchronize(c->stream));
        c->pool->put(gSum.ptr, gSum.bytes);
      }
      gSum.ptr = p;
      gSum.cols = need;
      gSum.bytes = sizeof(double) * need;
    }
    if (reorth) {
      const int64_t needp = (int64_t)std::max(nb, small_G) * 2 * reo_cols();
      if (gPR.cols < needp) {
        if (gPR.ptr) {
          RCG_CUDA(c, cudaStreamSynchronize(c->stream));
          c->pool->put(gPR.ptr, gPR.bytes);
        }
        gPR.ptr = (double*)c->pool->get(sizeof(double) * needp);
        if (!gPR.ptr) return set_error(c, RCG_ERR_OOM, "reorth partials alloc");
        gPR.cols = needp;
        gPR.bytes = sizeof(double) * needp;
      }
    }
    return RCG_OK;
  };
  if ((rc = ensure_sums())) return fail(rc);
  if (H && (rc = halo_prepare(c, H))) return fail(rc);    // staging for the loop's graph-capturable exchange

  if (!c->dargs && cudaMalloc(&c->dargs, 4096) != cudaSuccess) return fail(set_error(c, RCG_ERR_OOM, "args"));
  static_assert(sizeof(IterArgs) <= 4096, "IterArgs too large");
  IterArgs* dargs = (IterArgs*)c->dargs;
  double* small_sp = nullptr;
  unsigned int* small_bar = nullptr;
  const int small_sps = 3 + (int)n_c;
  if (small) {
    if ((rc = alloc(sizeof(double) * (size_t)small_G * small_sps + 256, (void**)&small_sp))) return fail(rc);
    small_bar = (unsigned int*)(small_sp + (size_t)small_G * small_sps);
    RCG_CUDA_F(cudaMemsetAsync(small_bar, 0, 64, c->stream));
  }
  const int64_t nc_bucket = ((n_c + 1 + 63) / 64) * 64;
  const size_t smem_upd = sizeof(double) * (n_c ? Ru : 1);
  // z / w_j tiles only when reorthogonalizing (they feed the AW GEMV-T); the
  // coarse solution s joins them in smem while it fits (a TRKS basis can grow
  // past the opt-in limit: then K3 reads s from s_ext, L2-resident)
  const size_t smem_tiles = sizeof(double) * (reorth ? 2 * (size_t)R : 0);
  const bool s_smem = n_c <= NC_INLINE || smem_tiles + sizeof(double) * nc_bucket <= c->smem_optin;
  const size_t smem_pre = smem_tiles + (s_smem ? sizeof(double) * nc_bucket : 0);
  if (smem_pre > c->smem_optin)
    return fail(set_error(c, RCG_ERR_CONTRACT, "K3 tile of %d rows needs %zu B of shared memory (limit %zu)", R,
                          smem_pre, c->smem_optin));
  IterArgs a{};
  auto refresh = [&]() {
    a.n = n;
    a.inv_diag = inv_diag;
    a.n_c = n_c;
    a.C = D ? D->C : nullptr;
    a.ldc = D ? D->ldc : 0;
    a.AC = D ? D->AC : nullptr;
    a.ldac = D ? D->ldac : 0;
    a.Ginv = D ? D->Ginv : nullptr;
    a.s_ext = s_ext;
    a.x = x;
    a.r = r;
    a.W = colsel(gW.ptr, ld, storeW ? 0 : 2);
    a.AW = colsel(gAW.ptr, ld, reorth ? 0 : 1);
    a.Z = colsel(gZ.ptr, ld, capture ? 0 : 2, 0, zcap);
    a.R = colsel(store ? gR.ptr : nullptr, ld, 0);
    a.waw_diag = wawd;
    a.alphas = alphas;
    a.betas = betas;
    a.rz_hist = rzh;
    a.rnorms = rnorms;
    a.sums = gSum.ptr;
    a.rz_off = 2 + n_c;
    a.part_upd = part_upd;
    a.part_z = part_z;
    a.part_reo = gPR.ptr;
    a.part_wu = part_wu;
    a.reo_stride = 2 * reo_cols();
    a.counters = counters;
    a.st = st;
    a.reorth = reorth ? 1 : 0;
    a.rows_per_block = R;
    a.s_smem = s_smem ? 1 : 0;
    a.rows_per_block_upd = Ru;
    a.rows_per_block_actr = Ra;
    a.nb_pre = nb;
    a.nb_upd = nbu;
    a.nb_wu = wu_grid;
    spmv_args_fill(A, &a.spmv);
    a.spmv.xs = a.W;
    a.spmv.ys = a.AW;
    a.spmv.st = st;
    a.spmv.part = part_spmv;
    a.spmv.rem_part = part_spmv + 2 * (size_t)spmv_main_partials(c, A);
    a.spmv.counter = counters + 0;
    a.spmv.claim = counters + 5;   // [5] tile claims, [6] mode-0 arrivals (3x3 block-DIA)
    a.spmv.out = gSum.ptr;
    // device copy read by every iteration kernel (pageable source: staged
    // before return, so the host struct may change right after)
    return cudaMemcpyAsync(dargs, &a, sizeof(IterArgs), cudaMemcpyHostToDevice, c->stream);
  };
  RCG_CUDA_F(refresh());

  // dynamic smem sized by n_c bucket so graphs are reusable across the
  // systems of a sequence (n_c changes from system to system)
  RCG_CUDA_F(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(smem_upd, 1024)));
  static const int pre_cg = env_int("RCG_PRE_CG", 8);
  static const bool pre_pf = env_int("RCG_PF", 0) != 0;
  auto pre = !reorth ? precond_kernel<8, false, false>
             : (pre_cg == 4 ? precond_kernel<4, false, true>
                            : (pre_cg == 2 ? precond_kernel<2, false, true>
                                           : (pre_pf ? precond_kernel<8, true, true> : precond_kernel<8, false, true>)));
  RCG_CUDA_F(cudaFuncSetAttribute(pre, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(smem_pre, 1024)));

  // ---- initial guess and residual (solver.py:208-219) ----
  SolveState hs{};
  hs.j = 0;
  hs.iterations = 0;
  hs.done = 0;
  RCG_CUDA_F(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  double* norms2 = nullptr;  // ||r0||^2, ||b||^2
  if ((rc = alloc(sizeof(double) * 16, (void**)&norms2))) return fail(rc);
  if (n_c) {
    // x0 = C G^{-1} C^T b; r0 = b - A x0 (x0 needs its ghosts for the SpMV)
    double* xext = nullptr;
    if ((rc = alloc(sizeof(double) * ld, (void**)&xext))) return fail(rc);
    if ((rc = gemv_t(c, n, n_c, D->C, D->ldc, b, gSum.ptr + 2))) return fail(rc);
    if ((rc = allreduce_h(H, c, gSum.ptr + 2, (size_t)n_c))) return fail(rc);
    if ((rc = coarse_combine(c, D, gSum.ptr + 2, nullptr, xext))) return fail(rc);
    if ((rc = halo_exchange(c, H, colsel(xext), nullptr, xext))) return fail(rc);
    if ((rc = launch_spmv(c, A, 2, colsel(xext), colsel(r), b, nullptr, part_spmv, counters + 0, norms2, counters + 5)))
      return fail(rc);
    RCG_CUDA_F(cudaMemcpyAsync(x, xext, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    copy_norms_kernel<<<elementwise_grid(c, n), kThreads, 0, c->stream>>>(n, b, r, x, part_spmv, counters + 0,
                                                                        norms2);
    RCG_LAUNCH_CHECK_F();
  }
  if ((rc = allreduce_h(H, c, norms2, 2))) return fail(rc);
  double hn[2] = {0.0, 0.0};
  RCG_CUDA_F(cudaMemcpyAsync(hn, norms2, sizeof(hn), cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA_F(cudaStreamSynchronize(c->stream));
  const double r0 = std::sqrt(hn[0]);
  const double bn = std::sqrt(hn[1]);
  T->view.n = n;
  T->view.r0_norm = r0;
  T->view.b_norm = bn;
  T->view.ld = ld;
  RCG_CUDA_F(cudaMemcpyAsync(rnorms, &r0, sizeof(double), cudaMemcpyHostToDevice, c->stream));

  auto finish_view = [&](void) {
    T->view.alphas = alphas;
    T->view.betas = betas;
    T->view.rz_inner = rzh;
    T->view.residual_norms = rnorms;
    T->view.Z = capture ? gZ.ptr : nullptr;
    T->view.W = storeW ? gW.ptr : nullptr;
    T->view.AW = reorth ? gAW.ptr : nullptr;
    T->view.R = store ? gR.ptr : nullptr;
    T->view.waw = wawd;
    for (Hist* h : {&gW, &gAW, &gZ, &gR}) {
      if (h->v.base) T->vbufs.push_back(h->v);
      h->v = VmmBuf();
    }
    T->allocs.emplace_back(gPR.ptr, gPR.bytes);
    T->allocs.emplace_back(gSum.ptr, gSum.bytes);
    gW.ptr = gAW.ptr = gZ.ptr = gR.ptr = gPR.ptr = gSum.ptr = nullptr;
  };

  if (r0 == 0.0 || r0 <= 1e-13 * bn) {                     // solver.py:217-219
    T->view.iterations = 0;
    T->view.n_betas = 0;
    T->view.converged = 1;
    T->view.early_exit = 1;
    finish_view();
    *trace_out = T;
    return RCG_OK;
  }
  hs.tol_abs = cfg->tol * r0;
  RCG_CUDA_F(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));

  auto launch_coarse = [&](int check_done) -> int {
    if (n_c > NC_INLINE) {
      coarse_kernel<<<2 * c->num_sms, kThreads, 0, c->stream>>>(dargs, check_done);
      RCG_LAUNCH_CHECK(c);
    }
    return RCG_OK;
  };

  // ---- z0, rz0, w0 (solver.py:221-231) ----
  update_kernel<<<nbu_l, kThreads, 0, c->stream>>>(dargs, 1);
  RCG_LAUNCH_CHECK_F();
  if (n_c) {
    actr_kernel<<<dim3(nta, (unsigned)ngr), kThreads, 0, c->stream>>>(dargs);
    RCG_LAUNCH_CHECK_F();
  }
  if ((rc = allreduce_h(H, c, gSum.ptr + 1, (size_t)(1 + n_c)))) return fail(rc);
  if ((rc = launch_coarse(1))) return fail(rc);
  pre<<<nb_l, kThreads, smem_pre, c->stream>>>(dargs, 1);
  RCG_LAUNCH_CHECK_F();
  if ((rc = allreduce_h(H, c, gSum.ptr + a.rz_off, 1))) return fail(rc);
  init_finish_kernel<<<1, 1, 0, c->stream>>>(dargs);
  RCG_LAUNCH_CHECK_F();

  // ---- the loop (solver.py:241-288), batched ----
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, c->stream);
  SolveState* hst = (SolveState*)c->pinned;
  int64_t it = 0;
  // the persistent loop stops by itself at convergence (blocks return), so it
  // runs long batches: one host round trip per solve once m is known
  int64_t batch = cfg->batch > 0 ? cfg->batch : (small ? std::max<int64_t>(64, hint) : 4);

  const double jac = inv_diag ? 1.0 : 0.0;
  // algorithmic bytes of the format actually streamed (BSR3: one index per block)
  const double bytes_spmv =
      A->dia_count > 0
          ? 8.0 * A->dia_count * A->dia_block * (double)n + 16.0 * (double)n   // stored upper blocks + x, y
      : (A->block == 3 && A->bsr_row_offsets)
          ? 8.0 * (double)A->nnz + 4.0 * (double)A->nnz / 9.0 + 4.0 * (double)(n / 3 + 1) + 16.0 * (double)n
          : 12.0 * (double)A->nnz + (A->row_offsets_64 ? 8.0 : 4.0) * (double)(n + 1) + 16.0 * (double)n;
  static const int use_graphs = env_int("RCG_GRAPHS", 1);
  // sharded: halo exchange beside the local SpMV (needs the DIA + remainder slab format)
  const bool halo_overlap = H && env_int("RCG_HALO_OVERLAP", 1) && spmv_has_rem(A) && halo_active(c, H);
  if (halo_overlap && !c->halo_stream) {
    RCG_CUDA_F(cudaStreamCreateWithFlags(&c->halo_stream, cudaStreamNonBlocking));
    RCG_CUDA_F(cudaEventCreateWithFlags(&c->halo_fork, cudaEventDisableTiming));
    RCG_CUDA_F(cudaEventCreateWithFlags(&c->halo_join, cudaEventDisableTiming));
  }
  const double halo_bytes = H ? 8.0 * ((double)H->send_off[H->nranks] + (double)H->n_ghost) : 0.0;
  bool direct_now = false;   // set by launch_batch: profile the collectives too
  auto allreduce_p = [&](double* buf, size_t count, int64_t jj) -> int {
    if (!H) return RCG_OK;
    if (direct_now) prof_begin(c, RCG_K_ALLREDUCE, 8.0 * (double)count, jj);
    const int r = allreduce_sum(c, buf, count);
    if (direct_now) prof_end(c);
    return r;
  };
  const int cr_grid = 2 * c->num_sms;
  // queue B iterations; `direct` allows the host-side per-iteration work
  // (profiling events, halo exchanges with jj-dependent addresses)
  auto launch_batch = [&](int64_t B, int64_t it0, bool direct) -> int {
    int rc2;
    direct_now = direct;
    for (int64_t q = 0; q < B; ++q) {
      const int64_t jj = it0 + q;  // the device-side j unless the solve already stopped
      const double nd = (double)n, js = (double)(jj + 1);
      if (halo_overlap && !direct) {
        // the exchange of w_j's ghosts runs on a second stream beside the local
        // part of the slab SpMV (block-DIA of the local-local block: it reads
        // only local x) and joins before the ghost-column remainder; inside a
        // captured batch this is the fork / join of two captured streams
        RCG_CUDA(c, cudaEventRecord(c->halo_fork, c->stream));
        RCG_CUDA(c, cudaStreamWaitEvent(c->halo_stream, c->halo_fork, 0));
        cudaStream_t main_stream = c->stream;
        c->stream = c->halo_stream;
        rc2 = halo_exchange_dev(c, H, &dargs->W, &dargs->st, &dargs->W);
        c->stream = main_stream;
        if (rc2) return rc2;
        RCG_CUDA(c, cudaEventRecord(c->halo_join, c->halo_stream));
        if ((rc2 = launch_spmv_ind_main(c, A, &dargs->spmv))) return rc2;
        RCG_CUDA(c, cudaStreamWaitEvent(c->stream, c->halo_join, 0));
        if ((rc2 = launch_spmv_ind_rem(c, A, &dargs->spmv))) return rc2;
      } else {
        if (H) {  // ghosts of w_j from the neighbouring slabs (column at device j: graph-capturable)
          if (direct) prof_begin(c, RCG_K_HALO, halo_bytes, jj);
          if ((rc2 = halo_exchange_dev(c, H, &dargs->W, &dargs->st, &dargs->W))) return rc2;
          if (direct) prof_end(c);
        }
        // algorithmic bytes per launch (each operand touched once)
        if (direct) prof_begin(c, RCG_K_SPMV, bytes_spmv, jj);
        if ((rc2 = launch_spmv_ind(c, A, &dargs->spmv))) return rc2;
        if (direct) prof_end(c);
      }
      if ((rc2 = allreduce_p(gSum.ptr, 1, jj))) return rc2;
      if (direct) prof_begin(c, RCG_K_UPDATE, 8.0 * nd * (6 + (store ? 1 : 0)), jj);
      RCG_CUDA(c, launch_k(update_kernel, dim3(nbu_l), dim3(kThreads), 0, c->stream, (const IterArgs*)dargs, 0));
      c->launches++;
      if (direct) prof_end(c);
      if (n_c) {
        if (direct) prof_begin(c, RCG_K_ACTR, 8.0 * nd * (1 + jac + n_c), jj);
        RCG_CUDA(c, launch_k(actr_kernel, dim3(nta, (unsigned)ngr), dim3(kThreads), 0, c->stream,
                             (const IterArgs*)dargs));
        c->launches++;
        if (direct) prof_end(c);
      }
      if ((rc2 = allreduce_p(gSum.ptr + 1, (size_t)(1 + n_c), jj))) return rc2;
      if (n_c > NC_INLINE) {
        if (direct) prof_begin(c, RCG_K_COARSE, 8.0 * (double)n_c * (double)n_c, jj);
        if ((rc2 = launch_coarse(1))) return rc2;
        if (direct) prof_end(c);
      }
      if (direct) prof_begin(c, RCG_K_PRECOND, 8.0 * nd * (2 + jac + n_c + (reorth ? 1.0 + js : 0.0)), jj);
      RCG_CUDA(c, launch_k(pre, dim3(nb_l, pre_split), dim3(kThreads), smem_pre, c->stream, (const IterArgs*)dargs, 0));
      c->launches++;
      if (direct) prof_end(c);
      if (reorth) {
        if (direct) prof_begin(c, RCG_K_COLREDUCE, 8.0 * 2.0 * js * (nb + 1), jj);
        RCG_CUDA(c, launch_k(colreduce_kernel, dim3(cr_grid), dim3(256), 0, c->stream, (const IterArgs*)dargs));
        c->launches++;
        if (direct) prof_end(c);
      }
      // one packed allreduce: (r, z) and the reorth dot products, over the
      // history capacity (fixed between regrows, so the graph replays it;
      // colreduce zeroes the slots past 2(j+1))
      if ((rc2 = allreduce_p(gSum.ptr + a.rz_off, (size_t)(1 + (reorth ? a.reo_stride : 0)), jj))) return rc2;
      if (direct) prof_begin(c, RCG_K_WUPDATE, 8.0 * nd * (3 + (reorth ? js : 0.0)), jj);
      if (!reorth)
        RCG_CUDA(c, launch_k(wupdate_plain_kernel<8>, dim3(wu_plain_grid), dim3(kThreads), 0, c->stream,
                             (const IterArgs*)dargs));
      else if (wu_rpt == 8)
        RCG_CUDA(c, launch_k(wupdate_kernel<8>, dim3(wu_grid, wu_split), dim3(kThreads), 0, c->stream,
                             (const IterArgs*)dargs));
      else
        RCG_CUDA(c, launch_k(wupdate_kernel<WU_RPT>, dim3(wu_grid, wu_split), dim3(kThreads), 0, c->stream,
                             (const IterArgs*)dargs));
      c->launches++;
      if (direct) prof_end(c);
    }
    return RCG_OK;
  };
  bool done = false;
  while (it < max_it && !done) {
    const int64_t B = std::min<int64_t>(batch, max_it - it);
    // capacity for columns up to it + B + 1
    const int64_t need = it + B + 2;
    bool regrown = false;
    if (storeW && need > gW.cols) {
      if ((rc = hist_grow(c, gW, need, ld))) return fail(rc);
      regrown = true;
    }
    if (reorth && need > gAW.cols) {
      if ((rc = hist_grow(c, gAW, need, ld))) return fail(rc);
      regrown = true;
    }
    if (capture && !zcap && need > gZ.cols) {
      if ((rc = hist_grow(c, gZ, need, ld))) return fail(rc);
      regrown = true;
    }
    if (store && need > gR.cols) {
      if ((rc = hist_grow(c, gR, need, ld))) return fail(rc);
      regrown = true;
    }
    if (regrown) {
      if ((rc = ensure_sums())) return fail(rc);
      RCG_CUDA_F(refresh());
    }
    const bool graph_ok = use_graphs && !c->profiling && (!H || comm_graphable(c));
    if (small && !c->profiling) {
      long long Bl = (long long)B;
      const IterArgs* ap = dargs;
      void* kargs[] = {(void*)&ap, (void*)&small_sp, (void*)&small_sps, (void*)&small_bar, (void*)&Bl};
      RCG_CUDA_F(cudaLaunchCooperativeKernel((const void*)small_solve_kernel, dim3(small_G), dim3(kThreads), kargs, 0,
                                              c->stream));
      c->launches++;
    } else if (graph_ok) {
      // one graph per (shape, batch size): parameters are all device-resident
      char key[256];
      // (sharded: the halo plan enters by its device buffers and sizes, which the send / recv / pack nodes
      //  bake in, not by the host struct's address, which a later plan may reuse)
      snprintf(key, sizeof(key), "%p|%lld|%d|%d|%d|%d|%zu|%zu|%d|%d|%lld|%d|%d|%p|%p|%p|%lld|%lld|%lld", (void*)pre, (long long)n,
               spmv_width(A), nbs, nb, nbu, smem_upd, smem_pre, reorth ? 1 : 0, n_c > NC_INLINE ? 1 : 0,
               (long long)B, A->block + 100 * A->bsr_slice + 10000 * (A->dia_count * 4 + A->dia_block),
               A->row_offsets_64 + 2 * (int)ceil_div(n_c, 8) + (halo_overlap ? 1 << 20 : 0),
               (const void*)(H ? H->send_idx : nullptr), (const void*)(H ? H->send_buf : nullptr),
               (const void*)(H ? gSum.ptr : nullptr),   // the allreduce nodes' buffer (a per-solve pool block)
               (long long)(H ? H->n_ghost : 0), (long long)(H ? H->send_off[H->nranks] : 0),
               (long long)(H ? reo_cols() : 0));   // sharded: halo plan and allreduce width
      cudaGraphExec_t exec = nullptr;
      auto gi = c->graphs.find(key);
      if (gi != c->graphs.end()) {
        exec = gi->second.exec;
      } else {
        // bounded cache: evict the least recently used shape.  Every batch
        // ends with a stream synchronize, so no cached graph is in flight.
        if (c->graphs.size() >= Ctx::kMaxGraphs) {
          auto lru = c->graphs.begin();
          for (auto g = c->graphs.begin(); g != c->graphs.end(); ++g)
            if (g->second.last < lru->second.last) lru = g;
          cudaGraphExecDestroy(lru->second.exec);
          c->graphs.erase(lru);
        }
        cudaGraph_t graph = nullptr;
        // capture on a private stream (the caller's may be the legacy default
        // stream, which cannot capture); the graph is launched on c->stream
        if (!c->capture_stream) RCG_CUDA_F(cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking));
        cudaStream_t user_stream = c->stream;
        c->stream = c->capture_stream;
        cudaError_t ce = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) {
          c->stream = user_stream;
          return fail(set_error(c, RCG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce)));
        }
        const int64_t l0 = c->launches;
        int crc = launch_batch(B, it, false);
        ce = cudaStreamEndCapture(c->stream, &graph);
        c->stream = user_stream;
        if (crc) return fail(crc);
        if (ce != cudaSuccess) return fail(set_error(c, RCG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce)));
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(set_error(c, RCG_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce)));
        c->graphs[key] = Ctx::GraphEntry{exec, c->launches - l0, 0};
        c->launches = l0;
      }
      Ctx::GraphEntry& ge = c->graphs[key];
      ge.last = ++c->graph_tick;
      RCG_CUDA_F(cudaGraphLaunch(exec, c->stream));
      c->launches += ge.kernels;
    } else {
      if ((rc = launch_batch(B, it, true))) return fail(rc);
    }
    it += B;
    RCG_CUDA_F(cudaMemcpyAsync(hst, st, sizeof(SolveState), cudaMemcpyDeviceToHost, c->stream));
    RCG_CUDA_F(cudaStreamSynchronize(c->stream));
    done = hst->done != 0;
    prof_collect(c, done ? (hst->converged ? hst->iterations - 1 : hst->j) : -1);
    batch = std::min<int64_t>(batch * 2, small ? 4096 : 64);
  }
  cudaEventRecord(ev1, c->stream);
  RCG_CUDA_F(cudaMemcpyAsync(hst, st, sizeof(SolveState), cudaMemcpyDeviceToHost, c->stream));
  RCG_CUDA_F(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  T->view.device_seconds = ms * 1e-3;
  T->view.failure = hst->failure;
  T->view.converged = hst->converged;
  T->view.iterations = hst->converged ? hst->iterations : hst->j;
  if (hst->failure == RCG_FAIL_WAW) T->view.iterations = hst->j;
  T->view.n_betas = hst->converged ? T->view.iterations - 1 : hst->j;
  c->m_hint[n] = T->view.iterations;
  finish_view();
  *trace_out = T;
  if (hst->failure && getenv("RCG_DEBUG_FAIL")) {
    const int64_t jj = hst->j;
    std::vector<double> al(std::max<int64_t>(jj + 1, 1)), ww(std::max<int64_t>(jj + 1, 1));
    cudaMemcpy(al.data(), alphas, sizeof(double) * al.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(ww.data(), wawd, sizeof(double) * ww.size(), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[rcg debug] failure %d at j=%lld n=%lld n_c=%lld block=%d\n", hst->failure, (long long)jj,
            (long long)n, (long long)n_c, A->block);
    for (int64_t k = std::max<int64_t>(0, jj - 4); k <= jj; ++k)
      fprintf(stderr, "  k=%lld alpha=%.17g waw=%.17g\n", (long long)k, al[k], ww[k]);
  }
  if (hst->failure) {
    return set_error(c, RCG_ERR_NUMERICAL, "%s",
                     hst->failure == RCG_FAIL_RZ ? "(r, z) <= 0: preconditioner or operator not SPD"
                                                 : "(w, A w) <= 0: operator not SPD on search space");
  }
  return RCG_OK;
#undef RCG_CUDA_F
#undef RCG_LAUNCH_CHECK_F
}

extern "C" int rcg_apcg_solve(rcg_ctx* ctx, const rcg_csr* A, const double* inv_diag, const rcg_deflation* D,
                              const double* b, double* x, const rcg_solve_cfg* cfg, rcg_trace** trace_out) {
  return solve_impl(ctx, A, inv_diag, D, b, x, cfg, nullptr, trace_out);
}

extern "C" int rcg_apcg_solve_sharded(rcg_ctx* ctx, const rcg_csr* A, const double* inv_diag,
                                      const rcg_deflation* D, const double* b, double* x, const rcg_solve_cfg* cfg,
                                      const rcg_halo* halo, rcg_trace** trace_out) {
  if (!halo) return ctx ? set_error(ctx, RCG_ERR_CONTRACT, "sharded solve needs a halo plan") : RCG_ERR_CONTRACT;
  return solve_impl(ctx, A, inv_diag, D, b, x, cfg, halo, trace_out);
}

// ---------------------------------------------------------------------------
// deflation build / project / initial guess (solver.py:63-117)

static int deflation_build_impl(rcg_ctx* ctx, const rcg_csr* A, double* C, int64_t ldc, int64_t n_c, double* AC,
                                int64_t ldac, double* L, double* Ginv, const rcg_halo* H, int64_t* bad_col_host) {
  if (!ctx || !A) return RCG_ERR_CONTRACT;
  if (bad_col_host) *bad_col_host = -1;
  if (n_c == 0) return RCG_OK;
  Ctx* c = ctx;
  int rc = RCG_OK;
  if (H) {  // AC = A C column by column, each column's ghosts exchanged first
    for (int64_t k = 0; k < n_c && !rc; ++k) {
      double* col = C + k * ldc;
      rc = halo_exchange(c, H, colsel(col), nullptr, col);
      if (!rc) rc = rcg_spmv(ctx, A, col, AC + k * ldac);
    }
  } else {
    rc = rcg_spmm(ctx, A, C, ldc, n_c, AC, ldac);           // AC = A C
  }
  if (rc) return rc;
  double* G = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&G, sizeof(double) * (size_t)n_c * n_c, c->stream));
  rc = gemm_tn(c, A->n, n_c, n_c, C, ldc, AC, ldac, G, 1);   // 0.5 (C^T AC + (C^T AC)^T), local rows
  if (!rc) rc = allreduce_h(H, c, G, (size_t)(n_c * n_c));   // sum of the slabs' contributions
  if (!rc) {
    int64_t bad = -1;
    rc = cholesky(c, G, n_c, 1e-12, L, Ginv, &bad);        // pivot_rtol=1e-12 (solver.py:116)
    if (bad_col_host) *bad_col_host = bad;
  }
  cudaFreeAsync(G, c->stream);
  if (!rc) RCG_CUDA(c, cudaStreamSynchronize(c->stream));
  return rc;
}

extern "C" int rcg_deflation_build(rcg_ctx* ctx, const rcg_csr* A, const double* C, int64_t ldc, int64_t n_c,
                                   double* AC, int64_t ldac, double* L, double* Ginv, int64_t* bad_col_host) {
  return deflation_build_impl(ctx, A, (double*)C, ldc, n_c, AC, ldac, L, Ginv, nullptr, bad_col_host);
}

extern "C" int rcg_deflation_build_sharded(rcg_ctx* ctx, const rcg_csr* A, double* C, int64_t ldc, int64_t n_c,
                                           double* AC, int64_t ldac, double* L, double* Ginv, const rcg_halo* halo,
                                           int64_t* bad_col_host) {
  return deflation_build_impl(ctx, A, C, ldc, n_c, AC, ldac, L, Ginv, halo, bad_col_host);
}

extern "C" int rcg_project(rcg_ctx* ctx, const rcg_deflation* D, const double* x, double* out) {
  if (!ctx || !D) return RCG_ERR_CONTRACT;
  Ctx* c = ctx;
  if (D->n_c == 0) {
    RCG_CUDA(c, cudaMemcpyAsync(out, x, sizeof(double) * D->n, cudaMemcpyDeviceToDevice, c->stream));
    return RCG_OK;
  }
  double* u = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&u, sizeof(double) * (size_t)D->n_c, c->stream));
  int rc = gemv_t(c, D->n, D->n_c, D->AC, D->ldac, x, u);   // AC^T x
  if (!rc) rc = coarse_combine(c, D, u, x, out);            // x - C G^{-1} AC^T x
  cudaFreeAsync(u, c->stream);
  return rc;
}

extern "C" int rcg_initial_guess(rcg_ctx* ctx, const rcg_deflation* D, const double* b, double* x0) {
  if (!ctx || !D) return RCG_ERR_CONTRACT;
  Ctx* c = ctx;
  if (D->n_c == 0) {
    RCG_CUDA(c, cudaMemsetAsync(x0, 0, sizeof(double) * D->n, c->stream));
    return RCG_OK;
  }
  double* u = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&u, sizeof(double) * (size_t)D->n_c, c->stream));
  int rc = gemv_t(c, D->n, D->n_c, D->C, D->ldc, b, u);     // C^T b
  if (!rc) rc = coarse_combine(c, D, u, nullptr, x0);       // C G^{-1} C^T b
  cudaFreeAsync(u, c->stream);
  return rc;
}
