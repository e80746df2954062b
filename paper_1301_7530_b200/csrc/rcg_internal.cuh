// Internal helpers shared by the rcg CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <cstdio>
#include <cstdarg>
#include <vector>
#include <map>
#include <memory>
#include <mutex>

#include "../../include/rcg.h"

namespace rcg {

constexpr int kThreads = 256;           // default CTA size for streaming kernels
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// device buffer pool: Krylov histories are GBs per solve; recycling them
// across the solves of a sequence avoids cudaMalloc/cudaFree of multi-GB
// blocks (and the geometric-growth copies) on every system.  Shared by the
// context and the traces it hands out (a trace may outlive its context).

struct Pool {
  std::mutex mu;
  std::multimap<size_t, void*> free_;
  size_t free_bytes = 0;
  size_t keep_bytes = (size_t)96 << 30;  // cap on idle pooled memory
  ~Pool();
  void* get(size_t bytes);               // nullptr on OOM
  void put(void* p, size_t bytes);
  void trim();
};

struct Comm;       // comm.cu
struct ChunkPool;  // vmm.cuh
struct VmmPool;    // vmm.cuh

// ---------------------------------------------------------------------------
// context

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  std::string err;
  int64_t launches = 0;
  // generic scratch (grown on demand; stream-ordered)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  unsigned int* counters = nullptr;     // zero-initialised last-block counters
  int n_counters = 64;
  double* pinned = nullptr;             // small pinned host staging buffer
  // live kernel timing (rcg_ctx_set_profiling)
  int profiling = 0;
  rcg_kernel_stat stats[RCG_K_NUM] = {};
  struct Pending {
    int kclass;
    double bytes;
    int64_t jj;   // solve-loop iteration the launch was queued for (-1: not a loop launch)
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::shared_ptr<Pool> pool = std::make_shared<Pool>();
  std::shared_ptr<ChunkPool> chunks;     // physical chunks of the VA-range histories
  std::shared_ptr<VmmPool> vpool;        // whole mapped history ranges kept across solves
  std::map<int64_t, int64_t> m_hint;     // n -> iterations of the last solve
  Comm* comm = nullptr;                  // NCCL communicator (sharded runs)
  double* halo_recv = nullptr;           // received ghosts, unpacked into the column at device j
  size_t halo_recv_cap = 0;
  void* dargs = nullptr;                 // device-resident solve arguments (graph replay)
  cudaStream_t capture_stream = nullptr; // private stream for graph capture
  cudaStream_t halo_stream = nullptr;    // sharded: the halo exchange runs here beside the local SpMV
  cudaEvent_t halo_fork = nullptr, halo_join = nullptr;
  struct GraphEntry {
    cudaGraphExec_t exec;
    int64_t kernels;   // kernel launches one replay stands for
    uint64_t last;     // use tick (LRU eviction)
  };
  std::map<std::string, GraphEntry> graphs;   // batch shape -> executable graph
  uint64_t graph_tick = 0;
  static constexpr size_t kMaxGraphs = 48;    // TRKS (n_c grows every system) keeps adding shapes
};

// Brackets a launch with events when profiling; `collect` (after a stream
// sync) folds the elapsed times into the per-class stats.
void prof_begin(Ctx* c, int kclass, double bytes, int64_t jj = -1);
void prof_end(Ctx* c);
// stop_j >= 0: the solve stopped in iteration stop_j; launches queued for later
// iterations (and the precond / colreduce / w-update launches of stop_j itself,
// which return at their `done` test) were no-ops and are not counted
void prof_collect(Ctx* c, int64_t stop_j = -1);

int set_error(Ctx* c, int code, const char* fmt, ...);

#define RCG_CUDA(ctx, call)                                                   \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return ::rcg::set_error((ctx), RCG_ERR_CUDA, "%s: %s (%s:%d)", #call,   \
                              cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

#define RCG_LAUNCH_CHECK(ctx)                                                 \
  do {                                                                        \
    (ctx)->launches++;                                                        \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess)                                                    \
      return ::rcg::set_error((ctx), RCG_ERR_CUDA, "launch: %s (%s:%d)",      \
                              cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

// scratch of at least `bytes` (device, 256-B aligned); invalidates earlier pointers
int scratch(Ctx* c, size_t bytes, void** out);

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): the iteration kernels are launched
// with programmatic stream serialization, so a kernel's CTAs are scheduled
// while the previous kernel's last CTA (its fixed-order reduction) is still
// running; every such kernel starts with pdl_wait() (griddepcontrol.wait),
// which blocks until the previous grid has completed and its writes are
// visible -- the same ordering as a plain stream launch, minus the launch
// latency.  griddepcontrol.wait is a no-op for a normally launched grid.
// RCG_PDL=0 launches plainly.

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum; result valid in thread 0 (and returned to all via smem).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sm /* >= NT/32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < NT / 32 ? sm[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sm[0] = t;
  }
  __syncthreads();
  t = sm[0];
  __syncthreads();
  return t;
}

// Last-block-done: every block has written its K partials to part[blockIdx*K+k];
// returns true in exactly one block (the last to arrive), after which that
// block may read all partials.  The counter is reset by the last block.
// The barrier orders every thread's partial writes before thread 0's fence
// (fence.sc is cumulative), so only thread 0 fences: the other threads do not
// stall on the completion of their own streaming stores.
__device__ __forceinline__ bool arrive_last(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
    if (last) *counter = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// sum of p[b * stride] over b = lane, lane + 32, ... < nb, added in exactly
// that order (so the same bits as the plain loop); the loads of 8 steps are
// issued before their adds: in the last-block tails below a plain loop waits
// one L2 round trip per step
__device__ __forceinline__ double lane_strided_sum(const double* p, int nb, int64_t stride, int lane) {
  double s = 0.0;
  int b = lane;
  for (; b + 32 * 7 < nb; b += 32 * 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)(b + 32 * u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; b < nb; b += 32) s += __ldcg(p + (size_t)b * stride);
  return s;
}

// Deterministic reduction of part[b*K + k] over b < nb for k < K into out[k]
// by one block of NT threads: warps own k's; lanes stride over blocks in a
// fixed order then a fixed shuffle tree.
template <int NT>
__device__ void reduce_partials(const double* part, int nb, int K, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = wid; k < K; k += NT / 32) {
    double s = lane_strided_sum(part + k, nb, K, lane);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
}

// as reduce_partials, for `count` values at stride `stride` in each partial row
template <int NT>
__device__ void reduce_partials_strided(const double* part, int nb, int stride, int count, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = wid; k < count; k += NT / 32) {
    double s = lane_strided_sum(part + k, nb, stride, lane);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t pad_ld(int64_t n) { return ceil_div(n, 32) * 32; }

// A column of a column-major history buffer chosen by the device-side
// iteration counter: column (j + shift) (mod `mod` when mod > 0).
// (clamp > 0: columns >= clamp all map to column `clamp`, a scratch column
// past a capped history)
struct ColSel {
  double* base;
  int64_t ld;
  int64_t mod;
  int64_t shift;
  int64_t clamp;
  __device__ __forceinline__ double* at(long long j) const {
    long long c = j + shift;
    if (mod > 0) c %= mod;
    if (clamp > 0 && c > clamp) c = clamp;
    return base + (int64_t)c * ld;
  }
};

__host__ __forceinline__ ColSel colsel(double* base, int64_t ld = 0, int64_t mod = 1, int64_t shift = 0,
                                       int64_t clamp = 0) {
  ColSel s;
  s.base = base;
  s.ld = ld;
  s.mod = mod;
  s.shift = shift;
  s.clamp = clamp;
  return s;
}

// Device-resident solve state (one per apcg_solve), read by every kernel of
// the iteration so that a batch of iterations can be queued (or graph-
// replayed) with identical launch parameters and no host round trip.
struct SolveState {
  long long j;          // index of the current direction w_j
  long long iterations; // m so far
  int done;             // converged / failed: every later kernel is a no-op
  int converged;
  int failure;          // rcg_failure
  int pad;
  double rz;            // (r_j, z_j)
  double tol_abs;       // tol * ||r0||
};

// row-offset load for int32/int64 CSR
template <typename RO>
__device__ __forceinline__ int64_t ro_at(const RO* ro, int64_t i) { return (int64_t)__ldg(ro + i); }

}  // namespace rcg

struct rcg_ctx : public rcg::Ctx {};
