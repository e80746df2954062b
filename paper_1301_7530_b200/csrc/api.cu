// Context management and error plumbing of the C ABI (include/rcg.h).
#include "rcg_internal.cuh"
#include "comm.cuh"
#include "vmm.cuh"

#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>
#include <cstring>

namespace rcg {

int set_error(Ctx* c, int code, const char* fmt, ...) {
  if (!c) return code;
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  c->err = buf;
  return code;
}

static bool pool_guard();
static void guard_release(void* p);
static void* guard_alloc(size_t bytes);

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RCG_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

int scratch(Ctx* c, size_t bytes, void** out) {
  if (pool_guard()) {  // exact size + canary per call (see Pool::get)
    if (c->scratch) guard_release(c->scratch);
    c->scratch = guard_alloc(bytes);
    c->scratch_bytes = bytes;
    if (!c->scratch) return set_error(c, RCG_ERR_OOM, "scratch allocation of %zu bytes failed", bytes);
    *out = c->scratch;
    return RCG_OK;
  }
  bytes = (bytes + 255) & ~(size_t)255;
  if (bytes > c->scratch_bytes) {
    if (c->scratch) cudaFreeAsync(c->scratch, c->stream);
    c->scratch = nullptr;
    size_t want = bytes > 2 * c->scratch_bytes ? bytes : 2 * c->scratch_bytes;
    cudaError_t e = cudaMallocAsync(&c->scratch, want, c->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c->scratch_bytes = 0;
      return set_error(c, RCG_ERR_OOM, "scratch allocation of %zu bytes failed", want);
    }
    c->scratch_bytes = want;
  }
  *out = c->scratch;
  return RCG_OK;
}

Pool::~Pool() { trim(); }

void Pool::trim() {
  std::lock_guard<std::mutex> g(mu);
  for (auto& kv : free_) cudaFree(kv.second);
  free_.clear();
  free_bytes = 0;
}

// RCG_POOL_EXACT=1: no pooling, exact-size cudaMalloc/cudaFree, so that
// compute-sanitizer memcheck sees every out-of-bounds access (debug runs)
static bool pool_exact() {
  static const bool e = [] {
    const char* v = getenv("RCG_POOL_EXACT");
    return v && atoi(v) != 0;
  }();
  return e;
}

// RCG_POOL_GUARD=1: exact-size allocations followed by a canary zone that is
// verified when the buffer is returned (and at context teardown): catches
// kernels writing past the end of a pooled buffer (debug runs; slow)
static bool pool_guard() {
  static const bool e = [] {
    const char* v = getenv("RCG_POOL_GUARD");
    return v && atoi(v) != 0;
  }();
  return e;
}
static constexpr size_t kGuard = 64 << 10;
static constexpr unsigned char kCanary = 0xA5;
static std::mutex g_guard_mu;
static std::map<void*, size_t> g_guarded;  // ptr -> requested bytes
static int64_t g_guard_violations = 0;

static void guard_check(void* p, size_t bytes) {
  std::vector<unsigned char> h(kGuard);
  cudaDeviceSynchronize();
  if (cudaMemcpy(h.data(), (char*)p + bytes, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  for (size_t i = 0; i < kGuard; ++i)
    if (h[i] != kCanary) {
      fprintf(stderr, "[rcg guard] write past the end of a %zu-byte pool buffer at +%zu bytes\n", bytes, i);
      ++g_guard_violations;
      if (getenv("RCG_POOL_GUARD_ABORT")) abort();
      return;
    }
}

extern "C" int64_t rcg_debug_guard_violations() {
  std::lock_guard<std::mutex> g(g_guard_mu);
  for (auto& kv : g_guarded) guard_check(kv.first, kv.second);
  return g_guard_violations;
}

static void* guard_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes + kGuard) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaDeviceSynchronize();
  cudaMemset((char*)p + bytes, kCanary, kGuard);
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> g(g_guard_mu);
  g_guarded[p] = bytes;
  return p;
}

static void guard_release(void* p) {
  std::lock_guard<std::mutex> g(g_guard_mu);
  auto it = g_guarded.find(p);
  if (it != g_guarded.end()) {
    guard_check(p, it->second);
    g_guarded.erase(it);
  }
  cudaFree(p);
}

void* Pool::get(size_t bytes) {
  if (pool_guard()) return guard_alloc(bytes);
  if (pool_exact()) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  bytes = (bytes + 4095) & ~(size_t)4095;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = free_.lower_bound(bytes);
    // best fit, but do not hand a huge idle block to a small request
    if (it != free_.end() && it->first <= 2 * bytes + ((size_t)64 << 20)) {
      void* p = it->second;
      free_bytes -= it->first;
      free_.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    trim();
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  return p;
}

void Pool::put(void* p, size_t bytes) {
  if (!p) return;
  if (pool_guard()) {
    guard_release(p);
    return;
  }
  if (pool_exact()) {
    cudaFree(p);
    return;
  }
  bytes = (bytes + 4095) & ~(size_t)4095;
  std::lock_guard<std::mutex> g(mu);
  free_.emplace(bytes, p);
  free_bytes += bytes;
  while (free_bytes > keep_bytes && !free_.empty()) {
    auto it = std::prev(free_.end());
    cudaFree(it->second);
    free_bytes -= it->first;
    free_.erase(it);
  }
}

static cudaEvent_t pool_get(Ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(Ctx* c, int kclass, double bytes, int64_t jj) {
  if (!c->profiling) return;
  Ctx::Pending p;
  p.kclass = kclass;
  p.bytes = bytes;
  p.jj = jj;
  p.a = pool_get(c);
  p.b = pool_get(c);
  cudaEventRecord(p.a, c->stream);
  c->pending.push_back(p);
}

void prof_end(Ctx* c) {
  if (!c->profiling || c->pending.empty()) return;
  cudaEventRecord(c->pending.back().b, c->stream);
}

void prof_collect(Ctx* c, int64_t stop_j) {
  for (auto& p : c->pending) {
    float ms = 0.f;
    const bool late = p.kclass == RCG_K_PRECOND || p.kclass == RCG_K_COLREDUCE || p.kclass == RCG_K_WUPDATE;
    const bool noop = stop_j >= 0 && p.jj >= 0 && (p.jj > stop_j || (p.jj == stop_j && late));
    if (noop) {
      // queued after the solve stopped: returned at the done flag, no bytes moved
    } else if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      c->stats[p.kclass].launches += 1;
      c->stats[p.kclass].seconds += ms * 1e-3;
      c->stats[p.kclass].bytes += p.bytes;
    } else {
      cudaGetLastError();
    }
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.clear();
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_ctx_set_profiling(rcg_ctx* c, int enable) {
  if (!c) return RCG_ERR_CONTRACT;
  c->profiling = enable ? 1 : 0;
  return RCG_OK;
}

extern "C" int rcg_ctx_kernel_stats(const rcg_ctx* c, rcg_kernel_stat* out, int n) {
  if (!c || !out) return RCG_ERR_CONTRACT;
  for (int i = 0; i < n && i < RCG_K_NUM; ++i) out[i] = c->stats[i];
  return RCG_OK;
}

extern "C" int rcg_ctx_reset_stats(rcg_ctx* c) {
  if (!c) return RCG_ERR_CONTRACT;
  for (int i = 0; i < RCG_K_NUM; ++i) c->stats[i] = rcg_kernel_stat{0, 0.0, 0.0};
  return RCG_OK;
}

extern "C" int rcg_version(void) { return 1; }

extern "C" int rcg_ctx_create(int device, void* stream, rcg_ctx** out) {
  if (!out) return RCG_ERR_CONTRACT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return RCG_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return RCG_ERR_CUDA;
  rcg_ctx* c = new rcg_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
  }
  if (cudaMalloc((void**)&c->counters, sizeof(unsigned int) * c->n_counters) != cudaSuccess ||
      cudaMemset(c->counters, 0, sizeof(unsigned int) * c->n_counters) != cudaSuccess ||
      cudaMallocHost((void**)&c->pinned, 4096) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return RCG_ERR_CUDA;
  }
  c->chunks = std::make_shared<ChunkPool>();
  c->chunks->device = device;
  c->vpool = std::make_shared<VmmPool>();
  *out = c;
  return RCG_OK;
}

extern "C" void rcg_ctx_destroy(rcg_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  comm_free(c);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.second.exec);
  if (c->dargs) cudaFree(c->dargs);
  if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
  if (c->halo_stream) cudaStreamDestroy(c->halo_stream);
  if (c->halo_fork) cudaEventDestroy(c->halo_fork);
  if (c->halo_join) cudaEventDestroy(c->halo_join);
  if (c->scratch) {
    if (pool_guard()) guard_release(c->scratch);
    else cudaFree(c->scratch);
  }
  if (c->counters) cudaFree(c->counters);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  delete c;
}

extern "C" int rcg_ctx_set_stream(rcg_ctx* c, void* stream) {
  if (!c) return RCG_ERR_CONTRACT;
  if ((cudaStream_t)stream != c->stream) {
    cudaStreamSynchronize(c->stream);  // scratch is stream-ordered on the old stream
    c->stream = (cudaStream_t)stream;
  }
  return RCG_OK;
}

extern "C" const char* rcg_last_error(const rcg_ctx* c) { return c ? c->err.c_str() : "null context"; }

extern "C" int rcg_num_kernel_launches(const rcg_ctx* c, int64_t* out) {
  if (!c || !out) return RCG_ERR_CONTRACT;
  *out = c->launches;
  return RCG_OK;
}
