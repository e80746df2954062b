// Context management and error plumbing of the C ABI (include/rcg.h).
#include "rcg_internal.cuh"

#include <cstdlib>
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

int scratch(Ctx* c, size_t bytes, void** out) {
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

}  // namespace rcg

using namespace rcg;

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
  *out = c;
  return RCG_OK;
}

extern "C" void rcg_ctx_destroy(rcg_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  if (c->scratch) cudaFree(c->scratch);
  if (c->counters) cudaFree(c->counters);
  if (c->pinned) cudaFreeHost(c->pinned);
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
