// CUDA virtual-memory growable buffers (see vmm.cuh).  Driver entry points
// are resolved through cudaGetDriverEntryPoint, so librcg.so does not link
// libcuda (it still loads in the GPU-less build container).
#include "rcg_internal.cuh"
#include "vmm.cuh"

#include <algorithm>

namespace rcg {

namespace {

struct Api {
  bool ok = false;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
};

Api* api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess &&
             *fn != nullptr;
    };
    bool ok = true;
    ok &= get("cuMemAddressReserve", (void**)&a.reserve);
    ok &= get("cuMemAddressFree", (void**)&a.addrFree);
    ok &= get("cuMemCreate", (void**)&a.create);
    ok &= get("cuMemRelease", (void**)&a.release);
    ok &= get("cuMemMap", (void**)&a.map);
    ok &= get("cuMemUnmap", (void**)&a.unmap);
    ok &= get("cuMemSetAccess", (void**)&a.setAccess);
    ok &= get("cuMemGetAllocationGranularity", (void**)&a.granularity);
    a.ok = ok;
    if (!ok) cudaGetLastError();
  });
  return &a;
}

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  return p;
}

}  // namespace

bool vmm_available() { return api()->ok; }

size_t vmm_granularity(int device) {
  Api* a = api();
  size_t g = (size_t)2 << 20;
  if (!a->ok) return g;
  CUmemAllocationProp p = prop_for(device);
  size_t r = 0;
  if (a->granularity(&r, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && r) g = r;
  return g;
}

ChunkPool::~ChunkPool() { trim(); }

void ChunkPool::trim() {
  std::lock_guard<std::mutex> l(mu);
  for (auto& kv : free_) api()->release(kv.second);
  free_.clear();
  free_bytes = 0;
}

bool ChunkPool::get(size_t bytes, CUmemGenericAllocationHandle* h) {
  {
    std::lock_guard<std::mutex> l(mu);
    auto it = free_.find(bytes);
    if (it != free_.end()) {
      *h = it->second;
      free_.erase(it);
      free_bytes -= bytes;
      return true;
    }
  }
  CUmemAllocationProp p = prop_for(device);
  if (api()->create(h, bytes, &p, 0) == CUDA_SUCCESS) return true;
  trim();  // idle chunks of other sizes, then retry once
  return api()->create(h, bytes, &p, 0) == CUDA_SUCCESS;
}

void ChunkPool::put(size_t bytes, CUmemGenericAllocationHandle h) {
  std::lock_guard<std::mutex> l(mu);
  if (free_bytes + bytes > keep_bytes) {
    api()->release(h);
    return;
  }
  free_.emplace(bytes, h);
  free_bytes += bytes;
}

bool VmmBuf::reserve(std::shared_ptr<ChunkPool> p, int dev, size_t max_bytes, size_t chunk_hint) {
  Api* a = api();
  if (!a->ok) return false;
  pool = std::move(p);
  device = dev;
  const size_t g = vmm_granularity(dev);
  chunk = std::max(g, ((chunk_hint + g - 1) / g) * g);
  reserved = ((std::max<size_t>(max_bytes, 1) + chunk - 1) / chunk) * chunk;
  if (a->reserve(&base, reserved, g, 0, 0) != CUDA_SUCCESS) {
    base = 0;
    reserved = 0;
    return false;
  }
  return true;
}

bool VmmBuf::ensure(size_t bytes) {
  Api* a = api();
  if (bytes > reserved) return false;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  while (mapped < bytes) {
    CUmemGenericAllocationHandle h;
    if (!pool->get(chunk, &h)) return false;
    if (a->map(base + mapped, chunk, 0, h, 0) != CUDA_SUCCESS) {
      pool->put(chunk, h);
      return false;
    }
    if (a->setAccess(base + mapped, chunk, &acc, 1) != CUDA_SUCCESS) {
      a->unmap(base + mapped, chunk);
      pool->put(chunk, h);
      return false;
    }
    handles.push_back(h);
    mapped += chunk;
  }
  return true;
}

void VmmBuf::release() {
  Api* a = api();
  if (!base) return;
  for (size_t k = 0; k < handles.size(); ++k) a->unmap(base + k * chunk, chunk);
  for (auto h : handles) pool->put(chunk, h);
  handles.clear();
  a->addrFree(base, reserved);
  base = 0;
  mapped = reserved = 0;
}

bool VmmPool::take(size_t chunk, size_t reserved, VmmBuf* out) {
  std::lock_guard<std::mutex> l(mu);
  for (size_t i = 0; i < bufs.size(); ++i) {
    if (bufs[i].chunk == chunk && bufs[i].reserved == reserved) {
      *out = bufs[i];
      mapped_total -= bufs[i].mapped;
      bufs.erase(bufs.begin() + i);
      return true;
    }
  }
  return false;
}

void VmmPool::give(VmmBuf& b) {
  if (!b.base) return;
  {
    std::lock_guard<std::mutex> l(mu);
    if (mapped_total + b.mapped <= keep_bytes) {
      mapped_total += b.mapped;
      bufs.push_back(b);
      b = VmmBuf();
      return;
    }
  }
  b.release();
  b = VmmBuf();
}

void VmmPool::clear() {
  std::vector<VmmBuf> v;
  {
    std::lock_guard<std::mutex> l(mu);
    v.swap(bufs);
    mapped_total = 0;
  }
  for (auto& b : v) b.release();
}

}  // namespace rcg
