// Growable device buffers on CUDA virtual memory: one VA range is reserved
// up front and physical chunks are mapped behind it on demand, so a Krylov
// history grows without copies and without the 1.5-2x peak of
// allocate-copy-free growth (histories are the HBM budget).
// Physical chunks are recycled through a per-context pool across solves.
#pragma once
#include <cuda.h>

#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace rcg {

struct ChunkPool {
  int device = 0;
  std::mutex mu;
  std::multimap<size_t, CUmemGenericAllocationHandle> free_;  // size -> handle
  size_t free_bytes = 0;
  size_t keep_bytes = (size_t)64 << 30;
  ~ChunkPool();
  bool get(size_t bytes, CUmemGenericAllocationHandle* h);
  void put(size_t bytes, CUmemGenericAllocationHandle h);
  void trim();
};

struct VmmBuf {
  CUdeviceptr base = 0;
  size_t reserved = 0;
  size_t mapped = 0;
  size_t chunk = 0;
  int device = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  std::shared_ptr<ChunkPool> pool;
  // reserve max_bytes of VA; chunk = physical mapping granule for this buffer
  bool reserve(std::shared_ptr<ChunkPool> p, int dev, size_t max_bytes, size_t chunk_hint);
  bool ensure(size_t bytes);  // map chunks until >= bytes are backed
  void release();             // unmap, return chunks to the pool, free the VA
  double* ptr() const { return (double*)base; }
};

// Whole mapped VA ranges kept across solves: a sequence re-solves the same
// shape, so the next solve re-uses the previous histories' mappings as is.
struct VmmPool {
  std::mutex mu;
  std::vector<VmmBuf> bufs;
  size_t mapped_total = 0;
  size_t keep_bytes = (size_t)96 << 30;
  ~VmmPool() { clear(); }
  bool take(size_t chunk, size_t reserved, VmmBuf* out);
  void give(VmmBuf& b);  // takes ownership (b is reset)
  void clear();
};

bool vmm_available();
size_t vmm_granularity(int device);

}  // namespace rcg
