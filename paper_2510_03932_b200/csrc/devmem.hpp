// Device memory for plans and solver state (library-internal): a
// process-wide cache of large blocks in front of the stream-ordered pool.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <map>
#include <mutex>
#include <utility>

namespace ocg::mem {

// Device blocks of at least kCacheMin bytes go back to a process-wide cache
// instead of the stream-ordered pool, and later allocations of (nearly) the
// same size take them from there. A solve rebuilds plans of the same sizes
// every time; through the pool alone, fragmentation now and then made it map
// fresh physical memory (zeroed by the driver), and plan building took up to
// seconds longer at random. Blocks enter the cache after a device
// synchronization, so no stream still uses them; when an allocation fails the
// cache is returned to the pool and the allocation retried.
constexpr size_t kCacheMin = size_t{4} << 20;

struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> blocks;  // (device, bytes) -> block
};
inline BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // never destroyed: outlives static DBufs
  return *c;
}
inline void* cache_take(size_t bytes, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.blocks.lower_bound({dev, bytes});
  if (it == c.blocks.end() || it->first.first != dev || it->first.second > bytes + bytes / 4) return nullptr;
  void* p = it->second;
  *got = it->first.second;
  c.blocks.erase(it);
  return p;
}
inline void cache_put(void* p, size_t bytes) {
  cudaDeviceSynchronize();
  int dev = 0;
  cudaGetDevice(&dev);
  auto& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.blocks.emplace(std::make_pair(dev, bytes), p);
}
inline void cache_flush() {
  auto& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto it = c.blocks.begin(); it != c.blocks.end();) {
    if (it->first.first == dev) {
      cudaFreeAsync(it->second, cudaStreamPerThread);
      it = c.blocks.erase(it);
    } else {
      ++it;
    }
  }
  cudaStreamSynchronize(cudaStreamPerThread);
}
// *p: a device block of `bytes` (cached when large); *cap: the block's size
inline cudaError_t device_alloc(size_t bytes, void** p, size_t* cap) {
  bytes = std::max<size_t>(bytes, 1);
  *cap = bytes;
  *p = nullptr;
  if (bytes >= kCacheMin)
    if ((*p = cache_take(bytes, cap))) return cudaSuccess;
  cudaError_t e = cudaMallocAsync(p, bytes, cudaStreamPerThread);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cache_flush();
    e = cudaMallocAsync(p, bytes, cudaStreamPerThread);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(cudaStreamPerThread);
}
inline void device_free(void* p, size_t cap) {
  if (!p) return;
  if (cap >= kCacheMin)
    cache_put(p, cap);
  else
    cudaFreeAsync(p, cudaStreamPerThread);  // stream-ordered: no device-wide sync
}

}  // namespace ocg::mem
