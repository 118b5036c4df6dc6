// Device memory for plans and solver state (library-internal): a bounded
// process-wide cache of large blocks in front of a PRIVATE stream-ordered
// pool per device, plus the device-scope guard every entry point uses.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace ocg::mem {

// Makes `dev` current for the scope of an entry point and restores the
// caller's device afterwards (contexts on several GPUs in one process).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

// SMs of the current device (cached per device).
inline int sm_count() {
  static std::mutex mu;
  static std::map<int, int>* n = new std::map<int, int>;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = n->find(dev);
  if (it != n->end()) return it->second;
  int c = 0;
  if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0) c = 148;
  n->emplace(dev, c);
  return c;
}

// The library's own pool per device: what is freed stays mapped (release
// threshold = max), so rebuilding a plan is not paid in page mappings, and
// the device's DEFAULT pool (shared with the rest of the process) is left
// alone. ocg_release_cached_memory() trims it.
inline cudaMemPool_t pool_for(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t>* pools = new std::map<int, cudaMemPool_t>;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools->find(dev);
  if (it != pools->end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceGetDefaultMemPool(&pool, dev);  // fall back to the default pool, threshold untouched
  } else {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  pools->emplace(dev, pool);
  return pool;
}

// Device blocks of at least kCacheMin bytes go back to a process-wide cache
// instead of the pool, and later allocations of (nearly) the same size take
// them from there. A solve rebuilds plans of the same sizes every time;
// through the pool alone, fragmentation now and then made it map fresh
// physical memory, and plan building took up to seconds longer at random.
// - Blocks are filed under the device that OWNS them (pointer attributes),
//   not whichever device is current when they are freed.
// - A freed block may still be read by work queued on any stream, so it is
//   marked pending; the first reuse of a pending block synchronizes its
//   device once (freeing never synchronizes).
// - The cache is bounded (OCG_CACHE_MAX_MB, default 8192 MiB per device);
//   blocks beyond the bound go back to the pool (after a device sync).
constexpr size_t kCacheMin = size_t{4} << 20;

struct CachedBlock {
  void* p;
  bool pending;
};
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, CachedBlock> blocks;  // (device, bytes) -> block
  std::map<int, size_t> bytes_held;
};
inline BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // never destroyed: outlives static DBufs
  return *c;
}
inline size_t cache_limit() {
  static const size_t lim = [] {
    const char* e = std::getenv("OCG_CACHE_MAX_MB");
    const long long mb = e ? std::atoll(e) : 8192;
    return static_cast<size_t>(std::max(0LL, mb)) << 20;
  }();
  return lim;
}
inline int owner_device(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice) return a.device;
  cudaGetLastError();
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
inline void* cache_take(size_t bytes, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.blocks.lower_bound({dev, bytes});
  if (it == c.blocks.end() || it->first.first != dev || it->first.second > bytes + bytes / 4) return nullptr;
  if (it->second.pending) {
    // work queued before the block was freed may still use it: settle the
    // device once, which settles every pending block of it
    cudaDeviceSynchronize();
    for (auto jt = c.blocks.lower_bound({dev, 0}); jt != c.blocks.end() && jt->first.first == dev; ++jt)
      jt->second.pending = false;
  }
  void* p = it->second.p;
  *got = it->first.second;
  c.bytes_held[dev] -= *got;
  c.blocks.erase(it);
  return p;
}
inline void cache_put(void* p, size_t bytes) {
  const int dev = owner_device(p);
  auto& c = block_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.bytes_held[dev] + bytes <= cache_limit()) {
      c.blocks.emplace(std::make_pair(dev, bytes), CachedBlock{p, true});
      c.bytes_held[dev] += bytes;
      return;
    }
  }
  DeviceScope ds(dev);
  cudaDeviceSynchronize();  // over the bound: back to the pool once no queued work can use it
  cudaFreeAsync(p, cudaStreamPerThread);
}
// Every cached block of `dev` (all devices if dev < 0) back to the pool, and
// the pool trimmed: the memory returns to the driver.
inline void cache_flush(int dev) {
  auto& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  std::map<int, bool> touched;
  for (auto it = c.blocks.begin(); it != c.blocks.end();) {
    if (dev < 0 || it->first.first == dev) {
      const int d = it->first.first;
      DeviceScope ds(d);
      if (!touched[d]) {
        cudaDeviceSynchronize();
        touched[d] = true;
      }
      cudaFree(it->second.p);
      c.bytes_held[d] -= it->first.second;
      it = c.blocks.erase(it);
    } else {
      ++it;
    }
  }
}
inline void trim(int dev) {
  cache_flush(dev);
  int n = 0;
  cudaGetDeviceCount(&n);
  for (int d = 0; d < n; ++d) {
    if (dev >= 0 && d != dev) continue;
    DeviceScope ds(d);
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool_for(d), 0);
  }
}
// *p: a device block of `bytes` on the current device (cached when large);
// *cap: the block's size
inline cudaError_t device_alloc(size_t bytes, void** p, size_t* cap) {
  bytes = std::max<size_t>(bytes, 1);
  *cap = bytes;
  *p = nullptr;
  if (bytes >= kCacheMin)
    if ((*p = cache_take(bytes, cap))) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaMallocFromPoolAsync(p, bytes, pool_for(dev), cudaStreamPerThread);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cache_flush(dev);
    e = cudaMallocFromPoolAsync(p, bytes, pool_for(dev), cudaStreamPerThread);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(cudaStreamPerThread);
}
inline void device_free(void* p, size_t cap) {
  if (!p) return;
  if (cap >= kCacheMin) {
    cache_put(p, cap);
  } else {
    DeviceScope ds(owner_device(p));
    cudaFreeAsync(p, cudaStreamPerThread);  // stream-ordered: no device-wide sync
  }
}

}  // namespace ocg::mem
