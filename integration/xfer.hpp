// Host <-> device copies of the reference's pageable std::vectors at PCIe rate
// (drop-in only: the reference's EvalContext hands the library plain
// std::vector<double> buffers, and a pageable cudaMemcpy runs at a fraction
// of the link's bandwidth).
//
// Each transfer is cut into chunks staged through a ring of page-locked
// buffers: while the DMA engine moves chunk i+1.., a small fork-join pool of
// host threads copies chunk i between the staging slot and the caller's
// memory. Registering the caller's vectors instead (cudaHostRegister) is not
// an option: EvalContext has no destructor the drop-in could hook, so the
// registration would outlive the memory.
#pragma once

#include <cuda_runtime.h>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace octrans_accel {

// Copy whose destination lines are written with non-temporal (streaming)
// stores: the destination is not read for ownership first and does not
// displace the staging ring from the last-level cache. Used for the
// staging -> caller copies of device-to-host transfers, whose destinations
// (the reference's COO vectors, tens of MB) are not read again by this
// process before the next evaluation overwrites them.
#if defined(__x86_64__)
__attribute__((target("avx2"))) inline void copy_nt_avx2(char* dst, const char* src, size_t bytes) {
  size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head > bytes) head = bytes;
  if (head) std::memcpy(dst, src, head);
  dst += head;
  src += head;
  bytes -= head;
  size_t i = 0;
  for (; i + 128 <= bytes; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  if (i < bytes) std::memcpy(dst + i, src + i, bytes - i);
  _mm_sfence();  // the streamed lines are visible before the caller's completion signal
}
inline bool have_avx2() {
  static const bool yes = __builtin_cpu_supports("avx2");
  return yes;
}
#endif
inline void copy_bytes(void* dst, const void* src, size_t bytes, bool nt) {
#if defined(__x86_64__)
  if (nt && have_avx2()) {
    copy_nt_avx2(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    return;
  }
#endif
  (void)nt;
  std::memcpy(dst, src, bytes);
}

// fork-join memcpy over T threads (the caller is one of them). A transfer
// hands the pool one chunk after another every few tens of microseconds, so
// the workers spin on the generation counter for a while after each chunk
// (a futex wake-up per chunk cost as much as the chunk's memcpy) and park on
// the condition variable only when the pool has been idle for kSpin.
class CopyPool {
 public:
  explicit CopyPool(int threads) {
    nthreads_ = threads;
    for (int t = 1; t < threads; ++t) workers_.emplace_back([this, t] { run(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true, std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void copy(void* dst, const void* src, size_t bytes, bool nt = false) {
    if (bytes < (size_t{1} << 18) || nthreads_ == 1) {
      copy_bytes(dst, src, bytes, nt);
      return;
    }
    nt_ = nt;
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    pending_.store(nthreads_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);  // orders the publication against a worker about to park
      gen_.fetch_add(1, std::memory_order_release);
    }
    if (parked_.load(std::memory_order_acquire) > 0) cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) != 0) pause();
  }

 private:
  static constexpr auto kSpin = std::chrono::microseconds(300);
  static void pause() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  void part(int t) {
    const size_t per = (bytes_ / nthreads_ + 63) & ~size_t{63};
    const size_t lo = std::min(bytes_, per * static_cast<size_t>(t)), hi = std::min(bytes_, lo + per);
    if (hi > lo) copy_bytes(dst_ + lo, src_ + lo, hi - lo, nt_);
  }
  void run(int t) {
    size_t seen = 0;
    for (;;) {
      auto t0 = std::chrono::steady_clock::now();
      int spins = 0;
      while (gen_.load(std::memory_order_acquire) == seen) {
        pause();
        if (++spins == 1024) {
          spins = 0;
          if (std::chrono::steady_clock::now() - t0 > kSpin) {
            std::unique_lock<std::mutex> lk(mu_);
            parked_.fetch_add(1, std::memory_order_acq_rel);
            cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
            parked_.fetch_sub(1, std::memory_order_acq_rel);
            t0 = std::chrono::steady_clock::now();
          }
        }
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load(std::memory_order_relaxed)) return;
      part(t);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  int nthreads_ = 1;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<size_t> gen_{0};
  std::atomic<int> pending_{0}, parked_{0};
  std::atomic<bool> stop_{false};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  bool nt_ = false;
  size_t bytes_ = 0;
};

class Xfer {
 public:
  static constexpr int kMaxSlots = 8;

  // chunk: doubles per staging slot; slots <= kMaxSlots
  // nt: bit 0 = streaming stores into the caller's memory on device-to-host
  // transfers, bit 1 = streaming stores into the staging slots on host-to-
  // device transfers
  Xfer(cudaStream_t s, int threads, size_t chunk, int slots, int nt = 1)
      : kChunk(chunk), kSlots(std::clamp(slots, 2, kMaxSlots)), nt_d2h_(nt & 1), nt_h2d_(nt & 2), stream_(s), pool_(threads) {
    for (int i = 0; i < kSlots; ++i) {
      ck(cudaMallocHost(&stage_[i], kChunk * sizeof(double)), "cudaMallocHost");
      ck(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming), "event");
    }
  }
  ~Xfer() {
    cudaStreamSynchronize(stream_);
    for (int i = 0; i < kSlots; ++i) {
      cudaFreeHost(stage_[i]);
      cudaEventDestroy(ev_[i]);
    }
  }
  Xfer(const Xfer&) = delete;
  Xfer& operator=(const Xfer&) = delete;

  // enqueue host -> device; returns once the host source has been consumed
  void h2d(double* ddst, const double* src, size_t n) {
    for (size_t off = 0; off < n; off += kChunk) {
      const size_t len = std::min(kChunk, n - off);
      const int s = next_slot();
      ck(cudaEventSynchronize(ev_[s]), "slot sync");  // the slot's previous DMA is done
      pool_.copy(stage_[s], src + off, len * sizeof(double), nt_h2d_);
      ck(cudaMemcpyAsync(ddst + off, stage_[s], len * sizeof(double), cudaMemcpyHostToDevice, stream_), "H2D");
      ck(cudaEventRecord(ev_[s], stream_), "record");
    }
  }

  struct Part {
    double* dst;
    const double* dsrc;
    size_t n;
  };
  // device -> host for several arrays in one pipeline; synchronous
  void d2h(const std::vector<Part>& parts) {
    struct Chunk {
      double* dst;
      const double* dsrc;
      size_t len;
    };
    std::vector<Chunk> ch;
    for (const Part& p : parts)
      for (size_t off = 0; off < p.n; off += kChunk) ch.push_back({p.dst + off, p.dsrc + off, std::min(kChunk, p.n - off)});
    std::vector<int> slot(ch.size());
    auto issue = [&](size_t i) {
      const int s = next_slot();
      slot[i] = s;
      ck(cudaMemcpyAsync(stage_[s], ch[i].dsrc, ch[i].len * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H");
      ck(cudaEventRecord(ev_[s], stream_), "record");
    };
    const size_t ahead = std::min<size_t>(kSlots, ch.size());
    for (size_t i = 0; i < ahead; ++i) issue(i);
    for (size_t i = 0; i < ch.size(); ++i) {
      ck(cudaEventSynchronize(ev_[slot[i]]), "D2H sync");
      pool_.copy(ch[i].dst, stage_[slot[i]], ch[i].len * sizeof(double), nt_d2h_);
      if (i + kSlots < ch.size()) issue(i + kSlots);
    }
  }

 private:
  static void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("octrans_accel xfer ") + what + ": " + cudaGetErrorString(e));
  }
  int next_slot() {
    const int s = slot_;
    slot_ = (slot_ + 1) % kSlots;
    return s;
  }
  const size_t kChunk;
  const int kSlots;
  const bool nt_d2h_, nt_h2d_;
  cudaStream_t stream_;
  CopyPool pool_;
  double* stage_[kMaxSlots] = {};
  cudaEvent_t ev_[kMaxSlots] = {};
  int slot_ = 0;
};

}  // namespace octrans_accel
