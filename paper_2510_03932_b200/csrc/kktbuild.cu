// KKT pattern and gather maps built on the device (KktAssembler's
// constructor, proj/src/ipm/eval.cpp:318-427, as sorts instead of host loops).
//
// Every structural source (Hessian entry, Jacobian entry, slack -1, primal
// diagonal, dual diagonal) becomes a (col, row) key with its source code; a
// stable radix sort by key puts them in the reference's (col, row) CSC order
// with codes ascending within a slot — exactly the accumulation order of
// KktAssembler::assemble. Slots are the runs of equal keys. The full
// symmetric CSR used by the matvec and the per-column J^T lambda gather are
// built the same way. All integer work, deterministic (no floating point).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "devmem.hpp"
#include "kktbuild.hpp"

namespace ocg::dev {

namespace {

#define GRID_LOOP(i, n)                                                                  \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

constexpr unsigned long long kNone = ~0ull;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("kkt build: ") + what + ": " + cudaGetErrorString(e));
}

int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<int>(want < 1 ? 1 : (want > 148 * 32 ? 148 * 32 : want));
}

// blocks through the device block cache (devmem.hpp); their sizes are kept
// so temporaries go back to the cache, outputs are handed over (forget)
std::mutex g_cap_mu;
std::unordered_map<void*, size_t> g_caps;

template <class T>
T* dalloc(size_t n, cudaStream_t) {
  void* p = nullptr;
  size_t cap = 0;
  ck(ocg::mem::device_alloc((n ? n : 1) * sizeof(T), &p, &cap), "cudaMallocAsync");
  std::lock_guard<std::mutex> lk(g_cap_mu);
  g_caps[p] = cap;
  return static_cast<T*>(p);
}
void dfree(void* p) {
  if (!p) return;
  size_t cap = 0;
  {
    std::lock_guard<std::mutex> lk(g_cap_mu);
    auto it = g_caps.find(p);
    if (it != g_caps.end()) {
      cap = it->second;
      g_caps.erase(it);
    }
  }
  if (cap)
    ocg::mem::device_free(p, cap);
  else
    cudaFreeAsync(p, cudaStreamPerThread);
}
// an output adopted by the caller (freed with cudaFreeAsync)
void forget(void* p) {
  std::lock_guard<std::mutex> lk(g_cap_mu);
  g_caps.erase(p);
}

// sources -> (key, code); invalid (folded/fixed) sources get kNone
__global__ void keys_k(const int64_t* __restrict__ hr, const int64_t* __restrict__ hc, int64_t H,
                       const int64_t* __restrict__ jr, const int64_t* __restrict__ jc, int64_t J,
                       const int64_t* __restrict__ prim, const int64_t* __restrict__ dual,
                       const int64_t* __restrict__ slack_dual, int64_t nfree, int64_t S, int64_t ntot, int64_t m,
                       unsigned long long* __restrict__ key, int64_t* __restrict__ code) {
  const int64_t C = H + J + S + ntot + m;
  GRID_LOOP(q, C) {
    long long col = -1, row = -1;
    if (q < H) {
      const int64_t pi = prim[hr[q]], pj = prim[hc[q]];
      if (pi >= 0 && pj >= 0) {
        col = pi < pj ? pi : pj;
        row = pi < pj ? pj : pi;
      }
    } else if (q < H + J) {
      const int64_t e = q - H;
      const int64_t d = dual[jr[e]], pj = prim[jc[e]];
      if (d >= 0 && pj >= 0) {
        col = pj;
        row = ntot + d;
      }
    } else if (q < H + J + S) {
      const int64_t k = q - H - J;
      col = nfree + k;
      row = ntot + slack_dual[k];
    } else if (q < H + J + S + ntot) {
      col = row = q - H - J - S;
    } else {
      col = row = ntot + (q - H - J - S - ntot);  // dual diagonal: zero source
    }
    key[q] = col < 0 ? kNone : (static_cast<unsigned long long>(col) << 32) | static_cast<unsigned long long>(row);
    code[q] = q;  // source codes are the source ordinals (assemble: H, J, -1, sigma, 0)
  }
}

__global__ void fresh_k(const unsigned long long* __restrict__ key, int64_t n, int64_t* __restrict__ flag) {
  GRID_LOOP(i, n) flag[i] = (key[i] != kNone && (i == 0 || key[i] != key[i - 1])) ? 1 : 0;
}

// slot-level outputs from the sorted sources: rowi, src_ptr, per-column counts
__global__ void slots_k(const unsigned long long* __restrict__ key, const int64_t* __restrict__ slot_incl,
                        int64_t n, int64_t* __restrict__ rowi, int64_t* __restrict__ src_ptr,
                        int* __restrict__ colcnt) {
  GRID_LOOP(i, n) {
    if (key[i] == kNone) continue;
    if (i == 0 || key[i] != key[i - 1]) {
      const int64_t s = slot_incl[i] - 1;
      rowi[s] = static_cast<int64_t>(key[i] & 0xffffffffull);
      src_ptr[s] = i;
      atomicAdd(&colcnt[key[i] >> 32], 1);
    }
  }
}

// column of CSC entry q by binary search: the mirror is built one thread per
// entry, so a dense column (a free final time's) is not one thread's loop
__device__ __forceinline__ int64_t col_of(const int64_t* __restrict__ colp, int64_t dim, int64_t q) {
  int64_t lo = 0, hi = dim;  // colp[lo] <= q < colp[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (colp[mid] <= q)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// mirrored entries of the lower CSC for the full symmetric CSR: entry p gives
// keys (row, col) at 2p and, off the diagonal, (col, row) at 2p + 1 (kNone on
// the diagonal: sorts last and is cut off)
__global__ void mirror_k(const int64_t* __restrict__ colp, const int64_t* __restrict__ rowi, int64_t dim,
                         int64_t nnz, unsigned long long* __restrict__ key, int64_t* __restrict__ val,
                         unsigned long long* __restrict__ ndiag) {
  unsigned long long nd = 0;
  GRID_LOOP(p, nnz) {
    const int64_t j = col_of(colp, dim, p), i = rowi[p];
    key[2 * p] = (static_cast<unsigned long long>(i) << 32) | static_cast<unsigned long long>(j);
    val[2 * p] = p;
    key[2 * p + 1] = i != j ? (static_cast<unsigned long long>(j) << 32) | static_cast<unsigned long long>(i) : kNone;
    val[2 * p + 1] = p;
    nd += i == j ? 1 : 0;
  }
  if (nd) atomicAdd(ndiag, nd);
}

__global__ void split_key_k(const unsigned long long* __restrict__ key, int64_t n, int64_t* __restrict__ col,
                            int* __restrict__ rowcnt) {
  GRID_LOOP(i, n) {
    col[i] = static_cast<int64_t>(key[i] & 0xffffffffull);
    atomicAdd(&rowcnt[key[i] >> 32], 1);
  }
}

// J^T lambda: Jacobian entries of kept rows and free columns, keyed by column
__global__ void jt_keys_k(const int64_t* __restrict__ jr, const int64_t* __restrict__ jc, int64_t J,
                          const int64_t* __restrict__ prim, const int64_t* __restrict__ dual,
                          unsigned long long* __restrict__ key, int64_t* __restrict__ val) {
  GRID_LOOP(q, J) {
    const int64_t d = dual[jr[q]], pj = prim[jc[q]];
    key[q] = (d >= 0 && pj >= 0) ? static_cast<unsigned long long>(pj) : kNone;
    val[q] = q;
  }
}

__global__ void jt_fill_k(const unsigned long long* __restrict__ key, const int64_t* __restrict__ q,
                          const int64_t* __restrict__ jr, const int64_t* __restrict__ dual, int64_t n,
                          int64_t* __restrict__ dual_out, int* __restrict__ cnt) {
  GRID_LOOP(i, n) {
    dual_out[i] = dual[jr[q[i]]];
    atomicAdd(&cnt[key[i]], 1);
  }
}

__global__ void widen_k(const int* __restrict__ c, int64_t n, int64_t* __restrict__ out) {
  GRID_LOOP(i, n) out[i] = c[i];
}

void sort_pairs(unsigned long long*& keys, int64_t*& vals, int64_t n, int end_bit, cudaStream_t s) {
  unsigned long long* k2 = dalloc<unsigned long long>(static_cast<size_t>(n), s);
  int64_t* v2 = dalloc<int64_t>(static_cast<size_t>(n), s);
  size_t tmp_bytes = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, k2, vals, v2, n, 0, end_bit, s), "sort size");
  void* tmp = dalloc<char>(tmp_bytes, s);
  ck(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, k2, vals, v2, n, 0, end_bit, s), "sort");
  dfree(tmp);
  dfree(keys);
  dfree(vals);
  keys = k2;
  vals = v2;
}

// out[0] = 0, out[1 + i] = inclusive prefix of in[i] (n + 1 entries)
void exclusive_offsets(const int64_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  ck(cudaMemsetAsync(out, 0, sizeof(int64_t), s), "memset");
  if (n <= 0) return;
  size_t tmp_bytes = 0;
  ck(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, in, out + 1, n, s), "scan size");
  void* tmp = dalloc<char>(tmp_bytes, s);
  ck(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, in, out + 1, n, s), "scan");
  dfree(tmp);
}

int bits_for(int64_t v) {
  int b = 1;
  while (b < 64 && (1ull << b) <= static_cast<unsigned long long>(v)) ++b;
  return b;
}

}  // namespace

void build_kkt(const KktBuildIn& in, cudaStream_t s, KktBuildOut& out) {
  static const bool timing = std::getenv("OCG_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build_kkt] %-22s %8.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  const int64_t H = in.H, J = in.J, S = in.n_slack, ntot = in.n_free + in.n_slack, m = in.m;
  const int64_t dim = ntot + m;
  if (dim >= (1ll << 31)) throw std::runtime_error("KKT dimension exceeds the device pattern builder's 2^31");
  const int64_t C = H + J + S + ntot + m;
  // 1. sources -> keys, stable sort: (col, row) order, codes ascending in a slot
  auto* key = dalloc<unsigned long long>(static_cast<size_t>(C), s);
  auto* code = dalloc<int64_t>(static_cast<size_t>(C), s);
  keys_k<<<grid_for(C), 256, 0, s>>>(in.hr, in.hc, H, in.jr, in.jc, J, in.prim, in.dual, in.slack_dual, in.n_free,
                                     S, ntot, m, key, code);
  sort_pairs(key, code, C, 64, s);
  lap("sources sorted");
  // 2. slots: runs of equal keys
  auto* flag = dalloc<int64_t>(static_cast<size_t>(C), s);
  auto* slot = dalloc<int64_t>(static_cast<size_t>(C) + 1, s);
  fresh_k<<<grid_for(C), 256, 0, s>>>(key, C, flag);
  exclusive_offsets(flag, C, slot, s);  // slot[1 + i] = inclusive count
  int64_t nnz = 0, nvalid = 0;
  ck(cudaMemcpyAsync(&nnz, slot + C, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "nnz");
  ck(cudaStreamSynchronize(s), "sync");
  auto* rowi = dalloc<int64_t>(static_cast<size_t>(nnz), s);
  auto* src_ptr = dalloc<int64_t>(static_cast<size_t>(nnz) + 1, s);
  int* colcnt = dalloc<int>(static_cast<size_t>(dim), s);
  ck(cudaMemsetAsync(colcnt, 0, static_cast<size_t>(dim) * sizeof(int), s), "memset");
  slots_k<<<grid_for(C), 256, 0, s>>>(key, slot + 1, C, rowi, src_ptr, colcnt);
  // valid sources are a prefix of the sorted array (the sentinels sort last):
  // their count, the first sentinel's position, ends the last slot
  {
    unsigned long long last = 0;
    int64_t lo = 0, hi = C;  // first index with key == kNone
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      ck(cudaMemcpyAsync(&last, key + mid, sizeof(last), cudaMemcpyDeviceToHost, s), "probe");
      ck(cudaStreamSynchronize(s), "sync");
      if (last == kNone)
        hi = mid;
      else
        lo = mid + 1;
    }
    nvalid = lo;
  }
  ck(cudaMemcpyAsync(src_ptr + nnz, &nvalid, sizeof(int64_t), cudaMemcpyHostToDevice, s), "src end");
  auto* colp = dalloc<int64_t>(static_cast<size_t>(dim) + 1, s);
  auto* colcnt64 = dalloc<int64_t>(static_cast<size_t>(dim), s);
  widen_k<<<grid_for(dim), 256, 0, s>>>(colcnt, dim, colcnt64);
  exclusive_offsets(colcnt64, dim, colp, s);
  out.nnz = nnz;
  out.colp.resize(static_cast<size_t>(dim) + 1);
  out.rowi.resize(static_cast<size_t>(nnz));
  ck(cudaMemcpyAsync(out.colp.data(), colp, out.colp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "colp");
  ck(cudaMemcpyAsync(out.rowi.data(), rowi, out.rowi.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "rowi");
  out.src_ptr = src_ptr;
  out.src_code = code;  // sorted codes (first nvalid are the slots' sources)
  out.ncode = nvalid;

  lap("slots + host pattern");
  // 3. full symmetric CSR for matvec: mirrored entries keyed (row, col)
  auto* mkey = dalloc<unsigned long long>(2 * static_cast<size_t>(nnz), s);
  auto* mval = dalloc<int64_t>(2 * static_cast<size_t>(nnz), s);
  auto* ndiag = dalloc<unsigned long long>(1, s);
  ck(cudaMemsetAsync(ndiag, 0, sizeof(unsigned long long), s), "memset");
  mirror_k<<<grid_for(nnz), 256, 0, s>>>(colp, rowi, dim, nnz, mkey, mval, ndiag);
  unsigned long long nd = 0;
  ck(cudaMemcpyAsync(&nd, ndiag, sizeof(nd), cudaMemcpyDeviceToHost, s), "ndiag");
  ck(cudaStreamSynchronize(s), "sync");
  const int64_t mv_nnz = 2 * nnz - static_cast<int64_t>(nd);
  sort_pairs(mkey, mval, 2 * nnz, 64, s);
  auto* mv_col = dalloc<int64_t>(static_cast<size_t>(mv_nnz), s);
  int* rowcnt = dalloc<int>(static_cast<size_t>(dim), s);
  ck(cudaMemsetAsync(rowcnt, 0, static_cast<size_t>(dim) * sizeof(int), s), "memset");
  split_key_k<<<grid_for(mv_nnz), 256, 0, s>>>(mkey, mv_nnz, mv_col, rowcnt);
  auto* rowcnt64 = dalloc<int64_t>(static_cast<size_t>(dim), s);
  widen_k<<<grid_for(dim), 256, 0, s>>>(rowcnt, dim, rowcnt64);
  auto* mv_ptr = dalloc<int64_t>(static_cast<size_t>(dim) + 1, s);
  exclusive_offsets(rowcnt64, dim, mv_ptr, s);
  out.mv_ptr = mv_ptr;
  out.mv_col = mv_col;
  out.mv_vidx = mval;

  lap("symmetric CSR");
  // 4. J^T lambda gather: per free column, Jacobian entries in increasing order
  auto* jkey = dalloc<unsigned long long>(static_cast<size_t>(J), s);
  auto* jval = dalloc<int64_t>(static_cast<size_t>(J), s);
  jt_keys_k<<<grid_for(J), 256, 0, s>>>(in.jr, in.jc, J, in.prim, in.dual, jkey, jval);
  sort_pairs(jkey, jval, J, 64, s);
  int64_t njt = 0;
  {
    unsigned long long last = 0;
    int64_t lo = 0, hi = J;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      ck(cudaMemcpyAsync(&last, jkey + mid, sizeof(last), cudaMemcpyDeviceToHost, s), "probe");
      ck(cudaStreamSynchronize(s), "sync");
      if (last == kNone)
        hi = mid;
      else
        lo = mid + 1;
    }
    njt = lo;
  }
  auto* jt_dual = dalloc<int64_t>(static_cast<size_t>(njt), s);
  int* jcnt = dalloc<int>(static_cast<size_t>(ntot), s);
  ck(cudaMemsetAsync(jcnt, 0, static_cast<size_t>(std::max<int64_t>(ntot, 1)) * sizeof(int), s), "memset");
  if (njt > 0) jt_fill_k<<<grid_for(njt), 256, 0, s>>>(jkey, jval, in.jr, in.dual, njt, jt_dual, jcnt);
  auto* jcnt64 = dalloc<int64_t>(static_cast<size_t>(ntot), s);
  widen_k<<<grid_for(ntot), 256, 0, s>>>(jcnt, ntot, jcnt64);
  auto* jt_ptr = dalloc<int64_t>(static_cast<size_t>(ntot) + 1, s);
  exclusive_offsets(jcnt64, ntot, jt_ptr, s);
  out.jt_ptr = jt_ptr;
  out.jt_e = jval;
  out.jt_dual = jt_dual;

  lap("J^T gather");
  ck(cudaStreamSynchronize(s), "sync");
  for (void* p : {static_cast<void*>(key), static_cast<void*>(flag), static_cast<void*>(slot),
                  static_cast<void*>(colcnt), static_cast<void*>(colcnt64), static_cast<void*>(colp),
                  static_cast<void*>(rowi), static_cast<void*>(ndiag),
                  static_cast<void*>(mkey), static_cast<void*>(rowcnt), static_cast<void*>(rowcnt64),
                  static_cast<void*>(jkey), static_cast<void*>(jcnt), static_cast<void*>(jcnt64)})
    dfree(p);
  for (void* p : {static_cast<void*>(out.src_ptr), static_cast<void*>(out.src_code), static_cast<void*>(out.mv_ptr),
                  static_cast<void*>(out.mv_col), static_cast<void*>(out.mv_vidx), static_cast<void*>(out.jt_ptr),
                  static_cast<void*>(out.jt_e), static_cast<void*>(out.jt_dual)})
    forget(p);
  ck(cudaStreamSynchronize(s), "sync");
}

// Slots ordered by their first source code (kktbuild.hpp source_order).
__global__ void first_code_k(const int64_t* __restrict__ ptr, const int64_t* __restrict__ code, int64_t nnz,
                             int64_t max_code, unsigned long long* __restrict__ key, int64_t* __restrict__ slot) {
  GRID_LOOP(p, nnz) {
    key[p] = static_cast<unsigned long long>(ptr[p + 1] > ptr[p] ? code[ptr[p]] : max_code);
    slot[p] = p;
  }
}
__global__ void permute_codes_k(const int64_t* __restrict__ slot, const uint32_t* __restrict__ code32, int64_t nnz,
                                int32_t* __restrict__ order, uint32_t* __restrict__ code32_sorted) {
  GRID_LOOP(t, nnz) {
    const int64_t p = slot[t];
    order[t] = static_cast<int32_t>(p);
    code32_sorted[t] = code32[p];
  }
}

void source_order(const int64_t* ptr, const int64_t* code, const uint32_t* code32, int64_t nnz, int64_t max_code,
                  int32_t* order, uint32_t* code32_sorted, cudaStream_t s) {
  if (nnz <= 0) return;
  auto* key = dalloc<unsigned long long>(static_cast<size_t>(nnz), s);
  auto* slot = dalloc<int64_t>(static_cast<size_t>(nnz), s);
  first_code_k<<<grid_for(nnz), 256, 0, s>>>(ptr, code, nnz, max_code, key, slot);
  sort_pairs(key, slot, nnz, bits_for(max_code + 1), s);
  permute_codes_k<<<grid_for(nnz), 256, 0, s>>>(slot, code32, nnz, order, code32_sorted);
  ck(cudaStreamSynchronize(s), "sync");
  dfree(key);
  dfree(slot);
}

}  // namespace ocg::dev
