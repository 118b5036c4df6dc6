// Hand-written sm_100a kernels: deterministic reductions and gathers around
// the generated per-node kernels. See kernels.hpp for the reference each one
// mirrors. All of them are HBM-bound streaming/gather kernels; grids are
// sized in multiples of the 148 SMs x resident blocks.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.hpp"

namespace ocg::dev {

namespace {

constexpr int kChunk = 512;  // Backend::kChunkSize (backend.hpp:50)
constexpr int kSms = 148;

__device__ __forceinline__ bool finite(double v) { return fabs(v) <= 1.7976931348623157e308; }

// rows longer than kLongRow go to the one-block-per-row kernels below
__device__ __forceinline__ bool is_long(const int64_t* ptr, int64_t i) { return ptr[i + 1] - ptr[i] > kLongRow; }

// One warp per 512-instance chunk: coalesced loads into shared memory, then
// lane 0 adds in index order (the reference's `s += v` loop).
__global__ void __launch_bounds__(256) chunk_sums(const double* __restrict__ objv, const int64_t* __restrict__ goff,
                                                  const int64_t* __restrict__ gcount,
                                                  const int64_t* __restrict__ cbase, int64_t n_chunks,
                                                  int n_groups, double* __restrict__ partials) {
  __shared__ double buf[8][kChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (c >= n_chunks) return;
  int g = 0;
  while (g + 1 < n_groups && cbase[g + 1] <= c) ++g;
  const int64_t lo = (c - cbase[g]) * kChunk;
  const int64_t hi = min(gcount[g], lo + kChunk);
  const int64_t n = hi - lo;
  const double* src = objv + goff[g] + lo;
  for (int64_t i = lane; i < n; i += 32) buf[warp][i] = src[i];
  __syncwarp();
  if (lane == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += buf[warp][i];
    partials[c] = s;
  }
}

__global__ void combine_chunks(const double* __restrict__ partials, const int64_t* __restrict__ cbase,
                               const double* __restrict__ weights, int n_groups, double obj_scale,
                               double* __restrict__ f, int* __restrict__ flag) {
  // one warp: the lanes stage the chunk partials into shared memory a tile
  // at a time, lane 0 adds them in chunk order and closes each group in
  // group order (the same roundings as one thread reading global memory,
  // without a global-load round trip per chunk)
  if (blockIdx.x != 0) return;
  constexpr int kTile = 1024;
  __shared__ double buf[kTile];
  const int lane = threadIdx.x;
  double total = 0.0, part = 0.0;
  int g = 0;
  const int64_t c0 = n_groups > 0 ? cbase[0] : 0, c1 = n_groups > 0 ? cbase[n_groups] : 0;
  for (int64_t t0 = c0; t0 < c1; t0 += kTile) {
    const int n = static_cast<int>(c1 - t0 < kTile ? c1 - t0 : kTile);
    for (int i = lane; i < n; i += 32) buf[i] = partials[t0 + i];
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < n; ++i) {
        while (t0 + i >= cbase[g + 1]) {  // groups ending before this chunk, empty ones included
          total += weights[g] * part;
          part = 0.0;
          ++g;
        }
        part += buf[i];
      }
    __syncwarp();
  }
  if (lane != 0) return;
  for (; g < n_groups; ++g) {
    total += weights[g] * part;
    part = 0.0;
  }
  const double fs = obj_scale * total;
  *f = fs;
  if (!finite(fs)) *flag = 1;
}

__global__ void __launch_bounds__(256) gather_sum_k(const double* __restrict__ src, const int64_t* __restrict__ ptr,
                                                    const int32_t* __restrict__ idx, int64_t n,
                                                    double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (is_long(ptr, i)) continue;
    double s = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += src[idx[p]];
    out[i] = s;
  }
}

__global__ void __launch_bounds__(256) kkt_assemble_k(const double* __restrict__ hess, const double* __restrict__ jac,
                                                      const double* __restrict__ sigma,
                                                      const int64_t* __restrict__ ptr,
                                                      const int64_t* __restrict__ code, int64_t nnz, int64_t H,
                                                      int64_t J, int64_t S, int64_t ntot, double* __restrict__ val) {
  const int64_t HJ = H + J, HJS = H + J + S;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (is_long(ptr, p)) continue;
    double s = 0.0;
    for (int64_t q = ptr[p]; q < ptr[p + 1]; ++q) {
      const int64_t c = code[q];
      double v;
      if (c < H)
        v = hess[c];
      else if (c < HJ)
        v = jac[c - H];
      else if (c < HJS)
        v = -1.0;
      else if (c < HJS + ntot)
        v = sigma[c - HJS];
      else
        v = 0.0;  // dual diagonal: structural, no value (-delta_c is the factorization's)
      s += v;
    }
    val[p] = s;
  }
}

// Compact per-slot source codes (kkt_code32): single-source slots — most of
// K — gather through one 32-bit word (3-bit array tag, 29-bit index) instead
// of ptr[p], ptr[p+1] and an int64 code; slots with several sources keep the
// CSR walk in code order.
constexpr uint32_t kTagShift = 29, kIdxMask = (1u << kTagShift) - 1;
enum : uint32_t { kTagHess = 0, kTagJac = 1, kTagSigma = 2, kTagMinus1 = 3, kTagZero = 4, kTagMulti = 7 };

__global__ void __launch_bounds__(256) kkt_code32_k(const int64_t* __restrict__ ptr, const int64_t* __restrict__ code,
                                                    int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot,
                                                    uint32_t* __restrict__ out) {
  const int64_t HJ = H + J, HJS = H + J + S;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q0 = ptr[p], n = ptr[p + 1] - q0;
    uint32_t w = kTagMulti << kTagShift;
    if (n == 1) {
      const int64_t c = code[q0];
      if (c < H)
        w = (kTagHess << kTagShift) | static_cast<uint32_t>(c);
      else if (c < HJ)
        w = (kTagJac << kTagShift) | static_cast<uint32_t>(c - H);
      else if (c < HJS)
        w = kTagMinus1 << kTagShift;
      else if (c < HJS + ntot)
        w = (kTagSigma << kTagShift) | static_cast<uint32_t>(c - HJS);
      else
        w = kTagZero << kTagShift;
    } else if (n == 0) {
      w = kTagZero << kTagShift;
    }
    out[p] = w;
  }
}

// slot t (or order[t] when given: kktbuild.hpp source_order), code32[t] its
// compact code. Measured on Goddard / quadrotor N=1e5: the slot order (a
// gather, coalesced writes) beats the source order (coalesced reads,
// scattered writes: 110 -> 132 MB of DRAM reads, the partial-sector writes
// are filled from DRAM), so the library walks slots in slot order.
__global__ void __launch_bounds__(256) kkt_assemble_fast_k(const double* __restrict__ hess,
                                                           const double* __restrict__ jac,
                                                           const double* __restrict__ sigma,
                                                           const uint32_t* __restrict__ code32,
                                                           const int32_t* __restrict__ order,
                                                           const int64_t* __restrict__ ptr,
                                                           const int64_t* __restrict__ code, int64_t nnz, int64_t H,
                                                           int64_t J, int64_t S, int64_t ntot,
                                                           double* __restrict__ val) {
  const int64_t HJ = H + J, HJS = H + J + S;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < nnz;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = order ? static_cast<int64_t>(__ldg(order + t)) : t;
    const uint32_t w = __ldg(code32 + t);
    const uint32_t tag = w >> kTagShift, i = w & kIdxMask;
    double s;
    if (tag == kTagHess) {
      s = __ldg(hess + i);
    } else if (tag == kTagJac) {
      s = __ldg(jac + i);
    } else if (tag == kTagSigma) {
      s = __ldg(sigma + i);
    } else if (tag == kTagMinus1) {
      s = -1.0;
    } else if (tag == kTagZero) {
      s = 0.0;
    } else {  // several sources, in the reference's order (code order)
      if (is_long(ptr, p)) continue;
      s = 0.0;
      for (int64_t q = ptr[p]; q < ptr[p + 1]; ++q) {
        const int64_t c = code[q];
        double v;
        if (c < H)
          v = hess[c];
        else if (c < HJ)
          v = jac[c - H];
        else if (c < HJS)
          v = -1.0;
        else if (c < HJS + ntot)
          v = sigma[c - HJS];
        else
          v = 0.0;
        s += v;
      }
    }
    val[p] = s;
  }
}

// ---- tiled assembly (kkt_tile_*): a block owns kTileSlots consecutive slots;
// the sources its slots read from each source stream (one per COO group of
// hess / jac, and sigma) form one window [lo, lo + len) that the block copies
// into shared memory with coalesced loads, so every source byte leaves DRAM
// about once; slot codes then address shared memory (tag kTagSmem). Windows
// too sparse or too large for the block's budget stay in global memory.
constexpr uint32_t kTagSmem = 5;
// a slot with 2..kMultiMax sources whose codes sit in the tile's staged copy
// of mcode: (count << kMultiShift) | offset from the tile's first code
constexpr uint32_t kTagMultiLocal = 6;
constexpr uint32_t kMultiShift = 24, kMultiMax = 31;

__device__ __forceinline__ int stream_of(const int64_t* __restrict__ sb, int ns, int64_t c) {
  int lo = 0, hi = ns;  // sb[0..ns]: stream s covers [sb[s], sb[s+1])
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(sb + mid) <= c) lo = mid; else hi = mid;
  }
  return (c >= __ldg(sb) && c < __ldg(sb + ns)) ? lo : -1;
}

// unified code of a compact single-source word (-1: no data: constants, multi)
__device__ __forceinline__ int64_t unified_of(uint32_t w, int64_t H, int64_t HJS) {
  const uint32_t tag = w >> kTagShift, i = w & kIdxMask;
  if (tag == kTagHess) return i;
  if (tag == kTagJac) return H + i;
  if (tag == kTagSigma) return HJS + i;
  return -1;
}
__device__ __forceinline__ uint32_t word_of(int64_t c, int64_t H, int64_t J, int64_t S, int64_t ntot) {
  const int64_t HJ = H + J, HJS = HJ + S;
  if (c < H) return (kTagHess << kTagShift) | static_cast<uint32_t>(c);
  if (c < HJ) return (kTagJac << kTagShift) | static_cast<uint32_t>(c - H);
  if (c < HJS) return kTagMinus1 << kTagShift;
  if (c < HJS + ntot) return (kTagSigma << kTagShift) | static_cast<uint32_t>(c - HJS);
  return kTagZero << kTagShift;
}

__global__ void __launch_bounds__(256) kkt_tile_minmax_k(const uint32_t* __restrict__ code32,
                                                         const int64_t* __restrict__ ptr,
                                                         const int64_t* __restrict__ code, int64_t nnz,
                                                         const int64_t* __restrict__ sb, int ns, int64_t H,
                                                         int64_t J, int64_t S, unsigned long long* __restrict__ mn,
                                                         unsigned long long* __restrict__ mx,
                                                         unsigned int* __restrict__ cnt) {
  const int64_t HJS = H + J + S;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = p / kTileSlots;
    const uint32_t w = code32[p];
    auto note = [&](int64_t c) {
      const int st = c >= 0 ? stream_of(sb, ns, c) : -1;
      if (st < 0) return;
      atomicMin(mn + t * ns + st, static_cast<unsigned long long>(c));
      atomicMax(mx + t * ns + st, static_cast<unsigned long long>(c));
      atomicAdd(cnt + t * ns + st, 1u);
    };
    if ((w >> kTagShift) == kTagMulti) {
      if (is_long(ptr, p)) continue;
      for (int64_t q = ptr[p]; q < ptr[p + 1]; ++q) {
        const int64_t c = code[q];
        if (c < H + J || (c >= HJS)) note(c);
      }
    } else {
      note(unified_of(w, H, HJS));
    }
  }
}

// one thread per tile: window lengths and shared-memory offsets; a window is
// staged when it is dense (len <= kTileSparse * the sources read from it +
// 32) and fits the block's budget
__global__ void kkt_tile_plan_k(const unsigned long long* __restrict__ mn, const unsigned long long* __restrict__ mx,
                                const unsigned int* __restrict__ cnt,
                                int64_t ntile, int ns, int64_t nnz, int64_t* __restrict__ wlo,
                                int32_t* __restrict__ wlen, int32_t* __restrict__ woff) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= ntile) return;
  int32_t off = kTileConsts;  // win[0] = -1.0, win[1] = 0.0
  for (int st = 0; st < ns; ++st) {
    const unsigned long long a = mn[t * ns + st], b = mx[t * ns + st];
    int32_t len = 0;
    if (b >= a && b != ~0ull) {
      const int64_t l = static_cast<int64_t>(b - a) + 1;
      if (l <= static_cast<int64_t>(kTileSparse) * cnt[t * ns + st] + 32 && off + l + 2 <= kTileWindow)
        len = static_cast<int32_t>(l);
    }
    wlo[t * ns + st] = static_cast<int64_t>(a);
    wlen[t * ns + st] = len;
    woff[t * ns + st] = off;
    off += len + (len & 1);
  }
}

// rewrite the codes of staged sources to shared-memory offsets
__global__ void __launch_bounds__(256) kkt_tile_codes_k(uint32_t* __restrict__ code32, const int64_t* __restrict__ ptr,
                                                        const int64_t* __restrict__ code, uint32_t* __restrict__ mcode,
                                                        int64_t nnz, const int64_t* __restrict__ sb, int ns,
                                                        const int64_t* __restrict__ wlo, const int32_t* __restrict__ wlen,
                                                        const int32_t* __restrict__ woff, int64_t H, int64_t J,
                                                        int64_t S, int64_t ntot) {
  const int64_t HJS = H + J + S;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = p / kTileSlots;
    auto staged = [&](int64_t c, uint32_t& w) {
      const int st = c >= 0 ? stream_of(sb, ns, c) : -1;
      if (st < 0) return;
      const int64_t k = t * ns + st;
      if (wlen[k] > 0) w = (kTagSmem << kTagShift) | static_cast<uint32_t>(woff[k] + (c - wlo[k]));
    };
    auto consts = [](uint32_t& w) {
      if ((w >> kTagShift) == kTagMinus1) w = (kTagSmem << kTagShift) | 0u;
      if ((w >> kTagShift) == kTagZero) w = (kTagSmem << kTagShift) | 1u;
    };
    uint32_t w = code32[p];
    if ((w >> kTagShift) == kTagMulti) {
      if (is_long(ptr, p)) continue;
      for (int64_t q = ptr[p]; q < ptr[p + 1]; ++q) {
        const int64_t c = code[q];
        uint32_t mw = word_of(c, H, J, S, ntot);
        if (c < H + J || c >= HJS) staged(c, mw);
        consts(mw);
        mcode[q] = mw;
      }
      const int64_t n = ptr[p + 1] - ptr[p], off = ptr[p] - ptr[t * kTileSlots];
      if (n <= kMultiMax && off < (int64_t{1} << kMultiShift))
        code32[p] = (kTagMultiLocal << kTagShift) | (static_cast<uint32_t>(n) << kMultiShift) | static_cast<uint32_t>(off);
    } else {
      staged(unified_of(w, H, HJS), w);
      consts(w);
      code32[p] = w;
    }
  }
}

__device__ __forceinline__ double tile_fetch(uint32_t w, const double* __restrict__ win, const double* __restrict__ hess,
                                             const double* __restrict__ jac, const double* __restrict__ sigma) {
  const uint32_t tag = w >> kTagShift, i = w & kIdxMask;
  switch (tag) {
    case kTagSmem: return win[i];
    case kTagHess: return __ldg(hess + i);
    case kTagJac: return __ldg(jac + i);
    case kTagSigma: return __ldg(sigma + i);
    case kTagMinus1: return -1.0;
    default: return 0.0;
  }
}

__global__ void __launch_bounds__(256) kkt_assemble_tiled_k(const double* __restrict__ hess,
                                                            const double* __restrict__ jac,
                                                            const double* __restrict__ sigma,
                                                            const uint32_t* __restrict__ code32,
                                                            const int64_t* __restrict__ ptr,
                                                            const uint32_t* __restrict__ mcode, int64_t nnz,
                                                            int ns, const int64_t* __restrict__ wlo,
                                                            const int32_t* __restrict__ wlen,
                                                            const int32_t* __restrict__ woff, int64_t H, int64_t J,
                                                            int64_t S, double* __restrict__ val) {
  extern __shared__ __align__(16) double win[];
  constexpr int kPer = static_cast<int>(kTileSlots / 256);  // slots per thread (blockDim.x == 256)
  const int64_t t = blockIdx.x;
  const int64_t HJS = H + J + S;
  const int64_t p0 = t * kTileSlots;
  // the tile's codes first (one DRAM round trip for all of them) ...
  uint32_t w[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int64_t p = p0 + j * 256 + threadIdx.x;
    w[j] = p < nnz ? __ldg(code32 + p) : (kTagZero << kTagShift);
  }
  // ... while the tile's window table comes in (one load per stream, all in
  // flight together) ...
  __shared__ int64_t s_lo[kTileMaxStreams];
  __shared__ int32_t s_len[kTileMaxStreams], s_off[kTileMaxStreams];
  for (int st = threadIdx.x; st < ns; st += blockDim.x) {
    s_lo[st] = wlo[t * ns + st];
    s_len[st] = wlen[t * ns + st];
    s_off[st] = woff[t * ns + st];
  }
  __syncthreads();
  // ... and then the windows: warp w copies windows w, w + 8, ... (LDGSTS,
  // coalesced; every copy of the tile in flight together, one wait)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int st = warp; st < ns; st += 8) {
    const int32_t len = s_len[st];
    if (len == 0) continue;
    const int64_t lo = s_lo[st];
    const double* src = lo < H ? hess + lo : (lo < H + J ? jac + (lo - H) : sigma + (lo - HJS));
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(win + s_off[st]));
    for (int32_t i = lane; i < len; i += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * static_cast<unsigned>(i)), "l"(src + i)
                   : "memory");
  }
  // the codes of the tile's multi-source slots (one contiguous range of mcode)
  const int64_t q0 = __ldg(ptr + p0), q1 = __ldg(ptr + min(nnz, p0 + kTileSlots));
  const int nq = static_cast<int>(q1 - q0 < kTileMcode ? q1 - q0 : kTileMcode);
  uint32_t* const mloc = reinterpret_cast<uint32_t*>(win + kTileWindow);
  for (int i = threadIdx.x; i < nq; i += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(mloc + i))),
                 "l"(mcode + q0 + i)
                 : "memory");
  if (threadIdx.x == 0) {
    win[0] = -1.0;
    win[1] = 0.0;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int64_t p = p0 + j * 256 + threadIdx.x;
    if (p >= nnz) break;
    const uint32_t tag = w[j] >> kTagShift;
    double s;
    if (tag == kTagSmem) {
      s = win[w[j] & kIdxMask];
    } else if (tag == kTagMultiLocal) {
      const uint32_t off = w[j] & ((1u << kMultiShift) - 1);
      const int n = static_cast<int>((w[j] >> kMultiShift) & kMultiMax);
      // codes staged (or, past the staged range, from global memory)
      const uint32_t* c = static_cast<int>(off) + n <= nq ? mloc + off : mcode + q0 + off;
      s = 0.0;  // the reference's order
      for (int i = 0; i < n; ++i) {
        const uint32_t cw = c[i];
        s += (cw >> kTagShift) == kTagSmem ? win[cw & kIdxMask] : tile_fetch(cw, win, hess, jac, sigma);
      }
    } else if (tag != kTagMulti) {
      s = tile_fetch(w[j], win, hess, jac, sigma);
    } else {  // more than kMultiMax sources (long rows: kkt_assemble_long_k)
      if (is_long(ptr, p)) continue;
      s = 0.0;
      for (int64_t q = ptr[p]; q < ptr[p + 1]; ++q) s += tile_fetch(__ldg(mcode + q), win, hess, jac, sigma);
    }
    val[p] = s;
  }
}

template <class I>
__global__ void __launch_bounds__(256) sym_matvec_k(const double* __restrict__ val, const int64_t* __restrict__ rptr,
                                                    const I* __restrict__ col,
                                                    const I* __restrict__ vidx, int64_t n,
                                                    const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (is_long(rptr, i)) continue;
    double s = 0.0;
    for (int64_t p = rptr[i]; p < rptr[i + 1]; ++p) s += val[vidx[p]] * x[col[p]];
    y[i] = s;
  }
}

// max over rows of sum_j |K_ij| with the symmetric mirror (sparse::norm_inf_sym)
template <class I>
__global__ void __launch_bounds__(256) sym_norm_inf_k(const double* __restrict__ val, const int64_t* __restrict__ rptr,
                                                      const I* __restrict__ vidx, int64_t n,
                                                      unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (is_long(rptr, i)) continue;
    double s = 0.0;
    for (int64_t p = rptr[i]; p < rptr[i + 1]; ++p) s += fabs(val[vidx[p]]);
    m = fmax(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, wm[w]);
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

template <class I>
__global__ void __launch_bounds__(256) jt_lambda_k(const double* __restrict__ jac, const double* __restrict__ lam,
                                                   const int64_t* __restrict__ ptr, const I* __restrict__ e_idx,
                                                   const I* __restrict__ dual_idx, int64_t n_free,
                                                   const int64_t* __restrict__ slack_dual, int64_t n_slack,
                                                   double* __restrict__ out) {
  const int64_t ntot = n_free + n_slack;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ntot;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (is_long(ptr, i)) continue;
    double s = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += jac[e_idx[p]] * lam[dual_idx[p]];
    if (i >= n_free) s -= lam[slack_dual[i - n_free]];
    out[i] = s;
  }
}

__global__ void __launch_bounds__(256) max_abs_k(const double* __restrict__ v, int64_t n,
                                                 unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(v[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, wm[w]);
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// ---- long rows ------------------------------------------------------------------
// A row whose source list is longer than kLongRow (e.g. the free final time
// tf of a free-horizon problem: its KKT diagonal gathers one Hessian entry per
// time step, its J^T lambda entry one Jacobian entry per dynamics row) would
// be one thread's serial chain of dependent gathers. The thread-per-row
// kernels skip such rows; one block per long row sums it. Pure sums keep the
// reference's order (increasing source index, one `s += term` accumulator):
// threads 32.. gather the terms into shared memory, double-buffered, while
// thread 0 adds the previous stage in order.
constexpr int kStage = 2048;

template <class Term>
__device__ double ordered_block_sum(int64_t lo, int64_t hi, Term term) {
  __shared__ double sb[2][kStage];
  const int64_t n = hi - lo;
  const int tid = static_cast<int>(threadIdx.x), nl = static_cast<int>(blockDim.x) - 32;
  auto stage = [&](int64_t k, double* dst) {
    const int64_t b = lo + k * kStage, e = min(hi, b + kStage);
    for (int64_t p = b + (tid - 32); p < e; p += nl) dst[p - b] = term(p);
  };
  double s = 0.0;
  const int64_t nst = (n + kStage - 1) / kStage;
  if (tid >= 32 && nst > 0) stage(0, sb[0]);
  __syncthreads();
  for (int64_t k = 0; k < nst; ++k) {
    if (tid >= 32) {
      if (k + 1 < nst) stage(k + 1, sb[(k + 1) & 1]);
    } else if (tid == 0) {
      const double* c = sb[k & 1];
      const int m = static_cast<int>(min(static_cast<int64_t>(kStage), n - k * kStage));
      int i = 0;
      for (; i + 8 <= m; i += 8) {  // eight loads in flight, then the ordered adds
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = c[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[j];
      }
      for (; i < m; ++i) s += c[i];
    }
    __syncthreads();
  }
  return s;
}

// Products and norms of long rows (J^T lambda, K x, |K| row sums): a fixed-shape
// tree over kLongBlocks blocks per row — block b sums its contiguous share of
// the row with thread t taking terms t, t+256, ..., then the warps' shuffle
// trees and the warp partials in warp order into partials[row][b]; a second
// pass adds the kLongBlocks partials in block order. Deterministic; not the
// reference's left-to-right order (these sums are FMA-contracted in the
// thread-per-row path anyway), within 1e-12 relative of it.
template <class Term>
__device__ void tree_block_partial(int64_t lo, int64_t hi, Term term, double* partial) {
  __shared__ double wp[8];
  const int64_t len = hi - lo, per = (len + kLongBlocks - 1) / kLongBlocks;
  const int64_t a = lo + min(len, per * blockIdx.x), e = lo + min(len, per * (blockIdx.x + 1));
  double s = 0.0;
#pragma unroll 4
  for (int64_t p = a + threadIdx.x; p < e; p += blockDim.x) s += term(p);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += wp[w];
    *partial = s;
  }
}

// second pass: one thread per long row adds its partials in block order;
// mode 0 stores, 1 subtracts the slack term (J^T lambda), 2 takes the max (norm)
__global__ void long_finish_k(LongRows lr, double* __restrict__ out, int mode, const double* __restrict__ lam,
                              const int64_t* __restrict__ slack_dual, int64_t n_free) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= lr.n) return;
  const double* pp = lr.partials + r * kLongBlocks;
  double s = 0.0;
  for (int b = 0; b < kLongBlocks; ++b) s += pp[b];
  const int64_t i = lr.idx[r];
  if (mode == 2) {
    atomicMax(reinterpret_cast<unsigned long long*>(out), static_cast<unsigned long long>(__double_as_longlong(s)));
    return;
  }
  if (mode == 1 && i >= n_free) s -= lam[slack_dual[i - n_free]];
  out[i] = s;
}


__global__ void __launch_bounds__(256) gather_sum_long_k(const double* __restrict__ src,
                                                         const int64_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ idx, LongRows lr,
                                                         double* __restrict__ out) {
  const int64_t i = lr.idx[blockIdx.x];
  const double s = ordered_block_sum(ptr[i], ptr[i + 1], [&](int64_t p) { return src[idx[p]]; });
  if (threadIdx.x == 0) out[i] = s;
}

__global__ void __launch_bounds__(256) kkt_assemble_long_k(const double* __restrict__ hess,
                                                           const double* __restrict__ jac,
                                                           const double* __restrict__ sigma,
                                                           const int64_t* __restrict__ ptr,
                                                           const int64_t* __restrict__ code, LongRows lr, int64_t H,
                                                           int64_t J, int64_t S, int64_t ntot,
                                                           double* __restrict__ val) {
  const int64_t p = lr.idx[blockIdx.x];
  const int64_t HJ = H + J, HJS = H + J + S;
  const double s = ordered_block_sum(ptr[p], ptr[p + 1], [&](int64_t q) {
    const int64_t c = code[q];
    if (c < H) return hess[c];
    if (c < HJ) return jac[c - H];
    if (c < HJS) return -1.0;
    if (c < HJS + ntot) return sigma[c - HJS];
    return 0.0;
  });
  if (threadIdx.x == 0) val[p] = s;
}

template <class I>
__global__ void __launch_bounds__(256) sym_matvec_long_k(const double* __restrict__ val,
                                                         const int64_t* __restrict__ rptr,
                                                         const I* __restrict__ col,
                                                         const I* __restrict__ vidx, LongRows lr,
                                                         const double* __restrict__ x) {
  const int64_t r = blockIdx.y, i = lr.idx[r];
  tree_block_partial(rptr[i], rptr[i + 1], [&](int64_t p) { return val[vidx[p]] * x[col[p]]; },
                     lr.partials + r * kLongBlocks + blockIdx.x);
}

template <class I>
__global__ void __launch_bounds__(256) sym_norm_inf_long_k(const double* __restrict__ val,
                                                           const int64_t* __restrict__ rptr,
                                                           const I* __restrict__ vidx, LongRows lr) {
  const int64_t r = blockIdx.y, i = lr.idx[r];
  tree_block_partial(rptr[i], rptr[i + 1], [&](int64_t p) { return fabs(val[vidx[p]]); },
                     lr.partials + r * kLongBlocks + blockIdx.x);
}

template <class I>
__global__ void __launch_bounds__(256) jt_lambda_long_k(const double* __restrict__ jac, const double* __restrict__ lam,
                                                        const int64_t* __restrict__ ptr,
                                                        const I* __restrict__ e_idx,
                                                        const I* __restrict__ dual_idx, LongRows lr) {
  const int64_t r = blockIdx.y, i = lr.idx[r];
  tree_block_partial(ptr[i], ptr[i + 1], [&](int64_t p) { return jac[e_idx[p]] * lam[dual_idx[p]]; },
                     lr.partials + r * kLongBlocks + blockIdx.x);
}

int grid_for(int64_t n, int block) {
  const int64_t want = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(kSms) * 16;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void objective_chunk_sums(const double* objv, const int64_t* group_off, const int64_t* group_count,
                          const int64_t* chunk_base, int64_t n_chunks, int n_groups, double* partials,
                          cudaStream_t s) {
  if (n_chunks <= 0) return;
  const int blocks = static_cast<int>((n_chunks + 7) / 8);
  chunk_sums<<<blocks, 256, 0, s>>>(objv, group_off, group_count, chunk_base, n_chunks, n_groups, partials);
}

void objective_combine(const double* partials, const int64_t* chunk_base, const double* weights, int n_groups,
                       double obj_scale, double* f, int* flag, cudaStream_t s) {
  combine_chunks<<<1, 32, 0, s>>>(partials, chunk_base, weights, n_groups, obj_scale, f, flag);
}

void objective_reduce(const double* objv, const int64_t* group_off, const int64_t* group_count,
                      const int64_t* chunk_base, int64_t n_chunks, const double* weights, int n_groups,
                      double obj_scale, double* partials, double* f, int* flag, cudaStream_t s) {
  objective_chunk_sums(objv, group_off, group_count, chunk_base, n_chunks, n_groups, partials, s);
  objective_combine(partials, chunk_base, weights, n_groups, obj_scale, f, flag, s);
}

void gather_sum(const double* src, const int64_t* ptr, const int32_t* idx, int64_t n, double* out, LongRows lr,
                cudaStream_t s) {
  if (n <= 0) return;
  gather_sum_k<<<grid_for(n, 256), 256, 0, s>>>(src, ptr, idx, n, out);
  if (lr.n > 0) gather_sum_long_k<<<static_cast<unsigned>(lr.n), 256, 0, s>>>(src, ptr, idx, lr, out);
}

bool kkt_code32(const int64_t* ptr, const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot,
                uint32_t* out, cudaStream_t s) {
  if (H > kIdxMask || J > kIdxMask || ntot > kIdxMask) return false;  // indices do not fit 29 bits
  if (nnz > 0) kkt_code32_k<<<grid_for(nnz, 256), 256, 0, s>>>(ptr, code, nnz, H, J, S, ntot, out);
  return true;
}

void kkt_assemble(const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                  const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot, double* val,
                  LongRows lr, cudaStream_t s, const uint32_t* code32, const int32_t* order) {
  if (nnz <= 0) return;
  if (code32)
    kkt_assemble_fast_k<<<grid_for(nnz, 256), 256, 0, s>>>(hess, jac, sigma, code32, order, ptr, code, nnz, H, J, S,
                                                           ntot, val);
  else
    kkt_assemble_k<<<grid_for(nnz, 256), 256, 0, s>>>(hess, jac, sigma, ptr, code, nnz, H, J, S, ntot, val);
  if (lr.n > 0)
    kkt_assemble_long_k<<<static_cast<unsigned>(lr.n), 256, 0, s>>>(hess, jac, sigma, ptr, code, lr, H, J, S, ntot,
                                                                   val);
}

bool kkt_tile_plan(const uint32_t* code32_in, const int64_t* ptr, const int64_t* code, int64_t nnz, int64_t ncode,
                   const int64_t* stream_bounds_dev, int ns, int64_t H, int64_t J, int64_t S, int64_t ntot,
                   KktTiles& out, cudaStream_t s) {
  if (!code32_in || nnz <= 0 || ns <= 0 || ns > kTileMaxStreams) return false;
  const int64_t ntile = (nnz + kTileSlots - 1) / kTileSlots;
  const size_t nw = static_cast<size_t>(ntile) * static_cast<size_t>(ns);
  unsigned long long *mn = nullptr, *mx = nullptr;
  unsigned int* cnt = nullptr;
  if (cudaMallocAsync(&mn, nw * 8, s) != cudaSuccess || cudaMallocAsync(&mx, nw * 8, s) != cudaSuccess ||
      cudaMallocAsync(&cnt, nw * 4, s) != cudaSuccess)
    return false;
  cudaMemsetAsync(mn, 0xff, nw * 8, s);
  cudaMemsetAsync(mx, 0, nw * 8, s);
  cudaMemsetAsync(cnt, 0, nw * 4, s);
  // "max" starts at 0 and "min" at ~0: an untouched window has mx < mn
  kkt_tile_minmax_k<<<grid_for(nnz, 256), 256, 0, s>>>(code32_in, ptr, code, nnz, stream_bounds_dev, ns, H, J, S, mn,
                                                       mx, cnt);
  cudaMallocAsync(&out.wlo, nw * sizeof(int64_t), s);
  cudaMallocAsync(&out.wlen, nw * sizeof(int32_t), s);
  cudaMallocAsync(&out.woff, nw * sizeof(int32_t), s);
  cudaMallocAsync(&out.code32, static_cast<size_t>(nnz) * sizeof(uint32_t), s);
  cudaMallocAsync(&out.mcode, static_cast<size_t>(std::max<int64_t>(1, ncode)) * sizeof(uint32_t), s);
  kkt_tile_plan_k<<<static_cast<unsigned>((ntile + 127) / 128), 128, 0, s>>>(mn, mx, cnt, ntile, ns, nnz, out.wlo, out.wlen,
                                                                             out.woff);
  cudaMemcpyAsync(out.code32, code32_in, static_cast<size_t>(nnz) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  kkt_tile_codes_k<<<grid_for(nnz, 256), 256, 0, s>>>(out.code32, ptr, code, out.mcode, nnz, stream_bounds_dev, ns,
                                                      out.wlo, out.wlen, out.woff, H, J, S, ntot);
  if (std::getenv("OCG_KKT_TILE_STATS")) {  // diagnostic: where the slots' sources come from
    std::vector<uint32_t> c(static_cast<size_t>(nnz));
    std::vector<int32_t> len(nw);
    cudaMemcpyAsync(c.data(), out.code32, c.size() * 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(len.data(), out.wlen, len.size() * 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int64_t tags[8] = {0};
    for (uint32_t w : c) ++tags[w >> kTagShift];
    int64_t staged = 0, windows = 0;
    for (int32_t l : len) { staged += l; windows += l > 0; }
    std::fprintf(stderr, "[kkt_tile] nnz %lld tiles %lld streams %d: smem %lld hess %lld jac %lld sigma %lld -1 %lld 0 %lld multi %lld; staged %lld doubles in %lld windows (%.2f per slot)\n",
                 (long long)nnz, (long long)ntile, ns, (long long)tags[kTagSmem], (long long)tags[kTagHess],
                 (long long)tags[kTagJac], (long long)tags[kTagSigma], (long long)tags[kTagMinus1], (long long)tags[kTagZero],
                 (long long)tags[kTagMulti], (long long)staged, (long long)windows, double(staged) / double(nnz));
  }
  cudaFreeAsync(mn, s);
  cudaFreeAsync(mx, s);
  cudaFreeAsync(cnt, s);
  out.ntile = ntile;
  out.ns = ns;
  return cudaGetLastError() == cudaSuccess;
}

void kkt_assemble_tiled(const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                        const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot, double* val,
                        LongRows lr, const KktTiles& t, cudaStream_t s) {
  if (nnz <= 0) return;
  static bool attr = [] {
    return cudaFuncSetAttribute(kkt_assemble_tiled_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kTileWindow * static_cast<int>(sizeof(double)) + kTileMcode * 4) == cudaSuccess;
  }();
  (void)attr;
  kkt_assemble_tiled_k<<<static_cast<unsigned>(t.ntile), 256, kTileWindow * sizeof(double) + kTileMcode * 4, s>>>(
      hess, jac, sigma, t.code32, ptr, t.mcode, nnz, t.ns, t.wlo, t.wlen, t.woff, H, J, S, val);
  if (lr.n > 0)
    kkt_assemble_long_k<<<static_cast<unsigned>(lr.n), 256, 0, s>>>(hess, jac, sigma, ptr, code, lr, H, J, S, ntot,
                                                                   val);
}

template <class I>
void sym_matvec(const double* val, const int64_t* rptr, const I* col, const I* vidx, int64_t n,
                const double* x, double* y, LongRows lr, cudaStream_t s) {
  if (n <= 0) return;
  sym_matvec_k<<<grid_for(n, 256), 256, 0, s>>>(val, rptr, col, vidx, n, x, y);
  if (lr.n > 0) {
    sym_matvec_long_k<<<dim3(kLongBlocks, static_cast<unsigned>(lr.n)), 256, 0, s>>>(val, rptr, col, vidx, lr, x);
    long_finish_k<<<static_cast<unsigned>((lr.n + 127) / 128), 128, 0, s>>>(lr, y, 0, nullptr, nullptr, 0);
  }
}

template <class I>
void sym_norm_inf(const double* val, const int64_t* rptr, const I* vidx, int64_t n, double* out, LongRows lr,
                  cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  if (n <= 0) return;
  sym_norm_inf_k<<<grid_for(n, 256), 256, 0, s>>>(val, rptr, vidx, n, reinterpret_cast<unsigned long long*>(out));
  if (lr.n > 0) {
    sym_norm_inf_long_k<<<dim3(kLongBlocks, static_cast<unsigned>(lr.n)), 256, 0, s>>>(val, rptr, vidx, lr);
    long_finish_k<<<static_cast<unsigned>((lr.n + 127) / 128), 128, 0, s>>>(lr, out, 2, nullptr, nullptr, 0);
  }
}

template <class I>
void jt_lambda(const double* jac, const double* lam, const int64_t* ptr, const I* e_idx,
               const I* dual_idx, int64_t n_free, const int64_t* slack_dual, int64_t n_slack, double* out,
               LongRows lr, cudaStream_t s) {
  const int64_t n = n_free + n_slack;
  if (n <= 0) return;
  jt_lambda_k<<<grid_for(n, 256), 256, 0, s>>>(jac, lam, ptr, e_idx, dual_idx, n_free, slack_dual, n_slack, out);
  if (lr.n > 0) {
    jt_lambda_long_k<<<dim3(kLongBlocks, static_cast<unsigned>(lr.n)), 256, 0, s>>>(jac, lam, ptr, e_idx, dual_idx,
                                                                                   lr);
    long_finish_k<<<static_cast<unsigned>((lr.n + 127) / 128), 128, 0, s>>>(lr, out, 1, lam, slack_dual, n_free);
  }
}

void max_abs(const double* v, int64_t n, double* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  if (n <= 0) return;
  max_abs_k<<<grid_for(n, 256), 256, 0, s>>>(v, n, reinterpret_cast<unsigned long long*>(out));
}

namespace {
__global__ void long_rows_k(const int64_t* __restrict__ ptr, int64_t n, int64_t* __restrict__ out,
                            unsigned long long* __restrict__ count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (is_long(ptr, i)) out[atomicAdd(count, 1ull)] = i;
}
}  // namespace

int64_t long_rows_device(const int64_t* ptr, int64_t n, int64_t* out, cudaStream_t s) {
  unsigned long long* d = nullptr;
  cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), s);
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), s);
  if (n > 0) long_rows_k<<<grid_for(n, 256), 256, 0, s>>>(ptr, n, out, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  cudaStreamSynchronize(s);
  return static_cast<int64_t>(h);
}

std::vector<int64_t> long_rows(const std::vector<int64_t>& ptr) {
  std::vector<int64_t> out;
  for (size_t i = 0; i + 1 < ptr.size(); ++i)
    if (ptr[i + 1] - ptr[i] > kLongRow) out.push_back(static_cast<int64_t>(i));
  return out;
}

}  // namespace ocg::dev

namespace ocg::dev {

namespace {

__global__ void struct_fill_k(StructGroup g, int64_t* __restrict__ a, int64_t* __restrict__ b) {
  const int64_t cnt = g.endpoints ? (g.lo == g.hi ? 1 : 2) : g.hi - g.lo;
  const int64_t total = cnt * g.np;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = e / g.np;
    const int p = static_cast<int>(e - k * g.np);
    const int64_t idx = g.endpoints ? (k == 0 ? g.lo : g.hi) : g.lo + k;
    const int ib = g.pb[p];
    const int64_t sb = g.ibase[ib] + g.istride[ib] * idx;
    if (g.kind == 0) {
      a[g.off + e] = g.row_base + k * g.out_dim + g.pa[p];
      b[g.off + e] = sb;
    } else if (g.kind == 1) {
      const int ia = g.pa[p];
      const int64_t sa = g.ibase[ia] + g.istride[ia] * idx;
      a[g.off + e] = sa > sb ? sa : sb;
      b[g.off + e] = sa > sb ? sb : sa;
    } else {
      a[g.off + e] = sb;
    }
  }
}

__global__ void row_absmax_k(const double* __restrict__ v, const int64_t* __restrict__ row, int64_t n,
                             unsigned long long* __restrict__ out) {
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicMax(out + row[q], static_cast<unsigned long long>(__double_as_longlong(fabs(v[q]))));
}

__global__ void row_scale_rule_k(const double* __restrict__ jmax, int64_t m, double* __restrict__ rs) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rs[r] = jmax[r] > 0.0 ? fmin(1.0, 100.0 / jmax[r]) : 1.0;
}

__global__ void row_max_node_k(const int64_t* __restrict__ row, const int64_t* __restrict__ col, int64_t n,
                               const int64_t* __restrict__ col_node, unsigned long long* __restrict__ node1) {
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicMax(node1 + row[q], static_cast<unsigned long long>(col_node[col[q]] + 1));
}

__global__ void minus_one_k(unsigned long long* __restrict__ v, int64_t m) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    reinterpret_cast<int64_t*>(v)[r] = static_cast<int64_t>(v[r]) - 1;
}

int grid_n(int64_t n) {
  const int64_t want = (n + 255) / 256, cap = 148LL * 16;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void struct_fill(const StructGroup& g, int64_t* a, int64_t* b, cudaStream_t s) {
  const int64_t cnt = g.endpoints ? (g.lo == g.hi ? 1 : 2) : g.hi - g.lo;
  if (cnt * g.np <= 0) return;
  struct_fill_k<<<grid_n(cnt * g.np), 256, 0, s>>>(g, a, b);
}

void row_absmax(const double* v, const int64_t* row, int64_t n, double* out, cudaStream_t s) {
  if (n > 0) row_absmax_k<<<grid_n(n), 256, 0, s>>>(v, row, n, reinterpret_cast<unsigned long long*>(out));
}

void row_scale_rule(const double* jmax, int64_t m, double* rs, cudaStream_t s) {
  if (m > 0) row_scale_rule_k<<<grid_n(m), 256, 0, s>>>(jmax, m, rs);
}

void row_max_node(const int64_t* row, const int64_t* col, int64_t n, const int64_t* col_node, int64_t m,
                  int64_t* node, cudaStream_t s) {
  cudaMemsetAsync(node, 0, static_cast<size_t>(m) * sizeof(int64_t), s);
  if (n > 0)
    row_max_node_k<<<grid_n(n), 256, 0, s>>>(row, col, n, col_node, reinterpret_cast<unsigned long long*>(node));
  if (m > 0) minus_one_k<<<grid_n(m), 256, 0, s>>>(reinterpret_cast<unsigned long long*>(node), m);
}

template void sym_matvec<int64_t>(const double*, const int64_t*, const int64_t*, const int64_t*, int64_t, const double*,
                                   double*, LongRows, cudaStream_t);
template void sym_matvec<int32_t>(const double*, const int64_t*, const int32_t*, const int32_t*, int64_t, const double*,
                                   double*, LongRows, cudaStream_t);
template void sym_norm_inf<int64_t>(const double*, const int64_t*, const int64_t*, int64_t, double*, LongRows,
                                     cudaStream_t);
template void sym_norm_inf<int32_t>(const double*, const int64_t*, const int32_t*, int64_t, double*, LongRows,
                                     cudaStream_t);
template void jt_lambda<int64_t>(const double*, const double*, const int64_t*, const int64_t*, const int64_t*, int64_t,
                                  const int64_t*, int64_t, double*, LongRows, cudaStream_t);
template void jt_lambda<int32_t>(const double*, const double*, const int64_t*, const int32_t*, const int32_t*, int64_t,
                                  const int64_t*, int64_t, double*, LongRows, cudaStream_t);

namespace {
__global__ void narrow_k(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(in[i]);
}
}  // namespace

void narrow_i32(const int64_t* in, int64_t n, int32_t* out, cudaStream_t s) {
  if (n > 0) narrow_k<<<grid_for(n, 256), 256, 0, s>>>(in, n, out);
}

}  // namespace ocg::dev
