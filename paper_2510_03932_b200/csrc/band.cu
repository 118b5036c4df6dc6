// Device LDL^T in a node-major band-plus-border ordering, partitioned in time
// (see band.hpp for the structure and the conventions kept from the
// reference's sparse::factorize).
//
// Kernels:
//   factor_k   one thread block per banded block (segment or separator
//              system). The (b+1)x(b+1) trailing triangle of the band rolls
//              through a ring of column slots in shared memory, the border
//              rows' window likewise, and the band/border columns that enter
//              are prefetched kPrefetch columns ahead with cp.async (LDGSTS),
//              so no global-memory latency sits on the per-column path.
//   solve_k    one warp per block: forward (L), D, backward (L^T) passes with
//              the same prefetch ring; segments run their forward and
//              backward halves around the separator system's full solve.
//   schur/rhs  deterministic assembly of the segments' Schur complements and
//              right-hand-side contributions into the separator system:
//              segments of one parity touch disjoint separators; the global
//              border block is summed in segment order by one thread each.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "band.hpp"
#include "devmem.hpp"

namespace ocg {

namespace {

// factor_k's shared memory for a block of bandwidth b and w border rows with
// a kp-column prefetch ring; `owned`: compile-time shape (no pair table)
size_t factor_smem(int b, int w, int kp = 32, bool owned = false) {
  const size_t B1 = static_cast<size_t>(b) + 1, W = static_cast<size_t>(w);
  const size_t pairs = owned ? 0 : static_cast<size_t>(b) * (b + 1) / 2;
  return sizeof(double) * (B1 * B1 + B1 + W * B1 + W * (W + 1) / 2 + W + 2 * B1 + 2 * W +
                           static_cast<size_t>(kp) * (B1 + W + 2)) +
         sizeof(short) * 2 * pairs + 64;
}
// host loop [0, n) split over the host cores (iterations independent)
template <class F>
void par_range(int64_t n, F f) {
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 65536));
  if (nt <= 1) {
    f(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}

size_t solve_smem(int b, int w) {
  constexpr size_t kPre = 32;
  return sizeof(double) * (static_cast<size_t>(b) + 1 + 2 * static_cast<size_t>(w) +
                           kPre * (static_cast<size_t>(b) + 3 + w)) +
         64;
}

}  // namespace

BandPlan make_band_plan(int64_t dim, const std::vector<int64_t>& node, const std::vector<int64_t>& colp,
                        const std::vector<int64_t>& rowi, int64_t ntot, int target_segments, const DeviceCsc* dcsc,
                        int64_t** d_dst) {
  BandPlan P;
  P.dim = dim;
  P.nnz = static_cast<int64_t>(rowi.size());
  // flat node-major order: band part, then the global border
  // stable counting sort by node (border indices, node -1, last)
  std::vector<int64_t> flat(static_cast<size_t>(dim));
  std::vector<int64_t> node_start;
  {
    int64_t max_node = -1;
    for (int64_t i = 0; i < dim; ++i) max_node = std::max(max_node, node[static_cast<size_t>(i)]);
    std::vector<int64_t> start(static_cast<size_t>(max_node) + 3, 0);
    auto bucket = [&](int64_t i) {
      const int64_t v = node[static_cast<size_t>(i)];
      return static_cast<size_t>(v < 0 ? max_node + 1 : v);
    };
    for (int64_t i = 0; i < dim; ++i) start[bucket(i) + 1]++;
    for (size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
    node_start.assign(start.begin(), start.begin() + (max_node + 1));  // flat position of each node's first index
    for (int64_t i = 0; i < dim; ++i) flat[static_cast<size_t>(start[bucket(i)]++)] = i;
  }
  std::vector<int64_t> fpos(static_cast<size_t>(dim));
  par_range(dim, [&](int64_t p0, int64_t p1) {
    for (int64_t p = p0; p < p1; ++p) fpos[static_cast<size_t>(flat[static_cast<size_t>(p)])] = p;
  });
  int64_t wg = 0;
  for (int64_t i = 0; i < dim; ++i) wg += node[static_cast<size_t>(i)] < 0 ? 1 : 0;
  const int64_t n = dim - wg;
  int64_t b = 0;
  int64_t* d_fpos = nullptr;
  if (dcsc) {
    d_fpos = dev::upload_i64(fpos, dcsc->stream);
    b = dev::bandwidth(dcsc->colp, dcsc->rowi, d_fpos, n, dim, dcsc->stream);
  } else {
    for (int64_t j = 0; j < dim; ++j)
      for (int64_t q = colp[static_cast<size_t>(j)]; q < colp[static_cast<size_t>(j) + 1]; ++q) {
        const int64_t pi = fpos[static_cast<size_t>(rowi[static_cast<size_t>(q)])], pj = fpos[static_cast<size_t>(j)];
        if (pi < n && pj < n) b = std::max<int64_t>(b, pi > pj ? pi - pj : pj - pi);
      }
  }
  b = std::max<int64_t>(b, 1);
  if (b > 60) throw std::runtime_error("KKT bandwidth " + std::to_string(b) + " exceeds the band solver's limit (60)");
  P.b = static_cast<int>(b);
  P.wg = static_cast<int>(wg);

  // partition: P segments of >= 8b interior columns separated by b-wide
  // separators. Default: three segment blocks per SM (Goddard's 21 KB and
  // quadrotor's 72 KB factor blocks both fit three); two for the narrowest
  // bands (b < 12), whose iteration counts at N=2e4 moved with more segments.
  // The count follows the device's SMs (148 on B200: 444 / 296); the pinned
  // iteration counts were measured with those values.
  if (target_segments <= 0) {
    const int sms = ocg::mem::sm_count();
    target_segments = b >= 12 ? 3 * sms : 2 * sms;
  }
  int64_t nseg = std::min<int64_t>(target_segments, n / std::max<int64_t>(1, 8 * b));
  if (nseg < 2) nseg = 1;
  P.nseg = static_cast<int>(nseg);
  std::vector<int64_t> seg_lo(static_cast<size_t>(nseg)), seg_len(static_cast<size_t>(nseg));
  const int64_t interior = n - (nseg - 1) * b;
  {
    // Every segment after the first starts at a time node's first index (its
    // primal slots): the segment's first pivots are then primal blocks, not
    // duals whose primal partners sit in the separator before them — those
    // would be pivots of size ~delta_c and ruin the accuracy.
    int64_t f = 0;
    for (int64_t i = 0; i < nseg; ++i) {
      seg_lo[static_cast<size_t>(i)] = f;
      f += interior / nseg + (i < interior % nseg ? 1 : 0) + (i + 1 < nseg ? b : 0);
    }
    for (int64_t i = 1; i < nseg; ++i) {
      auto it = std::lower_bound(node_start.begin(), node_start.end(), seg_lo[static_cast<size_t>(i)]);
      if (it != node_start.end() && *it < n && *it - b > seg_lo[static_cast<size_t>(i) - 1]) seg_lo[static_cast<size_t>(i)] = *it;
    }
    for (int64_t i = 1; i < nseg; ++i)
      if (seg_lo[static_cast<size_t>(i)] - b <= seg_lo[static_cast<size_t>(i) - 1] ||
          seg_lo[static_cast<size_t>(i)] >= n)
        throw std::runtime_error("band plan: degenerate time partition");
    for (int64_t i = 0; i < nseg; ++i)
      seg_len[static_cast<size_t>(i)] =
          (i + 1 < nseg ? seg_lo[static_cast<size_t>(i) + 1] - b : n) - seg_lo[static_cast<size_t>(i)];
  }
  const int64_t n2 = (nseg - 1) * b;  // separator-system band columns
  const int wmax = nseg > 1 ? static_cast<int>(2 * b + wg) : static_cast<int>(wg);
  P.wmax = wmax;
  // positions: segment interiors in order, then separators, then the global border
  std::vector<int64_t> seg_pos(static_cast<size_t>(nseg));
  {
    int64_t p = 0;
    for (int64_t i = 0; i < nseg; ++i) {
      seg_pos[static_cast<size_t>(i)] = p;
      p += seg_len[static_cast<size_t>(i)];
    }
  }
  const int64_t sep_pos0 = interior;  // first separator-system position
  struct Loc {
    int kind;  // 0 interior of segment idx, 1 separator idx, 2 global border
    int64_t idx, local;
  };
  auto loc_of_flat = [&](int64_t f) -> Loc {
    if (f >= n) return {2, 0, f - n};
    if (nseg == 1) return {0, 0, f};
    const int64_t i = std::upper_bound(seg_lo.begin(), seg_lo.end(), f) - seg_lo.begin() - 1;
    const int64_t off = f - seg_lo[static_cast<size_t>(i)];
    if (off < seg_len[static_cast<size_t>(i)]) return {0, i, off};
    return {1, i, off - seg_len[static_cast<size_t>(i)]};
  };
  std::vector<Loc> loc(static_cast<size_t>(dim));
  P.perm.assign(static_cast<size_t>(dim), -1);
  par_range(dim, [&](int64_t f0, int64_t f1) {
    for (int64_t f = f0; f < f1; ++f) {
      const Loc L = loc_of_flat(f);
      loc[static_cast<size_t>(f)] = L;
      int64_t pos;
      if (L.kind == 0)
        pos = seg_pos[static_cast<size_t>(L.idx)] + L.local;
      else if (L.kind == 1)
        pos = sep_pos0 + L.idx * b + L.local;
      else
        pos = sep_pos0 + n2 + L.local;
      P.perm[static_cast<size_t>(pos)] = flat[static_cast<size_t>(f)];  // a permutation: disjoint writes
    }
  });
  P.primal.resize(static_cast<size_t>(dim));
  par_range(dim, [&](int64_t p0, int64_t p1) {
    for (int64_t p = p0; p < p1; ++p) P.primal[static_cast<size_t>(p)] = P.perm[static_cast<size_t>(p)] < ntot ? 1.0 : 0.0;
  });

  // blocks and their buffers
  int64_t off = 0;
  auto add_block = [&](long long nn, int bb, int ww, int early, int fin, long long pos, long long bpos) {
    BandSeg s;
    s.n = nn;
    s.b = bb;
    s.w = ww;
    s.w_early = early;
    s.finalize = fin;
    s.band = off;
    off += nn * (bb + 1);
    s.border = off;
    off += static_cast<int64_t>(ww) * nn;
    s.S = off;
    off += static_cast<int64_t>(ww) * ww;
    s.ps0 = off;
    off += nn + ww;
    s.pos = pos;
    s.bpos = bpos;
    P.segs.push_back(s);
  };
  if (nseg == 1) {
    add_block(n, static_cast<int>(b), static_cast<int>(wg), static_cast<int>(wg), 1, 0, n);
  } else {
    for (int64_t i = 0; i < nseg; ++i)
      add_block(seg_len[static_cast<size_t>(i)], static_cast<int>(b), wmax, static_cast<int>(b + wg), 0,
                seg_pos[static_cast<size_t>(i)], -1);
    add_block(n2, static_cast<int>(2 * b - 1), static_cast<int>(wg), static_cast<int>(wg), 1, sep_pos0,
              sep_pos0 + n2);
  }
  P.buf_len = off;
  // segment border rows [left sep | global | right sep] -> separator-system
  // local index (n2 + u = global row u), -1 = no such separator
  P.border_pos.assign(static_cast<size_t>(nseg) * static_cast<size_t>(std::max(wmax, 1)), -1);
  if (nseg > 1)
    for (int64_t i = 0; i < nseg; ++i)
      for (int t = 0; t < wmax; ++t) {
        int64_t v;
        if (t < b)
          v = i > 0 ? (i - 1) * b + t : -1;
        else if (t < b + wg)
          v = n2 + (t - b);
        else
          v = i + 1 < nseg ? i * b + (t - b - wg) : -1;
        P.border_pos[static_cast<size_t>(i * wmax + t)] = v;
      }

  // K entries -> buffer offsets
  auto sep_target = [&](int64_t R, int64_t C) -> int64_t {  // separator-system local indices
    const BandSeg& sep = P.segs.back();
    if (R < C) std::swap(R, C);
    if (R < n2) return sep.band + C * (sep.b + 1) + (R - C);
    if (C < n2) return sep.border + (R - n2) * n2 + C;
    return sep.S + (R - n2) * sep.w + (C - n2);
  };
  if (dcsc) {
    // the same classification per entry, on the device (dev::band_dst)
    std::vector<int8_t> lk(static_cast<size_t>(dim));
    std::vector<int64_t> li(static_cast<size_t>(dim)), ll(static_cast<size_t>(dim));
    par_range(dim, [&](int64_t f0, int64_t f1) {
      for (int64_t f = f0; f < f1; ++f) {
        lk[static_cast<size_t>(f)] = static_cast<int8_t>(loc[static_cast<size_t>(f)].kind);
        li[static_cast<size_t>(f)] = loc[static_cast<size_t>(f)].idx;
        ll[static_cast<size_t>(f)] = loc[static_cast<size_t>(f)].local;
      }
    });
    dev::BandDstIn in;
    in.colp = dcsc->colp;
    in.rowi = dcsc->rowi;
    in.fpos = d_fpos;
    in.dim = dim;
    in.n = n;
    in.b = b;
    in.wg = wg;
    in.n2 = n2;
    in.nseg = nseg;
    *d_dst = dev::band_dst(in, lk, li, ll, P.segs, dcsc->nnz, dcsc->stream);
    cudaFreeAsync(d_fpos, dcsc->stream);
  } else {
  P.dst.resize(rowi.size());
  for (int64_t j = 0; j < dim; ++j)
    for (int64_t q = colp[static_cast<size_t>(j)]; q < colp[static_cast<size_t>(j) + 1]; ++q) {
      Loc a = loc[static_cast<size_t>(fpos[static_cast<size_t>(rowi[static_cast<size_t>(q)])])];
      Loc c = loc[static_cast<size_t>(fpos[static_cast<size_t>(j)])];
      int64_t d = -1;
      if (nseg == 1) {
        const BandSeg& s = P.segs[0];
        int64_t r = a.kind == 2 ? n + a.local : a.local, cc = c.kind == 2 ? n + c.local : c.local;
        if (r < cc) std::swap(r, cc);
        if (r < n)
          d = s.band + cc * (b + 1) + (r - cc);
        else if (cc < n)
          d = s.border + (r - n) * n + cc;
        else
          d = s.S + (r - n) * s.w + (cc - n);
      } else {
        if (a.kind == 0 && c.kind != 0) std::swap(a, c);  // interior (if any) in c
        if (a.kind == 0 && c.kind == 0) {
          if (a.idx != c.idx) throw std::runtime_error("band plan: entry couples two segments");
          const BandSeg& s = P.segs[static_cast<size_t>(a.idx)];
          int64_t r = a.local, cc = c.local;
          if (r < cc) std::swap(r, cc);
          if (r - cc > b) throw std::runtime_error("band plan: entry outside the band");
          d = s.band + cc * (b + 1) + (r - cc);
        } else if (c.kind == 0) {
          const BandSeg& s = P.segs[static_cast<size_t>(c.idx)];
          int64_t t;
          if (a.kind == 2)
            t = b + a.local;
          else if (a.idx == c.idx - 1)
            t = a.local;
          else if (a.idx == c.idx)
            t = b + wg + a.local;
          else
            throw std::runtime_error("band plan: separator coupled to a distant segment");
          d = s.border + t * s.n + c.local;
        } else {
          auto sl = [&](const Loc& L) { return L.kind == 1 ? L.idx * b + L.local : n2 + L.local; };
          d = sep_target(sl(a), sl(c));
        }
      }
      P.dst[static_cast<size_t>(q)] = d;
    }
  }
  size_t sf = 0, ss = 0;
  for (const BandSeg& s : P.segs) {
    sf = std::max(sf, factor_smem(s.b, s.w));
    ss = std::max(ss, solve_smem(s.b, s.w));
  }
  P.smem_factor = sf;
  P.smem_solve = ss;
  return P;
}

namespace dev {

namespace {

constexpr int kPrefetch = 32;  // band columns in flight ahead of the window (power of two)
constexpr int kMask = kPrefetch - 1;
constexpr int kFactorThreads = 256;


__device__ __forceinline__ void cp8(double* s, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#define GRID_LOOP(i, n)                                                                  \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

// batched launches (BandBatch::ids != NULL): grid row y works on system ids[y]
__device__ __forceinline__ long long batch_id(const BandBatch& bb) { return bb.ids ? bb.ids[blockIdx.y] : 0; }

__global__ void scatter_k(const double* __restrict__ kval, const int64_t* __restrict__ dst, int64_t nnz,
                          double* __restrict__ buf, BandBatch bb) {
  const long long bi = batch_id(bb);
  kval += bi * nnz;
  buf += bi * bb.sbuf;
  GRID_LOOP(p, nnz) buf[dst[p]] = kval[p];
}

__global__ void zero_k(double* __restrict__ buf, int64_t len, BandBatch bb) {
  buf += batch_id(bb) * bb.sbuf;
  GRID_LOOP(p, len) buf[p] = 0.0;
}

__device__ __forceinline__ bool zero_pivot(double d, double scale) {
  return !(fabs(d) <= DBL_MAX) || fabs(d) <= 1e-14 * fmax(scale, 1e-30);
}

// One thread block per banded block (blockIdx.x indexes `segs` from seg0).
// Specialized at compile time on the bandwidth and border widths of the
// blocks a model produces (BC = b + 1, WC = border rows, WEC = rows coupled
// from column 0; 0 / -1 = read them from the descriptor), so the per-column
// loops have constant trip counts and constant divisors.
template <int BC, int WC, int WEC, int TT>
__global__ void __launch_bounds__(TT) factor_k(const BandSeg* __restrict__ segs, int seg0,
                                                           double* __restrict__ buf,
                                                           const double* __restrict__ primal, double dw, double dc,
                                                           double* __restrict__ Dinv,
                                                           long long* __restrict__ inertia_parts, BandBatch bb) {
  extern __shared__ double sm[];
  const BandSeg g = segs[seg0 + blockIdx.x];
  if (bb.ids) {
    const long long bi = bb.ids[blockIdx.y];
    buf += bi * bb.sbuf;
    Dinv += bi * bb.sdim;
    inertia_parts += bi * bb.sparts;
    if (bb.dw) {
      dw = bb.dw[blockIdx.y];
      dc = bb.dc[blockIdx.y];
    }
  }
  constexpr int T = TT;
  // compile-time shapes: deep windows prefetch 16 columns (shared memory for 3
  // blocks per SM), and the update pairs live in registers, not a table
  constexpr bool kOwned = BC > 0 && WEC >= 0;
  constexpr int KP = (BC > 0 && WC >= 0 && BC + WC > 96) ? 16 : kPrefetch;
  constexpr int KM = KP - 1;
  const int tid = threadIdx.x;
  const long long n = g.n;
  const int B1 = BC > 0 ? BC : g.b + 1;
  const int b = B1 - 1;
  const int w = WC >= 0 ? WC : g.w;
  const int we = WEC >= 0 ? WEC : g.w_early;
  double* W = sm;                 // B1 * B1 (slot-major)
  double* ps = W + B1 * B1;       // B1
  double* Wb = ps + B1;           // w * B1
  double* S = Wb + w * B1;        // w (w + 1) / 2: lower triangle, row-packed
  double* Sps = S + w * (w + 1) / 2;  // w
  double* y = Sps + w;            // B1
  double* l = y + B1;             // B1
  double* yb = l + B1;            // w
  double* lb = yb + w;            // w
  double* ring = lb + w;          // KP * RW
  const int RW = B1 + w + 2;      // ring row: band column, its border entries, regularization flag, pivot-scale seed
  short* pj1 = reinterpret_cast<short*>(ring + KP * RW);  // pair table (generic shapes only)
  const int P = b * (b + 1) / 2;
  short* pj2 = pj1 + P;
  double* band = buf + g.band;
  double* border = buf + g.border;
  double* Sg = buf + g.S;
  double* ps0 = buf + g.ps0;  // pivot-scale seeds: [n] interior, then [w] border
  const double* flag = primal + g.pos;
  double* dinvp = Dinv + g.pos;

  auto sidx = [](int t, int u) { return t * (t + 1) / 2 + u; };  // packed lower S
  if constexpr (!kOwned)
    for (int p = tid; p < P; p += T) {  // pairs j1 <= j2 in 1..b
      int j1 = 1, rem = p;
      while (rem >= b - j1 + 1) {
        rem -= b - j1 + 1;
        ++j1;
      }
      pj1[p] = static_cast<short>(j1);
      pj2[p] = static_cast<short>(j1 + rem);
    }
  auto delta_of = [&](double f) { return f != 0.0 ? dw : -dc; };
  auto fetch = [&](long long c, int r) {  // column c -> ring row r (async)
    double* dstp = ring + r * RW;
#pragma unroll
    for (int j = tid; j < B1; j += T) {
      if (c + j < n)
        cp8(dstp + j, band + c * B1 + j);
      else
        dstp[j] = 0.0;
    }
#pragma unroll
    for (int t = tid; t < w; t += T) cp8(dstp + B1 + t, border + static_cast<long long>(t) * n + c);
    if (tid == 0) {
      cp8(dstp + B1 + w, flag + c);
      cp8(dstp + B1 + w + 1, ps0 + c);
    }
  };
  for (long long c = 0; c < B1 && c < n; ++c) {
    for (int j = tid; j < B1; j += T) {
      double v = c + j < n ? band[c * B1 + j] : 0.0;
      if (j == 0) {
        v += delta_of(flag[c]);
        ps[c] = fmax(fabs(v), ps0[c]);
      }
      W[c * B1 + j] = v;
    }
    for (int t = tid; t < w; t += T) Wb[t * B1 + c] = border[static_cast<long long>(t) * n + c];
  }
  for (int r = 0; r < KP; ++r) {
    if (B1 + r < n) fetch(B1 + r, r);
    cp_commit();
  }
  for (int q = tid; q < w * w; q += T) {
    const int t = q / w, u = q % w;
    if (u > t) continue;
    double v = Sg[q];
    if (t == u) {
      if (g.finalize) v += delta_of(primal[g.bpos + t]);
      Sps[t] = fmax(fabs(v), ps0[n + t]);
    }
    S[sidx(t, u)] = v;
  }
  long long npos = 0, nneg = 0, nzero = 0;
  // compile-time shapes: each thread owns its rank-1-update pairs (j1, j2) and
  // early border entries (t, j) in registers, so a column's update is a few
  // shared-memory read-modify-writes with no index arithmetic or table loads
  constexpr int kPairs = BC > 0 ? (BC - 1) * BC / 2 : 0;
  constexpr int kPPT = kOwned && kPairs > 0 ? (kPairs + TT - 1) / TT : 1;
  constexpr int kWb = kOwned ? WEC * (BC - 1) : 0;
  constexpr int kWPT = kOwned && kWb > 0 ? (kWb + TT - 1) / TT : 1;
  int oj1[kPPT], oj2[kPPT], ot[kWPT], oj[kWPT];
  if constexpr (kOwned) {
#pragma unroll
    for (int i = 0; i < kPPT; ++i) {
      const int p = tid + i * TT;
      oj1[i] = oj2[i] = 0;
      if (p < kPairs) {
        int j1 = 1, rem = p;
        while (rem >= (BC - 1) - j1 + 1) {
          rem -= (BC - 1) - j1 + 1;
          ++j1;
        }
        oj1[i] = j1;
        oj2[i] = j1 + rem;
      }
    }
#pragma unroll
    for (int i = 0; i < kWPT; ++i) {
      const int q = tid + i * TT;
      ot[i] = q < kWb ? q / (BC - 1) : -1;
      oj[i] = q < kWb ? q - (q / (BC - 1)) * (BC - 1) + 1 : 0;
    }
  }
  __syncthreads();

  int s = 0;  // slot of column k = k mod B1
  for (long long k = 0; k < n; ++k, s = (s + 1 == B1 ? 0 : s + 1)) {
    const double d = W[s * B1];
    const bool zero = zero_pivot(d, ps[s]);
    const double dinv = zero ? 0.0 : 1.0 / d;
    if (tid == 0) {
      dinvp[k] = dinv;
      band[k * B1] = d;
      if (zero)
        ++nzero;
      else if (d > 0)
        ++npos;
      else
        ++nneg;
    }
    const bool late = k + b >= n;  // the last b columns: every border row coupled
    const int wa = late ? w : we;
#pragma unroll
    for (int j = tid + 1; j < B1; j += T) {
      const double yj = k + j < n ? W[s * B1 + j] : 0.0;
      const double lj = yj * dinv;
      y[j] = yj;
      l[j] = lj;
      if (k + j < n) band[k * B1 + j] = lj;
    }
#pragma unroll
    for (int t = tid; t < w; t += T) {
      const double v = t < wa ? Wb[t * B1 + s] : 0.0;
      yb[t] = v;
      lb[t] = v * dinv;
      border[static_cast<long long>(t) * n + k] = v * dinv;
    }
    __syncthreads();
    if constexpr (kOwned) {
#pragma unroll
      for (int i = 0; i < kPPT; ++i) {
        const int j1 = oj1[i], j2 = oj2[i];
        if (j1 > 0 && (!late || k + j2 < n)) {
          const int s1 = s + j1 >= B1 ? s + j1 - B1 : s + j1;
          const double upd = l[j2] * y[j1];
          W[s1 * B1 + (j2 - j1)] -= upd;
          if (j1 == j2) ps[s1] = fmax(ps[s1], fabs(upd));
        }
      }
    } else {
#pragma unroll 4
      for (int p = tid; p < P; p += T) {
        const int j1 = pj1[p], j2 = pj2[p];
        if (!late || k + j2 < n) {
          const int s1 = s + j1 >= B1 ? s + j1 - B1 : s + j1;
          const double upd = l[j2] * y[j1];
          W[s1 * B1 + (j2 - j1)] -= upd;
          if (j1 == j2) ps[s1] = fmax(ps[s1], fabs(upd));
        }
      }
    }
    if (!late) {
      if constexpr (kOwned) {
#pragma unroll
        for (int i = 0; i < kWPT; ++i) {
          const int t = ot[i], j = oj[i];
          if (t >= 0) Wb[t * B1 + (s + j >= B1 ? s + j - B1 : s + j)] -= lb[t] * y[j];
        }
      } else {
#pragma unroll 4
        for (int q = tid; q < we * b; q += T) {
          const int t = q / b, j = q - t * b + 1;
          Wb[t * B1 + (s + j >= B1 ? s + j - B1 : s + j)] -= lb[t] * y[j];
        }
      }
      // the early rows' border block S is updated after the loop, from the
      // stored border factor (one pass over the segment, not a per-column step)
    } else {
      for (int q = tid; q < w * b; q += T) {
        const int t = q / b, j = q - t * b + 1;
        if (k + j < n) Wb[t * B1 + (s + j >= B1 ? s + j - B1 : s + j)] -= lb[t] * y[j];
      }
      for (int q = tid; q < w * w; q += T) {
        const int t = q / w, u = q - t * w;
        if (u <= t) {
          const double upd = lb[t] * yb[u];
          S[sidx(t, u)] -= upd;
          if (t == u) Sps[t] = fmax(Sps[t], fabs(upd));
        }
      }
    }
    // column k is final: its slot takes column k + B1 from the prefetch ring.
    // No barrier before the refill: every thread reads back exactly the ring
    // entries its own cp.async copied (same j / t mapping as fetch), slot s
    // was last read before the barrier above (the multipliers), and this
    // column's updates above write only slots s+1 .. s+b and ps of those.
    cp_wait<KP - 1>();
    const long long cin = k + B1;
    if (cin < n) {
      const double* src = ring + static_cast<int>(k & KM) * RW;
#pragma unroll
      for (int j = tid; j < B1; j += T) {
        double v = src[j];
        if (j == 0) {
          v += delta_of(src[B1 + w]);
          ps[s] = fmax(fabs(v), src[B1 + w + 1]);
        }
        W[s * B1 + j] = v;
      }
#pragma unroll
      for (int t = tid; t < w; t += T) Wb[t * B1 + s] = src[B1 + t];
    }
    __syncthreads();
    if (cin + KP < n) fetch(cin + KP, static_cast<int>(k & KM));
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();
  {
    // deferred early updates of S: S[t][u] -= sum_k L[t][k] d_k L[u][k] over
    // the columns k < n - b (rows t, u < we), staged through the ring's shared
    // memory in chunks of columns
    const long long n_early = n > b ? n - b : 0;
    const int CH = min(32, (KP * RW) / max(1, 2 * we));
    double* lc = ring;            // we x CH: L[t][k]
    double* yc = ring + we * CH;  // we x CH: L[u][k] d_k
    const int npair = we * (we + 1) / 2;
    for (long long c0 = 0; c0 < n_early; c0 += CH) {
      const int m = static_cast<int>(min(static_cast<long long>(CH), n_early - c0));
      for (int e = tid; e < we * CH; e += T) {
        const int t = e / CH, j = e - t * CH;
        if (j < m) {
          const double lv = border[static_cast<long long>(t) * n + c0 + j];
          lc[e] = lv;
          yc[e] = lv * band[(c0 + j) * B1];
        }
      }
      __syncthreads();
      for (int q = tid; q < npair; q += T) {
        int t = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
        while ((t + 1) * (t + 2) / 2 <= q) ++t;
        while (t * (t + 1) / 2 > q) --t;
        const int u = q - t * (t + 1) / 2;
        double acc = S[sidx(t, u)], mx = 0.0;
        for (int j = 0; j < m; ++j) {
          const double upd = lc[t * CH + j] * yc[u * CH + j];
          acc -= upd;
          mx = fmax(mx, fabs(upd));
        }
        S[sidx(t, u)] = acc;
        if (t == u) Sps[t] = fmax(Sps[t], mx);
      }
      __syncthreads();
    }
  }
  if (g.finalize) {
    // dense border block: sequential LDL^T with the same pivot rule
    if (tid == 0) {
      for (int t = 0; t < w; ++t) {
        const double d = S[sidx(t, t)];
        const bool zero = zero_pivot(d, Sps[t]);
        const double dinv = zero ? 0.0 : 1.0 / d;
        Dinv[g.bpos + t] = dinv;
        Sg[t * w + t] = d;
        if (zero)
          ++nzero;
        else if (d > 0)
          ++npos;
        else
          ++nneg;
        for (int u = t + 1; u < w; ++u) {
          const double lu = S[sidx(u, t)] * dinv;
          for (int v = t + 1; v <= u; ++v) {
            const double upd = lu * S[sidx(v, t)];
            S[sidx(u, v)] -= upd;
            if (u == v) Sps[u] = fmax(Sps[u], fabs(upd));
          }
        }
        for (int u = t + 1; u < w; ++u) Sg[u * w + t] = S[sidx(u, t)] * dinv;
      }
    }
  } else {
    for (int q = tid; q < w * w; q += T) {  // Schur complement on the border rows (lower)
      const int t = q / w, u = q % w;
      if (u <= t) Sg[q] = S[sidx(t, u)];
    }
    for (int t = tid; t < w; t += T) ps0[n + t] = Sps[t];   // and its diagonal's largest single update
  }
  if (tid == 0) {
    long long* o = inertia_parts + 3 * (seg0 + blockIdx.x);
    o[0] = npos;
    o[1] = nneg;
    o[2] = nzero;
  }
}

using FactorKernel = void (*)(const BandSeg*, int, double*, const double*, double, double, double*, long long*,
                              BandBatch);

// instantiations for the blocks of the shipped models (segment: b + 1,
// 2b + wg, b + wg, many blocks of 256 threads; separator system: 2b, wg, wg,
// one block of 1024 threads), else the generic kernels
// *smem: the dynamic shared memory of the returned kernel
FactorKernel factor_kernel_for(int B1, int w, int we, bool single, int threads, size_t* smem) {
#define OCG_FK(a, c, e, t)                                                                          \
  if (B1 == (a) && w == (c) && we == (e) && single == ((t) == 1024) && (single || threads == (t))) { \
    *smem = factor_smem((a) - 1, (c), (a) + (c) > 96 ? 16 : kPrefetch, true);                       \
    return factor_k<a, c, e, t>;                                                                     \
  }
  OCG_FK(9, 16, 8, 128)    // small bands: 128-thread segment blocks (fewer warps per barrier)
  OCG_FK(13, 25, 13, 128)
  OCG_FK(17, 32, 16, 128)
  OCG_FK(9, 16, 8, 256)    // double integrator (b 8, wg 0)
  OCG_FK(16, 0, 0, 1024)
  OCG_FK(13, 25, 13, 256)  // Goddard (b 12, wg 1)
  OCG_FK(24, 1, 1, 1024)
  OCG_FK(17, 32, 16, 256)  // cart-pendulum (b 16, wg 0)
  OCG_FK(32, 0, 0, 1024)
  OCG_FK(18, 35, 18, 256)  // hang glider (b 17, wg 1)
  OCG_FK(34, 1, 1, 1024)
  OCG_FK(28, 55, 28, 256)  // shuttle (b 27, wg 1)
  OCG_FK(54, 1, 1, 1024)
  OCG_FK(38, 74, 37, 256)  // quadrotor (b 37, wg 0)
  OCG_FK(74, 0, 0, 1024)
#undef OCG_FK
  *smem = factor_smem(B1 - 1, w, kPrefetch, false);
  return single ? factor_k<0, -1, -1, 1024> : factor_k<0, -1, -1, 256>;
}

// ---- one warp per system: unpartitioned bands without a border, b + 1 <= 32 ----
//
// factor_k's algorithm and arithmetic for one small band per warp: the
// (b+1) x (b+1) window in the warp's shared memory as a ring of column slots
// (column k in slot k mod (b+1)), the rank-1 update spread over the lanes by
// a fixed pair assignment held in registers, __syncwarp instead of block
// barriers, and the column entering the window loaded PF columns ahead into
// registers (lane j holds its entry j: coalesced).
constexpr unsigned kFull = 0xffffffffu;

template <int B1, int PF>
__global__ void __launch_bounds__(128) factor_warp_k(const BandSeg* __restrict__ segs, double* __restrict__ buf,
                                                     const double* __restrict__ primal, double* __restrict__ Dinv,
                                                     long long* __restrict__ inertia, BandBatch bb, int nb) {
  constexpr int b = B1 - 1;
  constexpr int P = b * (b + 1) / 2;     // update pairs j1 <= j2 in 1..b
  constexpr int T = (P + 31) / 32;       // pairs per lane
  constexpr int WS = B1 * B1 + 3 * B1;   // shared doubles per warp: window, pivot scales, y, l
  __shared__ double smem[4 * WS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int yidx = blockIdx.x * 4 + wib;
  if (yidx >= nb) return;  // warp-uniform
  double* W = smem + wib * WS;
  double* ps = W + B1 * B1;
  double* yv = ps + B1;
  double* lv = yv + B1;
  const long long bi = bb.ids[yidx];
  const double dw = bb.dw[yidx], dc = bb.dc[yidx];
  const BandSeg g = segs[0];
  const long long n = g.n;
  double* band = buf + bi * bb.sbuf + g.band;
  double* dinvp = Dinv + bi * bb.sdim + g.pos;
  const double* flag = primal + g.pos;
  // this lane's update pairs (fixed for the whole factorization)
  int pj1[T], pj2[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int p = lane + 32 * t;
    int j1 = 1, rem = p < P ? p : 0;
    while (rem >= b - j1 + 1) {
      rem -= b - j1 + 1;
      ++j1;
    }
    pj1[t] = p < P ? j1 : 0;
    pj2[t] = p < P ? j1 + rem : 0;
  }
  // column c entry `lane` (+ delta on the diagonal), 0 outside the matrix
  auto column = [&](long long c) -> double {
    if (lane >= B1 || c >= n || c + lane >= n) return 0.0;
    double v = band[c * B1 + lane];
    if (lane == 0) v += flag[c] != 0.0 ? dw : -dc;
    return v;
  };
  for (int c = 0; c < B1; ++c) {
    const double v = column(c);
    if (lane < B1) W[c * B1 + lane] = v;
    if (lane == 0) ps[c] = fabs(v);
  }
  // prefetched raw column entries and (lane 0) regularization flags: the
  // delta is applied when the column enters the window, so no arithmetic
  // waits on a load at prefetch time
  auto raw = [&](long long c) -> double {
    return lane < B1 && c < n && c + lane < n ? band[c * B1 + lane] : 0.0;
  };
  auto rawflag = [&](long long c) -> double { return lane == 0 && c < n ? flag[c] : 0.0; };
  double pf[PF], pff[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    pf[q] = raw(B1 + q);
    pff[q] = rawflag(B1 + q);
  }
  __syncwarp();
  long long npos = 0, nneg = 0, nzero = 0;
  int s = 0;
  for (long long k0 = 0; k0 < n; k0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const long long k = k0 + q;
      if (k >= n) break;
      const double d = W[s * B1];
      const bool zero = zero_pivot(d, ps[s]);
      const double dinv = zero ? 0.0 : 1.0 / d;
      if (lane == 0) {
        dinvp[k] = dinv;
        band[k * B1] = d;
        if (zero)
          ++nzero;
        else if (d > 0)
          ++npos;
        else
          ++nneg;
      } else if (lane < B1) {
        const double yj = k + lane < n ? W[s * B1 + lane] : 0.0;
        const double lj = yj * dinv;
        yv[lane] = yj;
        lv[lane] = lj;
        if (k + lane < n) band[k * B1 + lane] = lj;
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (lane + 32 * t < P) {
          const int j1 = pj1[t], j2 = pj2[t];
          const int s1 = s + j1 >= B1 ? s + j1 - B1 : s + j1;
          const double upd = lv[j2] * yv[j1];
          W[s1 * B1 + (j2 - j1)] -= upd;
          if (j1 == j2) ps[s1] = fmax(ps[s1], fabs(upd));
        }
      }
      __syncwarp();
      // column k is final: its slot takes column k + B1
      double vin = pf[q];
      if (lane == 0 && k + B1 < n) vin += pff[q] != 0.0 ? dw : -dc;
      if (lane < B1) W[s * B1 + lane] = vin;
      if (lane == 0) ps[s] = fabs(vin);
      pf[q] = raw(k + B1 + PF);
      pff[q] = rawflag(k + B1 + PF);
      s = s + 1 == B1 ? 0 : s + 1;
      __syncwarp();
    }
  }
  if (lane == 0) {
    long long* o = inertia + bi * bb.sparts;
    o[0] = npos;
    o[1] = nneg;
    o[2] = nzero;
  }
}

// forward, diagonal and backward substitution with the factor of factor_warp_k
// (solve_k mode 0's arithmetic): the forward window z[c+j] and the backward
// window x[c+j] sit one entry per lane
template <int B1, int PF>
__global__ void __launch_bounds__(128) solve_warp_k(const BandSeg* __restrict__ segs, const double* __restrict__ buf,
                                                    const double* __restrict__ Dinv, double* __restrict__ work,
                                                    BandBatch bb, int nb) {
  const int lane = threadIdx.x & 31;
  const int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (y >= nb) return;
  const long long bi = bb.ids[y];
  const BandSeg g = segs[0];
  const long long n = g.n;
  constexpr int b = B1 - 1;
  const double* band = buf + bi * bb.sbuf + g.band;
  const double* dinv = Dinv + bi * bb.sdim + g.pos;
  double* v = work + bi * bb.swork + g.pos;
  const bool col_lane = lane >= 1 && lane < B1;
  auto lcol = [&](long long c) -> double {  // L(c + lane, c)
    return (col_lane && c >= 0 && c + lane < n) ? band[c * B1 + lane] : 0.0;
  };
  // ---- forward: L z = rhs
  double z = lane < B1 && lane < n ? v[lane] : 0.0;
  double pl[PF], pv[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    pl[q] = lcol(q);
    pv[q] = (lane == b && q + B1 < n) ? v[q + B1] : 0.0;
  }
  for (long long c0 = 0; c0 < n; c0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const long long c = c0 + q;
      if (c >= n) break;
      const double yc = __shfl_sync(kFull, z, 0);
      if (lane == 0) v[c] = yc;
      z -= pl[q] * yc;
      z = __shfl_down_sync(kFull, z, 1);
      if (lane == b) z = pv[q];
      pl[q] = lcol(c + PF);
      pv[q] = (lane == b && c + PF + B1 < n) ? v[c + PF + B1] : 0.0;
    }
  }
  // ---- backward: x_c = z_c * dinv_c - sum_j L(c+j, c) x_{c+j}
  double xw = 0.0;  // lane j: x[c + j]
  double pz[PF], pd[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    const long long c = n - 1 - q;
    pl[q] = lcol(c);
    pz[q] = c >= 0 ? v[c] : 0.0;
    pd[q] = c >= 0 ? dinv[c] : 0.0;
  }
  for (long long c0 = n - 1; c0 >= 0; c0 -= PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const long long c = c0 - q;
      if (c < 0) break;
      double part = pl[q] * xw;
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
      const double xc = pz[q] * pd[q] - part;
      if (lane == 0) v[c] = xc;
      xw = __shfl_up_sync(kFull, xw, 1);
      if (lane == 1) xw = xc;
      const long long cn = c - PF;
      pl[q] = lcol(cn);
      pz[q] = cn >= 0 ? v[cn] : 0.0;
      pd[q] = cn >= 0 ? dinv[cn] : 0.0;
    }
  }
}

using FactorWarpKernel = void (*)(const BandSeg*, double*, const double*, double*, long long*, BandBatch, int);
using SolveWarpKernel = void (*)(const BandSeg*, const double*, const double*, double*, BandBatch, int);

template <int B1>
void warp_kernels(FactorWarpKernel& f, SolveWarpKernel& s) {
  f = factor_warp_k<B1, 8>;
  s = solve_warp_k<B1, 8>;
}

bool warp_kernels_for(int B1, FactorWarpKernel& f, SolveWarpKernel& s) {
  switch (B1) {
#define OCG_WK(a) \
  case a:         \
    warp_kernels<a>(f, s); \
    return true;
    OCG_WK(2) OCG_WK(3) OCG_WK(4) OCG_WK(5) OCG_WK(6) OCG_WK(7) OCG_WK(8) OCG_WK(9) OCG_WK(10) OCG_WK(11)
    OCG_WK(12) OCG_WK(13) OCG_WK(14) OCG_WK(15) OCG_WK(16) OCG_WK(17) OCG_WK(18) OCG_WK(19) OCG_WK(20)
    OCG_WK(21) OCG_WK(22) OCG_WK(23) OCG_WK(24) OCG_WK(25) OCG_WK(26) OCG_WK(27) OCG_WK(28) OCG_WK(29)
    OCG_WK(30) OCG_WK(31) OCG_WK(32)
#undef OCG_WK
    default:
      return false;
  }
}

// unpartitioned bands of many small systems (batched solves): 128 threads per
// system, several systems per SM
FactorKernel factor_kernel_batch(int B1, int w, int we, size_t* smem) {
#define OCG_FKB(a, c, e)                                                        \
  if (B1 == (a) && w == (c) && we == (e)) {                                     \
    *smem = factor_smem((a) - 1, (c), (a) + (c) > 96 ? 16 : kPrefetch, true);   \
    return factor_k<a, c, e, 128>;                                              \
  }
  OCG_FKB(9, 0, 0)    // double integrator
  OCG_FKB(13, 1, 1)   // Goddard
  OCG_FKB(17, 0, 0)   // cart-pendulum
  OCG_FKB(18, 1, 1)   // hang glider
  OCG_FKB(28, 1, 1)   // shuttle
  OCG_FKB(38, 0, 0)   // quadrotor
#undef OCG_FKB
  *smem = factor_smem(B1 - 1, w, kPrefetch, false);
  return factor_k<0, -1, -1, 128>;
}

// segments of parity `par` add their Schur complements into the separator
// system (disjoint separators within a parity); global-global entries skipped
__global__ void schur_add_k(const BandSeg* __restrict__ segs, int nseg, int par, int wmax,
                            const int64_t* __restrict__ border_pos, double* __restrict__ buf, BandBatch bb) {
  buf += batch_id(bb) * bb.sbuf;
  const BandSeg sep = segs[nseg];
  const long long n2 = sep.n;
  const int64_t per = static_cast<int64_t>(wmax) * wmax;
  const int64_t cnt = static_cast<int64_t>((nseg - par + 1) / 2) * per;
  GRID_LOOP(q, cnt) {
    const int i = par + 2 * static_cast<int>(q / per);
    const int t = static_cast<int>((q % per) / wmax), u = static_cast<int>(q % wmax);
    if (u > t) continue;
    int64_t R = border_pos[static_cast<int64_t>(i) * wmax + t], C = border_pos[static_cast<int64_t>(i) * wmax + u];
    if (R < 0 || C < 0 || (R >= n2 && C >= n2)) continue;
    const double v = buf[segs[i].S + static_cast<int64_t>(t) * wmax + u];
    if (R < C) {
      const int64_t tmp = R;
      R = C;
      C = tmp;
    }
    int64_t dst;
    if (R < n2)
      dst = sep.band + C * (sep.b + 1) + (R - C);
    else
      dst = sep.border + (R - n2) * n2 + C;
    buf[dst] += v;
    if (t == u) {  // R == C < n2: a separator pivot; separators are disjoint within a parity
      double& sc = buf[sep.ps0 + R];
      sc = fmax(sc, buf[segs[i].ps0 + segs[i].n + t]);
    }
  }
}

// global-global block: every segment contributes, summed in segment order
__global__ void schur_global_k(const BandSeg* __restrict__ segs, int nseg, int wmax, int b, int wg,
                               double* __restrict__ buf, BandBatch bb) {
  buf += batch_id(bb) * bb.sbuf;
  const BandSeg sep = segs[nseg];
  GRID_LOOP(q, static_cast<int64_t>(wg) * wg) {
    const int u = static_cast<int>(q / wg), v = static_cast<int>(q % wg);
    if (v > u) continue;
    double acc = 0.0, sc = 0.0;
    for (int i = 0; i < nseg; ++i) {
      acc += buf[segs[i].S + static_cast<int64_t>(b + u) * wmax + (b + v)];
      if (u == v) sc = fmax(sc, buf[segs[i].ps0 + segs[i].n + b + u]);
    }
    buf[sep.S + static_cast<int64_t>(u) * sep.w + v] += acc;
    if (u == v) buf[sep.ps0 + sep.n + u] = sc;
  }
}

__global__ void inertia_sum_k(const long long* __restrict__ parts, int nblocks, long long* __restrict__ out,
                              BandBatch bb) {
  // integer counts: one warp, lane-strided sums and a shuffle tree (exact in
  // any order)
  if (blockIdx.x != 0) return;
  if (bb.ids) {
    const long long bi = bb.ids[blockIdx.y];
    parts += bi * bb.sparts;
    out += bi * 3;
  }
  long long a = 0, c = 0, z = 0;
  for (int i = threadIdx.x; i < nblocks; i += 32) {
    a += parts[3 * i];
    c += parts[3 * i + 1];
    z += parts[3 * i + 2];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
    z += __shfl_xor_sync(0xffffffffu, z, o);
  }
  if (threadIdx.x != 0) return;
  out[0] = a;
  out[1] = c;
  out[2] = z;
}

__global__ void gather_k(const double* __restrict__ rhs, const int64_t* __restrict__ perm, int64_t dim,
                         double* __restrict__ out, BandBatch bb) {
  const long long bi = batch_id(bb);
  rhs += bi * bb.sdim;
  out += bi * bb.swork;
  GRID_LOOP(p, dim) out[p] = rhs[perm[p]];
}

__global__ void scatter_back_k(const double* __restrict__ work, const int64_t* __restrict__ perm, int64_t dim,
                               double* __restrict__ x, BandBatch bb) {
  const long long bi = batch_id(bb);
  work += bi * bb.swork;
  x += bi * bb.sdim;
  GRID_LOOP(p, dim) x[perm[p]] = work[p];
}

// mode 0: full solve of a finalized block (forward, border block, D, backward)
// mode 1: segment forward; border accumulations -> gparts[blk * wmax + t]
// mode 2: segment backward with the separator system's solution as border values
// Segment forward (mode 1) / backward (mode 2) substitution with the window
// in registers: lane j holds window entries j, j + 32, ... (NW per lane) and
// border rows lane, lane + 32, ... (NBW per lane); a column is a broadcast,
// one FMA per held entry and a shuffle shift (forward) or a warp sum
// (backward) — no shared memory, no warp barriers. Column data is prefetched
// PF columns ahead into registers. solve_k's arithmetic per entry (the
// backward's warp sum groups the terms differently).
template <int PF, int NW, int NBW>
__global__ void __launch_bounds__(32) solve_seg_warp_k(const BandSeg* __restrict__ segs, int mode,
                                                       const double* __restrict__ buf,
                                                       const double* __restrict__ Dinv, double* __restrict__ work,
                                                       double* __restrict__ gparts, int wmax,
                                                       const int64_t* __restrict__ border_pos, long long sep_pos0) {
  const int blk = blockIdx.x;
  const BandSeg g = segs[blk];
  const int lane = threadIdx.x;
  const long long n = g.n;
  const int B1 = g.b + 1, w = g.w;
  const double* band = buf + g.band;
  const double* border = buf + g.border;
  double* v = work + g.pos;
  const double* dinv = Dinv + g.pos;
  const int last = B1 - 1;  // window entry that takes the incoming value
  auto colb = [&](long long c, int r) {
    const int e = lane + 32 * r;
    return e > 0 && e < B1 && c >= 0 && c < n && c + e < n ? band[c * B1 + e] : 0.0;
  };
  auto colw = [&](long long c, int r) {
    const int t = lane + 32 * r;
    return t < w && c >= 0 && c < n ? border[static_cast<long long>(t) * n + c] : 0.0;
  };
  if (mode == 1) {
    double Y[NW], yb[NBW];
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int e = lane + 32 * r;
      Y[r] = e < B1 && e < n ? v[e] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < NBW; ++r) yb[r] = 0.0;
    auto colv = [&](long long c) { return lane == last % 32 && c + B1 < n ? v[c + B1] : 0.0; };
    double pb[PF][NW], pw[PF][NBW], pv[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
#pragma unroll
      for (int r = 0; r < NW; ++r) pb[q][r] = colb(q, r);
#pragma unroll
      for (int r = 0; r < NBW; ++r) pw[q][r] = colw(q, r);
      pv[q] = colv(q);
    }
    for (long long c0 = 0; c0 < n; c0 += PF) {
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const long long c = c0 + q;
        if (c >= n) break;
        const double yc = __shfl_sync(0xffffffffu, Y[0], 0);
        if (lane == 0) v[c] = yc;
#pragma unroll
        for (int r = 0; r < NW; ++r) Y[r] -= pb[q][r] * yc;
#pragma unroll
        for (int r = 0; r < NBW; ++r) yb[r] -= pw[q][r] * yc;
        // shift: entry e takes entry e + 1; entry B1 - 1 takes v[c + B1]
#pragma unroll
        for (int r = 0; r < NW; ++r) {
          double dn = __shfl_down_sync(0xffffffffu, Y[r], 1);
          if (r + 1 < NW) {
            const double nx = __shfl_sync(0xffffffffu, Y[r + 1 < NW ? r + 1 : r], 0);
            if (lane == 31) dn = nx;
          }
          if (r == last / 32 && lane == last % 32) dn = pv[q];
          Y[r] = dn;
        }
#pragma unroll
        for (int r = 0; r < NW; ++r) pb[q][r] = colb(c + PF, r);
#pragma unroll
        for (int r = 0; r < NBW; ++r) pw[q][r] = colw(c + PF, r);
        pv[q] = colv(c + PF);
      }
    }
#pragma unroll
    for (int r = 0; r < NBW; ++r)
      if (lane + 32 * r < w) gparts[static_cast<int64_t>(blk) * wmax + lane + 32 * r] = yb[r];
    return;
  }
  // mode 2: backward with the separator system's solution as border values
  double xb[NBW], X[NW];
#pragma unroll
  for (int r = 0; r < NBW; ++r) {
    const int t = lane + 32 * r;
    xb[r] = 0.0;
    if (t < w) {
      const int64_t q = border_pos[static_cast<int64_t>(blk) * wmax + t];
      xb[r] = q >= 0 ? work[sep_pos0 + q] : 0.0;
    }
  }
#pragma unroll
  for (int r = 0; r < NW; ++r) X[r] = 0.0;  // entry e >= 1: x[c + e]
  // raw v[c] and dinv[c] (lane 0), multiplied when used: no arithmetic waits
  // on a load at prefetch time
  auto colv = [&](long long c) { return lane == 0 && c >= 0 ? v[c] : 0.0; };
  auto coli = [&](long long c) { return lane == 0 && c >= 0 ? dinv[c] : 0.0; };
  double pb[PF][NW], pw[PF][NBW], pv[PF], pi[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
#pragma unroll
    for (int r = 0; r < NW; ++r) pb[q][r] = colb(n - 1 - q, r);
#pragma unroll
    for (int r = 0; r < NBW; ++r) pw[q][r] = colw(n - 1 - q, r);
    pv[q] = colv(n - 1 - q);
    pi[q] = coli(n - 1 - q);
  }
  for (long long i0 = 0; i0 < n; i0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const long long c = n - 1 - (i0 + q);
      if (c < 0) break;
      double part = 0.0;
#pragma unroll
      for (int r = 0; r < NW; ++r) part += pb[q][r] * X[r];
#pragma unroll
      for (int r = 0; r < NBW; ++r) part += pw[q][r] * xb[r];
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double xc = __shfl_sync(0xffffffffu, pv[q] * pi[q], 0) - part;
      if (lane == 0) v[c] = xc;
      // shift: entry e takes entry e - 1; entry 1 takes x_c
#pragma unroll
      for (int r = NW - 1; r >= 0; --r) {
        double up = __shfl_up_sync(0xffffffffu, X[r], 1);
        if (r > 0) {
          const double pr = __shfl_sync(0xffffffffu, X[r > 0 ? r - 1 : 0], 31);
          if (lane == 0) up = pr;
        }
        if (r == 0 && lane == 1) up = xc;
        X[r] = up;
      }
#pragma unroll
      for (int r = 0; r < NW; ++r) pb[q][r] = colb(c - PF, r);
#pragma unroll
      for (int r = 0; r < NBW; ++r) pw[q][r] = colw(c - PF, r);
      pv[q] = colv(c - PF);
      pi[q] = coli(c - PF);
    }
  }
}

using SolveSegKernel = void (*)(const BandSeg*, int, const double*, const double*, double*, double*, int,
                                const int64_t*, long long);

SolveSegKernel solve_seg_kernel_for(int B1, int w) {
  if (B1 <= 32 && w <= 32) return solve_seg_warp_k<16, 1, 1>;
  if (B1 <= 32 && w <= 64) return solve_seg_warp_k<8, 1, 2>;
  if (B1 <= 64 && w <= 96) return solve_seg_warp_k<8, 2, 3>;
  return nullptr;
}

__global__ void __launch_bounds__(32) solve_k(const BandSeg* __restrict__ segs, int seg0, int mode,
                                              const double* __restrict__ buf, const double* __restrict__ Dinv,
                                              double* __restrict__ work, double* __restrict__ gparts, int wmax,
                                              const int64_t* __restrict__ border_pos, long long sep_pos0,
                                              BandBatch bb) {
  extern __shared__ double sm[];
  const int blk = seg0 + blockIdx.x;
  if (bb.ids) {
    const long long bi = bb.ids[blockIdx.y];
    buf += bi * bb.sbuf;
    Dinv += bi * bb.sdim;
    work += bi * bb.swork;
    gparts += bi * bb.swork;
  }
  const BandSeg g = segs[blk];
  const int lane = threadIdx.x;
  const long long n = g.n;
  const int b = g.b, w = g.w, B1 = b + 1;
  const int RW = B1 + w;
  const double* band = buf + g.band;
  const double* border = buf + g.border;
  const double* Sg = buf + g.S;
  double* v = work + g.pos;
  const double* dinv = Dinv + g.pos;
  double* Y = sm;          // B1 window of the vector
  double* yb = Y + B1;     // w
  double* xb = yb + w;     // w
  double* ring = xb + w;   // kPrefetch * (RW + 2)
  auto fetch = [&](long long c, int r, bool forward) {
    double* dstp = ring + r * (RW + 2);
    for (int j = lane; j < B1; j += 32) {
      if (c + j < n)
        cp8(dstp + j, band + c * B1 + j);
      else
        dstp[j] = 0.0;
    }
    for (int t = lane; t < w; t += 32) cp8(dstp + B1 + t, border + static_cast<long long>(t) * n + c);
    if (lane == 0) {
      if (forward) {
        if (c + B1 < n) cp8(dstp + RW, v + c + B1);
      } else {
        cp8(dstp + RW, v + c);
        cp8(dstp + RW + 1, dinv + c);
      }
    }
  };
  if (mode != 2) {
    // ---- forward: columns in increasing order
    for (int j = lane; j < B1; j += 32) Y[j] = j < n ? v[j] : 0.0;
    for (int t = lane; t < w; t += 32) yb[t] = mode == 0 ? work[g.bpos + t] : 0.0;
    for (int r = 0; r < kPrefetch; ++r) {
      if (r < n) fetch(r, r, true);
      cp_commit();
    }
    __syncwarp();
    int s = 0;
    for (long long c = 0; c < n; ++c, s = (s + 1 == B1 ? 0 : s + 1)) {
      cp_wait<kPrefetch - 1>();
      __syncwarp();
      const double* col = ring + static_cast<int>(c & kMask) * (RW + 2);
      const double yc = Y[s];
      if (lane == 0) v[c] = yc;
      for (int j = lane + 1; j < B1; j += 32)
        if (c + j < n) Y[s + j >= B1 ? s + j - B1 : s + j] -= col[j] * yc;
      for (int t = lane; t < w; t += 32) yb[t] -= col[B1 + t] * yc;
      __syncwarp();
      if (lane == 0 && c + B1 < n) Y[s] = col[RW];
      __syncwarp();
      if (c + kPrefetch < n) fetch(c + kPrefetch, static_cast<int>(c & kMask), true);
      cp_commit();
    }
    cp_wait<0>();
    __syncwarp();
    if (mode == 1) {
      for (int t = lane; t < w; t += 32) gparts[static_cast<int64_t>(blk) * wmax + t] = yb[t];
      return;
    }
    if (lane == 0) {
      for (int t = 0; t < w; ++t)
        for (int u = 0; u < t; ++u) yb[t] -= Sg[t * w + u] * yb[u];
      for (int t = 0; t < w; ++t) yb[t] *= Dinv[g.bpos + t];
      for (int t = w - 1; t >= 0; --t)
        for (int u = t + 1; u < w; ++u) yb[t] -= Sg[u * w + t] * yb[u];
      for (int t = 0; t < w; ++t) work[g.bpos + t] = yb[t];
    }
    __syncwarp();
    for (int t = lane; t < w; t += 32) xb[t] = yb[t];
  } else {
    // border values: the separator system's solution at this segment's rows
    for (int t = lane; t < w; t += 32) {
      const int64_t q = border_pos[static_cast<int64_t>(blk) * wmax + t];
      xb[t] = q >= 0 ? work[sep_pos0 + q] : 0.0;
    }
  }
  __syncwarp();
  // ---- backward: columns in decreasing order; X window holds x[c+1..c+b]
  double* X = Y;
  for (int r = 0; r < kPrefetch; ++r) {
    if (n - 1 - r >= 0) fetch(n - 1 - r, r, false);
    cp_commit();
  }
  int sc = static_cast<int>((n - 1) % B1);
  for (long long c = n - 1; c >= 0; --c, sc = (sc == 0 ? B1 - 1 : sc - 1)) {
    const long long it = n - 1 - c;
    cp_wait<kPrefetch - 1>();
    __syncwarp();
    const double* col = ring + static_cast<int>(it & kMask) * (RW + 2);
    double part = 0.0;
    for (int j = lane + 1; j < B1; j += 32)
      if (c + j < n) part += col[j] * X[sc + j >= B1 ? sc + j - B1 : sc + j];
    for (int t = lane; t < w; t += 32) part += col[B1 + t] * xb[t];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double xc = col[RW] * col[RW + 1] - part;
    __syncwarp();
    if (lane == 0) {
      X[sc] = xc;
      v[c] = xc;
    }
    __syncwarp();
    if (c - kPrefetch >= 0) fetch(c - kPrefetch, static_cast<int>(it & kMask), false);
    cp_commit();
  }
  cp_wait<0>();
}

// segment forward contributions into the separator system's right-hand side
__global__ void rhs_add_k(int nseg, int par, int wmax, long long n2, const int64_t* __restrict__ border_pos,
                          const double* __restrict__ gparts, double* __restrict__ sepv, BandBatch bb) {
  {
    const long long bi = batch_id(bb);
    gparts += bi * bb.swork;
    sepv += bi * bb.swork;
  }
  const int64_t cnt = static_cast<int64_t>((nseg - par + 1) / 2) * wmax;
  GRID_LOOP(q, cnt) {
    const int i = par + 2 * static_cast<int>(q / wmax), t = static_cast<int>(q % wmax);
    const int64_t R = border_pos[static_cast<int64_t>(i) * wmax + t];
    if (R < 0 || R >= n2) continue;
    sepv[R] += gparts[static_cast<int64_t>(i) * wmax + t];
  }
}
__global__ void rhs_global_k(int nseg, int wmax, int b, int wg, long long n2, const double* __restrict__ gparts,
                             double* __restrict__ sepv, BandBatch bb) {
  {
    const long long bi = batch_id(bb);
    gparts += bi * bb.swork;
    sepv += bi * bb.swork;
  }
  GRID_LOOP(u, wg) {
    double acc = 0.0;
    for (int i = 0; i < nseg; ++i) acc += gparts[static_cast<int64_t>(i) * wmax + b + u];
    sepv[n2 + u] += acc;
  }
}

int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 16)));
}

}  // namespace

namespace {
// column of CSC entry q (one thread per entry: a dense column — a free final
// time's — must not become one thread's serial loop)
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

__global__ void bandwidth_k(const int64_t* __restrict__ colp, const int64_t* __restrict__ rowi,
                            const int64_t* __restrict__ fpos, int64_t n, int64_t dim, int64_t nnz,
                            unsigned long long* out) {
  unsigned long long m = 0;
  GRID_LOOP(q, nnz) {
    const int64_t pj = fpos[col_of(colp, dim, q)];
    const int64_t pi = fpos[rowi[q]];
    if (pi < n && pj < n) m = max(m, static_cast<unsigned long long>(pi > pj ? pi - pj : pj - pi));
  }
  atomicMax(out, m);
}

__global__ void band_dst_k(BandDstIn in, const int8_t* __restrict__ lk, const int64_t* __restrict__ li,
                           const int64_t* __restrict__ ll, const BandSeg* __restrict__ segs,
                           int64_t* __restrict__ dst, int* __restrict__ err) {
  const int64_t n = in.n, b = in.b, wg = in.wg, n2 = in.n2;
  GRID_LOOP(q, in.nnz) {
    const int64_t fc = in.fpos[col_of(in.colp, in.dim, q)];
    {
      const int64_t fa = in.fpos[in.rowi[q]];
      int ak = lk[fa], ck_ = lk[fc];
      int64_t ai = li[fa], al = ll[fa], ci = li[fc], cl = ll[fc];
      int64_t d = -1;
      if (in.nseg == 1) {
        const BandSeg& sg = segs[0];
        int64_t r = ak == 2 ? n + al : al, cc = ck_ == 2 ? n + cl : cl;
        if (r < cc) {
          const int64_t t = r;
          r = cc;
          cc = t;
        }
        if (r < n)
          d = sg.band + cc * (b + 1) + (r - cc);
        else if (cc < n)
          d = sg.border + (r - n) * n + cc;
        else
          d = sg.S + (r - n) * sg.w + (cc - n);
      } else {
        if (ak == 0 && ck_ != 0) {  // interior (if any) in c
          int ti = ak;
          ak = ck_;
          ck_ = ti;
          int64_t t = ai;
          ai = ci;
          ci = t;
          t = al;
          al = cl;
          cl = t;
        }
        if (ak == 0 && ck_ == 0) {
          if (ai != ci) atomicOr(err, 1);
          const BandSeg& sg = segs[ai];
          int64_t r = al, cc = cl;
          if (r < cc) {
            const int64_t t = r;
            r = cc;
            cc = t;
          }
          if (r - cc > b) atomicOr(err, 2);
          d = sg.band + cc * (b + 1) + (r - cc);
        } else if (ck_ == 0) {
          const BandSeg& sg = segs[ci];
          int64_t t;
          if (ak == 2)
            t = b + al;
          else if (ai == ci - 1)
            t = al;
          else if (ai == ci)
            t = b + wg + al;
          else {
            atomicOr(err, 4);
            t = 0;
          }
          d = sg.border + t * sg.n + cl;
        } else {
          const BandSeg& sep = segs[in.nseg];
          int64_t R = ak == 1 ? ai * b + al : n2 + al, C = ck_ == 1 ? ci * b + cl : n2 + cl;
          if (R < C) {
            const int64_t t = R;
            R = C;
            C = t;
          }
          if (R < n2)
            d = sep.band + C * (sep.b + 1) + (R - C);
          else if (C < n2)
            d = sep.border + (R - n2) * n2 + C;
          else
            d = sep.S + (R - n2) * sep.w + (C - n2);
        }
      }
      dst[q] = d;
    }
  }
}
}  // namespace

int64_t* upload_i64(const std::vector<int64_t>& v, cudaStream_t s) {
  int64_t* p = nullptr;
  cudaMallocAsync(reinterpret_cast<void**>(&p), (v.empty() ? 1 : v.size()) * sizeof(int64_t), s);
  if (!v.empty()) cudaMemcpyAsync(p, v.data(), v.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  return p;
}

int64_t bandwidth(const int64_t* colp, const int64_t* rowi, const int64_t* fpos, int64_t n, int64_t dim,
                  cudaStream_t s) {
  unsigned long long* d = nullptr;
  cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), s);
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), s);
  int64_t nnz = 0;
  cudaMemcpyAsync(&nnz, colp + dim, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  bandwidth_k<<<grid_for(nnz), 256, 0, s>>>(colp, rowi, fpos, n, dim, nnz, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  cudaStreamSynchronize(s);
  return static_cast<int64_t>(h);
}

int64_t* band_dst(const BandDstIn& in, const std::vector<int8_t>& lk, const std::vector<int64_t>& li,
                  const std::vector<int64_t>& ll, const std::vector<BandSeg>& segs, int64_t nnz, cudaStream_t s) {
  int8_t* dlk = nullptr;
  BandSeg* dseg = nullptr;
  int* derr = nullptr;
  int64_t* dst = nullptr;
  cudaMallocAsync(reinterpret_cast<void**>(&dlk), std::max<size_t>(1, lk.size()), s);
  cudaMemcpyAsync(dlk, lk.data(), lk.size(), cudaMemcpyHostToDevice, s);
  int64_t* dli = upload_i64(li, s);
  int64_t* dll = upload_i64(ll, s);
  cudaMallocAsync(reinterpret_cast<void**>(&dseg), segs.size() * sizeof(BandSeg), s);
  cudaMemcpyAsync(dseg, segs.data(), segs.size() * sizeof(BandSeg), cudaMemcpyHostToDevice, s);
  cudaMallocAsync(reinterpret_cast<void**>(&derr), sizeof(int), s);
  cudaMemsetAsync(derr, 0, sizeof(int), s);
  cudaMallocAsync(reinterpret_cast<void**>(&dst), std::max<int64_t>(1, nnz) * sizeof(int64_t), s);
  BandDstIn in2 = in;
  in2.nnz = nnz;
  band_dst_k<<<grid_for(nnz), 256, 0, s>>>(in2, dlk, dli, dll, dseg, dst, derr);
  int err = 0;
  cudaMemcpyAsync(&err, derr, sizeof(int), cudaMemcpyDeviceToHost, s);
  for (void* p : {static_cast<void*>(dlk), static_cast<void*>(dli), static_cast<void*>(dll), static_cast<void*>(dseg),
                  static_cast<void*>(derr)})
    cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  if (err) throw std::runtime_error("band plan: KKT entry outside the partitioned band structure (" +
                                    std::to_string(err) + ")");
  return dst;
}

void band_assemble(const BandPlan& P, const BandDev& D, const double* kval, double* buf, cudaStream_t s) {
  zero_k<<<grid_for(P.buf_len), 256, 0, s>>>(buf, P.buf_len, BandBatch{});
  const int64_t nnz = P.nnz;
  if (nnz > 0) scatter_k<<<grid_for(nnz), 256, 0, s>>>(kval, D.dst, nnz, buf, BandBatch{});
}

void band_factor(const BandPlan& P, const BandDev& D, double* buf, double delta_w, double delta_c, double* Dinv,
                 long long* inertia_parts, long long* inertia, cudaStream_t s) {
  // many segments: 256-thread blocks, two per SM; a single sequential block
  // (the separator system, or an unpartitioned band): 1024 threads
  const BandSeg& s0 = P.segs[0];
  static const int env_threads = std::getenv("OCG_SEG_THREADS") ? std::atoi(std::getenv("OCG_SEG_THREADS")) : 0;
  const int seg_threads = env_threads > 0 ? env_threads : (s0.b <= 16 ? 128 : kFactorThreads);
  size_t sm_seg = 0, sm_sep = 0;
  const FactorKernel fseg = factor_kernel_for(s0.b + 1, s0.w, s0.w_early, P.nseg == 1, seg_threads, &sm_seg);
  const FactorKernel fsep =
      P.nseg > 1 ? factor_kernel_for(P.segs.back().b + 1, P.segs.back().w, P.segs.back().w_early, true, 1024, &sm_sep)
                 : fseg;
  const int tseg = P.nseg == 1 ? 1024 : seg_threads;
  if (sm_seg > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fseg), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm_seg));
  if (P.nseg > 1 && sm_sep > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fsep), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm_sep));
  static const bool timing = std::getenv("OCG_TIMING") != nullptr;
  cudaEvent_t ev[4];
  if (timing)
    for (auto& e : ev) cudaEventCreate(&e);
  if (timing) cudaEventRecord(ev[0], s);
  fseg<<<P.nseg, tseg, sm_seg, s>>>(D.segs, 0, buf, D.primal, delta_w, delta_c, Dinv, inertia_parts, BandBatch{});
  if (timing) cudaEventRecord(ev[1], s);
  int blocks = P.nseg;
  if (P.nseg > 1) {
    const int64_t per = static_cast<int64_t>(P.wmax) * P.wmax;
    for (int par = 0; par < 2; ++par)
      schur_add_k<<<grid_for(((P.nseg + 1) / 2) * per), 256, 0, s>>>(D.segs, P.nseg, par, P.wmax, D.border_pos, buf,
                                                                        BandBatch{});
    if (P.wg > 0) schur_global_k<<<1, 256, 0, s>>>(D.segs, P.nseg, P.wmax, P.b, P.wg, buf, BandBatch{});
    if (timing) cudaEventRecord(ev[2], s);
    if (D.cr)
      cr_factor(P, P.segs.back(), buf, D.primal, delta_w, delta_c, D.cr, D.crparts, inertia_parts + 3 * P.nseg, s);
    else
      fsep<<<1, 1024, sm_sep, s>>>(D.segs, P.nseg, buf, D.primal, delta_w, delta_c, Dinv, inertia_parts,
                                   BandBatch{});
    if (timing) cudaEventRecord(ev[3], s);
    blocks += 1;
  }
  if (timing && P.nseg > 1) {
    cudaEventSynchronize(ev[3]);
    float a = 0, b2 = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b2, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    std::fprintf(stderr, "[band_factor] segments %.3f ms  schur %.3f ms  separator system %.3f ms (%lld cols, b %d)\n",
                 a, b2, c, static_cast<long long>(P.segs.back().n), P.segs.back().b);
  }
  if (timing)
    for (auto& e : ev) cudaEventDestroy(e);
  inertia_sum_k<<<1, 32, 0, s>>>(inertia_parts, blocks, inertia, BandBatch{});
}

void band_solve(const BandPlan& P, const BandDev& D, const double* buf, const double* Dinv, const double* rhs,
                double* x, double* work, cudaStream_t s) {
  const int64_t dim = P.dim;
  double* gparts = work + dim;
  if (P.smem_solve > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(solve_k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P.smem_solve));
  static const bool timing = std::getenv("OCG_TIMING") != nullptr;
  cudaEvent_t ev[5];
  if (timing)
    for (auto& e : ev) {
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
    }
  gather_k<<<grid_for(dim), 256, 0, s>>>(rhs, D.perm, dim, work, BandBatch{});
  if (P.nseg == 1) {
    solve_k<<<1, 32, P.smem_solve, s>>>(D.segs, 0, 0, buf, Dinv, work, gparts, P.wmax, D.border_pos, 0, BandBatch{});
  } else {
    const BandSeg& sep = P.segs.back();
    if (timing) cudaEventRecord(ev[1], s);
    const SolveSegKernel regwin = solve_seg_kernel_for(P.b + 1, P.wmax);
    if (regwin)
      regwin<<<P.nseg, 32, 0, s>>>(D.segs, 1, buf, Dinv, work, gparts, P.wmax, D.border_pos, sep.pos);
    else
      solve_k<<<P.nseg, 32, P.smem_solve, s>>>(D.segs, 0, 1, buf, Dinv, work, gparts, P.wmax, D.border_pos, sep.pos,
                                               BandBatch{});
    if (timing) cudaEventRecord(ev[2], s);
    for (int par = 0; par < 2; ++par)
      rhs_add_k<<<grid_for(((P.nseg + 1) / 2) * P.wmax), 256, 0, s>>>(P.nseg, par, P.wmax, sep.n, D.border_pos,
                                                                        gparts, work + sep.pos, BandBatch{});
    if (P.wg > 0)
      rhs_global_k<<<1, 32, 0, s>>>(P.nseg, P.wmax, P.b, P.wg, sep.n, gparts, work + sep.pos, BandBatch{});
    if (D.cr)
      cr_solve(P, sep, D.cr, work, s);
    else
      solve_k<<<1, 32, P.smem_solve, s>>>(D.segs, P.nseg, 0, buf, Dinv, work, gparts, P.wmax, D.border_pos, sep.pos,
                                          BandBatch{});
    if (timing) cudaEventRecord(ev[3], s);
    if (regwin)
      regwin<<<P.nseg, 32, 0, s>>>(D.segs, 2, buf, Dinv, work, gparts, P.wmax, D.border_pos, sep.pos);
    else
      solve_k<<<P.nseg, 32, P.smem_solve, s>>>(D.segs, 0, 2, buf, Dinv, work, gparts, P.wmax, D.border_pos, sep.pos,
                                               BandBatch{});
  }
  scatter_back_k<<<grid_for(dim), 256, 0, s>>>(work, D.perm, dim, x, BandBatch{});
  if (timing) {
    cudaEventRecord(ev[4], s);
    cudaEventSynchronize(ev[4]);
    float t[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    std::fprintf(stderr, "[band_solve] gather %.3f ms  segments forward %.3f ms  separator system %.3f ms  "
                 "segments backward + scatter %.3f ms\n", t[0], t[1], t[2], t[3]);
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void band_factor_batch(const BandPlan& P, const BandDev& D, const double* kval, double* buf, double* Dinv,
                       long long* inertia, long long* parts, const int* ids, int nb, const double* dws,
                       const double* dcs, cudaStream_t s) {
  if (nb <= 0) return;
  BandBatch bb;
  bb.ids = ids;
  bb.sbuf = P.buf_len;
  bb.sdim = P.dim;
  bb.swork = P.dim + static_cast<long long>(P.nseg) * P.wmax;
  bb.sparts = 3;
  bb.dw = dws;
  bb.dc = dcs;
  if (P.nseg > 1) {
    // every system's segments in one launch (grid segments x systems), the
    // Schur complements, then every system's separator system
    const unsigned ny = static_cast<unsigned>(nb);
    zero_k<<<dim3(std::max(1, std::min(grid_for(P.buf_len), 16)), ny), 256, 0, s>>>(buf, P.buf_len, bb);
    if (P.nnz > 0)
      scatter_k<<<dim3(std::max(1, std::min(grid_for(P.nnz), 16)), ny), 256, 0, s>>>(kval, D.dst, P.nnz, buf, bb);
    const BandSeg& s0 = P.segs[0];
    size_t sm_seg = 0, sm_sep = 0;
    const FactorKernel fseg = factor_kernel_for(s0.b + 1, s0.w, s0.w_early, false, kFactorThreads, &sm_seg);
    const FactorKernel fsep =
        factor_kernel_for(P.segs.back().b + 1, P.segs.back().w, P.segs.back().w_early, true, 1024, &sm_sep);
    for (auto [f, sm] : {std::pair<FactorKernel, size_t>{fseg, sm_seg}, {fsep, sm_sep}})
      if (sm > 48 * 1024)
        cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    BandBatch pb = bb;
    pb.sparts = 3 * (P.nseg + 1);
    fseg<<<dim3(P.nseg, ny), kFactorThreads, sm_seg, s>>>(D.segs, 0, buf, D.primal, 0.0, 0.0, Dinv, parts, pb);
    const int64_t per = static_cast<int64_t>(P.wmax) * P.wmax;
    for (int par = 0; par < 2; ++par)
      schur_add_k<<<dim3(std::max(1, std::min(grid_for(((P.nseg + 1) / 2) * per), 8)), ny), 256, 0, s>>>(
          D.segs, P.nseg, par, P.wmax, D.border_pos, buf, pb);
    if (P.wg > 0) schur_global_k<<<dim3(1, ny), 256, 0, s>>>(D.segs, P.nseg, P.wmax, P.b, P.wg, buf, pb);
    fsep<<<dim3(1, ny), 1024, sm_sep, s>>>(D.segs, P.nseg, buf, D.primal, 0.0, 0.0, Dinv, parts, pb);
    inertia_sum_k<<<dim3(1, ny), 32, 0, s>>>(parts, P.nseg + 1, inertia, pb);
    return;
  }
  const unsigned ny = static_cast<unsigned>(nb);
  const int gz = std::max(1, std::min(grid_for(P.buf_len), 8));
  zero_k<<<dim3(gz, ny), 256, 0, s>>>(buf, P.buf_len, bb);
  if (P.nnz > 0) scatter_k<<<dim3(std::max(1, std::min(grid_for(P.nnz), 8)), ny), 256, 0, s>>>(kval, D.dst, P.nnz, buf, bb);
  const BandSeg& s0 = P.segs[0];
  FactorWarpKernel fw = nullptr;
  SolveWarpKernel sw = nullptr;
  if (s0.w == 0 && !std::getenv("OCG_BATCH_BLOCK_LDL") && warp_kernels_for(s0.b + 1, fw, sw)) {
    fw<<<(nb + 3) / 4, 128, 0, s>>>(D.segs, buf, D.primal, Dinv, inertia, bb, nb);
    return;
  }
  size_t sm_f = 0;
  const FactorKernel f = factor_kernel_batch(s0.b + 1, s0.w, s0.w_early, &sm_f);
  if (sm_f > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm_f));
  f<<<dim3(1, ny), 128, sm_f, s>>>(D.segs, 0, buf, D.primal, 0.0, 0.0, Dinv, inertia, bb);
}

void band_solve_batch(const BandPlan& P, const BandDev& D, const double* buf, const double* Dinv, const double* rhs,
                      double* x, double* work, const int* ids, int nb, cudaStream_t s) {
  if (nb <= 0) return;
  BandBatch bb;
  bb.ids = ids;
  bb.sbuf = P.buf_len;
  bb.sdim = P.dim;
  bb.swork = P.dim + static_cast<long long>(P.nseg) * P.wmax;
  const unsigned ny = static_cast<unsigned>(nb);
  if (P.nseg > 1) {
    if (P.smem_solve > 48 * 1024)
      cudaFuncSetAttribute(reinterpret_cast<const void*>(solve_k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(P.smem_solve));
    const int gd = std::max(1, std::min(grid_for(P.dim), 8));
    const BandSeg& sep = P.segs.back();
    double* gparts = work + P.dim;
    gather_k<<<dim3(gd, ny), 256, 0, s>>>(rhs, D.perm, P.dim, work, bb);
    solve_k<<<dim3(P.nseg, ny), 32, P.smem_solve, s>>>(D.segs, 0, 1, buf, Dinv, work, gparts, P.wmax, D.border_pos,
                                                       sep.pos, bb);
    for (int par = 0; par < 2; ++par)
      rhs_add_k<<<dim3(1, ny), 256, 0, s>>>(P.nseg, par, P.wmax, sep.n, D.border_pos, gparts, work + sep.pos, bb);
    if (P.wg > 0) rhs_global_k<<<dim3(1, ny), 32, 0, s>>>(P.nseg, P.wmax, P.b, P.wg, sep.n, gparts, work + sep.pos, bb);
    solve_k<<<dim3(1, ny), 32, P.smem_solve, s>>>(D.segs, P.nseg, 0, buf, Dinv, work, gparts, P.wmax, D.border_pos,
                                                 sep.pos, bb);
    solve_k<<<dim3(P.nseg, ny), 32, P.smem_solve, s>>>(D.segs, 0, 2, buf, Dinv, work, gparts, P.wmax, D.border_pos,
                                                       sep.pos, bb);
    scatter_back_k<<<dim3(gd, ny), 256, 0, s>>>(work, D.perm, P.dim, x, bb);
    return;
  }
  const int gd = std::max(1, std::min(grid_for(P.dim), 8));
  if (P.smem_solve > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(solve_k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P.smem_solve));
  gather_k<<<dim3(gd, ny), 256, 0, s>>>(rhs, D.perm, P.dim, work, bb);
  const BandSeg& s0 = P.segs[0];
  FactorWarpKernel fw = nullptr;
  SolveWarpKernel sw = nullptr;
  if (s0.w == 0 && !std::getenv("OCG_BATCH_BLOCK_LDL") && warp_kernels_for(s0.b + 1, fw, sw))
    sw<<<(nb + 3) / 4, 128, 0, s>>>(D.segs, buf, Dinv, work, bb, nb);
  else
    solve_k<<<dim3(1, ny), 32, P.smem_solve, s>>>(D.segs, 0, 0, buf, Dinv, work, work + P.dim, P.wmax, D.border_pos,
                                                 0, bb);
  scatter_back_k<<<dim3(gd, ny), 256, 0, s>>>(work, D.perm, P.dim, x, bb);
}

}  // namespace dev
}  // namespace ocg
