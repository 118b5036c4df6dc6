// Device LDL^T in a node-major band-plus-border ordering (see band.hpp).
//
// The factorization and the triangular solves are sequential along the band,
// so each runs on ONE warp with the active window of the band in shared
// memory: the (b+1) x (b+1) trailing triangle rolls through a ring of column
// slots, and the band columns that enter the window are prefetched kPrefetch
// columns ahead with cp.async (LDGSTS) so that no global-memory latency sits
// on the per-column critical path. Gathers/scatters between KKT order and
// band order are grid-wide streaming kernels.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "band.hpp"

namespace ocg {

BandPlan make_band_plan(int64_t dim, const std::vector<int64_t>& node, const std::vector<int64_t>& colp,
                        const std::vector<int64_t>& rowi, int64_t ntot) {
  BandPlan P;
  P.dim = dim;
  std::vector<int64_t> order(static_cast<size_t>(dim));
  for (int64_t i = 0; i < dim; ++i) order[static_cast<size_t>(i)] = i;
  auto key = [&](int64_t i) { return node[static_cast<size_t>(i)] < 0 ? INT64_MAX : node[static_cast<size_t>(i)]; };
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
  std::vector<int64_t> pos(static_cast<size_t>(dim));
  for (int64_t p = 0; p < dim; ++p) pos[static_cast<size_t>(order[static_cast<size_t>(p)])] = p;
  int64_t w = 0;
  for (int64_t i = 0; i < dim; ++i) w += node[static_cast<size_t>(i)] < 0 ? 1 : 0;
  P.n = dim - w;
  P.w = static_cast<int>(w);
  P.perm = order;
  P.primal.resize(static_cast<size_t>(dim));
  for (int64_t p = 0; p < dim; ++p) P.primal[static_cast<size_t>(p)] = order[static_cast<size_t>(p)] < ntot ? 1 : 0;
  int64_t b = 0;
  for (int64_t j = 0; j < dim; ++j)
    for (int64_t q = colp[static_cast<size_t>(j)]; q < colp[static_cast<size_t>(j) + 1]; ++q) {
      const int64_t pi = pos[static_cast<size_t>(rowi[static_cast<size_t>(q)])], pj = pos[static_cast<size_t>(j)];
      if (pi < P.n && pj < P.n) b = std::max<int64_t>(b, pi > pj ? pi - pj : pj - pi);
    }
  if (b > 62) throw std::runtime_error("KKT bandwidth " + std::to_string(b) + " exceeds the band solver's limit (62)");
  P.b = static_cast<int>(b);
  const int64_t B1 = b + 1, n = P.n;
  P.dst.resize(rowi.size());
  for (int64_t j = 0; j < dim; ++j)
    for (int64_t q = colp[static_cast<size_t>(j)]; q < colp[static_cast<size_t>(j) + 1]; ++q) {
      int64_t r = pos[static_cast<size_t>(rowi[static_cast<size_t>(q)])], c = pos[static_cast<size_t>(j)];
      if (r < c) std::swap(r, c);
      int64_t d;
      if (r < n)
        d = c * B1 + (r - c);  // band
      else if (c < n)
        d = n * B1 + (r - n) * n + c;  // border row r-n, band column c
      else
        d = n * B1 + w * n + (r - n) * w + (c - n);  // border block (lower)
      P.dst[static_cast<size_t>(q)] = d;
    }
  return P;
}

namespace dev {

namespace {

constexpr int kPrefetch = 32;  // band columns in flight ahead of the window (power of two)
constexpr int kMask = kPrefetch - 1;

__device__ __forceinline__ void cp8(double* s, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__global__ void scatter_k(const double* __restrict__ kval, const int64_t* __restrict__ dst, int64_t nnz,
                          double* __restrict__ buf) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    buf[dst[p]] = kval[p];
}

__global__ void zero_k(double* __restrict__ buf, int64_t len) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    buf[p] = 0.0;
}

__device__ __forceinline__ bool zero_pivot(double d, double scale) {
  return !(fabs(d) <= DBL_MAX) || fabs(d) <= 1e-14 * fmax(scale, 1e-30);
}

// One warp. Shared memory: window W[B1][B1] (slot-major), pivot scales ps[B1],
// border window Wb[w][B1], border block S[w][w] + scales, y/l/yb/lb vectors,
// the (j1, j2) update pairs and a prefetch ring of kPrefetch columns.
__global__ void __launch_bounds__(32) band_factor_k(double* __restrict__ buf, const double* __restrict__ primal,
                                                    long long n, int b, int w, double dw, double dc,
                                                    double* __restrict__ Dinv, long long* __restrict__ inertia) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x;
  const int B1 = b + 1;
  double* W = sm;                     // B1 * B1
  double* ps = W + B1 * B1;           // B1
  double* Wb = ps + B1;               // w * B1
  double* S = Wb + w * B1;            // w * w
  double* Sps = S + w * w;            // w
  double* y = Sps + w;                // B1
  double* l = y + B1;                 // B1
  double* yb = l + B1;                // w
  double* lb = yb + w;                // w
  double* ring = lb + w;              // kPrefetch * (B1 + w + 1)
  short* pj1 = reinterpret_cast<short*>(ring + kPrefetch * (B1 + w + 1));
  const int P = b * (b + 1) / 2;
  short* pj2 = pj1 + P;
  double* band = buf;
  double* border = buf + n * B1;
  double* Sg = border + static_cast<long long>(w) * n;
  const int RW = B1 + w + 1;  // ring row: band column, its border entries, its primal flag

  for (int p = lane; p < P; p += 32) {  // pairs j1 <= j2 in 1..b
    int j1 = 1, rem = p;
    while (rem >= b - j1 + 1) {
      rem -= b - j1 + 1;
      ++j1;
    }
    pj1[p] = static_cast<short>(j1);
    pj2[p] = static_cast<short>(j1 + rem);
  }
  auto delta_of = [&](double flag) { return flag != 0.0 ? dw : -dc; };
  // a column entering the window: band entries, its diagonal's regularization
  // and pivot scale, and its border entries
  auto enter = [&](long long c, int slot, const double* src) {
    for (int j = lane; j < B1; j += 32) {
      double v = src[j];
      if (j == 0) {
        v += delta_of(src[B1 + w]);
        ps[slot] = fabs(v);
      }
      W[slot * B1 + j] = v;
    }
    for (int t = lane; t < w; t += 32) Wb[t * B1 + slot] = src[B1 + t];
  };
  auto fetch = [&](long long c, int r) {  // column c -> ring row r (async)
    double* dstp = ring + r * RW;
    for (int j = lane; j < B1; j += 32) {
      if (c + j < n)
        cp8(dstp + j, band + c * B1 + j);
      else
        dstp[j] = 0.0;
    }
    for (int t = lane; t < w; t += 32) cp8(dstp + B1 + t, border + static_cast<long long>(t) * n + c);
    if (lane == 0) cp8(dstp + B1 + w, primal + c);
  };
  // initial window: columns 0..B1-1 directly; prefetch B1..B1+kPrefetch-1
  for (long long c = 0; c < B1 && c < n; ++c) {
    for (int j = lane; j < B1; j += 32) {
      double v = c + j < n ? band[c * B1 + j] : 0.0;
      if (j == 0) {
        v += delta_of(primal[c]);
        ps[c] = fabs(v);
      }
      W[c * B1 + j] = v;
    }
    for (int t = lane; t < w; t += 32) Wb[t * B1 + c] = border[static_cast<long long>(t) * n + c];
  }
  for (int r = 0; r < kPrefetch; ++r) {
    if (B1 + r < n) fetch(B1 + r, r);
    cp_commit();
  }
  for (int q = lane; q < w * w; q += 32) {
    const int t = q / w, u = q % w;
    double v = Sg[q];
    if (t == u) {
      v += delta_of(primal[n + t]);
      Sps[t] = fabs(v);
    }
    S[q] = v;
  }
  long long npos = 0, nneg = 0, nzero = 0;
  __syncwarp();

  int s = 0;  // slot of column k = k mod B1
  for (long long k = 0; k < n; ++k, s = (s + 1 == B1 ? 0 : s + 1)) {
    const double d = W[s * B1];
    const bool zero = zero_pivot(d, ps[s]);
    const double dinv = zero ? 0.0 : 1.0 / d;
    if (lane == 0) {
      Dinv[k] = dinv;
      band[k * B1] = d;
      if (zero)
        ++nzero;
      else if (d > 0)
        ++npos;
      else
        ++nneg;
    }
    for (int j = lane + 1; j < B1; j += 32) {
      const double yj = k + j < n ? W[s * B1 + j] : 0.0;
      const double lj = yj * dinv;
      y[j] = yj;
      l[j] = lj;
      if (k + j < n) band[k * B1 + j] = lj;
    }
    for (int t = lane; t < w; t += 32) {
      const double v = Wb[t * B1 + s];
      yb[t] = v;
      lb[t] = v * dinv;
      border[static_cast<long long>(t) * n + k] = v * dinv;
    }
    __syncwarp();
    for (int p = lane; p < P; p += 32) {
      const int j1 = pj1[p], j2 = pj2[p];
      if (k + j2 < n) {
        const int s1 = s + j1 >= B1 ? s + j1 - B1 : s + j1;
        const double upd = l[j2] * y[j1];
        W[s1 * B1 + (j2 - j1)] -= upd;
        if (j1 == j2) ps[s1] = fmax(ps[s1], fabs(upd));
      }
    }
    for (int q = lane; q < w * b; q += 32) {
      const int t = q / b, j = q % b + 1;
      if (k + j < n) Wb[t * B1 + (s + j >= B1 ? s + j - B1 : s + j)] -= lb[t] * y[j];
    }
    for (int q = lane; q < w * w; q += 32) {
      const int t = q / w, u = q % w;
      if (u <= t) {
        const double upd = lb[t] * yb[u];
        S[q] -= upd;
        if (t == u) Sps[t] = fmax(Sps[t], fabs(upd));
      }
    }
    // column k is final: its slot takes column k + B1 from the prefetch ring
    cp_wait<kPrefetch - 1>();
    __syncwarp();
    const long long cin = k + B1;
    if (cin < n) enter(cin, s, ring + static_cast<int>(k & kMask) * RW);
    __syncwarp();
    if (cin + kPrefetch < n) fetch(cin + kPrefetch, static_cast<int>(k & kMask));
    cp_commit();
  }
  cp_wait<0>();
  // dense border block: sequential LDL^T with the same pivot rule
  if (lane == 0) {
    for (int t = 0; t < w; ++t) {
      const double d = S[t * w + t];
      const bool zero = zero_pivot(d, Sps[t]);
      const double dinv = zero ? 0.0 : 1.0 / d;
      Dinv[n + t] = dinv;
      Sg[t * w + t] = d;
      if (zero)
        ++nzero;
      else if (d > 0)
        ++npos;
      else
        ++nneg;
      for (int u = t + 1; u < w; ++u) {
        const double yu = S[u * w + t];
        const double lu = yu * dinv;
        for (int v = t + 1; v <= u; ++v) {
          const double upd = lu * S[v * w + t];
          S[u * w + v] -= upd;
          if (u == v) Sps[u] = fmax(Sps[u], fabs(upd));
        }
      }
      for (int u = t + 1; u < w; ++u) Sg[u * w + t] = S[u * w + t] * dinv;
    }
  }
  // counts from lane 0 only
  if (lane == 0) {
    inertia[0] = npos;
    inertia[1] = nneg;
    inertia[2] = nzero;
  }
}

__global__ void gather_k(const double* __restrict__ rhs, const int64_t* __restrict__ perm, int64_t dim,
                         double* __restrict__ out) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < dim;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = rhs[perm[p]];
}

__global__ void scatter_back_k(const double* __restrict__ work, const int64_t* __restrict__ perm, int64_t dim,
                               double* __restrict__ x) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < dim;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[perm[p]] = work[p];
}

// One warp: forward L y = b, D scaling, backward L^T x = y, on work[] in
// band order (border last). L columns stream through a cp.async ring.
__global__ void __launch_bounds__(32) band_solve_k(const double* __restrict__ buf, const double* __restrict__ Dinv,
                                                   long long n, int b, int w, double* __restrict__ work) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x;
  const int B1 = b + 1;
  const int RW = B1 + w;
  const double* band = buf;
  const double* border = buf + n * B1;
  const double* Sg = border + static_cast<long long>(w) * n;
  double* Y = sm;            // B1 window of the vector
  double* yb = Y + B1;       // w
  double* ring = yb + w;     // kPrefetch * (RW + 2)
  // ring row of column c: L column, border entries, then two vector values
  // the step needs (forward: rhs of column c + B1; backward: y_c and Dinv_c)
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
        if (c + B1 < n) cp8(dstp + RW, work + c + B1);
      } else {
        cp8(dstp + RW, work + c);
        cp8(dstp + RW + 1, Dinv + c);
      }
    }
  };
  // ---- forward: columns in increasing order
  for (int j = lane; j < B1; j += 32) Y[j] = j < n ? work[j] : 0.0;
  for (int t = lane; t < w; t += 32) yb[t] = work[n + t];
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
    if (lane == 0) work[c] = yc;
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
  if (lane == 0) {
    for (int t = 0; t < w; ++t)
      for (int u = 0; u < t; ++u) yb[t] -= Sg[t * w + u] * yb[u];
    for (int t = 0; t < w; ++t) yb[t] *= Dinv[n + t];
    for (int t = w - 1; t >= 0; --t)
      for (int u = t + 1; u < w; ++u) yb[t] -= Sg[u * w + t] * yb[u];
    for (int t = 0; t < w; ++t) work[n + t] = yb[t];
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
    for (int t = lane; t < w; t += 32) part += col[B1 + t] * yb[t];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double xc = col[RW] * col[RW + 1] - part;
    __syncwarp();
    if (lane == 0) {
      X[sc] = xc;
      work[c] = xc;
    }
    __syncwarp();
    if (c - kPrefetch >= 0) fetch(c - kPrefetch, static_cast<int>(it & kMask), false);
    cp_commit();
  }
  cp_wait<0>();
}

int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 16)));
}

}  // namespace

void band_assemble(const double* kval, const int64_t* dst, int64_t nnz, double* buf, int64_t len, cudaStream_t s) {
  zero_k<<<grid_for(len), 256, 0, s>>>(buf, len);
  if (nnz > 0) scatter_k<<<grid_for(nnz), 256, 0, s>>>(kval, dst, nnz, buf);
}

void band_factor(double* buf, const double* primal, int64_t n, int b, int w, double delta_w, double delta_c,
                 double* Dinv, long long* inertia, cudaStream_t s) {
  const int B1 = b + 1, P = b * (b + 1) / 2;
  const size_t smem = sizeof(double) * (static_cast<size_t>(B1) * B1 + B1 + static_cast<size_t>(w) * B1 +
                                        static_cast<size_t>(w) * w + w + 2 * B1 + 2 * w +
                                        static_cast<size_t>(kPrefetch) * (B1 + w + 1)) +
                      sizeof(short) * 2 * static_cast<size_t>(P) + 16;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(band_factor_k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  band_factor_k<<<1, 32, smem, s>>>(buf, primal, n, b, w, delta_w, delta_c, Dinv, inertia);
}

void band_solve(const double* buf, const double* Dinv, const int64_t* perm, int64_t n, int b, int w,
                const double* rhs, double* x, double* work, cudaStream_t s) {
  const int64_t dim = n + w;
  gather_k<<<grid_for(dim), 256, 0, s>>>(rhs, perm, dim, work);
  const size_t smem = sizeof(double) * (static_cast<size_t>(b + 1) + w + static_cast<size_t>(kPrefetch) * (b + 3 + w));
  band_solve_k<<<1, 32, smem, s>>>(buf, Dinv, n, b, w, work);
  scatter_back_k<<<grid_for(dim), 256, 0, s>>>(work, perm, dim, x);
}

}  // namespace dev
}  // namespace ocg
