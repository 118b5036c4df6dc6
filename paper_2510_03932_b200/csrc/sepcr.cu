// Separator system of the time-partitioned band LDL^T by block cyclic
// reduction (band.hpp: CrLayout, cr_factor, cr_solve).
//
// After the segments are factored, the separators (ns blocks of b columns)
// form a block-tridiagonal system with a dense border of w rows (free
// variables such as a free final time). factor_k eliminates it as one band,
// one column after another in one thread block: a serial chain of ns*b
// columns. Here the separators are eliminated level by level instead:
// separator k is eliminated at level l = v2(k + 1) (the power of two dividing
// k + 1), when its nearest surviving neighbours are p = k - 2^l and
// q = k + 2^l. Every elimination of a level is independent: one thread block
// per separator factors its b x b diagonal block (1x1 pivots, the reference's
// zero-pivot rule with the pivot scale carried through every Schur update as
// the largest single update), forms W = A_xk L_k^-T D_k^-1 for the rows of
// p, q and the border, and subtracts W D_k W^T from p and q. Two separators
// of a level share a neighbour, so a level runs as two launches (even and odd
// members); border contributions go to per-separator slots summed in
// separator order at the end. Deterministic; a different (equally valid)
// elimination order than the band kernel, so the pivots differ by rounding.
// Depth log2(ns) instead of ns*b.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "band.hpp"

namespace ocg::dev {

namespace {

__device__ __forceinline__ bool zero_pivot(double d, double scale) {
  return !(fabs(d) <= DBL_MAX) || fabs(d) <= 1e-14 * fmax(scale, 1e-30);
}

// per-separator region: D (b*b, row-major lower: the working diagonal block,
// after elimination L strict-lower + pivots on the diagonal), E (b*b: coupling
// to the next surviving separator, rows there, columns here), G (w*b border
// coupling), Wp, Wq (b*b), Wg (w*b), dinv (b), ps (b), Sc (w*w border
// contribution), Sps (w), rg (w: forward-solve border contribution)
struct Cr {
  double* base;
  int b, w;
  long long per;
  __device__ double* D(long long j) const { return base + j * per; }
  __device__ double* E(long long j) const { return D(j) + b * b; }
  __device__ double* G(long long j) const { return E(j) + b * b; }
  __device__ double* Wp(long long j) const { return G(j) + w * b; }
  __device__ double* Wq(long long j) const { return Wp(j) + b * b; }
  __device__ double* Wg(long long j) const { return Wq(j) + b * b; }
  __device__ double* dinv(long long j) const { return Wg(j) + w * b; }
  __device__ double* ps(long long j) const { return dinv(j) + b; }
  __device__ double* Sc(long long j) const { return ps(j) + b; }
  __device__ double* Sps(long long j) const { return Sc(j) + w * w; }
  __device__ double* rg(long long j) const { return Sps(j) + w; }
};

__host__ __device__ inline long long cr_per(int b, int w) {
  return 5LL * b * b + 2LL * w * b + 2LL * b + static_cast<long long>(w) * w + 2LL * w;
}

// separator-system view of the factor buffer (the last BandSeg)
struct SepView {
  const double* band;    // (n2) x (2b) column-major band, entry (R, C) at C*2b + (R-C)
  const double* border;  // w x n2
  const double* S;       // w x w lower
  const double* ps0;     // n2 + w pivot-scale seeds
  const double* primal;  // by position, from sep.pos
  long long n2;
};

__global__ void cr_init_k(Cr cr, SepView sv, int ns, double dw, double dc, double* __restrict__ Sg,
                          double* __restrict__ Sps) {
  const int b = cr.b, w = cr.w, B2 = 2 * b;
  auto delta = [&](double f) { return f != 0.0 ? dw : -dc; };
  if (static_cast<int>(blockIdx.x) == ns) {
    for (int q = threadIdx.x; q < w * w; q += blockDim.x) {
      const int t = q / w, u = q % w;
      double v = u <= t ? sv.S[q] : 0.0;
      if (t == u) {
        v += delta(sv.primal[sv.n2 + t]);
        Sps[t] = fmax(fabs(v), sv.ps0[sv.n2 + t]);
      }
      Sg[q] = v;
    }
    return;
  }
  const long long j = blockIdx.x, c0 = j * b;
  double* D = cr.D(j);
  double* E = cr.E(j);
  double* G = cr.G(j);
  double* ps = cr.ps(j);
  for (int q = threadIdx.x; q < b * b; q += blockDim.x) {
    const int r = q / b, c = q % b;
    double v = 0.0;
    if (r >= c) v = sv.band[(c0 + c) * B2 + (r - c)];
    if (r == c) {
      v += delta(sv.primal[c0 + r]);
      ps[r] = fmax(fabs(v), sv.ps0[c0 + r]);
    }
    D[q] = v;
    E[q] = j + 1 < ns ? sv.band[(c0 + c) * B2 + (b + r - c)] : 0.0;
  }
  for (int q = threadIdx.x; q < w * b; q += blockDim.x) {
    const int t = q / b, c = q % b;
    G[q] = sv.border[static_cast<long long>(t) * sv.n2 + c0 + c];
  }
}

// eliminate the separators k = 2^l (2i + 1) - 1, i = 2i' + phase
__global__ void cr_elim_k(Cr cr, int ns, int level, int phase, long long* __restrict__ parts) {
  extern __shared__ double sm[];
  const int b = cr.b, w = cr.w, tid = threadIdx.x, T = blockDim.x;
  const long long i = 2LL * blockIdx.x + phase;
  const long long step = 1LL << level;
  const long long k = step * (2 * i + 1) - 1;
  if (k >= ns) return;
  const long long p = k - step, q = k + step;
  const bool hp = p >= 0, hq = q < ns;
  double* Dk = sm;            // b*b
  double* dv = Dk + b * b;    // b pivots' inverses
  double* ps = dv + b;        // b
  const int nrow = (hp ? b : 0) + (hq ? b : 0) + w;
  double* X = ps + b;         // nrow * b: rows [p | q | border] of A_xk L^-T
  double* W = X + nrow * b;   // nrow * b: X D^-1
  const double* Dg = cr.D(k);
  for (int e = tid; e < b * b; e += T) Dk[e] = Dg[e];
  for (int e = tid; e < b; e += T) ps[e] = cr.ps(k)[e];
  // rows of A(p,k) = E[p]^T, A(q,k) = E[k], G[k]
  const int rq = hp ? b : 0, rg = rq + (hq ? b : 0);
  for (int e = tid; e < nrow * b; e += T) {
    const int r = e / b, m = e % b;
    double v;
    if (r < rq)
      v = cr.E(p)[m * b + r];
    else if (r < rg)
      v = cr.E(k)[(r - rq) * b + m];
    else
      v = cr.G(k)[(r - rg) * b + m];
    X[e] = v;
  }
  __syncthreads();
  // LDL^T of the diagonal block, 1x1 pivots in order (factor_k's arithmetic)
  long long npos = 0, nneg = 0, nzero = 0;
  for (int m = 0; m < b; ++m) {
    const double d = Dk[m * b + m];
    const bool zero = zero_pivot(d, ps[m]);
    const double dinv = zero ? 0.0 : 1.0 / d;
    if (tid == 0) {
      dv[m] = dinv;
      if (zero)
        ++nzero;
      else if (d > 0)
        ++npos;
      else
        ++nneg;
    }
    const int rem = b - m - 1;
    for (int e = tid; e < rem * rem; e += T) {
      const int ii = m + 1 + e / rem, jj = m + 1 + e % rem;
      if (jj <= ii) {
        const double upd = Dk[ii * b + m] * dinv * Dk[jj * b + m];
        Dk[ii * b + jj] -= upd;
        if (ii == jj) ps[ii] = fmax(ps[ii], fabs(upd));
      }
    }
    __syncthreads();
    for (int ii = m + 1 + tid; ii < b; ii += T) Dk[ii * b + m] *= dinv;
    __syncthreads();
  }
  // X = A_xk L^-T (row-wise forward substitution), W = X D^-1
  for (int r = tid; r < nrow; r += T) {
    double* x = X + r * b;
    for (int m = 0; m < b; ++m) {
      double v = x[m];
      for (int n = 0; n < m; ++n) v -= Dk[m * b + n] * x[n];
      x[m] = v;
      W[r * b + m] = v * dv[m];
    }
  }
  __syncthreads();
  // factor of k and its W rows for the solves
  for (int e = tid; e < b * b; e += T) cr.D(k)[e] = Dk[e];
  for (int e = tid; e < b; e += T) cr.dinv(k)[e] = dv[e];
  for (int e = tid; e < b * b; e += T) {
    if (hp) cr.Wp(k)[e] = W[e];
    if (hq) cr.Wq(k)[e] = W[rq * b + e];
  }
  for (int e = tid; e < w * b; e += T) cr.Wg(k)[e] = W[rg * b + e];
  // Schur updates: entry -= sum_m X[i][m] W[j][m], m in order
  auto schur = [&](const double* Xi, const double* Wj) {
    double s = 0.0;
    for (int m = 0; m < b; ++m) s += Xi[m] * Wj[m];
    return s;
  };
  auto diag_scale = [&](const double* Xi, const double* Wi) {
    double s = 0.0;
    for (int m = 0; m < b; ++m) s = fmax(s, fabs(Xi[m] * Wi[m]));
    return s;
  };
  if (hp) {
    double* Dp = cr.D(p);
    for (int e = tid; e < b * b; e += T) {
      const int ii = e / b, jj = e % b;
      if (jj <= ii) {
        double v = Dp[e];
        for (int m = 0; m < b; ++m) v -= X[ii * b + m] * W[jj * b + m];
        Dp[e] = v;
      }
    }
    for (int ii = tid; ii < b; ii += T) cr.ps(p)[ii] = fmax(cr.ps(p)[ii], diag_scale(X + ii * b, W + ii * b));
    for (int e = tid; e < w * b; e += T) {
      const int t = e / b, jj = e % b;
      cr.G(p)[e] -= schur(X + (rg + t) * b, W + jj * b);
    }
    // new coupling A(q, p) = - W_q D W_p^T (rows q, columns p)
    for (int e = tid; e < b * b; e += T) {
      const int ii = e / b, jj = e % b;
      cr.E(p)[e] = hq ? -schur(X + (rq + ii) * b, W + jj * b) : 0.0;
    }
  }
  if (hq) {
    double* Dq = cr.D(q);
    for (int e = tid; e < b * b; e += T) {
      const int ii = e / b, jj = e % b;
      if (jj <= ii) {
        double v = Dq[e];
        for (int m = 0; m < b; ++m) v -= X[(rq + ii) * b + m] * W[(rq + jj) * b + m];
        Dq[e] = v;
      }
    }
    for (int ii = tid; ii < b; ii += T)
      cr.ps(q)[ii] = fmax(cr.ps(q)[ii], diag_scale(X + (rq + ii) * b, W + (rq + ii) * b));
    for (int e = tid; e < w * b; e += T) {
      const int t = e / b, jj = e % b;
      cr.G(q)[e] -= schur(X + (rg + t) * b, W + (rq + jj) * b);
    }
  }
  for (int e = tid; e < w * w; e += T) {
    const int t = e / w, u = e % w;
    cr.Sc(k)[e] = u <= t ? schur(X + (rg + t) * b, W + (rg + u) * b) : 0.0;
  }
  for (int t = tid; t < w; t += T) cr.Sps(k)[t] = diag_scale(X + (rg + t) * b, W + (rg + t) * b);
  if (tid == 0) {
    parts[3 * k] = npos;
    parts[3 * k + 1] = nneg;
    parts[3 * k + 2] = nzero;
  }
}

// border block: S minus every separator's contribution (separator order), its
// LDL^T, then the separator system's inertia into out[0..2]
__global__ void cr_border_k(Cr cr, int ns, double* __restrict__ S, double* __restrict__ Sps,
                            double* __restrict__ Sdinv, long long* __restrict__ parts, long long* __restrict__ out) {
  const int w = cr.w;
  if (threadIdx.x != 0) return;
  for (int t = 0; t < w; ++t)
    for (int u = 0; u <= t; ++u) {
      double v = S[t * w + u];
      for (long long k = 0; k < ns; ++k) v -= cr.Sc(k)[t * w + u];
      S[t * w + u] = v;
    }
  for (int t = 0; t < w; ++t)
    for (long long k = 0; k < ns; ++k) Sps[t] = fmax(Sps[t], cr.Sps(k)[t]);
  long long npos = 0, nneg = 0, nzero = 0;
  for (int t = 0; t < w; ++t) {
    const double d = S[t * w + t];
    const bool zero = zero_pivot(d, Sps[t]);
    const double dinv = zero ? 0.0 : 1.0 / d;
    Sdinv[t] = dinv;
    if (zero)
      ++nzero;
    else if (d > 0)
      ++npos;
    else
      ++nneg;
    for (int u = t + 1; u < w; ++u) {
      const double lu = S[u * w + t] * dinv;
      for (int v = t + 1; v <= u; ++v) {
        const double upd = lu * S[v * w + t];
        S[u * w + v] -= upd;
        if (u == v) Sps[u] = fmax(Sps[u], fabs(upd));
      }
    }
    for (int u = t + 1; u < w; ++u) S[u * w + t] *= dinv;
  }
  for (long long k = 0; k < ns; ++k) {
    npos += parts[3 * k];
    nneg += parts[3 * k + 1];
    nzero += parts[3 * k + 2];
  }
  out[0] = npos;
  out[1] = nneg;
  out[2] = nzero;
}

// forward: y_k = L_k^-1 r_k; r_p -= W_p y_k; r_q -= W_q y_k; rg_k = W_g y_k
__global__ void cr_fwd_k(Cr cr, int ns, int level, int phase, double* __restrict__ v) {
  __shared__ double y[64];
  const int b = cr.b, w = cr.w, lane = threadIdx.x;
  const long long i = 2LL * blockIdx.x + phase;
  const long long step = 1LL << level;
  const long long k = step * (2 * i + 1) - 1;
  if (k >= ns) return;
  const long long p = k - step, q = k + step;
  const double* L = cr.D(k);
  double* vk = v + k * b;
  for (int m = lane; m < b; m += 32) y[m] = vk[m];
  __syncwarp();
  for (int m = 1; m < b; ++m) {
    double part = 0.0;
    for (int n = lane; n < m; n += 32) part += L[m * b + n] * y[n];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) y[m] -= part;
    __syncwarp();
  }
  for (int m = lane; m < b; m += 32) vk[m] = y[m];
  if (p >= 0) {
    const double* Wp = cr.Wp(k);
    for (int r = lane; r < b; r += 32) {
      double s = 0.0;
      for (int m = 0; m < b; ++m) s += Wp[r * b + m] * y[m];
      v[p * b + r] -= s;
    }
  }
  if (q < ns) {
    const double* Wq = cr.Wq(k);
    for (int r = lane; r < b; r += 32) {
      double s = 0.0;
      for (int m = 0; m < b; ++m) s += Wq[r * b + m] * y[m];
      v[q * b + r] -= s;
    }
  }
  const double* Wg = cr.Wg(k);
  for (int t = lane; t < w; t += 32) {
    double s = 0.0;
    for (int m = 0; m < b; ++m) s += Wg[t * b + m] * y[m];
    cr.rg(k)[t] = s;
  }
}

// border: r_g minus the separators' contributions (separator order), then
// the border block's LDL^T solve; x_g in place
__global__ void cr_border_solve_k(Cr cr, int ns, const double* __restrict__ S, const double* __restrict__ Sdinv,
                                  double* __restrict__ vg) {
  const int w = cr.w;
  if (threadIdx.x != 0) return;
  for (int t = 0; t < w; ++t) {
    double s = vg[t];
    for (long long k = 0; k < ns; ++k) s -= cr.rg(k)[t];
    vg[t] = s;
  }
  for (int t = 0; t < w; ++t)
    for (int u = 0; u < t; ++u) vg[t] -= S[t * w + u] * vg[u];
  for (int t = 0; t < w; ++t) vg[t] *= Sdinv[t];
  for (int t = w - 1; t >= 0; --t)
    for (int u = t + 1; u < w; ++u) vg[t] -= S[u * w + t] * vg[u];
}

// backward: x_k = L_k^-T (D_k^-1 y_k - W_p^T x_p - W_q^T x_q - W_g^T x_g)
__global__ void cr_bwd_k(Cr cr, int ns, int level, double* __restrict__ v, const double* __restrict__ vg) {
  __shared__ double z[64];
  const int b = cr.b, w = cr.w, lane = threadIdx.x;
  const long long step = 1LL << level;
  const long long k = step * (2LL * blockIdx.x + 1) - 1;
  if (k >= ns) return;
  const long long p = k - step, q = k + step;
  const double* L = cr.D(k);
  const double* dv = cr.dinv(k);
  double* vk = v + k * b;
  for (int m = lane; m < b; m += 32) {
    double s = dv[m] * vk[m];
    if (p >= 0)
      for (int r = 0; r < b; ++r) s -= cr.Wp(k)[r * b + m] * v[p * b + r];
    if (q < ns)
      for (int r = 0; r < b; ++r) s -= cr.Wq(k)[r * b + m] * v[q * b + r];
    for (int t = 0; t < w; ++t) s -= cr.Wg(k)[t * b + m] * vg[t];
    z[m] = s;
  }
  __syncwarp();
  for (int m = b - 2; m >= 0; --m) {
    double part = 0.0;
    for (int n = m + 1 + lane; n < b; n += 32) part += L[n * b + m] * z[n];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) z[m] -= part;
    __syncwarp();
  }
  for (int m = lane; m < b; m += 32) vk[m] = z[m];
}

Cr make_cr(double* base, int b, int w) { return Cr{base, b, w, cr_per(b, w)}; }

int levels_of(int ns) {
  int L = 0;
  while ((1LL << (L + 1)) <= ns) ++L;
  return L;  // levels 0..L
}

}  // namespace

long long cr_length(int ns, int b, int w) {
  return static_cast<long long>(ns) * cr_per(b, w) + static_cast<long long>(w) * w + 2LL * w;
}

size_t cr_smem(int b, int w) {
  const size_t nrow = 2 * static_cast<size_t>(b) + w;
  return sizeof(double) * (static_cast<size_t>(b) * b + 2 * b + 2 * nrow * b);
}

void cr_factor(const BandPlan& P, const BandSeg& sep, const double* buf, const double* primal, double dw, double dc,
               double* cr, long long* crparts, long long* sep_inertia, cudaStream_t s) {
  const int ns = P.nseg - 1, b = P.b, w = P.wg;
  Cr c = make_cr(cr, b, w);
  double* S = cr + static_cast<long long>(ns) * c.per;
  double* Sps = S + w * w;
  double* Sdinv = Sps + w;
  SepView sv{buf + sep.band, buf + sep.border, buf + sep.S, buf + sep.ps0, primal + sep.pos, sep.n};
  cr_init_k<<<ns + 1, 256, 0, s>>>(c, sv, ns, dw, dc, S, Sps);
  const size_t smem = cr_smem(b, w);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(cr_elim_k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  const int L = levels_of(ns);
  for (int l = 0; l <= L; ++l) {
    const long long cnt = ((static_cast<long long>(ns) >> l) + 1) / 2;  // k = 2^l (2i+1) - 1 < ns
    for (int ph = 0; ph < 2; ++ph) {
      const long long blocks = (cnt + 1 - ph) / 2;
      if (blocks > 0) cr_elim_k<<<static_cast<unsigned>(blocks), 256, smem, s>>>(c, ns, l, ph, crparts);
    }
  }
  cr_border_k<<<1, 32, 0, s>>>(c, ns, S, Sps, Sdinv, crparts, sep_inertia);
}

void cr_solve(const BandPlan& P, const BandSeg& sep, double* cr, double* work, cudaStream_t s) {
  const int ns = P.nseg - 1, b = P.b, w = P.wg;
  Cr c = make_cr(cr, b, w);
  const double* S = cr + static_cast<long long>(ns) * c.per;
  const double* Sdinv = S + w * w + w;
  double* v = work + sep.pos;
  double* vg = v + sep.n;
  const int L = levels_of(ns);
  for (int l = 0; l <= L; ++l) {
    const long long cnt = ((static_cast<long long>(ns) >> l) + 1) / 2;
    for (int ph = 0; ph < 2; ++ph) {
      const long long blocks = (cnt + 1 - ph) / 2;
      if (blocks > 0) cr_fwd_k<<<static_cast<unsigned>(blocks), 32, 0, s>>>(c, ns, l, ph, v);
    }
  }
  cr_border_solve_k<<<1, 32, 0, s>>>(c, ns, S, Sdinv, vg);
  for (int l = L; l >= 0; --l) {
    const long long cnt = ((static_cast<long long>(ns) >> l) + 1) / 2;
    if (cnt > 0) cr_bwd_k<<<static_cast<unsigned>(cnt), 32, 0, s>>>(c, ns, l, v, vg);
  }
}

}  // namespace ocg::dev
