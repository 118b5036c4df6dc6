// Device numerics of the reference-order LDL^T (refldl.hpp).
//
// Factorization, per call (5 launches):
//   1. W = 0; K's values into the fronts' first columns and the leaves'
//      A columns, +delta_w / -delta_c on the diagonal (ldl.cpp:164-166).
//   2. leaves: pivot, zero test, L column (ldl.cpp:198-211 with an empty
//      pattern), one thread each.
//   3. leaf update matrices pre-assembled into their parents' fronts, one
//      thread per parent, leaves in ascending order.
//   4. the chain: ONE warp walks the remaining columns in elimination order;
//      per column it adds the stashed update matrices of children that are
//      not the previous column, takes the pivot, writes L's column and
//      extend-adds its own update matrix into the next column's front (its
//      parent) or stashes it for a later parent.
// Every product and difference is rounded separately (no FMA contraction),
// as in the reference's loop; only the order of the terms of a sum differs.
//
// Solve (sparse::solve, ldl.cpp:222-247): forward substitution as leaf
// terms (parallel) + the chain (one warp, update vectors), the diagonal, and
// backward substitution as the chain (one warp, reverse order) + leaves.
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <string>

#include "refldl.hpp"

namespace ocg::rl {
namespace {

constexpr int kThreads = 256;
constexpr int kTab = (kMaxFront - 1) * kMaxFront / 2;  // packed entries of the largest update matrix

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("refldl ") + what + ": " + cudaGetErrorString(e));
}

unsigned grid_for(int64_t n) {
  const int64_t b = (n + kThreads - 1) / kThreads;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

__device__ __forceinline__ int64_t tri(int64_t a) { return a * (a + 1) / 2; }  // entry (a, b) of a packed front: tri(a) + b

__device__ __forceinline__ bool zero_pivot(double d, double scale) {
  // ldl.cpp:203-205
  return !isfinite(d) || fabs(d) <= 1e-14 * fmax(scale, 1e-30);
}

__global__ void scatter_k(const int64_t* __restrict__ dst, const int64_t* __restrict__ dpos,
                          const int64_t* __restrict__ msd, const int8_t* __restrict__ primal,
                          const double* __restrict__ kval, int64_t nnz, double dw, double dc, double* __restrict__ W) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = kval[i];
    const int64_t d = dpos[i];
    if (d >= 0) v = __dadd_rn(v, primal[d] ? dw : -dc);
    W[dst[i]] = v;
    if (msd[i] >= 0) W[msd[i]] = fabs(v);  // pivot scale starts at |a_kk + delta| (ldl.cpp:169)
  }
}

__device__ __forceinline__ void count_pivot(double d, bool zero, unsigned long long* c) {
  if (zero)
    ++c[2];
  else if (d > 0)
    ++c[0];
  else
    ++c[1];
}

__global__ void leaf_k(Dev P, const double* __restrict__ W, double* __restrict__ D, double* __restrict__ Dinv,
                       double* __restrict__ Lx, unsigned long long* __restrict__ inertia) {
  unsigned long long c[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P.nleaf;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pos = P.lf_pos[i];
    const int f = P.lf_f[i];
    const double* A = W + P.lf_aoff[i];
    const double d = A[0];
    const bool zero = zero_pivot(d, fabs(d));  // no updates: the scale is |a_kk + delta|
    const double dinv = zero ? 0.0 : __drcp_rn(d);
    D[pos] = d;
    Dinv[pos] = dinv;
    count_pivot(d, zero, c);
    const int64_t lp = P.Lp[pos];
    for (int t = 1; t < f; ++t) Lx[lp + t - 1] = __dmul_rn(A[t], dinv);
  }
  for (int q = 0; q < 3; ++q) {
    unsigned long long v = c[q];
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(inertia + q, v);
  }
}

__global__ void preassemble_k(Dev P, double* __restrict__ W, const double* __restrict__ Lx) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < P.npa;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = P.pa_j[q];
    const int f = P.nl_f[j];
    double* F = W + P.nl_foff[j];
    double* ms = F + tri(f);
    for (int64_t t = P.pa_ptr[q]; t < P.pa_ptr[q + 1]; ++t) {
      const int i = P.pa_leaf[t];
      const int fc = P.lf_f[i];
      const double* A = W + P.lf_aoff[i];
      const int64_t lp = P.Lp[P.lf_pos[i]];
      const int32_t* r = P.rel + lp;
      // U(a, b) = 0 - L(b) * A(a): the leaf's updates of entries (r_a, r_b)
      for (int a = 1; a < fc; ++a) {
        const double Aa = A[a];
        const int64_t ra = tri(r[a - 1]);
        for (int b = 1; b <= a; ++b) F[ra + r[b - 1]] = __dsub_rn(F[ra + r[b - 1]], __dmul_rn(Lx[lp + b - 1], Aa));
        ms[r[a - 1]] = fmax(ms[r[a - 1]], fabs(__dmul_rn(Lx[lp + a - 1], Aa)));
      }
    }
  }
}

__device__ void build_tables(unsigned char* ta, unsigned char* tb) {
  for (int a = 1 + static_cast<int>(threadIdx.x); a < kMaxFront; a += blockDim.x)
    for (int b = 1; b <= a; ++b) {
      const int u = (a - 1) * a / 2 + b - 1;
      ta[u] = static_cast<unsigned char>(a);
      tb[u] = static_cast<unsigned char>(b);
    }
}

__global__ void __launch_bounds__(32) chain_factor_k(Dev P, double* __restrict__ W, double* __restrict__ stash,
                                                     double* __restrict__ D, double* __restrict__ Dinv,
                                                     double* __restrict__ Lx, unsigned long long* __restrict__ inertia) {
  __shared__ unsigned char ta[kTab], tb[kTab];
  build_tables(ta, tb);
  __syncwarp();
  const int lane = threadIdx.x;
  unsigned long long c[3] = {0, 0, 0};
  for (int64_t j = 0; j < P.nnl; ++j) {
    const int64_t pos = P.nl_pos[j];
    const int f = P.nl_f[j];
    double* F = W + P.nl_foff[j];
    double* ms = F + tri(f);
    const int64_t lp = P.Lp[pos];
    const int32_t* r = P.rel + lp;
    // update matrices of children that were not the previous column
    for (int64_t q = P.sc_ptr[j]; q < P.sc_ptr[j + 1]; ++q) {
      const int cj = P.sc_child[q];
      const int fc = P.nl_f[cj];
      const double* Us = stash + P.nl_soff[cj];
      const int32_t* rc = P.rel + P.Lp[P.nl_pos[cj]];
      const int tu = (fc - 1) * fc / 2;
      for (int u = lane; u < tu; u += 32) {
        const int64_t e = tri(rc[ta[u] - 1]) + rc[tb[u] - 1];
        F[e] = __dadd_rn(F[e], Us[u]);
      }
      for (int a = lane; a < fc - 1; a += 32) ms[rc[a]] = fmax(ms[rc[a]], Us[tu + a]);
      __syncwarp();
    }
    const double d = F[0];
    const bool zero = zero_pivot(d, ms[0]);
    const double dinv = zero ? 0.0 : __drcp_rn(d);
    if (lane == 0) {
      D[pos] = d;
      Dinv[pos] = dinv;
      count_pivot(d, zero, c);
    }
    for (int t = lane + 1; t < f; t += 32) Lx[lp + t - 1] = __dmul_rn(F[tri(t)], dinv);
    const int64_t so = P.nl_soff[j];
    if (so != kRoot) {
      double* Fn = nullptr;
      double* msn = nullptr;
      double* Us = nullptr;
      if (so == kChain) {
        const int fn = P.nl_f[j + 1];
        Fn = W + P.nl_foff[j + 1];
        msn = Fn + tri(fn);
      } else {
        Us = stash + so;
      }
      const int tu = (f - 1) * f / 2;
      for (int u = lane; u < tu; u += 32) {
        const int a = ta[u], b = tb[u];
        const double Lb = __dmul_rn(F[tri(b)], dinv);
        const double U = __dsub_rn(F[tri(a) + b], __dmul_rn(Lb, F[tri(a)]));
        if (Fn) {
          const int64_t e = tri(r[a - 1]) + r[b - 1];
          Fn[e] = __dadd_rn(Fn[e], U);
        } else {
          Us[u] = U;
        }
      }
      for (int a = lane + 1; a < f; a += 32) {
        const double Fa0 = F[tri(a)];
        const double m = fmax(ms[a], fabs(__dmul_rn(__dmul_rn(Fa0, dinv), Fa0)));
        if (Fn)
          msn[r[a - 1]] = fmax(msn[r[a - 1]], m);
        else
          Us[tu + a - 1] = m;
      }
    }
    __syncwarp();
  }
  if (lane == 0)
    for (int q = 0; q < 3; ++q)
      if (c[q]) atomicAdd(inertia + q, c[q]);
}

// ---- solves ------------------------------------------------------------------

__global__ void gather_k(const int64_t* __restrict__ perm, const double* __restrict__ rhs, double* __restrict__ y,
                         int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = rhs[perm[i]];
}

__global__ void scatter_out_k(const int64_t* __restrict__ perm, const double* __restrict__ xp, double* __restrict__ x,
                              int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[perm[i]] = xp[i];
}

// chain rows minus their leaf terms (leaf y = b: leaves have no incoming terms)
__global__ void fwd_leaf_k(Dev P, const double* __restrict__ Lx, double* __restrict__ y) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < P.nfl;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pos = P.nl_pos[P.fl_j[q]];
    double s = y[pos];
    for (int64_t t = P.fl_ptr[q]; t < P.fl_ptr[q + 1]; ++t) s = __dsub_rn(s, __dmul_rn(Lx[P.fl_lx[t]], y[P.fl_col[t]]));
    y[pos] = s;
  }
}

// vector fronts: V_j = [y_pos, 0, ...]
__global__ void vinit_k(Dev P, const double* __restrict__ y, double* __restrict__ V) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P.nnl;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double* v = V + P.nl_voff[j];
    v[0] = y[P.nl_pos[j]];
    for (int a = 1; a < P.nl_f[j]; ++a) v[a] = 0.0;
  }
}

__global__ void __launch_bounds__(32) fwd_chain_k(Dev P, const double* __restrict__ Lx, double* __restrict__ y,
                                                  double* __restrict__ V, double* __restrict__ Vs) {
  const int lane = threadIdx.x;
  for (int64_t j = 0; j < P.nnl; ++j) {
    const int f = P.nl_f[j];
    double* v = V + P.nl_voff[j];
    for (int64_t q = P.sc_ptr[j]; q < P.sc_ptr[j + 1]; ++q) {
      const int cj = P.sc_child[q];
      const int32_t* rc = P.rel + P.Lp[P.nl_pos[cj]];
      const double* us = Vs + P.nl_soff[cj];
      for (int a = lane; a < P.nl_f[cj] - 1; a += 32) v[rc[a]] = __dadd_rn(v[rc[a]], us[a]);
      __syncwarp();
    }
    const int64_t pos = P.nl_pos[j];
    const double yk = v[0];
    if (lane == 0) y[pos] = yk;
    const int64_t so = P.nl_soff[j];
    if (so != kRoot) {
      const int64_t lp = P.Lp[pos];
      const int32_t* r = P.rel + lp;
      double* vn = so == kChain ? V + P.nl_voff[j + 1] : nullptr;
      for (int a = lane + 1; a < f; a += 32) {
        const double u = __dsub_rn(v[a], __dmul_rn(Lx[lp + a - 1], yk));
        if (vn)
          vn[r[a - 1]] = __dadd_rn(vn[r[a - 1]], u);
        else
          Vs[so + a - 1] = u;
      }
    }
    __syncwarp();
  }
}

// backward: x-fronts X_j = [x_pos, x of the rows of column j]
__global__ void __launch_bounds__(32) bwd_chain_k(Dev P, const double* __restrict__ Lx, const double* __restrict__ Dinv,
                                                  const double* __restrict__ y, double* __restrict__ xp,
                                                  double* __restrict__ V) {
  const int lane = threadIdx.x;
  for (int64_t j = P.nnl - 1; j >= 0; --j) {
    const int64_t pos = P.nl_pos[j];
    const int f = P.nl_f[j];
    double* X = V + P.nl_voff[j];
    const int64_t lp = P.Lp[pos];
    const int32_t* r = P.rel + lp;
    const bool chain = P.nl_soff[j] == kChain;
    const double* Xn = chain ? V + P.nl_voff[j + 1] : nullptr;
    for (int a = lane + 1; a < f; a += 32) X[a] = chain ? Xn[r[a - 1]] : xp[P.Li[lp + a - 1]];
    __syncwarp();
    if (lane == 0) {
      double s = __dmul_rn(y[pos], Dinv[pos]);
      for (int a = 1; a < f; ++a) s = __dsub_rn(s, __dmul_rn(Lx[lp + a - 1], X[a]));
      X[0] = s;
      xp[pos] = s;
    }
    __syncwarp();
  }
}

__global__ void bwd_leaf_k(Dev P, const double* __restrict__ Lx, const double* __restrict__ Dinv,
                           const double* __restrict__ y, double* __restrict__ xp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P.nleaf;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pos = P.lf_pos[i];
    const int64_t lp = P.Lp[pos];
    double s = __dmul_rn(y[pos], Dinv[pos]);
    for (int t = 0; t < P.lf_f[i] - 1; ++t) s = __dsub_rn(s, __dmul_rn(Lx[lp + t], xp[P.Li[lp + t]]));
    xp[pos] = s;
  }
}

}  // namespace

void factor(const Dev& P, const double* kval, double delta_w, double delta_c, double* W, double* stash, double* D,
            double* Dinv, double* Lx, unsigned long long* inertia, cudaStream_t s) {
  ck(cudaMemsetAsync(W, 0, static_cast<size_t>(P.w_len) * sizeof(double), s), "memset W");
  ck(cudaMemsetAsync(inertia, 0, 3 * sizeof(unsigned long long), s), "memset inertia");
  scatter_k<<<grid_for(P.nnz), kThreads, 0, s>>>(P.sc_dst, P.sc_dpos, P.sc_ms, P.primal, kval, P.nnz, delta_w,
                                                delta_c, W);
  if (P.nleaf) leaf_k<<<grid_for(P.nleaf), kThreads, 0, s>>>(P, W, D, Dinv, Lx, inertia);
  if (P.npa) preassemble_k<<<grid_for(P.npa), kThreads, 0, s>>>(P, W, Lx);
  if (P.nnl) chain_factor_k<<<1, 32, 0, s>>>(P, W, stash, D, Dinv, Lx, inertia);
  ck(cudaGetLastError(), "factor launch");
}

void solve(const Dev& P, const double* Dinv, const double* Lx, const double* rhs, double* x, double* y, double* xp,
           double* V, double* Vs, cudaStream_t s) {
  gather_k<<<grid_for(P.dim), kThreads, 0, s>>>(P.perm, rhs, y, P.dim);
  if (P.nfl) fwd_leaf_k<<<grid_for(P.nfl), kThreads, 0, s>>>(P, Lx, y);
  if (P.nnl) {
    vinit_k<<<grid_for(P.nnl), kThreads, 0, s>>>(P, y, V);
    fwd_chain_k<<<1, 32, 0, s>>>(P, Lx, y, V, Vs);
    bwd_chain_k<<<1, 32, 0, s>>>(P, Lx, Dinv, y, xp, V);
  }
  if (P.nleaf) bwd_leaf_k<<<grid_for(P.nleaf), kThreads, 0, s>>>(P, Lx, Dinv, y, xp);
  scatter_out_k<<<grid_for(P.dim), kThreads, 0, s>>>(P.perm, xp, x, P.dim);
  ck(cudaGetLastError(), "solve launch");
}

}  // namespace ocg::rl
