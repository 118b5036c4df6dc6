// Batched interior-point kernels (batch_kernels.hpp). Every formula is the
// one of the single-instance kernel it batches (ipm_kernels.cu, kernels.cu,
// ipm.cpp's setup) — itself citing the reference line it follows — applied to
// instance ids[blockIdx.y]. Reductions: one block per instance, fixed
// thread partition and combine order, so an instance's result does not depend
// on which other instances share the launch.
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "batch_kernels.hpp"

namespace ocg::bdev {

namespace {

constexpr int kT = 256;
constexpr double kInfD = __builtin_huge_val();
constexpr double kPushIn = 1e-2;  // solver.cpp:52

__device__ __forceinline__ int64_t inst(const int* ids) { return ids[blockIdx.y]; }

// elementwise: grid (gx, nb) with a grid-stride loop over x
#define ELOOP(i, n)                                                                      \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
// reductions: one block per instance
#define BLOOP(i, n) for (int64_t i = threadIdx.x; i < (n); i += blockDim.x)

dim3 grid2(int64_t n, int nb) {
  int64_t want = (n + kT - 1) / kT;
  int64_t cap = 2048 / (nb > 0 ? nb : 1);
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return dim3(static_cast<unsigned>(want), static_cast<unsigned>(nb));
}
dim3 grid1(int nb) { return dim3(1, static_cast<unsigned>(nb)); }

template <int NV>
__device__ void block_reduce(double (&v)[NV], const int (&op)[NV], double* out, int os) {
  __shared__ double sh[NV][kT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double a = v[q];
    for (int o = 16; o > 0; o >>= 1) {
      const double b = __shfl_xor_sync(0xffffffffu, a, o);
      a = op[q] == 0 ? a + b : (op[q] == 1 ? fmax(a, b) : fmin(a, b));
    }
    if (lane == 0) sh[q][wid] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double a = sh[q][0];
      for (int w = 1; w < kT / 32; ++w) a = op[q] == 0 ? a + sh[q][w] : (op[q] == 1 ? fmax(a, sh[q][w]) : fmin(a, sh[q][w]));
      out[static_cast<int64_t>(blockIdx.y) * os + q] = a;
    }
  }
}

// reduced primal value v_i: x at the free slot, or the slack
__device__ __forceinline__ double v_at(const BDims& D, const BMaps& M, const double* x, const double* s, int64_t i) {
  return i < D.n_free ? x[M.free_slot[i]] : s[i - D.n_free];
}

// ipm.cpp setup(): push_into (solver.cpp:172-206), std::min / std::clamp semantics
__device__ __forceinline__ double push_into(double v, double l, double u) {
  const double d = u - l;
  const double w = d < 1.0 ? d : 1.0;
  const double wf = isfinite(w) ? w : 1.0;
  const double lo = isfinite(l) ? l + kPushIn * wf : -kInfD;
  const double hi = isfinite(u) ? u - kPushIn * wf : kInfD;
  return v < lo ? lo : (hi < v ? hi : v);
}

struct BV {  // per-instance bound pointers
  const double *lb, *ub;
  const int8_t *hl, *hu;
  const double* lcs;
};
__device__ __forceinline__ BV bounds_of(const BDims& D, const BBounds& B, int64_t b) {
  return {B.lb + b * D.ntot, B.ub + b * D.ntot, B.has_lb + b * D.ntot, B.has_ub + b * D.ntot,
          B.lcon_s + b * D.m_con};
}

// ---- evaluation reductions ----------------------------------------------------

constexpr int kChunk = 512;

__global__ void __launch_bounds__(256) obj_chunks_k(BDims D, const double* __restrict__ objv,
                                                    const int64_t* __restrict__ goff,
                                                    const int64_t* __restrict__ gcount,
                                                    const int64_t* __restrict__ cbase, double* __restrict__ partials,
                                                    const int* __restrict__ ids) {
  __shared__ double buf[8][kChunk];
  const int64_t b = inst(ids);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (c >= D.n_chunks) return;
  int g = 0;
  while (g + 1 < D.n_obj && cbase[g + 1] <= c) ++g;
  const int64_t lo = (c - cbase[g]) * kChunk;
  const int64_t hi = min(gcount[g], lo + kChunk);
  const int64_t n = hi - lo;
  const double* src = objv + b * D.objv_n + goff[g] + lo;
  for (int64_t i = lane; i < n; i += 32) buf[warp][i] = src[i];
  __syncwarp();
  if (lane == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += buf[warp][i];
    partials[b * D.n_chunks + c] = s;
  }
}

__global__ void obj_combine_k(BDims D, const double* __restrict__ partials, const int64_t* __restrict__ cbase,
                              const double* __restrict__ weights, const double* __restrict__ obj_scale,
                              double* __restrict__ f, int* __restrict__ flag, int os, const int* __restrict__ ids) {
  if (threadIdx.x != 0) return;
  const int64_t b = inst(ids);
  const double* p = partials + b * D.n_chunks;
  double total = 0.0;
  for (int g = 0; g < D.n_obj; ++g) {
    double part = 0.0;
    for (int64_t c = cbase[g]; c < cbase[g + 1]; ++c) part += p[c];
    total += weights[g] * part;
  }
  const double fs = obj_scale[b] * total;
  f[static_cast<int64_t>(blockIdx.y) * os] = fs;
  if (!(fabs(fs) <= DBL_MAX)) flag[b] = 1;
}

__global__ void __launch_bounds__(256) gather_grad_k(BDims D, const double* __restrict__ src,
                                                     const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                     double* __restrict__ out, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  src += b * D.gnnz;
  out += b * D.nvar;
  ELOOP(i, D.nvar) {
    double s = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += src[idx[p]];
    out[i] = s;
  }
}

__global__ void max_abs_k(const double* __restrict__ v, int64_t n, double* __restrict__ out,
                          int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  v += b * n;
  double r[1] = {0.0};
  const int op[1] = {1};
  BLOOP(i, n) r[0] = fmax(r[0], fabs(v[i]));
  block_reduce<1>(r, op, out, os);
}

__global__ void take_flags_k(int* __restrict__ flag, double* __restrict__ out, int stride, int slot, int nb,
                             const int* __restrict__ ids) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nb) return;
  const int b = ids[y];
  out[static_cast<int64_t>(y) * stride + slot] = flag[b] != 0 ? 1.0 : 0.0;
  flag[b] = 0;
}

// eval.cpp:260-280 with ipm.cpp's failure rule: a failed evaluation keeps unit scales
__global__ void scaling_k(BDims D, const double* __restrict__ grad, const double* __restrict__ jac,
                          const int64_t* __restrict__ jrow_ptr, const int64_t* __restrict__ jrow_e,
                          const int* __restrict__ flag, const double* __restrict__ weights, int enabled,
                          double* __restrict__ obj_scale, double* __restrict__ row_scale, double* __restrict__ objw,
                          const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  grad += b * D.nvar;
  jac += b * D.jnnz;
  double* rs = row_scale + b * D.m_con;
  const bool use = enabled && flag[b] == 0;
  __shared__ double sh[kT / 32];
  __shared__ double os_sh;
  double a = 0.0;
  if (use) BLOOP(i, D.nvar) a = fmax(a, fabs(grad[i]));
  for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double gmax = sh[0];
    for (int w = 1; w < kT / 32; ++w) gmax = fmax(gmax, sh[w]);
    double os = 1.0;
    if (use && gmax > 0.0) os = 100.0 / gmax < 1.0 ? 100.0 / gmax : 1.0;
    os_sh = os;
    obj_scale[b] = os;
  }
  __syncthreads();
  const double gm = os_sh;
  BLOOP(q, D.n_obj) objw[b * D.n_obj + q] = gm * weights[q];
  BLOOP(row, D.m_con) {
    double jm = 0.0;
    if (use)
      for (int64_t p = jrow_ptr[row]; p < jrow_ptr[row + 1]; ++p) jm = fmax(jm, fabs(jac[jrow_e[p]]));
    rs[row] = jm > 0.0 ? (100.0 / jm < 1.0 ? 100.0 / jm : 1.0) : 1.0;
  }
}

// ---- KKT ------------------------------------------------------------------------

__global__ void __launch_bounds__(256) kkt_assemble_k(BDims D, const double* __restrict__ hess,
                                                      const double* __restrict__ jac,
                                                      const double* __restrict__ sigma,
                                                      const int64_t* __restrict__ ptr,
                                                      const int64_t* __restrict__ code, double* __restrict__ val,
                                                      const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  hess += b * D.hnnz;
  jac += b * D.jnnz;
  sigma += b * D.ntot;
  val += b * D.knnz;
  const int64_t H = D.hnnz, HJ = D.hnnz + D.jnnz, HJS = HJ + D.n_slack;
  ELOOP(p, D.knnz) {
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
      else if (c < HJS + D.ntot)
        v = sigma[c - HJS];
      else
        v = 0.0;
      s += v;
    }
    val[p] = s;
  }
}

__global__ void __launch_bounds__(256) sym_matvec_k(BDims D, const double* __restrict__ val,
                                                    const int64_t* __restrict__ rptr, const int64_t* __restrict__ col,
                                                    const int64_t* __restrict__ vidx, const double* __restrict__ x,
                                                    double* __restrict__ y, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  val += b * D.knnz;
  x += b * D.dim;
  y += b * D.dim;
  ELOOP(i, D.dim) {
    double s = 0.0;
    for (int64_t p = rptr[i]; p < rptr[i + 1]; ++p) s += val[vidx[p]] * x[col[p]];
    y[i] = s;
  }
}

__global__ void sym_norm_inf_k(BDims D, const double* __restrict__ val, const int64_t* __restrict__ rptr,
                               const int64_t* __restrict__ vidx, double* __restrict__ out,
                               int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  val += b * D.knnz;
  double r[1] = {0.0};
  const int op[1] = {1};
  BLOOP(i, D.dim) {
    double s = 0.0;
    for (int64_t p = rptr[i]; p < rptr[i + 1]; ++p) s += fabs(val[vidx[p]]);
    r[0] = fmax(r[0], s);
  }
  block_reduce<1>(r, op, out, os);
}

__global__ void __launch_bounds__(256) jt_lambda_k(BDims D, const double* __restrict__ jac,
                                                   const double* __restrict__ lam, const int64_t* __restrict__ ptr,
                                                   const int64_t* __restrict__ e_idx,
                                                   const int64_t* __restrict__ dual_idx,
                                                   const int64_t* __restrict__ slack_dual, double* __restrict__ out,
                                                   const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  jac += b * D.jnnz;
  lam += b * D.m;
  out += b * D.ntot;
  ELOOP(i, D.ntot) {
    double s = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += jac[e_idx[p]] * lam[dual_idx[p]];
    if (i >= D.n_free) s -= lam[slack_dual[i - D.n_free]];
    out[i] = s;
  }
}

// ---- setup ----------------------------------------------------------------------

__global__ void broadcast_rows_k(double* __restrict__ a, int64_t n, int nb) {
  const int64_t total = n * (nb - 1);
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[n + q] = a[q % n];
}

// ipm.cpp setup(): xlo = max(lvar, lcon rows), xhi = min(uvar, ucon rows) per
// folded slot (std::max / std::min expressions, rows in index order)
__global__ void fold_bounds_k(BDims D, const int64_t* __restrict__ fptr, const int64_t* __restrict__ frow,
                              const int64_t* __restrict__ prim_index, double* __restrict__ xlo,
                              double* __restrict__ xhi, const double* __restrict__ lcon,
                              const double* __restrict__ ucon, int* __restrict__ contra, int* __restrict__ bad,
                              const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  xlo += b * D.nvar;
  xhi += b * D.nvar;
  lcon += b * D.m_con;
  ucon += b * D.m_con;
  ELOOP(sl, D.nvar) {
    double lo = xlo[sl], hi = xhi[sl];
    for (int64_t p = fptr[sl]; p < fptr[sl + 1]; ++p) {
      const int64_t r = frow[p];
      lo = lo < lcon[r] ? lcon[r] : lo;
      hi = ucon[r] < hi ? ucon[r] : hi;
    }
    xlo[sl] = lo;
    xhi[sl] = hi;
    if (lo > hi) atomicOr(contra + b, 1);
    if ((prim_index[sl] < 0) != (lo == hi)) atomicOr(bad + b, 1);
  }
}

// Solver::setup_bounds (solver.cpp:125-170) as ipm.cpp's setup() computes it
__global__ void setup_bounds_k(BDims D, BMaps M, const double* __restrict__ xlo, const double* __restrict__ xhi,
                               const double* __restrict__ lcon, const double* __restrict__ ucon,
                               const double* __restrict__ row_scale, double relax, double* __restrict__ lb,
                               double* __restrict__ ub, int8_t* __restrict__ hl, int8_t* __restrict__ hu,
                               double* __restrict__ lcon_s, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  xlo += b * D.nvar;
  xhi += b * D.nvar;
  lcon += b * D.m_con;
  ucon += b * D.m_con;
  row_scale += b * D.m_con;
  lb += b * D.ntot;
  ub += b * D.ntot;
  hl += b * D.ntot;
  hu += b * D.ntot;
  lcon_s += b * D.m_con;
  ELOOP(r, D.m_con) lcon_s[r] = row_scale[r] * lcon[r];
  ELOOP(i, D.ntot) {
    double l = -kInfD, u = kInfD;
    int8_t a = 0, c = 0;
    if (i < D.n_free) {
      const int64_t sl = M.free_slot[i];
      if (isfinite(xlo[sl])) {
        l = xlo[sl];
        a = 1;
      }
      if (isfinite(xhi[sl])) {
        u = xhi[sl];
        c = 1;
      }
    } else {
      const int64_t r = M.slack_of[i - D.n_free];
      const double ls = row_scale[r] * lcon[r], us = row_scale[r] * ucon[r];
      if (isfinite(ls)) {
        l = ls;
        a = 1;
      }
      if (isfinite(us)) {
        u = us;
        c = 1;
      }
    }
    if (relax > 0.0) {
      if (a) l -= relax * (1.0 < fabs(l) ? fabs(l) : 1.0);
      if (c) u += relax * (1.0 < fabs(u) ? fabs(u) : 1.0);
    }
    lb[i] = l;
    ub[i] = u;
    hl[i] = a;
    hu[i] = c;
  }
}

// Solver::initialize_iterate (solver.cpp:172-206): fixed slots at their
// value, free slots pushed inside their bounds
__global__ void init_x_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x0, const double* __restrict__ xlo,
                         const double* __restrict__ xhi, double* __restrict__ x, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  x0 += b * D.nvar;
  xlo += b * D.nvar;
  xhi += b * D.nvar;
  x += b * D.nvar;
  ELOOP(sl, D.nvar) {
    double v = x0[sl];
    if (xlo[sl] == xhi[sl]) v = xlo[sl];
    const int64_t i = M.prim_index[sl];
    if (i >= 0) v = push_into(v, V.lb[i], V.ub[i]);
    x[sl] = v;
  }
}

__global__ void init_slacks_duals_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x,
                                    const double* __restrict__ c, double mu, double* __restrict__ s,
                                    double* __restrict__ zl, double* __restrict__ zu, double* __restrict__ lambda,
                                    const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  x += b * D.nvar;
  c += b * D.m_con;
  s += b * D.n_slack;
  zl += b * D.ntot;
  zu += b * D.ntot;
  lambda += b * D.m;
  ELOOP(i, D.ntot) {
    double v;
    if (i < D.n_free) {
      v = x[M.free_slot[i]];
    } else {
      const int64_t k = i - D.n_free;
      v = push_into(c[M.slack_of[k]], V.lb[i], V.ub[i]);
      s[k] = v;
    }
    zl[i] = V.hl[i] ? mu / (v - V.lb[i]) : 0.0;
    zu[i] = V.hu[i] ? mu / (V.ub[i] - v) : 0.0;
  }
  ELOOP(d, D.m) lambda[d] = 0.0;
}

// ---- iteration vector work -----------------------------------------------------

// solver.cpp:206-215 + :219-223
__global__ void residual_theta_k(BDims D, BMaps M, BBounds B, const double* __restrict__ c,
                                 const double* __restrict__ s, double* __restrict__ g, double* __restrict__ out,
                                 int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  c += b * D.m_con;
  s += b * D.n_slack;
  g += b * D.m;
  double r[1] = {0.0};
  const int op[1] = {0};
  BLOOP(d, D.m) {
    const int64_t row = M.dual_row[d];
    const int64_t k = M.slack_index[row];
    const double gd = c[row] - (k >= 0 ? s[k] : V.lcs[row]);
    g[d] = gd;
    r[0] += fabs(gd);
  }
  block_reduce<1>(r, op, out, os);
}

// solver.cpp:367-373
__global__ void sigma_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                        const double* __restrict__ zl, const double* __restrict__ zu, double* __restrict__ out,
                        const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  x += b * D.nvar;
  s += b * D.n_slack;
  zl += b * D.ntot;
  zu += b * D.ntot;
  out += b * D.ntot;
  ELOOP(i, D.ntot) {
    const double v = v_at(D, M, x, s, i);
    double t = 0.0;
    if (V.hl[i]) t += zl[i] / (v - V.lb[i]);
    if (V.hu[i]) t += zu[i] / (V.ub[i] - v);
    out[i] = t;
  }
}

// solver.cpp:381-389
__global__ void rhs_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                      const double* __restrict__ grad, const double* __restrict__ jtlam, const double* __restrict__ g,
                      const double* __restrict__ mu_, double* __restrict__ out, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double mu = mu_[blockIdx.y];
  x += b * D.nvar;
  s += b * D.n_slack;
  grad += b * D.nvar;
  jtlam += b * D.ntot;
  g += b * D.m;
  out += b * D.dim;
  ELOOP(i, D.ntot + D.m) {
    if (i < D.ntot) {
      const double v = v_at(D, M, x, s, i);
      double rd = (i < D.n_free ? grad[M.free_slot[i]] : 0.0) + jtlam[i];
      if (V.hl[i]) rd -= mu / (v - V.lb[i]);
      if (V.hu[i]) rd += mu / (V.ub[i] - v);
      out[i] = -rd;
    } else {
      out[i] = -g[i - D.ntot];
    }
  }
}

// solver.cpp:434-441
__global__ void trial_k(BDims D, BMaps M, const double* __restrict__ x, const double* __restrict__ s,
                        const double* __restrict__ dir, const double* __restrict__ a_, double* __restrict__ xt,
                        double* __restrict__ st, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const double a = a_[blockIdx.y];
  x += b * D.nvar;
  s += b * D.n_slack;
  dir += b * D.dim;
  xt += b * D.nvar;
  st += b * D.n_slack;
  ELOOP(sl, D.nvar) {
    const int64_t i = M.prim_index[sl];
    xt[sl] = i >= 0 ? x[sl] + a * dir[i] : x[sl];
  }
  ELOOP(k, D.n_slack) st[k] = s[k] + a * dir[D.n_free + k];
}

// solver.cpp:641-646
__global__ void expand_k(BDims D, BMaps M, const double* __restrict__ lambda, double* __restrict__ full,
                         const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  lambda += b * D.m;
  full += b * D.m_con;
  ELOOP(r, D.m_con) {
    const int64_t d = M.dual_index[r];
    full[r] = d >= 0 ? lambda[d] : 0.0;
  }
}

__global__ void axpy_m_k(BDims D, const double* __restrict__ a_, const double* xv, const double* yv, double* out,
                         const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const double a = a_[blockIdx.y];
  xv += b * D.m;
  yv += b * D.m;
  out += b * D.m;
  ELOOP(i, D.m) out[i] = a * xv[i] + yv[i];
}

__global__ void rhs_soc_k(BDims D, const double* __restrict__ rhs, const double* __restrict__ gsoc,
                          double* __restrict__ out, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  rhs += b * D.dim;
  gsoc += b * D.m;
  out += b * D.dim;
  ELOOP(i, D.ntot + D.m) out[i] = i < D.ntot ? rhs[i] : -gsoc[i - D.ntot];
}

__global__ void add_dim_k(BDims D, double* __restrict__ x, const double* __restrict__ dx,
                          const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  x += b * D.dim;
  dx += b * D.dim;
  ELOOP(i, D.dim) x[i] += dx[i];
}

__global__ void commit_k(BDims D, double* __restrict__ x, const double* __restrict__ xt, double* __restrict__ s,
                         const double* __restrict__ st, double* __restrict__ c, const double* __restrict__ ct,
                         double* __restrict__ grad, const double* __restrict__ gradt, double* __restrict__ step,
                         const double* __restrict__ step2, const double* __restrict__ swap,
                         const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  ELOOP(i, D.nvar) {
    x[b * D.nvar + i] = xt[b * D.nvar + i];
    grad[b * D.nvar + i] = gradt[b * D.nvar + i];
  }
  ELOOP(i, D.n_slack) s[b * D.n_slack + i] = st[b * D.n_slack + i];
  ELOOP(i, D.m_con) c[b * D.m_con + i] = ct[b * D.m_con + i];
  if (swap && swap[blockIdx.y] != 0.0) ELOOP(i, D.dim) step[b * D.dim + i] = step2[b * D.dim + i];
}

// solver.cpp:598-617
__global__ void accept_k(BDims D, BMaps M, BBounds B, const double* __restrict__ step, const double* __restrict__ dzl,
                         const double* __restrict__ dzu, const double* __restrict__ scal,
                         const double* __restrict__ xn, const double* __restrict__ sn, double* __restrict__ lambda,
                         double* __restrict__ zl, double* __restrict__ zu, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double alpha = scal[blockIdx.y * 4], alpha_z = scal[blockIdx.y * 4 + 1], mu = scal[blockIdx.y * 4 + 2],
               kappa = scal[blockIdx.y * 4 + 3];
  step += b * D.dim;
  dzl += b * D.ntot;
  dzu += b * D.ntot;
  xn += b * D.nvar;
  sn += b * D.n_slack;
  lambda += b * D.m;
  zl += b * D.ntot;
  zu += b * D.ntot;
  ELOOP(i, D.ntot + D.m) {
    if (i >= D.ntot) {
      lambda[i - D.ntot] += alpha * step[i];
      continue;
    }
    double l = zl[i] + alpha_z * dzl[i];
    double u = zu[i] + alpha_z * dzu[i];
    const double v = v_at(D, M, xn, sn, i);
    if (V.hl[i]) {
      const double d = v - V.lb[i];
      l = fmin(fmax(l, mu / (kappa * d)), kappa * mu / d);
    }
    if (V.hu[i]) {
      const double d = V.ub[i] - v;
      u = fmin(fmax(u, mu / (kappa * d)), kappa * mu / d);
    }
    zl[i] = l;
    zu[i] = u;
  }
}

// ---- reductions ------------------------------------------------------------------

// solver.cpp:225-242
__global__ void barrier_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                          double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  x += b * D.nvar;
  s += b * D.n_slack;
  double r[2] = {0.0, 0.0};
  const int op[2] = {0, 0};
  BLOOP(i, D.ntot) {
    const double vi = v_at(D, M, x, s, i);
    if (V.hl[i]) {
      const double d = vi - V.lb[i];
      if (d <= 0.0)
        r[1] += 1.0;
      else
        r[0] += log(d);
    }
    if (V.hu[i]) {
      const double d = V.ub[i] - vi;
      if (d <= 0.0)
        r[1] += 1.0;
      else
        r[0] += log(d);
    }
  }
  block_reduce<2>(r, op, out, os);
}

// solver.cpp:260-287
__global__ void kkt_error_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                            const double* __restrict__ zl, const double* __restrict__ zu,
                            const double* __restrict__ lambda, const double* __restrict__ grad,
                            const double* __restrict__ jtlam, const double* __restrict__ g,
                            const double* __restrict__ mu_, double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double mu = mu_[blockIdx.y];
  x += b * D.nvar;
  s += b * D.n_slack;
  zl += b * D.ntot;
  zu += b * D.ntot;
  lambda += b * D.m;
  grad += b * D.nvar;
  jtlam += b * D.ntot;
  g += b * D.m;
  double r[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int op[5] = {0, 0, 1, 1, 1};
  BLOOP(i, D.ntot) {
    r[0] += fabs(zl[i]) + fabs(zu[i]);
    const double rd = (i < D.n_free ? grad[M.free_slot[i]] : 0.0) + jtlam[i] - zl[i] + zu[i];
    r[2] = fmax(r[2], fabs(rd));
    const double vi = v_at(D, M, x, s, i);
    if (V.hl[i]) r[4] = fmax(r[4], fabs((vi - V.lb[i]) * zl[i] - mu));
    if (V.hu[i]) r[4] = fmax(r[4], fabs((V.ub[i] - vi) * zu[i] - mu));
  }
  BLOOP(d, D.m) {
    r[1] += fabs(lambda[d]);
    r[3] = fmax(r[3], fabs(g[d]));
  }
  block_reduce<5>(r, op, out, os);
}

// solver.cpp:399-406 / :473-483
__global__ void ftb_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                      const double* __restrict__ dir, const double* __restrict__ tau_, double* __restrict__ out,
                      int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double tau = tau_[blockIdx.y];
  x += b * D.nvar;
  s += b * D.n_slack;
  dir += b * D.dim;
  double r[1] = {1.0};
  const int op[1] = {2};
  BLOOP(i, D.ntot) {
    const double dv = dir[i];
    const double vi = v_at(D, M, x, s, i);
    if (V.hl[i] && dv < 0.0) r[0] = fmin(r[0], -tau * (vi - V.lb[i]) / dv);
    if (V.hu[i] && dv > 0.0) r[0] = fmin(r[0], tau * (V.ub[i] - vi) / dv);
  }
  block_reduce<1>(r, op, out, os);
}

// solver.cpp:408-415
__global__ void dphi_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                       const double* __restrict__ grad, const double* __restrict__ dir, const double* __restrict__ mu_,
                       double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double mu = mu_[blockIdx.y];
  x += b * D.nvar;
  s += b * D.n_slack;
  grad += b * D.nvar;
  dir += b * D.dim;
  double r[1] = {0.0};
  const int op[1] = {0};
  BLOOP(i, D.ntot) {
    const double vi = v_at(D, M, x, s, i);
    double gphi = i < D.n_free ? grad[M.free_slot[i]] : 0.0;
    if (V.hl[i]) gphi -= mu / (vi - V.lb[i]);
    if (V.hu[i]) gphi += mu / (V.ub[i] - vi);
    r[0] += gphi * dir[i];
  }
  block_reduce<1>(r, op, out, os);
}

// solver.cpp:579-596
__global__ void dual_dir_k(BDims D, BMaps M, BBounds B, const double* __restrict__ x, const double* __restrict__ s,
                           const double* __restrict__ zl, const double* __restrict__ zu,
                           const double* __restrict__ step, const double* __restrict__ scal, double* __restrict__ dzl,
                           double* __restrict__ dzu, double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const BV V = bounds_of(D, B, b);
  const double mu = scal[blockIdx.y * 4], tau = scal[blockIdx.y * 4 + 1];
  x += b * D.nvar;
  s += b * D.n_slack;
  zl += b * D.ntot;
  zu += b * D.ntot;
  step += b * D.dim;
  dzl += b * D.ntot;
  dzu += b * D.ntot;
  double r[1] = {1.0};
  const int op[1] = {2};
  BLOOP(i, D.ntot) {
    const double dv = step[i];
    const double vi = v_at(D, M, x, s, i);
    double a = 0.0, c = 0.0;
    if (V.hl[i]) {
      const double d = vi - V.lb[i];
      a = mu / d - zl[i] - zl[i] / d * dv;
    }
    if (V.hu[i]) {
      const double d = V.ub[i] - vi;
      c = mu / d - zu[i] + zu[i] / d * dv;
    }
    dzl[i] = a;
    dzu[i] = c;
    if (a < 0.0 && zl[i] > 0.0) r[0] = fmin(r[0], -tau * zl[i] / a);
    if (c < 0.0 && zu[i] > 0.0) r[0] = fmin(r[0], -tau * zu[i] / c);
  }
  block_reduce<1>(r, op, out, os);
}

// solver.cpp:686-699 / ldl.cpp:257-268
__global__ void resid_k(BDims D, const double* __restrict__ bv, const double* __restrict__ kx,
                        const double* __restrict__ x, const double* __restrict__ dwdc, double* __restrict__ r,
                        double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  const double dw = dwdc[blockIdx.y * 4], dc = dwdc[blockIdx.y * 4 + 1];
  bv += b * D.dim;
  kx += b * D.dim;
  x += b * D.dim;
  if (r) r += b * D.dim;
  double v[3] = {0.0, 0.0, 0.0};
  const int op[3] = {1, 1, 1};
  BLOOP(i, D.dim) {
    const double delta = i < D.ntot ? dw : -dc;
    const double ri = bv[i] - kx[i] - delta * x[i];
    if (r) r[i] = ri;
    v[0] = fmax(v[0], fabs(ri));
    v[1] = fmax(v[1], fabs(bv[i]));
    v[2] = fmax(v[2], fabs(x[i]));
  }
  block_reduce<3>(v, op, out, os);
}

__global__ void theta_unscaled_k(BDims D, BMaps M, const double* __restrict__ g, const double* __restrict__ rs,
                                 double* __restrict__ out, int os, const int* __restrict__ ids) {
  const int64_t b = inst(ids);
  g += b * D.m;
  rs += b * D.m_con;
  double r[1] = {0.0};
  const int op[1] = {1};
  BLOOP(d, D.m) r[0] = fmax(r[0], fabs(g[d]) / rs[M.dual_row[d]]);
  block_reduce<1>(r, op, out, os);
}

__global__ void copy_dim_if_k(BDims D, double* __restrict__ dst, const double* __restrict__ src,
                              const double* __restrict__ flag, const int* __restrict__ ids) {
  if (flag[blockIdx.y] == 0.0) return;
  const int64_t b = inst(ids);
  ELOOP(i, D.dim) dst[b * D.dim + i] = src[b * D.dim + i];
}

__global__ void take_i64x3_k(const long long* __restrict__ src, double* __restrict__ out, int os, int nb,
                             const int* __restrict__ ids) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= nb) return;
  const int64_t b = ids[y];
  for (int k = 0; k < 3; ++k) out[static_cast<int64_t>(y) * os + k] = static_cast<double>(src[b * 3 + k]);
}

}  // namespace

// ---- host wrappers ------------------------------------------------------------------

void objective_chunks(const BDims& D, const double* objv, const int64_t* goff, const int64_t* gcount,
                      const int64_t* cbase, double* partials, const BL& L) {
  if (L.nb <= 0 || D.n_chunks <= 0) return;
  obj_chunks_k<<<dim3(static_cast<unsigned>((D.n_chunks + 7) / 8), L.nb), 256, 0, L.s>>>(D, objv, goff, gcount, cbase,
                                                                                         partials, L.ids);
}
void objective_combine(const BDims& D, const double* partials, const int64_t* cbase, const double* weights,
                       const double* obj_scale, double* f, int* flag, int os, const BL& L) {
  if (L.nb <= 0) return;
  obj_combine_k<<<grid1(L.nb), 32, 0, L.s>>>(D, partials, cbase, weights, obj_scale, f, flag, os, L.ids);
}
void gather_grad(const BDims& D, const double* gcoo, const int64_t* ptr, const int32_t* idx, double* out,
                 const BL& L) {
  if (L.nb <= 0 || D.nvar <= 0) return;
  gather_grad_k<<<grid2(D.nvar, L.nb), kT, 0, L.s>>>(D, gcoo, ptr, idx, out, L.ids);
}
void max_abs(const double* v, int64_t n, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  max_abs_k<<<grid1(L.nb), kT, 0, L.s>>>(v, n, out, os, L.ids);
}
void take_flags(int* flag, double* out, int stride, int slot, const BL& L) {
  if (L.nb <= 0) return;
  take_flags_k<<<(L.nb + 255) / 256, 256, 0, L.s>>>(flag, out, stride, slot, L.nb, L.ids);
}
void scaling(const BDims& D, const double* grad_dense, const double* jac, const int64_t* jrow_ptr,
             const int64_t* jrow_e, const int* flag, const double* weights, int enabled, double* obj_scale,
             double* row_scale, double* objw, const BL& L) {
  if (L.nb <= 0) return;
  scaling_k<<<grid1(L.nb), kT, 0, L.s>>>(D, grad_dense, jac, jrow_ptr, jrow_e, flag, weights, enabled, obj_scale,
                                         row_scale, objw, L.ids);
}

void copy_dim_if(const BDims& D, double* dst, const double* src, const double* flag, const BL& L) {
  if (L.nb <= 0) return;
  copy_dim_if_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, dst, src, flag, L.ids);
}
void take_i64x3(const long long* src, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  take_i64x3_k<<<(L.nb + 255) / 256, 256, 0, L.s>>>(src, out, os, L.nb, L.ids);
}

void kkt_assemble(const BDims& D, const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                  const int64_t* code, double* val, const BL& L) {
  if (L.nb <= 0 || D.knnz <= 0) return;
  kkt_assemble_k<<<grid2(D.knnz, L.nb), kT, 0, L.s>>>(D, hess, jac, sigma, ptr, code, val, L.ids);
}
void sym_matvec(const BDims& D, const double* val, const int64_t* rptr, const int64_t* col, const int64_t* vidx,
                const double* x, double* y, const BL& L) {
  if (L.nb <= 0 || D.dim <= 0) return;
  sym_matvec_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, val, rptr, col, vidx, x, y, L.ids);
}
void sym_norm_inf(const BDims& D, const double* val, const int64_t* rptr, const int64_t* vidx, double* out,
                  int os, const BL& L) {
  if (L.nb <= 0) return;
  sym_norm_inf_k<<<grid1(L.nb), kT, 0, L.s>>>(D, val, rptr, vidx, out, os, L.ids);
}
void jt_lambda(const BDims& D, const double* jac, const double* lam, const int64_t* ptr, const int64_t* e_idx,
               const int64_t* dual_idx, const int64_t* slack_dual, double* out, const BL& L) {
  if (L.nb <= 0 || D.ntot <= 0) return;
  jt_lambda_k<<<grid2(D.ntot, L.nb), kT, 0, L.s>>>(D, jac, lam, ptr, e_idx, dual_idx, slack_dual, out, L.ids);
}

void broadcast_rows(double* a, int64_t n, int nb, cudaStream_t s) {
  if (nb <= 1 || n <= 0) return;
  broadcast_rows_k<<<2 * 148 * 4, 256, 0, s>>>(a, n, nb);
}
void fold_bounds(const BDims& D, const int64_t* fptr, const int64_t* frow, const int64_t* prim_index, double* xlo,
                 double* xhi, const double* lcon, const double* ucon, int* contra, int* bad, const BL& L) {
  if (L.nb <= 0) return;
  fold_bounds_k<<<grid2(D.nvar, L.nb), kT, 0, L.s>>>(D, fptr, frow, prim_index, xlo, xhi, lcon, ucon, contra, bad,
                                                    L.ids);
}

void setup_bounds(const BDims& D, const BMaps& M, const double* xlo, const double* xhi, const double* lcon,
                  const double* ucon, const double* row_scale, double relax, double* lb, double* ub, int8_t* has_lb,
                  int8_t* has_ub, double* lcon_s, const BL& L) {
  if (L.nb <= 0) return;
  setup_bounds_k<<<grid2(D.ntot > D.m_con ? D.ntot : D.m_con, L.nb), kT, 0, L.s>>>(
      D, M, xlo, xhi, lcon, ucon, row_scale, relax, lb, ub, has_lb, has_ub, lcon_s, L.ids);
}
void init_x(const BDims& D, const BMaps& M, const BBounds& B, const double* x0, const double* xlo, const double* xhi,
            double* x, const BL& L) {
  if (L.nb <= 0) return;
  init_x_k<<<grid2(D.nvar, L.nb), kT, 0, L.s>>>(D, M, B, x0, xlo, xhi, x, L.ids);
}
void init_slacks_duals(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* c, double mu,
                       double* s, double* zl, double* zu, double* lambda, const BL& L) {
  if (L.nb <= 0) return;
  init_slacks_duals_k<<<grid2(D.ntot > D.m ? D.ntot : D.m, L.nb), kT, 0, L.s>>>(D, M, B, x, c, mu, s, zl, zu, lambda,
                                                                                L.ids);
}

void residual_theta(const BDims& D, const BMaps& M, const BBounds& B, const double* c, const double* s, double* g,
                    double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  residual_theta_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, c, s, g, out, os, L.ids);
}
void sigma(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* zl,
           const double* zu, double* out, const BL& L) {
  if (L.nb <= 0 || D.ntot <= 0) return;
  sigma_k<<<grid2(D.ntot, L.nb), kT, 0, L.s>>>(D, M, B, x, s, zl, zu, out, L.ids);
}
void rhs(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* grad,
         const double* jtlam, const double* g, const double* mu, double* out, const BL& L) {
  if (L.nb <= 0) return;
  rhs_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, M, B, x, s, grad, jtlam, g, mu, out, L.ids);
}
void trial(const BDims& D, const BMaps& M, const double* x, const double* s, const double* dir, const double* a,
           double* xt, double* st, const BL& L) {
  if (L.nb <= 0) return;
  trial_k<<<grid2(D.nvar, L.nb), kT, 0, L.s>>>(D, M, x, s, dir, a, xt, st, L.ids);
}
void expand_lambda(const BDims& D, const BMaps& M, const double* lambda, double* full, const BL& L) {
  if (L.nb <= 0 || D.m_con <= 0) return;
  expand_k<<<grid2(D.m_con, L.nb), kT, 0, L.s>>>(D, M, lambda, full, L.ids);
}
void axpy_m(const BDims& D, const double* a, const double* x, const double* yv, double* out, const BL& L) {
  if (L.nb <= 0 || D.m <= 0) return;
  axpy_m_k<<<grid2(D.m, L.nb), kT, 0, L.s>>>(D, a, x, yv, out, L.ids);
}
void rhs_soc(const BDims& D, const double* rhs, const double* gsoc, double* out, const BL& L) {
  if (L.nb <= 0) return;
  rhs_soc_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, rhs, gsoc, out, L.ids);
}
void add_dim(const BDims& D, double* x, const double* dx, const BL& L) {
  if (L.nb <= 0) return;
  add_dim_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, x, dx, L.ids);
}
void commit(const BDims& D, double* x, const double* xt, double* s, const double* st, double* c, const double* ct,
            double* grad, const double* gradt, double* step, const double* step2, const double* swap, const BL& L) {
  if (L.nb <= 0) return;
  commit_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, x, xt, s, st, c, ct, grad, gradt, step, step2, swap, L.ids);
}
void accept(const BDims& D, const BMaps& M, const BBounds& B, const double* step, const double* dzl,
            const double* dzu, const double* scal, const double* xn, const double* sn, double* lambda, double* zl,
            double* zu, const BL& L) {
  if (L.nb <= 0) return;
  accept_k<<<grid2(D.dim, L.nb), kT, 0, L.s>>>(D, M, B, step, dzl, dzu, scal, xn, sn, lambda, zl, zu, L.ids);
}

void barrier(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, double* out,
             int os, const BL& L) {
  if (L.nb <= 0) return;
  barrier_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, x, s, out, os, L.ids);
}
void kkt_error_parts(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                     const double* zl, const double* zu, const double* lambda, const double* grad,
                     const double* jtlam, const double* g, const double* mu, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  kkt_error_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, x, s, zl, zu, lambda, grad, jtlam, g, mu, out, os, L.ids);
}
void fraction_to_boundary(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                          const double* dir, const double* tau, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  ftb_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, x, s, dir, tau, out, os, L.ids);
}
void dphi(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* grad,
          const double* dir, const double* mu, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  dphi_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, x, s, grad, dir, mu, out, os, L.ids);
}
void dual_direction(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                    const double* zl, const double* zu, const double* step, const double* scal, double* dzl,
                    double* dzu, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  dual_dir_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, B, x, s, zl, zu, step, scal, dzl, dzu, out, os, L.ids);
}
void residual_norms(const BDims& D, const double* b, const double* kx, const double* x, const double* dwdc,
                    double* r, double* out, int os, const BL& L) {
  if (L.nb <= 0) return;
  resid_k<<<grid1(L.nb), kT, 0, L.s>>>(D, b, kx, x, dwdc, r, out, os, L.ids);
}
void theta_unscaled(const BDims& D, const BMaps& M, const double* g, const double* row_scale, double* out,
                    int os, const BL& L) {
  if (L.nb <= 0) return;
  theta_unscaled_k<<<grid1(L.nb), kT, 0, L.s>>>(D, M, g, row_scale, out, os, L.ids);
}

}  // namespace ocg::bdev
