// Interior-point vector kernels: the elementwise and
// reduction work of the reference's Solver::run (proj/src/ipm/solver.cpp),
// on device-resident iterates. Each kernel cites the reference lines whose
// arithmetic it performs; elementwise results are bit-identical to the
// reference's formulas, reductions are deterministic two-level trees (fixed
// block partition, fixed combine order) rather than the reference's
// left-to-right loops, so sums agree to rounding.
#include <cfloat>
#include <cstdint>

#include "ipm_kernels.hpp"

namespace ocg::ipmdev {

namespace {

constexpr int kBlock = 256;
constexpr int kMaxBlocks = 2 * 148;

__device__ __forceinline__ double v_at(const Iter& P, const double* x, const double* s, int64_t i) {
  return i < P.n_free ? x[P.free_slot[i]] : s[i - P.n_free];
}

// block-level reduction of NV values with per-slot op (0 sum, 1 max, 2 min)
template <int NV>
__device__ void block_reduce(double (&v)[NV], const int (&op)[NV], double* partials) {
  __shared__ double sh[NV][kBlock / 32];
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
      for (int w = 1; w < kBlock / 32; ++w)
        a = op[q] == 0 ? a + sh[q][w] : (op[q] == 1 ? fmax(a, sh[q][w]) : fmin(a, sh[q][w]));
      partials[static_cast<size_t>(blockIdx.x) * NV + q] = a;
    }
  }
}

// the block partials combined in block order by one thread (the fixed
// combine order); the block first stages them into shared memory so that the
// serial combine reads shared memory instead of waiting on one global load
// per partial (a one-thread loop over 296 x 5 global loads took 130 us)
template <int NV>
__global__ void __launch_bounds__(kBlock) finalize_k(const double* __restrict__ partials, int nblocks, Ops<NV> ops,
                                                    double* __restrict__ out) {
  __shared__ double sp[kMaxBlocks * NV];
  for (int i = threadIdx.x; i < nblocks * NV; i += blockDim.x) sp[i] = partials[i];
  __syncthreads();
  // thread q combines slot q (slots are independent), eight partials loaded
  // ahead of their in-order combine
  const int q = threadIdx.x;
  if (q >= NV) return;
  const int op = ops.op[q];
  double a = ops.init[q];
  int b = 0;
  for (; b + 8 <= nblocks; b += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = sp[(b + u) * NV + q];
#pragma unroll
    for (int u = 0; u < 8; ++u) a = op == 0 ? a + v[u] : (op == 1 ? fmax(a, v[u]) : fmin(a, v[u]));
  }
  for (; b < nblocks; ++b) {
    const double v = sp[b * NV + q];
    a = op == 0 ? a + v : (op == 1 ? fmax(a, v) : fmin(a, v));
  }
  out[q] = a;
}

int blocks_for(int64_t n) {
  const int64_t want = (n + kBlock - 1) / kBlock;
  return static_cast<int>(want < 1 ? 1 : (want > kMaxBlocks ? kMaxBlocks : want));
}

// unrolled by four so that the loads of later elements are issued before the
// earlier ones are consumed (each thread's elements stay in the same order:
// the reductions' roundings are unchanged)
#define GRID_LOOP(i, n)                                                                  \
  _Pragma("unroll 4")                                                                    \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

// ---- elementwise ----------------------------------------------------------

// solver.cpp:206-215 constraint_residual
__global__ void residual_k(Iter P, const double* __restrict__ c, const double* __restrict__ s, double* __restrict__ g) {
  GRID_LOOP(d, P.m) {
    const int64_t r = P.dual_row[d];
    const int64_t k = P.slack_index[r];
    g[d] = c[r] - (k >= 0 ? s[k] : P.lcon_s[r]);
  }
}

// solver.cpp:367-373 primal barrier diagonal
__global__ void sigma_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                        const double* __restrict__ zl, const double* __restrict__ zu, double* __restrict__ sigma) {
  GRID_LOOP(i, P.ntot) {
    const double v = v_at(P, x, s, i);
    double t = 0.0;
    if (P.has_lb[i]) t += zl[i] / (v - P.lb[i]);
    if (P.has_ub[i]) t += zu[i] / (P.ub[i] - v);
    sigma[i] = t;
  }
}

// solver.cpp:381-389 right-hand side
__global__ void rhs_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                      const double* __restrict__ grad, const double* __restrict__ jtlam, const double* __restrict__ g,
                      double mu, double* __restrict__ rhs) {
  GRID_LOOP(i, P.ntot + P.m) {
    if (i < P.ntot) {
      const double v = v_at(P, x, s, i);
      double rd = (i < P.n_free ? grad[P.free_slot[i]] : 0.0) + jtlam[i];
      if (P.has_lb[i]) rd -= mu / (v - P.lb[i]);
      if (P.has_ub[i]) rd += mu / (P.ub[i] - v);
      rhs[i] = -rd;
    } else {
      rhs[i] = -g[i - P.ntot];
    }
  }
}

// solver.cpp:434-441 build_trial: x_t = x + a*dir on free slots, s_t = s + a*dir
__global__ void trial_scatter_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                                const double* __restrict__ dir, double a, double* __restrict__ xt,
                                double* __restrict__ st) {
  GRID_LOOP(i, P.ntot) {
    if (i < P.n_free) {
      const int64_t slot = P.free_slot[i];
      xt[slot] = x[slot] + a * dir[i];
    } else {
      st[i - P.n_free] = s[i - P.n_free] + a * dir[i];
    }
  }
}

// the same with the step length read from device memory (graph-captured trials)
__global__ void trial_scatter_dev_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                                    const double* __restrict__ dir, const double* __restrict__ ap,
                                    double* __restrict__ xt, double* __restrict__ st) {
  const double a = *ap;
  GRID_LOOP(i, P.ntot) {
    if (i < P.n_free) {
      const int64_t slot = P.free_slot[i];
      xt[slot] = x[slot] + a * dir[i];
    } else {
      st[i - P.n_free] = s[i - P.n_free] + a * dir[i];
    }
  }
}

// solver.cpp:641-646 expand_lambda (zeros elsewhere)
__global__ void zero_k(double* __restrict__ v, int64_t n) {
  GRID_LOOP(i, n) v[i] = 0.0;
}
__global__ void expand_k(Iter P, const double* __restrict__ lambda, double* __restrict__ full) {
  GRID_LOOP(d, P.m) full[P.dual_row[d]] = lambda[d];
}

// solver.cpp:500-504 / :530-532 g_soc = a*g_soc + g_trial (first: a*g + g_trial)
__global__ void axpy_k(double a, const double* xv, const double* y, double* out,
                       int64_t n) {
  GRID_LOOP(i, n) out[i] = a * xv[i] + y[i];
}

// rhs_soc: copy rhs, replace the constraint block by -g_soc (solver.cpp:506-508)
__global__ void rhs_soc_k(Iter P, const double* __restrict__ rhs, const double* __restrict__ gsoc,
                          double* __restrict__ out) {
  GRID_LOOP(i, P.ntot + P.m) out[i] = i < P.ntot ? rhs[i] : -gsoc[i - P.ntot];
}

// solver.cpp:598-617 accept: lambda += a*step, z += a_z*dz, then safeguard
__global__ void accept_k(Iter P, const double* __restrict__ step, const double* __restrict__ dzl,
                         const double* __restrict__ dzu, double alpha, double alpha_z, double mu, double kappa,
                         const double* __restrict__ xn, const double* __restrict__ sn, double* __restrict__ lambda,
                         double* __restrict__ zl, double* __restrict__ zu) {
  GRID_LOOP(i, P.ntot + P.m) {
    if (i >= P.ntot) {
      lambda[i - P.ntot] += alpha * step[i];
      continue;
    }
    double l = zl[i] + alpha_z * dzl[i];
    double u = zu[i] + alpha_z * dzu[i];
    const double v = v_at(P, xn, sn, i);
    if (P.has_lb[i]) {
      const double d = v - P.lb[i];
      l = fmin(fmax(l, mu / (kappa * d)), kappa * mu / d);
    }
    if (P.has_ub[i]) {
      const double d = P.ub[i] - v;
      u = fmin(fmax(u, mu / (kappa * d)), kappa * mu / d);
    }
    zl[i] = l;
    zu[i] = u;
  }
}

// ---- reductions --------------------------------------------------------------

// solver.cpp:219-223 theta = sum |g|
__global__ void l1_k(const double* __restrict__ g, int64_t n, double* __restrict__ partials) {
  double v[1] = {0.0};
  const int op[1] = {0};
  GRID_LOOP(i, n) v[0] += fabs(g[i]);
  block_reduce<1>(v, op, partials);
}

// solver.cpp:225-242 barrier_terms: sum of logs; [1] counts d <= 0
__global__ void barrier_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                          double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  const int op[2] = {0, 0};
  GRID_LOOP(i, P.ntot) {
    const double vi = v_at(P, x, s, i);
    if (P.has_lb[i]) {
      const double d = vi - P.lb[i];
      if (d <= 0.0)
        v[1] += 1.0;
      else
        v[0] += log(d);
    }
    if (P.has_ub[i]) {
      const double d = P.ub[i] - vi;
      if (d <= 0.0)
        v[1] += 1.0;
      else
        v[0] += log(d);
    }
  }
  block_reduce<2>(v, op, partials);
}

// solver.cpp:260-287 kkt_error ingredients: [0] sum|zl|+|zu|, [1] sum|lambda|,
// [2] max|rd|, [3] max|g|, [4] max complementarity at mu
__global__ void kkt_error_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                            const double* __restrict__ zl, const double* __restrict__ zu,
                            const double* __restrict__ lambda, const double* __restrict__ grad,
                            const double* __restrict__ jtlam, const double* __restrict__ g, double mu,
                            double* __restrict__ partials) {
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int op[5] = {0, 0, 1, 1, 1};
  GRID_LOOP(i, P.ntot) {
    v[0] += fabs(zl[i]) + fabs(zu[i]);
    const double rd = (i < P.n_free ? grad[P.free_slot[i]] : 0.0) + jtlam[i] - zl[i] + zu[i];
    v[2] = fmax(v[2], fabs(rd));
    const double vi = v_at(P, x, s, i);
    if (P.has_lb[i]) v[4] = fmax(v[4], fabs((vi - P.lb[i]) * zl[i] - mu));
    if (P.has_ub[i]) v[4] = fmax(v[4], fabs((P.ub[i] - vi) * zu[i] - mu));
  }
  GRID_LOOP(d, P.m) {
    v[1] += fabs(lambda[d]);
    v[3] = fmax(v[3], fabs(g[d]));
  }
  block_reduce<5>(v, op, partials);
}

// solver.cpp:399-406 / :473-483 fraction to boundary (min, starting at 1)
__global__ void ftb_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                      const double* __restrict__ dir, double tau, double* __restrict__ partials) {
  double v[1] = {1.0};
  const int op[1] = {2};
  GRID_LOOP(i, P.ntot) {
    const double dv = dir[i];
    const double vi = v_at(P, x, s, i);
    if (P.has_lb[i] && dv < 0.0) v[0] = fmin(v[0], -tau * (vi - P.lb[i]) / dv);
    if (P.has_ub[i] && dv > 0.0) v[0] = fmin(v[0], tau * (P.ub[i] - vi) / dv);
  }
  block_reduce<1>(v, op, partials);
}

// solver.cpp:408-415 directional derivative of the barrier objective
__global__ void dphi_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                       const double* __restrict__ grad, const double* __restrict__ dir, double mu,
                       double* __restrict__ partials) {
  double v[1] = {0.0};
  const int op[1] = {0};
  GRID_LOOP(i, P.ntot) {
    const double vi = v_at(P, x, s, i);
    double gphi = i < P.n_free ? grad[P.free_slot[i]] : 0.0;
    if (P.has_lb[i]) gphi -= mu / (vi - P.lb[i]);
    if (P.has_ub[i]) gphi += mu / (P.ub[i] - vi);
    v[0] += gphi * dir[i];
  }
  block_reduce<1>(v, op, partials);
}

// solver.cpp:579-596 dual direction and its step (min, starting at 1)
__global__ void dual_dir_k(Iter P, const double* __restrict__ x, const double* __restrict__ s,
                           const double* __restrict__ zl, const double* __restrict__ zu,
                           const double* __restrict__ step, double mu, double tau, double* __restrict__ dzl,
                           double* __restrict__ dzu, double* __restrict__ partials) {
  double v[1] = {1.0};
  const int op[1] = {2};
  GRID_LOOP(i, P.ntot) {
    const double dv = step[i];
    const double vi = v_at(P, x, s, i);
    double a = 0.0, b = 0.0;
    if (P.has_lb[i]) {
      const double d = vi - P.lb[i];
      a = mu / d - zl[i] - zl[i] / d * dv;
    }
    if (P.has_ub[i]) {
      const double d = P.ub[i] - vi;
      b = mu / d - zu[i] + zu[i] / d * dv;
    }
    dzl[i] = a;
    dzu[i] = b;
    if (a < 0.0 && zl[i] > 0.0) v[0] = fmin(v[0], -tau * zl[i] / a);
    if (b < 0.0 && zu[i] > 0.0) v[0] = fmin(v[0], -tau * zu[i] / b);
  }
  block_reduce<1>(v, op, partials);
}

// solver.cpp:686-699 / ldl.cpp:257-268 residual of (K + deltas) x = b:
// r = b - Kx - delta x; [0] max|r|, [1] max|b|, [2] max|x|
__global__ void resid_k(const double* __restrict__ b, const double* __restrict__ kx, const double* __restrict__ x,
                        int64_t dim, int64_t ntot, double dw, double dc, double* __restrict__ r,
                        double* __restrict__ partials) {
  double v[3] = {0.0, 0.0, 0.0};
  const int op[3] = {1, 1, 1};
  GRID_LOOP(i, dim) {
    const double delta = i < ntot ? dw : -dc;
    const double ri = b[i] - kx[i] - delta * x[i];
    if (r) r[i] = ri;
    v[0] = fmax(v[0], fabs(ri));
    v[1] = fmax(v[1], fabs(b[i]));
    v[2] = fmax(v[2], fabs(x[i]));
  }
  block_reduce<3>(v, op, partials);
}

__global__ void add_k(double* __restrict__ x, const double* __restrict__ dx, int64_t n) {
  GRID_LOOP(i, n) x[i] += dx[i];
}

template <int NV>
void finish_reduce(Scratch& sc, int nb, const int (&op)[NV], const double (&init)[NV], double* host,
                   cudaStream_t s) {
  Ops<NV> ops;
  for (int q = 0; q < NV; ++q) {
    ops.op[q] = op[q];
    ops.init[q] = init[q];
  }
  finalize_k<NV><<<1, kBlock, 0, s>>>(sc.partials, nb, ops, sc.out);
  cudaMemcpyAsync(host, sc.out, NV * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
}

// the same reduction, its values left on the device (no host round trip)
template <int NV>
void finish_reduce_dev(Scratch& sc, int nb, const int (&op)[NV], const double (&init)[NV], double* out_dev,
                       cudaStream_t s) {
  Ops<NV> ops;
  for (int q = 0; q < NV; ++q) {
    ops.op[q] = op[q];
    ops.init[q] = init[q];
  }
  finalize_k<NV><<<1, kBlock, 0, s>>>(sc.partials, nb, ops, out_dev);
}

}  // namespace

void residual(const Iter& P, const double* c, const double* s, double* g, cudaStream_t st) {
  if (P.m > 0) residual_k<<<blocks_for(P.m), kBlock, 0, st>>>(P, c, s, g);
}
void sigma(const Iter& P, const double* x, const double* s, const double* zl, const double* zu, double* out,
           cudaStream_t st) {
  if (P.ntot > 0) sigma_k<<<blocks_for(P.ntot), kBlock, 0, st>>>(P, x, s, zl, zu, out);
}
void rhs(const Iter& P, const double* x, const double* s, const double* grad, const double* jtlam, const double* g,
         double mu, double* out, cudaStream_t st) {
  rhs_k<<<blocks_for(P.ntot + P.m), kBlock, 0, st>>>(P, x, s, grad, jtlam, g, mu, out);
}
void trial(const Iter& P, const double* x, const double* s, const double* dir, double a, double* xt, double* stv,
           cudaStream_t st) {
  cudaMemcpyAsync(xt, x, P.nvar * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (P.ntot > 0) trial_scatter_k<<<blocks_for(P.ntot), kBlock, 0, st>>>(P, x, s, dir, a, xt, stv);
}
void trial_dev(const Iter& P, const double* x, const double* s, const double* dir, const double* a_dev, double* xt,
               double* stv, cudaStream_t st) {
  cudaMemcpyAsync(xt, x, P.nvar * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (P.ntot > 0) trial_scatter_dev_k<<<blocks_for(P.ntot), kBlock, 0, st>>>(P, x, s, dir, a_dev, xt, stv);
}
void expand_lambda(const Iter& P, const double* lambda, double* full, cudaStream_t st) {
  zero_k<<<blocks_for(P.m_con), kBlock, 0, st>>>(full, P.m_con);
  if (P.m > 0) expand_k<<<blocks_for(P.m), kBlock, 0, st>>>(P, lambda, full);
}
void axpy(double a, const double* x, const double* y, double* out, int64_t n, cudaStream_t st) {
  if (n > 0) axpy_k<<<blocks_for(n), kBlock, 0, st>>>(a, x, y, out, n);
}
void rhs_soc(const Iter& P, const double* rhs, const double* gsoc, double* out, cudaStream_t st) {
  rhs_soc_k<<<blocks_for(P.ntot + P.m), kBlock, 0, st>>>(P, rhs, gsoc, out);
}
void accept(const Iter& P, const double* step, const double* dzl, const double* dzu, double alpha, double alpha_z,
            double mu, double kappa, const double* xn, const double* sn, double* lambda, double* zl, double* zu,
            cudaStream_t st) {
  accept_k<<<blocks_for(P.ntot + P.m), kBlock, 0, st>>>(P, step, dzl, dzu, alpha, alpha_z, mu, kappa, xn, sn, lambda,
                                                         zl, zu);
}
void add(double* x, const double* dx, int64_t n, cudaStream_t st) {
  if (n > 0) add_k<<<blocks_for(n), kBlock, 0, st>>>(x, dx, n);
}

double l1(const double* g, int64_t n, Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(n);
  l1_k<<<nb, kBlock, 0, st>>>(g, n, sc.partials);
  double h[1];
  finish_reduce<1>(sc, nb, {0}, {0.0}, h, st);
  return h[0];
}
void l1_async(const double* g, int64_t n, Scratch& sc, double* out_dev, cudaStream_t st) {
  const int nb = blocks_for(n);
  l1_k<<<nb, kBlock, 0, st>>>(g, n, sc.partials);
  finish_reduce_dev<1>(sc, nb, {0}, {0.0}, out_dev, st);
}
void barrier_async(const Iter& P, const double* x, const double* s, Scratch& sc, double* out2_dev, cudaStream_t st) {
  const int nb = blocks_for(P.ntot);
  barrier_k<<<nb, kBlock, 0, st>>>(P, x, s, sc.partials);
  finish_reduce_dev<2>(sc, nb, {0, 0}, {0.0, 0.0}, out2_dev, st);
}
bool barrier(const Iter& P, const double* x, const double* s, double& bar, Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(P.ntot);
  barrier_k<<<nb, kBlock, 0, st>>>(P, x, s, sc.partials);
  double h[2];
  finish_reduce<2>(sc, nb, {0, 0}, {0.0, 0.0}, h, st);
  bar = h[0];
  return h[1] == 0.0;
}
void kkt_error_parts(const Iter& P, const double* x, const double* s, const double* zl, const double* zu,
                     const double* lambda, const double* grad, const double* jtlam, const double* g, double mu,
                     double* out5, Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(P.ntot > P.m ? P.ntot : P.m);
  kkt_error_k<<<nb, kBlock, 0, st>>>(P, x, s, zl, zu, lambda, grad, jtlam, g, mu, sc.partials);
  finish_reduce<5>(sc, nb, {0, 0, 1, 1, 1}, {0.0, 0.0, 0.0, 0.0, 0.0}, out5, st);
}
double fraction_to_boundary(const Iter& P, const double* x, const double* s, const double* dir, double tau,
                            Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(P.ntot);
  ftb_k<<<nb, kBlock, 0, st>>>(P, x, s, dir, tau, sc.partials);
  double h[1];
  finish_reduce<1>(sc, nb, {2}, {1.0}, h, st);
  return h[0];
}
double dphi(const Iter& P, const double* x, const double* s, const double* grad, const double* dir, double mu,
            Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(P.ntot);
  dphi_k<<<nb, kBlock, 0, st>>>(P, x, s, grad, dir, mu, sc.partials);
  double h[1];
  finish_reduce<1>(sc, nb, {0}, {0.0}, h, st);
  return h[0];
}
double dual_direction(const Iter& P, const double* x, const double* s, const double* zl, const double* zu,
                      const double* step, double mu, double tau, double* dzl, double* dzu, Scratch& sc,
                      cudaStream_t st) {
  const int nb = blocks_for(P.ntot);
  dual_dir_k<<<nb, kBlock, 0, st>>>(P, x, s, zl, zu, step, mu, tau, dzl, dzu, sc.partials);
  double h[1];
  finish_reduce<1>(sc, nb, {2}, {1.0}, h, st);
  return h[0];
}
void residual_norms(const double* b, const double* kx, const double* x, int64_t dim, int64_t ntot, double dw,
                    double dc, double* r, double* out3, Scratch& sc, cudaStream_t st) {
  const int nb = blocks_for(dim);
  resid_k<<<nb, kBlock, 0, st>>>(b, kx, x, dim, ntot, dw, dc, r, sc.partials);
  finish_reduce<3>(sc, nb, {1, 1, 1}, {0.0, 0.0, 0.0}, out3, st);
}

int launches_per_reduction() { return 2; }

}  // namespace ocg::ipmdev
