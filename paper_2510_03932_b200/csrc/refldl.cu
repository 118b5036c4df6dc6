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
#include <cstdlib>
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

// ---- the chain: one warp, columns streamed through a ring of shared-memory
// slots by cp.async (LDGSTS) NS-1 columns ahead ----------------------------------

__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_n() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// wait until at most n groups are pending (n <= 14)
__device__ __forceinline__ void cp_wait(int n) {
  switch (n) {
    case 0: cp_wait_n<0>(); break;
    case 1: cp_wait_n<1>(); break;
    case 2: cp_wait_n<2>(); break;
    case 3: cp_wait_n<3>(); break;
    case 4: cp_wait_n<4>(); break;
    case 5: cp_wait_n<5>(); break;
    case 6: cp_wait_n<6>(); break;
    case 7: cp_wait_n<7>(); break;
    case 8: cp_wait_n<8>(); break;
    case 9: cp_wait_n<9>(); break;
    case 10: cp_wait_n<10>(); break;
    case 11: cp_wait_n<11>(); break;
    case 12: cp_wait_n<12>(); break;
    case 13: cp_wait_n<13>(); break;
    default: cp_wait_n<14>(); break;
  }
}

// Per chain column metadata (Dev::rec): streamed into a shared-memory ring of
// kMetaRing records two 32-column blocks ahead of the walk.
constexpr int kMetaRing = 128;

// copy the records of walk steps [blk*32, blk*32+32) (columns in walking
// direction) into the meta ring
__device__ __forceinline__ void issue_meta(const Dev& P, int dir, long long blk, ColRec* ring) {
  const long long k = blk * 32 + threadIdx.x;
  if (k < P.nnl) {
    const long long c = dir > 0 ? k : P.nnl - 1 - k;
    ColRec* dst = ring + (k & (kMetaRing - 1));
    const ColRec* src = P.rec + c;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst)) + 16u),
                 "l"(reinterpret_cast<const char*>(src) + 16)
                 : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst)) + 32u),
                 "l"(reinterpret_cast<const char*>(src) + 32)
                 : "memory");
  }
}
// meta blocks 0 and 1 before the walk starts
__device__ __forceinline__ void meta_prologue(const Dev& P, int dir, ColRec* ring) {
  issue_meta(P, dir, 0, ring);
  issue_meta(P, dir, 1, ring);
  cp_commit();
  cp_wait(0);
  __syncwarp();
}

__device__ __forceinline__ int tri32(int a) { return a * (a + 1) / 2; }
__device__ __forceinline__ int next_slot(int s, int ns) { return s + 1 == ns ? 0 : s + 1; }

// factor slot: [front: tri(f) packed lower + f diagonal maxima][rel: f-1 int32]
__device__ __forceinline__ void issue_factor_slot(const Dev& P, const double* W, const ColRec& m, double* slot) {
  const int f = m.f;
  const int nf = tri32(f) + f;
  const double* src = W + m.foff;
  for (int i = threadIdx.x; i < nf; i += 32) cp8(slot + i, src + i);
  int* rel = reinterpret_cast<int*>(slot + nf);
  for (int i = threadIdx.x; i < f - 1; i += 32) cp4(rel + i, P.rel + m.lp + i);
}

__global__ void __launch_bounds__(32) chain_factor_k(Dev P, int ns, int slotd, const double* __restrict__ W,
                                                     double* __restrict__ stash, double* __restrict__ D,
                                                     double* __restrict__ Dinv, double* __restrict__ Lx,
                                                     unsigned long long* __restrict__ inertia) {
  __shared__ unsigned char ta[kTab], tb[kTab];
  __shared__ __align__(16) ColRec ring[kMetaRing];
  extern __shared__ double slots[];
  build_tables(ta, tb);
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  const int L = ns - 1;  // slot lookahead
  meta_prologue(P, 1, ring);
  for (int q = 0; q < L; ++q) {
    if (q < n) issue_factor_slot(P, W, ring[q], slots + q * slotd);
    cp_commit();
  }
  // the lane's first update-matrix entry (a, b): fixed for the whole walk
  const int ua = ta[lane], ub = tb[lane];
  unsigned long long c[3] = {0, 0, 0};
  int sj = 0, sa = L % ns;  // slots of step j and of step j + L
  for (long long j = 0; j < n; ++j) {
    if ((j & 31) == 0) issue_meta(P, 1, (j >> 5) + 2, ring);
    if (j + L < n) issue_factor_slot(P, W, ring[(j + L) & (kMetaRing - 1)], slots + sa * slotd);
    cp_commit();
    cp_wait(L - 1);  // steps j and j+1 have landed
    __syncwarp();
    const ColRec m = ring[j & (kMetaRing - 1)];
    const int f = m.f;
    double* F = slots + sj * slotd;
    const int tf = tri32(f);
    double* ms = F + tf;
    const int* r = reinterpret_cast<const int*>(ms + f);
    // update matrices of children that were not the previous column (global stash)
    for (int q = m.sc0; q < m.sc1; ++q) {
      const ColRec mc = P.rec[P.sc_child[q]];
      const int32_t* rc = P.rel + mc.lp;
      const double* Us = stash + mc.soff;
      const int tu = (mc.f - 1) * mc.f / 2;
      for (int u = lane; u < tu; u += 32) {
        const int e = tri32(rc[ta[u] - 1]) + rc[tb[u] - 1];
        F[e] = __dadd_rn(F[e], Us[u]);
      }
      for (int a = lane; a < mc.f - 1; a += 32) ms[rc[a]] = fmax(ms[rc[a]], Us[tu + a]);
      __syncwarp();
    }
    const double d = F[0];
    const bool zero = zero_pivot(d, ms[0]);
    const double dinv = zero ? 0.0 : __drcp_rn(d);
    if (lane == 0) {
      D[m.pos] = d;
      Dinv[m.pos] = dinv;
      count_pivot(d, zero, c);
    }
    const int sn = next_slot(sj, ns);
    double* Fn = nullptr;
    double* msn = nullptr;
    double* Us = nullptr;
    if (m.soff == kChain) {
      Fn = slots + sn * slotd;
      msn = Fn + tri32(ring[(j + 1) & (kMetaRing - 1)].f);
    } else if (m.soff >= 0) {
      Us = stash + m.soff;
    }
    // L's column and the diagonal maxima of the update matrix: rows 1..f-1
    for (int a = lane + 1; a < f; a += 32) {
      const double Fa0 = F[tri32(a)];
      const double l = __dmul_rn(Fa0, dinv);
      Lx[m.lp + a - 1] = l;
      const double mx = fmax(ms[a], fabs(__dmul_rn(l, Fa0)));
      if (Fn)
        msn[r[a - 1]] = fmax(msn[r[a - 1]], mx);
      else if (Us)
        Us[tf - f + a - 1] = mx;  // after the (f-1)f/2 entries
    }
    if (Fn || Us) {
      const int tu = tf - f;  // (f-1) f / 2
      for (int u = lane; u < tu; u += 32) {
        const int a = u == lane ? ua : ta[u], b = u == lane ? ub : tb[u];
        const double Lb = __dmul_rn(F[tri32(b)], dinv);
        const double U = __dsub_rn(F[tri32(a) + b], __dmul_rn(Lb, F[tri32(a)]));
        if (Fn) {
          const int e = tri32(r[a - 1]) + r[b - 1];
          Fn[e] = __dadd_rn(Fn[e], U);
        } else {
          Us[u] = U;
        }
      }
    }
    __syncwarp();
    sj = sn;
    sa = next_slot(sa, ns);
  }
  cp_wait(0);
  if (lane == 0)
    for (int q = 0; q < 3; ++q)
      if (c[q]) atomicAdd(inertia + q, c[q]);
}

// ---- small fronts (f <= FM, FM <= 16): fixed slot layout, every lane owns
// fixed update-matrix entries and rows; no loops over the front ------------------

template <int FM>
struct Small {
  static constexpr int TF = FM * (FM + 1) / 2;     // packed front
  static constexpr int TU = (FM - 1) * FM / 2;     // packed update matrix
  static constexpr int UPL = (TU + 31) / 32;       // update entries per lane
  static constexpr int FSLOT = TF + FM + FM / 2 + 1;  // [front TF][maxima FM][rel FM-1 ints]
  static constexpr int VSLOT = 3 * FM + 2;            // solves
};
constexpr int kSmallSlots = 8;

template <int FM>
__global__ void __launch_bounds__(32) chain_factor_small_k(Dev P, const double* __restrict__ W,
                                                           double* __restrict__ stash, double* __restrict__ D,
                                                           double* __restrict__ Dinv, double* __restrict__ Lx,
                                                           unsigned long long* __restrict__ inertia) {
  using S = Small<FM>;
  constexpr int NS = kSmallSlots, L = NS - 1;
  __shared__ unsigned char ta[kTab], tb[kTab];
  __shared__ __align__(16) ColRec ring[kMetaRing];
  __shared__ __align__(16) double slots[NS * S::FSLOT];
  build_tables(ta, tb);
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  meta_prologue(P, 1, ring);
  auto issue = [&](const ColRec& m, double* slot) {
    const int tf = tri32(m.f);
    const double* src = W + m.foff;
#pragma unroll
    for (int k = 0; k < (S::TF + FM + 31) / 32; ++k) {
      const int i = lane + 32 * k;
      if (i < tf)
        cp8(slot + i, src + i);
      else if (i < tf + m.f)
        cp8(slot + S::TF + (i - tf), src + i);
    }
    if (lane < m.f - 1) cp4(reinterpret_cast<int*>(slot + S::TF + FM) + lane, P.rel + m.lp + lane);
  };
  for (int q = 0; q < L; ++q) {
    if (q < n) issue(ring[q], slots + q * S::FSLOT);
    cp_commit();
  }
  int ua[S::UPL], ub[S::UPL];
#pragma unroll
  for (int k = 0; k < S::UPL; ++k) {
    const int u = lane + 32 * k;
    ua[k] = u < S::TU ? ta[u] : 0;
    ub[k] = u < S::TU ? tb[u] : 0;
  }
  unsigned long long c[3] = {0, 0, 0};
  int sj = 0, sa = L;
  for (long long j = 0; j < n; ++j) {
    if ((j & 31) == 0) issue_meta(P, 1, (j >> 5) + 2, ring);
    if (j + L < n) issue(ring[(j + L) & (kMetaRing - 1)], slots + sa * S::FSLOT);
    cp_commit();
    cp_wait_n<L - 1>();
    __syncwarp();
    const ColRec m = ring[j & (kMetaRing - 1)];
    const int f = m.f;
    double* F = slots + sj * S::FSLOT;
    double* ms = F + S::TF;
    const int* r = reinterpret_cast<const int*>(F + S::TF + FM);
    for (int q = m.sc0; q < m.sc1; ++q) {  // stashed children (rare)
      const ColRec mc = P.rec[P.sc_child[q]];
      const int32_t* rc = P.rel + mc.lp;
      const double* Us = stash + mc.soff;
      const int tu = (mc.f - 1) * mc.f / 2;
      for (int u = lane; u < tu; u += 32) {
        const int e = tri32(rc[ta[u] - 1]) + rc[tb[u] - 1];
        F[e] = __dadd_rn(F[e], Us[u]);
      }
      for (int a = lane; a < mc.f - 1; a += 32) ms[rc[a]] = fmax(ms[rc[a]], Us[tu + a]);
      __syncwarp();
    }
    const double d = F[0];
    const bool zero = zero_pivot(d, ms[0]);
    const double dinv = zero ? 0.0 : __drcp_rn(d);
    if (lane == 0) {
      D[m.pos] = d;
      Dinv[m.pos] = dinv;
      count_pivot(d, zero, c);
    }
    const int sn = sj + 1 == NS ? 0 : sj + 1;
    double* Fn = m.soff == kChain ? slots + sn * S::FSLOT : nullptr;
    double* Us = m.soff >= 0 ? stash + m.soff : nullptr;
    const int tu = (f - 1) * f / 2;
    if (lane >= 1 && lane < f) {  // row `lane`: L's entry and the diagonal maximum
      const double Fa0 = F[tri32(lane)];
      const double l = __dmul_rn(Fa0, dinv);
      Lx[m.lp + lane - 1] = l;
      const double mx = fmax(ms[lane], fabs(__dmul_rn(l, Fa0)));
      if (Fn)
        Fn[S::TF + r[lane - 1]] = fmax(Fn[S::TF + r[lane - 1]], mx);
      else if (Us)
        Us[tu + lane - 1] = mx;
    }
#pragma unroll
    for (int k = 0; k < S::UPL; ++k) {
      const int u = lane + 32 * k;
      if (u < tu && (Fn || Us)) {
        const int a = ua[k], b = ub[k];
        const double U = __dsub_rn(F[tri32(a) + b], __dmul_rn(__dmul_rn(F[tri32(b)], dinv), F[tri32(a)]));
        if (Fn) {
          const int e = tri32(r[a - 1]) + r[b - 1];
          Fn[e] = __dadd_rn(Fn[e], U);
        } else {
          Us[u] = U;
        }
      }
    }
    __syncwarp();
    sj = sn;
    sa = sa + 1 == NS ? 0 : sa + 1;
  }
  cp_wait_n<0>();
  if (lane == 0)
    for (int q = 0; q < 3; ++q)
      if (c[q]) atomicAdd(inertia + q, c[q]);
}

// Fronts of at most 8 rows, register-resident: lane u owns update-matrix
// entry (a, b), u = tri(a-1) + b-1 (28 lanes), and holds F(a,b), F(a,0),
// F(b,0), the pivot F(0,0) and the diagonal maxima in registers. Along the
// chain (the next column is the parent and has no stashed children) the
// update matrix moves to the next front's owners by shuffles (ColRec::inv8),
// added to the pre-assembled values prefetched into the ring; the pivot's
// dependency chain per column is then shuffle -> add -> reciprocal -> three
// products. Other transitions go through the shared-memory front as in
// chain_factor_small_k.
__global__ void __launch_bounds__(32) chain_factor_reg_k(Dev P, const double* __restrict__ W,
                                                        double* __restrict__ stash, double* __restrict__ D,
                                                        double* __restrict__ Dinv, double* __restrict__ Lx,
                                                        unsigned long long* __restrict__ inertia) {
  constexpr int FM = 8;
  using S = Small<FM>;
  constexpr int NS = kSmallSlots, L = NS - 1;
  __shared__ unsigned char ta[kTab], tb[kTab];
  __shared__ __align__(16) ColRec ring[kMetaRing];
  __shared__ __align__(16) double slots[NS * S::FSLOT];
  build_tables(ta, tb);
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  meta_prologue(P, 1, ring);
  auto issue = [&](const ColRec& m, double* slot) {
    const int tf = tri32(m.f);
    const double* src = W + m.foff;
#pragma unroll
    for (int k = 0; k < (S::TF + FM + 31) / 32; ++k) {
      const int i = lane + 32 * k;
      if (i < tf)
        cp8(slot + i, src + i);
      else if (i < tf + m.f)
        cp8(slot + S::TF + (i - tf), src + i);
    }
    if (lane < m.f - 1) cp4(reinterpret_cast<int*>(slot + S::TF + FM) + lane, P.rel + m.lp + lane);
  };
  for (int q = 0; q < L; ++q) {
    if (q < n) issue(ring[q], slots + q * S::FSLOT);
    cp_commit();
  }
  // this lane's entry (la, lb); lanes 28..31 own none (la = 0)
  int la = 0, lb = 0;
#pragma unroll
  for (int a = 1; a < FM; ++a)
    if (lane >= tri32(a - 1) && lane < tri32(a)) {
      la = a;
      lb = lane - tri32(a - 1) + 1;
    }
  const bool diag = la > 0 && la == lb;
  double X = 0.0, Y = 0.0, Z = 0.0, Pv = 0.0, M0 = 0.0, Ma = 0.0;
  bool need_load = true;
  unsigned long long c[3] = {0, 0, 0};
  int sj = 0, sa = L;
  for (long long j = 0; j < n; ++j) {
    if ((j & 31) == 0) issue_meta(P, 1, (j >> 5) + 2, ring);
    if (j + L < n) issue(ring[(j + L) & (kMetaRing - 1)], slots + sa * S::FSLOT);
    cp_commit();
    cp_wait_n<L - 1>();
    __syncwarp();
    const ColRec m = ring[j & (kMetaRing - 1)];
    const int f = m.f;
    double* F = slots + sj * S::FSLOT;
    const int* r = reinterpret_cast<const int*>(F + S::TF + FM);
    if (need_load) {
      double* ms = F + S::TF;
      for (int q = m.sc0; q < m.sc1; ++q) {  // stashed children (rare)
        const ColRec mc = P.rec[P.sc_child[q]];
        const int32_t* rc = P.rel + mc.lp;
        const double* Us = stash + mc.soff;
        const int tu = (mc.f - 1) * mc.f / 2;
        for (int u = lane; u < tu; u += 32) {
          const int e = tri32(rc[ta[u] - 1]) + rc[tb[u] - 1];
          F[e] = __dadd_rn(F[e], Us[u]);
        }
        for (int a = lane; a < mc.f - 1; a += 32) ms[rc[a]] = fmax(ms[rc[a]], Us[tu + a]);
        __syncwarp();
      }
      X = F[tri32(la) + lb];
      Y = F[tri32(la)];
      Z = F[tri32(lb)];
      Pv = F[0];
      M0 = ms[0];
      Ma = ms[la];
    }
    const bool zero = zero_pivot(Pv, M0);
    const double dinv = zero ? 0.0 : __drcp_rn(Pv);
    if (lane == 0) {
      D[m.pos] = Pv;
      Dinv[m.pos] = dinv;
      count_pivot(Pv, zero, c);
    }
    const bool act = la > 0 && la < f;
    const double Lv = __dmul_rn(Y, dinv);  // L(la) on lanes with lb == 1
    if (act && lb == 1) Lx[m.lp + la - 1] = Lv;
    const double U = __dsub_rn(X, __dmul_rn(__dmul_rn(Z, dinv), Y));
    const double MU = diag ? fmax(Ma, fabs(__dmul_rn(Lv, Y))) : 0.0;
    const int sn = sj + 1 == NS ? 0 : sj + 1;
    need_load = true;
    if (m.soff != kRoot) {
      const ColRec mn = ring[(j + 1) & (kMetaRing - 1)];
      if (m.soff == kChain && mn.sc0 == mn.sc1 && m.inv8 != 0) {
        // register path: this lane's entry of the next front = pre-assembled + U of the row pair mapping here
        const double* Fn = slots + sn * S::FSLOT;
        const int ia = static_cast<int>((m.inv8 >> (8 * la)) & 0xff);
        const int ib = static_cast<int>((m.inv8 >> (8 * lb)) & 0xff);
        const int sx = ia && ib ? tri32(ia - 1) + ib - 1 : 0;
        const int sy = ia ? tri32(ia - 1) : 0;
        const int sz = ib ? tri32(ib - 1) : 0;
        const int sm = ia ? tri32(ia - 1) + ia - 1 : 0;
        const double vx = __shfl_sync(0xffffffffu, U, sx);
        const double vy = __shfl_sync(0xffffffffu, U, sy);
        const double vz = __shfl_sync(0xffffffffu, U, sz);
        const double vp = __shfl_sync(0xffffffffu, U, 0);
        const double m0 = __shfl_sync(0xffffffffu, MU, 0);
        const double ma = __shfl_sync(0xffffffffu, MU, sm);
        X = ia && ib ? __dadd_rn(Fn[tri32(la) + lb], vx) : Fn[tri32(la) + lb];
        Y = ia ? __dadd_rn(Fn[tri32(la)], vy) : Fn[tri32(la)];
        Z = ib ? __dadd_rn(Fn[tri32(lb)], vz) : Fn[tri32(lb)];
        Pv = __dadd_rn(Fn[0], vp);
        M0 = fmax(Fn[S::TF], m0);
        Ma = ia ? fmax(Fn[S::TF + la], ma) : Fn[S::TF + la];
        need_load = false;
      } else if (m.soff == kChain) {
        double* Fn = slots + sn * S::FSLOT;
        if (act) {
          const int e = tri32(r[la - 1]) + r[lb - 1];
          Fn[e] = __dadd_rn(Fn[e], U);
          if (diag) Fn[S::TF + r[la - 1]] = fmax(Fn[S::TF + r[la - 1]], MU);
        }
      } else {
        double* Us = stash + m.soff;
        const int tu = (f - 1) * f / 2;
        if (act) {
          Us[lane] = U;
          if (diag) Us[tu + la - 1] = MU;
        }
      }
    }
    __syncwarp();
    sj = sn;
    sa = sa + 1 == NS ? 0 : sa + 1;
  }
  cp_wait_n<0>();
  if (lane == 0)
    for (int q = 0; q < 3; ++q)
      if (c[q]) atomicAdd(inertia + q, c[q]);
}

template <int FM>
__global__ void __launch_bounds__(32) fwd_chain_small_k(Dev P, const double* __restrict__ Lx, double* __restrict__ y,
                                                        double* __restrict__ Vs) {
  using S = Small<FM>;
  constexpr int NS = kSmallSlots, L = NS - 1;
  __shared__ __align__(16) ColRec ring[kMetaRing];
  __shared__ __align__(16) double slots[NS * S::VSLOT];  // [v FM][Lx FM][rel FM ints]
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  meta_prologue(P, 1, ring);
  auto issue = [&](const ColRec& m, double* slot) {
    if (lane == 0) cp8(slot, y + m.pos);
    if (lane >= 1 && lane < FM) slot[lane] = 0.0;
    if (lane < m.f - 1) {
      cp8(slot + FM + lane, Lx + m.lp + lane);
      cp4(reinterpret_cast<int*>(slot + 2 * FM) + lane, P.rel + m.lp + lane);
    }
  };
  for (int q = 0; q < L; ++q) {
    if (q < n) issue(ring[q], slots + q * S::VSLOT);
    cp_commit();
  }
  int sj = 0, sa = L;
  for (long long j = 0; j < n; ++j) {
    if ((j & 31) == 0) issue_meta(P, 1, (j >> 5) + 2, ring);
    if (j + L < n) issue(ring[(j + L) & (kMetaRing - 1)], slots + sa * S::VSLOT);
    cp_commit();
    cp_wait_n<L - 1>();
    __syncwarp();
    const ColRec m = ring[j & (kMetaRing - 1)];
    double* v = slots + sj * S::VSLOT;
    const int* r = reinterpret_cast<const int*>(v + 2 * FM);
    for (int q = m.sc0; q < m.sc1; ++q) {
      const ColRec mc = P.rec[P.sc_child[q]];
      const int32_t* rc = P.rel + mc.lp;
      const double* us = Vs + mc.soff;
      for (int a = lane; a < mc.f - 1; a += 32) v[rc[a]] = __dadd_rn(v[rc[a]], us[a]);
      __syncwarp();
    }
    const double yk = v[0];
    if (lane == 0) y[m.pos] = yk;
    const int sn = sj + 1 == NS ? 0 : sj + 1;
    if (lane >= 1 && lane < m.f && m.soff != kRoot) {
      const double u = __dsub_rn(v[lane], __dmul_rn(v[FM + lane - 1], yk));
      if (m.soff == kChain) {
        double* vn = slots + sn * S::VSLOT;
        vn[r[lane - 1]] = __dadd_rn(vn[r[lane - 1]], u);
      } else {
        Vs[m.soff + lane - 1] = u;
      }
    }
    __syncwarp();
    sj = sn;
    sa = sa + 1 == NS ? 0 : sa + 1;
  }
  cp_wait_n<0>();
}

template <int FM>
__global__ void __launch_bounds__(32) bwd_chain_small_k(Dev P, const double* __restrict__ Lx,
                                                        const double* __restrict__ Dinv, const double* __restrict__ y,
                                                        double* __restrict__ xp) {
  using S = Small<FM>;
  constexpr int NS = kSmallSlots, L = NS - 2;
  __shared__ __align__(16) ColRec ring[kMetaRing];
  __shared__ __align__(16) double slots[NS * S::VSLOT];  // [X FM][Lx FM][y, Dinv][rel FM ints]
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  meta_prologue(P, -1, ring);
  auto issue = [&](const ColRec& m, double* slot) {
    if (lane < m.f - 1) {
      cp8(slot + FM + lane, Lx + m.lp + lane);
      cp4(reinterpret_cast<int*>(slot + 2 * FM + 2) + lane, P.rel + m.lp + lane);
    }
    if (lane == 30) cp8(slot + 2 * FM, y + m.pos);
    if (lane == 31) cp8(slot + 2 * FM + 1, Dinv + m.pos);
  };
  for (int q = 0; q < L; ++q) {
    if (q < n) issue(ring[q], slots + q * S::VSLOT);
    cp_commit();
  }
  int sk = 0, sp = NS - 1, sa = L;
  for (long long k = 0; k < n; ++k) {
    if ((k & 31) == 0) issue_meta(P, -1, (k >> 5) + 2, ring);
    if (k + L < n) issue(ring[(k + L) & (kMetaRing - 1)], slots + sa * S::VSLOT);
    cp_commit();
    cp_wait_n<L>();
    __syncwarp();
    const ColRec m = ring[k & (kMetaRing - 1)];
    const int f = m.f;
    double* X = slots + sk * S::VSLOT;
    const int* r = reinterpret_cast<const int*>(X + 2 * FM + 2);
    const bool chain = m.soff == kChain;
    const double* Xn = slots + sp * S::VSLOT;
    // X[a] = x of row a; the terms L(a) * X[a] summed in row order by lane 0
    double xa = 0.0;
    if (lane >= 1 && lane < f) {
      xa = chain ? Xn[r[lane - 1]] : xp[P.Li[m.lp + lane - 1]];
      X[lane] = xa;
    }
    const double term = lane >= 1 && lane < f ? __dmul_rn(X[FM + lane - 1], xa) : 0.0;
    double s = __dmul_rn(X[2 * FM], X[2 * FM + 1]);
#pragma unroll
    for (int a = 1; a < FM; ++a) {
      const double t = __shfl_sync(0xffffffffu, term, a);
      if (a < f) s = __dsub_rn(s, t);
    }
    if (lane == 0) {
      X[0] = s;
      xp[m.pos] = s;
    }
    __syncwarp();
    sp = sk;
    sk = sk + 1 == NS ? 0 : sk + 1;
    sa = sa + 1 == NS ? 0 : sa + 1;
  }
  cp_wait_n<0>();
}

// ---- streamed walks (fronts <= 8 rows) ------------------------------------------
// The chain's per-column data are contiguous in walk order (column records,
// pre-assembled fronts, L entries + Dinv, right-hand sides), so they stream
// into shared memory in chunks of kChunk columns by 1D bulk copies (TMA,
// cp.async.bulk) completing on an mbarrier: one wait per chunk instead of
// per-column asynchronous copies, and the per-column loop only reads shared
// memory and shuffles registers.

constexpr int kChunk = 16, kStages = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct FStage {
  ColRec rec[kChunk];
  double fr[kChunk * 44];  // fronts of <= 8 rows: 36 + 8 doubles each
};

// chain factorization, fronts <= 8 rows, register-resident (see
// chain_factor_reg_k) with the chunked bulk-copy stream. chunk_foff[c] = the
// W offset of chunk c's first front (c = 0..nchunks, the last = fronts_len).
// Chunks whose every column hands its update matrix to the next column by
// shuffles (ColRec::flags bit 0) run a branch-free loop; L's chain columns
// go to the walk-order records (P.sr), Lx is filled from them on demand
// (fill_lx).
__global__ void __launch_bounds__(32) chain_factor_stream_k(Dev P, const long long* __restrict__ chunk_foff,
                                                           const double* __restrict__ W, double* __restrict__ stash,
                                                           double* __restrict__ D, double* __restrict__ Dinv,
                                                           unsigned long long* __restrict__ inertia) {
  constexpr int FM = 8;
  __shared__ __align__(16) FStage stg[kStages];
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ unsigned char ta[kTab], tb[kTab];
  build_tables(ta, tb);
  const int lane = threadIdx.x;
  const long long n = P.nnl, nch = (n + kChunk - 1) / kChunk;
  if (lane == 0) {
    for (int q = 0; q < kStages; ++q) mbar_init(&bar[q]);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](long long c, long long fa, long long fb) {  // lane 0
    if (c >= nch) return;
    const int st = static_cast<int>(c % kStages);
    const long long j0 = c * kChunk;
    const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), n - j0));
    const unsigned rb = static_cast<unsigned>(cnt * sizeof(ColRec)), fbytes = static_cast<unsigned>((fb - fa) * 8);
    mbar_expect(&bar[st], rb + fbytes);
    bulk_load(stg[st].rec, P.rec + j0, rb, &bar[st]);
    if (fbytes) bulk_load(stg[st].fr, W + fa, fbytes, &bar[st]);
  };
  if (lane == 0)
    for (long long c = 0; c < kStages - 1 && c < nch; ++c) issue(c, chunk_foff[c], chunk_foff[c + 1]);
  // bounds of the chunk issued next, loaded one chunk ahead of their use
  long long pf0 = 0, pf1 = 0;
  if (kStages - 1 < nch) {
    pf0 = chunk_foff[kStages - 1];
    pf1 = chunk_foff[kStages];
  }
  int la = 0, lb = 0;
#pragma unroll
  for (int a = 1; a < FM; ++a)
    if (lane >= tri32(a - 1) && lane < tri32(a)) {
      la = a;
      lb = lane - tri32(a - 1) + 1;
    }
  const bool diag = la > 0 && la == lb;
  double X = 0.0, Y = 0.0, Z = 0.0, Pv = 0.0, M0 = 0.0, Ma = 0.0;
  bool need_load = true;
  unsigned long long np = 0, nn = 0, nz = 0;
  for (long long c = 0; c < nch; ++c) {
    if (lane == 0 && c + kStages - 1 < nch) issue(c + kStages - 1, pf0, pf1);
    if (c + kStages < nch) {
      pf0 = __ldg(chunk_foff + c + kStages);
      pf1 = __ldg(chunk_foff + c + kStages + 1);
    }
    const int st = static_cast<int>(c % kStages);
    mbar_wait(&bar[st], static_cast<unsigned>((c / kStages) & 1));
    const bool more = c + 1 < nch;
    const int st1 = static_cast<int>((c + 1) % kStages);
    if (more) mbar_wait(&bar[st1], static_cast<unsigned>(((c + 1) / kStages) & 1));
    const long long j0 = c * kChunk;
    const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), n - j0));
    const long long fa = stg[st].rec[0].foff, fa1 = more ? stg[st1].rec[0].foff : 0;
    const bool fast = !need_load && more && __all_sync(0xffffffffu, lane >= cnt || (stg[st].rec[lane & (kChunk - 1)].flags & 1));
    if (fast) {
      // every column: pivot, L, update matrix, shuffled into the next front's owners
#pragma unroll 2
      for (int jj = 0; jj < cnt; ++jj) {
        const long long j = j0 + jj;
        const ColRec m = stg[st].rec[jj];
        const bool zero = zero_pivot(Pv, M0);
        const double dinv = zero ? 0.0 : __drcp_rn(Pv);
        const double Lv = __dmul_rn(Y, dinv);
        const double U = __dsub_rn(X, __dmul_rn(__dmul_rn(Z, dinv), Y));
        const double MU = diag ? fmax(Ma, fabs(__dmul_rn(Lv, Y))) : 0.0;
        if (lane == 0) {
          D[m.pos] = Pv;
          Dinv[m.pos] = dinv;
          P.sr[j * 8 + 7] = dinv;
          np += !zero && Pv > 0;
          nn += !zero && !(Pv > 0);
          nz += zero;
        }
        if (la > 0 && la < m.f && lb == 1) P.sr[j * 8 + la - 1] = Lv;
        const bool same = jj + 1 < cnt;
        const ColRec& mn = same ? stg[st].rec[jj + 1] : stg[st1].rec[0];
        const double* Fn = same ? stg[st].fr + (mn.foff - fa) : stg[st1].fr + (mn.foff - fa1);
        const int fnn = mn.f;
        const int ia = static_cast<int>((m.inv8 >> (8 * la)) & 0xff);
        const int ib = static_cast<int>((m.inv8 >> (8 * lb)) & 0xff);
        const double vx = __shfl_sync(0xffffffffu, U, ia && ib ? tri32(ia - 1) + ib - 1 : 0);
        const double vy = __shfl_sync(0xffffffffu, U, ia ? tri32(ia - 1) : 0);
        const double vz = __shfl_sync(0xffffffffu, U, ib ? tri32(ib - 1) : 0);
        const double vp = __shfl_sync(0xffffffffu, U, 0);
        const double m0 = __shfl_sync(0xffffffffu, MU, 0);
        const double ma = __shfl_sync(0xffffffffu, MU, ia ? tri32(ia - 1) + ia - 1 : 0);
        const bool in = la < fnn;
        const double* msn = Fn + tri32(fnn);
        const double px = in ? Fn[tri32(la) + lb] : 0.0, py = in ? Fn[tri32(la)] : 0.0;
        const double pz = in ? Fn[tri32(lb)] : 0.0, pm = in ? msn[la] : 0.0;
        X = ia && ib ? __dadd_rn(px, vx) : px;
        Y = ia ? __dadd_rn(py, vy) : py;
        Z = ib ? __dadd_rn(pz, vz) : pz;
        Pv = __dadd_rn(Fn[0], vp);
        M0 = fmax(msn[0], m0);
        Ma = ia ? fmax(pm, ma) : pm;
      }
      __syncwarp();
      continue;
    }
    for (int jj = 0; jj < cnt; ++jj) {
      const long long j = j0 + jj;
      const ColRec m = stg[st].rec[jj];
      const int f = m.f;
      double* F = stg[st].fr + (m.foff - fa);
      double* ms = F + tri32(f);
      if (need_load) {
        for (int q = m.sc0; q < m.sc1; ++q) {  // stashed children (rare)
          const ColRec mc = P.rec[P.sc_child[q]];
          const int32_t* rc = P.rel + mc.lp;
          const double* Us = stash + mc.soff;
          const int tu = (mc.f - 1) * mc.f / 2;
          for (int u = lane; u < tu; u += 32) {
            const int e = tri32(rc[ta[u] - 1]) + rc[tb[u] - 1];
            F[e] = __dadd_rn(F[e], Us[u]);
          }
          for (int a = lane; a < mc.f - 1; a += 32) ms[rc[a]] = fmax(ms[rc[a]], Us[tu + a]);
          __syncwarp();
        }
        const bool in = la < f;
        X = in ? F[tri32(la) + lb] : 0.0;
        Y = in ? F[tri32(la)] : 0.0;
        Z = in ? F[tri32(lb)] : 0.0;
        Pv = F[0];
        M0 = ms[0];
        Ma = in ? ms[la] : 0.0;
      }
      const bool zero = zero_pivot(Pv, M0);
      const double dinv = zero ? 0.0 : __drcp_rn(Pv);
      const bool act = la > 0 && la < f;
      const double Lv = __dmul_rn(Y, dinv);
      const double U = __dsub_rn(X, __dmul_rn(__dmul_rn(Z, dinv), Y));
      const double MU = diag ? fmax(Ma, fabs(__dmul_rn(Lv, Y))) : 0.0;
      if (lane == 0) {
        D[m.pos] = Pv;
        Dinv[m.pos] = dinv;
        P.sr[j * 8 + 7] = dinv;
        np += !zero && Pv > 0;
        nn += !zero && !(Pv > 0);
        nz += zero;
      }
      if (act && lb == 1) P.sr[j * 8 + la - 1] = Lv;
      need_load = true;
      if (m.soff != kRoot && j + 1 < n) {
        const bool same = jj + 1 < cnt;
        const ColRec& mn = same ? stg[st].rec[jj + 1] : stg[st1].rec[0];
        double* Fn = same ? stg[st].fr + (mn.foff - fa) : stg[st1].fr + (mn.foff - fa1);
        const int fnn = mn.f;
        if (m.flags & 1) {
          const int ia = static_cast<int>((m.inv8 >> (8 * la)) & 0xff);
          const int ib = static_cast<int>((m.inv8 >> (8 * lb)) & 0xff);
          const double vx = __shfl_sync(0xffffffffu, U, ia && ib ? tri32(ia - 1) + ib - 1 : 0);
          const double vy = __shfl_sync(0xffffffffu, U, ia ? tri32(ia - 1) : 0);
          const double vz = __shfl_sync(0xffffffffu, U, ib ? tri32(ib - 1) : 0);
          const double vp = __shfl_sync(0xffffffffu, U, 0);
          const double m0 = __shfl_sync(0xffffffffu, MU, 0);
          const double ma = __shfl_sync(0xffffffffu, MU, ia ? tri32(ia - 1) + ia - 1 : 0);
          const bool in = la < fnn;
          const double* msn = Fn + tri32(fnn);
          const double px = in ? Fn[tri32(la) + lb] : 0.0, py = in ? Fn[tri32(la)] : 0.0;
          const double pz = in ? Fn[tri32(lb)] : 0.0, pm = in ? msn[la] : 0.0;
          X = ia && ib ? __dadd_rn(px, vx) : px;
          Y = ia ? __dadd_rn(py, vy) : py;
          Z = ib ? __dadd_rn(pz, vz) : pz;
          Pv = __dadd_rn(Fn[0], vp);
          M0 = fmax(msn[0], m0);
          Ma = ia ? fmax(pm, ma) : pm;
          need_load = false;
        } else if (m.soff == kChain) {
          if (act) {
            const int ra = static_cast<int>((m.rel8 >> (8 * (la - 1))) & 0xff);
            const int rb = static_cast<int>((m.rel8 >> (8 * (lb - 1))) & 0xff);
            const int e = tri32(ra) + rb;
            Fn[e] = __dadd_rn(Fn[e], U);
            if (diag) Fn[tri32(fnn) + ra] = fmax(Fn[tri32(fnn) + ra], MU);
          }
        } else if (m.soff >= 0) {
          double* Us = stash + m.soff;
          const int tu = (f - 1) * f / 2;
          if (act) {
            Us[lane] = U;
            if (diag) Us[tu + la - 1] = MU;
          }
        }
      }
      __syncwarp();
    }
  }
  if (lane == 0) {
    if (np) atomicAdd(inertia + 0, np);
    if (nn) atomicAdd(inertia + 1, nn);
    if (nz) atomicAdd(inertia + 2, nz);
  }
}

// Lx of the chain columns from the walk-order records (the streamed
// factorization writes only those): one thread per chain column
__global__ void fill_lx_k(Dev P, double* __restrict__ Lx) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P.nnl;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = P.nl_f[j];
    const int64_t lp = P.nl_lp[j];
    for (int a = 1; a < f; ++a) Lx[lp + a - 1] = P.sr[j * 8 + a - 1];
  }
}

// chain rows of the right-hand side minus their leaf terms, in walk order
__global__ void fwd_pre_k(Dev P, const double* __restrict__ Lx, const double* __restrict__ y) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P.nnl;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (P.fl_all_ptr[j + 1] - P.fl_all_ptr[j] > kPreLong) continue;  // fwd_pre_long_k
    double s = y[P.nl_pos[j]];
    for (int64_t t = P.fl_all_ptr[j]; t < P.fl_all_ptr[j + 1]; ++t)
      s = __dsub_rn(s, __dmul_rn(Lx[P.fl_lx[t]], y[P.fl_col[t]]));
    P.ypre[j] = s;
  }
}

struct VStage {
  ColRec rec[kChunk];
  double sr[kChunk * 8];
  double y[kChunk + 2];
};

// chunk c into stage (seq % kStages): seq is the chunk's place in the walk
// (c for the forward walk, nch-1-c for the backward one), which also sets
// the mbarrier phase of its wait, (seq / kStages) & 1
__device__ __forceinline__ void issue_vstage(const Dev& P, const double* yv, long long c, long long seq, long long nch,
                                             VStage* stg, uint64_t* bar) {
  if (c < 0 || c >= nch) return;
  const long long n = P.nnl;
  const int st = static_cast<int>(seq % kStages);
  const long long j0 = c * kChunk;
  const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), n - j0));
  const unsigned rb = static_cast<unsigned>(cnt * sizeof(ColRec)), sb = static_cast<unsigned>(cnt * 64),
                 yb = static_cast<unsigned>(((cnt + 1) & ~1) * 8);
  mbar_expect(&bar[st], rb + sb + yb);
  bulk_load(stg[st].rec, P.rec + j0, rb, &bar[st]);
  bulk_load(stg[st].sr, P.sr + j0 * 8, sb, &bar[st]);
  bulk_load(stg[st].y, yv + j0, yb, &bar[st]);
}

// forward substitution along the chain: lane a holds v(a) of the current
// front (v(0): the pivot row); v'(a') = pre + u(inv(a')) by shuffles
// one block per long chain column: the products L * y (each exact on its
// own) are staged into shared memory by threads 32.., double-buffered, while
// thread 0 subtracts the previous stage from the right-hand side in term
// order — the same sequence of roundings as fwd_pre_k's one thread
__global__ void __launch_bounds__(256) fwd_pre_long_k(Dev P, const double* __restrict__ Lx, const double* __restrict__ y) {
  constexpr int kStage = 2048;
  __shared__ double sb[2][kStage];
  const int64_t j = P.pre_long[blockIdx.x];
  const int64_t lo = P.fl_all_ptr[j], n = P.fl_all_ptr[j + 1] - lo;
  const int tid = threadIdx.x, nl = static_cast<int>(blockDim.x) - 32;
  auto stage = [&](int64_t k, double* dst) {
    const int64_t b = k * kStage, e = min(n, b + kStage);
    for (int64_t t = b + (tid - 32); t < e; t += nl) dst[t - b] = __dmul_rn(Lx[P.fl_lx[lo + t]], y[P.fl_col[lo + t]]);
  };
  double s = tid == 0 ? y[P.nl_pos[j]] : 0.0;
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
      for (; i + 8 <= m; i += 8) {  // eight loads in flight, then the ordered subtractions
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = c[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) s = __dsub_rn(s, v[q]);
      }
      for (; i < m; ++i) s = __dsub_rn(s, c[i]);
    }
    __syncthreads();
  }
  if (tid == 0) P.ypre[j] = s;
}

__global__ void __launch_bounds__(32) fwd_chain_stream_k(Dev P, double* __restrict__ Vs) {
  __shared__ __align__(16) VStage stg[kStages];
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ double vbuf[32];
  const int lane = threadIdx.x;
  const long long n = P.nnl, nch = (n + kChunk - 1) / kChunk;
  if (lane == 0) {
    for (int q = 0; q < kStages; ++q) mbar_init(&bar[q]);
    mbar_fence_init();
    for (long long c = 0; c < kStages - 1; ++c) issue_vstage(P, P.ypre, c, c, nch, stg, bar);
  }
  __syncwarp();
  double v = 0.0;
  bool need_load = true;
  for (long long c = 0; c < nch; ++c) {
    if (lane == 0) issue_vstage(P, P.ypre, c + kStages - 1, c + kStages - 1, nch, stg, bar);
    const int st = static_cast<int>(c % kStages);
    mbar_wait(&bar[st], static_cast<unsigned>((c / kStages) & 1));
    const bool more = c + 1 < nch;
    const int st1 = static_cast<int>((c + 1) % kStages);
    if (more) mbar_wait(&bar[st1], static_cast<unsigned>(((c + 1) / kStages) & 1));
    const long long j0 = c * kChunk;
    const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), n - j0));
    if (!need_load && more && __all_sync(0xffffffffu, lane >= cnt || (stg[st].rec[lane & (kChunk - 1)].flags & 1))) {
      // every column hands its update vector to the next one by a shuffle
#pragma unroll 2
      for (int jj = 0; jj < cnt; ++jj) {
        const ColRec m = stg[st].rec[jj];
        const double yk = __shfl_sync(0xffffffffu, v, 0);
        if (lane == 0) P.ych[j0 + jj] = yk;
        const double u = lane >= 1 && lane < m.f ? __dsub_rn(v, __dmul_rn(stg[st].sr[jj * 8 + lane - 1], yk)) : 0.0;
        const double pre = jj + 1 < cnt ? stg[st].y[jj + 1] : stg[st1].y[0];
        const int src = lane < 8 ? static_cast<int>((m.inv8 >> (8 * lane)) & 0xff) : 0;
        const double w = __shfl_sync(0xffffffffu, u, src);
        v = lane == 0 ? __dadd_rn(pre, w) : (src ? w : 0.0);
      }
      continue;
    }
    for (int jj = 0; jj < cnt; ++jj) {
      const long long j = j0 + jj;
      const ColRec m = stg[st].rec[jj];
      if (need_load) v = lane == 0 ? stg[st].y[jj] : 0.0;
      if (m.sc0 < m.sc1) {  // stashed children (rare): through shared memory
        vbuf[lane] = v;
        __syncwarp();
        for (int q = m.sc0; q < m.sc1; ++q) {
          const ColRec mc = P.rec[P.sc_child[q]];
          const int32_t* rc = P.rel + mc.lp;
          const double* us = Vs + mc.soff;
          for (int a = lane; a < mc.f - 1; a += 32) vbuf[rc[a]] = __dadd_rn(vbuf[rc[a]], us[a]);
          __syncwarp();
        }
        v = vbuf[lane];
        __syncwarp();
      }
      const double yk = __shfl_sync(0xffffffffu, v, 0);
      if (lane == 0) P.ych[j] = yk;
      const int f = m.f;
      const double u = lane >= 1 && lane < f ? __dsub_rn(v, __dmul_rn(stg[st].sr[jj * 8 + lane - 1], yk)) : 0.0;
      need_load = true;
      if (m.soff == kChain && m.inv8 != 0 && j + 1 < n) {
        const bool same = jj + 1 < cnt;
        const double pre = same ? stg[st].y[jj + 1] : stg[st1].y[0];
        const int src = lane < 8 ? static_cast<int>((m.inv8 >> (8 * lane)) & 0xff) : 0;
        const double w = __shfl_sync(0xffffffffu, u, src);
        v = lane == 0 ? __dadd_rn(pre, w) : (src ? w : 0.0);
        need_load = false;
      } else if (m.soff >= 0 && lane >= 1 && lane < f) {
        Vs[m.soff + lane - 1] = u;
      }
    }
  }
}

// backward substitution along the chain, last column first: lane a holds
// X(a), the solution at row a of the current front (X(0) its pivot row),
// gathered from the parent's front by shuffles (rel8)
__global__ void __launch_bounds__(32) bwd_chain_stream_k(Dev P, double* __restrict__ xp) {
  __shared__ __align__(16) VStage stg[kStages];
  __shared__ __align__(8) uint64_t bar[kStages];
  const int lane = threadIdx.x;
  const long long n = P.nnl, nch = (n + kChunk - 1) / kChunk;
  if (lane == 0) {
    for (int q = 0; q < kStages; ++q) mbar_init(&bar[q]);
    mbar_fence_init();
    for (long long k = 0; k < kStages - 1; ++k) issue_vstage(P, P.ych, nch - 1 - k, k, nch, stg, bar);
  }
  __syncwarp();
  double Xp = 0.0;  // X of the previous (higher) column
  for (long long k = 0; k < nch; ++k) {
    const long long c = nch - 1 - k;
    if (lane == 0) issue_vstage(P, P.ych, c - (kStages - 1), k + kStages - 1, nch, stg, bar);
    const int st = static_cast<int>(k % kStages);
    mbar_wait(&bar[st], static_cast<unsigned>((k / kStages) & 1));
    const long long j0 = c * kChunk;
    const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), n - j0));
    if (__all_sync(0xffffffffu, lane >= cnt || stg[st].rec[lane & (kChunk - 1)].soff == kChain)) {
      // every column's parent is the column walked just before: X by shuffles
#pragma unroll 2
      for (int jj = cnt - 1; jj >= 0; --jj) {
        const ColRec m = stg[st].rec[jj];
        const bool row = lane >= 1 && lane < m.f;
        const int ra = row ? static_cast<int>((m.rel8 >> (8 * (lane - 1))) & 0xff) : 0;
        const double xa = __shfl_sync(0xffffffffu, Xp, ra);
        // every lane gathers the front's X values by broadcast shuffles and
        // subtracts the terms in entry order: ldl.cpp:240-243's roundings
        double xs[7];
#pragma unroll
        for (int a = 1; a < 8; ++a) xs[a - 1] = __shfl_sync(0xffffffffu, Xp, static_cast<int>((m.rel8 >> (8 * (a - 1))) & 0xff));
        double s = __dmul_rn(stg[st].y[jj], stg[st].sr[jj * 8 + 7]);
#pragma unroll
        for (int a = 1; a < 8; ++a)
          if (a < m.f) s = __dsub_rn(s, __dmul_rn(stg[st].sr[jj * 8 + a - 1], xs[a - 1]));
        Xp = lane == 0 ? s : xa;
        if (lane == 0) xp[m.pos] = s;
      }
      continue;
    }
    for (int jj = cnt - 1; jj >= 0; --jj) {
      const ColRec m = stg[st].rec[jj];
      const int f = m.f;
      const int ra = lane >= 1 && lane < f ? static_cast<int>((m.rel8 >> (8 * (lane - 1))) & 0xff) : 0;
      double xa = __shfl_sync(0xffffffffu, Xp, ra);
      if (m.soff != kChain && lane >= 1 && lane < f) xa = xp[P.Li[m.lp + lane - 1]];  // parent not the previous column
      // X of row a on every lane (lane a's value broadcast), the terms
      // subtracted in entry order (ldl.cpp:240-243)
      double s = __dmul_rn(stg[st].y[jj], stg[st].sr[jj * 8 + 7]);
#pragma unroll
      for (int a = 1; a < 8; ++a) {
        const double x_a = __shfl_sync(0xffffffffu, xa, a);
        if (a < f) s = __dsub_rn(s, __dmul_rn(stg[st].sr[jj * 8 + a - 1], x_a));
      }
      Xp = lane == 0 ? s : xa;
      if (lane == 0) xp[m.pos] = s;
      __syncwarp();
    }
  }
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

// forward slot: [v: f][Lx: f-1][rel: f-1 int32]; v = [y_pos, 0, ...]
__device__ __forceinline__ void issue_fwd_slot(const Dev& P, const double* Lx, const double* y, const ColRec& m,
                                               double* slot) {
  const int f = m.f;
  if (threadIdx.x == 0) cp8(slot, y + m.pos);
  for (int i = 1 + threadIdx.x; i < f; i += 32) slot[i] = 0.0;
  for (int i = threadIdx.x; i < f - 1; i += 32) cp8(slot + f + i, Lx + m.lp + i);
  int* rel = reinterpret_cast<int*>(slot + 2 * f - 1);
  for (int i = threadIdx.x; i < f - 1; i += 32) cp4(rel + i, P.rel + m.lp + i);
}

__global__ void __launch_bounds__(32) fwd_chain_k(Dev P, int ns, int slotd, const double* __restrict__ Lx,
                                                  double* __restrict__ y, double* __restrict__ Vs) {
  __shared__ __align__(16) ColRec ring[kMetaRing];
  extern __shared__ double slots[];
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  const int L = ns - 1;
  meta_prologue(P, 1, ring);
  for (int q = 0; q < L; ++q) {
    if (q < n) issue_fwd_slot(P, Lx, y, ring[q], slots + q * slotd);
    cp_commit();
  }
  int sj = 0, sa = L % ns;
  for (long long j = 0; j < n; ++j) {
    if ((j & 31) == 0) issue_meta(P, 1, (j >> 5) + 2, ring);
    if (j + L < n) issue_fwd_slot(P, Lx, y, ring[(j + L) & (kMetaRing - 1)], slots + sa * slotd);
    cp_commit();
    cp_wait(L - 1);
    __syncwarp();
    const ColRec m = ring[j & (kMetaRing - 1)];
    const int f = m.f;
    double* v = slots + sj * slotd;
    const double* lx = v + f;
    const int* r = reinterpret_cast<const int*>(v + 2 * f - 1);
    for (int q = m.sc0; q < m.sc1; ++q) {
      const ColRec mc = P.rec[P.sc_child[q]];
      const int32_t* rc = P.rel + mc.lp;
      const double* us = Vs + mc.soff;
      for (int a = lane; a < mc.f - 1; a += 32) v[rc[a]] = __dadd_rn(v[rc[a]], us[a]);
      __syncwarp();
    }
    const double yk = v[0];
    if (lane == 0) y[m.pos] = yk;
    const int sn = next_slot(sj, ns);
    if (m.soff != kRoot) {
      double* vn = m.soff == kChain ? slots + sn * slotd : nullptr;
      for (int a = lane + 1; a < f; a += 32) {
        const double u = __dsub_rn(v[a], __dmul_rn(lx[a - 1], yk));
        if (vn)
          vn[r[a - 1]] = __dadd_rn(vn[r[a - 1]], u);
        else
          Vs[m.soff + a - 1] = u;
      }
    }
    __syncwarp();
    sj = sn;
    sa = next_slot(sa, ns);
  }
  cp_wait(0);
}

// backward slot: [X: f][Lx: f-1][y_pos, Dinv_pos][rel: f-1 int32]; X = [x_pos, x of the rows]
__device__ __forceinline__ void issue_bwd_slot(const Dev& P, const double* Lx, const double* Dinv, const double* y,
                                               const ColRec& m, double* slot) {
  const int f = m.f;
  for (int i = threadIdx.x; i < f - 1; i += 32) cp8(slot + f + i, Lx + m.lp + i);
  if (threadIdx.x == 0) cp8(slot + 2 * f - 1, y + m.pos);
  if (threadIdx.x == 1) cp8(slot + 2 * f, Dinv + m.pos);
  int* rel = reinterpret_cast<int*>(slot + 2 * f + 1);
  for (int i = threadIdx.x; i < f - 1; i += 32) cp4(rel + i, P.rel + m.lp + i);
}

__global__ void __launch_bounds__(32) bwd_chain_k(Dev P, int ns, int slotd, const double* __restrict__ Lx,
                                                  const double* __restrict__ Dinv, const double* __restrict__ y,
                                                  double* __restrict__ xp) {
  __shared__ __align__(16) ColRec ring[kMetaRing];
  extern __shared__ double slots[];
  const int lane = threadIdx.x;
  const long long n = P.nnl;
  // step k walks column n-1-k; it reads step k-1's slot, so the prefetch runs
  // L = ns-2 steps ahead and never lands in either
  const int L = ns - 2;
  meta_prologue(P, -1, ring);
  for (int q = 0; q < L; ++q) {
    if (q < n) issue_bwd_slot(P, Lx, Dinv, y, ring[q], slots + q * slotd);
    cp_commit();
  }
  int sk = 0, sp = ns - 1, sa = L % ns;  // slots of steps k, k-1, k+L
  for (long long k = 0; k < n; ++k) {
    if ((k & 31) == 0) issue_meta(P, -1, (k >> 5) + 2, ring);
    if (k + L < n) issue_bwd_slot(P, Lx, Dinv, y, ring[(k + L) & (kMetaRing - 1)], slots + sa * slotd);
    cp_commit();
    cp_wait(L);
    __syncwarp();
    const ColRec m = ring[k & (kMetaRing - 1)];
    const int f = m.f;
    double* X = slots + sk * slotd;
    const double* lx = X + f;
    const int* r = reinterpret_cast<const int*>(X + 2 * f + 1);
    const bool chain = m.soff == kChain;
    const double* Xn = slots + sp * slotd;  // column j+1, the previous step
    for (int a = lane + 1; a < f; a += 32) X[a] = chain ? Xn[r[a - 1]] : xp[P.Li[m.lp + a - 1]];
    if (lane == 0) {
      double s = __dmul_rn(X[2 * f - 1], X[2 * f]);
      for (int a = 1; a < f; ++a) s = __dsub_rn(s, __dmul_rn(lx[a - 1], chain ? Xn[r[a - 1]] : xp[P.Li[m.lp + a - 1]]));
      X[0] = s;
      xp[m.pos] = s;
    }
    __syncwarp();
    sp = sk;
    sk = next_slot(sk, ns);
    sa = next_slot(sa, ns);
  }
  cp_wait(0);
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

// Sequential solve, ldl.cpp:222-247 operation for operation: one block, the
// permuted right-hand side resident in shared memory; L's columns come in
// chunks (kSeqCols columns, kSeqEnt entries) that warps 1.. stage into a
// double buffer while thread 0 runs the previous chunk's columns:
//   forward, columns ascending: y[Li[p]] -= Lx[p] * y[k] (skipped when y[k]
//   is 0), each column's rows loaded together and stored together (the rows
//   of one column are distinct);
//   y[k] *= Dinv[k];
//   backward, columns descending: s = y[k]; s -= Lx[p] * y[Li[p]] in entry
//   order; y[k] = s.
// The same roundings in the same order as the reference, given L and D.
// The chain columns' L entries live in P.sr after a streamed factorization;
// they are written into Lx first (fill_lx_k's mapping).
struct SeqBuf {
  double* x;
  int32_t* i;
  int32_t* p;
};

__device__ __forceinline__ SeqBuf seq_buf(double* base, int64_t dim, int b) {
  double* x0 = base + ((dim + 1) & ~int64_t{1});
  char* q = reinterpret_cast<char*>(x0 + 2 * kSeqEnt);
  SeqBuf r;
  r.x = x0 + b * kSeqEnt;
  r.i = reinterpret_cast<int32_t*>(q) + b * kSeqEnt;
  r.p = reinterpret_cast<int32_t*>(q) + 2 * kSeqEnt + b * (kSeqCols + 1);
  return r;
}

__device__ __forceinline__ void seq_stage(const Dev& P, const double* Lx, int64_t c, SeqBuf B, int t0, int nt) {
  const int k0 = P.sq_col[c], k1 = P.sq_col[c + 1];
  const int e0 = P.Lp32[k0], ne = P.Lp32[k1] - e0;
  for (int t = t0; t <= k1 - k0; t += nt) B.p[t] = P.Lp32[k0 + t] - e0;
  for (int t = t0; t < ne; t += nt) {
    B.i[t] = P.Li32[e0 + t];
    B.x[t] = __ldcg(Lx + e0 + t);
  }
}

__global__ void __launch_bounds__(256) seq_solve_k(Dev P, const double* __restrict__ Dinv, double* Lx, bool fill,
                                                   const double* __restrict__ rhs, double* __restrict__ x) {
  extern __shared__ __align__(16) double ys[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t n = P.dim, nc = P.sq_nchunks;
  if (fill)
    for (int64_t j = tid; j < P.nnl; j += nt) {
      const int f = P.nl_f[j];
      const int64_t lp = P.nl_lp[j];
      for (int a = 1; a < f; ++a) Lx[lp + a - 1] = P.sr[j * 8 + a - 1];
    }
  for (int64_t k = tid; k < n; k += nt) ys[k] = rhs[P.perm[k]];
  __syncthreads();
  // L y = P b
  seq_stage(P, Lx, 0, seq_buf(ys, n, 0), tid, nt);
  __syncthreads();
  for (int64_t c = 0; c < nc; ++c) {
    const SeqBuf B = seq_buf(ys, n, static_cast<int>(c & 1));
    if (tid >= 32 && c + 1 < nc) seq_stage(P, Lx, c + 1, seq_buf(ys, n, static_cast<int>((c + 1) & 1)), tid - 32, nt - 32);
    if (tid == 0) {
      const int k0 = P.sq_col[c], nk = P.sq_col[c + 1] - k0;
      for (int kk = 0; kk < nk; ++kk) {
        const double yk = ys[k0 + kk];
        if (yk == 0.0) continue;
        const int pe = B.p[kk + 1];
        for (int p = B.p[kk]; p < pe; p += 8) {
          int r[8];
          double l[8], v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < pe) {
              r[u] = B.i[p + u];
              l[u] = B.x[p + u];
              v[u] = ys[r[u]];
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < pe) ys[r[u]] = __dsub_rn(v[u], __dmul_rn(l[u], yk));
        }
      }
    }
    __syncthreads();
  }
  for (int64_t k = tid; k < n; k += nt) ys[k] = __dmul_rn(ys[k], Dinv[k]);
  // L^T x = y, last chunk first
  seq_stage(P, Lx, nc - 1, seq_buf(ys, n, 0), tid, nt);
  __syncthreads();
  for (int64_t q = 0; q < nc; ++q) {
    const int64_t c = nc - 1 - q;
    const SeqBuf B = seq_buf(ys, n, static_cast<int>(q & 1));
    if (tid >= 32 && c > 0) seq_stage(P, Lx, c - 1, seq_buf(ys, n, static_cast<int>((q + 1) & 1)), tid - 32, nt - 32);
    if (tid == 0) {
      const int k0 = P.sq_col[c], nk = P.sq_col[c + 1] - k0;
      for (int kk = nk - 1; kk >= 0; --kk) {
        double s = ys[k0 + kk];
        const int pe = B.p[kk + 1];
        for (int p = B.p[kk]; p < pe; p += 8) {
          double l[8], v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < pe) {
              l[u] = B.x[p + u];
              v[u] = ys[B.i[p + u]];
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < pe) s = __dsub_rn(s, __dmul_rn(l[u], v[u]));
        }
        ys[k0 + kk] = s;
      }
    }
    __syncthreads();
  }
  for (int64_t k = tid; k < n; k += nt) x[P.perm[k]] = ys[k];
}

// ring depth: up to 16 slots, within 160 KB of dynamic shared memory
int ring_slots(int slotd) {
  const int by_smem = static_cast<int>((160 * 1024) / (static_cast<size_t>(slotd) * sizeof(double)));
  return std::max(2, std::min(15, by_smem));
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
  static const int variant = std::getenv("OCG_REFLDL_KERNEL") ? std::atoi(std::getenv("OCG_REFLDL_KERNEL")) : 0;
  if (P.nnl && P.fmax <= 8 && variant == 0 && P.chunk_foff) {
    chain_factor_stream_k<<<1, 32, 0, s>>>(P, P.chunk_foff, W, stash, D, Dinv, inertia);
  } else if (P.nnl && P.fmax <= 8 && variant == 1) {
    chain_factor_reg_k<<<1, 32, 0, s>>>(P, W, stash, D, Dinv, Lx, inertia);
  } else if (P.nnl && P.fmax <= 8) {
    chain_factor_small_k<8><<<1, 32, 0, s>>>(P, W, stash, D, Dinv, Lx, inertia);
  } else if (P.nnl && P.fmax <= 16) {
    chain_factor_small_k<16><<<1, 32, 0, s>>>(P, W, stash, D, Dinv, Lx, inertia);
  } else if (P.nnl) {
    const int slotd = static_cast<int>(P.fmax * (P.fmax + 1) / 2 + P.fmax + P.fmax / 2 + 1);
    const int ns = ring_slots(slotd);
    ck(cudaFuncSetAttribute(chain_factor_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024), "smem attr");
    chain_factor_k<<<1, 32, static_cast<size_t>(ns) * slotd * sizeof(double), s>>>(P, ns, slotd, W, stash, D, Dinv,
                                                                                   Lx, inertia);
  }
  ck(cudaGetLastError(), "factor launch");
}

bool streamed_factor(const Dev& P) {
  static const int variant = std::getenv("OCG_REFLDL_KERNEL") ? std::atoi(std::getenv("OCG_REFLDL_KERNEL")) : 0;
  return P.nnl && P.fmax <= 8 && variant == 0 && P.chunk_foff;
}

void fill_lx(const Dev& P, double* Lx, cudaStream_t s) {
  if (streamed_factor(P)) fill_lx_k<<<grid_for(P.nnl), kThreads, 0, s>>>(P, Lx);
}

std::vector<int32_t> seq_chunks(const std::vector<int64_t>& Lp) {
  const int64_t n = static_cast<int64_t>(Lp.size()) - 1;
  std::vector<int32_t> col{0};
  if (n <= 0 || seq_smem_bytes(n) > kSeqSmemMax || Lp[static_cast<size_t>(n)] >= (int64_t{1} << 31)) return {};
  int64_t k0 = 0;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t cnt = Lp[static_cast<size_t>(k) + 1] - Lp[static_cast<size_t>(k)];
    if (cnt > kSeqEnt) return {};
    if (k - k0 + 1 > kSeqCols || Lp[static_cast<size_t>(k) + 1] - Lp[static_cast<size_t>(k0)] > kSeqEnt) {
      col.push_back(static_cast<int32_t>(k));
      k0 = k;
    }
  }
  col.push_back(static_cast<int32_t>(n));
  return col;
}

size_t seq_smem_bytes(int64_t dim) {
  return static_cast<size_t>((dim + 1) & ~int64_t{1}) * sizeof(double) +
         2 * (kSeqEnt * (sizeof(double) + sizeof(int32_t)) + (kSeqCols + 1) * sizeof(int32_t));
}

// Opt-in (OCG_REFLDL_SOLVE=1, read per call): bit-exact with ldl.cpp's solve
// given L and D, but one thread's walk is latency-bound on its shared-memory
// round trips: Goddard N=1000 (dim 7001) 2.59 ms per solve against 1.19 ms
// for the warp-chain walks, Goddard@1000 parity solve time_solve 4.05 vs
// 1.89 s with the same 510 iterations (profiles/r2_seq_solve_ab.txt).
bool seq_solve_enabled(const Dev& P) {
  const char* e = std::getenv("OCG_REFLDL_SOLVE");
  return e && std::atoi(e) == 1 && P.sq_nchunks > 0;
}

void solve(const Dev& P, const double* Dinv, const double* Lx, const double* rhs, double* x, double* y, double* xp,
           double* V, double* Vs, cudaStream_t s) {
  (void)V;
  if (seq_solve_enabled(P)) {
    const size_t smem = seq_smem_bytes(P.dim);
    static bool attr = false;
    if (!attr) {
      ck(cudaFuncSetAttribute(seq_solve_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSeqSmemMax)),
         "smem attr");
      attr = true;
    }
    seq_solve_k<<<1, 256, smem, s>>>(P, Dinv, const_cast<double*>(Lx), streamed_factor(P), rhs, x);
    ck(cudaGetLastError(), "seq solve launch");
    return;
  }
  gather_k<<<grid_for(P.dim), kThreads, 0, s>>>(P.perm, rhs, y, P.dim);
  static const int variant = std::getenv("OCG_REFLDL_KERNEL") ? std::atoi(std::getenv("OCG_REFLDL_KERNEL")) : 0;
  const bool streamed = P.nnl && P.fmax <= 8 && variant == 0 && P.chunk_foff;
  if (P.nfl && !streamed) fwd_leaf_k<<<grid_for(P.nfl), kThreads, 0, s>>>(P, Lx, y);
  if (streamed) {
    fwd_pre_k<<<grid_for(P.nnl), kThreads, 0, s>>>(P, Lx, y);
    if (P.npre_long) fwd_pre_long_k<<<static_cast<unsigned>(P.npre_long), 256, 0, s>>>(P, Lx, y);
    fwd_chain_stream_k<<<1, 32, 0, s>>>(P, Vs);
    bwd_chain_stream_k<<<1, 32, 0, s>>>(P, xp);
  } else if (P.nnl && P.fmax <= 8) {
    fwd_chain_small_k<8><<<1, 32, 0, s>>>(P, Lx, y, Vs);
    bwd_chain_small_k<8><<<1, 32, 0, s>>>(P, Lx, Dinv, y, xp);
  } else if (P.nnl && P.fmax <= 16) {
    fwd_chain_small_k<16><<<1, 32, 0, s>>>(P, Lx, y, Vs);
    bwd_chain_small_k<16><<<1, 32, 0, s>>>(P, Lx, Dinv, y, xp);
  } else if (P.nnl) {
    const int slotd = static_cast<int>(3 * P.fmax + 2);
    const int ns = ring_slots(slotd);
    const size_t smem = static_cast<size_t>(ns) * slotd * sizeof(double);
    ck(cudaFuncSetAttribute(fwd_chain_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024), "smem attr");
    ck(cudaFuncSetAttribute(bwd_chain_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024), "smem attr");
    fwd_chain_k<<<1, 32, smem, s>>>(P, ns, slotd, Lx, y, Vs);
    bwd_chain_k<<<1, 32, smem, s>>>(P, ns, slotd, Lx, Dinv, y, xp);
  }
  if (P.nleaf) bwd_leaf_k<<<grid_for(P.nleaf), kThreads, 0, s>>>(P, Lx, Dinv, y, xp);
  scatter_out_k<<<grid_for(P.dim), kThreads, 0, s>>>(P.perm, xp, x, P.dim);
  ck(cudaGetLastError(), "solve launch");
}

}  // namespace ocg::rl
