// Hand-written sm_100a kernels around the generated per-node kernels:
// deterministic reductions, gathers and the KKT value assembly. Every sum is
// taken in the reference's accumulation order (starting from 0.0, sources in
// increasing order) so the results are bit-identical to the CPU reference;
// no floating-point atomics anywhere (max via integer atomics on the bit
// pattern of non-negative doubles is exact and order-free).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ocg::dev {

// Rows (source lists) longer than kLongRow — e.g. a free final time's J^T
// lambda entry or matvec row, which gather one entry per dynamics row — are
// skipped by the thread-per-row kernels and summed by one block each: pure
// sums (gradient gather, KKT assembly) in the same order (increasing source
// index, one accumulator), products and norms (J^T lambda, K x, |K|) by a
// fixed-shape tree. `idx`: device array of the long rows of that pointer
// array (long_rows() on its host copy); `partials`: device scratch of
// n * kLongBlocks doubles for the tree kernels.
constexpr int64_t kLongRow = 1024;
constexpr int kLongBlocks = 296;  // two blocks per SM for each long row
struct LongRows {
  const int64_t* idx = nullptr;
  int64_t n = 0;
  double* partials = nullptr;
};
std::vector<int64_t> long_rows(const std::vector<int64_t>& ptr);
// the same on the device: long rows of ptr[0..n] into out (capacity n, any
// order — each is summed on its own); returns their count
int64_t long_rows_device(const int64_t* ptr, int64_t n, int64_t* out, cudaStream_t s);

// Objective: per-instance values -> f (EvalContext::eval_objective + Backend::par_reduce,
// eval.cpp:175-200, backend.cpp:119-133): chunks of 512 summed in index
// order, chunk partials combined in chunk order, total += weight*part per group,
// f = obj_scale * total. group_* arrays are device arrays of length n_groups.
void objective_reduce(const double* objv, const int64_t* group_off, const int64_t* group_count,
                      const int64_t* chunk_base, int64_t n_chunks, const double* weights, int n_groups,
                      double obj_scale, double* partials, double* f, int* flag, cudaStream_t s);

// the two halves of objective_reduce, for node-range shards: per-chunk
// partials of this shard's instances, then the fixed-order combine of the
// chunk partials (gathered from every shard)
void objective_chunk_sums(const double* objv, const int64_t* group_off, const int64_t* group_count,
                          const int64_t* chunk_base, int64_t n_chunks, int n_groups, double* partials,
                          cudaStream_t s);
void objective_combine(const double* partials, const int64_t* chunk_base, const double* weights, int n_groups,
                       double obj_scale, double* f, int* flag, cudaStream_t s);

// out[i] = sum_{p in [ptr[i], ptr[i+1])} src[idx[p]]  (0.0-based, in p order)
void gather_sum(const double* src, const int64_t* ptr, const int32_t* idx, int64_t n, double* out, LongRows lr,
                cudaStream_t s);

// K.val[p] = sum of its sources in code order (KktAssembler::assemble,
// eval.cpp:429-440): code < H: hess[code]; < H+J: jac[code-H]; < H+J+S: -1.0;
// < H+J+S+ntot: sigma[code-H-J-S]; else 0 (the dual diagonal's structural slot).
// code32 / order (kkt_code32 + kktbuild.hpp source_order, may be NULL): the
// slots walked in source order, single-source slots through one 32-bit word.
void kkt_assemble(const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                  const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot, double* val,
                  LongRows lr, cudaStream_t s, const uint32_t* code32 = nullptr, const int32_t* order = nullptr);
// per slot: (array tag << 29) | index for a single source, a "several" tag
// otherwise; false (nothing written) when an index does not fit 29 bits
// Tiled assembly: a block owns kTileSlots consecutive K slots and stages the
// sources they read from each source stream (the COO segment of one hess /
// jac group, or sigma) into shared memory as one window with coalesced
// loads; slot codes address the window. kkt_tile_plan builds the windows and
// the rewritten codes on the device (stream_bounds: ns+1 ascending unified
// codes, hess [0,H), jac [H,H+J), sigma [H+J+S, ...)); same sums, same order.
constexpr int64_t kTileSlots = 1024;
constexpr int kTileWindow = 2560;  // doubles of shared memory per block (20 KB)
constexpr int kTileMaxStreams = 256;
constexpr int kTileConsts = 2;  // win[0] = -1.0 (slack entries), win[1] = 0.0 (structural zeros)  // source streams (COO groups + sigma) the tiled path takes
constexpr int kTileMcode = 2048;   // codes of the tile's multi-source slots staged (uint32)
constexpr int kTileSparse = 5;     // a window is staged when len <= kTileSparse * (sources read from it) + 32
struct KktTiles {
  int64_t ntile = 0;
  int ns = 0;
  int64_t* wlo = nullptr;
  int32_t *wlen = nullptr, *woff = nullptr;
  uint32_t *code32 = nullptr, *mcode = nullptr;
};
bool kkt_tile_plan(const uint32_t* code32, const int64_t* ptr, const int64_t* code, int64_t nnz, int64_t ncode,
                   const int64_t* stream_bounds_dev, int ns, int64_t H, int64_t J, int64_t S, int64_t ntot,
                   KktTiles& out, cudaStream_t s);
void kkt_assemble_tiled(const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                        const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot, double* val,
                        LongRows lr, const KktTiles& t, cudaStream_t s);
bool kkt_code32(const int64_t* ptr, const int64_t* code, int64_t nnz, int64_t H, int64_t J, int64_t S, int64_t ntot,
                uint32_t* out, cudaStream_t s);

// y[i] = sum over the full symmetric row i (increasing column) of K_ij x_j —
// the accumulation order of sparse::matvec_sym (sparse.cpp:51-61).
// (I = int64_t, or int32_t for the narrowed index copies)
template <class I>
void sym_matvec(const double* val, const int64_t* rptr, const I* col, const I* vidx, int64_t n,
                const double* x, double* y, LongRows lr, cudaStream_t s);

// *out = max_i sum_j |K_ij| over the full symmetric rows (sparse::norm_inf_sym)
template <class I>
void sym_norm_inf(const double* val, const int64_t* rptr, const I* vidx, int64_t n, double* out, LongRows lr,
                  cudaStream_t s);

// out[i] = sum_p jac[e_p] * lam[dual_p] (p in increasing e), then for slack
// rows out[i] -= lam[dual] (Solver::compute_jt_lambda, solver.cpp:244-257).
template <class I>
void jt_lambda(const double* jac, const double* lam, const int64_t* ptr, const I* e_idx,
               const I* dual_idx, int64_t n_free, const int64_t* slack_dual, int64_t n_slack, double* out,
               LongRows lr, cudaStream_t s);
// out[i] = (int32) in[i] (index arrays whose values fit 32 bits)
void narrow_i32(const int64_t* in, int64_t n, int32_t* out, cudaStream_t s);

// max |v| over n entries into *out (device scalar); exact.
void max_abs(const double* v, int64_t n, double* out, cudaStream_t s);

}  // namespace ocg::dev

namespace ocg::dev {

// COO structure of one group on the device (EvalContext's materialisation,
// eval.cpp:83-119): entry e = off + k * np + p for instance k of the group's
// range and pattern entry p. kind 0 Jacobian: a = row + k*out_dim + pa[p],
// b = slot(pb[p]); kind 1 Hessian: (a, b) = (max, min) of the two slots;
// kind 2 gradient: a = slot(pb[p]) (b unused). slot(i) = ibase[i] + istride[i] * idx.
struct StructGroup {
  int64_t lo = 0, hi = 0;
  int endpoints = 0, kind = 0, np = 0, out_dim = 0;
  int64_t off = 0, row_base = 0;
  const int* pa = nullptr;
  const int* pb = nullptr;
  const int64_t* ibase = nullptr;
  const int64_t* istride = nullptr;
};
void struct_fill(const StructGroup& g, int64_t* a, int64_t* b, cudaStream_t s);

// out[row[q]] = max(out[row[q]], |v[q]|) over q < n (out zeroed by the caller; exact)
void row_absmax(const double* v, const int64_t* row, int64_t n, double* out, cudaStream_t s);
// rs[r] = jmax[r] > 0 ? min(1, 100 / jmax[r]) : 1 (EvalContext::compute_scaling, eval.cpp:260-286)
void row_scale_rule(const double* jmax, int64_t m, double* rs, cudaStream_t s);
// node[r] = max over entries q of row r of col_node[col[q]] (-1 when none)
void row_max_node(const int64_t* row, const int64_t* col, int64_t n, const int64_t* col_node, int64_t m,
                  int64_t* node, cudaStream_t s);

}  // namespace ocg::dev
