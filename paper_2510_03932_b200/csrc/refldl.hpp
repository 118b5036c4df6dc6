// Device LDL^T of the KKT matrix in the REFERENCE's elimination order.
//
// The reference factors K with 1x1 pivots in the order KktAssembler::symbolic
// chooses (proj/src/ipm/eval.cpp:442-471): an AMD ordering of K's pattern
// (proj/src/sparse/ldl.cpp:54-76) in which every kept equality row whose
// Jacobian touches exactly one free column is moved to right after that
// column (pivot_after_, eval.cpp:409-426). Which 1x1 pivots fall under the
// zero-pivot threshold depends on that order, and on Goddard's near-singular
// KKT matrices the IPM's path follows those decisions. This
// factorization keeps the order exactly; only the summation order inside a
// pivot differs from the up-looking loop of ldl.cpp:166-211 (parity by order:
// a relative perturbation of 1e-14 of K leaves the reference's Goddard@1000
// solve at 510 iterations, profiles/r2_goddard_perturbation.txt).
//
// Ordering. SuiteSparse AMD is not in this image; the oracle build links a
// clean-room exact minimum-degree stand-in (oracle/amd_shim). The product
// computes the same order with its own implementation (min_degree_order):
// repeatedly eliminate the live vertex of smallest current degree (ties: the
// smallest index), its live neighbourhood becoming a clique; vertices of
// degree > max(16, 10 sqrt(n)) are left out and ordered last (AMD's dense-row
// rule). tests/test_refldl_symbolic.py checks perm, etree and the pattern of
// L against the reference's sparse::analyze_ordered.
//
// Numerics: multifrontal. Etree leaves (pattern-free rows: slack, bound and
// deferred dual pivots, ~2N of them) are factored in parallel and their
// update matrices pre-assembled into their parents' fronts; the rest of the
// tree — for a direct transcription a long chain in time — is eliminated in
// order by ONE warp that holds the current front and extend-adds its update
// matrix into the next front (usually the parent). The zero-pivot rule is the
// reference's: |d| <= 1e-14 * max(|a_kk + delta|, max |single update|), the
// max carried per diagonal through the update matrices; zero pivots get
// Dinv = 0 and are skipped by every later update. L comes out in the
// reference's layout (column-major, rows ascending, Lp/Li of analyze_ordered).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ocg::rl {

// sparse::amd_order's result for the full (both triangles, no diagonal)
// adjacency Fp/Fi of a symmetric pattern: position -> vertex
std::vector<int64_t> min_degree_order(int64_t n, const std::vector<int64_t>& Fp, const std::vector<int64_t>& Fi);

// KktAssembler::symbolic + sparse::analyze_ordered on the lower-CSC pattern
// of K (colp/rowi); indices [0, n_free) are free primal, [n_free, ntot)
// slacks, [ntot, dim) duals.
struct Symbolic {
  int64_t dim = 0, ntot = 0;
  std::vector<int64_t> perm, iperm;  // position -> KKT index, and back
  std::vector<int64_t> parent;       // elimination tree over positions, -1 = root
  std::vector<int64_t> Lp, Li;       // pattern of L by column (positions), rows ascending
};
Symbolic analyze(int64_t dim, const int64_t* colp, const int64_t* rowi, int64_t n_free, int64_t ntot);

constexpr int64_t kChain = -1, kRoot = -2;  // ColRec::soff / Dev::nl_soff markers

// Largest front (1 + column count of L) the warp kernels take.
constexpr int kMaxFront = 128;

// One chain column's metadata for the warp walks (48 bytes).
struct alignas(16) ColRec {
  long long foff;  // front in W
  int lp;          // first entry of the column in Li / Lx / rel
  int pos;         // position
  short f;         // front size
  short flags;     // bit 0: the next column is the parent, has no stashed children and both fronts <= 8 rows
  int soff;        // stash offset, or kChain / kRoot
  int sc0, sc1;    // stashed children: sc_child[sc0, sc1)
  // kChain with both fronts <= 8 rows: byte r of the parent's front is the
  // row of this front that lands there (0 = none) — the inverse of rel
  unsigned long long inv8;
  // fronts <= 8 rows: byte a-1 = rel of row a (where it lands in the parent's front)
  unsigned long long rel8;
};

// Host side of the device plan (below), built once per KKT pattern.
constexpr int64_t kPreLong = 256;

struct HostPlan {
  int64_t dim = 0, nnz = 0, lnz = 0;
  int fmax = 0;
  std::vector<int64_t> nl_pos, nl_lp, nl_foff, nl_soff, nl_voff, sc_ptr;
  std::vector<int32_t> nl_f, sc_child;
  std::vector<int64_t> lf_pos, lf_aoff;
  std::vector<int32_t> lf_f;
  std::vector<int32_t> pa_j, pa_leaf;
  std::vector<int64_t> pa_ptr;
  std::vector<int32_t> fl_j;
  std::vector<int64_t> fl_ptr, fl_lx, fl_col;
  std::vector<int64_t> fl_all_ptr;  // [nnl+1]: the same terms indexed by every chain column
  std::vector<int32_t> pre_long;    // chain columns with more than kPreLong leaf terms
  std::vector<int32_t> rel;
  std::vector<int64_t> sc_dst, sc_dpos, sc_ms;
  std::vector<int8_t> primal;
  std::vector<ColRec> rec;
  int64_t w_len = 0, stash_len = 0, v_len = 0, fronts_len = 0;
  std::vector<long long> chunk_foff;  // per 16 chain columns, then fronts_len
};
HostPlan build_plan(const Symbolic& S, const int64_t* colp, const int64_t* rowi);

// Device plan (refldl.cu). Columns of L are "leaves" (no etree child) or
// "chain" columns (all others, in elimination order: index j below).
struct Dev {
  int64_t dim = 0, nnz = 0, lnz = 0, nleaf = 0, nnl = 0, npa = 0, nfl = 0;
  int fmax = 0;
  // chain columns, j = 0..nnl-1
  const ColRec* rec = nullptr;       // [nnl] the same, packed for the walks
  const int64_t* nl_pos = nullptr;   // position
  const int64_t* nl_lp = nullptr;    // Lp[position]
  const int32_t* nl_f = nullptr;     // front size (1 + column count)
  const int64_t* nl_foff = nullptr;  // front (packed lower, row-major, then f diagonal maxima) in W
  // stash of the update matrix / vector when the parent is not column j+1:
  // offset >= 0; kChain: the parent is column j+1; kRoot: no parent
  const int64_t* nl_soff = nullptr;
  const int64_t* nl_voff = nullptr;  // vector front (solves), f doubles
  const int64_t* sc_ptr = nullptr;   // [nnl+1] stashed children of j (CSR) ...
  const int32_t* sc_child = nullptr; // ... as chain indices, ascending
  // leaves, i = 0..nleaf-1
  const int64_t* lf_pos = nullptr;
  const int32_t* lf_f = nullptr;
  const int64_t* lf_aoff = nullptr;  // A column (f values, diagonal first) in W
  // pre-assembly of leaf update matrices into chain fronts: chain index pa_j[q] gets its leaves
  const int32_t* pa_j = nullptr;     // [npa]
  const int64_t* pa_ptr = nullptr;   // [npa+1] -> pa_leaf
  const int32_t* pa_leaf = nullptr;  // leaf indices, ascending
  // forward solve: leaf terms of chain rows, rows j with any (CSR over fl_j)
  const int32_t* fl_j = nullptr;     // [nfl]
  const int64_t* fl_ptr = nullptr;   // [nfl+1]
  const int64_t* fl_lx = nullptr;    // L entry index
  const int64_t* fl_col = nullptr;   // leaf position
  const int64_t* fl_all_ptr = nullptr;  // [nnl+1] leaf terms of every chain column
  // chain columns with more than kPreLong leaf terms (a free final time's
  // row): summed by one block each, in order, instead of one thread
  const int32_t* pre_long = nullptr;
  int64_t npre_long = 0;
  // streamed walks (fronts <= 8): per chain column, its L entries and Dinv
  // (8 doubles, written by the factorization), the right-hand side after the
  // leaf terms and the forward result, all in walk order
  double* sr = nullptr;     // [nnl * 8]
  double* ypre = nullptr;   // [nnl]
  double* ych = nullptr;    // [nnl]
  int64_t fronts_len = 0;   // doubles of W holding the chain fronts
  const long long* chunk_foff = nullptr;  // [nchunks+1] W offset of every kChunk(16)-column chunk's fronts
  // L pattern
  const int64_t* Lp = nullptr;       // [dim+1] by position
  const int64_t* Li = nullptr;       // [lnz]
  const int32_t* rel = nullptr;      // [lnz] position of Li[p] in the parent's front (0 = the parent)
  // K entry p -> W index of its value; diagonal entries also carry their position
  const int64_t* sc_dst = nullptr;
  const int64_t* sc_dpos = nullptr;  // position (diagonal) or -1
  const int64_t* sc_ms = nullptr;    // W index of the front's diagonal max (chain diagonal) or -1
  const int64_t* perm = nullptr;     // position -> KKT index
  const int8_t* primal = nullptr;    // position: 1 = +delta_w, 0 = -delta_c
  int64_t w_len = 0, stash_len = 0, v_len = 0;
  // sequential solve (seq_solve_k): L's pattern as 32-bit Lp / Li and the
  // column chunks the block stages through shared memory (sq_col[c] = first
  // column of chunk c, sq_nchunks + 1 entries); sq_nchunks = 0: not planned
  const int32_t* Lp32 = nullptr;
  const int32_t* Li32 = nullptr;
  const int32_t* sq_col = nullptr;
  int64_t sq_nchunks = 0;
};

// Column chunks of at most kSeqCols columns and kSeqEnt entries of L for the
// sequential solve; empty when some column alone holds more than kSeqEnt
// entries or the solution vector does not fit shared memory beside the two
// staging buffers (the warp-chain solves are used then).
constexpr int kSeqCols = 256, kSeqEnt = 1536;
constexpr size_t kSeqSmemMax = 227 * 1024;
std::vector<int32_t> seq_chunks(const std::vector<int64_t>& Lp);
size_t seq_smem_bytes(int64_t dim);
// the sequential solve runs (planned, and OCG_REFLDL_SOLVE unset or 1)
bool seq_solve_enabled(const Dev& P);

// numeric factorization: W (w_len) and stash (stash_len) scratch; D, Dinv by
// position; Lx in the layout of Lp/Li; inertia (device, 3 counts) =
// (positive, negative, zero)
void factor(const Dev& P, const double* kval, double delta_w, double delta_c, double* W, double* stash, double* D,
            double* Dinv, double* Lx, unsigned long long* inertia, cudaStream_t s);
// the streamed factorization (fronts <= 8) leaves the chain columns of L in
// P.sr only; this writes them into Lx (the LdlFactor layout) on demand
void fill_lx(const Dev& P, double* Lx, cudaStream_t s);
// x = (K + deltas)^{-1} rhs in KKT index order; y, xp (dim), V (v_len), Vs
// (stash_len) scratch
void solve(const Dev& P, const double* Dinv, const double* Lx, const double* rhs, double* x, double* y, double* xp,
           double* V, double* Vs, cudaStream_t s);

}  // namespace ocg::rl
