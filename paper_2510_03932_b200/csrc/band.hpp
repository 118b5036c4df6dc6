// Device LDL^T of the KKT matrix in a node-major band-plus-border ordering.
//
// Stand-in for the sparse factorization the reference runs on the host
// (proj/src/sparse/ldl.cpp:139-272) and the paper runs in cuDSS, which this
// image does not ship. A direct transcription's KKT matrix,
// ordered by time node (each node's primal slots, then the slacks and the
// duals of the rows whose last coupled node it is), is banded with a
// bandwidth of a few node blocks; free variables such as a free final time
// couple every node and are ordered last as a dense border. The factorization
// keeps the reference's conventions: 1x1 pivots only, +delta_w on primal and
// -delta_c on dual diagonals, a pivot counts as zero when
// |d| <= 1e-14 * max(|a_kk + delta|, max |update|) and is then skipped by all
// later updates, and the inertia is reported as (positive, negative, zero).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ocg {

struct BandPlan {
  int64_t dim = 0;  // KKT dimension = n + w
  int64_t n = 0;    // banded part
  int b = 0;        // lower bandwidth
  int w = 0;        // border (dense) rows, ordered last
  std::vector<int64_t> perm;    // position -> KKT index
  std::vector<int64_t> dst;     // K entry p -> flat offset in the factor buffer
  std::vector<double> primal;   // per position: 1 = primal (+delta_w), 0 = dual (-delta_c)
  int64_t buf_len() const { return n * (b + 1) + static_cast<int64_t>(w) * n + static_cast<int64_t>(w) * w; }
};

// node[i]: time node of KKT index i, or -1 for a border index. Ordering:
// (node, i) for banded indices — callers number indices so that primal
// slots precede slacks precede duals. colp/rowi: lower CSC of K.
BandPlan make_band_plan(int64_t dim, const std::vector<int64_t>& node, const std::vector<int64_t>& colp,
                        const std::vector<int64_t>& rowi, int64_t ntot);

namespace dev {

// buf = P K P^T in band/border layout (zeroed first)
void band_assemble(const double* kval, const int64_t* dst, int64_t nnz, double* buf, int64_t len, cudaStream_t s);

// in-place LDL^T of buf; Dinv[dim] (position order); inertia[3] (device int64)
void band_factor(double* buf, const double* primal, int64_t n, int b, int w, double delta_w, double delta_c,
                 double* Dinv, long long* inertia, cudaStream_t s);

// x = (P^T L D L^T P)^{-1} rhs; rhs, x in KKT index order; work[dim] scratch
void band_solve(const double* buf, const double* Dinv, const int64_t* perm, int64_t n, int b, int w,
                const double* rhs, double* x, double* work, cudaStream_t s);

}  // namespace dev
}  // namespace ocg
