// Device LDL^T of the KKT matrix in a node-major band-plus-border ordering,
// partitioned in time for parallelism.
//
// Stand-in for the sparse factorization the reference runs on the host
// (proj/src/sparse/ldl.cpp:139-272) and the paper runs in cuDSS, which this
// image does not ship. A direct transcription's KKT matrix,
// ordered by time node (each node's primal slots, then the slacks and the
// duals of the rows whose last coupled node it is), is banded with a
// bandwidth of a few node blocks; free variables such as a free final time
// couple every node and are ordered last as a dense border.
//
// One level of nested dissection makes it parallel: the band is cut into P
// segments separated by b-wide separators. Every segment's interior is
// factored independently (one thread block each) together with its border
// rows (left separator, global border, right separator), leaving a Schur
// complement on those rows; the separators and the global border then form a
// block-tridiagonal band system that is factored last. Sylvester's law makes
// the inertia the sum of the parts'.
//
// Conventions of the reference kept: 1x1 pivots only, +delta_w on primal and
// -delta_c on dual diagonals, a pivot counts as zero when
// |d| <= 1e-14 * max(|a_kk + delta|, max |update|) and is then skipped by all
// later updates, and the inertia is reported as (positive, negative, zero).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ocg {

// One banded block with a dense border (a segment, or the separator system).
struct BandSeg {
  long long n = 0;       // interior (banded) columns
  int b = 0;             // lower bandwidth
  int w = 0;             // border rows
  int w_early = 0;       // rows [0, w_early) couple from column 0, the rest only to the last b columns
  int finalize = 0;      // 1: factor the border block too; 0: leave its Schur complement in S
  long long band = 0;    // offsets (doubles) into the factor buffer: band n*(b+1), column-major by column
  long long border = 0;  // w*n, row-major (t*n + c)
  long long S = 0;       // w*w
  long long pos = 0;     // first position (Dinv / flags / vector index) of the interior columns
  long long bpos = -1;   // finalize: first position of the border rows
  // n + w pivot-scale seeds (interior columns, then border rows): a block
  // factored after others starts each pivot's scale at max(|a_kk + delta|,
  // seed), the seed being the largest single update the earlier blocks
  // applied to that diagonal. A segment leaves its border rows' scales here.
  long long ps0 = 0;
};

struct BandPlan {
  int64_t dim = 0;
  int b = 0;        // segment bandwidth
  int wg = 0;       // global border rows
  int nseg = 0;     // P segments (1 = no partition: the single block is finalized)
  std::vector<BandSeg> segs;  // P segments, then the separator system (when P > 1)
  std::vector<int64_t> perm;  // position -> KKT index
  std::vector<int64_t> dst;   // K entry p -> flat offset in the factor buffer
  std::vector<double> primal; // per position: 1 = primal (+delta_w), 0 = dual (-delta_c)
  // separator-system position of every segment border row: [seg * wmax + t], -1 = none
  std::vector<int64_t> border_pos;
  int wmax = 0;                // border rows per segment (uniform stride)
  int64_t buf_len = 0;
  int64_t nnz = 0;  // KKT entries scattered by band_assemble
  size_t smem_factor = 0, smem_solve = 0;
};

// device copy of the KKT pattern: with it the O(nnz) parts of the plan
// (bandwidth, entry -> buffer offsets) run on the device
struct DeviceCsc {
  const int64_t* colp = nullptr;
  const int64_t* rowi = nullptr;
  int64_t nnz = 0;
  cudaStream_t stream = nullptr;
};

// node[i]: time node of KKT index i, or -1 for a border index. Indices of one
// node keep their KKT order (primal slots, slacks, duals). colp/rowi: lower
// CSC. With dcsc the entry offsets come back in *d_dst (device,
// cudaMallocAsync'd, caller owns) and P.dst stays empty.
BandPlan make_band_plan(int64_t dim, const std::vector<int64_t>& node, const std::vector<int64_t>& colp,
                        const std::vector<int64_t>& rowi, int64_t ntot, int target_segments = 0,
                        const DeviceCsc* dcsc = nullptr, int64_t** d_dst = nullptr);

namespace dev {

// Batched launches over many systems of one plan (ids != NULL): grid row y
// factors / solves system ids[y]; per-system arrays are [system][stride].
struct BandBatch {
  const int* ids = nullptr;
  long long sbuf = 0, sdim = 0, swork = 0, sparts = 0;  // strides: factor buffer, Dinv / vectors, work, inertia
  const double* dw = nullptr;  // [y] regularization per launched system (NULL: the scalar arguments)
  const double* dc = nullptr;
};

struct BandDstIn {
  const int64_t* colp = nullptr;
  const int64_t* rowi = nullptr;
  const int64_t* fpos = nullptr;
  int64_t dim = 0, n = 0, b = 0, wg = 0, n2 = 0, nseg = 1;
  int64_t nnz = 0;
};
int64_t* upload_i64(const std::vector<int64_t>& v, cudaStream_t s);
int64_t bandwidth(const int64_t* colp, const int64_t* rowi, const int64_t* fpos, int64_t n, int64_t dim,
                  cudaStream_t s);
int64_t* band_dst(const BandDstIn& in, const std::vector<int8_t>& lk, const std::vector<int64_t>& li,
                  const std::vector<int64_t>& ll, const std::vector<BandSeg>& segs, int64_t nnz, cudaStream_t s);

struct BandDev {  // device copies of the plan
  const BandSeg* segs = nullptr;
  const int64_t* dst = nullptr;
  const int64_t* perm = nullptr;
  const double* primal = nullptr;
  const int64_t* border_pos = nullptr;
  // separator system by block cyclic reduction (sepcr.cu); NULL: one band block
  double* cr = nullptr;        // cr_length(nseg - 1, b, wg) doubles
  long long* crparts = nullptr;  // 3 (nseg - 1) inertia counts
};

// block cyclic reduction of the separator system (sepcr.cu)
long long cr_length(int ns, int b, int w);
void cr_factor(const BandPlan& P, const BandSeg& sep, const double* buf, const double* primal, double dw, double dc,
               double* cr, long long* crparts, long long* sep_inertia, cudaStream_t s);
void cr_solve(const BandPlan& P, const BandSeg& sep, double* cr, double* work, cudaStream_t s);

// buf = P K P^T scattered into the segment and separator blocks (zeroed first)
void band_assemble(const BandPlan& P, const BandDev& D, const double* kval, double* buf, cudaStream_t s);

// in-place LDL^T; Dinv[dim] by position; inertia (device, 3 x int64) = (pos, neg, zero)
void band_factor(const BandPlan& P, const BandDev& D, double* buf, double delta_w, double delta_c, double* Dinv,
                 long long* inertia_parts, long long* inertia, cudaStream_t s);

// x = (K + deltas)^{-1} rhs (KKT index order); work[dim + nseg*wmax] scratch
void band_solve(const BandPlan& P, const BandDev& D, const double* buf, const double* Dinv, const double* rhs,
                double* x, double* work, cudaStream_t s);

// Batched factor / solve of the systems ids[0..nb): kval [system][nnz] -> buf
// [system][buf_len], Dinv [system][dim], inertia [system][3] = (pos, neg,
// zero), parts [system][3 (nseg + 1)] scratch; rhs, x [system][dim], work
// [system][dim + nseg * wmax]. Unpartitioned bands without a border and
// b + 1 <= 32 run one warp per system; partitioned plans run segments x
// systems in one launch.
void band_factor_batch(const BandPlan& P, const BandDev& D, const double* kval, double* buf, double* Dinv,
                       long long* inertia, long long* parts, const int* ids, int nb, const double* dws,
                       const double* dcs, cudaStream_t s);
void band_solve_batch(const BandPlan& P, const BandDev& D, const double* buf, const double* Dinv, const double* rhs,
                      double* x, double* work, const int* ids, int nb, cudaStream_t s);

}  // namespace dev
}  // namespace ocg
