// Device construction of the KKT pattern, the assembly's source lists, the
// symmetric-CSR matvec map and the J^T lambda gather (see kktbuild.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ocg::dev {

struct KktBuildIn {  // device arrays
  const int64_t *hr = nullptr, *hc = nullptr;  // Hessian COO (row >= col), H entries
  const int64_t *jr = nullptr, *jc = nullptr;  // Jacobian COO, J entries
  int64_t H = 0, J = 0;
  const int64_t* prim = nullptr;        // slot -> reduced primal index or -1
  const int64_t* dual = nullptr;        // row -> dual ordinal or -1
  const int64_t* slack_dual = nullptr;  // slack ordinal -> dual ordinal
  int64_t n_free = 0, n_slack = 0, m = 0;
};

struct KktBuildOut {
  std::vector<int64_t> colp, rowi;  // lower CSC (host copies)
  int64_t nnz = 0;
  // device arrays allocated with cudaMallocAsync; the caller owns them
  int64_t* src_ptr = nullptr;   // [nnz + 1] into src_code
  int64_t* src_code = nullptr;  // source codes: < H hess, < H+J jac, < +S slack (-1), < +ntot sigma, else 0
  int64_t ncode = 0;
  int64_t *mv_ptr = nullptr, *mv_col = nullptr, *mv_vidx = nullptr;
  int64_t *jt_ptr = nullptr, *jt_e = nullptr, *jt_dual = nullptr;
};

void build_kkt(const KktBuildIn& in, cudaStream_t s, KktBuildOut& out);

// The assembly's slots ordered by their first source code: order[t] = slot,
// code32_sorted[t] = code32[slot]. Walking slots in this order the assembly
// reads hess / jac / sigma nearly sequentially (coalesced) and scatters the
// writes, instead of gathering the sources slot by slot (kernels.cu
// kkt_assemble_fast_k).
void source_order(const int64_t* ptr, const int64_t* code, const uint32_t* code32, int64_t nnz, int64_t max_code,
                  int32_t* order, uint32_t* code32_sorted, cudaStream_t s);

}  // namespace ocg::dev
