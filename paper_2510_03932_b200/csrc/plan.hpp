// Device evaluation plan: COO offsets, thread mapping and generated kernels.
#pragma once

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "model.hpp"

namespace ocg {

// COO layout of the reference EvalContext (eval.cpp:44-81): constraint groups
// first (jac, hess), then objective groups (grad, hess), group-major then
// index-major. Thread mapping: every contiguous-range group is evaluated by
// the thread of its grid index (k = idx - lo); endpoint-pair groups are
// "special" instances handled by a short tail of extra threads.
struct Layout {
  std::vector<Index> jac_off, hess_off_con, hess_off_obj, grad_off, objv_off;
  Index jac_nnz = 0, hess_nnz = 0, grad_nnz = 0, objv_n = 0;
  Index idx_lo = 0, idx_hi = 0;  // main grid-index space [idx_lo, idx_hi)
  struct Special {
    bool objective;
    int group;
    Index k;
  };
  std::vector<Special> specials;
};

Layout make_layout(const Nlp& nlp);

// every index the generated kernels form (array slots, COO offsets, tile
// bases) fits 32-bit arithmetic, with room for a tile's overshoot
inline bool fits_idx32(const Nlp& nlp, const Layout& lay) {
  Index mx = std::max({lay.jac_nnz, lay.hess_nnz, lay.grad_nnz, lay.objv_n, nlp.nvar, nlp.m_con, lay.idx_hi});
  return mx < (Index{1} << 30);
}

struct GenOptions {
  bool fma = false;  // false: no FMA contraction (bit-compatible with the x86 reference)
  int block = 128;
  // __launch_bounds__ minimum resident blocks per SM (the register budget),
  // per kernel name; absent = 1
  std::map<std::string, int> min_blocks;
  // stage one output kind (c, J, H, ...) of a group at a time through a
  // single shared-memory region (less shared memory, more warps resident)
  bool split_kinds = false;
  // every group's outputs in their own shared region: one wait per tile
  // instead of one per group (more shared memory per warp)
  bool distinct_regions = false;
  // double-buffered input staging: the next tile's LDGSTS copies are in
  // flight while this tile computes (two input buffers per warp)
  bool prefetch = false;
  // TMA tiles (block 32 only): bulk copy-in on mbarriers, double-buffered
  bool tma = false;
  // 32-bit index arithmetic (every array index of the model < 2^31)
  bool idx32 = false;
};

struct Generated {
  std::string source;  // whole module (all kernels, OCG_MINB_* defined)
  // per-kernel compilation units: "#define OCG_MINB_<name> b" + prelude + kernels[name]
  std::string prelude;
  std::map<std::string, std::string> kernels;
  // kernel name -> gridDim.y it expects (1 for the merged mapping)
  std::map<std::string, int> slices;
  // kernel name -> threads of the tail (endpoint / small-range instances)
  std::map<std::string, int> tail;
  // kernel name -> dynamic shared memory bytes per block
  std::map<std::string, int> smem;
  // values of the by-value parameter block (first kernel argument)
  std::vector<long long> params;
  // options the module was generated with (filled by the budgeted generator)
  std::map<std::string, int> min_blocks;
  int block = 128;
  bool split_kinds = false;
  bool distinct_regions = false;
  bool prefetch = false;
  bool tma = false;
  bool idx32 = false;
};

// Kernel entry points in the generated module (all extern "C"):
//   ocg_c     (x, row_scale, c, flag, i0, n_main, n_spec)
//   ocg_cjac  (x, row_scale, c, jac, flag, i0, n_main, n_spec)
//   ocg_hess  (x, lambda, row_scale, objw, hess, flag, i0, n_main, n_spec)
//   ocg_cjh   (x, lambda, row_scale, objw, c, jac, hess, flag, i0, n_main, n_spec)
//   ocg_objv  (x, objv, flag, i0, n_main, n_spec)
//   ocg_grad  (x, objw, grad, flag, i0, n_main, n_spec)
Generated generate(const Nlp& nlp, const Layout& lay, const GenOptions& opt);
inline std::string generate_source(const Nlp& nlp, const Layout& lay, const GenOptions& opt) {
  return generate(nlp, lay, opt).source;
}

}  // namespace ocg
