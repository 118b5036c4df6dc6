// Library-internal definitions of the C ABI's opaque handles (include/octgpu.h),
// shared by the ABI implementation (capi.cpp) and the batched solver
// (batch.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/octgpu.h"
#include "band.hpp"
#include "devmem.hpp"
#include "jit.hpp"
#include "kernels.hpp"
#include "model.hpp"
#include "plan.hpp"
#include "refldl.hpp"

namespace ocg::hd {

using ocg::Index;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = true;
  size_t cap = 0;  // bytes of a block from device_alloc (0: adopted from cudaMallocAsync)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  // Stream-ordered pool allocations (device_alloc) on the calling thread's
  // default stream: unlike cudaMalloc/cudaFree they do not synchronize the
  // device, so plans built by concurrent host threads do not serialize.
  ~DBuf() { release(); }
  void release() {
    if (p && owned) {
      if (cap)
        ocg::mem::device_free(p, cap);
      else
        cudaFreeAsync(p, cudaStreamPerThread);
    }
    p = nullptr;
    cap = 0;
  }
  // caller-owned device memory of the same size replaces the library buffer
  void bind(T* ext) {
    release();
    p = ext;
    owned = false;
  }
  // take ownership of device memory from cudaMallocAsync
  void adopt(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
    owned = true;
  }
  void alloc(size_t count) {
    release();
    owned = true;
    n = count;
    void* q = nullptr;
    ck(ocg::mem::device_alloc(std::max<size_t>(count, 1) * sizeof(T), &q, &cap), "cudaMallocAsync");
    p = static_cast<T*>(q);
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) {
      ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, cudaStreamPerThread), "upload");
      ck(cudaStreamSynchronize(cudaStreamPerThread), "upload sync");
    }
  }
};

// by-value batch descriptor of the generated kernels (codegen.cpp OcgBatch)
struct GenBatch {
  const int* ids;
  long long s[10];
};
inline GenBatch kNoBatch{};

}  // namespace ocg::hd

using ocg::hd::DBuf;
using ocg::hd::GenBatch;
using ocg::Index;


struct ocg_model {
  ocg::Problem prob;
  ocg::Nlp nlp;
};

namespace ocg {
struct ShardPlan;  // shard.hpp
}

struct ocg_eval {
  const ocg_model* model = nullptr;
  int device = 0;
  // ocg_eval_create_sharded: the communicator (not owned) and this rank's plan
  ocg_comm* comm = nullptr;
  std::shared_ptr<ocg::ShardPlan> shard;
  ocg::Layout lay;
  std::map<std::string, std::shared_ptr<ocg::JitModule>> mods;  // one module per kernel (process-wide cache)
  cudaKernel_t k_c = nullptr, k_cjac = nullptr, k_hess = nullptr, k_cjh = nullptr, k_objv = nullptr,
               k_grad = nullptr;
  int block = 128;
  bool specials = true;
  std::map<std::string, int> slices, tail, smem;
  std::vector<long long> prm;  // by-value parameter block of the generated kernels
  std::vector<int> prm32;      // the same as 32-bit integers (modules with 32-bit indexing)
  bool idx32 = false;
  void set_idx32(bool on) {
    idx32 = on;
    prm32.assign(prm.begin(), prm.end());
  }
  void* prm_arg() { return idx32 ? static_cast<void*>(prm32.data()) : static_cast<void*>(prm.data()); }
  std::map<std::string, int> resident;  // resident blocks per SM per kernel
  int sm_count = 148;
  Index i0 = 0, n_main = 0;

  DBuf<double> jac, hess, grad, row_scale, objv, objw, partials, scratch;
  DBuf<int> flag;
  double obj_scale = 1.0;
  std::vector<double> obj_weight;  // group weights (host)

  // objective reduction plan
  DBuf<int64_t> og_off, og_count, og_cbase;
  Index n_chunks = 0;
  DBuf<double> og_weight;

  // dense gradient gather (slot -> grad COO entries)
  DBuf<int64_t> gg_ptr;
  DBuf<int32_t> gg_idx;
  DBuf<int64_t> gg_long;  // slots with more than kLongRow gradient entries
  int64_t n_gg_long = 0;

  int64_t launches = 0;
  std::map<std::string, int> min_blocks;  // register budget the kernels were compiled for

  // ocg_eval_jac_hess_host: device x / lambda / c, and the stream and events
  // that carry each node-range chunk's outputs back while the next computes
  DBuf<double> host_x, host_lam, host_c;
  cudaStream_t out_stream = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t join_ev = nullptr;
  ~ocg_eval() {
    for (cudaEvent_t ev : chunk_ev) cudaEventDestroy(ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (out_stream) cudaStreamDestroy(out_stream);
  }

  // tail instances this shard runs for kernel `name`
  Index n_spec(const char* name) const { return specials ? tail.at(name) : 0; }

  // persistent grid: min(tiles, SMs x resident blocks per SM)
  // batched (nz > 1): grid z = instances, the persistent cap shared out
  void launch(cudaKernel_t k, const char* name, void** args, cudaStream_t s, unsigned nz = 1) {
    const Index ns = n_spec(name);
    const Index tiles = (n_main + block - 1) / block;
    if (tiles <= 0 && ns <= 0) return;
    const Index cap = static_cast<Index>(sm_count) * std::max(1, resident.at(name));
    const unsigned grid =
        static_cast<unsigned>(std::max<Index>(1, std::min(tiles, std::max<Index>(1, cap / static_cast<Index>(nz)))));
    ocg::hd::ck(cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(grid, 1, nz), dim3(static_cast<unsigned>(block)), args,
                        static_cast<size_t>(smem.at(name)), s),
       "launch generated kernel");
    ++launches;
  }

  // one node range [i0, i0 + nm) of the main grid (+ ns tail instances):
  // the same persistent grid rule over the range's tiles
  void launch_range(cudaKernel_t k, const char* name, void** args, cudaStream_t s, Index nm, Index ns) {
    const Index tiles = (nm + block - 1) / block;
    if (tiles <= 0 && ns <= 0) return;
    const Index cap = static_cast<Index>(sm_count) * std::max(1, resident.at(name));
    const unsigned grid = static_cast<unsigned>(std::max<Index>(1, std::min(tiles, cap)));
    ocg::hd::ck(cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(grid, 1, 1), dim3(static_cast<unsigned>(block)), args,
                                 static_cast<size_t>(smem.at(name)), s),
                "launch generated kernel");
    ++launches;
  }

  void refresh_objw(cudaStream_t s) {
    std::vector<double> w(obj_weight.size());
    for (size_t g = 0; g < w.size(); ++g) w[g] = obj_scale * obj_weight[g];  // eval.cpp:206,246
    if (!w.empty()) ocg::hd::ck(cudaMemcpyAsync(objw.p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, s), "objw");
    ocg::hd::ck(cudaStreamSynchronize(s), "sync");
  }
};

struct ocg_kkt {
  ocg_eval* ev = nullptr;
  Index nvar = 0, m_con = 0;
  Index n_free = 0, n_slack = 0, ntot = 0, m = 0, dim = 0, nnz = 0;
  bool contradictory = false;
  std::vector<Index> prim_index, free_slot, slack_index, slack_of, dual_index, dual_row, row_slot;
  std::vector<double> xlo, xhi;
  std::vector<Index> colp, rowi;
  DBuf<double> val;
  DBuf<int64_t> src_ptr, src_code;
  DBuf<uint32_t> src_code32;  // per slot in source order: (tag << 29) | index (kernels.hpp kkt_code32)
  DBuf<int32_t> src_order;    // slots in order of their first source (kktbuild.hpp source_order)
  // tiled assembly (kernels.hpp KktTiles): per-tile source windows, rewritten codes
  ocg::dev::KktTiles tiles;
  DBuf<int64_t> t_sb, t_wlo;
  DBuf<int32_t> t_wlen, t_woff;
  DBuf<uint32_t> t_code32, t_mcode;
  Index H = 0, J = 0;
  // matvec (full symmetric CSR in increasing column order)
  DBuf<int64_t> mv_ptr, mv_col, mv_vidx;
  // J^T lambda
  DBuf<int64_t> jt_ptr, jt_e, jt_dual, jt_slack_dual;
  // 32-bit copies of the matvec and J^T lambda index arrays (when their values fit)
  DBuf<int32_t> mv_col32, mv_vidx32, jt_e32, jt_dual32;
  // rows of src_ptr / mv_ptr / jt_ptr longer than kLongRow (kernels.hpp)
  DBuf<int64_t> src_long, mv_long, jt_long;
  int64_t n_src_long = 0, n_mv_long = 0, n_jt_long = 0;
  DBuf<double> mv_long_part, jt_long_part;  // n_*_long x kLongBlocks partial sums
};

// Band LDL^T of the KKT matrix (band.hpp): plan + device buffers
struct ocg_ldl {
  ocg_kkt* kkt = nullptr;
  ocg::BandPlan plan;
  DBuf<int64_t> dst, perm, border_pos;
  DBuf<ocg::BandSeg> segs;
  DBuf<double> primal, buf, Dinv, work;
  DBuf<long long> inertia, inertia_parts;
  DBuf<double> cr;            // separator system by block cyclic reduction
  DBuf<long long> crparts;
  ocg::dev::BandDev dev;
  double delta_w = 0.0, delta_c = 0.0;
  int64_t factorizations = 0;
  // OCG_LDL_REFERENCE: the reference's elimination order (refldl.hpp) instead of the band
  struct Ref {
    ocg::rl::Symbolic S;
    int64_t nleaf = 0, nnl = 0;
    DBuf<int64_t> nl_pos, nl_lp, nl_foff, nl_soff, nl_voff, sc_ptr, lf_pos, lf_aoff, pa_ptr, fl_ptr, fl_lx, fl_col, Lp, Li,
        sc_dst, sc_dpos, sc_ms, perm;
    DBuf<int32_t> nl_f, sc_child, lf_f, pa_j, pa_leaf, fl_j, rel;
    DBuf<int8_t> primal;
    DBuf<ocg::rl::ColRec> rec;
    DBuf<double> W, stash, D, Dinv, Lx, y, xp, V, Vs, sr, ypre, ych;
    DBuf<int64_t> fl_all_ptr;
    DBuf<int32_t> pre_long;
    DBuf<int32_t> Lp32, Li32, sq_col;  // sequential solve (refldl.hpp seq_chunks)
    DBuf<long long> chunk_foff;
    DBuf<unsigned long long> inertia;
    ocg::rl::Dev dev;
    // speculative candidates (ocg_ldl_factor_many): numeric buffers and a
    // stream each; candidate 0 is the set above
    struct Cand {
      DBuf<double> W, stash, D, Dinv, Lx, sr;
      DBuf<unsigned long long> inertia;
      cudaStream_t st = nullptr;
      cudaEvent_t ev = nullptr;
      double dw = 0.0, dc = 0.0;
      ~Cand() {
        if (ev) cudaEventDestroy(ev);
        if (st) cudaStreamDestroy(st);
      }
    };
    std::vector<std::unique_ptr<Cand>> cand;
    cudaEvent_t ev0 = nullptr;
    ~Ref() {
      if (ev0) cudaEventDestroy(ev0);
    }
  };
  std::unique_ptr<Ref> ref;
};


namespace ocg::hd {
// ocg_ldl_create with an explicit segment target (1 = unpartitioned band)
int ldl_create(ocg_kkt* k, int target, ocg_ldl** out);
// ocg_last_error's message for this thread; returns code
int set_error(int code, const std::string& msg);
// ipm.cpp: drop ocg_ipm_solve's cached plans of a model (NULL: all)
void drop_ipm_plans(const ocg_model* m);
}  // namespace ocg::hd
