// extern "C" boundary (include/octgpu.h): model, EvalContext and KKT objects.
//
// ocg_eval mirrors octrans::ipm::detail::EvalContext (ipm_internal.hpp:40-95):
// identical COO structure, identical scaled outputs, bool results recovered
// from a device-side failure flag. ocg_kkt mirrors Reduction + KktAssembler
// (ipm_internal.hpp:102-146, eval.cpp:290-440): identical lower-CSC pattern,
// assembly as a precomputed segmented gather (no atomics) that adds the
// sources of every slot in the reference's order.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/octgpu.h"
#include "jit.hpp"
#include "band.hpp"
#include "kktbuild.hpp"
#include "kernels.hpp"
#include "model.hpp"
#include "plan.hpp"
#include "handles.hpp"

using ocg::Index;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

cudaStream_t st(ocg_stream s) { return static_cast<cudaStream_t>(s); }
using ocg::hd::ck;
using ocg::hd::CudaError;
using ocg::hd::kNoBatch;

}  // namespace

namespace {

// parallel loop over [0, n) in contiguous chunks on the host's cores
template <class F>
void parallel_for(Index n, F&& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const Index nt = std::min<Index>(static_cast<Index>(hw), std::max<Index>(1, n / 65536));
  if (nt <= 1) {
    f(Index{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (Index t = 0; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}

// host COO structure, exactly as EvalContext's constructor materialises it
// (eval.cpp:83-119): group-major, then index-major, pattern order within
void host_structure(const ocg::Nlp& nlp, std::vector<Index>* jr, std::vector<Index>* jc, std::vector<Index>* hr,
                    std::vector<Index>* hc, std::vector<Index>* gc) {
  Index nj = 0, nh = 0, ng = 0;
  for (const auto& g : nlp.cons) {
    nj += static_cast<Index>(g.pattern.jac.size()) * g.range.count();
    nh += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  }
  for (const auto& g : nlp.objs) {
    ng += static_cast<Index>(g.pattern.jac.size()) * g.range.count();
    nh += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  }
  if (jr) {
    jr->resize(static_cast<size_t>(nj));
    jc->resize(static_cast<size_t>(nj));
  }
  if (hr) {
    hr->resize(static_cast<size_t>(nh));
    hc->resize(static_cast<size_t>(nh));
  }
  if (gc) gc->resize(static_cast<size_t>(ng));
  Index joff = 0, hoff = 0, goff = 0;
  auto hess_fill = [&](const ocg::Group& g, Index base) {
    const auto& ins = g.kernel.graph.inputs();
    const Index nnz = static_cast<Index>(g.pattern.hess.size());
    parallel_for(g.range.count(), [&](Index k0, Index k1) {
      for (Index k = k0; k < k1; ++k) {
        const Index idx = g.range.at(k);
        Index e = base + k * nnz;
        for (const auto& [a, b] : g.pattern.hess) {
          const Index sa = ins[static_cast<size_t>(a)].slot(idx), sb = ins[static_cast<size_t>(b)].slot(idx);
          (*hr)[static_cast<size_t>(e)] = std::max(sa, sb);
          (*hc)[static_cast<size_t>(e++)] = std::min(sa, sb);
        }
      }
    });
  };
  for (const auto& g : nlp.cons) {
    const auto& ins = g.kernel.graph.inputs();
    const Index cnt = g.range.count();
    if (jr) {
      const Index nnz = static_cast<Index>(g.pattern.jac.size());
      parallel_for(cnt, [&](Index k0, Index k1) {
        for (Index k = k0; k < k1; ++k) {
          const Index idx = g.range.at(k);
          Index e = joff + k * nnz;
          for (const auto& [r, j] : g.pattern.jac) {
            (*jr)[static_cast<size_t>(e)] = g.row_base + k * g.out_dim() + r;
            (*jc)[static_cast<size_t>(e++)] = ins[static_cast<size_t>(j)].slot(idx);
          }
        }
      });
    }
    if (hr) hess_fill(g, hoff);
    joff += static_cast<Index>(g.pattern.jac.size()) * cnt;
    hoff += static_cast<Index>(g.pattern.hess.size()) * cnt;
  }
  for (const auto& g : nlp.objs) {
    const auto& ins = g.kernel.graph.inputs();
    const Index cnt = g.range.count();
    if (gc) {
      const Index nnz = static_cast<Index>(g.pattern.jac.size());
      parallel_for(cnt, [&](Index k0, Index k1) {
        for (Index k = k0; k < k1; ++k) {
          const Index idx = g.range.at(k);
          Index e = goff + k * nnz;
          for (const auto& pr : g.pattern.jac) (*gc)[static_cast<size_t>(e++)] = ins[static_cast<size_t>(pr.second)].slot(idx);
        }
      });
    }
    if (hr) hess_fill(g, hoff);
    goff += static_cast<Index>(g.pattern.jac.size()) * cnt;
    hoff += static_cast<Index>(g.pattern.hess.size()) * cnt;
  }
}

// the same COO structure built on the device (kernels.hpp struct_fill): one
// launch per group over its instances x pattern entries, from the groups'
// patterns and input addresses (a few KB uploaded once). jr/jc and/or hr/hc.
void device_structure(const ocg::Nlp& nlp, DBuf<int64_t>* jr, DBuf<int64_t>* jc, DBuf<int64_t>* hr,
                      DBuf<int64_t>* hc, cudaStream_t s) {
  Index nj = 0, nh = 0;
  for (const auto& g : nlp.cons) {
    nj += static_cast<Index>(g.pattern.jac.size()) * g.range.count();
    nh += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  }
  for (const auto& g : nlp.objs) nh += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  if (jr) {
    jr->alloc(static_cast<size_t>(nj));
    jc->alloc(static_cast<size_t>(nj));
  }
  if (hr) {
    hr->alloc(static_cast<size_t>(nh));
    hc->alloc(static_cast<size_t>(nh));
  }
  // flat pattern / address tables
  std::vector<int> pat;
  std::vector<int64_t> addr;
  struct Pending {
    ocg::dev::StructGroup g;
    size_t pa, pb, ia, n_in;
  };
  std::vector<Pending> todo;
  auto add = [&](const ocg::Group& g, int kind, const auto& pairs, Index off) {
    if (pairs.empty() || g.range.count() == 0) return;
    Pending t;
    t.g.lo = g.range.lo;
    t.g.hi = g.range.hi;
    t.g.endpoints = g.range.endpoints ? 1 : 0;
    t.g.kind = kind;
    t.g.np = static_cast<int>(pairs.size());
    t.g.out_dim = g.out_dim();
    t.g.off = off;
    t.g.row_base = g.row_base;
    t.pa = pat.size();
    for (const auto& pr : pairs) pat.push_back(static_cast<int>(pr.first));
    t.pb = pat.size();
    for (const auto& pr : pairs) pat.push_back(static_cast<int>(pr.second));
    const auto& ins = g.kernel.graph.inputs();
    t.ia = addr.size();
    t.n_in = ins.size();
    for (const auto& a : ins) addr.push_back(a.base);
    for (const auto& a : ins) addr.push_back(a.stride);
    todo.push_back(t);
  };
  Index joff = 0, hoff = 0;
  for (const auto& g : nlp.cons) {
    if (jr) add(g, 0, g.pattern.jac, joff);
    if (hr) add(g, 1, g.pattern.hess, hoff);
    joff += static_cast<Index>(g.pattern.jac.size()) * g.range.count();
    hoff += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  }
  for (const auto& g : nlp.objs) {
    if (hr) add(g, 1, g.pattern.hess, hoff);
    hoff += static_cast<Index>(g.pattern.hess.size()) * g.range.count();
  }
  if (todo.empty()) return;
  DBuf<int> dpat;
  DBuf<int64_t> daddr;
  dpat.upload(pat);
  daddr.upload(addr);
  for (auto& t : todo) {
    t.g.pa = dpat.p + t.pa;
    t.g.pb = dpat.p + t.pb;
    t.g.ibase = daddr.p + t.ia;
    t.g.istride = daddr.p + t.ia + t.n_in;
    if (t.g.kind == 0)
      ocg::dev::struct_fill(t.g, jr->p, jc->p, s);
    else
      ocg::dev::struct_fill(t.g, hr->p, hc->p, s);
  }
  ck(cudaStreamSynchronize(s), "structure sync");
}

const char* const kKernelNames[] = {"ocg_c", "ocg_cjac", "ocg_hess", "ocg_cjh", "ocg_objv", "ocg_grad"};

// per-kernel (registers, spill-store bytes) from the ptxas -v part of an NVRTC log
std::map<std::string, std::pair<int, int>> ptxas_stats(const std::string& log) {
  std::map<std::string, std::pair<int, int>> out;
  std::string cur;
  size_t pos = 0;
  while (pos < log.size()) {
    size_t eol = log.find('\n', pos);
    if (eol == std::string::npos) eol = log.size();
    const std::string ln = log.substr(pos, eol - pos);
    pos = eol + 1;
    size_t a = ln.find("entry function '");
    if (a != std::string::npos) {
      a += 16;
      cur = ln.substr(a, ln.find('\'', a) - a);
      continue;
    }
    a = ln.find("Function properties for ");
    if (a != std::string::npos) {  // also device functions (e.g. libdevice slow paths)
      cur = ln.substr(a + 24);
      while (!cur.empty() && (cur.back() == ' ' || cur.back() == '\r')) cur.pop_back();
      continue;
    }
    if (cur.empty()) continue;
    a = ln.find("bytes spill stores");
    if (a != std::string::npos) {
      size_t b = ln.rfind(',', a);
      b = b == std::string::npos ? ln.find(':') + 1 : b + 1;
      out[cur].second = std::atoi(ln.c_str() + b);
    }
    a = ln.find("Used ");
    if (a != std::string::npos) out[cur].first = std::atoi(ln.c_str() + a + 5);
  }
  return out;
}

// Code generation + NVRTC with a register budget per kernel: each kernel is
// compiled for `target` resident blocks per SM (capped by what its shared
// memory allows), stepping the budget down for kernels whose code would spill.
ocg::Generated generate_budgeted(const ocg::Nlp& nlp, const ocg::Layout& lay, ocg::GenOptions go, int target,
                                 int split, int staging, int smem_per_sm, int smem_per_block_max, std::string* log_out,
                                 std::map<std::string, std::string>* cubins_out = nullptr) {
  auto max_smem = [](const ocg::Generated& g) {
    int mx = 0;
    for (const auto& kv : g.smem) mx = std::max(mx, kv.second);
    return mx;
  };
  if (const char* e = std::getenv("OCG_SPLIT")) split = std::atoi(e);
  // output staging: 0 one region reused group after group, 1 one region per
  // output kind in turn, 2 a region per group (one wait per tile). Auto: a
  // region per group while three 4-warp blocks of the fused kernel still fit
  // (the register budget of these kernels rarely allows more), else shared.
  if (split < 0) {
    go.split_kinds = false;
    go.distinct_regions = true;
    const ocg::Generated g2 = ocg::generate(nlp, lay, go);
    const int per_block = g2.smem.at("ocg_cjh") * 128 / std::max(1, go.block) + 1024;
    go.distinct_regions = 3 * per_block <= smem_per_sm;
  } else {
    go.split_kinds = split == 1;
    go.distinct_regions = split == 2;
  }
  if (const char* e = std::getenv("OCG_STAGING")) staging = std::atoi(e);
  go.idx32 = ocg::fits_idx32(nlp, lay);
  if (const char* e = std::getenv("OCG_IDX64")) go.idx32 = go.idx32 && std::atoi(e) == 0;
  go.tma = staging == 2;
  if (go.tma) go.block = 32;
  go.prefetch = staging == 1;
  ocg::Generated gen = ocg::generate(nlp, lay, go);
  // shared memory per block scales with warps per block: halve the block
  // until every kernel fits the per-block limit
  while (max_smem(gen) > smem_per_block_max && go.block > 32) {
    go.block /= 2;
    gen = ocg::generate(nlp, lay, go);
  }
  // auto staging: double-buffer the inputs when the second buffer costs no
  // resident blocks of the fused kernel (its budget is rarely above 3-4
  // blocks per SM), else stage once per tile
  if (staging < 0 && go.distinct_regions && !go.split_kinds) {
    auto blocks = [&](const ocg::Generated& g) {
      return std::min(std::max(1, smem_per_sm / (g.smem.at("ocg_cjh") + 1024)), 4 * std::max(1, 128 / go.block));
    };
    go.prefetch = true;
    ocg::Generated g2 = ocg::generate(nlp, lay, go);
    if (max_smem(g2) <= smem_per_block_max && blocks(g2) >= blocks(gen))
      gen = std::move(g2);
    else
      go.prefetch = false;
  }
  if (max_smem(gen) > smem_per_block_max)
    throw std::runtime_error("model needs more shared memory per warp than one block provides");
  // the target counts 128-thread blocks; one-warp blocks (TMA tiles) scale it
  // to the same warps per SM, within the 32 resident blocks an SM holds
  const int per128 = std::max(1, 128 / go.block);
  for (const char* k : kKernelNames) {
    const int sm = gen.smem.at(k) + 1024;  // + per-block reservation
    const int by_smem = std::max(1, smem_per_sm / std::max(sm, 1));
    const int by_threads = std::min(32, std::max(1, 2048 / go.block));
    go.min_blocks[k] = std::max(1, std::min({target * per128, by_smem, by_threads}));
  }
  // every kernel is its own compilation unit, compiled concurrently; each
  // steps its register budget down while ptxas reports spills
  int spill_ok = 256;
  if (const char* e = std::getenv("OCG_SPILL_OK")) spill_ok = std::atoi(e);
  std::vector<std::thread> th;
  std::vector<std::string> errs(std::size(kKernelNames));
  std::vector<int> mbs(std::size(kKernelNames));
  std::vector<std::string> cubins(std::size(kKernelNames)), klogs(std::size(kKernelNames));
  for (size_t i = 0; i < std::size(kKernelNames); ++i) {
    mbs[i] = go.min_blocks[kKernelNames[i]];
    th.emplace_back([&, i] {
      try {
        const std::string name = kKernelNames[i];
        for (int it = 0; it < 8; ++it) {
          const std::string src =
              "#define OCG_MINB_" + name + " " + std::to_string(mbs[i]) + "\n" + gen.prelude + gen.kernels.at(name);
          ocg::jit_compile_only(src, go.fma, cubins[i], &klogs[i]);
          const auto st = ptxas_stats(klogs[i]);
          const auto f = st.find(name);
          // a few spilled registers (served from L1) cost less than a lost
          // block of occupancy: step the budget down only past spill_ok bytes
          if (f == st.end() || f->second.second <= spill_ok || mbs[i] <= 1) break;
          mbs[i] = std::max(1, mbs[i] - (mbs[i] > per128 ? per128 : 1));
        }
      } catch (const std::exception& ex) {
        errs[i] = ex.what();
      }
    });
  }
  for (auto& t : th) t.join();
  for (size_t i = 0; i < std::size(kKernelNames); ++i) {
    if (!errs[i].empty()) throw std::runtime_error(errs[i]);
    go.min_blocks[kKernelNames[i]] = mbs[i];
    if (cubins_out) (*cubins_out)[kKernelNames[i]] = cubins[i];
    if (log_out) *log_out += klogs[i];
  }
  gen.min_blocks = go.min_blocks;
  gen.block = go.block;
  gen.split_kinds = go.split_kinds;
  gen.distinct_regions = go.distinct_regions;
  gen.prefetch = go.prefetch;
  gen.tma = go.tma;
  gen.idx32 = go.idx32;
  return gen;
}

// Loaded modules are shared by every eval context whose kernel compiled to the
// same cubin (e.g. batch instances that differ only in bounds): one
// cudaLibrary per distinct cubin per device per process.
std::shared_ptr<ocg::JitModule> loaded_module(const std::string& cubin) {
  static std::mutex mu;
  static std::map<std::pair<size_t, size_t>, std::shared_ptr<ocg::JitModule>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(std::hash<std::string>{}(cubin) ^ static_cast<size_t>(dev), cubin.size());
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto mod = std::make_shared<ocg::JitModule>();
  ocg::jit_load(cubin, *mod);
  cache.emplace(key, mod);
  return mod;
}

int auto_min_blocks(const ocg_eval_options& o) {
  if (o.min_blocks > 0) return o.min_blocks;
  if (const char* e = std::getenv("OCG_MINB")) return std::max(1, std::atoi(e));
  return 6;
}

}  // namespace

extern "C" {

const char* ocg_last_error(void) { return g_err.c_str(); }
void ocg_free(void* p) { std::free(p); }
const char* ocg_version(void) { return "octgpu 0.1 (sm_100a)"; }

// ---- model --------------------------------------------------------------------

int ocg_model_create(const char* source, int scheme, int64_t N, int boxes_as_bounds, ocg_model** out) {
  if (!source || !out) return fail(OCG_ERR_ARG, "null argument");
  try {
    auto m = std::make_unique<ocg_model>();
    m->prob = ocg::parse_problem(source);
    m->nlp = ocg::transcribe(m->prob, scheme == 0 ? ocg::Scheme::euler : ocg::Scheme::trapezoid, N,
                             boxes_as_bounds != 0);
    *out = m.release();
    return OCG_OK;
  } catch (const ocg::ParseError& e) {
    return fail(OCG_ERR_PARSE, e.what());
  } catch (const std::exception& e) {
    return fail(OCG_ERR_ARG, e.what());
  }
}

int ocg_model_create_from_nlp(const ocg_nlp_desc* d, ocg_model** out) {
  if (!d || !out) return fail(OCG_ERR_ARG, "null argument");
  try {
    auto m = std::make_unique<ocg_model>();
    ocg::Nlp& nlp = m->nlp;
    nlp.scheme = d->scheme == 0 ? ocg::Scheme::euler : ocg::Scheme::trapezoid;
    nlp.N = d->N;
    nlp.nvar = d->nvar;
    nlp.m_con = d->m_con;
    nlp.maximize = d->maximize != 0;
    for (int s = 0; s < d->n_slabs; ++s) {
      ocg::Slab sl;
      sl.kind = static_cast<ocg::VarKind>(d->slab_kind[s]);
      sl.dim = d->slab_dim[s];
      sl.base = d->slab_base[s];
      sl.nodes = d->slab_nodes[s];
      nlp.slabs.push_back(sl);
    }
    const auto nv = static_cast<size_t>(d->nvar), mc = static_cast<size_t>(d->m_con);
    auto vec = [](const double* p, size_t n, double fill) {
      return p ? std::vector<double>(p, p + n) : std::vector<double>(n, fill);
    };
    nlp.lvar = vec(d->lvar, nv, -INFINITY);
    nlp.uvar = vec(d->uvar, nv, INFINITY);
    nlp.x_start = vec(d->x_start, nv, 0.0);
    nlp.clip_lo = d->clip_lo ? vec(d->clip_lo, nv, 0.0) : nlp.lvar;
    nlp.clip_hi = d->clip_hi ? vec(d->clip_hi, nv, 0.0) : nlp.uvar;
    nlp.lcon = vec(d->lcon, mc, 0.0);
    nlp.ucon = vec(d->ucon, mc, 0.0);
    auto group = [](const ocg_group_desc& gd, bool objective) {
      ocg::Group g;
      g.kind = static_cast<ocg::Group::Kind>(objective ? 1 : gd.kind);
      for (int i = 0; i < gd.n_inputs; ++i)
        g.kernel.graph.append_raw_input({gd.input_base[i], gd.input_stride[i]},
                                        gd.input_labels && gd.input_labels[i] ? gd.input_labels[i] : "");
      if (gd.label) g.label = gd.label;
      for (int k = 0; k < gd.n_nodes; ++k) {
        ocg::Node n;
        n.op = static_cast<ocg::Op>(gd.node_op[k]);
        n.a = gd.node_a[k];
        n.b = gd.node_b[k];
        n.c = gd.node_c[k];
        if (n.op > ocg::Op::pow || n.a >= (n.op == ocg::Op::input ? gd.n_inputs : k) || n.b >= k)
          throw std::invalid_argument("group graph is not a topologically ordered kernel::Graph");
        g.kernel.graph.append_raw(n);
      }
      for (int r = 0; r < gd.out_dim; ++r) g.kernel.roots.push_back(gd.roots[r]);
      g.pattern = ocg::sparsity_of(g.kernel);
      if (gd.jac) {
        bool same = static_cast<size_t>(gd.n_jac) == g.pattern.jac.size();
        for (int e = 0; same && e < gd.n_jac; ++e)
          same = g.pattern.jac[static_cast<size_t>(e)] == std::pair<int, int>(gd.jac[2 * e], gd.jac[2 * e + 1]);
        if (!same) throw std::invalid_argument("Jacobian pattern differs from the graph's structural pattern");
      }
      if (gd.hess) {
        bool same = static_cast<size_t>(gd.n_hess) == g.pattern.hess.size();
        for (int e = 0; same && e < gd.n_hess; ++e)
          same = g.pattern.hess[static_cast<size_t>(e)] == std::pair<int, int>(gd.hess[2 * e], gd.hess[2 * e + 1]);
        if (!same) throw std::invalid_argument("Hessian pattern differs from the graph's structural pattern");
      }
      g.range.lo = gd.range_lo;
      g.range.hi = gd.range_hi;
      g.range.endpoints = gd.range_endpoints != 0;
      g.row_base = gd.row_base;
      if (!objective && gd.lower) g.lower.assign(gd.lower, gd.lower + gd.out_dim);
      if (!objective && gd.upper) g.upper.assign(gd.upper, gd.upper + gd.out_dim);
      g.weight = gd.weight;
      return g;
    };
    for (int i = 0; i < d->n_con_groups; ++i) nlp.cons.push_back(group(d->con_groups[i], false));
    for (int i = 0; i < d->n_obj_groups; ++i) nlp.objs.push_back(group(d->obj_groups[i], true));
    *out = m.release();
    return OCG_OK;
  } catch (const std::exception& e) {
    return fail(OCG_ERR_ARG, e.what());
  }
}

void ocg_model_destroy(ocg_model* m) {
  if (!m) return;
  ocg::hd::drop_ipm_plans(m);  // ocg_ipm_solve's cached plans of this model
  delete m;
}
int64_t ocg_model_nvar(const ocg_model* m) { return m ? m->nlp.nvar : -1; }
int64_t ocg_model_mcon(const ocg_model* m) { return m ? m->nlp.m_con : -1; }
int64_t ocg_model_grid(const ocg_model* m) { return m ? m->nlp.N : -1; }

int ocg_model_arrays(const ocg_model* m, double* lvar, double* uvar, double* x_start, double* clip_lo, double* clip_hi,
                     double* lcon, double* ucon) {
  if (!m) return fail(OCG_ERR_ARG, "null model");
  auto cp = [](double* d, const std::vector<double>& v) {
    if (d && !v.empty()) std::memcpy(d, v.data(), v.size() * sizeof(double));
  };
  const auto& n = m->nlp;
  cp(lvar, n.lvar);
  cp(uvar, n.uvar);
  cp(x_start, n.x_start);
  cp(clip_lo, n.clip_lo);
  cp(clip_hi, n.clip_hi);
  cp(lcon, n.lcon);
  cp(ucon, n.ucon);
  return OCG_OK;
}

char* ocg_model_structure_json(const ocg_model* m) {
  if (!m) return nullptr;
  const std::string s = m->nlp.structure_json();
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

int ocg_model_synth_acceptance(const ocg_model* m, uint32_t seed, double* x, double* lambda) {
  if (!m || !x) return fail(OCG_ERR_ARG, "null argument");
  const auto& n = m->nlp;
  std::mt19937 rng(seed);
  for (Index i = 0; i < n.nvar; ++i) {
    double lo = n.clip_lo[static_cast<size_t>(i)], hi = n.clip_hi[static_cast<size_t>(i)];
    if (!std::isfinite(lo) || !std::isfinite(hi)) {
      lo = std::isfinite(lo) ? lo + 0.05 : 0.4;
      hi = std::isfinite(hi) ? hi - 0.05 : 1.2;
      if (lo >= hi) {
        lo = 0.4;
        hi = 1.2;
      }
    } else {
      const double w = hi - lo;
      lo += 0.05 * w;
      hi -= 0.05 * w;
    }
    std::uniform_real_distribution<double> d(lo, hi);
    x[i] = d(rng);
  }
  if (lambda) {
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    for (Index r = 0; r < n.m_con; ++r) lambda[r] = d(rng);
  }
  return OCG_OK;
}

int ocg_synth_uniform(uint32_t seed, double lo, double hi, int64_t n, double* out) {
  if (!out) return fail(OCG_ERR_ARG, "null argument");
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> d(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = d(rng);
  return OCG_OK;
}

// ---- eval ---------------------------------------------------------------------

void ocg_eval_default_options(ocg_eval_options* o) {
  o->device = 0;
  o->fma = 0;
  o->block = 128;
  o->idx_lo = 0;
  o->idx_hi = -1;
  o->specials = 1;
  o->min_blocks = 0;
  o->split_kinds = -1;
  o->input_staging = -1;
}

int ocg_eval_create(const ocg_model* m, const ocg_eval_options* opts, ocg_eval** out) {
  if (!m || !out) return fail(OCG_ERR_ARG, "null argument");
  ocg_eval_options o;
  ocg_eval_default_options(&o);
  if (opts) o = *opts;
  try {
    const bool timing = std::getenv("OCG_TIMING") != nullptr;
    auto tprev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[ocg_eval_create] %-16s %8.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
      tprev = now;
    };
    auto e = std::make_unique<ocg_eval>();
    e->model = m;
    e->device = o.device;
    e->block = o.block > 0 ? o.block : 128;
    ck(cudaSetDevice(o.device), "cudaSetDevice");
    // device properties once per device and process (the query itself takes
    // from milliseconds to a tenth of a second)
    static std::mutex prop_mu;
    static std::map<int, cudaDeviceProp> props;
    cudaDeviceProp prop;
    {
      std::lock_guard<std::mutex> lk(prop_mu);
      auto it = props.find(o.device);
      if (it == props.end()) {
        ck(cudaGetDeviceProperties(&prop, o.device), "cudaGetDeviceProperties");
        props.emplace(o.device, prop);
      } else {
        prop = it->second;
      }
    }
    if (prop.major != 10) return fail(OCG_ERR_CUDA, "octgpu kernels target sm_100a; device is sm_" +
                                                        std::to_string(prop.major) + std::to_string(prop.minor));
    const ocg::Nlp& nlp = m->nlp;
    e->lay = ocg::make_layout(nlp);
    const Index lo = std::max(e->lay.idx_lo, o.idx_lo);
    const Index hi = o.idx_hi < 0 ? e->lay.idx_hi : std::min(e->lay.idx_hi, o.idx_hi);
    e->i0 = lo;
    e->n_main = std::max<Index>(0, hi - lo);
    e->specials = o.specials != 0;

    ocg::GenOptions go;
    go.fma = o.fma != 0;
    go.block = e->block;
    lap("device props");
    std::map<std::string, std::string> cubins;
    ocg::Generated gen =
        generate_budgeted(nlp, e->lay, go, auto_min_blocks(o), o.split_kinds, o.input_staging,
                          static_cast<int>(prop.sharedMemPerMultiprocessor),
                          static_cast<int>(prop.sharedMemPerBlockOptin), nullptr, &cubins);
    go.block = gen.block;
    e->block = go.block;
    e->min_blocks = gen.min_blocks;
    e->slices = gen.slices;
    e->tail = gen.tail;
    e->smem = gen.smem;
    e->prm = gen.params;
    e->set_idx32(gen.idx32);
    lap("generate+compile");
    for (const char* k : kKernelNames) e->mods[k] = loaded_module(cubins.at(k));
    lap("load modules");
    e->k_c = e->mods.at("ocg_c")->kernel("ocg_c");
    e->k_cjac = e->mods.at("ocg_cjac")->kernel("ocg_cjac");
    e->k_hess = e->mods.at("ocg_hess")->kernel("ocg_hess");
    e->k_cjh = e->mods.at("ocg_cjh")->kernel("ocg_cjh");
    e->k_objv = e->mods.at("ocg_objv")->kernel("ocg_objv");
    e->k_grad = e->mods.at("ocg_grad")->kernel("ocg_grad");
    for (auto [k, name] : {std::pair{e->k_c, "ocg_c"}, {e->k_cjac, "ocg_cjac"}, {e->k_hess, "ocg_hess"},
                           {e->k_cjh, "ocg_cjh"}, {e->k_objv, "ocg_objv"}, {e->k_grad, "ocg_grad"}}) {
      const int bytes = e->smem.at(name);
      if (bytes > 48 * 1024)
        ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
           "dynamic shared memory attribute");

      int nb = 0;
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, reinterpret_cast<const void*>(k), e->block, bytes),
         "occupancy");
      e->resident[name] = nb;
    }
    e->sm_count = prop.multiProcessorCount;

    lap("kernel attrs");
    e->jac.alloc(static_cast<size_t>(e->lay.jac_nnz));
    e->hess.alloc(static_cast<size_t>(e->lay.hess_nnz));
    e->grad.alloc(static_cast<size_t>(e->lay.grad_nnz));
    e->objv.alloc(static_cast<size_t>(e->lay.objv_n));
    e->row_scale.upload(std::vector<double>(static_cast<size_t>(nlp.m_con), 1.0));
    e->flag.upload(std::vector<int>{0});
    e->scratch.alloc(4);
    for (const auto& g : nlp.objs) e->obj_weight.push_back(g.weight);
    e->objw.alloc(std::max<size_t>(1, nlp.objs.size()));
    e->refresh_objw(nullptr);

    // objective reduction plan: chunks of 512 per group
    std::vector<int64_t> off, cnt, cbase{0};
    for (size_t g = 0; g < nlp.objs.size(); ++g) {
      off.push_back(e->lay.objv_off[g]);
      cnt.push_back(nlp.objs[g].range.count());
      cbase.push_back(cbase.back() + (cnt.back() + 511) / 512);
    }
    e->n_chunks = cbase.back();
    e->og_off.upload(off);
    e->og_count.upload(cnt);
    e->og_cbase.upload(cbase);
    e->og_weight.upload(e->obj_weight);
    e->partials.alloc(static_cast<size_t>(std::max<Index>(1, e->n_chunks)));

    lap("buffers");
    // dense gradient: per slot, grad COO entries in increasing order
    std::vector<Index> gc;
    host_structure(nlp, nullptr, nullptr, nullptr, nullptr, &gc);
    std::vector<int64_t> ptr(static_cast<size_t>(nlp.nvar) + 1, 0);
    for (Index c : gc) ptr[static_cast<size_t>(c) + 1]++;
    for (Index i = 0; i < nlp.nvar; ++i) ptr[static_cast<size_t>(i) + 1] += ptr[static_cast<size_t>(i)];
    std::vector<int32_t> idx(gc.size());
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (size_t q = 0; q < gc.size(); ++q) idx[static_cast<size_t>(fill[static_cast<size_t>(gc[q])]++)] = static_cast<int32_t>(q);
    e->gg_ptr.upload(ptr);
    e->gg_idx.upload(idx);
    {
      const auto lr = ocg::dev::long_rows(ptr);
      e->gg_long.upload(lr);
      e->n_gg_long = static_cast<int64_t>(lr.size());
    }
    ck(cudaStreamSynchronize(cudaStreamPerThread), "sync");
    lap("gradient gather");
    *out = e.release();
    return OCG_OK;
  } catch (const CudaError& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_JIT, ex.what());
  }
}

void ocg_eval_destroy(ocg_eval* e) {
  if (!e) return;
  ocg::mem::DeviceScope ds(e->device);
  cudaDeviceSynchronize();  // no queued work may still use the buffers
  delete e;
}

int ocg_eval_sizes(const ocg_eval* e, int64_t* jn, int64_t* hn, int64_t* gn) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  if (jn) *jn = e->lay.jac_nnz;
  if (hn) *hn = e->lay.hess_nnz;
  if (gn) *gn = e->lay.grad_nnz;
  return OCG_OK;
}

int ocg_eval_structure(const ocg_eval* e, int64_t* jr, int64_t* jc, int64_t* hr, int64_t* hc, int64_t* gc) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  std::vector<Index> a, b, c, d, g;
  host_structure(e->model->nlp, &a, &b, &c, &d, &g);
  auto cp = [](int64_t* dst, const std::vector<Index>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(Index));
  };
  cp(jr, a);
  cp(jc, b);
  cp(hr, c);
  cp(hc, d);
  cp(gc, g);
  return OCG_OK;
}

double* ocg_eval_buffer(ocg_eval* e, int which) {
  if (!e) return nullptr;
  switch (which) {
    case OCG_BUF_JAC: return e->jac.p;
    case OCG_BUF_HESS: return e->hess.p;
    case OCG_BUF_GRAD: return e->grad.p;
    case OCG_BUF_ROWSCALE: return e->row_scale.p;
    case OCG_BUF_OBJV: return e->objv.p;
  }
  return nullptr;
}

int ocg_eval_bind_buffer(ocg_eval* e, int which, double* dev_ptr) {
  if (!e || !dev_ptr) return fail(OCG_ERR_ARG, "null argument");
  try {
    ocg::mem::DeviceScope ds_(e->device);
    switch (which) {
      case OCG_BUF_JAC: e->jac.bind(dev_ptr); break;
      case OCG_BUF_HESS: e->hess.bind(dev_ptr); break;
      case OCG_BUF_GRAD: e->grad.bind(dev_ptr); break;
      case OCG_BUF_ROWSCALE: {
        const size_t m = static_cast<size_t>(e->model->nlp.m_con);
        if (m) ck(cudaMemcpy(dev_ptr, e->row_scale.p, m * sizeof(double), cudaMemcpyDeviceToDevice), "rs copy");
        e->row_scale.bind(dev_ptr);
        break;
      }
      case OCG_BUF_OBJV: e->objv.bind(dev_ptr); break;
      default: return fail(OCG_ERR_ARG, "unknown buffer");
    }
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_set_scaling(ocg_eval* e, double obj_scale, const double* row_scale) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  try {
    ocg::mem::DeviceScope ds_(e->device);
    const size_t m = static_cast<size_t>(e->model->nlp.m_con);
    std::vector<double> rs(m, 1.0);
    if (row_scale) std::copy(row_scale, row_scale + m, rs.begin());
    if (m) ck(cudaMemcpy(e->row_scale.p, rs.data(), m * sizeof(double), cudaMemcpyHostToDevice), "row_scale");
    e->obj_scale = obj_scale;
    e->refresh_objw(nullptr);
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_get_scaling(ocg_eval* e, double* obj_scale, double* row_scale) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  try {
    ocg::mem::DeviceScope ds_(e->device);
    if (obj_scale) *obj_scale = e->obj_scale;
    const size_t m = static_cast<size_t>(e->model->nlp.m_con);
    if (row_scale && m) ck(cudaMemcpy(row_scale, e->row_scale.p, m * sizeof(double), cudaMemcpyDeviceToHost), "rs");
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

#define OCG_GUARD_BEGIN try {
#define OCG_GUARD_END                          \
  }                                            \
  catch (const std::exception& ex) {           \
    return fail(OCG_ERR_CUDA, ex.what());      \
  }

int ocg_eval_constraints(ocg_eval* e, const double* x, double* c, ocg_stream s) {
  if (!e || !x || !c) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const double* rs = e->row_scale.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_c");
  void* args[] = {e->prm_arg(), &x, &rs, &c, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_c, "ocg_c", args, st(s));
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_constraints_jacobian(ocg_eval* e, const double* x, double* c, ocg_stream s) {
  if (!e || !x || !c) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const double* rs = e->row_scale.p;
  double* jac = e->jac.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_cjac");
  void* args[] = {e->prm_arg(), &x, &rs, &c, &jac, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_cjac, "ocg_cjac", args, st(s));
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_hessian(ocg_eval* e, const double* x, const double* lambda, ocg_stream s) {
  if (!e || !x || !lambda) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const double* rs = e->row_scale.p;
  const double* ow = e->objw.p;
  double* hess = e->hess.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_hess");
  void* args[] = {e->prm_arg(), &x, &lambda, &rs, &ow, &hess, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_hess, "ocg_hess", args, st(s));
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_jac_hess(ocg_eval* e, const double* x, const double* lambda, double* c, ocg_stream s) {
  if (!e || !x || !lambda || !c) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const double* rs = e->row_scale.p;
  const double* ow = e->objw.p;
  double* jac = e->jac.p;
  double* hess = e->hess.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_cjh");
  void* args[] = {e->prm_arg(), &x, &lambda, &rs, &ow, &c, &jac, &hess, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_cjh, "ocg_cjh", args, st(s));
  return OCG_OK;
  OCG_GUARD_END
}

namespace {

// One COO / c segment a node range writes: (buffer 0 = c, 1 = jac, 2 = hess,
// offset, count). Groups are laid out group-major, instance-major inside a
// group (eval.cpp:44-119), so a range's outputs are one segment per group
// and output kind; tail groups (endpoint pairs, boundary kind) go with the
// chunk that runs the specials.
struct OutSeg {
  int buf;
  Index off, n;
};

std::vector<OutSeg> range_segments(const ocg::Nlp& nlp, const ocg::Layout& L, Index a, Index b, bool specials) {
  std::vector<OutSeg> v;
  auto span = [&](const ocg::Group& g, Index& k0, Index& k1) {
    const bool tail = g.range.endpoints || g.kind == ocg::Group::Kind::boundary;
    if (tail) {
      k0 = 0;
      k1 = specials ? g.range.count() : 0;
    } else {
      k0 = std::max<Index>(0, std::max(g.range.lo, a) - g.range.lo);
      k1 = std::max<Index>(0, std::min(g.range.hi, b) - g.range.lo);
    }
  };
  for (size_t gi = 0; gi < nlp.cons.size(); ++gi) {
    const ocg::Group& g = nlp.cons[gi];
    Index k0 = 0, k1 = 0;
    span(g, k0, k1);
    if (k1 <= k0) continue;
    const Index od = g.out_dim(), nj = static_cast<Index>(g.pattern.jac.size()),
                nh = static_cast<Index>(g.pattern.hess.size());
    v.push_back({0, g.row_base + k0 * od, (k1 - k0) * od});
    if (nj) v.push_back({1, L.jac_off[gi] + k0 * nj, (k1 - k0) * nj});
    if (nh) v.push_back({2, L.hess_off_con[gi] + k0 * nh, (k1 - k0) * nh});
  }
  for (size_t gi = 0; gi < nlp.objs.size(); ++gi) {
    const ocg::Group& g = nlp.objs[gi];
    Index k0 = 0, k1 = 0;
    span(g, k0, k1);
    const Index nh = static_cast<Index>(g.pattern.hess.size());
    if (k1 > k0 && nh) v.push_back({2, L.hess_off_obj[gi] + k0 * nh, (k1 - k0) * nh});
  }
  // adjacent segments of one buffer merged (fewer, larger copies)
  std::sort(v.begin(), v.end(), [](const OutSeg& p, const OutSeg& q) { return p.buf != q.buf ? p.buf < q.buf : p.off < q.off; });
  std::vector<OutSeg> m;
  for (const OutSeg& sg : v) {
    if (!m.empty() && m.back().buf == sg.buf && m.back().off + m.back().n == sg.off)
      m.back().n += sg.n;
    else
      m.push_back(sg);
  }
  return m;
}

}  // namespace

int ocg_eval_jac_hess_host(ocg_eval* e, const double* x, const double* lambda, double* c, double* jac, double* hess,
                           int chunks, int64_t* bytes, ocg_stream s) {
  if (!e || !x || !lambda || !c || !jac || !hess) return fail(OCG_ERR_ARG, "null argument");
  if (e->shard) return fail(OCG_ERR_ARG, "ocg_eval_jac_hess_host: a sharded context uploads its shard (ocg_eval_scatter_x)");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const ocg::Nlp& nlp = e->model->nlp;
  const size_t nv = static_cast<size_t>(nlp.nvar), mc = static_cast<size_t>(nlp.m_con);
  if (!e->host_x.p) {
    e->host_x.alloc(nv);
    e->host_lam.alloc(std::max<size_t>(mc, 1));
    e->host_c.alloc(std::max<size_t>(mc, 1));
    ck(cudaStreamCreateWithFlags(&e->out_stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&e->join_ev, cudaEventDisableTiming), "event");
  }
  const cudaStream_t cs = st(s);
  // chunk boundaries on the 32-node tile grid; the specials with the last
  // chunk (every x node is on the device by then)
  const Index lo = e->i0, hi = e->i0 + e->n_main;
  const Index nch = std::max<Index>(1, std::min<Index>(chunks > 0 ? chunks : 1, (hi - lo + 31) / 32));
  while (static_cast<Index>(e->chunk_ev.size()) < nch) {
    cudaEvent_t ev = nullptr;
    ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    e->chunk_ev.push_back(ev);
  }
  double* const dx = e->host_x.p;
  double* const dl = e->host_lam.p;
  double* const dc = e->host_c.p;
  int64_t moved = 0;
  // x whole first: a chunk's kernels read its right halo and the free
  // variables (tf), and x is the smallest array
  ck(cudaMemcpyAsync(dx, x, nv * sizeof(double), cudaMemcpyHostToDevice, cs), "x h2d");
  moved += static_cast<int64_t>(nv * sizeof(double));
  const double* rs = e->row_scale.p;
  const double* ow = e->objw.p;
  double* dj = e->jac.p;
  double* dh = e->hess.p;
  int* fl = e->flag.p;
  double* const hbuf[3] = {c, jac, hess};
  const double* const dbuf[3] = {dc, dj, dh};
  for (Index q = 0; q < nch; ++q) {
    // [a, b): boundaries on the tile grid
    const Index a = q == 0 ? lo : std::min(hi, lo + ((hi - lo) * q / nch + 31) / 32 * 32);
    const Index b = q + 1 == nch ? hi : std::min(hi, lo + ((hi - lo) * (q + 1) / nch + 31) / 32 * 32);
    const bool last = q + 1 == nch;
    const std::vector<OutSeg> segs = range_segments(nlp, e->lay, a, b, last && e->specials);
    // this chunk's multiplier rows are exactly its c rows
    for (const OutSeg& sg : segs)
      if (sg.buf == 0) {
        ck(cudaMemcpyAsync(dl + sg.off, lambda + sg.off, static_cast<size_t>(sg.n) * sizeof(double),
                            cudaMemcpyHostToDevice, cs),
            "lambda h2d");
        moved += sg.n * static_cast<int64_t>(sizeof(double));
      }
    Index i0 = a, nm = b - a;
    Index ns = last ? e->n_spec("ocg_cjh") : 0;
    const double* xin = dx;
    const double* lin = dl;
    double* cout = dc;
    void* args[] = {e->prm_arg(), &xin, &lin, &rs, &ow, &cout, &dj, &dh, &fl, &i0, &nm, &ns, &kNoBatch};
    e->launch_range(e->k_cjh, "ocg_cjh", args, cs, nm, ns);
    ck(cudaEventRecord(e->chunk_ev[static_cast<size_t>(q)], cs), "record");
    ck(cudaStreamWaitEvent(e->out_stream, e->chunk_ev[static_cast<size_t>(q)], 0), "wait");
    for (const OutSeg& sg : segs) {
      ck(cudaMemcpyAsync(hbuf[sg.buf] + sg.off, dbuf[sg.buf] + sg.off, static_cast<size_t>(sg.n) * sizeof(double),
                          cudaMemcpyDeviceToHost, e->out_stream),
          "d2h");
      moved += sg.n * static_cast<int64_t>(sizeof(double));
    }
  }
  // the caller's stream is done when the last copy out is
  ck(cudaEventRecord(e->join_ev, e->out_stream), "record");
  ck(cudaStreamWaitEvent(cs, e->join_ev, 0), "wait");
  if (bytes) *bytes = moved;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_objective(ocg_eval* e, const double* x, double* f, ocg_stream s) {
  if (!e || !x || !f) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  double* ov = e->objv.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_objv");
  void* args[] = {e->prm_arg(), &x, &ov, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_objv, "ocg_objv", args, st(s));
  ocg::dev::objective_reduce(e->objv.p, e->og_off.p, e->og_count.p, e->og_cbase.p, e->n_chunks, e->og_weight.p,
                             static_cast<int>(e->obj_weight.size()), e->obj_scale, e->partials.p, f, e->flag.p, st(s));
  e->launches += 2;
  return OCG_OK;
  OCG_GUARD_END
}

int64_t ocg_eval_objective_chunks(const ocg_eval* e) { return e ? e->n_chunks : -1; }

int ocg_eval_objective_partials(ocg_eval* e, const double* x, double* partials, ocg_stream s) {
  if (!e || !x || !partials) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  double* ov = e->objv.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_objv");
  void* args[] = {e->prm_arg(), &x, &ov, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_objv, "ocg_objv", args, st(s));
  ocg::dev::objective_chunk_sums(e->objv.p, e->og_off.p, e->og_count.p, e->og_cbase.p, e->n_chunks,
                                 static_cast<int>(e->obj_weight.size()), partials, st(s));
  e->launches += 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_objective_combine(ocg_eval* e, const double* partials, double* f, ocg_stream s) {
  if (!e || !partials || !f) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  ocg::dev::objective_combine(partials, e->og_cbase.p, e->og_weight.p, static_cast<int>(e->obj_weight.size()),
                              e->obj_scale, f, e->flag.p, st(s));
  e->launches += 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_gradient(ocg_eval* e, const double* x, double* grad_dense, ocg_stream s) {
  if (!e || !x || !grad_dense) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const double* ow = e->objw.p;
  double* g = e->grad.p;
  int* fl = e->flag.p;
  Index ns = e->n_spec("ocg_grad");
  void* args[] = {e->prm_arg(), &x, &ow, &g, &fl, &e->i0, &e->n_main, &ns, &kNoBatch};
  e->launch(e->k_grad, "ocg_grad", args, st(s));
  ocg::dev::gather_sum(e->grad.p, e->gg_ptr.p, e->gg_idx.p, e->model->nlp.nvar, grad_dense,
                       {e->gg_long.p, e->n_gg_long}, st(s));
  e->launches += 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_max_abs_hessian(ocg_eval* e, double* out, ocg_stream s) {
  if (!e || !out) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  ocg::dev::max_abs(e->hess.p, e->lay.hess_nnz, out, st(s));
  e->launches += 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_status(ocg_eval* e, ocg_stream s) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  int h = 0;
  ck(cudaMemcpyAsync(&h, e->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st(s)), "flag d2h");
  ck(cudaStreamSynchronize(st(s)), "sync");
  if (h) {
    ck(cudaMemsetAsync(e->flag.p, 0, sizeof(int), st(s)), "flag reset");
    ck(cudaStreamSynchronize(st(s)), "sync");
    return OCG_EVAL_DOMAIN;
  }
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_eval_status_async(ocg_eval* e, int* host_flag, ocg_stream s) {
  if (!e || !host_flag) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  ck(cudaMemcpyAsync(host_flag, e->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st(s)), "flag d2h");
  ck(cudaMemsetAsync(e->flag.p, 0, sizeof(int), st(s)), "flag reset");
  return OCG_OK;
  OCG_GUARD_END
}

int64_t ocg_eval_launch_count(const ocg_eval* e) { return e ? e->launches : -1; }

// EvalContext::compute_scaling (eval.cpp:266-286): gradient and Jacobian at x0
// with unit scales on the device, the max-abs rules on the host.
int ocg_eval_compute_scaling(ocg_eval* e, const double* x0, int enabled, ocg_stream s) {
  if (!e || !x0) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(e->device);
  const auto& nlp = e->model->nlp;
  const size_t m = static_cast<size_t>(nlp.m_con), nv = static_cast<size_t>(nlp.nvar);
  int rc = ocg_eval_set_scaling(e, 1.0, nullptr);
  if (rc != OCG_OK || !enabled) return rc;
  DBuf<double> gd, cd;
  gd.alloc(nv);
  cd.alloc(m);
  ocg_eval_gradient(e, x0, gd.p, s);
  if (ocg_eval_status(e, s) != OCG_OK) return OCG_OK;  // keep unit scales
  ocg_eval_constraints_jacobian(e, x0, cd.p, s);
  if (ocg_eval_status(e, s) != OCG_OK) return OCG_OK;
  // the max rules on the device: max|grad| and per-row max|J| (exact)
  const cudaStream_t cs = st(s);
  DBuf<double> gm;
  gm.alloc(1);
  ocg::dev::max_abs(gd.p, static_cast<int64_t>(nv), gm.p, cs);
  double gmax = 0.0;
  ck(cudaMemcpyAsync(&gmax, gm.p, sizeof(double), cudaMemcpyDeviceToHost, cs), "gmax d2h");
  double os = 1.0;
  if (gmax > 0.0) os = std::min(1.0, 100.0 / gmax);
  DBuf<int64_t> djr, djc;
  device_structure(nlp, &djr, &djc, nullptr, nullptr, cs);
  DBuf<double> jmax;
  jmax.alloc(m);
  ck(cudaMemsetAsync(jmax.p, 0, std::max<size_t>(m, 1) * sizeof(double), cs), "memset");
  ocg::dev::row_absmax(e->jac.p, djr.p, static_cast<int64_t>(djr.n), jmax.p, cs);
  ocg::dev::row_scale_rule(jmax.p, static_cast<int64_t>(m), e->row_scale.p, cs);
  ck(cudaStreamSynchronize(cs), "scaling sync");
  e->obj_scale = os;
  e->refresh_objw(nullptr);
  return OCG_OK;
  OCG_GUARD_END
}

// ---- KKT ----------------------------------------------------------------------

int ocg_kkt_create(const ocg_model* mdl, ocg_eval* e, ocg_kkt** out) {
  if (!mdl || !e || !out) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  const bool timing = std::getenv("OCG_TIMING") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ocg_kkt_create] %-16s %8.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
    tprev = now;
  };
  const ocg::Nlp& nlp = mdl->nlp;
  auto K = std::make_unique<ocg_kkt>();
  K->ev = e;
  K->nvar = nlp.nvar;
  K->m_con = nlp.m_con;
  const auto nv = static_cast<size_t>(nlp.nvar), mc = static_cast<size_t>(nlp.m_con);

  // Reduction (eval.cpp:290-316): fold rows whose root is a bare input
  K->xlo = nlp.lvar;
  K->xhi = nlp.uvar;
  K->row_slot.assign(mc, -1);
  for (const auto& g : nlp.cons) {
    const auto& gr = g.kernel.graph;
    for (int r = 0; r < g.out_dim(); ++r) {
      const ocg::Node& root = gr.at(g.kernel.roots[static_cast<size_t>(r)]);
      if (root.op != ocg::Op::input) continue;
      const ocg::Addr a = gr.inputs()[static_cast<size_t>(root.a)];
      for (Index k = 0; k < g.range.count(); ++k) {
        const auto row = static_cast<size_t>(g.row_base + k * g.out_dim() + r);
        const auto slot = static_cast<size_t>(a.slot(g.range.at(k)));
        K->row_slot[row] = static_cast<Index>(slot);
        K->xlo[slot] = std::max(K->xlo[slot], nlp.lcon[row]);
        K->xhi[slot] = std::min(K->xhi[slot], nlp.ucon[row]);
        if (K->xlo[slot] > K->xhi[slot]) K->contradictory = true;
      }
    }
  }
  K->dual_index.assign(mc, -1);
  for (size_t r = 0; r < mc; ++r) {
    if (K->row_slot[r] >= 0) continue;
    K->dual_index[r] = K->m++;
    K->dual_row.push_back(static_cast<Index>(r));
  }
  lap("reduction");
  // KktAssembler (eval.cpp:318-403)
  K->prim_index.assign(nv, -1);
  for (size_t s = 0; s < nv; ++s) {
    if (K->xlo[s] == K->xhi[s]) continue;
    K->prim_index[s] = K->n_free++;
    K->free_slot.push_back(static_cast<Index>(s));
  }
  K->slack_index.assign(mc, -1);
  for (size_t r = 0; r < mc; ++r) {
    if (K->dual_index[r] < 0 || nlp.lcon[r] == nlp.ucon[r]) continue;
    K->slack_index[r] = K->n_slack++;
    K->slack_of.push_back(static_cast<Index>(r));
  }
  K->ntot = K->n_free + K->n_slack;
  K->dim = K->ntot + K->m;

  lap("maps");
  DBuf<int64_t> dhr, dhc, djr, djc;
  device_structure(nlp, &djr, &djc, &dhr, &dhc, cudaStreamPerThread);
  K->H = static_cast<Index>(dhr.n);
  K->J = static_cast<Index>(djr.n);
  lap("structure");
  // pattern, assembly sources, matvec CSR and J^T lambda gather: sorted on
  // the device (kktbuild.cu); sources keep the reference's accumulation order
  {
    std::vector<int64_t> sd(static_cast<size_t>(K->n_slack));
    for (Index k = 0; k < K->n_slack; ++k)
      sd[static_cast<size_t>(k)] = K->dual_index[static_cast<size_t>(K->slack_of[static_cast<size_t>(k)])];
    DBuf<int64_t> dprim, ddual;
    dprim.upload(K->prim_index);
    ddual.upload(K->dual_index);
    K->jt_slack_dual.upload(sd);
    ocg::dev::KktBuildIn bi;
    bi.hr = dhr.p;
    bi.hc = dhc.p;
    bi.jr = djr.p;
    bi.jc = djc.p;
    bi.H = K->H;
    bi.J = K->J;
    bi.prim = dprim.p;
    bi.dual = ddual.p;
    bi.slack_dual = K->jt_slack_dual.p;
    bi.n_free = K->n_free;
    bi.n_slack = K->n_slack;
    bi.m = K->m;
    ocg::dev::KktBuildOut bo;
    ocg::dev::build_kkt(bi, cudaStreamPerThread, bo);
    K->colp = std::move(bo.colp);
    K->rowi = std::move(bo.rowi);
    K->nnz = bo.nnz;
    K->src_ptr.adopt(bo.src_ptr, static_cast<size_t>(bo.nnz) + 1);
    K->src_code.adopt(bo.src_code, static_cast<size_t>(bo.ncode));
    K->mv_ptr.adopt(bo.mv_ptr, static_cast<size_t>(K->dim) + 1);
    K->mv_col.adopt(bo.mv_col, 0);
    K->mv_vidx.adopt(bo.mv_vidx, 0);
    K->jt_ptr.adopt(bo.jt_ptr, static_cast<size_t>(K->ntot) + 1);
    K->jt_e.adopt(bo.jt_e, 0);
    K->jt_dual.adopt(bo.jt_dual, 0);
  }
  {
    // long rows of the three gathers (a free final time's diagonal, J^T lambda entry, matvec row)
    auto longs = [&](const DBuf<int64_t>& ptr, size_t n, DBuf<int64_t>& out, int64_t& count) {
      out.alloc(n);
      count = ocg::dev::long_rows_device(ptr.p, static_cast<int64_t>(n), out.p, cudaStreamPerThread);
    };
    longs(K->src_ptr, static_cast<size_t>(K->nnz), K->src_long, K->n_src_long);
    longs(K->mv_ptr, static_cast<size_t>(K->dim), K->mv_long, K->n_mv_long);
    longs(K->jt_ptr, static_cast<size_t>(K->ntot), K->jt_long, K->n_jt_long);
    K->mv_long_part.alloc(static_cast<size_t>(K->n_mv_long) * ocg::dev::kLongBlocks);
    K->jt_long_part.alloc(static_cast<size_t>(K->n_jt_long) * ocg::dev::kLongBlocks);
  }
  // compact single-source codes for the assembly (kernels.hpp kkt_code32);
  // slots in slot order (see kkt_assemble_fast_k for the source-order A/B)
  K->src_code32.alloc(static_cast<size_t>(std::max<Index>(1, K->nnz)));
  if (!ocg::dev::kkt_code32(K->src_ptr.p, K->src_code.p, K->nnz, K->H, K->J, K->n_slack, K->ntot, K->src_code32.p,
                            cudaStreamPerThread))
    K->src_code32.release();
  // 32-bit copies of the matvec / J^T lambda indices (values < nnz_K, dim, nnz_J, m)
  if (K->nnz < (Index{1} << 31) && K->dim < (Index{1} << 31) && K->J < (Index{1} << 31) &&
      !(std::getenv("OCG_IDX64") && std::atoi(std::getenv("OCG_IDX64")) != 0)) {
    int64_t nmv = 0, njt = 0;
    ck(cudaMemcpyAsync(&nmv, K->mv_ptr.p + K->dim, sizeof(int64_t), cudaMemcpyDeviceToHost, cudaStreamPerThread), "mv n");
    ck(cudaMemcpyAsync(&njt, K->jt_ptr.p + K->ntot, sizeof(int64_t), cudaMemcpyDeviceToHost, cudaStreamPerThread), "jt n");
    ck(cudaStreamSynchronize(cudaStreamPerThread), "sync");
    K->mv_col32.alloc(static_cast<size_t>(std::max<int64_t>(1, nmv)));
    K->mv_vidx32.alloc(static_cast<size_t>(std::max<int64_t>(1, nmv)));
    K->jt_e32.alloc(static_cast<size_t>(std::max<int64_t>(1, njt)));
    K->jt_dual32.alloc(static_cast<size_t>(std::max<int64_t>(1, njt)));
    ocg::dev::narrow_i32(K->mv_col.p, nmv, K->mv_col32.p, cudaStreamPerThread);
    ocg::dev::narrow_i32(K->mv_vidx.p, nmv, K->mv_vidx32.p, cudaStreamPerThread);
    ocg::dev::narrow_i32(K->jt_e.p, njt, K->jt_e32.p, cudaStreamPerThread);
    ocg::dev::narrow_i32(K->jt_dual.p, njt, K->jt_dual32.p, cudaStreamPerThread);
  }
  // tiled assembly: one source stream per COO group of hess and jac, and sigma
  if (K->src_code32.p && !(std::getenv("OCG_KKT_TILED") && std::atoi(std::getenv("OCG_KKT_TILED")) == 0)) {
    const ocg::Layout& lay = e->lay;
    std::vector<int64_t> sb;
    for (Index o : lay.hess_off_con) sb.push_back(o);
    for (Index o : lay.hess_off_obj) sb.push_back(o);
    for (Index o : lay.jac_off) sb.push_back(K->H + o);
    sb.push_back(K->H + K->J + K->n_slack);
    sb.push_back(K->H + K->J + K->n_slack + K->ntot);
    bool sorted = std::is_sorted(sb.begin(), sb.end()) && !sb.empty() && sb.front() == 0;
    if (sorted) {
      K->t_sb.alloc(sb.size());
      ck(cudaMemcpyAsync(K->t_sb.p, sb.data(), sb.size() * sizeof(int64_t), cudaMemcpyHostToDevice, cudaStreamPerThread),
         "stream bounds");
      ocg::dev::KktTiles t;
      const Index ncode = static_cast<Index>(K->src_code.n);
      if (ocg::dev::kkt_tile_plan(K->src_code32.p, K->src_ptr.p, K->src_code.p, K->nnz, ncode, K->t_sb.p,
                                  static_cast<int>(sb.size()) - 1, K->H, K->J, K->n_slack, K->ntot, t,
                                  cudaStreamPerThread)) {
        const size_t nw = static_cast<size_t>(t.ntile) * static_cast<size_t>(t.ns);
        K->t_wlo.adopt(t.wlo, nw);
        K->t_wlen.adopt(t.wlen, nw);
        K->t_woff.adopt(t.woff, nw);
        K->t_code32.adopt(t.code32, static_cast<size_t>(K->nnz));
        K->t_mcode.adopt(t.mcode, static_cast<size_t>(std::max<Index>(1, ncode)));
        K->tiles = t;
      }
    }
  }
  K->val.alloc(static_cast<size_t>(K->nnz));
  ck(cudaMemsetAsync(K->val.p, 0, static_cast<size_t>(K->nnz) * sizeof(double), cudaStreamPerThread), "memset");
  ck(cudaStreamSynchronize(cudaStreamPerThread), "sync");
  lap("jt gather");
  *out = K.release();
  return OCG_OK;
  OCG_GUARD_END
}

void ocg_kkt_destroy(ocg_kkt* k) {
  if (!k) return;
  ocg::mem::DeviceScope ds(k->ev->device);
  cudaDeviceSynchronize();
  delete k;
}

int ocg_kkt_dims(const ocg_kkt* k, int64_t* out) {
  if (!k || !out) return fail(OCG_ERR_ARG, "null argument");
  out[0] = k->n_free;
  out[1] = k->n_slack;
  out[2] = k->ntot;
  out[3] = k->m;
  out[4] = k->dim;
  out[5] = k->nnz;
  out[6] = k->contradictory ? 1 : 0;
  return OCG_OK;
}

int ocg_kkt_pattern(const ocg_kkt* k, int64_t* colp, int64_t* rowi) {
  if (!k) return fail(OCG_ERR_ARG, "null kkt");
  if (colp) std::memcpy(colp, k->colp.data(), k->colp.size() * sizeof(Index));
  if (rowi && !k->rowi.empty()) std::memcpy(rowi, k->rowi.data(), k->rowi.size() * sizeof(Index));
  return OCG_OK;
}

int ocg_kkt_maps(const ocg_kkt* k, int64_t* prim_index, int64_t* slack_index, int64_t* dual_index, int64_t* row_slot,
                 double* xlo, double* xhi) {
  if (!k) return fail(OCG_ERR_ARG, "null kkt");
  auto cpi = [](int64_t* d, const std::vector<Index>& v) {
    if (d && !v.empty()) std::memcpy(d, v.data(), v.size() * sizeof(Index));
  };
  auto cpd = [](double* d, const std::vector<double>& v) {
    if (d && !v.empty()) std::memcpy(d, v.data(), v.size() * sizeof(double));
  };
  cpi(prim_index, k->prim_index);
  cpi(slack_index, k->slack_index);
  cpi(dual_index, k->dual_index);
  cpi(row_slot, k->row_slot);
  cpd(xlo, k->xlo);
  cpd(xhi, k->xhi);
  return OCG_OK;
}

double* ocg_kkt_values(ocg_kkt* k) { return k ? k->val.p : nullptr; }

int ocg_kkt_assemble(ocg_kkt* k, const double* sigma, ocg_stream s) {
  if (!k || !sigma) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(k->ev->device);
  if (k->tiles.ntile > 0)
    ocg::dev::kkt_assemble_tiled(k->ev->hess.p, k->ev->jac.p, sigma, k->src_ptr.p, k->src_code.p, k->nnz, k->H, k->J,
                                 k->n_slack, k->ntot, k->val.p, {k->src_long.p, k->n_src_long}, k->tiles, st(s));
  else
    ocg::dev::kkt_assemble(k->ev->hess.p, k->ev->jac.p, sigma, k->src_ptr.p, k->src_code.p, k->nnz, k->H, k->J,
                           k->n_slack, k->ntot, k->val.p, {k->src_long.p, k->n_src_long}, st(s), k->src_code32.p,
                           k->src_order.p);
  k->ev->launches += k->n_src_long > 0 ? 2 : 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_kkt_matvec(ocg_kkt* k, const double* x, double* y, ocg_stream s) {
  if (!k || !x || !y) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(k->ev->device);
  if (k->mv_col32.p)
    ocg::dev::sym_matvec(k->val.p, k->mv_ptr.p, k->mv_col32.p, k->mv_vidx32.p, k->dim, x, y,
                         {k->mv_long.p, k->n_mv_long, k->mv_long_part.p}, st(s));
  else
    ocg::dev::sym_matvec(k->val.p, k->mv_ptr.p, k->mv_col.p, k->mv_vidx.p, k->dim, x, y,
                         {k->mv_long.p, k->n_mv_long, k->mv_long_part.p}, st(s));
  k->ev->launches += k->n_mv_long > 0 ? 3 : 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_kkt_norm_inf(ocg_kkt* k, double* out, ocg_stream s) {
  if (!k || !out) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(k->ev->device);
  if (k->mv_vidx32.p)
    ocg::dev::sym_norm_inf(k->val.p, k->mv_ptr.p, k->mv_vidx32.p, k->dim, out,
                           {k->mv_long.p, k->n_mv_long, k->mv_long_part.p}, st(s));
  else
    ocg::dev::sym_norm_inf(k->val.p, k->mv_ptr.p, k->mv_vidx.p, k->dim, out,
                           {k->mv_long.p, k->n_mv_long, k->mv_long_part.p}, st(s));
  k->ev->launches += k->n_mv_long > 0 ? 3 : 1;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_kkt_jt_lambda(ocg_kkt* k, const double* lambda, double* out, ocg_stream s) {
  if (!k || !lambda || !out) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(k->ev->device);
  if (k->jt_e32.p)
    ocg::dev::jt_lambda(k->ev->jac.p, lambda, k->jt_ptr.p, k->jt_e32.p, k->jt_dual32.p, k->n_free, k->jt_slack_dual.p,
                        k->n_slack, out, {k->jt_long.p, k->n_jt_long, k->jt_long_part.p}, st(s));
  else
    ocg::dev::jt_lambda(k->ev->jac.p, lambda, k->jt_ptr.p, k->jt_e.p, k->jt_dual.p, k->n_free, k->jt_slack_dual.p,
                        k->n_slack, out, {k->jt_long.p, k->n_jt_long, k->jt_long_part.p}, st(s));
  k->ev->launches += k->n_jt_long > 0 ? 3 : 1;
  return OCG_OK;
  OCG_GUARD_END
}

// ---- band LDL^T (band.hpp) ---------------------------------------------------

int ocg_ldl_create(ocg_kkt* k, ocg_ldl** out) {
  int target = 0;  // the band plan's default (band.cu make_band_plan)
  if (const char* e = std::getenv("OCG_LDL_SEGMENTS")) target = std::max(1, std::atoi(e));
  return ocg::hd::ldl_create(k, target, out);
}

}  // extern "C"

int ocg::hd::set_error(int code, const std::string& msg) { return fail(code, msg); }

int ocg::hd::ldl_create(ocg_kkt* k, int target, ocg_ldl** out) {
  if (!k || !out) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  const bool timing = std::getenv("OCG_TIMING") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ocg_ldl_create] %-16s %8.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
    tprev = now;
  };
  const ocg::Nlp& nlp = k->ev->model->nlp;
  // time node of every KKT index: slots by their slab, rows by the last node
  // their Jacobian touches; free variables (and rows touching only them) are
  // the dense border
  std::vector<Index> slot_node(static_cast<size_t>(nlp.nvar), -1);
  for (const auto& sl : nlp.slabs)
    if (sl.nodes > 1)
      for (Index q = 0; q < sl.dim * sl.nodes; ++q) slot_node[static_cast<size_t>(sl.base + q)] = q / sl.dim;
  std::vector<Index> row_node(static_cast<size_t>(nlp.m_con), -1);
  {
    DBuf<int64_t> djr, djc, dsn, drn;
    device_structure(nlp, &djr, &djc, nullptr, nullptr, cudaStreamPerThread);
    dsn.upload(slot_node);
    drn.alloc(row_node.size());
    ocg::dev::row_max_node(djr.p, djc.p, static_cast<int64_t>(djr.n), dsn.p, static_cast<int64_t>(row_node.size()),
                           drn.p, cudaStreamPerThread);
    if (!row_node.empty())
      ck(cudaMemcpyAsync(row_node.data(), drn.p, row_node.size() * sizeof(int64_t), cudaMemcpyDeviceToHost,
                         cudaStreamPerThread),
         "row_node d2h");
    ck(cudaStreamSynchronize(cudaStreamPerThread), "sync");
  }
  std::vector<int64_t> node(static_cast<size_t>(k->dim), -1);
  for (Index i = 0; i < k->n_free; ++i) node[static_cast<size_t>(i)] = slot_node[static_cast<size_t>(k->free_slot[static_cast<size_t>(i)])];
  for (Index q = 0; q < k->n_slack; ++q)
    node[static_cast<size_t>(k->n_free + q)] = row_node[static_cast<size_t>(k->slack_of[static_cast<size_t>(q)])];
  for (Index d = 0; d < k->m; ++d)
    node[static_cast<size_t>(k->ntot + d)] = row_node[static_cast<size_t>(k->dual_row[static_cast<size_t>(d)])];
  lap("node map");
  auto L = std::make_unique<ocg_ldl>();
  L->kkt = k;
  {
    // the O(nnz) parts of the plan on the device
    DBuf<int64_t> dcolp, drowi;
    dcolp.upload(k->colp);
    drowi.upload(k->rowi);
    ocg::DeviceCsc csc;
    csc.colp = dcolp.p;
    csc.rowi = drowi.p;
    csc.nnz = static_cast<int64_t>(k->rowi.size());
    csc.stream = cudaStreamPerThread;
    int64_t* ddst = nullptr;
    L->plan = ocg::make_band_plan(k->dim, node, k->colp, k->rowi, k->ntot, target, &csc, &ddst);
    L->dst.adopt(ddst, static_cast<size_t>(csc.nnz));
  }
  lap("band plan");
  const ocg::BandPlan& P = L->plan;
  L->perm.upload(P.perm);
  L->primal.upload(P.primal);
  L->border_pos.upload(P.border_pos.empty() ? std::vector<int64_t>{-1} : P.border_pos);
  L->segs.upload(P.segs);
  L->buf.alloc(static_cast<size_t>(std::max<int64_t>(1, P.buf_len)));
  L->Dinv.alloc(static_cast<size_t>(std::max<int64_t>(1, k->dim)));
  L->work.alloc(static_cast<size_t>(std::max<int64_t>(1, k->dim + static_cast<int64_t>(P.nseg) * P.wmax)));
  L->inertia.alloc(3);
  L->inertia_parts.alloc(static_cast<size_t>(3 * (P.nseg + 1)));
  L->dev.segs = L->segs.p;
  L->dev.dst = L->dst.p;
  L->dev.perm = L->perm.p;
  L->dev.primal = L->primal.p;
  L->dev.border_pos = L->border_pos.p;
  const char* sep_mode = std::getenv("OCG_SEP");  // "band": the separator system as one band block
  if (P.nseg > 1 && !(sep_mode && std::string(sep_mode) == "band")) {
    L->cr.alloc(static_cast<size_t>(ocg::dev::cr_length(P.nseg - 1, P.b, P.wg)));
    L->crparts.alloc(static_cast<size_t>(3 * (P.nseg - 1)));
    L->dev.cr = L->cr.p;
    L->dev.crparts = L->crparts.p;
  }
  lap("buffers");
  *out = L.release();
  return OCG_OK;
  OCG_GUARD_END
}

namespace {

// the reference-order factorization's plan (refldl.hpp) on the device
std::unique_ptr<ocg_ldl::Ref> make_ref_ldl(ocg_kkt* k) {
  auto R = std::make_unique<ocg_ldl::Ref>();
  R->S = ocg::rl::analyze(k->dim, k->colp.data(), k->rowi.data(), k->n_free, k->ntot);
  const ocg::rl::HostPlan H = ocg::rl::build_plan(R->S, k->colp.data(), k->rowi.data());
  R->nleaf = static_cast<int64_t>(H.lf_pos.size());
  R->nnl = static_cast<int64_t>(H.nl_pos.size());
  auto up64 = [](DBuf<int64_t>& b, const std::vector<int64_t>& v) { b.upload(v.empty() ? std::vector<int64_t>{0} : v); };
  auto up32 = [](DBuf<int32_t>& b, const std::vector<int32_t>& v) { b.upload(v.empty() ? std::vector<int32_t>{0} : v); };
  up64(R->nl_pos, H.nl_pos);
  up64(R->nl_lp, H.nl_lp);
  up64(R->nl_foff, H.nl_foff);
  up64(R->nl_soff, H.nl_soff);
  up64(R->nl_voff, H.nl_voff);
  up64(R->sc_ptr, H.sc_ptr);
  up64(R->lf_pos, H.lf_pos);
  up64(R->lf_aoff, H.lf_aoff);
  up64(R->pa_ptr, H.pa_ptr);
  up64(R->fl_ptr, H.fl_ptr);
  up64(R->fl_lx, H.fl_lx);
  up64(R->fl_col, H.fl_col);
  up64(R->Lp, R->S.Lp);
  up64(R->Li, R->S.Li);
  up64(R->sc_dst, H.sc_dst);
  up64(R->sc_dpos, H.sc_dpos);
  up64(R->sc_ms, H.sc_ms);
  up64(R->perm, R->S.perm);
  up32(R->nl_f, H.nl_f);
  up32(R->sc_child, H.sc_child);
  up32(R->lf_f, H.lf_f);
  up32(R->pa_j, H.pa_j);
  up32(R->pa_leaf, H.pa_leaf);
  up32(R->fl_j, H.fl_j);
  up32(R->rel, H.rel);
  R->primal.upload(H.primal.empty() ? std::vector<int8_t>{0} : H.primal);
  R->rec.upload(H.rec.empty() ? std::vector<ocg::rl::ColRec>(1) : H.rec);
  const size_t dim = static_cast<size_t>(std::max<int64_t>(1, k->dim));
  R->W.alloc(static_cast<size_t>(H.w_len));
  R->stash.alloc(static_cast<size_t>(H.stash_len));
  R->D.alloc(dim);
  R->Dinv.alloc(dim);
  R->Lx.alloc(static_cast<size_t>(std::max<int64_t>(1, H.lnz)));
  R->y.alloc(dim);
  R->xp.alloc(dim);
  R->V.alloc(static_cast<size_t>(H.v_len));
  R->Vs.alloc(static_cast<size_t>(H.stash_len));
  R->inertia.alloc(3);
  const size_t nnl = static_cast<size_t>(std::max<int64_t>(1, R->nnl));
  R->sr.alloc(nnl * 8);
  R->ypre.alloc(nnl + 2);  // + the double a rounded-up bulk copy reads past the end
  R->ych.alloc(nnl + 2);
  R->chunk_foff.upload(H.chunk_foff);
  up64(R->fl_all_ptr, H.fl_all_ptr);
  up32(R->pre_long, H.pre_long);
  ocg::rl::Dev& d = R->dev;
  d.dim = H.dim;
  d.nnz = H.nnz;
  d.lnz = H.lnz;
  d.nleaf = R->nleaf;
  d.nnl = R->nnl;
  d.npa = static_cast<int64_t>(H.pa_j.size());
  d.nfl = static_cast<int64_t>(H.fl_j.size());
  d.fmax = H.fmax;
  d.rec = R->rec.p;
  d.nl_pos = R->nl_pos.p;
  d.nl_lp = R->nl_lp.p;
  d.nl_f = R->nl_f.p;
  d.nl_foff = R->nl_foff.p;
  d.nl_soff = R->nl_soff.p;
  d.nl_voff = R->nl_voff.p;
  d.sc_ptr = R->sc_ptr.p;
  d.sc_child = R->sc_child.p;
  d.lf_pos = R->lf_pos.p;
  d.lf_f = R->lf_f.p;
  d.lf_aoff = R->lf_aoff.p;
  d.pa_j = R->pa_j.p;
  d.pa_ptr = R->pa_ptr.p;
  d.pa_leaf = R->pa_leaf.p;
  d.fl_j = R->fl_j.p;
  d.fl_ptr = R->fl_ptr.p;
  d.fl_lx = R->fl_lx.p;
  d.fl_col = R->fl_col.p;
  d.Lp = R->Lp.p;
  d.Li = R->Li.p;
  d.rel = R->rel.p;
  d.sc_dst = R->sc_dst.p;
  d.sc_dpos = R->sc_dpos.p;
  d.sc_ms = R->sc_ms.p;
  d.perm = R->perm.p;
  d.primal = R->primal.p;
  d.w_len = H.w_len;
  d.fronts_len = H.fronts_len;
  d.chunk_foff = H.fmax <= 8 ? R->chunk_foff.p : nullptr;
  d.fl_all_ptr = R->fl_all_ptr.p;
  d.pre_long = R->pre_long.p;
  d.npre_long = static_cast<int64_t>(H.pre_long.size());
  d.sr = R->sr.p;
  d.ypre = R->ypre.p;
  d.ych = R->ych.p;
  d.stash_len = H.stash_len;
  d.v_len = H.v_len;
  {
    const std::vector<int32_t> col = ocg::rl::seq_chunks(R->S.Lp);
    if (!col.empty()) {
      std::vector<int32_t> lp(R->S.Lp.begin(), R->S.Lp.end()), li(R->S.Li.begin(), R->S.Li.end());
      up32(R->Lp32, lp);
      up32(R->Li32, li);
      up32(R->sq_col, col);
      d.Lp32 = R->Lp32.p;
      d.Li32 = R->Li32.p;
      d.sq_col = R->sq_col.p;
      d.sq_nchunks = static_cast<int64_t>(col.size()) - 1;
    }
  }
  return R;
}

}  // namespace

extern "C" {

int ocg_ldl_create_ex(ocg_kkt* k, int order, ocg_ldl** out) {
  if (!k || !out) return fail(OCG_ERR_ARG, "null argument");
  if (order == OCG_LDL_BAND) return ocg_ldl_create(k, out);
  if (order != OCG_LDL_REFERENCE) return fail(OCG_ERR_ARG, "ocg_ldl_create_ex: unknown order");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(k->ev->device);
  auto L = std::make_unique<ocg_ldl>();
  L->kkt = k;
  L->plan.dim = k->dim;
  L->ref = make_ref_ldl(k);
  *out = L.release();
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_ldl_order(const ocg_ldl* l) { return l && l->ref ? OCG_LDL_REFERENCE : OCG_LDL_BAND; }

int64_t ocg_ldl_factor_nnz(const ocg_ldl* l) { return l && l->ref ? static_cast<int64_t>(l->ref->S.Li.size()) : 0; }

int ocg_ldl_factors(const ocg_ldl* l, int64_t* perm, int64_t* Lp, int64_t* Li, double* D, double* Lx) {
  if (!l) return fail(OCG_ERR_ARG, "null argument");
  if (!l->ref) return fail(OCG_ERR_STATE, "ocg_ldl_factors: not a reference-order factorization");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(l->kkt->ev->device);
  const auto& R = *l->ref;
  const size_t n = R.S.perm.size(), lnz = R.S.Li.size();
  if (perm) std::copy(R.S.perm.begin(), R.S.perm.end(), perm);
  if (Lp) std::copy(R.S.Lp.begin(), R.S.Lp.end(), Lp);
  if (Li) std::copy(R.S.Li.begin(), R.S.Li.end(), Li);
  ocg::rl::fill_lx(R.dev, R.Lx.p, cudaStreamPerThread);
  ck(cudaDeviceSynchronize(), "sync");
  if (D && n) ck(cudaMemcpy(D, R.D.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D d2h");
  if (Lx && lnz) ck(cudaMemcpy(Lx, R.Lx.p, lnz * sizeof(double), cudaMemcpyDeviceToHost), "Lx d2h");
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_ldl_ref_symbolic(int64_t dim, const int64_t* colp, const int64_t* rowi, int64_t n_free, int64_t ntot,
                         int64_t* perm, int64_t* parent, int64_t* Lp, int64_t* Li, int64_t* lnz) {
  if (dim < 0 || (dim > 0 && (!colp || !rowi)) || n_free < 0 || ntot < n_free || ntot > dim)
    return fail(OCG_ERR_ARG, "ocg_ldl_ref_symbolic: bad arguments");
  try {
    const ocg::rl::Symbolic S = ocg::rl::analyze(dim, colp, rowi, n_free, ntot);
    if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
    if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
    if (Lp) std::copy(S.Lp.begin(), S.Lp.end(), Lp);
    if (Li) std::copy(S.Li.begin(), S.Li.end(), Li);
    if (lnz) *lnz = static_cast<int64_t>(S.Li.size());
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_ARG, std::string("ocg_ldl_ref_symbolic: ") + ex.what());
  }
}

void ocg_ldl_destroy(ocg_ldl* l) {
  if (!l) return;
  ocg::mem::DeviceScope ds(l->kkt->ev->device);
  cudaDeviceSynchronize();
  delete l;
}

int ocg_release_cached_memory(int device) {
  ocg::hd::drop_ipm_plans(nullptr);
  ocg::mem::trim(device);
  return OCG_OK;
}

int ocg_ldl_info(const ocg_ldl* l, int64_t* out) {
  if (!l || !out) return fail(OCG_ERR_ARG, "null argument");
  if (l->ref) {  // reference order: no segments; "bandwidth" = the largest column count of L
    out[0] = l->ref->S.dim;
    out[1] = 0;
    out[2] = l->ref->dev.fmax - 1;
    out[3] = 0;
    out[4] = l->factorizations;
    return OCG_OK;
  }
  out[0] = l->plan.dim;
  out[1] = l->plan.nseg;
  out[2] = l->plan.b;
  out[3] = l->plan.wg;
  out[4] = l->factorizations;
  return OCG_OK;
}

int ocg_ldl_factor(ocg_ldl* l, double delta_w, double delta_c, int64_t* inertia, ocg_stream s) {
  if (!l) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(l->kkt->ev->device);
  if (l->ref) {
    auto& R = *l->ref;
    ocg::rl::factor(R.dev, l->kkt->val.p, delta_w, delta_c, R.W.p, R.stash.p, R.D.p, R.Dinv.p, R.Lx.p, R.inertia.p,
                    st(s));
    l->kkt->ev->launches += 2 + (R.nleaf > 0) + (R.dev.npa > 0) + (R.nnl > 0);
    l->delta_w = delta_w;
    l->delta_c = delta_c;
    ++l->factorizations;
    if (inertia) {
      unsigned long long h[3];
      ck(cudaMemcpyAsync(h, R.inertia.p, sizeof h, cudaMemcpyDeviceToHost, st(s)), "inertia d2h");
      ck(cudaStreamSynchronize(st(s)), "sync");
      for (int i = 0; i < 3; ++i) inertia[i] = static_cast<int64_t>(h[i]);
    }
    return OCG_OK;
  }
  const ocg::BandPlan& P = l->plan;
  ocg::dev::band_assemble(P, l->dev, l->kkt->val.p, l->buf.p, st(s));
  ocg::dev::band_factor(P, l->dev, l->buf.p, delta_w, delta_c, l->Dinv.p, l->inertia_parts.p, l->inertia.p, st(s));
  l->kkt->ev->launches += P.nseg > 1 ? 7 : 4;
  l->delta_w = delta_w;
  l->delta_c = delta_c;
  ++l->factorizations;
  if (inertia) {
    long long h[3];
    ck(cudaMemcpyAsync(h, l->inertia.p, sizeof h, cudaMemcpyDeviceToHost, st(s)), "inertia d2h");
    ck(cudaStreamSynchronize(st(s)), "sync");
    for (int i = 0; i < 3; ++i) inertia[i] = h[i];
  }
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_ldl_factor_many(ocg_ldl* l, int n, const double* delta_w, const double* delta_c, int64_t* inertia,
                        ocg_stream s) {
  if (!l || n < 1 || !delta_w || !delta_c || !inertia) return fail(OCG_ERR_ARG, "null argument");
  if (!l->ref) {
    if (n != 1) return fail(OCG_ERR_ARG, "ocg_ldl_factor_many: the band order takes one candidate");
    return ocg_ldl_factor(l, delta_w[0], delta_c[0], inertia, s);
  }
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(l->kkt->ev->device);
  auto& R = *l->ref;
  const cudaStream_t s0 = st(s);
  const ocg::rl::Dev& d0 = R.dev;
  while (static_cast<int>(R.cand.size()) < n - 1) {
    auto c = std::make_unique<ocg_ldl::Ref::Cand>();
    c->W.alloc(static_cast<size_t>(std::max<int64_t>(1, d0.w_len)));
    c->stash.alloc(static_cast<size_t>(std::max<int64_t>(1, d0.stash_len)));
    c->D.alloc(static_cast<size_t>(d0.dim));
    c->Dinv.alloc(static_cast<size_t>(d0.dim));
    c->Lx.alloc(static_cast<size_t>(std::max<int64_t>(1, d0.lnz)));
    c->sr.alloc(static_cast<size_t>(std::max<int64_t>(1, R.nnl * 8)));
    c->inertia.alloc(3);
    ck(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "candidate stream");
    ck(cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming), "candidate event");
    R.cand.push_back(std::move(c));
  }
  if (!R.ev0) ck(cudaEventCreateWithFlags(&R.ev0, cudaEventDisableTiming), "event");
  const double* kval = l->kkt->val.p;
  ck(cudaEventRecord(R.ev0, s0), "record");
  for (int i = 1; i < n; ++i) {  // candidates 1.. on their streams, after the caller's work so far
    auto& c = *R.cand[static_cast<size_t>(i - 1)];
    ck(cudaStreamWaitEvent(c.st, R.ev0, 0), "wait");
    ocg::rl::Dev d = d0;
    d.sr = c.sr.p;
    ocg::rl::factor(d, kval, delta_w[i], delta_c[i], c.W.p, c.stash.p, c.D.p, c.Dinv.p, c.Lx.p, c.inertia.p, c.st);
    c.dw = delta_w[i];
    c.dc = delta_c[i];
    ck(cudaEventRecord(c.ev, c.st), "record");
  }
  ocg::rl::factor(d0, kval, delta_w[0], delta_c[0], R.W.p, R.stash.p, R.D.p, R.Dinv.p, R.Lx.p, R.inertia.p, s0);
  std::vector<unsigned long long> h(static_cast<size_t>(3 * n));
  ck(cudaMemcpyAsync(h.data(), R.inertia.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s0), "inertia");
  for (int i = 1; i < n; ++i) {
    auto& c = *R.cand[static_cast<size_t>(i - 1)];
    ck(cudaStreamWaitEvent(s0, c.ev, 0), "wait");
    ck(cudaMemcpyAsync(h.data() + 3 * i, c.inertia.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s0),
       "inertia");
  }
  ck(cudaStreamSynchronize(s0), "sync");
  for (int i = 0; i < 3 * n; ++i) inertia[i] = static_cast<int64_t>(h[static_cast<size_t>(i)]);
  l->kkt->ev->launches += static_cast<int64_t>(n) * (2 + (R.nleaf > 0) + (R.dev.npa > 0) + (R.nnl > 0));
  l->delta_w = delta_w[0];
  l->delta_c = delta_c[0];
  l->factorizations += n;
  return OCG_OK;
  OCG_GUARD_END
}

int ocg_ldl_select(ocg_ldl* l, int i) {
  if (!l) return fail(OCG_ERR_ARG, "null argument");
  if (i == 0) return OCG_OK;
  if (!l->ref || i < 0 || i > static_cast<int>(l->ref->cand.size()))
    return fail(OCG_ERR_ARG, "ocg_ldl_select: no such candidate");
  auto& R = *l->ref;
  auto& c = *R.cand[static_cast<size_t>(i - 1)];
  auto sw = [](auto& a, auto& b) {
    std::swap(a.p, b.p);
    std::swap(a.n, b.n);
    std::swap(a.cap, b.cap);
    std::swap(a.owned, b.owned);
  };
  sw(R.W, c.W);
  sw(R.stash, c.stash);
  sw(R.D, c.D);
  sw(R.Dinv, c.Dinv);
  sw(R.Lx, c.Lx);
  sw(R.sr, c.sr);
  sw(R.inertia, c.inertia);
  R.dev.sr = R.sr.p;
  std::swap(l->delta_w, c.dw);
  std::swap(l->delta_c, c.dc);
  return OCG_OK;
}

int ocg_ldl_solve(ocg_ldl* l, const double* rhs, double* x, ocg_stream s) {
  if (!l || !rhs || !x) return fail(OCG_ERR_ARG, "null argument");
  OCG_GUARD_BEGIN
  ocg::mem::DeviceScope ds_(l->kkt->ev->device);
  if (l->ref) {
    auto& R = *l->ref;
    ocg::rl::solve(R.dev, R.Dinv.p, R.Lx.p, rhs, x, R.y.p, R.xp.p, R.V.p, R.Vs.p, st(s));
    l->kkt->ev->launches += ocg::rl::seq_solve_enabled(R.dev) ? 1 : 2 + (R.dev.nfl > 0) + (R.nnl > 0 ? 3 : 0) + (R.nleaf > 0);
    return OCG_OK;
  }
  const ocg::BandPlan& P = l->plan;
  ocg::dev::band_solve(P, l->dev, l->buf.p, l->Dinv.p, rhs, x, l->work.p, st(s));
  l->kkt->ev->launches += P.nseg > 1 ? 8 : 3;
  return OCG_OK;
  OCG_GUARD_END
}

}  // extern "C"

extern "C" char* ocg_debug_generated_source(const ocg_model* m, int fma, int block) {
  return ocg_debug_generated_source_ex(m, fma, block, 0);
}

extern "C" char* ocg_debug_generated_source_ex(const ocg_model* m, int fma, int block, int input_staging) {
  if (!m) return nullptr;
  ocg::GenOptions go;
  go.fma = fma != 0;
  go.block = block > 0 ? block : 128;
  go.prefetch = input_staging == 1;
  go.tma = input_staging == 2;
  go.idx32 = ocg::fits_idx32(m->nlp, ocg::make_layout(m->nlp));
  if (go.tma && go.block != 32) return nullptr;
  if (const char* e = std::getenv("OCG_SPLIT")) {
    go.split_kinds = std::atoi(e) == 1;
    go.distinct_regions = std::atoi(e) == 2;
  }
  const ocg::Generated gen = ocg::generate(m->nlp, ocg::make_layout(m->nlp), go);
  std::string s = gen.source + "// ocg-meta {";
  bool first = true;
  for (const auto& [name, y] : gen.slices) {
    s += std::string(first ? "" : ", ") + "\"" + name + "\": [" + std::to_string(y) + ", " +
         std::to_string(gen.tail.at(name)) + ", " + std::to_string(gen.smem.at(name)) + "]";
    first = false;
  }
  s += ", \"params\": [";
  for (size_t i = 0; i < gen.params.size(); ++i) s += (i ? ", " : "") + std::to_string(gen.params[i]);
  s += "]}\n";
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

extern "C" char* ocg_debug_compile_log(const ocg_model* m, const ocg_eval_options* opts) {
  if (!m) {
    fail(OCG_ERR_ARG, "null model");
    return nullptr;
  }
  try {
    ocg_eval_options o;
    ocg_eval_default_options(&o);
    if (opts) o = *opts;
    ocg::GenOptions go;
    go.fma = o.fma != 0;
    go.block = o.block > 0 ? o.block : 128;
    std::string log;
    // B200: 228 KB shared memory per SM, 227 KB per block (opt-in)
    const ocg::Generated gen =
        generate_budgeted(m->nlp, ocg::make_layout(m->nlp), go, auto_min_blocks(o), o.split_kinds, o.input_staging,
                          233472, 232448,
                          &log);
    std::string s = log + "\n// min_blocks:";
    for (const auto& [k, v] : gen.min_blocks) s += " " + k + "=" + std::to_string(v);
    s += " block=" + std::to_string(gen.block) + " staging=" +
         std::to_string(gen.split_kinds ? 1 : (gen.distinct_regions ? 2 : 0)) +
         " input_staging=" + std::to_string(gen.tma ? 2 : (gen.prefetch ? 1 : 0)) + "\n";
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
  } catch (const std::exception& ex) {
    fail(OCG_ERR_JIT, ex.what());
    return nullptr;
  }
}

extern "C" int ocg_debug_compile(const ocg_model* m, int fma, int block) {
  if (!m) return fail(OCG_ERR_ARG, "null model");
  try {
    ocg::GenOptions go;
    go.fma = fma != 0;
    go.block = block > 0 ? block : 128;
    std::string cubin;
    ocg::jit_compile_only(ocg::generate_source(m->nlp, ocg::make_layout(m->nlp), go), go.fma, cubin);
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_JIT, ex.what());
  }
}
