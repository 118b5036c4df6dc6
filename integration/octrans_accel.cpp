// Drop-in device implementation of the reference's evaluation layer.
//
// This translation unit REPLACES /root/reference/proj/src/ipm/eval.cpp at link
// time: it defines the same classes declared by the unchanged
// reference header proj/src/ipm/ipm_internal.hpp —
//   EvalContext   (ipm_internal.hpp:40-95;  reference eval.cpp:40-286)
//   Reduction     (ipm_internal.hpp:102-111; reference eval.cpp:290-316)
//   KktAssembler  (ipm_internal.hpp:119-146; reference eval.cpp:318-471)
// — over libocgpu's C ABI (include/octgpu.h), so the reference's own Solver
// (proj/src/ipm/solver.cpp), factorization and tests run unmodified with every
// derivative evaluation and the KKT value assembly on the B200.
//
// The reference StructuredNlp is handed to the library as flat arrays
// (ocg_model_create_from_nlp); the library re-derives each group's structural
// pattern and refuses a mismatch, and its COO structure equals the reference's
// bit for bit. Values computed on the device are mirrored into the public
// host vectors (jac_val, hess_val, grad_val, row_scale, obj_scale) because the
// reference Solver reads them directly (solver.cpp:133, :246-251, :626).
//
// The class layout is fixed by the reference header, so per-object device
// state lives in a side table keyed by the object address; it is released
// when a new object is built at the same address or by
// octrans_accel_release_all() (the harness calls it after each solve).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ipm/ipm_internal.hpp"
#include "octgpu.h"
#include "xfer.hpp"

namespace octrans::ipm::detail {

namespace {

void ck(int rc, const char* what) {
  if (rc < 0) throw std::runtime_error(std::string("octgpu ") + what + ": " + ocg_last_error());
}

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda ") + what + ": " + cudaGetErrorString(e));
}

// OCTRANS_ACCEL_TIMING=1: per-phase wall times of the eval calls on stderr
class Lap {
 public:
  explicit Lap(const char* what) : what_(what), on_(std::getenv("OCTRANS_ACCEL_TIMING") != nullptr) {}
  void operator()(const char* phase) {
    if (!on_) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[octrans_accel] %s %-16s %8.3f ms\n", what_, phase,
                 std::chrono::duration<double, std::milli>(now - t_).count());
    t_ = now;
  }

 private:
  const char* what_;
  bool on_;
  std::chrono::steady_clock::time_point t_ = std::chrono::steady_clock::now();
};

class Timer {
 public:
  explicit Timer(double& acc) : acc_(acc), t0_(std::chrono::steady_clock::now()) {}
  ~Timer() { acc_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count(); }

 private:
  double& acc_;
  std::chrono::steady_clock::time_point t0_;
};

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    n = std::max<size_t>(count, 1);
    ckc(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)), "cudaMalloc");
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
};

// Flattened copy of the reference StructuredNlp in the shape of ocg_nlp_desc.
struct NlpFlat {
  struct G {
    std::vector<int32_t> op, a, b, roots, jac, hess;
    std::vector<double> c;
    std::vector<int64_t> base, stride;
    std::vector<const char*> labels;
  };
  std::vector<G> gs;
  std::vector<ocg_group_desc> con, obj;
  std::vector<int32_t> slab_kind, slab_dim;
  std::vector<int64_t> slab_base, slab_nodes;
  ocg_nlp_desc d{};

  ocg_group_desc group(const kernel::Evaluator& ev, G& g) {
    const auto& graph = ev.kernel().graph;
    for (const auto& nd : graph.nodes()) {
      g.op.push_back(static_cast<int32_t>(nd.op));
      g.a.push_back(nd.a);
      g.b.push_back(nd.b);
      g.c.push_back(nd.c);
    }
    for (const auto& in : graph.inputs()) {
      g.base.push_back(in.base);
      g.stride.push_back(in.stride);
    }
    for (const auto& l : graph.input_labels()) g.labels.push_back(l.c_str());
    for (int r : ev.kernel().roots) g.roots.push_back(r);
    for (auto [r, j] : ev.pattern().jac) {
      g.jac.push_back(r);
      g.jac.push_back(j);
    }
    for (auto [i, j] : ev.pattern().hess) {
      g.hess.push_back(i);
      g.hess.push_back(j);
    }
    ocg_group_desc gd{};
    gd.n_nodes = static_cast<int32_t>(g.op.size());
    gd.node_op = g.op.data();
    gd.node_a = g.a.data();
    gd.node_b = g.b.data();
    gd.node_c = g.c.data();
    gd.n_inputs = static_cast<int32_t>(g.base.size());
    gd.input_base = g.base.data();
    gd.input_stride = g.stride.data();
    gd.out_dim = static_cast<int32_t>(g.roots.size());
    gd.roots = g.roots.data();
    gd.n_jac = static_cast<int32_t>(g.jac.size() / 2);
    gd.jac = g.jac.data();
    gd.n_hess = static_cast<int32_t>(g.hess.size() / 2);
    gd.hess = g.hess.data();
    gd.input_labels = g.labels.size() == g.base.size() ? g.labels.data() : nullptr;
    return gd;
  }

  explicit NlpFlat(const StructuredNlp& nlp) {
    gs.resize(nlp.con_groups.size() + nlp.obj_groups.size());
    size_t q = 0;
    for (const auto& cg : nlp.con_groups) {
      ocg_group_desc gd = group(cg.eval, gs[q++]);
      gd.kind = static_cast<int32_t>(cg.kind);
      gd.label = cg.label.c_str();
      gd.range_lo = cg.range.lo;
      gd.range_hi = cg.range.hi;
      gd.range_endpoints = cg.range.endpoints ? 1 : 0;
      gd.row_base = cg.row_base;
      gd.lower = cg.lower.data();
      gd.upper = cg.upper.data();
      con.push_back(gd);
    }
    for (const auto& og : nlp.obj_groups) {
      ocg_group_desc gd = group(og.eval, gs[q++]);
      gd.range_lo = og.range.lo;
      gd.range_hi = og.range.hi;
      gd.range_endpoints = og.range.endpoints ? 1 : 0;
      gd.weight = og.weight;
      gd.label = og.label.c_str();
      obj.push_back(gd);
    }
    for (const auto& s : nlp.layout.slabs) {
      slab_kind.push_back(static_cast<int32_t>(s.kind));
      slab_dim.push_back(s.dim);
      slab_base.push_back(s.base);
      slab_nodes.push_back(s.nodes);
    }
    d.scheme = nlp.scheme == transcribe::Scheme::euler ? 0 : 1;
    d.N = nlp.N;
    d.n_slabs = static_cast<int32_t>(slab_kind.size());
    d.slab_kind = slab_kind.data();
    d.slab_dim = slab_dim.data();
    d.slab_base = slab_base.data();
    d.slab_nodes = slab_nodes.data();
    d.nvar = nlp.nvar();
    d.m_con = nlp.m_con;
    d.lvar = nlp.lvar.data();
    d.uvar = nlp.uvar.data();
    d.x_start = nlp.x_start.data();
    d.clip_lo = nlp.clip_lo.empty() ? nullptr : nlp.clip_lo.data();
    d.clip_hi = nlp.clip_hi.empty() ? nullptr : nlp.clip_hi.data();
    d.lcon = nlp.lcon.data();
    d.ucon = nlp.ucon.data();
    d.maximize = nlp.maximize ? 1 : 0;
    d.n_con_groups = static_cast<int32_t>(con.size());
    d.con_groups = con.data();
    d.n_obj_groups = static_cast<int32_t>(obj.size());
    d.obj_groups = obj.data();
  }
};

// Device state of one EvalContext.
struct Accel {
  ocg_model* model = nullptr;
  ocg_eval* ev = nullptr;
  cudaStream_t stream = nullptr;
  size_t nvar = 0, m = 0;
  Dev<double> x, lam, c, grad, f, scratch;
  ~Accel() {
    xfer.reset();  // synchronises the stream destroyed below
    if (flag) cudaFreeHost(flag);
    if (ev) ocg_eval_destroy(ev);
    if (model) ocg_model_destroy(model);
    if (stream) cudaStreamDestroy(stream);
  }
  // large arrays move through the pipelined page-locked staging of xfer.hpp
  static constexpr size_t kStaged = size_t{1} << 16;
  std::unique_ptr<octrans_accel::Xfer> xfer;
  void upload(const double* src, Dev<double>& dst, size_t n) {
    if (n >= kStaged)
      xfer->h2d(dst.p, src, n);
    else if (n)
      ckc(cudaMemcpyAsync(dst.p, src, n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
  }
  void download(const Dev<double>& src, double* dst, size_t n) {
    if (n) ckc(cudaMemcpyAsync(dst, src.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
  }
  void download_buf(int which, double* dst, size_t n) {
    if (n)
      ckc(cudaMemcpyAsync(dst, ocg_eval_buffer(ev, which), n * sizeof(double), cudaMemcpyDeviceToHost, stream),
          "D2H");
  }
  // several device arrays to host, synchronous on return
  void download_all(const std::vector<octrans_accel::Xfer::Part>& parts) {
    std::vector<octrans_accel::Xfer::Part> big;
    for (const auto& p : parts)
      if (p.n >= kStaged)
        big.push_back(p);
      else if (p.n)
        ckc(cudaMemcpyAsync(p.dst, p.dsrc, p.n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    if (!big.empty()) xfer->d2h(big);
    ckc(cudaStreamSynchronize(stream), "sync");
  }
  // the reference's bool without a synchronisation of its own: the flag is
  // copied behind the outputs and read once the downloads are done
  int* flag = nullptr;  // page-locked
  void status_async() { ck(ocg_eval_status_async(ev, flag, stream), "eval_status_async"); }
  bool flag_ok() const { return *flag == 0; }
  // the reference's bool: synchronises, reports and clears the device flag
  bool status() {
    const int rc = ocg_eval_status(ev, stream);
    ck(rc, "eval_status");
    return rc == OCG_OK;
  }
};

struct KktDev {
  ocg_kkt* k = nullptr;
  Dev<double> sigma;
  ~KktDev() {
    if (k) ocg_kkt_destroy(k);
  }
};

std::mutex g_mu;
std::map<const void*, std::unique_ptr<KktDev>> g_kkt;
std::map<const void*, std::unique_ptr<Accel>> g_ec;

Accel& accel(const EvalContext* e) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ec.find(e);
  if (it == g_ec.end()) throw std::runtime_error("octrans_accel: EvalContext without device state");
  return *it->second;
}

int device_ordinal() {
  const char* d = std::getenv("OCTRANS_ACCEL_DEVICE");
  return d ? std::atoi(d) : 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// EvalContext (ipm_internal.hpp:40-95)
// ---------------------------------------------------------------------------

EvalContext::EvalContext(const StructuredNlp& nlp, const backend::Backend& backend) : nlp_(nlp), backend_(backend) {
  auto a = std::make_unique<Accel>();
  NlpFlat flat(nlp);
  ck(ocg_model_create_from_nlp(&flat.d, &a->model), "model_create_from_nlp");
  ocg_eval_options o;
  ocg_eval_default_options(&o);
  o.device = device_ordinal();
  ckc(cudaSetDevice(o.device), "cudaSetDevice");
  ck(ocg_eval_create(a->model, &o, &a->ev), "eval_create");
  ckc(cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking), "stream");
  ckc(cudaMallocHost(&a->flag, sizeof(int)), "cudaMallocHost");
  *a->flag = 0;
  {
    // staging: 6 slots of 2^18 doubles (2 MiB), half the host threads (at most
    // 8) copying -- the best of a sweep on the B200 box (Goddard N=1e5 J+H
    // step 1.47 ms; 4 MiB x 4: 2.4 ms, 1 MiB x 8: 1.75 ms, profiles/
    // r2_dropin_xfer_sweep.txt); OCTRANS_ACCEL_XFER="chunk_doubles,slots,threads"
    size_t chunk = size_t{1} << 18;
    int slots = 6, threads = static_cast<int>(std::clamp(std::thread::hardware_concurrency() / 2, 1u, 8u));
    int nt = 0;
    if (const char* e = std::getenv("OCTRANS_ACCEL_XFER")) std::sscanf(e, "%zu,%d,%d,%d", &chunk, &slots, &threads, &nt);
    a->xfer =
        std::make_unique<octrans_accel::Xfer>(a->stream, std::max(1, threads), std::max<size_t>(chunk, 1024), slots, nt);
  }
  a->nvar = static_cast<size_t>(nlp.nvar());
  a->m = static_cast<size_t>(nlp.m_con);
  a->x.alloc(a->nvar);
  a->lam.alloc(a->m);
  a->c.alloc(a->m);
  a->grad.alloc(a->nvar);
  a->f.alloc(1);
  a->scratch.alloc(1);

  int64_t jn = 0, hn = 0, gn = 0;
  ck(ocg_eval_sizes(a->ev, &jn, &hn, &gn), "sizes");
  jac_row.resize(static_cast<size_t>(jn));
  jac_col.resize(static_cast<size_t>(jn));
  hess_row.resize(static_cast<size_t>(hn));
  hess_col.resize(static_cast<size_t>(hn));
  grad_col.resize(static_cast<size_t>(gn));
  ck(ocg_eval_structure(a->ev, jac_row.data(), jac_col.data(), hess_row.data(), hess_col.data(), grad_col.data()),
     "structure");
  jac_val.assign(static_cast<size_t>(jn), 0.0);
  hess_val.assign(static_cast<size_t>(hn), 0.0);
  grad_val.assign(static_cast<size_t>(gn), 0.0);
  c_raw_.assign(a->m, 0.0);
  row_scale.assign(a->m, 1.0);

  std::lock_guard<std::mutex> lk(g_mu);
  g_ec[this] = std::move(a);
}

void EvalContext::compute_scaling(std::span<const double> x0, bool enabled) {
  Accel& a = accel(this);
  a.upload(x0.data(), a.x, a.nvar);
  ck(ocg_eval_compute_scaling(a.ev, a.x.p, enabled ? 1 : 0, a.stream), "compute_scaling");
  ck(ocg_eval_get_scaling(a.ev, &obj_scale, row_scale.data()), "get_scaling");
}

bool EvalContext::eval_constraints(std::span<const double> x, std::vector<double>& c_scaled) {
  Timer t(time_derivatives);
  Accel& a = accel(this);
  a.upload(x.data(), a.x, a.nvar);
  ck(ocg_eval_constraints(a.ev, a.x.p, a.c.p, a.stream), "eval_constraints");
  if (!a.status()) return false;
  c_scaled.resize(a.m);
  a.download_all({{c_scaled.data(), a.c.p, a.m}});
  return true;
}

bool EvalContext::eval_constraints_jacobian(std::span<const double> x, std::vector<double>& c_scaled) {
  Timer t(time_derivatives);
  Accel& a = accel(this);
  Lap lap("eval_constraints_jacobian");
  a.upload(x.data(), a.x, a.nvar);
  lap("h2d x");
  ck(ocg_eval_constraints_jacobian(a.ev, a.x.p, a.c.p, a.stream), "eval_constraints_jacobian");
  a.status_async();
  lap("kernel enqueued");
  // c and jac_val come back unconditionally (on a domain error the reference
  // also leaves partial values behind); the bool is read after the copies
  c_scaled.resize(a.m);
  a.download_all({{c_scaled.data(), a.c.p, a.m},
                  {jac_val.data(), static_cast<const double*>(ocg_eval_buffer(a.ev, OCG_BUF_JAC)), jac_val.size()}});
  lap("d2h c, jac_val");
  return a.flag_ok();
}

bool EvalContext::eval_objective(std::span<const double> x, double& f_scaled) {
  Timer t(time_derivatives);
  Accel& a = accel(this);
  a.upload(x.data(), a.x, a.nvar);
  ck(ocg_eval_objective(a.ev, a.x.p, a.f.p, a.stream), "eval_objective");
  if (!a.status()) return false;
  a.download(a.f, &f_scaled, 1);
  ckc(cudaStreamSynchronize(a.stream), "sync");
  return std::isfinite(f_scaled);
}

bool EvalContext::eval_gradient(std::span<const double> x, std::vector<double>& grad_dense) {
  Timer t(time_derivatives);
  Accel& a = accel(this);
  a.upload(x.data(), a.x, a.nvar);
  ck(ocg_eval_gradient(a.ev, a.x.p, a.grad.p, a.stream), "eval_gradient");
  if (!a.status()) return false;
  grad_dense.resize(a.nvar);
  a.download_all({{grad_dense.data(), a.grad.p, a.nvar},
                  {grad_val.data(), static_cast<const double*>(ocg_eval_buffer(a.ev, OCG_BUF_GRAD)), grad_val.size()}});
  return true;
}

bool EvalContext::eval_hessian(std::span<const double> x, std::span<const double> lambda_scaled) {
  Timer t(time_derivatives);
  Accel& a = accel(this);
  Lap lap("eval_hessian");
  a.upload(x.data(), a.x, a.nvar);
  a.upload(lambda_scaled.data(), a.lam, a.m);
  lap("h2d x, lambda");
  ck(ocg_eval_hessian(a.ev, a.x.p, a.lam.p, a.stream), "eval_hessian");
  a.status_async();
  lap("kernel enqueued");
  // hess_val is public: keep the host mirror current (the reference leaves
  // partial values behind on failure too)
  a.download_all({{hess_val.data(), static_cast<const double*>(ocg_eval_buffer(a.ev, OCG_BUF_HESS)), hess_val.size()}});
  lap("d2h hess_val");
  return a.flag_ok();
}

double EvalContext::max_abs_hessian() const {
  Accel& a = accel(this);
  ck(ocg_eval_max_abs_hessian(a.ev, a.scratch.p, a.stream), "max_abs_hessian");
  double m = 0.0;
  a.download(a.scratch, &m, 1);
  ckc(cudaStreamSynchronize(a.stream), "sync");
  return m;
}

// ---------------------------------------------------------------------------
// Reduction (ipm_internal.hpp:102-111): rows whose kernel root is a bare
// decision slot become slot bounds; the remaining rows get dual ordinals.
// ---------------------------------------------------------------------------

Reduction::Reduction(const StructuredNlp& nlp) : xlo(nlp.lvar), xhi(nlp.uvar) {
  const auto mc = static_cast<size_t>(nlp.m_con);
  row_slot.assign(mc, -1);
  for (const auto& grp : nlp.con_groups) {
    const auto& graph = grp.eval.kernel().graph;
    const auto& roots = grp.eval.kernel().roots;
    for (int r = 0; r < grp.out_dim; ++r) {
      const kernel::Node& root = graph.node(roots[static_cast<size_t>(r)]);
      if (root.op != kernel::Op::input) continue;
      const kernel::InputAddress in = graph.inputs()[static_cast<size_t>(root.a)];
      for (Index k = 0; k < grp.range.count(); ++k) {
        const auto row = static_cast<size_t>(grp.row_base + k * grp.out_dim + r);
        const auto slot = static_cast<size_t>(in.slot(grp.range.at(k)));
        row_slot[row] = static_cast<Index>(slot);
        xlo[slot] = std::max(xlo[slot], nlp.lcon[row]);
        xhi[slot] = std::min(xhi[slot], nlp.ucon[row]);
        contradictory = contradictory || xlo[slot] > xhi[slot];
      }
    }
  }
  dual_index.assign(mc, -1);
  for (size_t r = 0; r < mc; ++r) {
    if (row_slot[r] >= 0) continue;
    dual_index[r] = m_active++;
    dual_row.push_back(static_cast<Index>(r));
  }
}

// ---------------------------------------------------------------------------
// KktAssembler (ipm_internal.hpp:119-146): pattern and maps from the device
// library (bit-identical to the reference's lower CSC), values assembled on
// the device from the device-resident Jacobian/Hessian, K.val mirrored to the
// host for the reference factorization.
// ---------------------------------------------------------------------------

KktAssembler::KktAssembler(const StructuredNlp& nlp, const EvalContext& ec, const Reduction& red) : red_(red) {
  Accel& a = accel(&ec);
  auto kd = std::make_unique<KktDev>();
  ck(ocg_kkt_create(a.model, a.ev, &kd->k), "kkt_create");
  int64_t dims[7];
  ck(ocg_kkt_dims(kd->k, dims), "kkt_dims");
  n_free = dims[0];
  n_slack = dims[1];
  ntot = dims[2];
  m = dims[3];
  dim = dims[4];
  if (m != red.m_active) throw std::runtime_error("octrans_accel: reduction mismatch");
  K.n = dim;
  K.colp.resize(static_cast<size_t>(dim) + 1);
  K.rowi.resize(static_cast<size_t>(dims[5]));
  ck(ocg_kkt_pattern(kd->k, K.colp.data(), K.rowi.data()), "kkt_pattern");
  K.val.assign(static_cast<size_t>(dims[5]), 0.0);
  const auto nv = static_cast<size_t>(nlp.nvar()), mc = static_cast<size_t>(nlp.m_con);
  prim_index.resize(nv);
  slack_index.resize(mc);
  std::vector<Index> dual_index(mc), row_slot(mc);
  std::vector<double> xlo(nv), xhi(nv);
  ck(ocg_kkt_maps(kd->k, prim_index.data(), slack_index.data(), dual_index.data(), row_slot.data(), xlo.data(),
                  xhi.data()),
     "kkt_maps");
  free_slot.assign(static_cast<size_t>(n_free), -1);
  for (size_t s = 0; s < nv; ++s)
    if (prim_index[s] >= 0) free_slot[static_cast<size_t>(prim_index[s])] = static_cast<Index>(s);
  slack_of.assign(static_cast<size_t>(n_slack), -1);
  for (size_t r = 0; r < mc; ++r)
    if (slack_index[r] >= 0) slack_of[static_cast<size_t>(slack_index[r])] = static_cast<Index>(r);
  kd->sigma.alloc(static_cast<size_t>(ntot));

  // single-column kept equality rows: their dual is pivoted right after that
  // primal column (zero-diagonal 1x1 pivots otherwise hit exact zeros)
  std::vector<Index> col_of(mc, -1);
  std::vector<int> count(mc, 0);
  for (size_t e = 0; e < ec.jac_row.size(); ++e) {
    const Index pj = prim_index[static_cast<size_t>(ec.jac_col[e])];
    if (pj < 0) continue;
    const auto r = static_cast<size_t>(ec.jac_row[e]);
    if (count[r] == 0) {
      col_of[r] = pj;
      count[r] = 1;
    } else if (col_of[r] != pj) {
      count[r] = 2;
    }
  }
  for (size_t r = 0; r < mc; ++r)
    if (red.dual_index[r] >= 0 && slack_index[r] < 0 && count[r] == 1)
      pivot_after_.emplace_back(col_of[r], ntot + red.dual_index[r]);

  std::lock_guard<std::mutex> lk(g_mu);
  g_kkt[this] = std::move(kd);
}

void KktAssembler::assemble(const EvalContext& ec, std::span<const double> sigma) {
  Accel& a = accel(&ec);
  KktDev* kd;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    kd = g_kkt.at(this).get();
  }
  a.upload(sigma.data(), kd->sigma, static_cast<size_t>(ntot));
  ck(ocg_kkt_assemble(kd->k, kd->sigma.p, a.stream), "kkt_assemble");
  if (!K.val.empty())
    ckc(cudaMemcpyAsync(K.val.data(), ocg_kkt_values(kd->k), K.val.size() * sizeof(double), cudaMemcpyDeviceToHost,
                        a.stream),
        "D2H K");
  ckc(cudaStreamSynchronize(a.stream), "sync");
}

const sparse::SymbolicLdl& KktAssembler::symbolic() {
  if (!analyzed_) {
    std::vector<Index> perm = sparse::amd_order(K);
    if (!pivot_after_.empty()) {
      // each deferred dual follows its primal column, in the order the pairs
      // were recorded (latest first)
      std::vector<std::vector<Index>> after(static_cast<size_t>(dim));
      std::vector<char> skip(static_cast<size_t>(dim), 0);
      for (const auto& [col, dual] : pivot_after_) {
        after[static_cast<size_t>(col)].insert(after[static_cast<size_t>(col)].begin(), dual);
        skip[static_cast<size_t>(dual)] = 1;
      }
      std::vector<Index> order;
      order.reserve(static_cast<size_t>(dim));
      for (Index node : perm) {
        if (skip[static_cast<size_t>(node)]) continue;
        order.push_back(node);
        for (Index d : after[static_cast<size_t>(node)]) order.push_back(d);
      }
      perm.swap(order);
    }
    sym_ = sparse::analyze_ordered(K, perm);
    analyzed_ = true;
    ++analyze_count;
  }
  return sym_;
}

}  // namespace octrans::ipm::detail

extern "C" void octrans_accel_release_all() {
  using namespace octrans::ipm::detail;
  std::lock_guard<std::mutex> lk(g_mu);
  g_kkt.clear();
  g_ec.clear();
}

// Diagnostics for the CPU test suite: the library's structure dump of a
// reference StructuredNlp handed over through ocg_model_create_from_nlp
// (needs no GPU). Caller frees with ocg_free.
extern "C" char* octrans_accel_nlp_json(const void* structured_nlp) {
  using namespace octrans::ipm::detail;
  NlpFlat flat(*static_cast<const octrans::transcribe::StructuredNlp*>(structured_nlp));
  ocg_model* m = nullptr;
  if (ocg_model_create_from_nlp(&flat.d, &m) != OCG_OK) return nullptr;
  char* s = ocg_model_structure_json(m);
  ocg_model_destroy(m);
  return s;
}
