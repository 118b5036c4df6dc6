// Device-resident filter line-search interior-point solve.
//
// Host control flow of the reference's Solver (proj/src/ipm/solver.cpp:304-702):
// monotone barrier update, inertia-corrected regularization, backtracking
// filter line search with up to 4 second-order corrections, the single-shot
// restoration fallback and the dual safeguard — the same decisions in the
// same order. Every vector lives on the device: evaluations (octgpu eval
// kernels), the KKT assembly, the vector work (ipm_kernels.cu) and the
// factorization (band.cu, the stand-in for the reference's LDL^T / cuDSS).
// Per line-search trial the host receives a handful of scalars (ok flags,
// theta, barrier sum, objective).
//
// This file is a client of the public C ABI only (include/octgpu.h), like the
// reference's Solver is a client of EvalContext / KktAssembler / sparse::.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/octgpu.h"
#include "devmem.hpp"
#include "ipm_kernels.hpp"

namespace ocg::hd {
int set_error(int code, const std::string& msg);  // capi.cpp: ocg_last_error's message
int ldl_create(ocg_kkt* k, int target, ocg_ldl** out);  // capi.cpp: band LDL^T with a segment target
}

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
// filter line-search constants (solver.cpp:38-52)
constexpr double kGammaTheta = 1e-5;
constexpr double kGammaPhi = 1e-5;
constexpr double kSTheta = 1.1;
constexpr double kSPhi = 2.3;
constexpr double kDeltaSwitch = 1.0;
constexpr double kEtaPhi = 1e-4;
constexpr double kAlphaMin = 1e-12;
constexpr double kKappaSigma = 1e10;
constexpr double kKappaEps = 10.0;
constexpr double kKappaMu = 0.2;
constexpr double kThetaMu = 1.5;
constexpr double kPushIn = 1e-2;

struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaErr(std::string(what) + ": " + cudaGetErrorString(e));
}
void cko(int rc, const char* what) {
  if (rc < 0) throw CudaErr(std::string(what) + ": " + ocg_last_error());
}

struct Clock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double elapsed() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

template <class T>
struct DVec {
  T* p = nullptr;
  size_t n = 0;
  DVec() = default;
  explicit DVec(size_t count) { alloc(count); }
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  size_t cap = 0;
  ~DVec() { ocg::mem::device_free(p, cap); }  // large blocks back to the cache (devmem.hpp)
  void alloc(size_t count) {
    ocg::mem::device_free(p, cap);
    n = count;
    void* q = nullptr;
    ckc(ocg::mem::device_alloc(std::max<size_t>(count, 1) * sizeof(T), &q, &cap), "cudaMallocAsync");
    p = static_cast<T*>(q);
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    if (!v.empty()) ckc(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
  }
  void download(std::vector<T>& v, cudaStream_t s) const {
    v.resize(n);
    if (n) ckc(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    ckc(cudaStreamSynchronize(s), "sync");
  }
  // exchange whole blocks (pointer, length and the block size the cache files them under)
  void swap(DVec& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(cap, o.cap);
  }
};

// an instance whose data do not fit the model's structure (OCG_ERR_ARG)
struct InvalidInstance : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class DeviceSolver {
 public:
  DeviceSolver(ocg_model* model, const ocg_ipm_options& o, int device) : model_(model), o_(o), device_(device) {
    Clock t;
    ckc(cudaSetDevice(device), "cudaSetDevice");
    ckc(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
    ocg_eval_options eo;
    ocg_eval_default_options(&eo);
    eo.device = device;
    cko(ocg_eval_create(model, &eo, &ev_), "eval_create");
    r_.time_plan_eval = t.elapsed();
    Clock t2;
    cko(ocg_kkt_create(model, ev_, &kkt_), "kkt_create");
    r_.time_plan_kkt = t2.elapsed();
  }
  ~DeviceSolver() {
    ocg::mem::DeviceScope ds(device_);
    if (s_) cudaStreamSynchronize(s_);
    for (ocg_ldl* l : ldls_)
      if (l) ocg_ldl_destroy(l);
    if (ldl_retry_) ocg_ldl_destroy(ldl_retry_);
    if (kkt_) ocg_kkt_destroy(kkt_);
    if (ev_) ocg_eval_destroy(ev_);
    if (s_) cudaStreamDestroy(s_);
    drop_graphs();
    if (hpin_) cudaFreeHost(hpin_);
  }

  int run(ocg_ipm_result* res, double* x_out);
  // run(); on the band factorization, a solve that ends infeasible or failed
  // is solved again with a quarter of the segments (longer segments change
  // the rounding of the inertia decisions on near-singular KKT matrices —
  // Goddard at N = 3e4 / 5e4 — and converge where the default did not);
  // OCG_IPM_RETRY=0 off
  int run_with_retry(ocg_ipm_result* res, double* x_out);
  int device() const { return device_; }
  // instance data for the next run (NULL = the model's own arrays)
  void set_instance(const ocg_ipm_options& o, const double* lvar, const double* uvar, const double* x0,
                    const double* lcon, const double* ucon) {
    o_ = o;
    inst_[0] = lvar;
    inst_[1] = uvar;
    inst_[2] = x0;
    inst_[3] = lcon;
    inst_[4] = ucon;
  }

 private:
  const double* inst_[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool allocated_ = false;
  ocg_model* model_;
  ocg_ipm_options o_;
  int device_ = 0;
  cudaStream_t s_ = nullptr;
  ocg_eval* ev_ = nullptr;
  ocg_kkt* kkt_ = nullptr;
  ocg_ldl* ldl_ = nullptr;      // the factorization of this run: ldls_[o_.kkt_order]
  ocg_ldl* ldls_[2] = {nullptr, nullptr};
  // band fallback of run_with_retry: a quarter of the segments
  ocg_ldl* ldl_retry_ = nullptr;
  bool use_retry_ldl_ = false;
  // the factorization plan of the requested elimination order, built on first use
  void select_ldl() {
    const int order = o_.kkt_order == OCG_LDL_REFERENCE ? OCG_LDL_REFERENCE : OCG_LDL_BAND;
    if (!ldls_[order]) {
      Clock t;
      cko(ocg_ldl_create_ex(kkt_, order, &ldls_[order]), "ldl_create");
      plan_ldl_s_[order] = t.elapsed();
    }
    ldl_ = use_retry_ldl_ && order == OCG_LDL_BAND && ldl_retry_ ? ldl_retry_ : ldls_[order];
    r_.time_plan_ldl = plan_ldl_s_[order];
    const char* e = std::getenv("OCG_IPM_SPECULATE");
    speculate_ = order == OCG_LDL_REFERENCE && !(e && std::atoi(e) == 0);
    const char* g = std::getenv("OCG_IPM_GRAPHS");
    graphs_ = !(g && std::atoi(g) == 0);
    // captured graphs hold this solve's scalars (e.g. the objective scale) by
    // value: every solve captures its own
    drop_graphs();
  }
  double plan_ldl_s_[2] = {0.0, 0.0};
  ocg::ipmdev::Iter P_;
  ocg::ipmdev::Scratch sc_;

  int64_t nvar_ = 0, mcon_ = 0, nfree_ = 0, nslack_ = 0, ntot_ = 0, m_ = 0, dim_ = 0;
  bool contradictory_ = false;
  double mu_ = 0.1, tau_ = 0.99, delta_last_ = 0.0, obj_scale_ = 1.0;
  // OCG_TIMING diagnostics: solves, refinement rounds, line-search trials
  long long n_solves_ = 0, n_refine_ = 0, n_trials_ = 0;
  double t_err_ = 0, t_assemble_ = 0, t_pre_ = 0, t_search_ = 0, t_accept_ = 0;
  double dw_ = 0.0, dc_ = 0.0;  // regularization of the current factorization
  // page-locked landing slots of the fused trial evaluation's scalars
  struct HostPinned {
    double v[4];
    double alpha;
    int flag_c, flag_f;
  };
  // graph-captured line-search trials (OCG_IPM_GRAPHS=0 off), one executable
  // graph per pointer set of the iterate, trial and direction buffers
  bool graphs_ = true;
  using TrialKey = std::array<const void*, 6>;
  std::map<TrialKey, cudaGraphExec_t> trial_graphs_;
  void drop_graphs() {
    for (auto& [k, g] : trial_graphs_)
      if (g) cudaGraphExecDestroy(g);
    trial_graphs_.clear();
  }
  HostPinned* hpin_ = nullptr;
  // setup's host arrays, reused across solves of this context
  struct HostScratch {
    std::vector<double> lvar, uvar, x0, lcon, ucon, xlo, xhi, lcon_s, ucon_s, lb, ub, x, c, s, zl, zu;
    std::vector<int64_t> prim, slack, dual, rslot, free_slot, slack_of, dual_row;
    std::vector<int8_t> hl, hu;
  } hs_;
  // speculative inertia correction (reference order only, OCG_IPM_SPECULATE=0 off)
  bool speculate_ = false;
  long long r_speculative_ = 0;
  double theta_min_ = 0.0, theta_max_ = kInf;
  std::vector<std::pair<double, double>> filter_;
  ocg_ipm_result r_{};

  // device state
  DVec<int64_t> free_slot_, dual_row_, slack_index_;
  DVec<double> lb_, ub_, lcon_s_;
  DVec<int8_t> has_lb_, has_ub_;
  std::unique_ptr<DVec<double>> x_, s_v_, c_, grad_, xt_, st_, ct_, gradt_;
  DVec<double> lambda_, zl_, zu_, g_, gt_, gsoc_, sigma_, rhs_, rhs2_, jtlam_, lamfull_, step_, step2_, kx_, r_v_,
      dx_, dzl_, dzu_, dscal_, partials_, out_;

  // ---- wrappers with the reference's bool semantics ----
  bool ok() {
    const int rc = ocg_eval_status(ev_, s_);
    cko(rc, "eval_status");
    return rc == OCG_OK;
  }
  bool eval_c(const double* x, double* c) {
    Clock t;
    cko(ocg_eval_constraints(ev_, x, c, s_), "eval_constraints");
    const bool b = ok();
    r_.time_derivatives += t.elapsed();
    return b;
  }
  bool eval_cj(const double* x, double* c) {
    Clock t;
    cko(ocg_eval_constraints_jacobian(ev_, x, c, s_), "eval_constraints_jacobian");
    const bool b = ok();
    r_.time_derivatives += t.elapsed();
    return b;
  }
  bool eval_f(const double* x, double& f) {
    Clock t;
    cko(ocg_eval_objective(ev_, x, dscal_.p, s_), "eval_objective");
    const bool b = ok();
    ckc(cudaMemcpyAsync(&f, dscal_.p, sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H f");
    ckc(cudaStreamSynchronize(s_), "sync");
    r_.time_derivatives += t.elapsed();
    return b && std::isfinite(f);
  }
  bool eval_grad(const double* x, double* g) {
    Clock t;
    cko(ocg_eval_gradient(ev_, x, g, s_), "eval_gradient");
    const bool b = ok();
    r_.time_derivatives += t.elapsed();
    return b;
  }
  bool eval_h(const double* x, const double* lam_full) {
    Clock t;
    cko(ocg_eval_hessian(ev_, x, lam_full, s_), "eval_hessian");
    const bool b = ok();
    r_.time_derivatives += t.elapsed();
    return b;
  }
  double max_abs_h() {
    cko(ocg_eval_max_abs_hessian(ev_, dscal_.p, s_), "max_abs_hessian");
    double v = 0.0;
    ckc(cudaMemcpyAsync(&v, dscal_.p, sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H");
    ckc(cudaStreamSynchronize(s_), "sync");
    return v;
  }

  void setup(std::vector<double>& row_scale);
  void alloc_state(size_t nv, size_t mc);
  // OCG_IPM_DUMP=<dir> OCG_IPM_DUMP_ITERS=i,j,...: the iterate and the vector
  // kernels' results at those iterations, for tests against the reference's
  // Solver math (tests/test_ipm_kernels_gpu.py)
  void dump_iterate(int iter, double alpha_max, double dphi);
  double theta_of(const double* g) { return ocg::ipmdev::l1(g, m_, sc_, s_); }
  double kkt_error(double mu, const double* g, double& comp_out, double& stat_out);
  void add_to_filter(double theta, double phi);
  bool filter_rejects(double theta, double phi) const;
  bool solve_kkt(double wmax, bool& numeric_failure);
  void resolve(const double* rhs, double* step);
  void refine_if_needed(const double* rhs, double* step);
  void finish(int status, int iter, const std::vector<double>& row_scale);
};

void DeviceSolver::alloc_state(size_t nv, size_t mc) {
  const auto nt = static_cast<size_t>(ntot_);
  free_slot_.alloc(static_cast<size_t>(nfree_));
  dual_row_.alloc(static_cast<size_t>(m_));
  slack_index_.alloc(mc);
  lb_.alloc(nt);
  ub_.alloc(nt);
  has_lb_.alloc(nt);
  has_ub_.alloc(nt);
  lcon_s_.alloc(mc);
  for (auto* v : {&x_, &xt_, &grad_, &gradt_}) *v = std::make_unique<DVec<double>>(nv);
  for (auto* v : {&c_, &ct_}) *v = std::make_unique<DVec<double>>(mc);
  for (auto* v : {&s_v_, &st_}) *v = std::make_unique<DVec<double>>(static_cast<size_t>(nslack_));
  const auto dm = static_cast<size_t>(dim_), mm = static_cast<size_t>(m_);
  lambda_.alloc(mm);
  g_.alloc(mm);
  gt_.alloc(mm);
  gsoc_.alloc(mm);
  zl_.alloc(nt);
  zu_.alloc(nt);
  sigma_.alloc(nt);
  jtlam_.alloc(nt);
  dzl_.alloc(nt);
  dzu_.alloc(nt);
  rhs_.alloc(dm);
  rhs2_.alloc(dm);
  step_.alloc(dm);
  step2_.alloc(dm);
  kx_.alloc(dm);
  r_v_.alloc(dm);
  dx_.alloc(dm);
  lamfull_.alloc(mc);
  dscal_.alloc(8);
  if (!hpin_) ckc(cudaMallocHost(reinterpret_cast<void**>(&hpin_), sizeof(HostPinned)), "pinned trial scalars");
  partials_.alloc(2 * 148 * 8);
  out_.alloc(8);
  sc_.partials = partials_.p;
  sc_.out = out_.p;
}

void DeviceSolver::setup(std::vector<double>& row_scale) {
  static const bool timing = std::getenv("OCG_TIMING") != nullptr;
  Clock lapc;
  auto lap = [&](const char* what) {
    if (!timing) return;
    std::fprintf(stderr, "[ipm setup] %-18s %8.3f s\n", what, lapc.elapsed());
    lapc = Clock();
  };
  nvar_ = ocg_model_nvar(model_);
  mcon_ = ocg_model_mcon(model_);
  int64_t d[7];
  cko(ocg_kkt_dims(kkt_, d), "kkt_dims");
  nfree_ = d[0];
  nslack_ = d[1];
  ntot_ = d[2];
  m_ = d[3];
  dim_ = d[4];
  contradictory_ = d[6] != 0;
  r_.kkt_dim = dim_;
  r_.kkt_nnz = d[5];
  const auto nv = static_cast<size_t>(nvar_), mc = static_cast<size_t>(mcon_);
  // host arrays live in hs_ and keep their memory across solves of this
  // context (cached with the plans): no fresh pages to fault in per solve
  auto& lvar = hs_.lvar; auto& uvar = hs_.uvar; auto& x0 = hs_.x0; auto& lcon = hs_.lcon; auto& ucon = hs_.ucon;
  auto& xlo = hs_.xlo; auto& xhi = hs_.xhi;
  for (auto* v : {&lvar, &uvar, &x0, &xlo, &xhi}) v->resize(nv);
  lcon.resize(mc);
  ucon.resize(mc);
  cko(ocg_model_arrays(model_, lvar.data(), uvar.data(), x0.data(), nullptr, nullptr, lcon.data(), ucon.data()),
      "model_arrays");
  auto& prim = hs_.prim; auto& slack = hs_.slack; auto& dual = hs_.dual; auto& rslot = hs_.rslot;
  prim.resize(nv);
  for (auto* v : {&slack, &dual, &rslot}) v->resize(mc);
  cko(ocg_kkt_maps(kkt_, prim.data(), slack.data(), dual.data(), rslot.data(), xlo.data(), xhi.data()), "kkt_maps");
  if (inst_[0] || inst_[1] || inst_[2] || inst_[3] || inst_[4]) {
    // another instance of the same structure: its bounds and start point, and
    // the Reduction's folded bounds recomputed from them (eval.cpp:290-316)
    auto take = [](std::vector<double>& v, const double* p) {
      if (p) std::copy(p, p + v.size(), v.begin());
    };
    take(lvar, inst_[0]);
    take(uvar, inst_[1]);
    take(x0, inst_[2]);
    take(lcon, inst_[3]);
    take(ucon, inst_[4]);
    xlo = lvar;
    xhi = uvar;
    contradictory_ = false;
    for (size_t r = 0; r < mc; ++r) {
      if (rslot[r] < 0) continue;
      const auto sl = static_cast<size_t>(rslot[r]);
      xlo[sl] = std::max(xlo[sl], lcon[r]);
      xhi[sl] = std::min(xhi[sl], ucon[r]);
      if (xlo[sl] > xhi[sl]) contradictory_ = true;
    }
    for (size_t sl = 0; sl < nv; ++sl)
      if ((prim[sl] < 0) != (xlo[sl] == xhi[sl]))
        throw InvalidInstance("instance bounds change which slots are fixed: the KKT structure differs");
    // the slack map is the model's (eval.cpp:330-336): a kept equality row
    // must stay an equality and a kept range row a range
    for (size_t r = 0; r < mc; ++r)
      if (dual[r] >= 0 && (lcon[r] == ucon[r]) != (slack[r] < 0))
        throw InvalidInstance("instance row " + std::to_string(r) +
                              (slack[r] < 0 ? " loosens an equality of the model into a range"
                                            : " turns a range row of the model into an equality"));
  }
  auto& free_slot = hs_.free_slot; auto& slack_of = hs_.slack_of; auto& dual_row = hs_.dual_row;
  free_slot.resize(static_cast<size_t>(nfree_));
  slack_of.resize(static_cast<size_t>(nslack_));
  dual_row.resize(static_cast<size_t>(m_));
  for (size_t sl = 0; sl < nv; ++sl)
    if (prim[sl] >= 0) free_slot[static_cast<size_t>(prim[sl])] = static_cast<int64_t>(sl);
  for (size_t r = 0; r < mc; ++r) {
    if (slack[r] >= 0) slack_of[static_cast<size_t>(slack[r])] = static_cast<int64_t>(r);
    if (dual[r] >= 0) dual_row[static_cast<size_t>(dual[r])] = static_cast<int64_t>(r);
  }

  lap("arrays + maps");
  // EvalContext::compute_scaling at x_start (solver.cpp:318)
  DVec<double> xs(nv);
  xs.upload(x0, s_);
  cko(ocg_eval_compute_scaling(ev_, xs.p, o_.scale, s_), "compute_scaling");
  row_scale.assign(mc, 1.0);
  cko(ocg_eval_get_scaling(ev_, &obj_scale_, row_scale.data()), "get_scaling");

  lap("scaling");
  // Solver::setup_bounds (solver.cpp:125-170)
  auto& lcon_s = hs_.lcon_s; auto& ucon_s = hs_.ucon_s;
  lcon_s.resize(mc);
  ucon_s.resize(mc);
  for (size_t r = 0; r < mc; ++r) {
    lcon_s[r] = row_scale[r] * lcon[r];
    ucon_s[r] = row_scale[r] * ucon[r];
  }
  const auto nt = static_cast<size_t>(ntot_);
  auto& lb = hs_.lb; auto& ub = hs_.ub; auto& hl = hs_.hl; auto& hu = hs_.hu;
  lb.assign(nt, -kInf);
  ub.assign(nt, kInf);
  hl.assign(nt, 0);
  hu.assign(nt, 0);
  for (int64_t i = 0; i < nfree_; ++i) {
    const auto sl = static_cast<size_t>(free_slot[static_cast<size_t>(i)]);
    if (std::isfinite(xlo[sl])) {
      lb[static_cast<size_t>(i)] = xlo[sl];
      hl[static_cast<size_t>(i)] = 1;
    }
    if (std::isfinite(xhi[sl])) {
      ub[static_cast<size_t>(i)] = xhi[sl];
      hu[static_cast<size_t>(i)] = 1;
    }
  }
  for (int64_t k = 0; k < nslack_; ++k) {
    const auto r = static_cast<size_t>(slack_of[static_cast<size_t>(k)]);
    const auto i = static_cast<size_t>(nfree_ + k);
    if (std::isfinite(lcon_s[r])) {
      lb[i] = lcon_s[r];
      hl[i] = 1;
    }
    if (std::isfinite(ucon_s[r])) {
      ub[i] = ucon_s[r];
      hu[i] = 1;
    }
  }
  const double relax = std::min(o_.bound_relax_factor, o_.tol);
  if (relax > 0.0)
    for (size_t i = 0; i < nt; ++i) {
      if (hl[i]) lb[i] -= relax * std::max(1.0, std::abs(lb[i]));
      if (hu[i]) ub[i] += relax * std::max(1.0, std::abs(ub[i]));
    }

  // Solver::initialize_iterate (solver.cpp:172-206)
  auto& x = hs_.x;
  x = x0;
  for (size_t sl = 0; sl < nv; ++sl)
    if (xlo[sl] == xhi[sl]) x[sl] = xlo[sl];
  auto push_into = [](double v, double l, double u) {
    const double w = std::min(1.0, u - l);
    const double lo = std::isfinite(l) ? l + kPushIn * (std::isfinite(w) ? w : 1.0) : -kInf;
    const double hi = std::isfinite(u) ? u - kPushIn * (std::isfinite(w) ? w : 1.0) : kInf;
    return std::clamp(v, lo, hi);
  };
  for (int64_t i = 0; i < nfree_; ++i) {
    const auto sl = static_cast<size_t>(free_slot[static_cast<size_t>(i)]);
    x[sl] = push_into(x[sl], lb[static_cast<size_t>(i)], ub[static_cast<size_t>(i)]);
  }

  lap("bounds + start");
  // device state (allocated on the first run, reused by later instances)
  if (!allocated_) {
    allocated_ = true;
    alloc_state(nv, mc);
  }
  lap("alloc state");
  free_slot_.upload(free_slot, s_);
  dual_row_.upload(dual_row, s_);
  slack_index_.upload(slack, s_);
  lb_.upload(lb, s_);
  ub_.upload(ub, s_);
  has_lb_.upload(hl, s_);
  has_ub_.upload(hu, s_);
  lcon_s_.upload(lcon_s, s_);
  P_.nvar = nvar_;
  P_.m_con = mcon_;
  P_.n_free = nfree_;
  P_.n_slack = nslack_;
  P_.ntot = ntot_;
  P_.m = m_;
  P_.free_slot = free_slot_.p;
  P_.dual_row = dual_row_.p;
  P_.slack_index = slack_index_.p;
  P_.lb = lb_.p;
  P_.ub = ub_.p;
  P_.has_lb = has_lb_.p;
  P_.has_ub = has_ub_.p;
  P_.lcon_s = lcon_s_.p;
  x_->upload(x, s_);

  lap("uploads");
  // slacks from the constraint values at the start point, multipliers
  auto& c = hs_.c;
  eval_c(x_->p, c_->p);
  c_->download(c, s_);
  auto& s = hs_.s;
  s.resize(static_cast<size_t>(nslack_));
  for (int64_t k = 0; k < nslack_; ++k) {
    const auto r = static_cast<size_t>(slack_of[static_cast<size_t>(k)]);
    const auto i = static_cast<size_t>(nfree_ + k);
    s[static_cast<size_t>(k)] = push_into(c[r], lb[i], ub[i]);
  }
  s_v_->upload(s, s_);
  auto& zl = hs_.zl; auto& zu = hs_.zu;
  zl.assign(nt, 0.0);
  zu.assign(nt, 0.0);
  for (size_t i = 0; i < nt; ++i) {
    const double v = static_cast<int64_t>(i) < nfree_ ? x[static_cast<size_t>(free_slot[i])]
                                                      : s[i - static_cast<size_t>(nfree_)];
    if (hl[i]) zl[i] = mu_ / (v - lb[i]);
    if (hu[i]) zu[i] = mu_ / (ub[i] - v);
  }
  zl_.upload(zl, s_);
  zu_.upload(zu, s_);
  ckc(cudaMemsetAsync(lambda_.p, 0, std::max<size_t>(static_cast<size_t>(m_), 1) * sizeof(double), s_), "memset");
  ckc(cudaStreamSynchronize(s_), "sync");
  lap("slacks + duals");
}

void DeviceSolver::dump_iterate(int iter, double alpha_max, double dphi) {
  const char* dir = std::getenv("OCG_IPM_DUMP");
  const char* which = std::getenv("OCG_IPM_DUMP_ITERS");
  if (!dir || !which) return;
  bool hit = false;
  for (const char* p = which; *p;) {
    if (std::atoi(p) == iter) hit = true;
    while (*p && *p != ',') ++p;
    if (*p == ',') ++p;
  }
  if (!hit) return;
  const std::string base = std::string(dir) + "/it" + std::to_string(iter) + "_";
  auto put = [&](const char* name, const void* dev, size_t bytes) {
    std::vector<char> h(bytes);
    if (bytes) ckc(cudaMemcpyAsync(h.data(), dev, bytes, cudaMemcpyDeviceToHost, s_), "dump d2h");
    ckc(cudaStreamSynchronize(s_), "sync");
    if (FILE* f = std::fopen((base + name).c_str(), "wb")) {
      if (bytes) std::fwrite(h.data(), 1, bytes, f);
      std::fclose(f);
    }
  };
  const size_t D = sizeof(double);
  put("x.f64", x_->p, static_cast<size_t>(nvar_) * D);
  put("s.f64", s_v_->p, static_cast<size_t>(nslack_) * D);
  put("zl.f64", zl_.p, static_cast<size_t>(ntot_) * D);
  put("zu.f64", zu_.p, static_cast<size_t>(ntot_) * D);
  put("lambda.f64", lambda_.p, static_cast<size_t>(m_) * D);
  put("grad.f64", grad_->p, static_cast<size_t>(nvar_) * D);
  put("jtlam.f64", jtlam_.p, static_cast<size_t>(ntot_) * D);
  put("g.f64", g_.p, static_cast<size_t>(m_) * D);
  put("c.f64", c_->p, static_cast<size_t>(mcon_) * D);
  put("step.f64", step_.p, static_cast<size_t>(dim_) * D);
  put("sigma.f64", sigma_.p, static_cast<size_t>(ntot_) * D);
  put("rhs.f64", rhs_.p, static_cast<size_t>(dim_) * D);
  put("free_slot.i64", free_slot_.p, static_cast<size_t>(nfree_) * sizeof(int64_t));
  put("dual_row.i64", dual_row_.p, static_cast<size_t>(m_) * sizeof(int64_t));
  put("slack_index.i64", slack_index_.p, static_cast<size_t>(mcon_) * sizeof(int64_t));
  put("lb.f64", lb_.p, static_cast<size_t>(ntot_) * D);
  put("ub.f64", ub_.p, static_cast<size_t>(ntot_) * D);
  put("has_lb.i8", has_lb_.p, static_cast<size_t>(ntot_));
  put("has_ub.i8", has_ub_.p, static_cast<size_t>(ntot_));
  put("lcon_s.f64", lcon_s_.p, static_cast<size_t>(mcon_) * D);
  // the remaining kernels on scratch copies (the solver's state is untouched)
  double p5[5] = {0, 0, 0, 0, 0};
  ocg::ipmdev::kkt_error_parts(P_, x_->p, s_v_->p, zl_.p, zu_.p, lambda_.p, grad_->p, jtlam_.p, g_.p, mu_, p5, sc_, s_);
  double bar = 0.0;
  const bool bar_ok = ocg::ipmdev::barrier(P_, x_->p, s_v_->p, bar, sc_, s_);
  const double theta = theta_of(g_.p);
  DVec<double> dzl(static_cast<size_t>(std::max<int64_t>(1, ntot_))), dzu(static_cast<size_t>(std::max<int64_t>(1, ntot_)));
  const double alpha_z = ocg::ipmdev::dual_direction(P_, x_->p, s_v_->p, zl_.p, zu_.p, step_.p, mu_, tau_, dzl.p, dzu.p,
                                                     sc_, s_);
  put("dzl.f64", dzl.p, static_cast<size_t>(ntot_) * D);
  put("dzu.f64", dzu.p, static_cast<size_t>(ntot_) * D);
  // a trial point at alpha_max and the accepted multipliers there
  DVec<double> xn(static_cast<size_t>(std::max<int64_t>(1, nvar_))), sn(static_cast<size_t>(std::max<int64_t>(1, nslack_)));
  DVec<double> lam2(static_cast<size_t>(std::max<int64_t>(1, m_))), zl2(static_cast<size_t>(std::max<int64_t>(1, ntot_))),
      zu2(static_cast<size_t>(std::max<int64_t>(1, ntot_)));
  ckc(cudaMemcpyAsync(xn.p, x_->p, static_cast<size_t>(nvar_) * D, cudaMemcpyDeviceToDevice, s_), "copy");
  ckc(cudaMemcpyAsync(lam2.p, lambda_.p, static_cast<size_t>(m_) * D, cudaMemcpyDeviceToDevice, s_), "copy");
  ckc(cudaMemcpyAsync(zl2.p, zl_.p, static_cast<size_t>(ntot_) * D, cudaMemcpyDeviceToDevice, s_), "copy");
  ckc(cudaMemcpyAsync(zu2.p, zu_.p, static_cast<size_t>(ntot_) * D, cudaMemcpyDeviceToDevice, s_), "copy");
  ocg::ipmdev::trial(P_, x_->p, s_v_->p, step_.p, alpha_max, xn.p, sn.p, s_);
  const double az = std::min(alpha_z, std::max(alpha_max, 1e-2));
  ocg::ipmdev::accept(P_, step_.p, dzl.p, dzu.p, alpha_max, az, mu_, kKappaSigma, xn.p, sn.p, lam2.p, zl2.p, zu2.p, s_);
  put("x_trial.f64", xn.p, static_cast<size_t>(nvar_) * D);
  put("s_trial.f64", sn.p, static_cast<size_t>(nslack_) * D);
  put("lambda_acc.f64", lam2.p, static_cast<size_t>(m_) * D);
  put("zl_acc.f64", zl2.p, static_cast<size_t>(ntot_) * D);
  put("zu_acc.f64", zu2.p, static_cast<size_t>(ntot_) * D);
  if (FILE* f = std::fopen((base + "meta.json").c_str(), "w")) {
    std::fprintf(f,
                 "{\"iter\": %d, \"nvar\": %lld, \"m_con\": %lld, \"n_free\": %lld, \"n_slack\": %lld, "
                 "\"ntot\": %lld, \"m\": %lld, \"dim\": %lld, \"mu\": %.17g, \"tau\": %.17g, "
                 "\"alpha_max\": %.17g, \"dphi\": %.17g, \"kkt_parts\": [%.17g, %.17g, %.17g, %.17g, %.17g], "
                 "\"barrier\": %.17g, \"barrier_ok\": %s, \"theta\": %.17g, \"alpha_z\": %.17g, "
                 "\"alpha_z_used\": %.17g, \"kappa_sigma\": %.17g}\n",
                 iter, static_cast<long long>(nvar_), static_cast<long long>(mcon_), static_cast<long long>(nfree_),
                 static_cast<long long>(nslack_), static_cast<long long>(ntot_), static_cast<long long>(m_),
                 static_cast<long long>(dim_), mu_, tau_, alpha_max, dphi, p5[0], p5[1], p5[2], p5[3], p5[4], bar,
                 bar_ok ? "true" : "false", theta, alpha_z, az, kKappaSigma);
    std::fclose(f);
  }
}

// Solver::kkt_error (solver.cpp:260-287)
double DeviceSolver::kkt_error(double mu, const double* g, double& comp_out, double& stat_out) {
  double p[5];
  ocg::ipmdev::kkt_error_parts(P_, x_->p, s_v_->p, zl_.p, zu_.p, lambda_.p, grad_->p, jtlam_.p, g, mu, p, sc_, s_);
  const double znorm1 = p[0], lnorm1 = p[1], stat = p[2], feas = p[3], comp = p[4];
  const double denom = static_cast<double>(std::max<int64_t>(1, m_ + ntot_));
  const double sd = std::max(100.0, (lnorm1 + znorm1) / denom) / 100.0;
  const double sc = std::max(100.0, znorm1 / static_cast<double>(std::max<int64_t>(1, ntot_))) / 100.0;
  comp_out = comp / sc;
  stat_out = stat / sd;
  return std::max({stat / sd, feas, comp / sc});
}

void DeviceSolver::add_to_filter(double theta, double phi) {
  const std::pair<double, double> e{(1.0 - kGammaTheta) * theta, phi - kGammaPhi * theta};
  filter_.erase(std::remove_if(filter_.begin(), filter_.end(),
                               [&](const auto& f) { return f.first >= e.first && f.second >= e.second; }),
                filter_.end());
  filter_.push_back(e);
}

bool DeviceSolver::filter_rejects(double theta, double phi) const {
  if (theta > theta_max_) return true;
  for (const auto& f : filter_)
    if (theta >= f.first && phi >= f.second) return true;
  return false;
}

// sparse::refine (ldl.cpp:249-272) when the first solve's residual is large
void DeviceSolver::refine_if_needed(const double* rhs, double* step) {
  double nr[3];
  cko(ocg_kkt_matvec(kkt_, step, kx_.p, s_), "matvec");
  ocg::ipmdev::residual_norms(rhs, kx_.p, step, dim_, ntot_, dw_, dc_, nullptr, nr, sc_, s_);
  if (!(nr[0] > o_.refine_trigger * (1.0 + nr[1]))) return;
  double anorm = 0.0;
  cko(ocg_kkt_norm_inf(kkt_, dscal_.p, s_), "norm_inf");
  ckc(cudaMemcpyAsync(&anorm, dscal_.p, sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H");
  ckc(cudaStreamSynchronize(s_), "sync");
  anorm += std::abs(dw_) + std::abs(dc_);
  for (int round = 0; round < o_.refine_rounds; ++round) {
    cko(ocg_kkt_matvec(kkt_, step, kx_.p, s_), "matvec");
    ocg::ipmdev::residual_norms(rhs, kx_.p, step, dim_, ntot_, dw_, dc_, r_v_.p, nr, sc_, s_);
    if (nr[0] <= 1e-12 * (anorm * nr[2] + nr[1])) break;
    cko(ocg_ldl_solve(ldl_, r_v_.p, dx_.p, s_), "ldl_solve");
    ++n_refine_;
    ocg::ipmdev::add(step, dx_.p, dim_, s_);
  }
}

// Solver::solve_kkt (solver.cpp:648-702): inertia-corrected factorization,
// solve into step_
bool DeviceSolver::solve_kkt(double wmax, bool& numeric_failure) {
  numeric_failure = false;
  Clock tf;
  double dw = 0.0, dc = 0.0;
  bool first_bump = true;
  // the reference's next regularization after a rejected inertia `in`
  auto next_delta = [&](const int64_t* in) {
    if (first_bump) {
      dw = delta_last_ > 0.0 ? std::max(1e-20, delta_last_ / o_.reg_shrink)
                             : o_.reg_initial_scale * std::max(1.0, wmax);
      first_bump = false;
    } else if (in[2] > 0 && dc == 0.0) {
      dc = o_.reg_dual_scale * std::pow(mu_, o_.reg_dual_power);
    } else {
      dw *= o_.reg_grow;
    }
  };
  auto accepted = [&](const int64_t* in) { return in[0] == ntot_ && in[1] == m_ && in[2] == 0; };
  bool done = false;
  if (speculate_) {
    // Reference order: the factorization is one sequential chain on one SM,
    // so the first four attempts of the reference's decision tree run
    // concurrently — (0, 0); (dw1, 0); then (dw1, dc1) if that one found zero
    // pivots, else (dw1 grow, 0) — and the walk below takes exactly the
    // sequential loop's decisions over their inertias; factorizations counts
    // the attempts the sequential loop would have made.
    const double dw1 = delta_last_ > 0.0 ? std::max(1e-20, delta_last_ / o_.reg_shrink)
                                         : o_.reg_initial_scale * std::max(1.0, wmax);
    const double dc1 = o_.reg_dual_scale * std::pow(mu_, o_.reg_dual_power);
    const double cdw[4] = {0.0, dw1, dw1, dw1 * o_.reg_grow}, cdc[4] = {0.0, 0.0, dc1, 0.0};
    int nc = 4;
    while (nc > 1 && cdw[nc - 1] > o_.reg_max_delta) --nc;
    int64_t in[4][3];
    cko(ocg_ldl_factor_many(ldl_, nc, cdw, cdc, &in[0][0], s_), "ldl_factor_many");
    r_speculative_ += nc;
    int cur = 0;
    for (;;) {
      ++r_.factorizations;
      if (accepted(in[cur])) {
        cko(ocg_ldl_select(ldl_, cur), "ldl_select");
        done = true;
        break;
      }
      next_delta(in[cur]);
      if (dw > o_.reg_max_delta) {
        numeric_failure = true;
        r_.time_factorize += tf.elapsed();
        return false;
      }
      int nxt = -1;
      for (int i = cur + 1; i < nc; ++i)
        if (cdw[i] == dw && cdc[i] == dc && (cur > 0 || i == 1) && (cur != 1 || i >= 2)) {
          nxt = i;
          break;
        }
      if (nxt < 0) break;  // past the speculated attempts: on sequentially from (dw, dc)
      cur = nxt;
    }
  }
  while (!done) {
    int64_t in[3];
    cko(ocg_ldl_factor(ldl_, dw, dc, in, s_), "ldl_factor");
    ++r_.factorizations;
    if (accepted(in)) break;
    next_delta(in);
    if (dw > o_.reg_max_delta) {
      numeric_failure = true;
      r_.time_factorize += tf.elapsed();
      return false;
    }
  }
  if (dw > 0.0) delta_last_ = dw;
  dw_ = dw;
  dc_ = dc;
  r_.time_factorize += tf.elapsed();
  Clock ts;
  cko(ocg_ldl_solve(ldl_, rhs_.p, step_.p, s_), "ldl_solve");
  ++n_solves_;
  refine_if_needed(rhs_.p, step_.p);
  ckc(cudaStreamSynchronize(s_), "sync");
  r_.time_solve += ts.elapsed();
  return true;
}

// Solver::resolve_rhs (solver.cpp:704-721): solve with the current factor
void DeviceSolver::resolve(const double* rhs, double* step) {
  Clock ts;
  cko(ocg_ldl_solve(ldl_, rhs, step, s_), "ldl_solve");
  ++n_solves_;
  refine_if_needed(rhs, step);
  ckc(cudaStreamSynchronize(s_), "sync");
  r_.time_solve += ts.elapsed();
}

void DeviceSolver::finish(int status, int iter, const std::vector<double>& row_scale) {
  r_.status = status;
  r_.iterations = iter;
  double f = 0.0;
  eval_f(x_->p, f);
  const double f_raw = f / obj_scale_;
  int maximize = 0;
  {
    // the model's objective sense: structure JSON carries it; read cheaply
    char* js = ocg_model_structure_json(model_);
    if (js) {
      maximize = std::string(js).find("\"maximize\":true") != std::string::npos ? 1 : 0;
      ocg_free(js);
    }
  }
  r_.objective = maximize ? -f_raw : f_raw;
  if (m_ > 0) {
    std::vector<double> g;
    g_.download(g, s_);
    std::vector<int64_t> dr(static_cast<size_t>(m_));
    ckc(cudaMemcpy(dr.data(), dual_row_.p, dr.size() * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    double th = 0.0;
    for (size_t d = 0; d < g.size(); ++d) th = std::max(th, std::abs(g[d]) / row_scale[static_cast<size_t>(dr[d])]);
    r_.theta = th;
  }
  cko(ocg_kkt_jt_lambda(kkt_, lambda_.p, jtlam_.p, s_), "jt_lambda");
  double comp = 0.0, stat = 0.0;
  kkt_error(0.0, g_.p, comp, stat);
  r_.stationarity = stat / obj_scale_;
  r_.complementarity = comp / obj_scale_;
}

int DeviceSolver::run_with_retry(ocg_ipm_result* res, double* x_out) {
  use_retry_ldl_ = false;
  int rc = run(res, x_out);
  const char* e = std::getenv("OCG_IPM_RETRY");
  if (rc != OCG_OK || (e && std::atoi(e) == 0) || o_.kkt_order == OCG_LDL_REFERENCE) return rc;
  if (res->status != 2 && res->status != 3) return rc;
  int64_t li[5];
  cko(ocg_ldl_info(ldl_, li), "ldl_info");
  const int64_t target = std::max<int64_t>(1, li[1] / 4);
  if (li[1] <= 1) return rc;
  if (!ldl_retry_) cko(ocg::hd::ldl_create(kkt_, static_cast<int>(target), &ldl_retry_), "ldl_create (retry)");
  const ocg_ipm_result first = *res;
  use_retry_ldl_ = true;
  rc = run(res, x_out);
  use_retry_ldl_ = false;
  res->time_total += first.time_total;
  if (std::getenv("OCG_TIMING"))
    std::fprintf(stderr, "[ipm] band path: status %d with %lld segments, retried with %lld: status %d\n", first.status,
                 static_cast<long long>(li[1]), static_cast<long long>(target), res->status);
  return rc;
}

int DeviceSolver::run(ocg_ipm_result* res, double* x_out) {
  Clock total;
  {
    // fresh per-run state; the plan timings stay with the context
    const double pe = r_.time_plan_eval, pk = r_.time_plan_kkt, pl = r_.time_plan_ldl;
    r_ = ocg_ipm_result{};
    r_.time_plan_eval = pe;
    r_.time_plan_kkt = pk;
    r_.time_plan_ldl = pl;
    filter_.clear();
    r_speculative_ = 0;
    n_solves_ = n_refine_ = n_trials_ = 0;
    t_err_ = t_assemble_ = t_pre_ = t_search_ = t_accept_ = 0.0;
    delta_last_ = 0.0;
    dw_ = dc_ = 0.0;
    theta_min_ = 0.0;
    theta_max_ = kInf;
  }
  select_ldl();
  std::vector<double> row_scale;
  mu_ = o_.mu_init;
  tau_ = std::max(o_.tau_min, 1.0 - mu_);
  setup(row_scale);
  r_.time_setup = total.elapsed();
  if (contradictory_) {
    r_.status = 2;
    r_.time_total = total.elapsed();
    *res = r_;
    return OCG_OK;
  }
  const double mu_min = o_.tol / 10.0;
  auto done = [&](int status, int iter) {
    finish(status, iter, row_scale);
    r_.time_total = total.elapsed();
    if (x_out) ckc(cudaMemcpy(x_out, x_->p, static_cast<size_t>(nvar_) * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    int64_t li[5];
    ocg_ldl_info(ldl_, li);
    r_.bandwidth = li[2];
    *res = r_;
    if (std::getenv("OCG_TIMING"))
      std::fprintf(stderr,
                   "[ipm] %d iterations: total %.3f s, factorize %.3f s (%d; %lld speculative), solve %.3f s (%lld "
                   "solves + %lld refinement rounds), derivatives %.3f s, %lld line-search trials\n",
                   iter, r_.time_total, r_.time_factorize, r_.factorizations, r_speculative_, r_.time_solve, n_solves_,
                   n_refine_, r_.time_derivatives, n_trials_);
    if (std::getenv("OCG_TIMING"))
      std::fprintf(stderr,
                   "[ipm] phases: kkt error + mu %.3f s, H + assembly + rhs %.3f s, step stats %.3f s, line search "
                   "%.3f s, accept %.3f s\n",
                   t_err_, t_assemble_, t_pre_, t_search_, t_accept_);
  };
  if (!eval_cj(x_->p, c_->p) || !eval_grad(x_->p, grad_->p)) {
    done(3, 0);
    return OCG_OK;
  }
  ocg::ipmdev::residual(P_, c_->p, s_v_->p, g_.p, s_);
  {
    const double th = theta_of(g_.p);
    theta_min_ = 1e-4 * std::max(1.0, th);
    theta_max_ = 1e4 * std::max(1.0, th);
  }
  int consecutive_restorations = 0;
  bool hold_mu = false;
  for (int iter = 0;; ++iter) {
    Clock ph;
    auto mark = [&](double& acc) {
      acc += ph.elapsed();
      ph = Clock();
    };
    cko(ocg_kkt_jt_lambda(kkt_, lambda_.p, jtlam_.p, s_), "jt_lambda");
    double comp = 0.0, stat = 0.0;
    const double e0 = kkt_error(0.0, g_.p, comp, stat);
    if (e0 <= o_.tol) {
      done(0, iter);
      return OCG_OK;
    }
    if (iter >= o_.max_iter) {
      done(1, iter);
      return OCG_OK;
    }
    {
      double cmu = 0.0, smu = 0.0;
      if (!hold_mu && mu_ > mu_min && kkt_error(mu_, g_.p, cmu, smu) <= kKappaEps * mu_) {
        mu_ = std::max(mu_min, std::min(kKappaMu * mu_, std::pow(mu_, kThetaMu)));
        tau_ = std::max(o_.tau_min, 1.0 - mu_);
        filter_.clear();
      }
    }
    mark(t_err_);
    ocg::ipmdev::expand_lambda(P_, lambda_.p, lamfull_.p, s_);
    if (!eval_h(x_->p, lamfull_.p)) {
      done(3, iter);
      return OCG_OK;
    }
    ocg::ipmdev::sigma(P_, x_->p, s_v_->p, zl_.p, zu_.p, sigma_.p, s_);
    cko(ocg_kkt_assemble(kkt_, sigma_.p, s_), "kkt_assemble");
    ocg::ipmdev::rhs(P_, x_->p, s_v_->p, grad_->p, jtlam_.p, g_.p, mu_, rhs_.p, s_);
    const double wmax = max_abs_h();
    mark(t_assemble_);
    bool numeric_failure = false;
    if (!solve_kkt(wmax, numeric_failure)) {
      done(3, iter);
      return OCG_OK;
    }
    ph = Clock();
    const double alpha_max = ocg::ipmdev::fraction_to_boundary(P_, x_->p, s_v_->p, step_.p, tau_, sc_, s_);
    const double dphi = ocg::ipmdev::dphi(P_, x_->p, s_v_->p, grad_->p, step_.p, mu_, sc_, s_);
    if (std::getenv("OCG_IPM_DUMP")) dump_iterate(iter, alpha_max, dphi);
    const double theta_k = theta_of(g_.p);
    double phi_k = 0.0;
    {
      double f_k = 0.0, bar = 0.0;
      if (!eval_f(x_->p, f_k) || !ocg::ipmdev::barrier(P_, x_->p, s_v_->p, bar, sc_, s_)) {
        done(3, iter);
        return OCG_OK;
      }
      phi_k = f_k - mu_ * bar;
    }

    mark(t_pre_);
    double alpha = alpha_max;
    bool accepted = false, armijo_path = false, saw_eval_error = false;
    double theta_t = 0.0, phi_t = 0.0;
    const double* dir = step_.p;
    // the trial point and its evaluation replay as one CUDA graph per
    // (iterate, trial buffer, direction) pointer set; the step length goes
    // in through a page-locked slot the graph copies to the device first
    const double* trial_dir = step_.p;
    double trial_alpha = 0.0;
    auto build_trial = [&](const double* d, double a) {
      trial_dir = d;
      trial_alpha = a;
      if (!graphs_) ocg::ipmdev::trial(P_, x_->p, s_v_->p, d, a, xt_->p, st_->p, s_);
    };
    // one host round trip per trial: c, residual, theta, barrier and f are
    // launched back to back and their scalars and finiteness flags come back
    // together; the decisions below are the sequential ones (solver.cpp:444-455)
    auto enqueue_eval = [&]() {
      cko(ocg_eval_constraints(ev_, xt_->p, ct_->p, s_), "eval_constraints");
      cko(ocg_eval_status_async(ev_, &hpin_->flag_c, s_), "status");
      ocg::ipmdev::residual(P_, ct_->p, st_->p, gt_.p, s_);
      ocg::ipmdev::l1_async(gt_.p, m_, sc_, dscal_.p, s_);
      ocg::ipmdev::barrier_async(P_, xt_->p, st_->p, sc_, dscal_.p + 1, s_);
      cko(ocg_eval_objective(ev_, xt_->p, dscal_.p + 3, s_), "eval_objective");
      cko(ocg_eval_status_async(ev_, &hpin_->flag_f, s_), "status");
      ckc(cudaMemcpyAsync(hpin_->v, dscal_.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H trial");
    };
    auto eval_trial = [&]() {
      ++n_trials_;
      Clock t;
      if (graphs_) {
        hpin_->alpha = trial_alpha;
        const TrialKey key{x_->p, xt_->p, s_v_->p, st_->p, trial_dir, ct_->p};
        cudaGraphExec_t& ge = trial_graphs_[key];
        if (!ge) {
          cudaGraph_t g = nullptr;
          ckc(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal), "capture");
          ckc(cudaMemcpyAsync(dscal_.p + 4, &hpin_->alpha, sizeof(double), cudaMemcpyHostToDevice, s_), "alpha");
          ocg::ipmdev::trial_dev(P_, x_->p, s_v_->p, trial_dir, dscal_.p + 4, xt_->p, st_->p, s_);
          enqueue_eval();
          ckc(cudaStreamEndCapture(s_, &g), "end capture");
          ckc(cudaGraphInstantiate(&ge, g, 0), "instantiate");
          cudaGraphDestroy(g);
        }
        ckc(cudaGraphLaunch(ge, s_), "graph launch");
      } else {
        enqueue_eval();
      }
      ckc(cudaStreamSynchronize(s_), "sync");
      r_.time_derivatives += t.elapsed();
      if (hpin_->flag_c) return false;
      theta_t = hpin_->v[0];
      const double bar = hpin_->v[1], f_t = hpin_->v[3];
      if (hpin_->v[2] != 0.0 || hpin_->flag_f || !std::isfinite(f_t)) return false;
      phi_t = f_t - mu_ * bar;
      return std::isfinite(phi_t);
    };
    auto acceptable = [&](double a) {
      if (filter_rejects(theta_t, phi_t)) return false;
      const bool descent = dphi < 0.0;
      const bool switching = descent && a * std::pow(-dphi, kSPhi) > kDeltaSwitch * std::pow(theta_k, kSTheta);
      if (theta_k <= theta_min_ && switching) {
        if (phi_t <= phi_k + kEtaPhi * a * dphi) {
          armijo_path = true;
          return true;
        }
        return false;
      }
      return theta_t <= (1.0 - kGammaTheta) * theta_k || phi_t <= phi_k - kGammaPhi * theta_k;
    };

    bool first_trial = true;
    while (alpha >= kAlphaMin) {
      build_trial(dir, alpha);
      if (!eval_trial()) {
        saw_eval_error = true;
        first_trial = false;
        alpha *= 0.5;
        continue;
      }
      accepted = acceptable(alpha);
      if (!accepted && first_trial && theta_t >= theta_k && m_ > 0) {
        // second-order corrections (solver.cpp:496-534)
        ocg::ipmdev::axpy(alpha, g_.p, gt_.p, gsoc_.p, m_, s_);
        double theta_prev = theta_t;
        for (int soc = 0; soc < 4 && !accepted; ++soc) {
          ocg::ipmdev::rhs_soc(P_, rhs_.p, gsoc_.p, rhs2_.p, s_);
          resolve(rhs2_.p, step2_.p);
          const double alpha_soc = ocg::ipmdev::fraction_to_boundary(P_, x_->p, s_v_->p, step2_.p, tau_, sc_, s_);
          build_trial(step2_.p, alpha_soc);
          if (!eval_trial()) break;
          if (acceptable(alpha_soc)) {
            accepted = true;
            step_.swap(step2_);
            dir = step_.p;
            alpha = alpha_soc;
            break;
          }
          if (theta_t >= 0.99 * theta_prev) break;
          theta_prev = theta_t;
          ocg::ipmdev::axpy(alpha_soc, gsoc_.p, gt_.p, gsoc_.p, m_, s_);
        }
        if (!accepted) {
          build_trial(dir, alpha);
          if (!eval_trial()) {
            saw_eval_error = true;
            first_trial = false;
            alpha *= 0.5;
            continue;
          }
        }
      }
      if (accepted) {
        if (!eval_cj(xt_->p, ct_->p) || !eval_grad(xt_->p, gradt_->p)) {
          saw_eval_error = true;
          accepted = false;
          armijo_path = false;
          first_trial = false;
          alpha *= 0.5;
          continue;
        }
        break;
      }
      first_trial = false;
      alpha *= 0.5;
    }

    if (!accepted) {
      if (consecutive_restorations >= 5) {
        done(saw_eval_error ? 3 : 2, iter);
        return OCG_OK;
      }
      ++consecutive_restorations;
      hold_mu = true;
      mu_ = std::min(mu_ * 10.0, 1e4);
      tau_ = std::max(o_.tau_min, 1.0 - mu_);
      filter_.clear();
      if (!eval_cj(x_->p, c_->p) || !eval_grad(x_->p, grad_->p)) {
        done(3, iter);
        return OCG_OK;
      }
      ocg::ipmdev::residual(P_, c_->p, s_v_->p, g_.p, s_);
      continue;
    }
    mark(t_search_);
    consecutive_restorations = 0;
    hold_mu = false;
    if (!armijo_path) add_to_filter(theta_k, phi_k);

    double alpha_z = ocg::ipmdev::dual_direction(P_, x_->p, s_v_->p, zl_.p, zu_.p, dir, mu_, tau_, dzl_.p, dzu_.p,
                                                 sc_, s_);
    alpha_z = std::min(alpha_z, std::max(alpha, 1e-2));
    std::swap(x_, xt_);
    std::swap(s_v_, st_);
    ocg::ipmdev::accept(P_, dir, dzl_.p, dzu_.p, alpha, alpha_z, mu_, kKappaSigma, x_->p, s_v_->p, lambda_.p, zl_.p,
                        zu_.p, s_);
    std::swap(c_, ct_);
    std::swap(grad_, gradt_);
    ocg::ipmdev::residual(P_, c_->p, s_v_->p, g_.p, s_);
    if (o_.verbose) {
      double f_raw = 0.0;
      eval_f(x_->p, f_raw);
      std::printf("iter %4d  f %+.8e  theta %.3e  mu %.2e  alpha %.2e  alpha_z %.2e  delta_w %.1e\n", iter + 1,
                  f_raw / obj_scale_, theta_of(g_.p), mu_, alpha, alpha_z, delta_last_);
    }
    mark(t_accept_);
  }
}

}  // namespace

struct ocg_ipm_ctx {
  std::unique_ptr<DeviceSolver> solver;
};

namespace {

// Process-wide plans of ocg_ipm_solve, per (model, device): the evaluation
// plan, the KKT pattern and the factorization plans are built by the first
// solve and reused by the next ones, as an ocg_ipm_ctx would. Dropped when
// the model is destroyed (ocg_model_destroy) or by ocg_release_cached_memory;
// OCG_IPM_PLAN_CACHE=0 turns the cache off.
struct PlanCacheEntry {
  std::mutex mu;  // held while a solve uses the plans
  std::unique_ptr<DeviceSolver> solver;
};
std::mutex g_plan_mu;
std::map<std::pair<const ocg_model*, int>, std::shared_ptr<PlanCacheEntry>>& plan_cache() {
  static auto* c = new std::map<std::pair<const ocg_model*, int>, std::shared_ptr<PlanCacheEntry>>;
  return *c;
}
std::shared_ptr<PlanCacheEntry> plan_cache_entry(const ocg_model* m, int device) {
  if (const char* e = std::getenv("OCG_IPM_PLAN_CACHE"); e && std::atoi(e) == 0) return nullptr;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto& c = plan_cache();
  auto& slot = c[{m, device}];
  if (!slot) slot = std::make_shared<PlanCacheEntry>();
  return slot;
}

}  // namespace

namespace ocg::hd {
// drop the cached solve plans of model m (every device; all models when m is NULL)
void drop_ipm_plans(const ocg_model* m) {
  std::vector<std::shared_ptr<PlanCacheEntry>> gone;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto& c = plan_cache();
    for (auto it = c.begin(); it != c.end();) {
      if (!m || it->first.first == m) {
        gone.push_back(it->second);
        it = c.erase(it);
      } else {
        ++it;
      }
    }
  }
  for (auto& e : gone) {
    std::lock_guard<std::mutex> lk(e->mu);  // wait for a solve in flight
    e->solver.reset();
  }
}
}  // namespace ocg::hd

extern "C" {

void ocg_ipm_default_options(ocg_ipm_options* o) {
  if (!o) return;
  o->tol = 1e-8;
  o->max_iter = 3000;
  o->mu_init = 1e-1;
  o->tau_min = 0.99;
  o->reg_initial_scale = 1e-4;
  o->reg_grow = 8.0;
  o->reg_shrink = 3.0;
  o->reg_dual_scale = 1e-8;
  o->reg_dual_power = 0.25;
  o->reg_max_delta = 1e40;
  o->scale = 1;
  o->bound_relax_factor = 1e-8;
  o->refine_rounds = 5;
  o->refine_trigger = 1e-8;
  o->verbose = 0;
  o->kkt_order = OCG_LDL_BAND;
}



int ocg_ipm_ctx_create(ocg_model* m, int device, ocg_ipm_ctx** out) {
  if (!m || !out) return ocg::hd::set_error(OCG_ERR_ARG, "ocg_ipm_ctx_create: null argument");
  try {
    ocg::mem::DeviceScope ds(device);
    ocg_ipm_options o;
    ocg_ipm_default_options(&o);
    auto c = std::make_unique<ocg_ipm_ctx>();
    c->solver = std::make_unique<DeviceSolver>(m, o, device);
    *out = c.release();
    return OCG_OK;
  } catch (const std::exception& ex) {
    return ocg::hd::set_error(OCG_ERR_CUDA, std::string("ocg_ipm_ctx_create: ") + ex.what());
  }
}

void ocg_ipm_ctx_destroy(ocg_ipm_ctx* c) { delete c; }  // ~DeviceSolver makes its device current

int ocg_ipm_ctx_solve(ocg_ipm_ctx* c, const ocg_ipm_options* opts, const double* lvar, const double* uvar,
                      const double* x_start, const double* lcon, const double* ucon, ocg_ipm_result* out,
                      double* x_out) {
  if (!c || !out) return ocg::hd::set_error(OCG_ERR_ARG, "ocg_ipm_ctx_solve: null argument");
  ocg_ipm_options o;
  ocg_ipm_default_options(&o);
  if (opts) o = *opts;
  try {
    ocg::mem::DeviceScope ds(c->solver->device());
    c->solver->set_instance(o, lvar, uvar, x_start, lcon, ucon);
    return c->solver->run_with_retry(out, x_out);
  } catch (const InvalidInstance& ex) {
    return ocg::hd::set_error(OCG_ERR_ARG, std::string("ocg_ipm_ctx_solve: ") + ex.what());
  } catch (const std::exception& ex) {
    return ocg::hd::set_error(OCG_ERR_CUDA, std::string("ocg_ipm_ctx_solve: ") + ex.what());
  }
}

int ocg_ipm_solve(ocg_model* m, const ocg_ipm_options* opts, int device, ocg_ipm_result* out, double* x_out) {
  if (!m || !out) return ocg::hd::set_error(OCG_ERR_ARG, "ocg_ipm_solve: null argument");
  ocg_ipm_options o;
  ocg_ipm_default_options(&o);
  if (opts) o = *opts;
  try {
    ocg::mem::DeviceScope ds(device);
    // plans of this model and device from a previous solve, unless another
    // thread is solving with them right now (then this solve builds its own)
    std::shared_ptr<PlanCacheEntry> e = plan_cache_entry(m, device);
    std::unique_lock<std::mutex> lk;
    if (e) lk = std::unique_lock<std::mutex>(e->mu, std::try_to_lock);
    if (e && lk.owns_lock()) {
      if (!e->solver) e->solver = std::make_unique<DeviceSolver>(m, o, device);
      e->solver->set_instance(o, nullptr, nullptr, nullptr, nullptr, nullptr);
      return e->solver->run_with_retry(out, x_out);
    }
    DeviceSolver solver(m, o, device);
    return solver.run_with_retry(out, x_out);
  } catch (const std::exception& ex) {
    return ocg::hd::set_error(OCG_ERR_CUDA, std::string("ocg_ipm_solve: ") + ex.what());
  }
}

}  // extern "C"
