// Batched device IPM: many independent instances of one transcribed structure
// (BASELINE config 5; SURVEY.md §8e "batched in one launch over instance x
// node", §8f item 4).
//
// Every instance runs the control flow of the single-instance solver
// (ipm.cpp, itself the reference's Solver::run, proj/src/ipm/solver.cpp:
// 304-702) as a C++20 coroutine: wherever the single solver would launch
// device work and wait for a scalar, the coroutine posts a request and
// suspends. A scheduler collects the requests of every instance, issues one
// launch sequence per request kind over all instances that asked for it (the
// generated evaluation kernels with a batch grid dimension, the batched vector
// kernels of batch_kernels.cu, the batched band LDL^T of band.cu), copies the
// per-instance scalars back once per round, and resumes the coroutines. The
// decisions per instance are exactly the single solver's; only the device
// launches are shared, so a batch of 4096 instances costs a few hundred
// launch rounds instead of 4096 x (thousands of launches).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <coroutine>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/octgpu.h"
#include "batch_kernels.hpp"
#include "handles.hpp"

namespace {
// an instance whose data do not fit the model's structure (OCG_ERR_ARG)
struct InvalidInstance : std::runtime_error {
  using std::runtime_error::runtime_error;
};
}  // namespace

namespace {

using ocg::Index;
using ocg::hd::ck;
namespace bd = ocg::bdev;

constexpr double kInf = std::numeric_limits<double>::infinity();
// filter line-search constants (solver.cpp:38-52), as in ipm.cpp
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

// request kinds; a kind fixes which buffers the launch reads and writes
enum Op : int {
  CJG_X,      // c, J, grad at x                         -> ok_cj, ok_grad
  CJG_T,      // same at the trial point (a0: step <- step2 first) -> ok_cj, ok_grad
  RESID_X,    // g = c - (s or lcon_s) at x              -> theta
  KKTERR,     // J^T lambda, kkt_error parts at mu = a0  -> 5 parts
  ITER,       // expand lambda, H, max|H|, sigma, K, rhs (mu = a0) -> ok_h, max|H|
  FACTOR,     // band LDL^T with (a0, a1) = (delta_w, delta_c) -> inertia
  SOLVE_0,    // rhs -> step, residual norms (a0, a1 = deltas) -> 3 norms
  SOLVE_1,    // rhs_soc -> rhs2 -> step2, residual norms
  NORMINF,    // ||K||_inf
  REFINE_0,   // residual r of step -> 3 norms
  REFINE_1,
  APPLY_0,    // step += K^-1 r, new residual -> 3 norms
  APPLY_1,
  LSPREP,     // alpha_max (tau a0), dphi (mu a1), theta, f(x), barrier(x)
  TRIAL_0,    // x_t = x + a0 * step: c, theta, barrier, f (mu a1)
  TRIAL_1,    // with step2
  GSOC_0,     // gsoc = a0 * g + g_t
  GSOC_1,     // gsoc = a0 * gsoc + g_t
  FTB2,       // alpha_soc = fraction to boundary along step2 (tau a0)
  DUALDIR,    // dz and alpha_z (mu a0, tau a1)
  ACCEPT,     // commit the trial point, update lambda / z (alpha a0, alpha_z a1, mu a2), residual
  FINISH,     // f(x), unscaled theta, kkt_error parts at mu 0
  NOPS
};
constexpr int kArgs = 4;  // per-request arguments (column-major in the staging buffer)
constexpr int kRes = 8;   // per-request results

struct Inst;
class Batch;

// ---- coroutine plumbing --------------------------------------------------------

struct Task {
  struct promise_type {
    std::exception_ptr ex;
    Task get_return_object() { return Task{std::coroutine_handle<promise_type>::from_promise(*this)}; }
    std::suspend_always initial_suspend() noexcept { return {}; }
    std::suspend_always final_suspend() noexcept { return {}; }
    void return_void() {}
    void unhandled_exception() { ex = std::current_exception(); }
  };
  std::coroutine_handle<promise_type> h;
  explicit Task(std::coroutine_handle<promise_type> hh) : h(hh) {}
  Task(Task&& o) noexcept : h(std::exchange(o.h, {})) {}
  Task(const Task&) = delete;
  ~Task() {
    if (h) h.destroy();
  }
};

// a child coroutine the parent co_awaits (symmetric transfer back on completion)
struct Sub {
  struct promise_type {
    std::coroutine_handle<> parent;
    std::exception_ptr ex;
    Sub get_return_object() { return Sub{std::coroutine_handle<promise_type>::from_promise(*this)}; }
    std::suspend_always initial_suspend() noexcept { return {}; }
    struct Final {
      bool await_ready() noexcept { return false; }
      std::coroutine_handle<> await_suspend(std::coroutine_handle<promise_type> h) noexcept {
        return h.promise().parent ? h.promise().parent : std::noop_coroutine();
      }
      void await_resume() noexcept {}
    };
    Final final_suspend() noexcept { return {}; }
    void return_void() {}
    void unhandled_exception() { ex = std::current_exception(); }
  };
  std::coroutine_handle<promise_type> h;
  explicit Sub(std::coroutine_handle<promise_type> hh) : h(hh) {}
  Sub(Sub&& o) noexcept : h(std::exchange(o.h, {})) {}
  ~Sub() {
    if (h) h.destroy();
  }
  bool await_ready() const noexcept { return false; }
  std::coroutine_handle<> await_suspend(std::coroutine_handle<> p) noexcept {
    h.promise().parent = p;
    return h;
  }
  void await_resume() const {
    if (h.promise().ex) std::rethrow_exception(h.promise().ex);
  }
};

struct Inst {
  int id = 0;
  std::coroutine_handle<> h;
  double a[kArgs] = {0, 0, 0, 0};
  double r[kRes] = {0, 0, 0, 0, 0, 0, 0, 0};
  // solver state (ipm.cpp DeviceSolver members)
  double mu = 0.1, tau = 0.99, delta_last = 0.0, dw = 0.0, dc = 0.0, theta_min = 0.0, theta_max = kInf;
  double obj_scale = 1.0;
  bool contradictory = false;
  std::vector<std::pair<double, double>> filter;
  ocg_ipm_result res{};
};

struct Await {
  Batch* B;
  Inst* I;
  int op;
  bool await_ready() const noexcept { return false; }
  void await_suspend(std::coroutine_handle<> h);
  void await_resume() const noexcept {}
};

class Batch {
 public:
  Batch(ocg_model* m, const ocg_ipm_options& o, int device, int nb) : model_(m), o_(o), nb_(nb) {
    auto t0 = std::chrono::steady_clock::now();
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
    for (auto& h : hs_) ck(cudaStreamCreateWithFlags(&h, cudaStreamNonBlocking), "stream");
    for (auto& e : join_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
    ocg_eval_options eo;
    ocg_eval_default_options(&eo);
    eo.device = device;
    if (ocg_eval_create(m, &eo, &ev_) != OCG_OK) throw std::runtime_error(ocg_last_error());
    auto t1 = std::chrono::steady_clock::now();
    if (ocg_kkt_create(m, ev_, &kkt_) != OCG_OK) throw std::runtime_error(ocg_last_error());
    auto t2 = std::chrono::steady_clock::now();
    // a few time segments per instance: short sequential chains per factor /
    // solve, the batch supplying the rest of the parallelism (OCG_BATCH_SEGMENTS)
    int target = 1;
    if (const char* e = std::getenv("OCG_BATCH_SEGMENTS")) target = std::max(1, std::atoi(e));
    if (ocg::hd::ldl_create(kkt_, target, &ldl_) != OCG_OK) throw std::runtime_error(ocg_last_error());
    auto t3 = std::chrono::steady_clock::now();
    plan_eval_ = std::chrono::duration<double>(t1 - t0).count();
    plan_kkt_ = std::chrono::duration<double>(t2 - t1).count();
    plan_ldl_ = std::chrono::duration<double>(t3 - t2).count();
  }
  ~Batch() {
    insts_.clear();
    if (ldl_) ocg_ldl_destroy(ldl_);
    if (kkt_) ocg_kkt_destroy(kkt_);
    if (ev_) ocg_eval_destroy(ev_);
    for (auto& h : hs_)
      if (h) cudaStreamDestroy(h);
    for (auto& e : join_)
      if (e) cudaEventDestroy(e);
    if (fork_) cudaEventDestroy(fork_);
    if (arena_) cudaFree(arena_);
    if (harena_) cudaFreeHost(harena_);
    if (s_) cudaStreamDestroy(s_);
  }

  void run(const double* lvar, const double* uvar, const double* x0, const double* lcon, const double* ucon,
           ocg_ipm_result* out, double* x_out);

  void post(Inst* I, int op, std::coroutine_handle<> h) {
    I->h = h;
    pending_[op].push_back(I);
  }

 private:
  ocg_model* model_;
  ocg_ipm_options o_;
  int nb_;
  cudaStream_t s_ = nullptr;
  ocg_eval* ev_ = nullptr;
  ocg_kkt* kkt_ = nullptr;
  ocg_ldl* ldl_ = nullptr;
  double plan_eval_ = 0, plan_kkt_ = 0, plan_ldl_ = 0;
  bool maximize_ = false;

  bd::BDims D_;
  bd::BMaps M_;
  bd::BBounds Bd_;
  // shared structure
  DBuf<int64_t> free_slot_, prim_index_, dual_row_, dual_index_, slack_index_, slack_of_, jrow_ptr_, jrow_e_;
  DBuf<int> flag_;
  // per-instance state [instance][len]
  DBuf<double> x_, xt_, grad_, gradt_, xlo_, xhi_, x0_, gcoo_, c_, ct_, lamfull_, lcon_, ucon_, rs_, lcon_s_, sv_,
      st_, lambda_, g_, gt_, gsoc_, zl_, zu_, sigma_, jtlam_, dzl_, dzu_, lb_, ub_, rhs_, rhs2_, step_, step2_, kx_,
      rv_, dx_, jac_, hess_, objv_, partials_, kval_, band_, dinv_, work_, objs_, objw_, tmpf_;
  DBuf<int8_t> hl_, hu_;
  DBuf<long long> inertia_, parts_;
  // per-kind staging
  DBuf<int> ids_[NOPS];
  DBuf<double> args_[NOPS], res_[NOPS];
  int* ids_h_[NOPS] = {};
  double* args_h_[NOPS] = {};
  double* res_h_[NOPS] = {};
  void* arena_ = nullptr;   // device memory of every per-instance array
  void* harena_ = nullptr;  // pinned staging
  std::vector<Inst*> pending_[NOPS];
  std::vector<Inst> insts_;
  std::vector<Task> tasks_;
  int64_t rounds_ = 0, launch_groups_ = 0;
  // heavy request kinds run on their own streams (fork / join on s_)
  cudaStream_t hs_[NOPS] = {};
  cudaEvent_t fork_ = nullptr, join_[NOPS] = {};
  static bool heavy(int k) {
    return k == FACTOR || k == SOLVE_0 || k == SOLVE_1 || k == APPLY_0 || k == APPLY_1;
  }
  // OCG_TIMING: device time per request kind
  bool timing_ = false;
  cudaEvent_t ev_t_[2 * NOPS] = {};
  double t_kind_[NOPS] = {}, w_kind_[NOPS] = {};
  int64_t n_kind_[NOPS] = {};

  Await op(Inst& I, int kind, double a0 = 0, double a1 = 0, double a2 = 0, double a3 = 0) {
    I.a[0] = a0;
    I.a[1] = a1;
    I.a[2] = a2;
    I.a[3] = a3;
    return Await{this, &I, kind};
  }

  void alloc_all();
  void setup(const double* lvar, const double* uvar, const double* x0, const double* lcon, const double* ucon);
  void gen(cudaKernel_t k, const char* name, std::vector<void*> ptr_args, const bd::BL& L);
  void objective(const double* x, double* f, int os, const bd::BL& L);
  void execute(int kind, int nb, cudaStream_t st);
  void drive();

  Task solve_one(Inst& I);
  Sub solve_kkt(Inst& I, double wmax, bool& ok);
  Sub resolve(Inst& I, int sel);
  Sub finish(Inst& I, int status, int iter);
  double kkt_error(const double* p, double& comp, double& stat) const;
  static void add_to_filter(Inst& I, double theta, double phi);
  static bool filter_rejects(const Inst& I, double theta, double phi);
};

void Await::await_suspend(std::coroutine_handle<> h) { B->post(I, op, h); }

// ---- allocation and setup --------------------------------------------------------

void Batch::alloc_all() {
  int64_t d[7];
  ocg_kkt_dims(kkt_, d);
  D_.nvar = ocg_model_nvar(model_);
  D_.m_con = ocg_model_mcon(model_);
  D_.n_free = d[0];
  D_.n_slack = d[1];
  D_.ntot = d[2];
  D_.m = d[3];
  D_.dim = d[4];
  D_.knnz = d[5];
  int64_t jn = 0, hn = 0, gn = 0;
  ocg_eval_sizes(ev_, &jn, &hn, &gn);
  D_.jnnz = jn;
  D_.hnnz = hn;
  D_.gnnz = gn;
  D_.objv_n = ev_->lay.objv_n;
  D_.n_chunks = ev_->n_chunks;
  D_.n_obj = static_cast<int>(ev_->obj_weight.size());

  const auto nv = static_cast<size_t>(D_.nvar), mc = static_cast<size_t>(D_.m_con);
  std::vector<int64_t> prim(nv), slack(mc), dual(mc), rslot(mc);
  ocg_kkt_maps(kkt_, prim.data(), slack.data(), dual.data(), rslot.data(), nullptr, nullptr);
  std::vector<int64_t> free_slot(static_cast<size_t>(D_.n_free)), slack_of(static_cast<size_t>(D_.n_slack)),
      dual_row(static_cast<size_t>(D_.m));
  for (size_t sl = 0; sl < nv; ++sl)
    if (prim[sl] >= 0) free_slot[static_cast<size_t>(prim[sl])] = static_cast<int64_t>(sl);
  for (size_t r = 0; r < mc; ++r) {
    if (slack[r] >= 0) slack_of[static_cast<size_t>(slack[r])] = static_cast<int64_t>(r);
    if (dual[r] >= 0) dual_row[static_cast<size_t>(dual[r])] = static_cast<int64_t>(r);
  }
  // Jacobian rows -> entries (compute_scaling's per-row max)
  std::vector<int64_t> jr(static_cast<size_t>(D_.jnnz));
  ocg_eval_structure(ev_, jr.data(), nullptr, nullptr, nullptr, nullptr);
  std::vector<int64_t> rptr(mc + 1, 0), re(jr.size());
  for (int64_t r : jr) ++rptr[static_cast<size_t>(r) + 1];
  for (size_t r = 0; r < mc; ++r) rptr[r + 1] += rptr[r];
  {
    std::vector<int64_t> fill(rptr.begin(), rptr.end() - 1);
    for (size_t q = 0; q < jr.size(); ++q) re[static_cast<size_t>(fill[static_cast<size_t>(jr[q])]++)] = static_cast<int64_t>(q);
  }
  free_slot_.upload(free_slot);
  prim_index_.upload(prim);
  dual_row_.upload(dual_row);
  dual_index_.upload(dual);
  slack_index_.upload(slack);
  slack_of_.upload(slack_of);
  jrow_ptr_.upload(rptr);
  jrow_e_.upload(re);
  M_.free_slot = free_slot_.p;
  M_.prim_index = prim_index_.p;
  M_.dual_row = dual_row_.p;
  M_.dual_index = dual_index_.p;
  M_.slack_index = slack_index_.p;
  M_.slack_of = slack_of_.p;

  // every per-instance array and staging buffer carved from one device and
  // one pinned host allocation (a batch allocates once, not ~130 times)
  const auto B = static_cast<size_t>(nb_);
  std::vector<std::pair<void**, size_t>> dev, host;
  auto A = [&](auto& buf, int64_t n) {
    using T = std::remove_reference_t<decltype(*buf.p)>;
    dev.push_back({reinterpret_cast<void**>(&buf.p), B * static_cast<size_t>(std::max<int64_t>(1, n)) * sizeof(T)});
  };
  for (auto* v : {&x_, &xt_, &grad_, &gradt_, &xlo_, &xhi_, &x0_}) A(*v, D_.nvar);
  for (auto* v : {&c_, &ct_, &lamfull_, &lcon_, &ucon_, &rs_, &lcon_s_}) A(*v, D_.m_con);
  for (auto* v : {&sv_, &st_}) A(*v, D_.n_slack);
  for (auto* v : {&lambda_, &g_, &gt_, &gsoc_}) A(*v, D_.m);
  for (auto* v : {&zl_, &zu_, &sigma_, &jtlam_, &dzl_, &dzu_, &lb_, &ub_}) A(*v, D_.ntot);
  for (auto* v : {&rhs_, &rhs2_, &step_, &step2_, &kx_, &rv_, &dx_, &dinv_}) A(*v, D_.dim);
  A(gcoo_, D_.gnnz);
  A(jac_, D_.jnnz);
  A(hess_, D_.hnnz);
  A(objv_, D_.objv_n);
  A(partials_, D_.n_chunks);
  A(kval_, D_.knnz);
  A(band_, ldl_->plan.buf_len);
  A(work_, D_.dim + static_cast<int64_t>(ldl_->plan.nseg) * ldl_->plan.wmax);
  A(objs_, 1);
  A(objw_, D_.n_obj);
  A(tmpf_, kRes);
  A(hl_, D_.ntot);
  A(hu_, D_.ntot);
  A(inertia_, 3);
  A(parts_, 3 * (ldl_->plan.nseg + 1));
  A(flag_, 1);
  for (int k = 0; k < NOPS; ++k) {
    A(ids_[k], 1);
    A(args_[k], kArgs + 4);  // column-major args + an interleaved copy of the first four
    A(res_[k], kRes);
    host.push_back({reinterpret_cast<void**>(&ids_h_[k]), B * sizeof(int)});
    host.push_back({reinterpret_cast<void**>(&args_h_[k]), B * (kArgs + 4) * sizeof(double)});
    host.push_back({reinterpret_cast<void**>(&res_h_[k]), B * kRes * sizeof(double)});
  }
  auto carve = [](std::vector<std::pair<void**, size_t>>& parts, char* base) {
    size_t off = 0;
    for (auto& [pp, bytes] : parts) {
      if (base) *pp = base + off;
      off += (bytes + 255) / 256 * 256;
    }
    return off;
  };
  const size_t dbytes = carve(dev, nullptr), hbytes = carve(host, nullptr);
  ck(cudaMalloc(&arena_, dbytes), "batch arena");
  ck(cudaMallocHost(&harena_, hbytes), "batch pinned arena");
  carve(dev, static_cast<char*>(arena_));
  carve(host, static_cast<char*>(harena_));
  for (DBuf<double>* v : {&x_, &xt_, &grad_, &gradt_, &xlo_, &xhi_, &x0_, &gcoo_, &c_, &ct_, &lamfull_, &lcon_, &ucon_,
                          &rs_, &lcon_s_, &sv_, &st_, &lambda_, &g_, &gt_, &gsoc_, &zl_, &zu_, &sigma_, &jtlam_, &dzl_,
                          &dzu_, &lb_, &ub_, &rhs_, &rhs2_, &step_, &step2_, &kx_, &rv_, &dx_, &jac_, &hess_, &objv_,
                          &partials_, &kval_, &band_, &dinv_, &work_, &objs_, &objw_, &tmpf_})
    v->owned = false;
  hl_.owned = hu_.owned = false;
  inertia_.owned = parts_.owned = false;
  flag_.owned = false;
  for (int k = 0; k < NOPS; ++k) ids_[k].owned = args_[k].owned = res_[k].owned = false;
  ck(cudaMemsetAsync(flag_.p, 0, B * sizeof(int), s_), "memset");
  Bd_.lb = lb_.p;
  Bd_.ub = ub_.p;
  Bd_.has_lb = hl_.p;
  Bd_.has_ub = hu_.p;
  Bd_.lcon_s = lcon_s_.p;
}

// one generated evaluation kernel over the launch's instances
void Batch::gen(cudaKernel_t k, const char* name, std::vector<void*> ptr_args, const bd::BL& L) {
  GenBatch gb{};
  gb.ids = L.ids;
  gb.s[0] = D_.nvar;
  gb.s[1] = D_.m_con;
  gb.s[2] = D_.m_con;
  gb.s[3] = D_.n_obj;
  gb.s[4] = D_.m_con;
  gb.s[5] = D_.jnnz;
  gb.s[6] = D_.hnnz;
  gb.s[7] = D_.objv_n;
  gb.s[8] = D_.gnnz;
  gb.s[9] = 1;
  Index ns = ev_->n_spec(name);
  std::vector<void*> args;
  args.push_back(ev_->prm_arg());
  for (void* p : ptr_args) args.push_back(p);
  args.push_back(&ev_->i0);
  args.push_back(&ev_->n_main);
  args.push_back(&ns);
  args.push_back(&gb);
  ev_->launch(k, name, args.data(), L.s, static_cast<unsigned>(L.nb));
}

// scaled objective of every launched instance into f[y * os] (flag set if not finite)
void Batch::objective(const double* x, double* f, int os, const bd::BL& L) {
  double* ov = objv_.p;
  int* fl = flag_.p;
  gen(ev_->k_objv, "ocg_objv", {&x, &ov, &fl}, L);
  bd::objective_chunks(D_, objv_.p, ev_->og_off.p, ev_->og_count.p, ev_->og_cbase.p, partials_.p, L);
  bd::objective_combine(D_, partials_.p, ev_->og_cbase.p, ev_->og_weight.p, objs_.p, f, flag_.p, os, L);
}

void Batch::setup(const double* lvar, const double* uvar, const double* x0, const double* lcon, const double* ucon) {
  const auto nv = static_cast<size_t>(D_.nvar), mc = static_cast<size_t>(D_.m_con), B = static_cast<size_t>(nb_);
  std::vector<double> mlv(nv), muv(nv), mx0(nv), mlc(mc), muc(mc);
  ocg_model_arrays(model_, mlv.data(), muv.data(), mx0.data(), nullptr, nullptr, mlc.data(), muc.data());
  std::vector<int64_t> prim(nv), slack(mc), dual(mc), rslot(mc);
  ocg_kkt_maps(kkt_, prim.data(), slack.data(), dual.data(), rslot.data(), nullptr, nullptr);
  // the slack map is the model's (eval.cpp:330-336): every instance must keep
  // each kept row's kind (equality stays equality, range stays range)
  for (size_t b = 0; b < B; ++b)
    for (size_t r = 0; r < mc; ++r) {
      if (dual[r] < 0) continue;
      const double lo = lcon ? lcon[b * mc + r] : mlc[r], hi = ucon ? ucon[b * mc + r] : muc[r];
      if ((lo == hi) != (slack[r] < 0))
        throw InvalidInstance("instance " + std::to_string(b) + " row " + std::to_string(r) +
                              (slack[r] < 0 ? " loosens an equality of the model into a range"
                                            : " turns a range row of the model into an equality"));
    }
  {
    char* js = ocg_model_structure_json(model_);
    if (js) {
      maximize_ = std::string(js).find("\"maximize\":true") != std::string::npos;
      ocg_free(js);
    }
  }
  // every instance's data on the device (the model's own, uploaded once and
  // broadcast, where the caller passes NULL), then the Reduction's folded
  // bounds (eval.cpp:290-316) per instance
  auto put = [&](DBuf<double>& d, const double* p, const std::vector<double>& def, size_t n) {
    if (p) {
      ck(cudaMemcpyAsync(d.p, p, B * n * sizeof(double), cudaMemcpyHostToDevice, s_), "H2D");
    } else {
      ck(cudaMemcpyAsync(d.p, def.data(), n * sizeof(double), cudaMemcpyHostToDevice, s_), "H2D");
      bd::broadcast_rows(d.p, static_cast<int64_t>(n), nb_, s_);
    }
  };
  put(xlo_, lvar, mlv, nv);
  put(xhi_, uvar, muv, nv);
  put(x0_, x0, mx0, nv);
  put(lcon_, lcon, mlc, mc);
  put(ucon_, ucon, muc, mc);
  std::vector<int64_t> fptr(nv + 1, 0), frow;
  for (size_t r = 0; r < mc; ++r)
    if (rslot[r] >= 0) ++fptr[static_cast<size_t>(rslot[r]) + 1];
  for (size_t sl = 0; sl < nv; ++sl) fptr[sl + 1] += fptr[sl];
  frow.resize(static_cast<size_t>(fptr[nv]));
  {
    std::vector<int64_t> fill(fptr.begin(), fptr.end() - 1);
    for (size_t r = 0; r < mc; ++r)  // rows in index order per slot, like the host loop
      if (rslot[r] >= 0) frow[static_cast<size_t>(fill[static_cast<size_t>(rslot[r])]++)] = static_cast<int64_t>(r);
  }
  DBuf<int64_t> dfptr, dfrow;
  dfptr.upload(fptr);
  dfrow.upload(frow.empty() ? std::vector<int64_t>{0} : frow);
  DBuf<int> dflags;
  dflags.alloc(2 * B);
  ck(cudaMemsetAsync(dflags.p, 0, 2 * B * sizeof(int), s_), "memset");
  std::vector<int> all(B);
  for (size_t b = 0; b < B; ++b) all[b] = static_cast<int>(b);
  ck(cudaMemcpyAsync(ids_[0].p, all.data(), B * sizeof(int), cudaMemcpyHostToDevice, s_), "ids");
  bd::fold_bounds(D_, dfptr.p, dfrow.p, prim_index_.p, xlo_.p, xhi_.p, lcon_.p, ucon_.p, dflags.p, dflags.p + B,
                  bd::BL{ids_[0].p, nb_, s_});
  std::vector<int> flags(2 * B);
  ck(cudaMemcpyAsync(flags.data(), dflags.p, 2 * B * sizeof(int), cudaMemcpyDeviceToHost, s_), "D2H");
  ck(cudaStreamSynchronize(s_), "fold sync");
  for (size_t b = 0; b < B; ++b)
    if (flags[B + b])
      throw InvalidInstance("instance " + std::to_string(b) +
                            ": its bounds change which slots are fixed (the KKT structure differs)");

  insts_.resize(B);
  for (size_t b = 0; b < B; ++b) {
    insts_[b].id = static_cast<int>(b);
    insts_[b].contradictory = flags[b] != 0;
  }
  const bd::BL L{ids_[0].p, nb_, s_};

  // EvalContext::compute_scaling at x_start (solver.cpp:318): unit-scale
  // gradient and Jacobian, then the reference's max rules
  {
    std::vector<double> ones(mc, 1.0);
    ck(cudaMemcpyAsync(rs_.p, ones.data(), mc * sizeof(double), cudaMemcpyHostToDevice, s_), "H2D");
    bd::broadcast_rows(rs_.p, static_cast<int64_t>(mc), nb_, s_);
    if (D_.n_obj > 0) {
      ck(cudaMemcpyAsync(objw_.p, ev_->obj_weight.data(), static_cast<size_t>(D_.n_obj) * sizeof(double),
                         cudaMemcpyHostToDevice, s_),
         "H2D");
      bd::broadcast_rows(objw_.p, D_.n_obj, nb_, s_);
    }
    const double* xp = x0_.p;
    const double* ow = objw_.p;
    double* gc = gcoo_.p;
    int* fl = flag_.p;
    gen(ev_->k_grad, "ocg_grad", {&xp, &ow, &gc, &fl}, L);
    bd::gather_grad(D_, gcoo_.p, ev_->gg_ptr.p, ev_->gg_idx.p, grad_.p, L);
    const double* rsp = rs_.p;
    double* cp = c_.p;
    double* jp = jac_.p;
    gen(ev_->k_cjac, "ocg_cjac", {&xp, &rsp, &cp, &jp, &fl}, L);
    bd::scaling(D_, grad_.p, jac_.p, jrow_ptr_.p, jrow_e_.p, flag_.p, ev_->og_weight.p, o_.scale, objs_.p, rs_.p,
                objw_.p, L);
    ck(cudaMemsetAsync(flag_.p, 0, B * sizeof(int), s_), "flags");
  }
  // Solver::setup_bounds / initialize_iterate (solver.cpp:125-206)
  const double relax = std::min(o_.bound_relax_factor, o_.tol);
  bd::setup_bounds(D_, M_, xlo_.p, xhi_.p, lcon_.p, ucon_.p, rs_.p, relax, lb_.p, ub_.p, hl_.p, hu_.p, lcon_s_.p, L);
  bd::init_x(D_, M_, Bd_, x0_.p, xlo_.p, xhi_.p, x_.p, L);
  {
    const double* xp = x_.p;
    const double* rsp = rs_.p;
    double* cp = c_.p;
    int* fl = flag_.p;
    gen(ev_->k_c, "ocg_c", {&xp, &rsp, &cp, &fl}, L);
  }
  bd::init_slacks_duals(D_, M_, Bd_, x_.p, c_.p, o_.mu_init, sv_.p, zl_.p, zu_.p, lambda_.p, L);
  ck(cudaMemsetAsync(flag_.p, 0, B * sizeof(int), s_), "flags");
  std::vector<double> os(B);
  ck(cudaMemcpyAsync(os.data(), objs_.p, B * sizeof(double), cudaMemcpyDeviceToHost, s_), "D2H");
  ck(cudaStreamSynchronize(s_), "setup sync");
  for (size_t b = 0; b < B; ++b) insts_[b].obj_scale = os[b];
}

// ---- one launch group: every instance that posted `kind` this round -------------

void Batch::execute(int kind, int nb, cudaStream_t st) {
  const bd::BL L{ids_[kind].p, nb, st};
  const double* a0 = args_[kind].p;
  const double* a1 = a0 + nb_;
  const double* a2 = a1 + nb_;
  const double* a3 = a2 + nb_;
  const double* ai = a3 + nb_;  // interleaved [y * 4 + k]
  double* R = res_[kind].p;
  int* fl = flag_.p;
  const double* rsp = rs_.p;
  const double* ow = objw_.p;
  auto cjg = [&](const double* xw, double* cw, double* gw) {
    double* jp = jac_.p;
    gen(ev_->k_cjac, "ocg_cjac", {&xw, &rsp, &cw, &jp, &fl}, L);
    bd::take_flags(fl, R, kRes, 0, L);
    double* gc = gcoo_.p;
    gen(ev_->k_grad, "ocg_grad", {&xw, &ow, &gc, &fl}, L);
    bd::gather_grad(D_, gcoo_.p, ev_->gg_ptr.p, ev_->gg_idx.p, gw, L);
    bd::take_flags(fl, R, kRes, 1, L);
  };
  auto solve_norms = [&](const double* rhs, double* step, bool refine_r) {
    bd::sym_matvec(D_, kval_.p, kkt_->mv_ptr.p, kkt_->mv_col.p, kkt_->mv_vidx.p, step, kx_.p, L);
    bd::residual_norms(D_, rhs, kx_.p, step, ai, refine_r ? rv_.p : nullptr, R, kRes, L);
  };
  const ocg::BandPlan& P = ldl_->plan;
  switch (kind) {
    case CJG_X:
      cjg(x_.p, c_.p, grad_.p);
      break;
    case CJG_T:
      bd::copy_dim_if(D_, step_.p, step2_.p, a0, L);
      cjg(xt_.p, ct_.p, gradt_.p);
      break;
    case RESID_X:
      bd::residual_theta(D_, M_, Bd_, c_.p, sv_.p, g_.p, R, kRes, L);
      break;
    case KKTERR:
      bd::jt_lambda(D_, jac_.p, lambda_.p, kkt_->jt_ptr.p, kkt_->jt_e.p, kkt_->jt_dual.p, kkt_->jt_slack_dual.p,
                    jtlam_.p, L);
      bd::kkt_error_parts(D_, M_, Bd_, x_.p, sv_.p, zl_.p, zu_.p, lambda_.p, grad_.p, jtlam_.p, g_.p, a0, R, kRes, L);
      break;
    case ITER: {
      bd::expand_lambda(D_, M_, lambda_.p, lamfull_.p, L);
      const double* xp = x_.p;
      const double* lp = lamfull_.p;
      double* hp = hess_.p;
      gen(ev_->k_hess, "ocg_hess", {&xp, &lp, &rsp, &ow, &hp, &fl}, L);
      bd::take_flags(fl, R, kRes, 0, L);
      bd::max_abs(hess_.p, D_.hnnz, R + 1, kRes, L);
      bd::sigma(D_, M_, Bd_, x_.p, sv_.p, zl_.p, zu_.p, sigma_.p, L);
      bd::kkt_assemble(D_, hess_.p, jac_.p, sigma_.p, kkt_->src_ptr.p, kkt_->src_code.p, kval_.p, L);
      bd::rhs(D_, M_, Bd_, x_.p, sv_.p, grad_.p, jtlam_.p, g_.p, a0, rhs_.p, L);
      break;
    }
    case FACTOR:
      ocg::dev::band_factor_batch(P, ldl_->dev, kval_.p, band_.p, dinv_.p, inertia_.p, parts_.p, L.ids, nb, a0, a1,
                                  st);
      bd::take_i64x3(inertia_.p, R, kRes, L);
      break;
    case SOLVE_0:
      ocg::dev::band_solve_batch(P, ldl_->dev, band_.p, dinv_.p, rhs_.p, step_.p, work_.p, L.ids, nb, st);
      solve_norms(rhs_.p, step_.p, false);
      break;
    case SOLVE_1:
      bd::rhs_soc(D_, rhs_.p, gsoc_.p, rhs2_.p, L);
      ocg::dev::band_solve_batch(P, ldl_->dev, band_.p, dinv_.p, rhs2_.p, step2_.p, work_.p, L.ids, nb, st);
      solve_norms(rhs2_.p, step2_.p, false);
      break;
    case NORMINF:
      bd::sym_norm_inf(D_, kval_.p, kkt_->mv_ptr.p, kkt_->mv_vidx.p, R, kRes, L);
      break;
    case REFINE_0:
      solve_norms(rhs_.p, step_.p, true);
      break;
    case REFINE_1:
      solve_norms(rhs2_.p, step2_.p, true);
      break;
    case APPLY_0:
    case APPLY_1: {
      double* stp = kind == APPLY_0 ? step_.p : step2_.p;
      ocg::dev::band_solve_batch(P, ldl_->dev, band_.p, dinv_.p, rv_.p, dx_.p, work_.p, L.ids, nb, st);
      bd::add_dim(D_, stp, dx_.p, L);
      solve_norms(kind == APPLY_0 ? rhs_.p : rhs2_.p, stp, true);
      break;
    }
    case LSPREP:
      bd::fraction_to_boundary(D_, M_, Bd_, x_.p, sv_.p, step_.p, a0, R, kRes, L);
      bd::dphi(D_, M_, Bd_, x_.p, sv_.p, grad_.p, step_.p, a1, R + 1, kRes, L);
      bd::residual_theta(D_, M_, Bd_, c_.p, sv_.p, g_.p, R + 2, kRes, L);
      objective(x_.p, R + 3, kRes, L);
      bd::take_flags(fl, R, kRes, 4, L);
      bd::barrier(D_, M_, Bd_, x_.p, sv_.p, R + 5, kRes, L);
      break;
    case TRIAL_0:
    case TRIAL_1: {
      bd::trial(D_, M_, x_.p, sv_.p, kind == TRIAL_0 ? step_.p : step2_.p, a0, xt_.p, st_.p, L);
      const double* xp = xt_.p;
      double* cp = ct_.p;
      gen(ev_->k_c, "ocg_c", {&xp, &rsp, &cp, &fl}, L);
      bd::take_flags(fl, R, kRes, 0, L);
      bd::residual_theta(D_, M_, Bd_, ct_.p, st_.p, gt_.p, R + 1, kRes, L);
      bd::barrier(D_, M_, Bd_, xt_.p, st_.p, R + 2, kRes, L);
      objective(xt_.p, R + 4, kRes, L);
      bd::take_flags(fl, R, kRes, 5, L);
      break;
    }
    case GSOC_0:
      bd::axpy_m(D_, a0, g_.p, gt_.p, gsoc_.p, L);
      break;
    case GSOC_1:
      bd::axpy_m(D_, a0, gsoc_.p, gt_.p, gsoc_.p, L);
      break;
    case FTB2:
      bd::fraction_to_boundary(D_, M_, Bd_, x_.p, sv_.p, step2_.p, a0, R, kRes, L);
      break;
    case DUALDIR:
      bd::dual_direction(D_, M_, Bd_, x_.p, sv_.p, zl_.p, zu_.p, step_.p, ai, dzl_.p, dzu_.p, R, kRes, L);
      break;
    case ACCEPT:
      bd::commit(D_, x_.p, xt_.p, sv_.p, st_.p, c_.p, ct_.p, grad_.p, gradt_.p, step_.p, step2_.p, nullptr, L);
      bd::accept(D_, M_, Bd_, step_.p, dzl_.p, dzu_.p, ai, x_.p, sv_.p, lambda_.p, zl_.p, zu_.p, L);
      bd::residual_theta(D_, M_, Bd_, c_.p, sv_.p, g_.p, R, kRes, L);
      break;
    case FINISH:
      objective(x_.p, R, kRes, L);
      bd::take_flags(fl, R, kRes, 1, L);
      bd::theta_unscaled(D_, M_, g_.p, rs_.p, R + 2, kRes, L);
      bd::jt_lambda(D_, jac_.p, lambda_.p, kkt_->jt_ptr.p, kkt_->jt_e.p, kkt_->jt_dual.p, kkt_->jt_slack_dual.p,
                    jtlam_.p, L);
      bd::kkt_error_parts(D_, M_, Bd_, x_.p, sv_.p, zl_.p, zu_.p, lambda_.p, grad_.p, jtlam_.p, g_.p, a0, R + 3,
                          kRes, L);
      break;
    default:
      throw std::runtime_error("unknown batch request");
  }
}

// rounds: every pending request kind is launched once over its instances, one
// device->host copy per kind, one synchronization per round
void Batch::drive() {
  timing_ = std::getenv("OCG_TIMING") != nullptr;
  if (timing_)
    for (auto& e : ev_t_) cudaEventCreate(&e);
  for (auto& t : tasks_) t.h.resume();
  for (;;) {
    // Light requests first: the factorizations and triangular solves (whose
    // cost is a per-instance dependency chain, nearly independent of how many
    // instances share the launch) run only once every instance has reached
    // its next one, so each runs in as few launch groups as possible; the
    // heavy kinds of one round go out on separate streams and overlap.
    int kinds[NOPS], nk = 0;
    bool light = false;
    for (int k = 0; k < NOPS; ++k)
      if (!pending_[k].empty() && !heavy(k)) light = true;
    for (int k = 0; k < NOPS; ++k)
      if (!pending_[k].empty() && heavy(k) != light) kinds[nk++] = k;
    if (nk == 0) break;
    ++rounds_;
    if (!light) ck(cudaEventRecord(fork_, s_), "fork");
    for (int q = 0; q < nk; ++q) {
      const int k = kinds[q];
      cudaStream_t st = light ? s_ : hs_[q];
      if (!light) ck(cudaStreamWaitEvent(st, fork_, 0), "fork wait");
      const auto& P = pending_[k];
      const int nb = static_cast<int>(P.size());
      int* ih = ids_h_[k];
      double* ah = args_h_[k];
      for (int y = 0; y < nb; ++y) {
        ih[y] = P[static_cast<size_t>(y)]->id;
        for (int j = 0; j < kArgs; ++j) {
          ah[static_cast<size_t>(j) * static_cast<size_t>(nb_) + static_cast<size_t>(y)] = P[static_cast<size_t>(y)]->a[j];
          ah[static_cast<size_t>(kArgs) * static_cast<size_t>(nb_) + static_cast<size_t>(y) * 4 + static_cast<size_t>(j)] =
              P[static_cast<size_t>(y)]->a[j];
        }
      }
      ck(cudaMemcpyAsync(ids_[k].p, ih, static_cast<size_t>(nb) * sizeof(int), cudaMemcpyHostToDevice, st), "ids H2D");
      ck(cudaMemcpyAsync(args_[k].p, ah, static_cast<size_t>(nb_) * (kArgs + 4) * sizeof(double),
                         cudaMemcpyHostToDevice, st),
         "args H2D");
      if (timing_) cudaEventRecord(ev_t_[2 * q], st);
      execute(k, nb, st);
      if (timing_) cudaEventRecord(ev_t_[2 * q + 1], st);
      ++launch_groups_;
      ck(cudaMemcpyAsync(res_h_[k], res_[k].p, static_cast<size_t>(nb) * kRes * sizeof(double),
                         cudaMemcpyDeviceToHost, st),
         "results D2H");
      if (!light) {
        ck(cudaEventRecord(join_[q], st), "join");
        ck(cudaStreamWaitEvent(s_, join_[q], 0), "join wait");
      }
    }
    ck(cudaStreamSynchronize(s_), "round sync");
    ck(cudaGetLastError(), "batched launch");
    if (timing_)
      for (int q = 0; q < nk; ++q) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, ev_t_[2 * q], ev_t_[2 * q + 1]);
        t_kind_[kinds[q]] += ms;
        n_kind_[kinds[q]] += 1;
        w_kind_[kinds[q]] += static_cast<double>(pending_[kinds[q]].size());
      }
    std::vector<Inst*> ready;
    for (int q = 0; q < nk; ++q) {
      const int k = kinds[q];
      auto& P = pending_[k];
      for (size_t y = 0; y < P.size(); ++y) {
        std::memcpy(P[y]->r, res_h_[k] + y * kRes, kRes * sizeof(double));
        ready.push_back(P[y]);
      }
      P.clear();
    }
    for (Inst* I : ready) I->h.resume();
  }
  if (timing_) {
    static const char* const names[NOPS] = {"CJG_X",   "CJG_T",  "RESID_X", "KKTERR",  "ITER",   "FACTOR",
                                            "SOLVE_0", "SOLVE_1", "NORMINF", "REFINE_0", "REFINE_1", "APPLY_0",
                                            "APPLY_1", "LSPREP", "TRIAL_0", "TRIAL_1", "GSOC_0", "GSOC_1",
                                            "FTB2",    "DUALDIR", "ACCEPT",  "FINISH"};
    double tot = 0.0;
    for (int k = 0; k < NOPS; ++k) tot += t_kind_[k];
    std::fprintf(stderr, "[batch] %lld rounds, %lld launch groups, device %.1f ms\n", static_cast<long long>(rounds_),
                 static_cast<long long>(launch_groups_), tot);
    for (int k = 0; k < NOPS; ++k)
      if (n_kind_[k])
        std::fprintf(stderr, "[batch] %-9s %5lld groups  %9.2f ms  %7.3f ms/group  %7.1f instances/group\n", names[k],
                     static_cast<long long>(n_kind_[k]), t_kind_[k], t_kind_[k] / n_kind_[k], w_kind_[k] / n_kind_[k]);
    for (auto& e : ev_t_) cudaEventDestroy(e);
  }
  for (auto& t : tasks_)
    if (t.h.promise().ex) std::rethrow_exception(t.h.promise().ex);
}

// ---- the per-instance control flow (ipm.cpp DeviceSolver::run) -------------------

double Batch::kkt_error(const double* p, double& comp_out, double& stat_out) const {
  const double znorm1 = p[0], lnorm1 = p[1], stat = p[2], feas = p[3], comp = p[4];
  const double denom = static_cast<double>(std::max<int64_t>(1, D_.m + D_.ntot));
  const double sd = std::max(100.0, (lnorm1 + znorm1) / denom) / 100.0;
  const double sc = std::max(100.0, znorm1 / static_cast<double>(std::max<int64_t>(1, D_.ntot))) / 100.0;
  comp_out = comp / sc;
  stat_out = stat / sd;
  return std::max({stat / sd, feas, comp / sc});
}

void Batch::add_to_filter(Inst& I, double theta, double phi) {
  const std::pair<double, double> e{(1.0 - kGammaTheta) * theta, phi - kGammaPhi * theta};
  I.filter.erase(std::remove_if(I.filter.begin(), I.filter.end(),
                                [&](const auto& f) { return f.first >= e.first && f.second >= e.second; }),
                 I.filter.end());
  I.filter.push_back(e);
}

bool Batch::filter_rejects(const Inst& I, double theta, double phi) {
  if (theta > I.theta_max) return true;
  for (const auto& f : I.filter)
    if (theta >= f.first && phi >= f.second) return true;
  return false;
}

// sparse::refine (ldl.cpp:249-272) after a solve into step (sel 0) or step2 (sel 1)
Sub Batch::resolve(Inst& I, int sel) {
  co_await op(I, sel == 0 ? SOLVE_0 : SOLVE_1, I.dw, I.dc);
  if (!(I.r[0] > o_.refine_trigger * (1.0 + I.r[1]))) co_return;
  co_await op(I, NORMINF);
  const double anorm = I.r[0] + std::abs(I.dw) + std::abs(I.dc);
  co_await op(I, sel == 0 ? REFINE_0 : REFINE_1, I.dw, I.dc);
  for (int round = 0; round < o_.refine_rounds; ++round) {
    if (I.r[0] <= 1e-12 * (anorm * I.r[2] + I.r[1])) break;
    co_await op(I, sel == 0 ? APPLY_0 : APPLY_1, I.dw, I.dc);
  }
}

// Solver::solve_kkt (solver.cpp:648-702)
Sub Batch::solve_kkt(Inst& I, double wmax, bool& ok) {
  ok = false;
  double dw = 0.0, dc = 0.0;
  bool first_bump = true;
  for (;;) {
    co_await op(I, FACTOR, dw, dc);
    ++I.res.factorizations;
    if (static_cast<int64_t>(I.r[0]) == D_.ntot && static_cast<int64_t>(I.r[1]) == D_.m && I.r[2] == 0.0) break;
    if (first_bump) {
      dw = I.delta_last > 0.0 ? std::max(1e-20, I.delta_last / o_.reg_shrink) : o_.reg_initial_scale * std::max(1.0, wmax);
      first_bump = false;
    } else if (I.r[2] > 0.0 && dc == 0.0) {
      dc = o_.reg_dual_scale * std::pow(I.mu, o_.reg_dual_power);
    } else {
      dw *= o_.reg_grow;
    }
    if (dw > o_.reg_max_delta) co_return;
  }
  if (dw > 0.0) I.delta_last = dw;
  I.dw = dw;
  I.dc = dc;
  co_await resolve(I, 0);
  ok = true;
}

Sub Batch::finish(Inst& I, int status, int iter) {
  co_await op(I, FINISH, 0.0);
  I.res.status = status;
  I.res.iterations = iter;
  const double f_raw = I.r[0] / I.obj_scale;
  I.res.objective = maximize_ ? -f_raw : f_raw;
  if (D_.m > 0) I.res.theta = I.r[2];
  double comp = 0.0, stat = 0.0;
  kkt_error(I.r + 3, comp, stat);
  I.res.stationarity = stat / I.obj_scale;
  I.res.complementarity = comp / I.obj_scale;
}

Task Batch::solve_one(Inst& I) {
  I.mu = o_.mu_init;
  I.tau = std::max(o_.tau_min, 1.0 - I.mu);
  if (I.contradictory) {
    I.res.status = 2;
    co_return;
  }
  const double mu_min = o_.tol / 10.0;
  co_await op(I, CJG_X);
  if (I.r[0] != 0.0 || I.r[1] != 0.0) {
    co_await finish(I, 3, 0);
    co_return;
  }
  co_await op(I, RESID_X);
  {
    const double th = I.r[0];
    I.theta_min = 1e-4 * std::max(1.0, th);
    I.theta_max = 1e4 * std::max(1.0, th);
  }
  int consecutive_restorations = 0;
  bool hold_mu = false;
  for (int iter = 0;; ++iter) {
    co_await op(I, KKTERR, 0.0);
    double comp = 0.0, stat = 0.0;
    const double e0 = kkt_error(I.r, comp, stat);
    if (e0 <= o_.tol) {
      co_await finish(I, 0, iter);
      co_return;
    }
    if (iter >= o_.max_iter) {
      co_await finish(I, 1, iter);
      co_return;
    }
    if (!hold_mu && I.mu > mu_min) {
      co_await op(I, KKTERR, I.mu);
      double cmu = 0.0, smu = 0.0;
      if (kkt_error(I.r, cmu, smu) <= kKappaEps * I.mu) {
        I.mu = std::max(mu_min, std::min(kKappaMu * I.mu, std::pow(I.mu, kThetaMu)));
        I.tau = std::max(o_.tau_min, 1.0 - I.mu);
        I.filter.clear();
      }
    }
    co_await op(I, ITER, I.mu);
    if (I.r[0] != 0.0) {
      co_await finish(I, 3, iter);
      co_return;
    }
    bool ok = false;
    co_await solve_kkt(I, I.r[1], ok);
    if (!ok) {
      co_await finish(I, 3, iter);
      co_return;
    }
    co_await op(I, LSPREP, I.tau, I.mu);
    const double alpha_max = I.r[0], dphi = I.r[1], theta_k = I.r[2];
    double phi_k = 0.0;
    {
      const double f_k = I.r[3];
      const bool f_ok = I.r[4] == 0.0 && std::isfinite(f_k);
      if (!f_ok || I.r[6] != 0.0) {
        co_await finish(I, 3, iter);
        co_return;
      }
      phi_k = f_k - I.mu * I.r[5];
    }

    double alpha = alpha_max;
    bool accepted = false, armijo_path = false, saw_eval_error = false;
    double theta_t = 0.0, phi_t = 0.0;
    int dir = 0;  // 0: step, 1: step2 (a second-order correction)
    bool swapped = false;
    // the outcome of the last TRIAL request (ipm.cpp eval_trial)
    auto trial_ok = [&]() {
      if (I.r[0] != 0.0) return false;
      theta_t = I.r[1];
      const double f_t = I.r[4];
      if (I.r[3] != 0.0 || !(I.r[5] == 0.0 && std::isfinite(f_t))) return false;
      phi_t = f_t - I.mu * I.r[2];
      return std::isfinite(phi_t);
    };
    auto acceptable = [&](double a) {
      if (filter_rejects(I, theta_t, phi_t)) return false;
      const bool descent = dphi < 0.0;
      const bool switching = descent && a * std::pow(-dphi, kSPhi) > kDeltaSwitch * std::pow(theta_k, kSTheta);
      if (theta_k <= I.theta_min && switching) {
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
      co_await op(I, dir == 0 ? TRIAL_0 : TRIAL_1, alpha, I.mu);
      if (!trial_ok()) {
        saw_eval_error = true;
        first_trial = false;
        alpha *= 0.5;
        continue;
      }
      accepted = acceptable(alpha);
      if (!accepted && first_trial && theta_t >= theta_k && D_.m > 0) {
        // second-order corrections (solver.cpp:496-534)
        co_await op(I, GSOC_0, alpha);
        double theta_prev = theta_t;
        for (int soc = 0; soc < 4 && !accepted; ++soc) {
          co_await resolve(I, 1);
          co_await op(I, FTB2, I.tau);
          const double alpha_soc = I.r[0];
          co_await op(I, TRIAL_1, alpha_soc, I.mu);
          if (!trial_ok()) break;
          if (acceptable(alpha_soc)) {
            accepted = true;
            swapped = true;  // the correction becomes the step (ipm.cpp swaps the buffers)
            dir = 1;
            alpha = alpha_soc;
            break;
          }
          if (theta_t >= 0.99 * theta_prev) break;
          theta_prev = theta_t;
          co_await op(I, GSOC_1, alpha_soc);
        }
        if (!accepted) {
          co_await op(I, dir == 0 ? TRIAL_0 : TRIAL_1, alpha, I.mu);
          if (!trial_ok()) {
            saw_eval_error = true;
            first_trial = false;
            alpha *= 0.5;
            continue;
          }
        }
      }
      if (accepted) {
        // the accepted point's derivatives; a correction step moves into step
        co_await op(I, CJG_T, swapped ? 1.0 : 0.0);
        if (swapped) {
          dir = 0;
          swapped = false;
        }
        if (I.r[0] != 0.0 || I.r[1] != 0.0) {
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
        co_await finish(I, saw_eval_error ? 3 : 2, iter);
        co_return;
      }
      ++consecutive_restorations;
      hold_mu = true;
      I.mu = std::min(I.mu * 10.0, 1e4);
      I.tau = std::max(o_.tau_min, 1.0 - I.mu);
      I.filter.clear();
      co_await op(I, CJG_X);
      if (I.r[0] != 0.0 || I.r[1] != 0.0) {
        co_await finish(I, 3, iter);
        co_return;
      }
      co_await op(I, RESID_X);
      continue;
    }
    consecutive_restorations = 0;
    hold_mu = false;
    if (!armijo_path) add_to_filter(I, theta_k, phi_k);

    co_await op(I, DUALDIR, I.mu, I.tau);
    double alpha_z = I.r[0];
    alpha_z = std::min(alpha_z, std::max(alpha, 1e-2));
    co_await op(I, ACCEPT, alpha, alpha_z, I.mu, kKappaSigma);
  }
}

void Batch::run(const double* lvar, const double* uvar, const double* x0, const double* lcon, const double* ucon,
                ocg_ipm_result* out, double* x_out) {
  auto t0 = std::chrono::steady_clock::now();
  alloc_all();
  setup(lvar, uvar, x0, lcon, ucon);
  auto t1 = std::chrono::steady_clock::now();
  tasks_.reserve(insts_.size());
  for (auto& I : insts_) tasks_.push_back(solve_one(I));
  drive();
  auto t2 = std::chrono::steady_clock::now();
  if (x_out)
    ck(cudaMemcpy(x_out, x_.p, static_cast<size_t>(nb_) * static_cast<size_t>(D_.nvar) * sizeof(double),
                  cudaMemcpyDeviceToHost),
       "x D2H");
  int64_t li[5];
  ocg_ldl_info(ldl_, li);
  const double setup_s = std::chrono::duration<double>(t1 - t0).count();
  const double total = std::chrono::duration<double>(t2 - t0).count();
  for (size_t b = 0; b < insts_.size(); ++b) {
    ocg_ipm_result r = insts_[b].res;
    r.time_total = total;  // the batch's wall time (every instance ran in it)
    r.time_setup = setup_s;
    r.time_plan_eval = plan_eval_;
    r.time_plan_kkt = plan_kkt_;
    r.time_plan_ldl = plan_ldl_;
    r.kkt_dim = D_.dim;
    r.kkt_nnz = D_.knnz;
    r.bandwidth = li[2];
    // rounds and launch groups of the whole batch, in the timing slots that
    // have no per-instance meaning here
    r.time_derivatives = static_cast<double>(rounds_);
    r.time_solve = static_cast<double>(launch_groups_);
    out[b] = r;
  }
}

}  // namespace

extern "C" int ocg_ipm_batch_solve(ocg_model* m, const ocg_ipm_options* opts, int device, int nb, const double* lvar,
                                   const double* uvar, const double* x_start, const double* lcon, const double* ucon,
                                   ocg_ipm_result* out, double* x_out) {
  if (!m || !out || nb <= 0) return ocg::hd::set_error(OCG_ERR_ARG, "null argument or empty batch");
  ocg_ipm_options o;
  ocg_ipm_default_options(&o);
  if (opts) o = *opts;
  try {
    ocg::mem::DeviceScope ds(device);
    const bool timing = std::getenv("OCG_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::chrono::steady_clock::time_point t1, t2;
    {
      Batch b(m, o, device, nb);
      t1 = std::chrono::steady_clock::now();
      b.run(lvar, uvar, x_start, lcon, ucon, out, x_out);
      t2 = std::chrono::steady_clock::now();
    }
    if (timing) {
      const auto t3 = std::chrono::steady_clock::now();
      auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
      std::fprintf(stderr, "[ocg_ipm_batch_solve] plans %.3f s, run %.3f s, release %.3f s\n", sec(t0, t1), sec(t1, t2),
                   sec(t2, t3));
    }
    return OCG_OK;
  } catch (const InvalidInstance& ex) {
    return ocg::hd::set_error(OCG_ERR_ARG, std::string("ocg_ipm_batch_solve: ") + ex.what());
  } catch (const std::exception& ex) {
    return ocg::hd::set_error(OCG_ERR_CUDA, std::string("ocg_ipm_batch_solve: ") + ex.what());
  }
}
