// Test infrastructure only — the checker, never the product.
//
// extern "C" harness over the UNMODIFIED reference sources under
// /root/reference/proj/src (compiled by oracle/Makefile into oracle/_ref/).
// It exposes exactly the reference objects on the hot path so that tests and
// bench.py's reference arm can drive them through ctypes:
//   dsl::parse_ocp + transcribe::transcribe   (proj/src/dsl/parser.cpp:733,
//                                               proj/src/transcribe/transcribe.cpp:180)
//   ipm::detail::EvalContext                   (proj/src/ipm/eval.cpp:40-286)
//   ipm::detail::Reduction / KktAssembler      (proj/src/ipm/eval.cpp:290-440)
//   sparse::matvec_sym                          (proj/src/sparse/sparse.cpp:51-61)
//   ipm::solve                                  (proj/src/ipm/solver.cpp:789)
// plus the acceptance-suite input recipe (proj/tests/acceptance/acceptance_main.cpp:179-193)
// so that inputs are drawn with the same libstdc++ mt19937/uniform_real_distribution.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <json.hpp>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "ipm/ipm_internal.hpp"
#include "octrans/dsl/parser.hpp"
#include "octrans/ipm/solver.hpp"
#include "octrans/sparse/sparse.hpp"
#include "octrans/transcribe/transcribe.hpp"

using namespace octrans;
using kernel::Index;

namespace {

struct RefModel {
  dsl::OcpProblem prob;
  transcribe::StructuredNlp nlp;
};

struct RefEval {
  RefModel* model;
  std::unique_ptr<backend::Backend> be;
  std::unique_ptr<ipm::detail::EvalContext> ec;
  std::vector<double> c;
};

struct RefKkt {
  RefEval* ev;
  std::unique_ptr<ipm::detail::Reduction> red;
  std::unique_ptr<ipm::detail::KktAssembler> kkt;
};

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), static_cast<size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
}

nlohmann::json kernel_json(const kernel::Evaluator& ev) {
  nlohmann::json j;
  const auto& g = ev.kernel().graph;
  nlohmann::json nodes = nlohmann::json::array();
  for (const auto& nd : g.nodes()) nodes.push_back({static_cast<int>(nd.op), nd.a, nd.b, nd.c});
  j["nodes"] = nodes;
  j["roots"] = ev.kernel().roots;
  nlohmann::json inputs = nlohmann::json::array();
  for (size_t i = 0; i < g.inputs().size(); ++i)
    inputs.push_back({g.inputs()[i].base, g.inputs()[i].stride, g.input_labels()[i]});
  j["inputs"] = inputs;
  nlohmann::json jac = nlohmann::json::array(), hess = nlohmann::json::array();
  for (auto [r, c] : ev.pattern().jac) jac.push_back({r, c});
  for (auto [a, b] : ev.pattern().hess) hess.push_back({a, b});
  j["jac"] = jac;
  j["hess"] = hess;
  return j;
}

nlohmann::json range_json(const transcribe::IndexRange& r) { return {r.lo, r.hi, r.endpoints}; }

char* dup_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

}  // namespace

// Defined only when the harness is linked into integration/_out/libref_accel.so
// (the drop-in build): releases the device state of finished solves.
extern "C" void octrans_accel_release_all() __attribute__((weak));

extern "C" {

void ref_free(void* p) { std::free(p); }

void* ref_model_create(const char* src, int scheme, int64_t N, int boxes_as_bounds, char* err, int errlen) {
  try {
    auto m = std::make_unique<RefModel>();
    m->prob = dsl::parse_ocp(src);
    transcribe::TranscribeOptions opts;
    opts.boxes_as_bounds = boxes_as_bounds != 0;
    m->nlp = transcribe::transcribe(m->prob, scheme == 0 ? transcribe::Scheme::euler : transcribe::Scheme::trapezoid,
                                    N, opts);
    return m.release();
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// the StructuredNlp itself (for the drop-in build's descriptor checks)
const void* ref_model_nlp_ptr(void* h) { return &static_cast<RefModel*>(h)->nlp; }

int64_t ref_model_nvar(void* h) { return static_cast<RefModel*>(h)->nlp.nvar(); }
int64_t ref_model_mcon(void* h) { return static_cast<RefModel*>(h)->nlp.m_con; }

void ref_model_arrays(void* h, double* lvar, double* uvar, double* x_start, double* clip_lo, double* clip_hi,
                      double* lcon, double* ucon) {
  const auto& n = static_cast<RefModel*>(h)->nlp;
  auto cp = [](double* dst, const std::vector<double>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  };
  cp(lvar, n.lvar);
  cp(uvar, n.uvar);
  cp(x_start, n.x_start);
  cp(clip_lo, n.clip_lo);
  cp(clip_hi, n.clip_hi);
  cp(lcon, n.lcon);
  cp(ucon, n.ucon);
}

// Structure description (graphs, patterns, ranges, layout) as JSON.
char* ref_model_json(void* h) {
  const auto& n = static_cast<RefModel*>(h)->nlp;
  nlohmann::json j;
  j["N"] = n.N;
  j["nvar"] = n.nvar();
  j["m_con"] = n.m_con;
  j["maximize"] = n.maximize;
  j["scheme"] = transcribe::scheme_name(n.scheme);
  nlohmann::json slabs = nlohmann::json::array();
  for (const auto& s : n.layout.slabs) slabs.push_back({static_cast<int>(s.kind), s.dim, s.base, s.nodes});
  j["layout"] = slabs;
  nlohmann::json cons = nlohmann::json::array();
  for (const auto& g : n.con_groups) {
    nlohmann::json c = kernel_json(g.eval);
    c["kind"] = static_cast<int>(g.kind);
    c["label"] = g.label;
    c["range"] = range_json(g.range);
    c["out_dim"] = g.out_dim;
    c["row_base"] = g.row_base;
    c["lower"] = g.lower;
    c["upper"] = g.upper;
    cons.push_back(c);
  }
  j["con_groups"] = cons;
  nlohmann::json objs = nlohmann::json::array();
  for (const auto& g : n.obj_groups) {
    nlohmann::json o = kernel_json(g.eval);
    o["label"] = g.label;
    o["range"] = range_json(g.range);
    o["weight"] = g.weight;
    objs.push_back(o);
  }
  j["obj_groups"] = objs;
  return dup_string(j.dump());
}

// ---- EvalContext ----------------------------------------------------------

void* ref_eval_create(void* model, int parallel, int workers) {
  auto* m = static_cast<RefModel*>(model);
  auto e = std::make_unique<RefEval>();
  e->model = m;
  e->be = std::make_unique<backend::Backend>(parallel ? backend::Backend::Kind::parallel
                                                      : backend::Backend::Kind::serial,
                                             workers);
  e->ec = std::make_unique<ipm::detail::EvalContext>(m->nlp, *e->be);
  return e.release();
}

void ref_eval_destroy(void* h) { delete static_cast<RefEval*>(h); }

int ref_eval_workers(void* h) { return static_cast<RefEval*>(h)->be->workers(); }

void ref_eval_sizes(void* h, int64_t* out) {
  auto& ec = *static_cast<RefEval*>(h)->ec;
  out[0] = static_cast<int64_t>(ec.jac_row.size());
  out[1] = static_cast<int64_t>(ec.hess_row.size());
  out[2] = static_cast<int64_t>(ec.grad_col.size());
}

void ref_eval_structure(void* h, int64_t* jr, int64_t* jc, int64_t* hr, int64_t* hc, int64_t* gc) {
  auto& ec = *static_cast<RefEval*>(h)->ec;
  auto cp = [](int64_t* dst, const std::vector<Index>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(Index));
  };
  cp(jr, ec.jac_row);
  cp(jc, ec.jac_col);
  cp(hr, ec.hess_row);
  cp(hc, ec.hess_col);
  cp(gc, ec.grad_col);
}

void ref_eval_set_scaling(void* h, double obj_scale, const double* row_scale) {
  auto& ec = *static_cast<RefEval*>(h)->ec;
  ec.obj_scale = obj_scale;
  for (size_t r = 0; r < ec.row_scale.size(); ++r) ec.row_scale[r] = row_scale ? row_scale[r] : 1.0;
}

void ref_eval_compute_scaling(void* h, const double* x0, int enabled) {
  auto* e = static_cast<RefEval*>(h);
  e->ec->compute_scaling(std::span<const double>(x0, static_cast<size_t>(e->model->nlp.nvar())), enabled != 0);
}

void ref_eval_get_scaling(void* h, double* obj_scale, double* row_scale) {
  auto& ec = *static_cast<RefEval*>(h)->ec;
  *obj_scale = ec.obj_scale;
  if (row_scale) std::memcpy(row_scale, ec.row_scale.data(), ec.row_scale.size() * sizeof(double));
}

int ref_eval_c(void* h, const double* x, double* c) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  bool ok = e->ec->eval_constraints(xs, e->c);
  if (ok && c) std::memcpy(c, e->c.data(), e->c.size() * sizeof(double));
  return ok ? 1 : 0;
}

int ref_eval_cjac(void* h, const double* x, double* c, double* jac) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  bool ok = e->ec->eval_constraints_jacobian(xs, e->c);
  if (ok && c) std::memcpy(c, e->c.data(), e->c.size() * sizeof(double));
  if (ok && jac) std::memcpy(jac, e->ec->jac_val.data(), e->ec->jac_val.size() * sizeof(double));
  return ok ? 1 : 0;
}

int ref_eval_obj(void* h, const double* x, double* f) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  return e->ec->eval_objective(xs, *f) ? 1 : 0;
}

int ref_eval_grad(void* h, const double* x, double* grad_dense, double* grad_coo) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  std::vector<double> g;
  bool ok = e->ec->eval_gradient(xs, g);
  if (ok && grad_dense) std::memcpy(grad_dense, g.data(), g.size() * sizeof(double));
  if (ok && grad_coo) std::memcpy(grad_coo, e->ec->grad_val.data(), e->ec->grad_val.size() * sizeof(double));
  return ok ? 1 : 0;
}

int ref_eval_hess(void* h, const double* x, const double* lambda, double* hess) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  std::span<const double> ls(lambda, static_cast<size_t>(e->model->nlp.m_con));
  bool ok = e->ec->eval_hessian(xs, ls);
  if (ok && hess) std::memcpy(hess, e->ec->hess_val.data(), e->ec->hess_val.size() * sizeof(double));
  return ok ? 1 : 0;
}

double ref_eval_max_abs_hessian(void* h) { return static_cast<RefEval*>(h)->ec->max_abs_hessian(); }

// One J+H "step" (eval_constraints_jacobian + eval_hessian) timed with
// steady_clock; returns seconds. Used by bench.py's reference arm.
double ref_eval_step_seconds(void* h, const double* x, const double* lambda, int reps, int* ok_out) {
  auto* e = static_cast<RefEval*>(h);
  std::span<const double> xs(x, static_cast<size_t>(e->model->nlp.nvar()));
  std::span<const double> ls(lambda, static_cast<size_t>(e->model->nlp.m_con));
  bool ok = true;
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    ok &= e->ec->eval_constraints_jacobian(xs, e->c);
    ok &= e->ec->eval_hessian(xs, ls);
  }
  auto t1 = std::chrono::steady_clock::now();
  if (ok_out) *ok_out = ok ? 1 : 0;
  return std::chrono::duration<double>(t1 - t0).count();
}

// ---- Reduction / KktAssembler ------------------------------------------------

void* ref_kkt_create(void* eval) {
  auto* e = static_cast<RefEval*>(eval);
  auto k = std::make_unique<RefKkt>();
  k->ev = e;
  k->red = std::make_unique<ipm::detail::Reduction>(e->model->nlp);
  k->kkt = std::make_unique<ipm::detail::KktAssembler>(e->model->nlp, *e->ec, *k->red);
  return k.release();
}

void ref_kkt_destroy(void* h) { delete static_cast<RefKkt*>(h); }

void ref_kkt_dims(void* h, int64_t* out) {
  auto& k = *static_cast<RefKkt*>(h)->kkt;
  out[0] = k.n_free;
  out[1] = k.n_slack;
  out[2] = k.ntot;
  out[3] = k.m;
  out[4] = k.dim;
  out[5] = k.K.nnz();
  out[6] = static_cast<RefKkt*>(h)->red->contradictory ? 1 : 0;
}

void ref_kkt_pattern(void* h, int64_t* colp, int64_t* rowi) {
  auto& K = static_cast<RefKkt*>(h)->kkt->K;
  std::memcpy(colp, K.colp.data(), K.colp.size() * sizeof(Index));
  std::memcpy(rowi, K.rowi.data(), K.rowi.size() * sizeof(Index));
}

// Per-slot / per-row maps: prim_index[nvar], xlo/xhi[nvar] (effective bounds),
// slack_index/dual_index/row_slot[m_con].
void ref_kkt_maps(void* h, int64_t* prim_index, int64_t* slack_index, int64_t* dual_index, int64_t* row_slot,
                  double* xlo, double* xhi) {
  auto* r = static_cast<RefKkt*>(h);
  auto cpi = [](int64_t* dst, const std::vector<Index>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(Index));
  };
  auto cpd = [](double* dst, const std::vector<double>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  };
  cpi(prim_index, r->kkt->prim_index);
  cpi(slack_index, r->kkt->slack_index);
  cpi(dual_index, r->red->dual_index);
  cpi(row_slot, r->red->row_slot);
  cpd(xlo, r->red->xlo);
  cpd(xhi, r->red->xhi);
}

// assemble() from the EvalContext's current jac_val/hess_val buffers.
void ref_kkt_assemble(void* h, const double* sigma, double* val_out) {
  auto* r = static_cast<RefKkt*>(h);
  r->kkt->assemble(*r->ev->ec, std::span<const double>(sigma, static_cast<size_t>(r->kkt->ntot)));
  std::memcpy(val_out, r->kkt->K.val.data(), r->kkt->K.val.size() * sizeof(double));
}

// y = K x with the mirror, for given K values on the assembled pattern.
void ref_kkt_matvec(void* h, const double* val, const double* x, double* y) {
  auto* r = static_cast<RefKkt*>(h);
  sparse::SparseSym A = r->kkt->K;
  std::memcpy(A.val.data(), val, A.val.size() * sizeof(double));
  const auto n = static_cast<size_t>(A.n);
  sparse::matvec_sym(A, std::span<const double>(x, n), std::span<double>(y, n));
}


// KktAssembler::symbolic() (proj/src/ipm/eval.cpp:442-471): the AMD order with
// the pivot_after_ deferral, then sparse::analyze_ordered (ldl.cpp:78-133).
// sizes: out[0] = dim, out[1] = nnz(L).
void ref_kkt_symbolic_sizes(void* h, int64_t* out) {
  const auto& S = static_cast<RefKkt*>(h)->kkt->symbolic();
  out[0] = S.n;
  out[1] = S.lnz;
}
void ref_kkt_symbolic(void* h, int64_t* perm, int64_t* parent, int64_t* Lp) {
  const auto& S = static_cast<RefKkt*>(h)->kkt->symbolic();
  std::memcpy(perm, S.perm.data(), S.perm.size() * sizeof(Index));
  std::memcpy(parent, S.parent.data(), S.parent.size() * sizeof(Index));
  std::memcpy(Lp, S.Lp.data(), S.Lp.size() * sizeof(Index));
}

// sparse::factorize (ldl.cpp:139-213) of the given K values with the
// reference's split (ntot) and shifts; D, Li, Lx, Dinv out (permuted order),
// inertia[3] = (pos, neg, zero).
void ref_kkt_factorize(void* h, const double* val, double dw, double dc, double* D, int64_t* Li, double* Lx,
                       int64_t* inertia) {
  auto* r = static_cast<RefKkt*>(h);
  const auto& S = r->kkt->symbolic();
  sparse::SparseSym A = r->kkt->K;
  std::memcpy(A.val.data(), val, A.val.size() * sizeof(double));
  sparse::LdlFactor F;
  sparse::factorize(A, S, dw, dc, r->kkt->ntot, F);
  if (D) std::memcpy(D, F.D.data(), F.D.size() * sizeof(double));
  if (Li) std::memcpy(Li, F.Li.data(), F.Li.size() * sizeof(Index));
  if (Lx) std::memcpy(Lx, F.Lx.data(), F.Lx.size() * sizeof(double));
  inertia[0] = F.inertia.positive;
  inertia[1] = F.inertia.negative;
  inertia[2] = F.inertia.zero;
}

// sparse::solve (ldl.cpp:222-247) against a fresh factorization; returns 0 if
// the factorization had zero pivots (the reference throws there).
int ref_kkt_factor_solve(void* h, const double* val, double dw, double dc, const double* b, double* x) {
  auto* r = static_cast<RefKkt*>(h);
  const auto& S = r->kkt->symbolic();
  sparse::SparseSym A = r->kkt->K;
  std::memcpy(A.val.data(), val, A.val.size() * sizeof(double));
  sparse::LdlFactor F;
  sparse::factorize(A, S, dw, dc, r->kkt->ntot, F);
  if (F.inertia.zero > 0) return 0;
  auto y = sparse::solve(F, std::span<const double>(b, static_cast<size_t>(S.n)));
  std::memcpy(x, y.data(), y.size() * sizeof(double));
  return 1;
}

// ---- full solve ---------------------------------------------------------------

// out: [objective, iterations, time_total, time_derivatives, time_factorize,
//       time_solve, factorizations, kkt_nnz, factor_nnz, theta]; returns status.
int ref_solve(void* model, int parallel, int workers, int max_iter, double tol, double* out) {
  auto* m = static_cast<RefModel*>(model);
  backend::Backend be(parallel ? backend::Backend::Kind::parallel : backend::Backend::Kind::serial, workers);
  ipm::IpmOptions opts;
  if (max_iter > 0) opts.max_iter = max_iter;
  if (tol > 0) opts.tol = tol;
  opts.verbose = std::getenv("REF_VERBOSE") != nullptr;  // per-iteration trace (solver.cpp:623-628)
  if (const char* d = std::getenv("REF_DUMP_KKT")) opts.dump_kkt = d;  // first assembled KKT, Matrix Market
  auto sol = ipm::solve(m->nlp, opts, be);
  if (octrans_accel_release_all) octrans_accel_release_all();
  out[0] = sol.objective;
  out[1] = sol.iterations;
  out[2] = sol.stats.time_total;
  out[3] = sol.stats.time_derivatives;
  out[4] = sol.stats.time_factorize;
  out[5] = sol.stats.time_solve;
  out[6] = sol.stats.factorizations;
  out[7] = static_cast<double>(sol.stats.kkt_nnz);
  out[8] = static_cast<double>(sol.stats.factor_nnz);
  out[9] = sol.theta;
  return static_cast<int>(sol.status);
}

// ---- synthetic inputs (libstdc++ RNG, reference recipes) -------------------------

// Acceptance recipe (proj/tests/acceptance/acceptance_main.cpp:179-193): x per
// slot uniform inside the clip box shrunk 5% (half-open/infinite boxes use
// [lo+0.05, 1.2] / [0.4, 1.2]); then lambda ~ U(-1, 1) per row, same generator.
void ref_synth_acceptance(void* model, uint32_t seed, double* x, double* lambda) {
  auto& nlp = static_cast<RefModel*>(model)->nlp;
  std::mt19937 rng(seed);
  for (Index i = 0; i < nlp.nvar(); ++i) {
    double lo = nlp.clip_lo[static_cast<size_t>(i)], hi = nlp.clip_hi[static_cast<size_t>(i)];
    if (!std::isfinite(lo) || !std::isfinite(hi)) {
      lo = std::isfinite(lo) ? lo + 0.05 : 0.4;
      hi = std::isfinite(hi) ? hi - 0.05 : 1.2;
      if (lo >= hi) {
        lo = 0.4;
        hi = 1.2;
      }
    } else {
      double w = hi - lo;
      lo += 0.05 * w;
      hi -= 0.05 * w;
    }
    std::uniform_real_distribution<double> dist(lo, hi);
    x[i] = dist(rng);
  }
  std::uniform_real_distribution<double> ldist(-1.0, 1.0);
  if (lambda)
    for (Index r = 0; r < nlp.m_con; ++r) lambda[r] = ldist(rng);
}

// Quadrotor eval recipe (proj/tests/unit/ipm_test.cpp:398-403): U(lo, hi) per slot.
void ref_synth_uniform(uint32_t seed, double lo, double hi, int64_t n, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
