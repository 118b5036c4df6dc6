/* Test infrastructure only: CPU restatement of the reference's evaluation
 * hot path (see oc_oracle.h). Plain C11, glibc libm, compiled without FMA
 * contraction, so it performs the reference's floating-point operations in
 * the reference's order. Each function cites the reference lines it restates
 * (paths relative to /root/reference/proj/src). */
#include "oc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OP_CNST, OP_INPUT, OP_INDEX, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG, OP_SIN, OP_COS, OP_TAN, OP_EXP, OP_LOG,
       OP_SQRT, OP_POW };

typedef struct {
  double *v, *p1, *p2, *dv, *av, *ad, *grad;
  int32_t* input_node;
} ws_t;

static void ws_init(ws_t* w, const oc_group* g) {
  const size_t n = (size_t)g->n_nodes > 0 ? (size_t)g->n_nodes : 1;
  w->v = calloc(n, sizeof(double));
  w->p1 = calloc(n, sizeof(double));
  w->p2 = calloc(n, sizeof(double));
  w->dv = calloc(n, sizeof(double));
  w->av = calloc(n, sizeof(double));
  w->ad = calloc(n, sizeof(double));
  w->grad = calloc((size_t)g->n_inputs + 1, sizeof(double));
  w->input_node = malloc(((size_t)g->n_inputs + 1) * sizeof(int32_t));
  for (int32_t i = 0; i < g->n_inputs; ++i) w->input_node[i] = -1;
  for (int32_t k = 0; k < g->n_nodes; ++k)
    if (g->op[k] == OP_INPUT) w->input_node[g->a[k]] = k;
}

static void ws_free(ws_t* w) {
  free(w->v);
  free(w->p1);
  free(w->p2);
  free(w->dv);
  free(w->av);
  free(w->ad);
  free(w->grad);
  free(w->input_node);
}

static int64_t range_count(const oc_group* g) {
  return g->endpoints ? (g->lo == g->hi ? 1 : 2) : g->hi - g->lo;
}
static int64_t range_at(const oc_group* g, int64_t k) { return g->endpoints ? (k == 0 ? g->lo : g->hi) : g->lo + k; }

/* Evaluator::forward (kernel/evaluator.cpp:47-87) */
static int forward(const oc_group* g, const double* x, int64_t idx, ws_t* w, int partials) {
  int ok = 1;
  for (int32_t k = 0; k < g->n_nodes; ++k) {
    const int32_t a = g->a[k], b = g->b[k];
    double r = 0.0, q1 = 0.0, q2 = 0.0;
    const double* v = w->v;
    switch (g->op[k]) {
      case OP_CNST: r = g->c[k]; break;
      case OP_INPUT: r = x[g->base[a] + g->stride[a] * idx]; break;
      case OP_INDEX: r = (double)idx + g->c[k]; break;
      case OP_ADD: r = v[a] + v[b]; q1 = 1.0; q2 = 1.0; break;
      case OP_SUB: r = v[a] - v[b]; q1 = 1.0; q2 = -1.0; break;
      case OP_MUL: r = v[a] * v[b]; q1 = v[b]; q2 = v[a]; break;
      case OP_DIV: r = v[a] / v[b]; q1 = 1.0 / v[b]; q2 = -r / v[b]; break;
      case OP_NEG: r = -v[a]; q1 = -1.0; break;
      case OP_SIN: r = sin(v[a]); q1 = cos(v[a]); break;
      case OP_COS: r = cos(v[a]); q1 = -sin(v[a]); break;
      case OP_TAN: r = tan(v[a]); q1 = 1.0 + r * r; break;
      case OP_EXP: r = exp(v[a]); q1 = r; break;
      case OP_LOG: r = log(v[a]); q1 = 1.0 / v[a]; break;
      case OP_SQRT: r = sqrt(v[a]); q1 = 0.5 / r; break;
      case OP_POW: r = pow(v[a], g->c[k]); q1 = g->c[k] * pow(v[a], g->c[k] - 1.0); break;
    }
    w->v[k] = r;
    ok &= isfinite(r) ? 1 : 0;
    if (partials) {
      w->p1[k] = q1;
      w->p2[k] = q2;
      ok &= (g->op[k] < OP_ADD || (isfinite(q1) && isfinite(q2))) ? 1 : 0;
    }
  }
  return ok;
}

/* Evaluator::reverse_row (evaluator.cpp:96-112) */
static void reverse_row(const oc_group* g, int32_t root, double* grad, ws_t* w) {
  memset(w->av, 0, (size_t)g->n_nodes * sizeof(double));
  w->av[root] = 1.0;
  for (int32_t k = g->n_nodes; k-- > 0;) {
    const double ak = w->av[k];
    if (ak == 0.0) continue;
    if (g->op[k] == OP_INPUT) {
      grad[g->a[k]] += ak;
    } else if (g->a[k] >= 0) {
      w->av[g->a[k]] += ak * w->p1[k];
      if (g->b[k] >= 0) w->av[g->b[k]] += ak * w->p2[k];
    }
  }
}

/* Evaluator::jacobian_rows (evaluator.cpp:114-130): pattern rows in order */
static int jacobian_rows(const oc_group* g, double* jac, ws_t* w) {
  int ok = 1;
  int32_t e = 0;
  for (int32_t r = 0; r < g->out_dim; ++r) {
    const int32_t lo = e;
    while (e < g->n_jac && g->jac[2 * e] == r) ++e;
    if (lo == e) continue;
    memset(w->grad, 0, (size_t)g->n_inputs * sizeof(double));
    reverse_row(g, g->roots[r], w->grad, w);
    for (int32_t q = lo; q < e; ++q) {
      jac[q] = w->grad[g->jac[2 * q + 1]];
      ok &= isfinite(jac[q]) ? 1 : 0;
    }
  }
  return ok;
}

/* Evaluator::hess_direction (evaluator.cpp:145-212) */
static int hess_direction(const oc_group* g, int32_t j, const double* weights, ws_t* w) {
  const int32_t n = g->n_nodes;
  double *v = w->v, *p1 = w->p1, *p2 = w->p2, *dv = w->dv, *a = w->av, *ad = w->ad;
  for (int32_t k = 0; k < n; ++k) {
    switch (g->op[k]) {
      case OP_CNST:
      case OP_INDEX: dv[k] = 0.0; break;
      case OP_INPUT: dv[k] = g->a[k] == j ? 1.0 : 0.0; break;
      default: dv[k] = p1[k] * dv[g->a[k]] + (g->b[k] >= 0 ? p2[k] * dv[g->b[k]] : 0.0); break;
    }
  }
  memset(a, 0, (size_t)n * sizeof(double));
  memset(ad, 0, (size_t)n * sizeof(double));
  for (int32_t r = 0; r < g->out_dim; ++r) a[g->roots[r]] += weights[r];
  int ok = 1;
  for (int32_t k = n; k-- > 0;) {
    const double ak = a[k], adk = ad[k];
    if (ak == 0.0 && adk == 0.0) continue;
    const int32_t ia = g->a[k], ib = g->b[k];
    if (ia < 0 || g->op[k] == OP_INPUT) continue;
    double p1d = 0.0, p2d = 0.0;
    switch (g->op[k]) {
      case OP_MUL: p1d = dv[ib]; p2d = dv[ia]; break;
      case OP_DIV:
        p1d = -p1[k] * p1[k] * dv[ib];
        p2d = -(dv[k] * p1[k] + v[k] * p1d);
        break;
      case OP_SIN:
      case OP_COS: p1d = -v[k] * dv[ia]; break;
      case OP_TAN: p1d = 2.0 * v[k] * dv[k]; break;
      case OP_EXP: p1d = dv[k]; break;
      case OP_LOG: p1d = -p1[k] * p1[k] * dv[ia]; break;
      case OP_SQRT: p1d = v[k] != 0.0 ? -p1[k] * dv[k] / v[k] : 0.0; break;
      case OP_POW: {
        const double s = g->c[k] * (g->c[k] - 1.0) * pow(v[ia], g->c[k] - 2.0);
        p1d = s * dv[ia];
        ok &= (isfinite(s) || ak == 0.0) ? 1 : 0;
        break;
      }
      default: break;
    }
    a[ia] += ak * p1[k];
    ad[ia] += adk * p1[k] + ak * p1d;
    if (ib >= 0) {
      a[ib] += ak * p2[k];
      ad[ib] += adk * p2[k] + ak * p2d;
    }
  }
  return ok;
}

/* Evaluator::eval_hessian (evaluator.cpp:214-233) */
static int eval_hessian(const oc_group* g, const double* x, int64_t idx, const double* weights, double* hess,
                        ws_t* w) {
  if (g->n_hess == 0) return 1;
  if (!forward(g, x, idx, w, 1)) return 0;
  int ok = 1;
  int32_t e = 0;
  for (int32_t j = 0; j < g->n_inputs; ++j) {
    const int32_t lo = e;
    while (e < g->n_hess && g->hess[2 * e + 1] == j) ++e;
    if (lo == e) continue;
    ok &= hess_direction(g, j, weights, w);
    for (int32_t q = lo; q < e; ++q) {
      const int32_t node = w->input_node[g->hess[2 * q]];
      hess[q] = node >= 0 ? w->ad[node] : 0.0;
      ok &= isfinite(hess[q]) ? 1 : 0;
    }
  }
  return ok;
}

/* EvalContext::eval_constraints_jacobian (ipm/eval.cpp:148-173) */
int oc_constraints_jacobian(const oc_nlp* p, const double* x, const double* row_scale, double* c, double* jac) {
  int ok = 1;
  int64_t joff = 0;
  double* c_raw = calloc((size_t)p->m_con + 1, sizeof(double));
  for (int32_t gi = 0; gi < p->n_con; ++gi) {
    const oc_group* g = &p->con[gi];
    ws_t w;
    ws_init(&w, g);
    for (int64_t k = 0; k < range_count(g); ++k) {
      double* out = &c_raw[g->row_base + k * g->out_dim];
      double* jv = &jac[joff + k * g->n_jac];
      int kok = forward(g, x, range_at(g, k), &w, 1);
      if (kok) {
        for (int32_t r = 0; r < g->out_dim; ++r) out[r] = w.v[g->roots[r]];
        kok = jacobian_rows(g, jv, &w);
      }
      ok &= kok;
      for (int32_t e = 0; e < g->n_jac; ++e) jv[e] *= row_scale[g->row_base + k * g->out_dim + g->jac[2 * e]];
    }
    joff += range_count(g) * g->n_jac;
    ws_free(&w);
  }
  if (ok)
    for (int64_t r = 0; r < p->m_con; ++r) c[r] = row_scale[r] * c_raw[r];
  free(c_raw);
  return ok;
}

/* EvalContext::eval_hessian (ipm/eval.cpp:225-258) */
int oc_hessian(const oc_nlp* p, const double* x, const double* lambda, const double* row_scale, double obj_scale,
               double* hess) {
  int ok = 1;
  int64_t hoff = 0;
  for (int32_t gi = 0; gi < p->n_con; ++gi) {
    const oc_group* g = &p->con[gi];
    if (g->n_hess > 0) {
      ws_t w;
      ws_init(&w, g);
      double* weights = calloc((size_t)g->out_dim + 1, sizeof(double));
      for (int64_t k = 0; k < range_count(g); ++k) {
        const int64_t row0 = g->row_base + k * g->out_dim;
        for (int32_t r = 0; r < g->out_dim; ++r) weights[r] = lambda[row0 + r] * row_scale[row0 + r];
        ok &= eval_hessian(g, x, range_at(g, k), weights, &hess[hoff + k * g->n_hess], &w);
      }
      free(weights);
      ws_free(&w);
    }
    hoff += range_count(g) * g->n_hess;
  }
  for (int32_t gi = 0; gi < p->n_obj; ++gi) {
    const oc_group* g = &p->obj[gi];
    if (g->n_hess > 0) {
      ws_t w;
      ws_init(&w, g);
      const double wt = obj_scale * g->weight;
      for (int64_t k = 0; k < range_count(g); ++k)
        ok &= eval_hessian(g, x, range_at(g, k), &wt, &hess[hoff + k * g->n_hess], &w);
      ws_free(&w);
    }
    hoff += range_count(g) * g->n_hess;
  }
  return ok;
}

/* EvalContext::eval_objective (ipm/eval.cpp:175-200) + Backend::par_reduce
 * (backend/backend.cpp:119-133): 512-index chunks summed in index order,
 * chunk partials combined in chunk order */
int oc_objective(const oc_nlp* p, const double* x, double obj_scale, double* f) {
  double total = 0.0;
  for (int32_t gi = 0; gi < p->n_obj; ++gi) {
    const oc_group* g = &p->obj[gi];
    ws_t w;
    ws_init(&w, g);
    const int64_t cnt = range_count(g);
    double part = 0.0;
    int ok = 1;
    for (int64_t lo = 0; lo < cnt; lo += 512) {
      const int64_t hi = lo + 512 < cnt ? lo + 512 : cnt;
      double s = 0.0;
      for (int64_t k = lo; k < hi; ++k) {
        ok &= forward(g, x, range_at(g, k), &w, 0);
        s += w.v[g->roots[0]];
      }
      part += s;
    }
    ws_free(&w);
    if (!ok) return 0;
    total += g->weight * part;
  }
  *f = obj_scale * total;
  return isfinite(*f) ? 1 : 0;
}

/* EvalContext::eval_gradient (ipm/eval.cpp:202-223) */
int oc_gradient(const oc_nlp* p, const double* x, double obj_scale, double* grad_coo, double* grad_dense) {
  int ok = 1;
  int64_t goff = 0;
  for (int32_t gi = 0; gi < p->n_obj; ++gi) {
    const oc_group* g = &p->obj[gi];
    ws_t w;
    ws_init(&w, g);
    const double wt = obj_scale * g->weight;
    for (int64_t k = 0; k < range_count(g); ++k) {
      double* out = &grad_coo[goff + k * g->n_jac];
      int kok = forward(g, x, range_at(g, k), &w, 1);
      if (kok) kok = jacobian_rows(g, out, &w);
      ok &= kok;
      for (int32_t e = 0; e < g->n_jac; ++e) out[e] *= wt;
    }
    goff += range_count(g) * g->n_jac;
    ws_free(&w);
  }
  if (!ok) return 0;
  memset(grad_dense, 0, (size_t)p->nvar * sizeof(double));
  goff = 0;
  for (int32_t gi = 0; gi < p->n_obj; ++gi) {
    const oc_group* g = &p->obj[gi];
    for (int64_t k = 0; k < range_count(g); ++k)
      for (int32_t e = 0; e < g->n_jac; ++e) {
        const int32_t in = g->jac[2 * e + 1];
        grad_dense[g->base[in] + g->stride[in] * range_at(g, k)] += grad_coo[goff + k * g->n_jac + e];
      }
    goff += range_count(g) * g->n_jac;
  }
  return 1;
}
