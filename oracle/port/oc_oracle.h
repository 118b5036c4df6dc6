/* Test infrastructure only — the CPU restatement of the reference's
 * evaluation hot path that the parity tests check the GPU against (alongside
 * the reference itself, oracle/_ref/libref.so). Never linked by the product.
 *
 * Inputs are the reference's StructuredNlp in flat form (the structure dump
 * of ref_model_json / ocg_model_structure_json): per group the kernel graph
 * (kernel::Node list), the input addresses, the roots, the structural
 * pattern, the index range, row_base / weight. */
#ifndef OC_ORACLE_H_
#define OC_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_nodes;
  const int32_t* op; /* kernel::Op numbering, graph.hpp:43-59 */
  const int32_t* a;
  const int32_t* b;
  const double* c;
  int32_t n_inputs;
  const int64_t* base; /* InputAddress: slot(i) = base + stride*i */
  const int64_t* stride;
  int32_t out_dim;
  const int32_t* roots;
  int32_t n_jac;
  const int32_t* jac; /* (row, input) pairs */
  int32_t n_hess;
  const int32_t* hess; /* (i, j) pairs, i >= j, sorted by (j, i) */
  int64_t lo, hi;      /* IndexRange */
  int32_t endpoints;
  int64_t row_base;    /* constraint groups */
  double weight;       /* objective groups */
} oc_group;

typedef struct {
  int64_t nvar, m_con;
  int32_t n_con, n_obj;
  const oc_group* con;
  const oc_group* obj;
} oc_nlp;

/* EvalContext::eval_constraints_jacobian (eval.cpp:148-173): c (scaled) and
 * jac (COO, row-scaled). Returns 1 ok / 0 (non-finite value somewhere). */
int oc_constraints_jacobian(const oc_nlp* p, const double* x, const double* row_scale, double* c, double* jac);
/* EvalContext::eval_hessian (eval.cpp:225-258) */
int oc_hessian(const oc_nlp* p, const double* x, const double* lambda, const double* row_scale, double obj_scale,
               double* hess);
/* EvalContext::eval_objective (eval.cpp:175-200) with Backend::par_reduce's
 * 512-chunk partials combined in chunk order (backend.cpp:119-133) */
int oc_objective(const oc_nlp* p, const double* x, double obj_scale, double* f);
/* EvalContext::eval_gradient (eval.cpp:202-223): COO and dense */
int oc_gradient(const oc_nlp* p, const double* x, double obj_scale, double* grad_coo, double* grad_dense);

#ifdef __cplusplus
}
#endif

#endif
