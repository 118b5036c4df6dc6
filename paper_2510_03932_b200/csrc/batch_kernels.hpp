// Batched interior-point kernels: the vector work of ipm_kernels.cu, the
// KKT gathers of kernels.cu and the objective / gradient reductions, for many
// independent instances of ONE transcribed structure in one launch each
// (SURVEY.md §8e "replicas ... batched in one launch over instance x node",
// §8f item 4). Grid row y works on instance ids[y]; per-instance arrays are
// [instance][length] with the lengths in BDims. Reductions run one block per
// instance and write their values to out[y * os + q] in launch order, so one
// device->host copy returns every instance's scalars.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ocg::bdev {

struct BDims {
  int64_t nvar = 0, m_con = 0, n_free = 0, n_slack = 0, ntot = 0, m = 0, dim = 0;
  int64_t jnnz = 0, hnnz = 0, gnnz = 0, knnz = 0, objv_n = 0, n_chunks = 0;
  int n_obj = 0;
};

// structure shared by every instance (device)
struct BMaps {
  const int64_t* free_slot = nullptr;    // [n_free] reduced primal -> slot
  const int64_t* prim_index = nullptr;   // [nvar] slot -> reduced primal or -1
  const int64_t* dual_row = nullptr;     // [m] dual ordinal -> row
  const int64_t* dual_index = nullptr;   // [m_con] row -> dual ordinal or -1
  const int64_t* slack_index = nullptr;  // [m_con] row -> slack ordinal or -1
  const int64_t* slack_of = nullptr;     // [n_slack] slack ordinal -> row
};

// per-instance bounds (device, [instance][len])
struct BBounds {
  const double* lb = nullptr;  // [ntot]
  const double* ub = nullptr;
  const int8_t* has_lb = nullptr;
  const int8_t* has_ub = nullptr;
  const double* lcon_s = nullptr;  // [m_con]
};

struct BL {  // launch: instance list on the device, its length, stream
  const int* ids;
  int nb;
  cudaStream_t s;
};

// ---- evaluation reductions ----
// per-instance chunk partials of objv [inst][objv_n] -> partials [inst][n_chunks]
void objective_chunks(const BDims& D, const double* objv, const int64_t* goff, const int64_t* gcount,
                      const int64_t* cbase, double* partials, const BL& L);
// f[y] = obj_scale[inst] * sum_g w_g * sum_chunks; flag[inst] = 1 if not finite
void objective_combine(const BDims& D, const double* partials, const int64_t* cbase, const double* weights,
                       const double* obj_scale, double* f, int* flag, int os, const BL& L);
// dense gradient [inst][nvar] from grad COO [inst][gnnz]
void gather_grad(const BDims& D, const double* gcoo, const int64_t* ptr, const int32_t* idx, double* out,
                 const BL& L);
// out[y] = max |v[inst][0..n)|
void max_abs(const double* v, int64_t n, double* out, int os, const BL& L);
// out[y * stride + slot] = flag[inst]; flag[inst] = 0
void take_flags(int* flag, double* out, int stride, int slot, const BL& L);
// unit-scale evaluation at x0 -> obj_scale[inst], row_scale [inst][m_con],
// objw [inst][n_obj] (EvalContext::compute_scaling, eval.cpp:260-280)
void scaling(const BDims& D, const double* grad_dense, const double* jac, const int64_t* jrow_ptr,
             const int64_t* jrow_e, const int* flag, const double* weights, int enabled, double* obj_scale,
             double* row_scale, double* objw, const BL& L);

// dst <- src on dim-vectors where flag[y] != 0
void copy_dim_if(const BDims& D, double* dst, const double* src, const double* flag, const BL& L);
// out[y * os + k] = src[inst * 3 + k] (inertia triples)
void take_i64x3(const long long* src, double* out, int os, const BL& L);

// ---- KKT ----
void kkt_assemble(const BDims& D, const double* hess, const double* jac, const double* sigma, const int64_t* ptr,
                  const int64_t* code, double* val, const BL& L);
void sym_matvec(const BDims& D, const double* val, const int64_t* rptr, const int64_t* col, const int64_t* vidx,
                const double* x, double* y, const BL& L);
void sym_norm_inf(const BDims& D, const double* val, const int64_t* rptr, const int64_t* vidx, double* out,
                  int os, const BL& L);
void jt_lambda(const BDims& D, const double* jac, const double* lam, const int64_t* ptr, const int64_t* e_idx,
               const int64_t* dual_idx, const int64_t* slack_dual, double* out, const BL& L);

// ---- setup (Solver::setup_bounds / initialize_iterate, solver.cpp:125-206) ----
// rows 1..nb-1 of a [nb][n] array <- row 0 (instances sharing the model's data)
void broadcast_rows(double* a, int64_t n, int nb, cudaStream_t s);
// Reduction's folded bounds (eval.cpp:290-316) in place on xlo / xhi (holding
// lvar / uvar): slot sl takes the rows frow[fptr[sl]..fptr[sl+1]); contra[inst]
// = 1 if some slot ends with lo > hi, bad[inst] = 1 if the fixed slots differ
// from the structure's (prim_index < 0 <=> lo == hi)
void fold_bounds(const BDims& D, const int64_t* fptr, const int64_t* frow, const int64_t* prim_index, double* xlo,
                 double* xhi, const double* lcon, const double* ucon, int* contra, int* bad, const BL& L);
void setup_bounds(const BDims& D, const BMaps& M, const double* xlo, const double* xhi, const double* lcon,
                  const double* ucon, const double* row_scale, double relax, double* lb, double* ub, int8_t* has_lb,
                  int8_t* has_ub, double* lcon_s, const BL& L);
void init_x(const BDims& D, const BMaps& M, const BBounds& B, const double* x0, const double* xlo, const double* xhi,
            double* x, const BL& L);
void init_slacks_duals(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* c, double mu,
                       double* s, double* zl, double* zu, double* lambda, const BL& L);

// ---- iteration vector work (per-instance scalars a[y] in launch order) ----
// g = c - (s or lcon_s) on the kept rows; out[y] = sum |g|
void residual_theta(const BDims& D, const BMaps& M, const BBounds& B, const double* c, const double* s, double* g,
                    double* out, int os, const BL& L);
void sigma(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* zl,
           const double* zu, double* out, const BL& L);
void rhs(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* grad,
         const double* jtlam, const double* g, const double* mu, double* out, const BL& L);
void trial(const BDims& D, const BMaps& M, const double* x, const double* s, const double* dir, const double* a,
           double* xt, double* st, const BL& L);
void expand_lambda(const BDims& D, const BMaps& M, const double* lambda, double* full, const BL& L);
// out = a[y] * x + y_ on m-vectors
void axpy_m(const BDims& D, const double* a, const double* x, const double* yv, double* out, const BL& L);
void rhs_soc(const BDims& D, const double* rhs, const double* gsoc, double* out, const BL& L);
void add_dim(const BDims& D, double* x, const double* dx, const BL& L);
// x <- xt, s <- st, c <- ct, grad <- gradt; step <- step2 when swap (may be NULL) [y] != 0
void commit(const BDims& D, double* x, const double* xt, double* s, const double* st, double* c, const double* ct,
            double* grad, const double* gradt, double* step, const double* step2, const double* swap, const BL& L);
// scal[y*4 + 0..3] = alpha, alpha_z, mu, kappa
void accept(const BDims& D, const BMaps& M, const BBounds& B, const double* step, const double* dzl,
            const double* dzu, const double* scal, const double* xn, const double* sn, double* lambda, double* zl,
            double* zu, const BL& L);

// reductions, out[y * os + q]
void barrier(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, double* out,
             int os, const BL& L);  // NV 2: sum log, count d <= 0
void kkt_error_parts(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                     const double* zl, const double* zu, const double* lambda, const double* grad,
                     const double* jtlam, const double* g, const double* mu, double* out, int os, const BL& L);  // NV 5
void fraction_to_boundary(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                          const double* dir, const double* tau, double* out, int os, const BL& L);  // NV 1
void dphi(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s, const double* grad,
          const double* dir, const double* mu, double* out, int os, const BL& L);  // NV 1
// scal[y*4 + 0..1] = mu, tau
void dual_direction(const BDims& D, const BMaps& M, const BBounds& B, const double* x, const double* s,
                    const double* zl, const double* zu, const double* step, const double* scal, double* dzl,
                    double* dzu, double* out, int os, const BL& L);  // NV 1
// r = b - Kx - delta x (r may be NULL); dwdc[y*4 + 0..1]; out NV 3: max|r|, max|b|, max|x|
void residual_norms(const BDims& D, const double* b, const double* kx, const double* x, const double* dwdc,
                    double* r, double* out, int os, const BL& L);
// out[y] = max_d |g_d| / row_scale[dual_row[d]] (the unscaled constraint violation)
void theta_unscaled(const BDims& D, const BMaps& M, const double* g, const double* row_scale, double* out,
                    int os, const BL& L);

}  // namespace ocg::bdev
