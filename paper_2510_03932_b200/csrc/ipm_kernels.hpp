// Interior-point vector kernels on device-resident iterates (SURVEY.md §8a
// row a18; reference proj/src/ipm/solver.cpp). See ipm_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ocg::ipmdev {

// Index maps and bounds of the reduced primal vector v = (x_free, s) and of
// the kept rows (Solver::setup_bounds, solver.cpp:125-170). Device pointers.
struct Iter {
  int64_t nvar = 0, m_con = 0, n_free = 0, n_slack = 0, ntot = 0, m = 0;
  const int64_t* free_slot = nullptr;    // [n_free] reduced primal -> slot
  const int64_t* dual_row = nullptr;     // [m] dual ordinal -> row
  const int64_t* slack_index = nullptr;  // [m_con] row -> slack ordinal or -1
  const double* lb = nullptr;            // [ntot]
  const double* ub = nullptr;
  const int8_t* has_lb = nullptr;
  const int8_t* has_ub = nullptr;
  const double* lcon_s = nullptr;        // [m_con] scaled lower row bounds
};

template <int NV>
struct Ops {
  int op[NV];       // 0 sum, 1 max, 2 min
  double init[NV];
};

// device scratch for two-level reductions
struct Scratch {
  double* partials = nullptr;  // >= 2*148 blocks x 5 values
  double* out = nullptr;       // >= 5
};

void residual(const Iter& P, const double* c, const double* s, double* g, cudaStream_t st);
void sigma(const Iter& P, const double* x, const double* s, const double* zl, const double* zu, double* out,
           cudaStream_t st);
void rhs(const Iter& P, const double* x, const double* s, const double* grad, const double* jtlam, const double* g,
         double mu, double* out, cudaStream_t st);
void trial(const Iter& P, const double* x, const double* s, const double* dir, double a, double* xt, double* stv,
           cudaStream_t st);
// the same with the step length at a_dev (device), for graph capture
void trial_dev(const Iter& P, const double* x, const double* s, const double* dir, const double* a_dev, double* xt,
               double* stv, cudaStream_t st);
void expand_lambda(const Iter& P, const double* lambda, double* full, cudaStream_t st);
void axpy(double a, const double* x, const double* y, double* out, int64_t n, cudaStream_t st);
void rhs_soc(const Iter& P, const double* rhs, const double* gsoc, double* out, cudaStream_t st);
void accept(const Iter& P, const double* step, const double* dzl, const double* dzu, double alpha, double alpha_z,
            double mu, double kappa, const double* xn, const double* sn, double* lambda, double* zl, double* zu,
            cudaStream_t st);
void add(double* x, const double* dx, int64_t n, cudaStream_t st);

// reductions: synchronous, result on the host
double l1(const double* g, int64_t n, Scratch& sc, cudaStream_t st);
bool barrier(const Iter& P, const double* x, const double* s, double& bar, Scratch& sc, cudaStream_t st);
// the same values left on the device: out_dev = sum |g|; out2_dev = (barrier, invalid count)
void l1_async(const double* g, int64_t n, Scratch& sc, double* out_dev, cudaStream_t st);
void barrier_async(const Iter& P, const double* x, const double* s, Scratch& sc, double* out2_dev, cudaStream_t st);
// out5 = sum|z|, sum|lambda|, max|stationarity|, max|g|, max|complementarity - mu|
void kkt_error_parts(const Iter& P, const double* x, const double* s, const double* zl, const double* zu,
                     const double* lambda, const double* grad, const double* jtlam, const double* g, double mu,
                     double* out5, Scratch& sc, cudaStream_t st);
double fraction_to_boundary(const Iter& P, const double* x, const double* s, const double* dir, double tau,
                            Scratch& sc, cudaStream_t st);
double dphi(const Iter& P, const double* x, const double* s, const double* grad, const double* dir, double mu,
            Scratch& sc, cudaStream_t st);
double dual_direction(const Iter& P, const double* x, const double* s, const double* zl, const double* zu,
                      const double* step, double mu, double tau, double* dzl, double* dzu, Scratch& sc,
                      cudaStream_t st);
// r = b - kx - delta x (r may be NULL); out3 = max|r|, max|b|, max|x|
void residual_norms(const double* b, const double* kx, const double* x, int64_t dim, int64_t ntot, double dw,
                    double dc, double* r, double* out3, Scratch& sc, cudaStream_t st);

int launches_per_reduction();

}  // namespace ocg::ipmdev
