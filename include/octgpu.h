/* octgpu — B200-native evaluation of direct-transcription OCP NLPs.
 *
 * C ABI of the drop-in for the reference's evaluation layer:
 *   octrans::ipm::detail::EvalContext     /root/reference/proj/src/ipm/ipm_internal.hpp:40-95
 *   octrans::ipm::detail::Reduction       /root/reference/proj/src/ipm/ipm_internal.hpp:102-111
 *   octrans::ipm::detail::KktAssembler    /root/reference/proj/src/ipm/ipm_internal.hpp:119-146
 * fed by a StructuredNlp built from the same model text
 *   octrans::dsl::parse_ocp + octrans::transcribe::transcribe
 *                                         /root/reference/proj/include/octrans/dsl/parser.hpp:33
 *                                         /root/reference/proj/include/octrans/transcribe/transcribe.hpp:56-59
 *
 * Conventions: integer status returns (OCG_OK = 0,
 * OCG_EVAL_DOMAIN = 1 when an evaluation met a non-finite value or a domain
 * error — the reference's `false` — and negative codes for API/CUDA errors);
 * no C++ exceptions cross the ABI; library-owned device buffers; an explicit
 * CUDA stream argument (cudaStream_t passed as void*; NULL = legacy default
 * stream). Evaluation calls are asynchronous: they enqueue kernels and set a
 * device-side failure flag; ocg_eval_status() synchronises the stream and
 * reports (and clears) the flag, which is how the blocking bool semantics of
 * the reference are recovered. Index arrays are int64 like the reference's
 * `Index`. There is no CPU fallback: without a usable sm_100 device every
 * call that needs one returns OCG_ERR_CUDA.
 */
#ifndef OCTGPU_H_
#define OCTGPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCG_OK 0
#define OCG_EVAL_DOMAIN 1
#define OCG_ERR_ARG (-1)
#define OCG_ERR_CUDA (-2)
#define OCG_ERR_PARSE (-3)
#define OCG_ERR_JIT (-4)
#define OCG_ERR_STATE (-5)

typedef struct ocg_model ocg_model; /* StructuredNlp */
typedef struct ocg_eval ocg_eval;   /* EvalContext on one device */
typedef struct ocg_kkt ocg_kkt;     /* Reduction + KktAssembler */
typedef void* ocg_stream;           /* cudaStream_t */

/* Thread-local message for the last failed call. */
const char* ocg_last_error(void);
void ocg_free(void* p);
const char* ocg_version(void);
/* Library-internal device memory: large plan blocks are kept in a bounded
 * cache (OCG_CACHE_MAX_MB, default 8192 MiB per device) and a private
 * stream-ordered pool per device; this returns both to the driver for
 * `device` (< 0: every device), after dropping ocg_ipm_solve's cached plans.
 * Call with no work of the library in flight. */
int ocg_release_cached_memory(int device);

/* ---- model: parse + transcribe (reference transcribe.hpp:56-59) ---------- */
/* scheme: 0 = euler, 1 = trapezoid (transcribe::Scheme) */
int ocg_model_create(const char* source, int scheme, int64_t N, int boxes_as_bounds, ocg_model** out);
void ocg_model_destroy(ocg_model* m);
int64_t ocg_model_nvar(const ocg_model* m);
int64_t ocg_model_mcon(const ocg_model* m);
int64_t ocg_model_grid(const ocg_model* m);
/* Host copies of StructuredNlp's lvar/uvar/x_start/clip_lo/clip_hi (nvar)
 * and lcon/ucon (m_con); any pointer may be NULL. */
int ocg_model_arrays(const ocg_model* m, double* lvar, double* uvar, double* x_start, double* clip_lo,
                     double* clip_hi, double* lcon, double* ucon);
/* A StructuredNlp built by another front end (the reference's own
 * dsl::parse_ocp + transcribe::transcribe), handed over as flat arrays — the
 * drop-in path of INTEGRATION.md. Field meanings follow
 * /root/reference/proj/include/octrans/transcribe/nlp.hpp:36-117 and
 * kernel/graph.hpp:35-133; node ops use the kernel::Op numbering. The
 * structural pattern is re-derived and checked against jac/hess when given. */
typedef struct {
  int32_t kind;            /* ConstraintGroup::Kind: 0 dynamics, 1 path, 2 boundary (objective: ignored) */
  int32_t n_nodes;
  const int32_t* node_op;  /* kernel::Op */
  const int32_t* node_a;
  const int32_t* node_b;
  const double* node_c;
  int32_t n_inputs;
  const int64_t* input_base;   /* InputAddress */
  const int64_t* input_stride;
  int32_t out_dim;
  const int32_t* roots;
  int64_t range_lo, range_hi;  /* IndexRange */
  int32_t range_endpoints;
  int64_t row_base;        /* constraint groups */
  const double* lower;     /* [out_dim] constraint groups */
  const double* upper;
  double weight;           /* objective groups */
  int32_t n_jac, n_hess;   /* Pattern (pairs, optional: NULL/0 = derive only) */
  const int32_t* jac;
  const int32_t* hess;
  const char* label;              /* optional */
  const char* const* input_labels; /* [n_inputs], optional */
} ocg_group_desc;

typedef struct {
  int32_t scheme;          /* 0 euler, 1 trapezoid */
  int64_t N;
  int32_t n_slabs;         /* VariableLayout::slabs */
  const int32_t* slab_kind;  /* dsl::VarKind: 0 state, 1 control, 2 variable */
  const int32_t* slab_dim;
  const int64_t* slab_base;
  const int64_t* slab_nodes;
  int64_t nvar, m_con;
  const double* lvar;      /* [nvar] */
  const double* uvar;
  const double* x_start;
  const double* clip_lo;   /* [nvar], may be NULL */
  const double* clip_hi;
  const double* lcon;      /* [m_con] */
  const double* ucon;
  int32_t maximize;
  int32_t n_con_groups;
  const ocg_group_desc* con_groups;
  int32_t n_obj_groups;
  const ocg_group_desc* obj_groups;
} ocg_nlp_desc;

int ocg_model_create_from_nlp(const ocg_nlp_desc* d, ocg_model** out);

/* Graphs, patterns, ranges, layout as JSON (caller frees with ocg_free). */
char* ocg_model_structure_json(const ocg_model* m);
/* Synthetic inputs with libstdc++'s mt19937 (reference recipes):
 * acceptance_main.cpp:179-193 (x in the shrunk clip box, then lambda~U(-1,1))
 * and ipm_test.cpp:398-403 (U(lo,hi) per slot). Host arrays. */
int ocg_model_synth_acceptance(const ocg_model* m, uint32_t seed, double* x, double* lambda);
int ocg_synth_uniform(uint32_t seed, double lo, double hi, int64_t n, double* out);

/* ---- EvalContext (eval.cpp:40-286) ---------------------------------------- */
typedef struct {
  int device;       /* CUDA ordinal */
  int fma;          /* 0: no FMA contraction (bit-compatible with the x86 reference); 1: allow */
  int block;        /* threads per block, a multiple of 32; each warp owns 32-index tiles (0 = 128) */
  int64_t idx_lo;   /* shard: first main grid index (0 with idx_hi = -1: whole grid) */
  int64_t idx_hi;   /* shard: one past the last main grid index, -1 = all */
  int specials;     /* evaluate the endpoint-pair instances on this shard (1 = yes) */
  int min_blocks;   /* resident blocks per SM the kernels are register-budgeted for
                       (__launch_bounds__); 0 = auto: the largest budget <= 6 that the
                       shared memory allows and that compiles without spills */
  int split_kinds;  /* shared-memory staging of the outputs: 0 = one region reused group
                       after group, 1 = one region per output kind in turn, 2 = a region
                       per group (one wait per tile); -1 = auto */
  int input_staging; /* how a tile's inputs (node slabs, row_scale and lambda rows) reach
                       shared memory: 0 = per-lane LDGSTS, waited for before the tile computes;
                       1 = per-lane LDGSTS double-buffered (the next tile's copies in flight
                       while this one computes); 2 = TMA bulk copies on mbarriers,
                       double-buffered, one-warp blocks (forces block = 32); -1 = auto (1
                       when the second buffer costs no resident blocks, else 0) */
} ocg_eval_options;

void ocg_eval_default_options(ocg_eval_options* o);
int ocg_eval_create(const ocg_model* m, const ocg_eval_options* opts, ocg_eval** out);
void ocg_eval_destroy(ocg_eval* e);

/* jac_row/jac_col, hess_row/hess_col (row >= col), grad_col sizes */
int ocg_eval_sizes(const ocg_eval* e, int64_t* jac_nnz, int64_t* hess_nnz, int64_t* grad_nnz);
/* host copies of the global COO structure, bit-identical to EvalContext's */
int ocg_eval_structure(const ocg_eval* e, int64_t* jac_row, int64_t* jac_col, int64_t* hess_row,
                       int64_t* hess_col, int64_t* grad_col);

#define OCG_BUF_JAC 0       /* jac_val  [jac_nnz]   */
#define OCG_BUF_HESS 1      /* hess_val [hess_nnz]  */
#define OCG_BUF_GRAD 2      /* grad_val [grad_nnz]  */
#define OCG_BUF_ROWSCALE 3  /* row_scale [m_con]    */
#define OCG_BUF_OBJV 4      /* per-instance objective values */
/* library-owned device buffers */
double* ocg_eval_buffer(ocg_eval* e, int which);
/* Replace one of those buffers by caller-owned device memory of the same
 * length (e.g. a framework tensor); the caller keeps it alive. */
int ocg_eval_bind_buffer(ocg_eval* e, int which, double* dev_ptr);

/* obj_scale and row_scale (host array of m_con, NULL = ones) */
int ocg_eval_set_scaling(ocg_eval* e, double obj_scale, const double* row_scale);
int ocg_eval_get_scaling(ocg_eval* e, double* obj_scale, double* row_scale);
/* EvalContext::compute_scaling (eval.cpp:266-286) at device x0; synchronous */
int ocg_eval_compute_scaling(ocg_eval* e, const double* x0, int enabled, ocg_stream s);

/* Device pointers in, device pointers out; asynchronous. */
int ocg_eval_constraints(ocg_eval* e, const double* x, double* c, ocg_stream s);
int ocg_eval_constraints_jacobian(ocg_eval* e, const double* x, double* c, ocg_stream s);
int ocg_eval_objective(ocg_eval* e, const double* x, double* f, ocg_stream s); /* f: device scalar */
int ocg_eval_gradient(ocg_eval* e, const double* x, double* grad_dense, ocg_stream s);
int ocg_eval_hessian(ocg_eval* e, const double* x, const double* lambda, ocg_stream s);
/* fused eval_constraints_jacobian + eval_hessian at one x (one forward pass) */
int ocg_eval_jac_hess(ocg_eval* e, const double* x, const double* lambda, double* c, ocg_stream s);
int ocg_eval_max_abs_hessian(ocg_eval* e, double* out, ocg_stream s); /* out: device scalar */
/* The fused J+H evaluation from host buffers to host buffers, pipelined over
 * `chunks` node ranges of the main grid (boundaries on the 32-node tile grid,
 * the endpoint instances with the last): x goes up whole, then per chunk its
 * multiplier rows go up and its kernel runs on `s` while the previous chunk's
 * c / jac_val / hess_val segments come back on a second stream, so the two
 * copy directions overlap (host buffers page-locked for that). Reference
 * counterpart: EvalContext::eval_constraints_jacobian + eval_hessian at one x
 * with host vectors (proj/src/ipm/eval.cpp:148-173, 225-258). Stream-ordered:
 * the host outputs are complete when `s` is; *bytes (may be NULL) = bytes
 * copied in both directions. Not for sharded contexts. Measured on the B200
 * box: host<->device traffic in both directions together saturates at about
 * 55 GB/s, so overlapping the directions gains nothing there and each extra
 * chunk adds per-copy overhead (profiles/r2_host_pipeline_sweep.jsonl):
 * chunks = 1 (no pipelining) is the fastest setting on that host. */
int ocg_eval_jac_hess_host(ocg_eval* e, const double* x_host, const double* lambda_host, double* c_host,
                           double* jac_host, double* hess_host, int chunks, int64_t* bytes, ocg_stream s);
/* Node-range shards: the objective's 512-instance chunk
 * partials (Backend::par_reduce, backend.cpp:119-133) of this context's
 * instances — device array of ocg_eval_objective_chunks() doubles, chunks of
 * other shards left as whatever the kernel computes from the stale values —
 * and the fixed-order combine of a partials array gathered over all shards
 * (each chunk taken from its owner) into the scaled objective. With shard
 * boundaries on chunk boundaries the result equals ocg_eval_objective's
 * bit for bit. */
int64_t ocg_eval_objective_chunks(const ocg_eval* e);
int ocg_eval_objective_partials(ocg_eval* e, const double* x, double* partials, ocg_stream s);
int ocg_eval_objective_combine(ocg_eval* e, const double* partials, double* f, ocg_stream s);
/* Synchronise s; OCG_OK if every evaluation since the last call was finite,
 * else OCG_EVAL_DOMAIN. Clears the flag. */
int ocg_eval_status(ocg_eval* e, ocg_stream s);
/* Asynchronous form: enqueue on s the copy of the finiteness flag into
 * *host_flag (page-locked host memory) and its reset; once s has been
 * synchronized, *host_flag != 0 means some evaluation since the last status
 * call was not finite (ocg_eval_status's OCG_EVAL_DOMAIN). */
int ocg_eval_status_async(ocg_eval* e, int* host_flag, ocg_stream s);
/* number of kernels this context has launched (all entry points) */
int64_t ocg_eval_launch_count(const ocg_eval* e);

/* Diagnostics: the CUDA source generated for a model (ocg_free it; a final
 * "// ocg-meta {...}" line gives gridDim.y, tail threads and shared memory per
 * kernel and the parameter-block values), and an NVRTC compile of it for
 * sm_100a without loading (works without a GPU).
 */
char* ocg_debug_generated_source(const ocg_model* m, int fma, int block);
/* the same for an input_staging mode (0, 1, 2 as in ocg_eval_options) */
char* ocg_debug_generated_source_ex(const ocg_model* m, int fma, int block, int input_staging);
int ocg_debug_compile(const ocg_model* m, int fma, int block);
/* NVRTC/ptxas log (registers, spills per kernel) of the module an eval
 * context with these options would load; NULL on failure (ocg_free it). */
char* ocg_debug_compile_log(const ocg_model* m, const ocg_eval_options* opts);

/* ---- node-range shards over several GPUs -------------------
 * A communicator between the ranks of one evaluation: NCCL (the library
 * loads libnccl.so.2 at run time; rank 0 makes the unique id and the caller
 * broadcasts it), or host callbacks (e.g. torch.distributed over gloo), whose
 * buffers are host memory. Callbacks return 0 on success; a zero count means
 * "nothing to send / receive" and must not communicate. */
typedef struct ocg_comm ocg_comm;
typedef struct {
  void* ctx;
  /* in place over all ranks: element-wise sum of n doubles / max of n int32 */
  int (*allreduce_sum_f64)(void* ctx, double* buf, int64_t n);
  int (*allreduce_max_i32)(void* ctx, int32_t* buf, int64_t n);
  /* send n_send doubles to rank `to` and receive n_recv doubles from rank `from` */
  int (*sendrecv_f64)(void* ctx, const double* send, int64_t n_send, int to, double* recv, int64_t n_recv, int from);
} ocg_comm_host_fns;
int ocg_comm_nccl_unique_id(unsigned char id[128]);
int ocg_comm_create_nccl(const unsigned char id[128], int rank, int world, int device, ocg_comm** out);
int ocg_comm_create_host(const ocg_comm_host_fns* fns, int rank, int world, int device, ocg_comm** out);
void ocg_comm_destroy(ocg_comm* c);
/* The shard of `comm`'s rank: main grid indices [lo, hi) with boundaries on
 * multiples of 512 (no objective chunk straddles two ranks), the endpoint
 * instances on rank 0. opts->idx_lo / idx_hi / specials are ignored. The
 * context keeps `comm` (which must outlive it). */
int ocg_eval_create_sharded(const ocg_model* m, const ocg_eval_options* opts, ocg_comm* comm, ocg_eval** out);
/* out[6] = idx_lo, idx_hi, specials, rank, world, halo doubles per exchange */
int ocg_eval_shard(const ocg_eval* e, int64_t* out);
/* x_dev (device, nvar): the slots this rank owns copied from x_host (host,
 * nvar), then the halo nodes from their owners (ocg_eval_halo_exchange).
 * Returns the host->device bytes in *h2d_bytes (may be NULL). */
int ocg_eval_scatter_x(ocg_eval* e, const double* x_host, double* x_dev, int64_t* h2d_bytes, ocg_stream s);
/* the nodes this rank reads but does not own, from their owners, into x_dev */
int ocg_eval_halo_exchange(ocg_eval* e, double* x_dev, ocg_stream s);
/* lambda_dev (device, m_con): the rows this rank's instances read, from lambda_host */
int ocg_eval_scatter_rows(ocg_eval* e, const double* lambda_host, double* lambda_dev, int64_t* h2d_bytes,
                          ocg_stream s);
/* ocg_eval_status over all ranks (the ok flags max-reduced): OCG_OK or OCG_EVAL_DOMAIN on every rank */
int ocg_eval_status_all(ocg_eval* e, ocg_stream s);
/* the scaled objective over all ranks into *f (host): each rank's chunk
 * partials, the chunks it does not own zeroed, summed over the ranks (one
 * nonzero term per chunk) and combined in the reference's order; equal bit
 * for bit to ocg_eval_objective on one device. OCG_EVAL_DOMAIN if any rank
 * saw a non-finite value. */
int ocg_eval_objective_all(ocg_eval* e, const double* x_dev, double* f, ocg_stream s);

/* Host only: rank's shard plan as JSON (ocg_free it): {"lo", "hi", "specials",
 * "x_own": [[off, len]...], "send_to"/"recv_from": [[[off, len]...] per peer],
 * "rows": [[off, len]...], "chunk_owned": [0/1...], "halo_doubles"}. */
char* ocg_shard_plan_json(const ocg_model* m, int rank, int world);

/* ---- Reduction + KktAssembler (eval.cpp:290-440) -------------------------- */
int ocg_kkt_create(const ocg_model* m, ocg_eval* e, ocg_kkt** out);
void ocg_kkt_destroy(ocg_kkt* k);
/* out[7] = n_free, n_slack, ntot, m, dim, nnz, contradictory */
int ocg_kkt_dims(const ocg_kkt* k, int64_t* out);
/* lower-CSC pattern of K (colp[dim+1], rowi[nnz]), bit-identical to KktAssembler::K */
int ocg_kkt_pattern(const ocg_kkt* k, int64_t* colp, int64_t* rowi);
/* prim_index/xlo/xhi [nvar]; slack_index/dual_index/row_slot [m_con] */
int ocg_kkt_maps(const ocg_kkt* k, int64_t* prim_index, int64_t* slack_index, int64_t* dual_index,
                 int64_t* row_slot, double* xlo, double* xhi);
double* ocg_kkt_values(ocg_kkt* k); /* device K.val [nnz] */
/* K.val from the eval context's current jac/hess buffers + sigma[ntot] (device) */
int ocg_kkt_assemble(ocg_kkt* k, const double* sigma, ocg_stream s);
/* y = K x with the symmetric mirror (sparse::matvec_sym, sparse.cpp:51-61) */
int ocg_kkt_matvec(ocg_kkt* k, const double* x, double* y, ocg_stream s);
/* *out (device scalar) = max row sum of |K| with the mirror (sparse::norm_inf_sym, sparse.cpp) */
int ocg_kkt_norm_inf(ocg_kkt* k, double* out, ocg_stream s);
/* out[ntot] = J^T lambda over kept rows, minus lambda on slacks
 * (Solver::compute_jt_lambda, solver.cpp:244-257); lambda indexed by dual ordinal */
int ocg_kkt_jt_lambda(ocg_kkt* k, const double* lambda, double* out, ocg_stream s);

/* ---- KKT factorization on the device ---------------------------------------
 * Stand-in for sparse::factorize / solve (proj/src/sparse/ldl.cpp:139-247) and
 * for the paper's cuDSS (absent from this image): LDL^T with 1x1 pivots of
 * P (K + diag(delta_w I_ntot, -delta_c I_m)) P^T in a node-major band-plus-
 * border ordering, the reference's zero-pivot rule, inertia (pos, neg, zero). */
typedef struct ocg_ldl ocg_ldl;
int ocg_ldl_create(ocg_kkt* k, ocg_ldl** out);
void ocg_ldl_destroy(ocg_ldl* l);
/* out[5] = dim, time segments, bandwidth, global border rows, factorizations so far */
int ocg_ldl_info(const ocg_ldl* l, int64_t* out);
/* factor the current K.val of `k`; inertia[3] (host, may be NULL) — synchronous when given */
int ocg_ldl_factor(ocg_ldl* l, double delta_w, double delta_c, int64_t* inertia, ocg_stream s);
/* x = (K + deltas)^{-1} rhs with the last factorization (device vectors) */
int ocg_ldl_solve(ocg_ldl* l, const double* rhs, double* x, ocg_stream s);

/* Elimination orders of ocg_ldl_create_ex:
 * OCG_LDL_BAND       the node-major band above (ocg_ldl_create; fast, parallel
 *                    in time; its 1x1 pivots are not the reference's);
 * OCG_LDL_REFERENCE  the reference's order: KktAssembler::symbolic's AMD
 *                    ordering with the pivot_after_ deferral (eval.cpp:442-471,
 *                    ldl.cpp:54-137), the same 1x1 pivots and zero-pivot rule
 *                    as sparse::factorize (ldl.cpp:139-213), so inertia
 *                    corrections follow the reference's. The sequential part
 *                    (the elimination tree's chain) runs on one warp. */
#define OCG_LDL_BAND 0
#define OCG_LDL_REFERENCE 1
int ocg_ldl_create_ex(ocg_kkt* k, int order, ocg_ldl** out);
/* Speculative inertia correction (reference order): factor n candidate
 * regularizations (delta_w[i], delta_c[i]) concurrently — independent numeric
 * buffers, one stream each, the same arithmetic as n calls of
 * ocg_ldl_factor — and return their inertias in inertia[3 i .. 3 i + 2].
 * Candidate 0's factors are then current; ocg_ldl_select(l, i) makes
 * candidate i's current for ocg_ldl_solve / ocg_ldl_factors. The band order
 * takes n = 1 only (its factorization already fills the device). */
int ocg_ldl_factor_many(ocg_ldl* l, int n, const double* delta_w, const double* delta_c, int64_t* inertia,
                        ocg_stream s);
int ocg_ldl_select(ocg_ldl* l, int i);
int ocg_ldl_order(const ocg_ldl* l);
/* OCG_LDL_REFERENCE: nnz of L (sparse::SymbolicLdl::lnz); 0 for the band */
int64_t ocg_ldl_factor_nnz(const ocg_ldl* l);
/* OCG_LDL_REFERENCE: host copies of the last factorization in the reference's
 * layout (LdlFactor: perm[dim], Lp[dim+1], Li[lnz], D[dim] by pivot position,
 * Lx[lnz]); any pointer may be NULL. Synchronizes the device. */
int ocg_ldl_factors(const ocg_ldl* l, int64_t* perm, int64_t* Lp, int64_t* Li, double* D, double* Lx);
/* Host only (no device needed): the reference-order symbolic analysis of a
 * lower-CSC KKT pattern colp[dim+1]/rowi (indices [0, n_free) free primal,
 * [n_free, ntot) slacks, [ntot, dim) duals) -- KktAssembler::symbolic +
 * sparse::analyze_ordered: perm[dim] (position -> index), etree parent[dim],
 * Lp[dim+1], Li[*lnz] (pass Li = NULL to get *lnz first). Any output may be
 * NULL. */
int ocg_ldl_ref_symbolic(int64_t dim, const int64_t* colp, const int64_t* rowi, int64_t n_free, int64_t ntot,
                         int64_t* perm, int64_t* parent, int64_t* Lp, int64_t* Li, int64_t* lnz);

/* ---- device-resident interior-point solve -----------------------------------
 * ipm::solve (proj/src/ipm/solver.cpp:304-702, options solver.hpp:31-56): the
 * reference's filter line-search IPM with every vector on the device —
 * evaluations, KKT assembly, the vector kernels and the factorization
 * (ocg_ldl_*). */
typedef struct {
  double tol;
  int max_iter;
  double mu_init, tau_min;
  double reg_initial_scale, reg_grow, reg_shrink, reg_dual_scale, reg_dual_power, reg_max_delta;
  int scale;
  double bound_relax_factor;
  int refine_rounds;
  double refine_trigger;
  int verbose;
  int kkt_order; /* OCG_LDL_BAND (default) or OCG_LDL_REFERENCE (ocg_ldl_create_ex) */
} ocg_ipm_options;

typedef struct {
  int status; /* 0 optimal, 1 max_iter, 2 infeasible_detected, 3 eval_error (SolveStatus) */
  int iterations;
  double objective; /* sign-corrected like Solution::objective */
  double theta, stationarity, complementarity;
  int factorizations;
  double time_total, time_derivatives, time_factorize, time_solve;
  int64_t kkt_dim, kkt_nnz, bandwidth;
  /* one-time host/device setup, not in time_total: eval plan (incl. NVRTC),
   * KKT pattern, factorization plan; then bounds/start point (in time_total) */
  double time_plan_eval, time_plan_kkt, time_plan_ldl, time_setup;
} ocg_ipm_result;

void ocg_ipm_default_options(ocg_ipm_options* o);

/* A reusable solver context: the evaluation plan, KKT pattern and
 * factorization plan are built once per model structure; each solve then
 * takes an instance's bounds and start point (NULL = the model's), e.g. the
 * members of a batch that differ only in boundary values (BASELINE config 5).
 * The instance must fix the same slots (equal folded bounds) as the model,
 * and keep every kept row's kind: a row that is an equality (lcon == ucon) in
 * the model must stay one, a range row must stay a range (the slack map is
 * the model's); otherwise the solve returns OCG_ERR_ARG. */
typedef struct ocg_ipm_ctx ocg_ipm_ctx;
int ocg_ipm_ctx_create(ocg_model* m, int device, ocg_ipm_ctx** out);
void ocg_ipm_ctx_destroy(ocg_ipm_ctx* c);
int ocg_ipm_ctx_solve(ocg_ipm_ctx* c, const ocg_ipm_options* opts, const double* lvar, const double* uvar,
                      const double* x_start, const double* lcon, const double* ucon, ocg_ipm_result* out,
                      double* x_out);
/* x_out[nvar] (host, may be NULL): final iterate. The plans (evaluation,
 * KKT pattern, factorization) are kept per (model, device) and reused by the
 * next ocg_ipm_solve of the same model, as an ocg_ipm_ctx would; they go with
 * ocg_model_destroy or ocg_release_cached_memory (OCG_IPM_PLAN_CACHE=0: off). */
int ocg_ipm_solve(ocg_model* m, const ocg_ipm_options* opts, int device, ocg_ipm_result* out, double* x_out);

/* nb independent instances of the model's structure solved together
 * (BASELINE config 5): each instance follows exactly the
 * decisions of ocg_ipm_solve / the reference Solver, while every device step
 * is ONE launch over all instances that reached it (instance x node grids).
 * Instance arrays are host [nb][nvar] (lvar, uvar, x_start) and [nb][m_con]
 * (lcon, ucon), NULL = the model's own for every instance; each instance must
 * fix the same slots as the model. out[nb]; x_out[nb][nvar] may be NULL.
 * time_total / time_setup / time_plan_* are the batch's; time_derivatives and
 * time_solve carry the batch's launch rounds and launch groups. nb <= 65535. */
int ocg_ipm_batch_solve(ocg_model* m, const ocg_ipm_options* opts, int device, int nb, const double* lvar,
                        const double* uvar, const double* x_start, const double* lcon, const double* ucon,
                        ocg_ipm_result* out, double* x_out);

#ifdef __cplusplus
}
#endif

#endif /* OCTGPU_H_ */
