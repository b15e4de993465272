/* bipm_gpu.h -- C-ABI of the B200 reduced-space KKT engine.
 *
 * Drop-in boundary for the reduced KKT path of the reference solver
 * (/root/reference/proj/core).  Every entry point takes plain pointers and
 * sizes; host arrays use the reference layout: a per-scenario array is
 * scenario-major, i.e. the reference's column-major Matrix(len, M)
 * (types.hpp:56-78), and shared patterns are int32 CSR.  No C++ exception
 * crosses this boundary: functions return a BIPM_* status and the message of
 * the last failure is available from bipm_last_error().  The status codes map
 * one-to-one onto the reference exception types, so a host shim can rethrow
 * them.
 *
 * Reference interfaces replaced (file:line under proj/core):
 *   bipm_problem_create[_ex] opf::parse_matpower_file + generate_scenarios +
 *                            build_block_opf + make_ad_plan
 *                            (opf_parse.cpp:216, scenarios.cpp:44,
 *                             opf_model.cpp:624, autodiff.cpp:180)
 *   bipm_problem_create_tables  the same from the reference's in-memory
 *                            tables: opf::CaseData + opf::ScenarioSet
 *                            (opf.hpp:54-82; build_block_opf, opf_model.cpp:624)
 *   bipm_problem_create_patterns  make_ad_plan's split patterns +
 *                            make_condense_work (autodiff.hpp:40-60,
 *                            kkt.cpp:111-117): the KKT operators only
 *   bipm_eval_bundle         eval_bundle_range            (autodiff.hpp:131-133)
 *   bipm_eval_values         batch_eval                   (autodiff.hpp:96-97)
 *   bipm_condense            condense                     (kkt.hpp:110, kkt.cpp:123-170)
 *   bipm_factor_gx           factor_gx_range / BlockDiagFactor::factor
 *                                                         (kkt.hpp:162, linalg.cpp:51-89)
 *   bipm_reduce              reduce + finish_reduce       (kkt.hpp:139-142)
 *   bipm_reduce_rhs          reduce_rhs_group + all_reduce_sum (kkt.cpp:209-239)
 *   bipm_dense_factor_solve  factor_dense_sym + solve     (linalg.hpp:116, kkt.cpp:965-976)
 *   bipm_recover             recover_state_adjoint + recover_slack_dual
 *                                                         (kkt.hpp:114,147-148)
 *   bipm_solve_reduced       solve_reduced                (kkt.hpp:170-172, kkt.cpp:945-1006)
 *   bipm_solve               solve (the IPM driver)       (ipm.hpp:361)
 *   bipm_solver_iterate      SolveResult::iterate         (ipm.hpp:41-52, model.hpp:41-55)
 */
#ifndef BIPM_GPU_H
#define BIPM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (reference exception in parentheses) */
#define BIPM_OK 0
#define BIPM_SINGULAR_BLOCK 1   /* SingularBlockError */
#define BIPM_NONFINITE 2        /* NonFiniteError */
#define BIPM_NOT_PD 3           /* reduced matrix not positive definite */
#define BIPM_CUDA_ERROR 4
#define BIPM_INVALID_ARGUMENT 5 /* DimensionError / std::invalid_argument */
#define BIPM_NON_INTERIOR 6     /* NonInteriorError */
#define BIPM_LINEAR_SOLVE 7     /* LinearSolveError */
#define BIPM_PARSE_ERROR 8      /* opf::ParseError */
#define BIPM_UNSUPPORTED 9      /* augmented fallback (not on the GPU path) */

typedef struct bipm_problem bipm_problem; /* host model + symbolic plans */
typedef struct bipm_ctx bipm_ctx;         /* one GPU owning scenarios [lo, hi) */

const char* bipm_last_error(void);
/* global scenario index the last failure names (SingularBlockError::block,
 * NonFiniteError::block; types.hpp:99-109), -1 when none */
int32_t bipm_last_error_block(void);
int bipm_version(void);

/* ---- problem (host, no GPU needed) ---------------------------------- */
/* MATPOWER file + generate_scenarios(cs, N, sigma, {}, seed) */
int bipm_problem_create(const char* case_path, int32_t N, double sigma, uint64_t seed,
                        bipm_problem** out);
/* the same with contingencies: branch indices (into mpc.branch, in service),
 * the k-th outaged in scenario k mod N (scenarios.cpp:44-80) */
int bipm_problem_create_ex(const char* case_path, int32_t N, double sigma, uint64_t seed,
                           const int32_t* contingencies, int32_t n_contingencies,
                           bipm_problem** out);

/* opf::CaseData (opf.hpp:19-62) as row-major tables, file units (MW, MVAr,
 * degrees).  Columns follow the reference's row structs:
 *   bus     [nbus][10]   id type Pd Qd Gs Bs Vm Va Vmax Vmin       (BusRow)
 *   gen     [ngen][9]    bus Pg Qg Qmax Qmin Vg status Pmax Pmin   (GenRow)
 *   branch  [nbranch][9] from to r x b rateA tap shift status      (BranchRow)
 *   gencost [ngencost][4] model startup shutdown ncost, with the ncost
 *           coefficients of row i (highest order first) consecutive in
 *           gencost_coef                                          (GenCostRow) */
#define BIPM_BUS_COLS 10
#define BIPM_GEN_COLS 9
#define BIPM_BRANCH_COLS 9
#define BIPM_GENCOST_COLS 4
typedef struct {
  const char* name;
  double base_mva;
  int32_t nbus, ngen, nbranch, ngencost;
  const double* bus;
  const double* gen;
  const double* branch;
  const double* gencost;
  const double* gencost_coef;
} bipm_case_tables;
/* opf::ScenarioSet (opf.hpp:64-74): multipliers [N][nbus] (the reference's
 * Matrix(nbus, N)); outages of scenario s are outage_branch[outage_ptr[s] ..
 * outage_ptr[s+1]) (branch indices); outage_ptr may be NULL (no outages) */
typedef struct {
  int32_t N;
  double sigma;
  uint64_t seed;
  const double* multipliers;
  const int32_t* outage_ptr;
  const int32_t* outage_branch;
} bipm_scenario_tables;
int bipm_problem_create_tables(const bipm_case_tables* cs, const bipm_scenario_tables* sc,
                               bipm_problem** out);

/* a shared int32 CSR pattern (SparsityPattern, sparse.hpp:13-30) */
typedef struct {
  int32_t rows, cols;
  const int32_t* row_ptr; /* rows + 1 */
  const int32_t* col_ind; /* row_ptr[rows], strictly increasing per row */
} bipm_csr;
/* KKT-operator problem from the derivative patterns of a reference AdPlan:
 * G_x | G_u = g_split.x_pat | u_pat, H_x | H_u = h_split.x_pat | u_pat,
 * W_xx, W_xu, W_uu = w_split.xx, xu, uu.  Contexts of such a problem serve
 * the KKT operators (condense ... solve_reduced); the AD and the IPM driver
 * need an OPF problem. */
int bipm_problem_create_patterns(int32_t N, const bipm_csr* gx, const bipm_csr* gu,
                                 const bipm_csr* hx, const bipm_csr* hu, const bipm_csr* wxx,
                                 const bipm_csr* wxu, const bipm_csr* wuu, bipm_problem** out);
void bipm_problem_destroy(bipm_problem* p);
/* dims[0..9] = N, n_x, n_u, m, n_b, nbus, nbranch, ngen, nnz(L+U) factor, levels(fwd) */
int bipm_problem_dims(const bipm_problem* p, int32_t dims[10]);
/* Read-only view of a named host array (model maps, bounds, patterns, LU
 * plan): *is_int = 1 for int32 data, 0 for float64. */
int bipm_problem_array(const bipm_problem* p, const char* name, const void** data,
                       int64_t* count, int32_t* is_int);

/* ---- engine ---------------------------------------------------------- */
int bipm_ctx_create(const bipm_problem* p, int32_t device, int32_t lo, int32_t hi,
                    bipm_ctx** out);
void bipm_ctx_destroy(bipm_ctx* c);

/* Host inputs of the reduction, all scenario-major over the ctx's M = hi-lo
 * scenarios and laid out on the problem's shared patterns. */
typedef struct {
  const double* gu;      /* [M][nnz G_u] */
  const double* kxx;     /* [M][nnz K_xx] */
  const double* kxu;     /* [M][nnz K_xu] */
  const double* kuu;     /* [M][nnz K_uu] */
  const double* sigma_x; /* [M][n_x] */
  const double* rhat1;   /* [M][n_x] */
  const double* rhat3;   /* [M][n_x] */
  const double* sigma_u; /* [n_u] */
  const double* rhat2;   /* [n_u] */
} bipm_condensed;

/* G_x values [M][nnz G_x] -> batched LU on the device.  On a tiny or
 * non-finite pivot returns BIPM_SINGULAR_BLOCK with *singular_block set to
 * the lowest global scenario index. */
int bipm_factor_gx(bipm_ctx* c, const double* gx, int32_t* singular_block);

/* K_hat (n_u x n_u column-major) and rhs (n_u) of the reduced system at
 * delta_w, exactly as reduce()+finish_reduce(): K_hat includes
 * diag(sigma_u + delta_w), rhs includes -rhat2.  Requires bipm_factor_gx. */
int bipm_reduce(bipm_ctx* c, const bipm_condensed* in, double delta_w, double* khat,
                double* rhs);

/* ---- reduced-strategy operators (kkt.hpp:53-172) --------------------------
 * The augmented system of one ctx (AugmentedSystem, kkt.hpp:53-80) with the
 * bundle blocks it references, scenario-major over the ctx's M scenarios.
 * sigma_u and r1u are the full coupling rows (summed over ALL N scenarios,
 * as assemble_augmented builds them), identical on every rank. */
typedef struct {
  const double *gx, *gu, *hx, *hu, *wxx, *wxu, *wuu; /* [M][nnz] */
  const double *sigma_x, *r1x, *r3;                  /* [M][n_x]; r3 = g */
  const double *sigma_s, *r2, *r4;                   /* [M][m] */
  const double *sigma_u, *r1u;                       /* [n_u] */
} bipm_augmented;
/* CondensedSystem outputs (kkt.hpp:86-103); NULL members are skipped.
 * rhat2 is the full coupling row (all ranks). */
typedef struct {
  double *kxx, *kxu, *kuu; /* [M][nnz K_..] on the condensed patterns (kxx_p, ...) */
  double *rhat1, *rhat3;   /* [M][n_x] */
  double *rhat2;           /* [n_u] */
} bipm_condensed_out;
/* condense(sys, work): BIPM_NON_INTERIOR when a Sigma_s entry is not positive */
int bipm_condense(bipm_ctx* c, const bipm_augmented* a, const bipm_condensed_out* out);
/* reduce_rhs_group over the ctx's scenarios, all-reduced over the ranks:
 * rhs = sum_b [G_u' G_x^{-T} (rhat1 - K~_xx a) + K_xu' a], a = G_x^{-1} rhat3
 * (no -rhat2 term).  Requires bipm_factor_gx. */
int bipm_reduce_rhs(bipm_ctx* c, const bipm_condensed* in, double delta_w, double* rhs);
/* slack-side rows recover_slack_dual needs (kkt.cpp:172-188) */
typedef struct {
  const double *hx, *hu;            /* [M][nnz H_x], [M][nnz H_u] */
  const double *sigma_s, *r2, *r4;  /* [M][m] */
} bipm_slack_rows;
/* recover_state_adjoint + recover_slack_dual at p_u (n_u): p_x, p_y [M][n_x],
 * p_z, p_s [M][m].  Requires bipm_factor_gx. */
int bipm_recover(bipm_ctx* c, const bipm_condensed* in, const bipm_slack_rows* s,
                 double delta_w, const double* pu, double* px, double* py, double* pz,
                 double* ps);
/* RegSchedule (kkt.hpp:20-29); zero fields take the reference default */
typedef struct {
  double delta_w0, delta_w_min, delta_w_max, kappa_minus, kappa_plus, kappa_plus_emergency;
} bipm_reg_schedule;
typedef struct { /* Step (kkt.hpp:38-44); NULL members are skipped */
  double *px, *pu, *ps, *pz, *py;
} bipm_step;
typedef struct { /* StepInfo (kkt.hpp:46-51) + the refinement rounds taken */
  double delta_w;
  int32_t corrections, refinements;
  int64_t reductions;
} bipm_step_info;
/* solve_reduced: condense, batched G_x refactor, inertia loop of reduce +
 * shift + dense Cholesky, recovery and up to 3 refinement rounds, all on the
 * device.  delta_w_last is the warm start carried across calls (in/out).
 * BIPM_SINGULAR_BLOCK (+ the reference's augmented fallback on the caller's
 * side), BIPM_NON_INTERIOR, BIPM_LINEAR_SOLVE map onto the reference's
 * exceptions. */
int bipm_solve_reduced(bipm_ctx* c, const bipm_augmented* a, const bipm_reg_schedule* reg,
                       double* delta_w_last, const bipm_step* out, bipm_step_info* info);

/* Derivative bundle outputs (host, scenario-major over M; any may be NULL):
 * DerivativeBundle (autodiff.hpp:117-127). */
typedef struct {
  double* f;        /* [M] */
  double* g;        /* [M][n_x] */
  double* h;        /* [M][m] */
  double* gx;       /* [M][nnz G_x] */
  double* gu;       /* [M][nnz G_u] */
  double* hx;       /* [M][nnz H_x] */
  double* hu;       /* [M][nnz H_u] */
  double* wxx;      /* [M][nnz W_xx] */
  double* wxu;      /* [M][nnz W_xu] */
  double* wuu;      /* [M][nnz W_uu] */
  double* grad_lag; /* [M][n_x + n_u] */
} bipm_bundle;

/* eval_bundle_range: X, y [M][n_x], u [n_u], z [M][m].  Returns
 * BIPM_NONFINITE (with *bad_block the lowest scenario) when a basis value or
 * derivative is not finite (autodiff.cpp:11-22). */
int bipm_eval_bundle(bipm_ctx* c, const double* X, const double* u, const double* y,
                     const double* z, double obj_weight, const bipm_bundle* out,
                     int32_t* bad_block);
/* batch_eval: values only (line-search trials). */
int bipm_eval_values(bipm_ctx* c, const double* X, const double* u, double* f, double* g,
                     double* h, int32_t* bad_block);

/* ---- multi-GPU: one bipm_ctx per GPU owning a contiguous scenario group
 * (partition, executor.cpp:7-19).  The reduced matrix / rhs partial sums and
 * the scalar norms are all-reduced (all_reduce_sum, executor.cpp:39-61). */
/* ranges[2g], ranges[2g+1] = [lo, hi) of group g: sizes differ by at most
 * one, leading groups take the extra scenario */
int bipm_partition(int32_t N, int32_t G, int32_t* ranges);
/* NCCL (loaded with dlopen): rank 0 creates the id, every rank joins */
int bipm_nccl_unique_id(uint8_t out[128]);
int bipm_ctx_set_nccl(bipm_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank);
/* out = {kind (0 none, 1 NCCL, 2 host callback), communicator ranks, rank} */
int bipm_ctx_comm(const bipm_ctx* c, int32_t out[3]);
/* host-staged exchange through a callback (op: 0 sum, 1 max, 2 min, in place) */
typedef void (*bipm_allreduce_fn)(void* user, double* buf, int64_t n, int32_t op);
int bipm_ctx_set_host_comm(bipm_ctx* c, bipm_allreduce_fn fn, void* user, int32_t nranks,
                           int32_t rank);

/* ---- interior-point driver (ipm.cpp:435-664 on the reduced strategy) ---- */
typedef struct bipm_solver bipm_solver;

typedef struct { /* IpmOptions (ipm.hpp:7-25); zero fields take the default */
  double tol;      /* 1e-6 */
  double mu0;      /* 0.1 */
  int32_t max_iter; /* 300 */
} bipm_solve_options;

#define BIPM_STATUS_NOT_STARTED -2 /* bipm_solver_step before bipm_solver_start: BIPM_INVALID_ARGUMENT */
#define BIPM_STATUS_RUNNING -1
#define BIPM_STATUS_OPTIMAL 0
#define BIPM_STATUS_MAX_ITER 1
#define BIPM_STATUS_INFEASIBLE 2 /* step too small (no restoration, as the reference) */

typedef struct {
  int32_t status;     /* BIPM_STATUS_* */
  int32_t iterations;
  double objective;
  double t_total, t_ad, t_kkt; /* seconds, host clock around device phases */
  int64_t reductions;         /* K_hat assemblies (inertia attempts) */
} bipm_solve_result;

int bipm_solver_create(bipm_ctx* c, const bipm_solve_options* opts, bipm_solver** out);
void bipm_solver_destroy(bipm_solver* s);
/* initial_iterate (ipm.cpp:59-105) */
int bipm_solver_start(bipm_solver* s);
/* one IPM iteration; *status receives BIPM_STATUS_* */
int bipm_solver_step(bipm_solver* s, int32_t* status);
/* result so far; u (n_u, may be NULL) receives the current controls */
int bipm_solver_result(bipm_solver* s, bipm_solve_result* r, double* u);
/* the solver's current primal-dual point (Iterate, model.hpp:41-55), host
 * arrays: x, y, kappa_lo, kappa_up [M][n_x]; s, z, nu_lo, nu_up [M][m];
 * u, lambda_lo, lambda_up [n_u]; NULL members are skipped */
typedef struct {
  double *x, *u, *s, *y, *z, *kappa_lo, *kappa_up, *nu_lo, *nu_up, *lambda_lo, *lambda_up;
} bipm_iterate;
int bipm_solver_iterate(bipm_solver* s, const bipm_iterate* out);
/* IterationLog k: rec[15] = iter, objective, inf_pr, inf_du, complementarity,
 * mu, alpha_primal, alpha_dual, t_ad, t_kkt, t_total, corrections,
 * refinements, delta_w, full_step */
int bipm_solver_log(bipm_solver* s, int32_t k, double rec[15]);
/* one iteration bracketed by CUDA events on the engine stream; restarts the
 * solve when the previous one terminated (bench harness) */
int bipm_solver_step_timed(bipm_solver* s, int32_t* status, double* device_ms);
/* instrumentation: out = kernels launched by this library, H2D bytes, D2H bytes */
int bipm_counters(int64_t out[3]);
/* CUDA-event timing of the named kernel groups (lu_refactor, reduce_tiles,
 * reduce_rhs, cholesky, recover_state, condense, ad_bundle, ad_values);
 * enabling starts a new window (clears), disabling keeps the totals */
int bipm_ctx_profile(bipm_ctx* c, int32_t enable);
int bipm_ctx_kernel_time(bipm_ctx* c, const char* name, double* ms, int64_t* count);
/* debug: clock64 stamps of the reduction phases of CTA (0,0) (16 slots) */
int bipm_ctx_phase_stamps(bipm_ctx* c, int32_t enable, int64_t out[16]);
/* out = reduce tile width, scenarios per CTA, chunks, panel-in-smem, nnz(L),
 * nnz(L+U), LU multiply-adds, SM count, reduction flags (1 streamed, 2
 * presolved forward half, 4 adjoint identity), steps, ring bytes, nnz(VS) */
int bipm_ctx_info(bipm_ctx* c, int64_t out[12]);
/* debug: (step kind, clock64 before its data wait, after it) of every step of
   the streamed reduction's first scenario in CTA (0,0) from the previous
   reduction; n_out triples written */
/* host only: build the streamed reduction's step program for tile width K,
   `consumers` threads and a ring of ring_bytes, and validate it (sweep value
   coverage, ring placement).  out = {violations, steps, nnz_vs, sweep steps,
   dense steps, acc steps, spmv steps, accumulator registers, t0, tl} */
int bipm_problem_stream_check(const bipm_problem* p, int32_t K, int32_t consumers,
                              int32_t ring_bytes, int64_t out[10]);
/* the same for the round-2 program variants: mode bit 1 presolved forward
   half (no L sweep), bit 2 adjoint identity (no L' sweep, y_N accumulation),
   bit 4 deferred tail (Z_T stored for the batch-sum GEMM) */
int bipm_problem_stream_check_ex(const bipm_problem* p, int32_t K, int32_t consumers,
                                 int32_t ring_bytes, int32_t mode, int64_t out[10]);
/* debug: raw copy of the reduction's stamp/trace buffer */
int bipm_ctx_debug_buffer(bipm_ctx* c, int64_t* out, int64_t cap, int64_t* n_out);
int bipm_ctx_step_stamps(bipm_ctx* c, int32_t enable, int64_t* out, int32_t cap, int32_t* n_out);
/* factor_dense_sym + solve (linalg.hpp:116, kkt.cpp:965-976): K (n x n,
 * column-major) shifted by 1e-13 max(1,|K|_inf), Cholesky; *pd = 1 when
 * positive definite, then rhs is overwritten by K^{-1} rhs */
int bipm_dense_factor_solve(int32_t n, const double* k_colmajor, double* rhs, int32_t* pd);
/* The Bunch-Kaufman branch of DenseSymFactor::factor (dsytrf 'L' on the
 * shifted K, linalg.cpp:136-145, lapack.cpp:40-97): inertia = {pos, neg,
 * zero} of D; rhs (may be NULL) is overwritten by K^{-1} rhs when zero = 0.
 * bipm_dense_factor_solve and the engine's inertia loop use it when the
 * Cholesky rejects a pivot within rounding of zero: *pd then reports the BK
 * verdict neg = 0 and zero = 0, as the reference's attempt does
 * (kkt.cpp:969-971). */
int bipm_dense_inertia(int32_t n, const double* k_colmajor, double* rhs, int32_t inertia[3]);
/* out = {attempts decided by the Bunch-Kaufman inertia so far, the accepted
 * K_hat factor is Bunch-Kaufman (1) or Cholesky (0)} */
int bipm_ctx_factor_stats(bipm_ctx* c, int64_t out[2]);
/* whole solve: start + steps until a terminal status */
int bipm_solve(bipm_ctx* c, const bipm_solve_options* opts, bipm_solve_result* r, double* u);

#ifdef __cplusplus
}
#endif

#endif /* BIPM_GPU_H */
