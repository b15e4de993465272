// Host-side launchers for the reduced-KKT kernels (kkt_kernels.cu).
// All pointers are device pointers; per-scenario arrays are scenario-major
// ([scenario][slot]), the reference boundary layout.
#pragma once

#include <cuda_runtime.h>

#include "device_plan.cuh"

namespace bipm {

// Batched static-pivot refactor of G_x: F[s] = LU(P G_x[s] P').  status[s]
// is set to 1 when a pivot falls below piv_tol * max|G_x[s]| (or is not
// finite), mirroring SingularBlockError (linalg.cpp:69-73).
// Also writes the transposed copy FT [M][nnz_f] and the dense tail blocks
// D [M][4 tl tl] used by the solve kernels.
// VS (optional, [M][nnz_vs]): VS[s][q] = F[s][vs_src[q]] (0 where -1), the
// sweep-ordered factor values of the streamed reduction (reduce_stream.cu).
// Dp (optional, [M][2 tl dense_ld(tl)]): W, W' with rows padded to
// (tl + 15) & ~15 doubles, zero-filled, for the streamed reduction's dense step.
void launch_lu_refactor(const DevLu& P, int M, const double* gx, int nnz_gx, double* F,
                        double* FT, double* D, int* status, double piv_tol, const int* vs_src,
                        int nnz_vs, double* VS, double* Dp, double* scale, cudaStream_t st,
                        int dp_slot = -1, cudaEvent_t after_levels = nullptr);
// scale: [M] doubles of scratch (per-scenario max |G_x| for the pivot guard);
// dp_slot >= 0: only W (0) or W' (1) is padded into Dp (the other is unread);
// after_levels: recorded on st once the non-tail factor (L_NN, L_TN, U_N*)
// is final, before the dense tail (the reach solve needs nothing more)

struct ReduceLaunch {
  DevLu lu;
  DevCsr gu, kxx, kxu, kuu;
  int n_x, n_u, M;
  const double *F, *FT, *D, *gu_v, *kxx_v, *kxu_v, *kuu_v, *sigma_x;
  double dw;
  int kc;           // right-hand-side columns per tile
  int chunk;        // scenarios per CTA
  int nchunks;
  bool panel_in_smem;
  double* partial;  // [nchunks][n_u * n_u] column-major
  double* scratch;  // per-CTA L_x staging (+ panel when not in shared memory)
  long long* phase; // optional: clock64 stamps of CTA (0,0), first scenario (16 slots)
};
void plan_reduce_launch(ReduceLaunch& a, int smem_budget_bytes, int sm_count);
size_t reduce_scratch_doubles(const ReduceLaunch& a);
size_t reduce_smem_bytes(const ReduceLaunch& a);
void launch_reduce_tiles(const ReduceLaunch& a, cudaStream_t st);

// out[j] = sum_c parts[c][j] (fixed pairwise order) + (diag_add ? diag_add[u] + dw on the
// diagonal of an n x n column-major matrix : 0); n_mat = n (0: plain vector of length len)
// out = a + t (b - a) over len doubles (the inertia loop's affine K_hat(dw))
void launch_affine_mix(const double* a, const double* b, double t, long long len, double* out,
                       cudaStream_t st);
void launch_sum_parts(const double* parts, int nparts, long long len, double* out,
                      const double* diag_add, double dw, int n_mat, const double* sub_vec,
                      cudaStream_t st, int sym_n = 0);

struct RhsLaunch {
  DevLu lu;
  DevCsr gu, kxx, kxu;
  int n_x, n_u, M;
  const double *F, *FT, *D, *gu_v, *kxx_v, *kxu_v, *sigma_x;
  const double *rhat1, *rhat3;  // [M][n_x]
  double dw;
  double* part;  // [M][n_u] per-scenario contributions
  double* scratch;  // [M][2 n_x] when single_rhs_smem(n_x) == 0, else unused
  long long* phase = nullptr;  // debug: clock64 per phase of scenario 0
};
// shared memory of the single-RHS kernels' two n_x vectors, 0 when they do
// not fit (the caller then provides RhsLaunch/RecoverLaunch::scratch)
size_t single_rhs_smem(int n_x);
void launch_reduce_rhs(const RhsLaunch& a, cudaStream_t st);

struct RecoverLaunch {
  DevLu lu;
  DevCsr gu, kxx, kxu;
  int n_x, n_u, M;
  const double *F, *FT, *D, *gu_v, *kxx_v, *kxu_v, *sigma_x;
  const double *rhat1, *rhat3, *pu;
  double dw;
  double *px, *py;  // [M][n_x]
  double* scratch;  // [M][2 n_x] when single_rhs_smem(n_x) == 0, else unused
};
void launch_recover_state(const RecoverLaunch& a, cudaStream_t st);

// p_z = Sigma_s (H_x p_x + H_u p_u + r4) - r2;  p_s = -(r2 + p_z) / Sigma_s
void launch_recover_slack(const DevCsr& hx, const DevCsr& hu, int m, int n_x, int M,
                          const double* hx_v, const double* hu_v, const double* px,
                          const double* pu, const double* sigma_s, const double* r2,
                          const double* r4, double* pz, double* ps, cudaStream_t st);

// K = W + A' diag(sigma) B per scenario with the host gather program.
struct CondenseDev {
  int nout;
  const int *w_of, *ptr, *ka, *kb, *r;
};
void launch_condense(const CondenseDev& c, int M, const double* W, int ldw, const double* A,
                     int lda, const double* B, int ldb, const double* sigma, int lds, double* out,
                     cudaStream_t st);

// Dense symmetric factor of the n x n column-major K (lower Cholesky in place)
// with the reference's diagonal shift 1e-13 max(1, |K|_inf) (kkt.cpp:965-968).
// info (device int): 0 when positive definite, else 1 + failing column.
// info: 8 ints = {status (0, or the failing column + 1), pad, |K|_inf (double),
// the rejected pivot (double), pad}
void launch_shift_cholesky(double* K, int n, int* info, double* work, cudaStream_t st);
// Bunch-Kaufman LDL' of the shifted K (dense_bk.cu): factor in place, ipiv
// (LAPACK convention, 1-based), inertia[3] = pos, neg, zero; state: bk_work_bytes
size_t bk_work_bytes(int n);
void launch_bk_factor(double* K, int n, int* ipiv, void* state, int* inertia, cudaStream_t st);
void launch_bk_solve(const double* F, int n, const int* ipiv, double* b, cudaStream_t st);
void launch_cholesky_solve(const double* Lfac, int n, double* b, cudaStream_t st);
// n above the shared-memory kernel's range (dense_chol.cu)
void launch_blocked_cholesky(double* K, int n, int* info, cudaStream_t st);
void launch_blocked_solve(const double* L, int n, double* b, cudaStream_t st);

}  // namespace bipm
