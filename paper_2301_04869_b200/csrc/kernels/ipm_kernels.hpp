// Device kernels of the interior-point iteration around the reduced KKT path
// (residuals, augmented/condensed right-hand sides, refinement residual,
// bound steps, fraction to boundary, step application, merit terms).
//
// Reference (proj/core/src): ipm.cpp:59-172 (start point, bound steps,
// fraction to boundary), ipm.cpp:256-432 (merit terms, scaled error,
// apply_step), autodiff.cpp:441-482 (assemble_residuals), kkt.cpp:67-109
// (assemble_augmented), kkt.cpp:155-168 and 342-358 (condensed rhs),
// kkt.cpp:252-339 (augmented residual, long double -> double-double here).
#pragma once

#include <cuda_runtime.h>

#include "device_plan.cuh"

namespace bipm {

struct IpmDims {
  int M, n_x, n_u, m, n_d;
};

// a primal-dual point; u-sized arrays replicated on every engine
struct DevIter {
  double *x, *u, *s, *y, *z, *klo, *kup, *nlo, *nup, *llo, *lup;
};

struct DevBounds {
  const double *xlo, *xup, *ulo, *uup, *slo, *sup;
};

struct DevStep {
  double *px, *pu, *ps, *pz, *py;
};

struct DevBoundStep {
  double *klo, *kup, *nlo, *nup, *llo, *lup;
};

// Reduction slots are combined across blocks in a fixed order (deterministic).
enum RedOp : int { kSum = 0, kMax = 1, kMin = 2 };

// ---- residuals -----------------------------------------------------------
// out[0..5] = max|stat_x|, max|stat_s|, max|g|, max|h+s|, comp(mu) over x/s,
//             sum|multipliers| over x/s entries
void launch_kkt_error_xs(const IpmDims& d, const DevIter& it, const DevBounds& b,
                         const double* grad, const double* g, const double* h, double mu,
                         double* partial, double* out6, cudaStream_t st);
// gsum_u[i] = sum_s grad[s][n_x+i]   (fixed scenario order)
void launch_grad_u_sum(const IpmDims& d, const double* grad, double* gsum_u, cudaStream_t st);
// out[0..2] = max|stat_u|, comp(mu) over u, sum|lambda| (finite sides)
void launch_kkt_error_u(const IpmDims& d, const DevIter& it, const DevBounds& b,
                        const double* gsum_u, double mu, double* out3, cudaStream_t st);

// Fused residual evaluation (assemble_residuals + scaled_error ingredients,
// autodiff.cpp:441-482, ipm.cpp:345-379) for up to 4 barrier parameters in one
// pass; the last block to finish combines the block partials in a fixed order
// and adds the control part.  out[17]:
//   0 max|stat_x|  1 max|stat_s|  2 max|g|  3 max|h+s|  4..7 comp(mu_k) x/s
//   8 sum|mult| x/s  9 sum f  10 lowest non-finite global scenario (1e300: none)
//   11 max|stat_u| 12..15 comp(mu_k) u  16 sum|lambda|
void launch_kkt_eval(const IpmDims& d, const DevIter& it, const DevBounds& b, const double* grad,
                     const double* g, const double* h, const double* f, const int* bad, int lo,
                     const double* gsum_u, const double mus[4], double* partial,
                     unsigned int* counter, double* out, cudaStream_t st);

// ---- augmented / condensed systems -----------------------------------------
// sigma_x, r1x, sigma_s, r2, r4 (kkt.cpp:83-99); *flag = 1 if not interior
void launch_assemble_xs(const IpmDims& d, const DevIter& it, const DevBounds& b,
                        const double* grad, const double* h, double mu, double* sigma_x,
                        double* r1x, double* sigma_s, double* r2, double* r4, int* flag,
                        cudaStream_t st);
// sigma_u, r1u (kkt.cpp:101-107) from gsum_u
void launch_assemble_u(const IpmDims& d, const DevIter& it, const DevBounds& b,
                       const double* gsum_u, double mu, double* sigma_u, double* r1u, int* flag,
                       cudaStream_t st);
// rhat1 = r1x + H_x' t and part[s] = H_u' t, t = Sigma_s r4 - r2
void launch_condensed_rhs(const IpmDims& d, const DevCsr& hx, const DevCsr& hu,
                          const double* hx_v, const double* hu_v, const double* sigma_s,
                          const double* r4, const double* r2, const double* r1x, double* rhat1,
                          double* part_u, cudaStream_t st);
// out[i] = base[i] + sum_s part[s][i]   (fixed order)
void launch_scenario_sum(int M, int n, const double* part, const double* base, double* out,
                         cudaStream_t st);

// ---- refinement residual (double-double accumulation) --------------------
struct AugResidualArgs {
  IpmDims d;
  DevCsr gx, gu, hx, hu, wxx, wxu, wuu;
  const double *gx_v, *gu_v, *hx_v, *hu_v, *wxx_v, *wxu_v, *wuu_v;
  const double *sigma_x, *sigma_s, *sigma_u;
  const double *r1x, *r1u, *r2, *r3, *r4;  // system rhs
  DevStep p;
  double dw;
  double *o1x, *o2, *o3, *o4;  // residual rows [M][.]
  double *o1u_part;            // [M][2 n_u] double-double partials
};
// Writes the residual rows and max|row| partials; the u row is finished by
// launch_aug_residual_u.  out[0] = max over x/s rows.
void launch_aug_residual(const AugResidualArgs& a, double* partial, double* out1,
                         cudaStream_t st);
// o1u = r1u + (sigma_u + dw) p_u + sum_s part (double-double); out[0] = max|o1u|
// dd: 2 n_u doubles of scratch (double-double sums), owned by the caller
void launch_aug_residual_u(const AugResidualArgs& a, double* dd, double* o1u, double* out1,
                           cudaStream_t st);
// sharded variant: dd[2 n_u] = local sum of the per-scenario u-row partials
// (hi, lo); after the cross-rank all-reduce, finish adds r1u + (sigma_u+dw) p_u
void launch_aug_residual_u_local(const AugResidualArgs& a, double* dd, cudaStream_t st);
void launch_aug_residual_u_finish(const AugResidualArgs& a, const double* dd, double* o1u,
                                  double* out1, cudaStream_t st);
// max(1, |r1x|, |r1u|, |r2|, |r3|, |r4|) partial pieces
void launch_rhs_scale(const IpmDims& d, const double* r1x, const double* r1u, const double* r2,
                      const double* r3, const double* r4, double* partial, double* out1,
                      cudaStream_t st);
void launch_axpy_step(const IpmDims& d, DevStep a, DevStep q, cudaStream_t st);  // a += q

// ---- step sizes and updates --------------------------------------------------
// BoundSteps::compute + fraction_to_boundary: out[0] = alpha_p, out[1] = alpha_d
void launch_bound_steps(const IpmDims& d, const DevIter& it, const DevBounds& b, const DevStep& p,
                        double mu, double tau, DevBoundStep bs, double* partial, double* out2,
                        cudaStream_t st);
// trial = it + (ap, ad) step, then the kappa_sigma multiplier safeguard
void launch_apply_step(const IpmDims& d, const DevIter& it, DevIter trial, const DevBounds& b,
                       const DevStep& p, const DevBoundStep& bs, double ap, double ad, double mu,
                       cudaStream_t st);
// primal-only trial for the l1-merit line search
void launch_primal_trial(const IpmDims& d, const DevIter& it, DevIter trial, const DevStep& p,
                         double alpha, cudaStream_t st);

// merit terms at the iterate: out[0..7] = viol, max|y+py|, max|z+pz|, barrier
// log sum (x/s part), barrier directional (x/s), objective directional,
// sum f, sum |f|
void launch_merit(const IpmDims& d, const DevIter& it, const DevBounds& b, const DevStep& p,
                  const double* grad, const double* f, const double* g, const double* h,
                  const DevCsr& gx, const DevCsr& gu, const DevCsr& hx, const DevCsr& hu,
                  const double* gx_v, const double* gu_v, const double* hx_v,
                  const double* hu_v, double mu, double* partial, double* out8,
                  cudaStream_t st);
// u-part of the barrier terms: out[0] = log sum, out[1] = directional
void launch_merit_u(const IpmDims& d, const DevIter& it, const DevBounds& b, const double* pu,
                    double mu, double* out2, cudaStream_t st);
// line-search trial values: out[0..2] = sum f, barrier log sum (x/s), viol
void launch_ls_values(const IpmDims& d, const DevIter& trial, const DevBounds& b,
                      const double* f, const double* g, const double* h, double* partial,
                      double* out3, cudaStream_t st);

// p_u right-hand side: first solve (kkt.cpp:983-985) pu = ((S - r) + r) - r,
// refinement solves (kkt.cpp:975, 996) pu = S - r
void launch_pu_rhs(int n, const double* S, const double* r, double* pu, bool first,
                   cudaStream_t st);

// ---- start point ---------------------------------------------------------------
void launch_init_slacks(const IpmDims& d, DevIter it, const DevBounds& b, const double* h,
                        double mu0, cudaStream_t st);
void launch_init_x(const IpmDims& d, DevIter it, const DevBounds& b, const double* x0,
                   double mu0, cudaStream_t st);

}  // namespace bipm
