// The reduced-strategy Newton step as one device-resident operator.
//
// Restates solve_reduced (proj/core/src/kkt.cpp:945-1006) from an assembled
// augmented system onwards: condense (kkt.cpp:123-170), factor_gx_range for
// every owned scenario (kkt.cpp:190-196), the inertia-correction loop
// (kkt.cpp:742-772) whose attempts run reduce + finish_reduce + shift +
// dense factor (kkt.cpp:954-971), the p_u solve and recovery
// (kkt.cpp:507-532, 172-188) and up to three refinement rounds against the
// unreduced augmented system (kkt.cpp:988-999).
//
// Inputs live in the engine (bundle e.bd(): G/H/W values and g = r3;
// e.sigma_x, e.sigma_s, e.sigma_u, e.r2, e.r4) and here (r1x, r1u).  The
// interior-point driver (solver.cu) assembles them on the device; the C-ABI
// operator bipm_solve_reduced uploads them from the host.  The step lands in
// p[] = (p_x, p_u, p_s, p_z, p_y).
#pragma once

#include "../kernels/ipm_kernels.hpp"
#include "host_link.hpp"

namespace bipm {

struct RegOptions {  // RegSchedule (kkt.hpp:20-29)
  double delta_w0 = 1e-4, delta_w_min = 1e-20, delta_w_max = 1e40;
  double kappa_minus = 1.0 / 3.0, kappa_plus = 8.0, kappa_plus_emergency = 100.0;
};

class KktStep {
 public:
  explicit KktStep(Engine& e, int refine_rounds = 3);

  // augmented-system rows the engine does not hold
  DArr<double> r1x, r1u;  // [M][n_x], [n_u]
  // the step: p_x [M][n_x], p_u [n_u], p_s [M][m], p_z [M][m], p_y [M][n_x]
  DArr<double> p[5];
  int corrections = 0, refinements = 0;
  double last_dw = 0;        // delta_w of the accepted attempt
  long long reductions = 0;  // Schur reductions run (full K_hat assemblies)
  long long mixed = 0;       // attempts whose K_hat came from the affine identity
  int refine_rounds = 3;
  // K_hat and the reduced rhs are affine in delta_w (K~_xx = K_xx +
  // diag(sigma_x + dw): K_hat(dw) = K_hat(0) + dw (I + sum T'T)),
  // so from the third attempt of a step on they are interpolated from the
  // first two reductions instead of re-running the reduction (kkt.cpp:954-959
  // re-reduces every attempt).  BIPM_RETRY_EXACT=1 re-reduces every attempt.
  bool exact_retries = false;

  // condense (kkt.cpp:123-170): K blocks and rhat1 / rhat2 / rhat3 (= g)
  void condense();
  // the same split around the refactor: condense_begin forks the per-scenario
  // part onto the engine's side stream (it only reads the bundle and writes
  // the condensed blocks, so it runs beside the refactor's levels kernel);
  // condense_end joins it and does the cross-scenario rhat2 sum on st
  void condense_begin();
  void condense_end();
  // batched refactor of G_x (statuses stay on the device until check_factor)
  void factor_launch();
  // one host round trip for the refactor statuses and, when given, a device
  // interiority flag: throws NonInterior (flag set on any rank) or
  // SingularBlock (lowest singular global scenario over the ranks)
  void check_factor(const DArr<int>* interior_flag);
  // inertia loop + attempts; delta_w_last carries the warm start across
  // steps (solve_reduced's in/out argument)
  void solve(double& delta_w_last, const RegOptions& reg);

  DevStep step_view() { return view(p); }

 private:
  bool attempt(double dw, int k);
  void condensed_u_sum(const double* part, const double* base, double* out);
  DevStep view(DArr<double>* s) {
    return DevStep{s[0].get(), s[1].get(), s[2].get(), s[3].get(), s[4].get()};
  }

  Engine& e;
  IpmDims d{};
  HostLink io;
  DArr<double> q[5];  // refinement correction
  DArr<double> o1x, o1u, o2, o3, o4, o1u_part;
  DArr<double> c_rhat1, c_rhat2, rhs_sum, red_u, dd_u, rhat2_part;
  DArr<double> partial, scal;
  DArr<double> khat0, khat1, rhs0, rhs1;  // attempts 0 and 1 of the current step
  double dw0 = 0.0, dw1 = 0.0;
  // condense_begin / condense_end (events owned here, destroyed with the step)
  cudaEvent_t ev_cond0 = nullptr, ev_cond1 = nullptr;
  bool cond_forked = false;

 public:
  KktStep(const KktStep&) = delete;
  KktStep& operator=(const KktStep&) = delete;
  ~KktStep() {
    if (ev_cond0) cudaEventDestroy(ev_cond0);
    if (ev_cond1) cudaEventDestroy(ev_cond1);
  }
};

}  // namespace bipm
