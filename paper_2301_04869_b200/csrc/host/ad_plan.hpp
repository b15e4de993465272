// Gather programs for the analytic batched AD of the polar basis on the GPU.
//
// The reference evaluates first derivatives by colored forward mode and the
// Lagrangian Hessian by forward-over-reverse over a hand-coded adjoint
// (autodiff.cpp:283-415, opf_model.cpp:199-576).  On the GPU every basis
// element (bus, branch, generator, slack) differentiates itself analytically
// and the sparse products with L_f, L_g, L_h become fixed gather lists built
// here once per solve.  Outputs land on the reference's patterns
// (plan.hpp: DerivPlan), so values line up slot for slot.
//
// Per-scenario scratch arrays:
//   psi[n_b]     basis values
//   dp[n_dp]     first partials of every lane w.r.t. its jac deps, lane-major
//   w[n_b]       Lagrangian lane weights  obj_w L_f' + L_g' y + L_h' z
//   c[n_c]       element-local gradient / Hessian contributions:
//                  branch l: 14 at 14 l  (grad th_f th_t v_f v_t, then the 10
//                           upper-triangle Hessian entries of that order)
//                  bus b:    2 at c_bus + 2 b   (grad v, H(v,v))
//                  gen g:    2 at c_gen + 2 g   (grad p, H(p,p))
//                  slack:    |sd|^2 at c_slack  (2 w_sl2 grad p grad p')
#pragma once

#include <vector>

#include "plan.hpp"

namespace bipm {

struct Gather {
  std::vector<idx> ptr{0};
  std::vector<idx> src;
  std::vector<double> coef;  // empty: all coefficients are 1
  void push(idx s, double c) {
    src.push_back(s);
    coef.push_back(c);
  }
  void push(idx s) { src.push_back(s); }
  void close() { ptr.push_back(idx(src.size())); }
  idx outputs() const { return idx(ptr.size()) - 1; }
};

struct AdProgram {
  idx n_dp = 0, n_c = 0, c_bus = 0, c_gen = 0, c_slack = 0;
  std::vector<idx> dp_off;            // per lane (n_b + 1)
  std::vector<idx> sd;                // slack dependencies (inputs), sorted
  std::vector<idx> branch_ref;        // per branch: bit0 from-end at ref, bit1 to-end at ref
  std::vector<idx> gen_ref_other;     // per live gen: 1 if a non-slack gen at the ref bus
  Gather slack_val;   // 1 output: (coef, lane) after starting from psi[pd_ref]
  Gather slack_grad;  // |sd| outputs: (coef, dp index)
  Gather w;           // per lane: (coef, src) src<0 obj weight, <n_x y, else z
  Gather gx, gu, hx, hu;   // per slot: (coef, dp index)
  Gather grad;             // per input (n_d): contribution indices
  Gather wxx, wxu, wuu;    // per slot: contribution indices
};

AdProgram make_ad_program(const OpfModel& M, const LaneDeps& deps, const DerivPlan& D);

}  // namespace bipm
