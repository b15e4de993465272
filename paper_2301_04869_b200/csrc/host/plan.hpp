// Symbolic, scenario-independent plans built once per solve on the host.
//
//  * derivative patterns: the reference detects G, H and the Lagrangian
//    Hessian supports by index propagation through the basis
//    (autodiff.cpp:93-124, opf_model.cpp:277-327) and splits them into state
//    and control blocks (autodiff.cpp:126-178).  The same patterns are
//    reproduced here so per-scenario value arrays line up slot for slot with
//    the reference boundary.
//  * condense gather programs: K = W + A' diag(sigma) B as, for every output
//    slot, its W slot and the (a slot, b slot, row) triples that feed it, in
//    the reference's accumulation order (sparse.cpp:176-214).
//  * the static-pivot sparse LU of G_x: one symmetric minimum-degree ordering
//    shared by every scenario, its factor pattern, level schedules for the
//    four triangular sweeps, and the numeric refactor program.  This replaces
//    the reference's per-scenario Eigen::SparseLU (linalg.cpp:76-104).
#pragma once

#include <vector>

#include "common.hpp"
#include "grid_model.hpp"

namespace bipm {

struct LaneDeps {
  std::vector<std::vector<idx>> jac;   // first-derivative support per lane
  std::vector<std::vector<idx>> hess;  // inputs entering nonlinearly
};
LaneDeps basis_deps(const OpfModel& M);

struct SplitMap {
  Csr x, u;                 // column split at n_x
  std::vector<idx> x_src, u_src;  // slot in the unsplit pattern
};

struct CondenseProgram {
  Csr out;                       // pattern of W + A' S B
  std::vector<idx> w_of;         // per out slot: W slot or -1
  std::vector<idx> ptr;          // per out slot: range into (ka, kb, r)
  std::vector<idx> ka, kb, r;
};

struct DerivPlan {
  Csr jac_g, jac_h, hess;        // n_x x n_d, m x n_d, n_d x n_d
  SplitMap g, h;                 // G_x | G_u, H_x | H_u
  Csr wxx, wxu, wuu;             // Hessian split blocks
  std::vector<idx> wxx_src, wxu_src, wuu_src;  // slot in `hess`
  CondenseProgram kxx, kxu, kuu;
};

DerivPlan make_deriv_plan(const OpfModel& M, const LaneDeps& deps);
CondenseProgram plan_condense_program(const Csr& W, const Csr& A, const Csr& B);

// One triangular sweep over the permuted rows in "direct value" form: entry t
// of row i has column col[t] and value V[t] of the sweep's value array (F or
// FT below); with has_diag the first entry of each row is its diagonal.
// Rows [t0, n) (the trailing separator block) are not level-scheduled: they
// are solved as a dense triangle in registers; forward sweeps first gather
// their entries with col < t0 (tail_items).
struct SweepPlan {
  bool has_diag = false, forward = true;
  std::vector<idx> ptr, col;
  std::vector<idx> lvl_ptr;     // item ranges per level
  std::vector<idx> items;       // 4 ints per item: row, beg, end, 0
  std::vector<idx> tail_items;  // 4 ints per tail row (forward sweeps): row, beg, split, 0
};

// Static-pivot LU of a structurally symmetric n x n pattern (P A P' = L U).
// Factor values of one scenario live in one array of length nnz_f:
//   [0, nnz_l)        strict lower L, row-major by permuted row
//   [nnz_l, nnz_f)    upper U including the diagonal, row-major
struct LuPlan {
  idx n = 0, nnz_l = 0, nnz_f = 0;
  std::vector<idx> perm, iperm;  // permuted k <-> original perm[k]
  // row access (permuted indices): L strict lower / U strict upper / diag slot
  std::vector<idx> l_ptr, l_col, l_slot;
  std::vector<idx> u_ptr, u_col, u_slot;
  std::vector<idx> diag;
  // column access for the transposed sweeps: column i of U above the
  // diagonal (rows k < i) and column i of L below it (rows r > i)
  std::vector<idx> ut_ptr, ut_row, ut_slot;
  std::vector<idx> lt_ptr, lt_row, lt_slot;
  // level schedules: forward (L, U') and backward (U, L') sweeps
  std::vector<idx> fwd_ptr, fwd_rows, bwd_ptr, bwd_rows;
  // numeric refactor: per level of the forward schedule, the U-row entries
  // then the L-column entries of its pivot steps (factor slots); each entry
  // e: value = A[a_src[e]] (or 0) - sum_t F[mul_l[t]] * F[mul_u[t]]
  // over t in [mul_ptr[e], mul_ptr[e+1]); L entries then divide by the pivot.
  std::vector<idx> lvl_u_ptr, lvl_u_slot, lvl_l_ptr, lvl_l_slot;
  // the same program split at the dense tail (refactor_levels_kernel /
  // refactor_tail_kernel): levels of the pivots j < t0 only, then for every
  // factor slot of the tail block the terms k < t0 of its sum (the tail block
  // is then factorised densely)
  std::vector<idx> nt_lvl_u_ptr, nt_lvl_u_slot, nt_lvl_l_ptr, nt_lvl_l_slot;
  std::vector<idx> tail_slot, tail_mul_ptr, tail_mul_l, tail_mul_u;
  // the same split program flattened for refactor_levels_kernel: phases (U
  // entries of a level, L entries of a level, ..., tail block), one record per
  // factor slot {slot, pair begin, pair end, G_x slot or -1} + its pivot slot
  // (-1: no division), multiply pairs (L position, U slot) contiguous
  std::vector<idx> rf_phase_ptr, rf_rec, rf_piv, rf_pair;
  std::vector<idx> a_src;       // per factor slot: G_x slot or -1 (fill)
  std::vector<idx> piv_of;      // per factor slot: pivot slot for L entries, -1 for U
  std::vector<idx> mul_ptr, mul_l, mul_u;
  long long flops() const { return 2LL * (long long)mul_l.size(); }

  // ---- sweep layouts for the solve kernels
  // F  = [L strict rows | U rows (diag first)]      (the refactor output)
  // FT = [U' rows (diag first, then U(k,i), k<i) | L' rows (L(r,i), r>i)]
  idx t0 = 0, tl = 0;             // dense tail rows [t0, n), tl = n - t0
  std::vector<idx> ft_src;        // FT[p] = F[ft_src[p]]
  // dense tail blocks, column-major tl x tl, source F slot or -1 (zero):
  //   0: L_TT (unit lower)   1: U_TT (upper)
  // The refactor turns them into W = (L_TT U_TT)^{-1} (row-major) and W'
  // (row-major), so a solve's tail is one dense product per sweep pair.
  std::vector<idx> dense_src[2];
  SweepPlan sL, sU, sUt, sLt;
};

// dense tail selection (make_lu_plan): top etree levels of at most
// kTailWidth rows, at most kMaxTail rows (env BIPM_TAIL_WIDTH / BIPM_TAIL_MAX,
// the latter clamped to kMaxTailLimit).  Measured at 1354: width 6 (tl 233)
// -> 16 (tl 307): the reduction loses more sweep levels than it gains DMMA
// work, -10 % per reduction, +1.2 ms per refactor, -6 % per iteration; wider
// tails (width 32: tl 452, 64: tl 489) shave another 5 % off the reduction
// but the Gauss-Jordan inverse grows as tl^3 (7-12 ms per refactor): net loss.
// Round 2 (presolved reduction, same box): width 8 (tl 262) 19.40, 10 (tl 272)
// 18.85, 12-20 (tl 307) 19.23 ms per reduction + refactor at 1354/256.
constexpr idx kTailWidth = 10;
constexpr idx kMaxTail = 320;
constexpr idx kMaxTailLimit = 512;  // the Gauss-Jordan kernel's limit (env BIPM_TAIL_MAX up to it)
constexpr idx kWideTailN = 4000;    // n >= this: width 32, up to kMaxTailLimit rows

std::vector<idx> min_degree_order(const Csr& sym_pattern);
LuPlan make_lu_plan(const Csr& gx_pattern);
void build_sweeps(LuPlan& P, const std::vector<std::vector<idx>>& lrow,
                  const std::vector<std::vector<idx>>& urow, const std::vector<idx>& fwd_level);

}  // namespace bipm
