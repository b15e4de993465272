// Reference-side drop-in of the B200 engine (the C++ shim INTEGRATION.md
// describes), linked UNDER the reference's own interior-point driver.
//
// The reference's ipm.cpp calls three functions of the hot path across
// object-file boundaries:
//   compute_step   -> solve_reduced      (ipm.cpp:186-188; kkt.cpp:945-1006)
//   Engine::eval_bundle_into -> eval_bundle_range   (ipm.cpp:227-232;
//                                                     autodiff.cpp:484-516)
//   Engine::eval_values -> batch_eval    (ipm.cpp:237-254; autodiff.cpp:256-281)
// Linking the unmodified reference objects with
//   -Wl,--wrap=<mangled solve_reduced> [--wrap=<eval_bundle_range> --wrap=<batch_eval>]
// routes those calls here; each wrapper forwards to the C-ABI
// (include/bipm_gpu.h) and maps status codes back onto the reference's
// exception types, so ipm.cpp's own control flow -- including the
// SingularBlockError -> augmented fallback (ipm.cpp:502-507) and the
// NonFiniteError trial rejection (ipm.cpp:539-541) -- is unchanged.
// Disabled wrappers call the original (__real_) function.
//
//  * solve_reduced: a KKT-only GPU problem built from the bundle's own
//    patterns (DerivativeBundle::plan, bipm_problem_create_patterns) and one
//    context over all N scenarios; each call uploads the augmented system
//    and runs bipm_solve_reduced.
//  * eval_bundle_range / batch_eval: an OPF GPU problem built from the
//    caller's CaseData + ScenarioSet (bipm_problem_create_tables), one
//    context per scenario group [lo, lo + ws.batch()).
#include "bipm_reference_shim.hpp"

#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bipm_gpu.h"
#include "blockipm/autodiff.hpp"
#include "blockipm/kkt.hpp"

using namespace blockipm;

#define BIPM_SYM_SOLVE_REDUCED                                                                   \
  "_ZN8blockipm13solve_reducedERNS_15AugmentedSystemERKNS_12CondenseWorkERKNS_11RegScheduleERdi" \
  "RNS_8ExecutorERKNS_9PartitionEPNS_8StepInfoE"
#define BIPM_SYM_EVAL_BUNDLE_RANGE                                                               \
  "_ZN8blockipm17eval_bundle_rangeERKNS_8BlockNlpERKNS_6AdPlanERNS_11AdWorkspaceERKNS_6MatrixE" \
  "RKSt6vectorIdSaIdEESA_SA_diRNS_16DerivativeBundleE"
#define BIPM_SYM_BATCH_EVAL                                                                      \
  "_ZN8blockipm10batch_evalERKNS_8BlockNlpERKNS_6MatrixERKSt6vectorIdSaIdEEiRNS_11AdWorkspaceER" \
  "S8_RS3_SE_"

// the originals (resolved by the linker's --wrap)
Step real_solve_reduced(AugmentedSystem&, const CondenseWork&, const RegSchedule&, double&,
                        index_t, Executor&, const Partition&, StepInfo*)
    __asm__("__real_" BIPM_SYM_SOLVE_REDUCED);
void real_eval_bundle_range(const BlockNlp&, const AdPlan&, AdWorkspace&, const Matrix&,
                            const Vector&, const Matrix&, const Matrix&, double, index_t,
                            DerivativeBundle&) __asm__("__real_" BIPM_SYM_EVAL_BUNDLE_RANGE);
void real_batch_eval(const BlockNlp&, const Matrix&, const Vector&, index_t, AdWorkspace&,
                     Vector&, Matrix&, Matrix&) __asm__("__real_" BIPM_SYM_BATCH_EVAL);

namespace {

struct ShimState {
  int device = 0;
  bool kkt = false, ad = false;
  long long kkt_calls = 0, ad_calls = 0;
  // solve_reduced: keyed on the bundle's plan (one problem per solve)
  const void* kkt_key = nullptr;
  bipm_problem* kkt_prob = nullptr;
  bipm_ctx* kkt_ctx = nullptr;
  // AD: one problem, one context per scenario group
  bipm_problem* opf_prob = nullptr;
  std::map<std::pair<index_t, index_t>, bipm_ctx*> ad_ctx;

  ~ShimState() { release(); }
  void release_kkt() {
    if (kkt_ctx) bipm_ctx_destroy(kkt_ctx);
    if (kkt_prob) bipm_problem_destroy(kkt_prob);
    kkt_ctx = nullptr;
    kkt_prob = nullptr;
    kkt_key = nullptr;
  }
  void release() {
    release_kkt();
    for (auto& kv : ad_ctx) bipm_ctx_destroy(kv.second);
    ad_ctx.clear();
    if (opf_prob) bipm_problem_destroy(opf_prob);
    opf_prob = nullptr;
  }
};

ShimState& state() {
  static ShimState s;
  return s;
}

// status code -> the reference's exception (types.hpp:99-109, kkt.hpp:31-36)
[[noreturn]] void rethrow(int code, const char* where) {
  const std::string msg = std::string(where) + ": " + bipm_last_error();
  const index_t block = bipm_last_error_block();
  switch (code) {
    case BIPM_SINGULAR_BLOCK:
      throw SingularBlockError(block);
    case BIPM_NONFINITE:
      throw NonFiniteError(msg, block);
    case BIPM_NON_INTERIOR:
      throw NonInteriorError(msg);
    case BIPM_LINEAR_SOLVE:
    case BIPM_NOT_PD:
      throw LinearSolveError(msg);
    case BIPM_INVALID_ARGUMENT:
      throw DimensionError(msg);
    default:
      throw std::runtime_error(msg);
  }
}

void check(int code, const char* where) {
  if (code != BIPM_OK) rethrow(code, where);
}

bipm_csr csr_of(const SparsityPattern& p) {
  return bipm_csr{p.rows, p.cols, p.row_ptr.data(), p.col_ind.data()};
}

bipm_ctx* kkt_context(const AugmentedSystem& sys) {
  ShimState& S = state();
  const AdPlan& plan = sys.d->plan;
  if (S.kkt_ctx && S.kkt_key == static_cast<const void*>(sys.d)) return S.kkt_ctx;
  S.release_kkt();
  const bipm_csr gx = csr_of(plan.g_split.x_pat), gu = csr_of(plan.g_split.u_pat),
                 hx = csr_of(plan.h_split.x_pat), hu = csr_of(plan.h_split.u_pat),
                 wxx = csr_of(plan.w_split.xx), wxu = csr_of(plan.w_split.xu),
                 wuu = csr_of(plan.w_split.uu);
  check(bipm_problem_create_patterns(sys.nlp->dims.N, &gx, &gu, &hx, &hu, &wxx, &wxu, &wuu,
                                     &S.kkt_prob),
        "bipm_problem_create_patterns");
  check(bipm_ctx_create(S.kkt_prob, S.device, 0, sys.nlp->dims.N, &S.kkt_ctx), "bipm_ctx_create");
  S.kkt_key = sys.d;
  return S.kkt_ctx;
}

bipm_ctx* ad_context(index_t lo, index_t hi) {
  ShimState& S = state();
  auto it = S.ad_ctx.find({lo, hi});
  if (it != S.ad_ctx.end()) return it->second;
  bipm_ctx* c = nullptr;
  check(bipm_ctx_create(S.opf_prob, S.device, lo, hi, &c), "bipm_ctx_create");
  S.ad_ctx[{lo, hi}] = c;
  return c;
}

}  // namespace

namespace bipm_shim {

void enable_kkt(bool on, int device) {
  state().kkt = on;
  state().device = device;
}

void enable_ad(const blockipm::opf::CaseData& cs, const blockipm::opf::ScenarioSet& sc,
               int device) {
  ShimState& S = state();
  S.device = device;
  std::vector<double> bus, gen, branch, gc, coef;
  for (const auto& b : cs.bus)
    bus.insert(bus.end(), {double(b.id), double(b.type), b.Pd, b.Qd, b.Gs, b.Bs, b.Vm, b.Va,
                           b.Vmax, b.Vmin});
  for (const auto& g : cs.gen)
    gen.insert(gen.end(), {double(g.bus), g.Pg, g.Qg, g.Qmax, g.Qmin, g.Vg, double(g.status),
                           g.Pmax, g.Pmin});
  for (const auto& l : cs.branch)
    branch.insert(branch.end(), {double(l.from), double(l.to), l.r, l.x, l.b, l.rateA, l.tap,
                                 l.shift, double(l.status)});
  for (const auto& c : cs.gencost) {
    gc.insert(gc.end(), {double(c.model), c.startup, c.shutdown, double(c.ncost)});
    coef.insert(coef.end(), c.coef.begin(), c.coef.begin() + c.ncost);
  }
  const bipm_case_tables t{cs.name.c_str(),
                           cs.baseMVA,
                           int32_t(cs.bus.size()),
                           int32_t(cs.gen.size()),
                           int32_t(cs.branch.size()),
                           int32_t(cs.gencost.size()),
                           bus.data(),
                           gen.data(),
                           branch.data(),
                           gc.data(),
                           coef.data()};
  std::vector<int32_t> optr{0}, oidx;
  for (const auto& o : sc.outages) {
    oidx.insert(oidx.end(), o.begin(), o.end());
    optr.push_back(int32_t(oidx.size()));
  }
  // ScenarioSet::multipliers is Matrix(nbus, N): column b = scenario b, i.e.
  // the [N][nbus] table the C-ABI takes
  const bipm_scenario_tables st{sc.N, sc.sigma, sc.seed, sc.multipliers.data(), optr.data(),
                                oidx.data()};
  if (S.opf_prob) {
    for (auto& kv : S.ad_ctx) bipm_ctx_destroy(kv.second);
    S.ad_ctx.clear();
    bipm_problem_destroy(S.opf_prob);
    S.opf_prob = nullptr;
  }
  check(bipm_problem_create_tables(&t, &st, &S.opf_prob), "bipm_problem_create_tables");
  S.ad = true;
}

void disable() {
  state().kkt = false;
  state().ad = false;
  state().release();
}

long long kkt_calls() { return state().kkt_calls; }
long long ad_calls() { return state().ad_calls; }

}  // namespace bipm_shim

// ---- the wrappers -----------------------------------------------------------

Step wrap_solve_reduced(AugmentedSystem& sys, const CondenseWork& work, const RegSchedule& reg,
                        double& delta_w_last, index_t n_batch, Executor& exec,
                        const Partition& part, StepInfo* info)
    __asm__("__wrap_" BIPM_SYM_SOLVE_REDUCED);

Step wrap_solve_reduced(AugmentedSystem& sys, const CondenseWork& work, const RegSchedule& reg,
                        double& delta_w_last, index_t n_batch, Executor& exec,
                        const Partition& part, StepInfo* info) {
  ShimState& S = state();
  if (!S.kkt) return real_solve_reduced(sys, work, reg, delta_w_last, n_batch, exec, part, info);
  ++S.kkt_calls;
  const DerivativeBundle& d = *sys.d;
  const BlockDims& dm = sys.nlp->dims;
  bipm_ctx* c = kkt_context(sys);
  const bipm_augmented a{d.gx.data(),      d.gu.data(),      d.hx.data(),     d.hu.data(),
                         d.wxx.data(),     d.wxu.data(),     d.wuu.data(),    sys.sigma_x.data(),
                         sys.r1x.data(),   sys.r3.data(),    sys.sigma_s.data(), sys.r2.data(),
                         sys.r4.data(),    sys.sigma_u.data(), sys.r1u.data()};
  const bipm_reg_schedule rs{reg.delta_w0,   reg.delta_w_min, reg.delta_w_max,
                             reg.kappa_minus, reg.kappa_plus, reg.kappa_plus_emergency};
  Step st;
  st.px = Matrix(dm.n_x, dm.N);
  st.pu.assign(size_t(dm.n_u), 0.0);
  st.ps = Matrix(dm.m, dm.N);
  st.pz = Matrix(dm.m, dm.N);
  st.py = Matrix(dm.n_x, dm.N);
  const bipm_step out{st.px.data(), st.pu.data(), st.ps.data(), st.pz.data(), st.py.data()};
  bipm_step_info si{};
  check(bipm_solve_reduced(c, &a, &rs, &delta_w_last, &out, &si), "bipm_solve_reduced");
  if (info) {
    info->delta_w = si.delta_w;
    info->delta_c = 0;
    info->corrections = si.corrections;
  }
  sys.delta_w = si.delta_w;  // as solve_reduced leaves it (kkt.cpp:1003-1004)
  sys.delta_c = 0;
  return st;
}

void wrap_eval_bundle_range(const BlockNlp& nlp, const AdPlan& plan, AdWorkspace& ws,
                            const Matrix& X, const Vector& u, const Matrix& y, const Matrix& z,
                            double obj_weight, index_t block_begin, DerivativeBundle& out)
    __asm__("__wrap_" BIPM_SYM_EVAL_BUNDLE_RANGE);

void wrap_eval_bundle_range(const BlockNlp& nlp, const AdPlan& plan, AdWorkspace& ws,
                            const Matrix& X, const Vector& u, const Matrix& y, const Matrix& z,
                            double obj_weight, index_t block_begin, DerivativeBundle& out) {
  ShimState& S = state();
  if (!S.ad)
    return real_eval_bundle_range(nlp, plan, ws, X, u, y, z, obj_weight, block_begin, out);
  ++S.ad_calls;
  const index_t M = ws.batch();
  bipm_ctx* c = ad_context(block_begin, block_begin + M);
  // the group's columns are contiguous in the N-wide reference matrices
  // (column-major, one column per scenario) and land in place in `out`
  const size_t b0 = size_t(block_begin);
  auto col = [&](Matrix& m) { return m.data() + b0 * size_t(m.rows()); };
  const bipm_bundle o{out.f.data() + b0, col(out.g),   col(out.h),   col(out.gx),
                      col(out.gu),       col(out.hx),  col(out.hu),  col(out.wxx),
                      col(out.wxu),      col(out.wuu), col(out.grad_lag)};
  out.obj_weight = obj_weight;
  int32_t bad = -1;
  check(bipm_eval_bundle(c, X.col(block_begin), u.data(), y.col(block_begin), z.col(block_begin),
                         obj_weight, &o, &bad),
        "bipm_eval_bundle");
}

void wrap_batch_eval(const BlockNlp& nlp, const Matrix& X, const Vector& u, index_t block_begin,
                     AdWorkspace& ws, Vector& f, Matrix& g, Matrix& h)
    __asm__("__wrap_" BIPM_SYM_BATCH_EVAL);

void wrap_batch_eval(const BlockNlp& nlp, const Matrix& X, const Vector& u, index_t block_begin,
                     AdWorkspace& ws, Vector& f, Matrix& g, Matrix& h) {
  ShimState& S = state();
  if (!S.ad) return real_batch_eval(nlp, X, u, block_begin, ws, f, g, h);
  ++S.ad_calls;
  const index_t M = ws.batch();
  bipm_ctx* c = ad_context(block_begin, block_begin + M);
  f.assign(size_t(M), 0.0);
  g = Matrix(nlp.dims.n_x, M);
  h = Matrix(nlp.dims.m, M);
  int32_t bad = -1;
  check(bipm_eval_values(c, X.data(), u.data(), f.data(), g.data(), h.data(), &bad),
        "bipm_eval_values");
}
