#include <algorithm>
// extern "C" boundary (include/bipm_gpu.h): exceptions become status codes.
#include "../../include/bipm_gpu.h"

#include <cstring>
#include <map>
#include <memory>
#include <string>

#include "engine/engine.hpp"
#include "engine/kkt_step.hpp"
#include "engine/solver.hpp"

using namespace bipm;

struct bipm_problem {
  std::unique_ptr<Problem> p;
  std::map<std::string, std::pair<std::vector<int>, std::vector<double>>> cache;
};

struct bipm_ctx {
  const bipm_problem* prob = nullptr;
  std::unique_ptr<Engine> eng;
  std::unique_ptr<KktStep> kkt;  // operator-level solve_reduced state (created on first use)
  KktStep& step_op() {
    if (!kkt) kkt = std::make_unique<KktStep>(*eng);
    return *kkt;
  }
};

struct bipm_solver {
  bipm_ctx* ctx = nullptr;
  std::unique_ptr<Solver> s;
};

namespace {

thread_local std::string g_err;
thread_local int32_t g_err_block = -1;

template <typename F>
int guarded(F&& f) {
  try {
    g_err_block = -1;
    f();
    return BIPM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_block = e.block;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    const std::string w = e.what();
    if (w.find("cuda") != std::string::npos || w.find("CUDA") != std::string::npos)
      return BIPM_CUDA_ERROR;
    return BIPM_INVALID_ARGUMENT;
  }
}

// Named host arrays exposed read-only for tests and integration shims.
const void* lookup(bipm_problem* bp, const std::string& name, int64_t* count, int32_t* is_int) {
  const Problem& P = *bp->p;
  const OpfModel& M = P.M;
  auto ints = [&](const std::vector<idx>& v) {
    *count = int64_t(v.size());
    *is_int = 1;
    return static_cast<const void*>(v.data());
  };
  auto dbls = [&](const std::vector<double>& v) {
    *count = int64_t(v.size());
    *is_int = 0;
    return static_cast<const void*>(v.data());
  };
  const std::map<std::string, const Csr*> pats = {
      {"L_f", &M.L_f},       {"L_g", &M.L_g},     {"L_h", &M.L_h},         {"gx_p", &P.D.g.x},
      {"gu_p", &P.D.g.u},    {"hx_p", &P.D.h.x},  {"hu_p", &P.D.h.u},      {"wxx_p", &P.D.wxx},
      {"wxu_p", &P.D.wxu},   {"wuu_p", &P.D.wuu}, {"hess_p", &P.D.hess},   {"kxx_p", &P.D.kxx.out},
      {"kxu_p", &P.D.kxu.out}, {"kuu_p", &P.D.kuu.out}};
  for (const auto& [pre, c] : pats) {
    if (name == pre + "_rowptr") return ints(c->ptr);
    if (name == pre + "_colind") return ints(c->ind);
    if (name == pre + "_val") return dbls(c->val);
  }
  const std::map<std::string, const std::vector<double>*> vecs = {
      {"x_lo", &M.x_lo}, {"x_up", &M.x_up}, {"u_lo", &M.u_lo},       {"u_up", &M.u_up},
      {"s_lo", &M.s_lo}, {"s_up", &M.s_up}, {"x_start", &M.x_start}, {"u_start", &M.u_start},
      {"pd", &M.pd},     {"qd", &M.qd},     {"mult", &P.sc.mult}};
  if (auto it = vecs.find(name); it != vecs.end()) return dbls(*it->second);
  const std::map<std::string, const std::vector<idx>*> ivecs = {
      {"lu_perm", &P.LU.perm},       {"lu_fwd_ptr", &P.LU.fwd_ptr}, {"lu_bwd_ptr", &P.LU.bwd_ptr},
      {"lu_l_ptr", &P.LU.l_ptr},     {"lu_l_col", &P.LU.l_col},     {"lu_u_ptr", &P.LU.u_ptr},
      {"lu_u_col", &P.LU.u_col},     {"lu_mul_ptr", &P.LU.mul_ptr},
      {"lu_rf_phase_ptr", &P.LU.rf_phase_ptr}, {"lu_rf_rec", &P.LU.rf_rec},
      {"lu_rf_piv", &P.LU.rf_piv},   {"lu_rf_pair", &P.LU.rf_pair},
      {"lu_u_slot", &P.LU.u_slot},   {"lu_diag", &P.LU.diag}};
  if (auto it = ivecs.find(name); it != ivecs.end()) return ints(*it->second);
  static thread_local std::vector<idx> scalars;
  if (name == "lu_shape") {
    scalars = {P.LU.n, P.LU.nnz_l, P.LU.nnz_f, P.LU.t0, P.LU.tl};
    return ints(scalars);
  }
  const std::map<std::string, const std::vector<idx>*> lu_more = {
      {"lu_ft_src", &P.LU.ft_src},     {"lu_a_src", &P.LU.a_src},
      {"lu_dense_src0", &P.LU.dense_src[0]}, {"lu_dense_src1", &P.LU.dense_src[1]}};
  if (auto it = lu_more.find(name); it != lu_more.end()) return ints(*it->second);
  if (name.rfind("reach_", 0) == 0) {  // presolved forward half (ReachPlan)
    static thread_local ReachPlan R;
    R = build_reach_plan(P.LU, P.D.g.u, P.D.g.u.cols);
    const std::map<std::string, const std::vector<idx>*> rv = {
        {"reach_yn_ptr", &R.yn_ptr}, {"reach_yn_row", &R.yn_row}, {"reach_op_ptr", &R.op_ptr},
        {"reach_ops", &R.ops},       {"reach_ent", &R.ent},
        {"reach_yt_ptr", &R.yt_ptr}, {"reach_yt_row", &R.yt_row}};
    if (auto it = rv.find(name); it != rv.end()) return ints(*it->second);
  }
  const std::map<std::string, const SweepPlan*> sweeps = {
      {"sL", &P.LU.sL}, {"sU", &P.LU.sU}, {"sUt", &P.LU.sUt}, {"sLt", &P.LU.sLt}};
  for (const auto& [pre, sw] : sweeps) {
    if (name == "lu_" + pre + "_ptr") return ints(sw->ptr);
    if (name == "lu_" + pre + "_col") return ints(sw->col);
    if (name == "lu_" + pre + "_lvl_ptr") return ints(sw->lvl_ptr);
    if (name == "lu_" + pre + "_items") return ints(sw->items);
    if (name == "lu_" + pre + "_tail_items") return ints(sw->tail_items);
  }
  throw Error(kInvalidArgument, "unknown problem array '" + name + "'");
}

}  // namespace

namespace {
void upload_condensed(Engine& e, const bipm_condensed* in);
}

extern "C" {

const char* bipm_last_error(void) { return g_err.c_str(); }
int32_t bipm_last_error_block(void) { return g_err_block; }
int bipm_version(void) { return 1; }

int bipm_problem_create(const char* case_path, int32_t N, double sigma, uint64_t seed,
                        bipm_problem** out) {
  return guarded([&] {
    if (!case_path || !out) throw Error(kInvalidArgument, "null argument");
    auto bp = std::make_unique<bipm_problem>();
    bp->p = Problem::from_case_file(case_path, N, sigma, seed);
    *out = bp.release();
  });
}

int bipm_problem_create_ex(const char* case_path, int32_t N, double sigma, uint64_t seed,
                           const int32_t* contingencies, int32_t n_contingencies,
                           bipm_problem** out) {
  return guarded([&] {
    if (!case_path || !out || n_contingencies < 0 || (n_contingencies > 0 && !contingencies))
      throw Error(kInvalidArgument, "null argument");
    auto bp = std::make_unique<bipm_problem>();
    bp->p = Problem::from_case_file(
        case_path, N, sigma, seed,
        std::vector<idx>(contingencies, contingencies + n_contingencies));
    *out = bp.release();
  });
}

int bipm_problem_create_tables(const bipm_case_tables* t, const bipm_scenario_tables* sc,
                               bipm_problem** out) {
  return guarded([&] {
    if (!t || !sc || !out) throw Error(kInvalidArgument, "null argument");
    if (t->nbus < 1 || t->ngen < 1 || t->nbranch < 1 || !t->bus || !t->gen || !t->branch)
      throw Error(kInvalidArgument, "case tables: need buses, generators and branches");
    GridCase cs;
    cs.name = t->name ? t->name : "tables";
    cs.baseMVA = t->base_mva;
    for (int32_t i = 0; i < t->nbus; ++i) {
      const double* r = t->bus + size_t(i) * BIPM_BUS_COLS;
      CaseBus b;
      b.id = int(r[0]);
      b.type = int(r[1]);
      b.Pd = r[2], b.Qd = r[3], b.Gs = r[4], b.Bs = r[5], b.Vm = r[6], b.Va = r[7];
      b.Vmax = r[8], b.Vmin = r[9];
      cs.bus.push_back(b);
    }
    for (int32_t i = 0; i < t->ngen; ++i) {
      const double* r = t->gen + size_t(i) * BIPM_GEN_COLS;
      CaseGen g;
      g.bus = int(r[0]);
      g.Pg = r[1], g.Qg = r[2], g.Qmax = r[3], g.Qmin = r[4], g.Vg = r[5];
      g.status = int(r[6]);
      g.Pmax = r[7], g.Pmin = r[8];
      cs.gen.push_back(g);
    }
    for (int32_t i = 0; i < t->nbranch; ++i) {
      const double* r = t->branch + size_t(i) * BIPM_BRANCH_COLS;
      CaseBranch l;
      l.from = int(r[0]);
      l.to = int(r[1]);
      l.r = r[2], l.x = r[3], l.b = r[4], l.rateA = r[5], l.tap = r[6], l.shift = r[7];
      l.status = int(r[8]);
      cs.branch.push_back(l);
    }
    if (t->ngencost > 0) {
      if (!t->gencost || !t->gencost_coef || t->ngencost != t->ngen)
        throw Error(kInvalidArgument, "case tables: one gencost row per generator");
      size_t off = 0;
      for (int32_t i = 0; i < t->ngencost; ++i) {
        const double* r = t->gencost + size_t(i) * BIPM_GENCOST_COLS;
        CaseCost c;
        c.model = int(r[0]);
        c.ncost = int(r[3]);
        if (c.model != 2 || c.ncost < 0 || c.ncost > 3)
          throw Error(kInvalidArgument, "case tables: polynomial costs of degree <= 2 only");
        c.coef.assign(t->gencost_coef + off, t->gencost_coef + off + c.ncost);
        off += size_t(c.ncost);
        cs.cost.push_back(c);
      }
    }
    (void)cs.ref_bus();  // exactly one reference bus (throws otherwise)
    if (sc->N < 1 || !sc->multipliers) throw Error(kInvalidArgument, "scenarios: need N >= 1");
    ScenarioDraw d;
    d.N = sc->N;
    d.sigma = sc->sigma;
    d.seed = sc->seed;
    d.mult.assign(sc->multipliers, sc->multipliers + size_t(sc->N) * size_t(t->nbus));
    d.outages.assign(size_t(sc->N), {});
    if (sc->outage_ptr) {
      for (int32_t s = 0; s < sc->N; ++s)
        for (int32_t k = sc->outage_ptr[s]; k < sc->outage_ptr[s + 1]; ++k) {
          const int32_t l = sc->outage_branch[k];
          if (l < 0 || l >= t->nbranch || !cs.branch[size_t(l)].status)
            throw Error(kInvalidArgument, "scenario outage names an unknown or out-of-service branch");
          d.outages[size_t(s)].push_back(l);
        }
    }
    auto bp = std::make_unique<bipm_problem>();
    bp->p = Problem::from_parts(std::move(cs), std::move(d));
    *out = bp.release();
  });
}

int bipm_problem_create_patterns(int32_t N, const bipm_csr* gx, const bipm_csr* gu,
                                 const bipm_csr* hx, const bipm_csr* hu, const bipm_csr* wxx,
                                 const bipm_csr* wxu, const bipm_csr* wuu, bipm_problem** out) {
  return guarded([&] {
    if (!gx || !gu || !hx || !hu || !wxx || !wxu || !wuu || !out)
      throw Error(kInvalidArgument, "null argument");
    auto csr = [](const bipm_csr* c) {
      if (c->rows < 0 || c->cols < 0 || !c->row_ptr)
        throw Error(kInvalidArgument, "pattern: bad shape");
      Csr r;
      r.rows = c->rows;
      r.cols = c->cols;
      r.ptr.assign(c->row_ptr, c->row_ptr + c->rows + 1);
      if (r.ptr.back() > 0 && !c->col_ind) throw Error(kInvalidArgument, "pattern: null col_ind");
      r.ind.assign(c->col_ind, c->col_ind + r.ptr.back());
      return r;
    };
    auto bp = std::make_unique<bipm_problem>();
    bp->p = Problem::from_patterns(N, csr(gx), csr(gu), csr(hx), csr(hu), csr(wxx), csr(wxu),
                                   csr(wuu));
    *out = bp.release();
  });
}

void bipm_problem_destroy(bipm_problem* p) { delete p; }

int bipm_problem_dims(const bipm_problem* bp, int32_t d[10]) {
  return guarded([&] {
    const Problem& P = *bp->p;
    const OpfModel& M = P.M;
    const int32_t v[10] = {M.N,  M.n_x, M.n_u, M.m, M.n_b(), M.nbus, M.nbr, M.ngen, P.LU.nnz_f,
                           int32_t(P.LU.fwd_ptr.size()) - 1};
    std::memcpy(d, v, sizeof v);
  });
}

int bipm_problem_array(const bipm_problem* bp, const char* name, const void** data,
                       int64_t* count, int32_t* is_int) {
  return guarded([&] {
    *data = lookup(const_cast<bipm_problem*>(bp), name, count, is_int);
  });
}

int bipm_ctx_create(const bipm_problem* bp, int32_t device, int32_t lo, int32_t hi,
                    bipm_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<bipm_ctx>();
    c->prob = bp;
    c->eng = std::make_unique<Engine>(*bp->p, device, lo, hi);
    *out = c.release();
  });
}

void bipm_ctx_destroy(bipm_ctx* c) { delete c; }

int bipm_factor_gx(bipm_ctx* c, const double* gx, int32_t* singular_block) {
  return guarded([&] {
    Engine& e = *c->eng;
    e.bd().gx.copy_from(gx, e.bd().gx.size(), e.st);
    const idx bad = e.factor_gx();
    if (singular_block) *singular_block = bad;
    if (bad >= 0) throw Error(kSingularBlock, "singular block " + std::to_string(bad), bad);
  });
}

int bipm_reduce(bipm_ctx* c, const bipm_condensed* in, double delta_w, double* khat,
                double* rhs) {
  return guarded([&] {
    Engine& e = *c->eng;
    upload_condensed(e, in);
    e.reduce_local(delta_w);
    e.finish_reduce(delta_w);
    e.reduce_rhs_local(delta_w, e.rhs.get());
    // rhs = sum_b (...) - rhat2
    std::vector<double> r(e.rhs.size()), r2(e.rhat2.size());
    e.rhs.download(r.data(), r.size(), e.st);
    e.khat.download(khat, e.khat.size(), e.st);
    e.sync();
    for (size_t i = 0; i < r.size(); ++i) rhs[i] = r[i] - in->rhat2[i];
  });
}

}  // extern "C"

namespace {

void upload_condensed(Engine& e, const bipm_condensed* in) {
  if (!in || !in->gu || !in->kxx || !in->kxu || !in->kuu || !in->sigma_x || !in->rhat1 ||
      !in->rhat3 || !in->sigma_u || !in->rhat2)
    throw Error(kInvalidArgument, "condensed system: null array");
  const size_t Ms = size_t(e.M), nx = Ms * size_t(e.pb.M.n_x);
  const DerivPlan& D = e.pb.D;
  e.invalidate_reach();  // G_u changes: the reach solve of the last factor is stale
  e.bd().gu.copy_from(in->gu, Ms * size_t(D.g.u.nnz()), e.st);
  e.kxx.copy_from(in->kxx, Ms * size_t(D.kxx.out.nnz()), e.st);
  e.kxu.copy_from(in->kxu, Ms * size_t(D.kxu.out.nnz()), e.st);
  e.kuu.copy_from(in->kuu, Ms * size_t(D.kuu.out.nnz()), e.st);
  e.sigma_x.copy_from(in->sigma_x, nx, e.st);
  e.rhat1.copy_from(in->rhat1, nx, e.st);
  e.rhat3.copy_from(in->rhat3, nx, e.st);
  e.sigma_u.copy_from(in->sigma_u, size_t(e.pb.M.n_u), e.st);
  e.rhat2.copy_from(in->rhat2, size_t(e.pb.M.n_u), e.st);
}

// the augmented system (and the bundle blocks it references) into the engine
// and the KKT step; NonInterior when a Sigma_s entry is not positive, as
// condense does (kkt.cpp:138-141)
void upload_augmented(Engine& e, KktStep& k, const bipm_augmented* a) {
  if (!a || !a->gx || !a->gu || !a->hx || !a->hu || !a->wxx || !a->wxu || !a->wuu ||
      !a->sigma_x || !a->r1x || !a->r3 || !a->sigma_s || !a->r2 || !a->r4 || !a->sigma_u ||
      !a->r1u)
    throw Error(kInvalidArgument, "augmented system: null array");
  const size_t nm = size_t(e.M) * size_t(e.pb.M.m);
  for (size_t i = 0; i < nm; ++i)
    if (!(a->sigma_s[i] > 0))
      throw Error(kNonInterior, "condense: Sigma_s not positive (zero slack gap)",
                  e.lo + idx(i / size_t(std::max(1, e.pb.M.m))));
  Engine::Bundle& b = e.bd();
  const size_t nx = size_t(e.M) * size_t(e.pb.M.n_x);
  e.invalidate_reach();
  b.gx.copy_from(a->gx, b.gx.size(), e.st);
  b.gu.copy_from(a->gu, b.gu.size(), e.st);
  b.hx.copy_from(a->hx, b.hx.size(), e.st);
  b.hu.copy_from(a->hu, b.hu.size(), e.st);
  b.wxx.copy_from(a->wxx, b.wxx.size(), e.st);
  b.wxu.copy_from(a->wxu, b.wxu.size(), e.st);
  b.wuu.copy_from(a->wuu, b.wuu.size(), e.st);
  b.g.copy_from(a->r3, b.g.size(), e.st);
  e.sigma_x.copy_from(a->sigma_x, nx, e.st);
  e.sigma_s.copy_from(a->sigma_s, nm, e.st);
  e.r2.copy_from(a->r2, nm, e.st);
  e.r4.copy_from(a->r4, nm, e.st);
  e.sigma_u.copy_from(a->sigma_u, size_t(e.pb.M.n_u), e.st);
  k.r1x.copy_from(a->r1x, nx, e.st);
  k.r1u.copy_from(a->r1u, size_t(e.pb.M.n_u), e.st);
}

}  // namespace

extern "C" {

int bipm_condense(bipm_ctx* c, const bipm_augmented* a, const bipm_condensed_out* out) {
  return guarded([&] {
    Engine& e = *c->eng;
    KktStep& k = c->step_op();
    upload_augmented(e, k, a);
    k.condense();
    if (out) {
      auto dl = [&](const DArr<double>& v, double* dst, size_t n) {
        if (dst) v.download(dst, n, e.st);
      };
      dl(e.kxx, out->kxx, size_t(e.M) * size_t(e.pb.D.kxx.out.nnz()));
      dl(e.kxu, out->kxu, e.kxu.size());
      dl(e.kuu, out->kuu, e.kuu.size());
      dl(e.rhat1, out->rhat1, e.rhat1.size());
      dl(e.rhat2, out->rhat2, e.rhat2.size());
      dl(e.rhat3, out->rhat3, e.rhat3.size());
    }
    e.sync();
  });
}

int bipm_reduce_rhs(bipm_ctx* c, const bipm_condensed* in, double delta_w, double* rhs) {
  return guarded([&] {
    Engine& e = *c->eng;
    if (!rhs) throw Error(kInvalidArgument, "null argument");
    upload_condensed(e, in);
    e.reduce_rhs_local(delta_w, e.rhs.get());
    e.rhs.download(rhs, e.rhs.size(), e.st);
    e.sync();
  });
}

int bipm_recover(bipm_ctx* c, const bipm_condensed* in, const bipm_slack_rows* sr,
                 double delta_w, const double* pu, double* px, double* py, double* pz,
                 double* ps) {
  return guarded([&] {
    Engine& e = *c->eng;
    if (!sr || !sr->hx || !sr->hu || !sr->sigma_s || !sr->r2 || !sr->r4 || !pu || !px || !py ||
        !pz || !ps)
      throw Error(kInvalidArgument, "null argument");
    upload_condensed(e, in);
    e.bd().hx.copy_from(sr->hx, e.bd().hx.size(), e.st);
    e.bd().hu.copy_from(sr->hu, e.bd().hu.size(), e.st);
    e.sigma_s.copy_from(sr->sigma_s, e.sigma_s.size(), e.st);
    e.r2.copy_from(sr->r2, e.r2.size(), e.st);
    e.r4.copy_from(sr->r4, e.r4.size(), e.st);
    const OpfModel& M = e.pb.M;
    const size_t nx = size_t(e.M) * M.n_x, nm = size_t(e.M) * M.m;
    DArr<double> dpu, dpx(nx), dpy(nx), dpz(nm), dps(nm);
    dpu.upload(pu, size_t(M.n_u), e.st);
    e.recover(delta_w, dpu.get(), dpx.get(), dpy.get(), dpz.get(), dps.get());
    dpx.download(px, nx, e.st);
    dpy.download(py, nx, e.st);
    dpz.download(pz, nm, e.st);
    dps.download(ps, nm, e.st);
    e.sync();
  });
}

int bipm_solve_reduced(bipm_ctx* c, const bipm_augmented* a, const bipm_reg_schedule* reg,
                       double* delta_w_last, const bipm_step* out, bipm_step_info* info) {
  return guarded([&] {
    Engine& e = *c->eng;
    if (!delta_w_last || !out) throw Error(kInvalidArgument, "null argument");
    KktStep& k = c->step_op();
    RegOptions r;
    if (reg) {
      if (reg->delta_w0 > 0) r.delta_w0 = reg->delta_w0;
      if (reg->delta_w_min > 0) r.delta_w_min = reg->delta_w_min;
      if (reg->delta_w_max > 0) r.delta_w_max = reg->delta_w_max;
      if (reg->kappa_minus > 0) r.kappa_minus = reg->kappa_minus;
      if (reg->kappa_plus > 0) r.kappa_plus = reg->kappa_plus;
      if (reg->kappa_plus_emergency > 0) r.kappa_plus_emergency = reg->kappa_plus_emergency;
    }
    upload_augmented(e, k, a);
    k.condense();
    k.factor_launch();
    k.check_factor(nullptr);
    k.solve(*delta_w_last, r);
    double* dst[5] = {out->px, out->pu, out->ps, out->pz, out->py};
    for (int j = 0; j < 5; ++j)
      if (dst[j]) k.p[j].download(dst[j], k.p[j].size(), e.st);
    e.sync();
    if (info) {
      info->delta_w = k.last_dw;
      info->corrections = k.corrections;
      info->refinements = k.refinements;
      info->reductions = k.reductions;
    }
  });
}

int bipm_eval_bundle(bipm_ctx* c, const double* X, const double* u, const double* y,
                     const double* z, double obj_weight, const bipm_bundle* out,
                     int32_t* bad_block) {
  return guarded([&] {
    Engine& e = *c->eng;
    const OpfModel& M = e.pb.M;
    const size_t Ms = size_t(e.M);
    DArr<double> dX, du, dY, dZ;
    dX.upload(X, Ms * M.n_x, e.st);
    du.upload(u, size_t(M.n_u), e.st);
    dY.upload(y, Ms * M.n_x, e.st);
    dZ.upload(z, Ms * M.m, e.st);
    Engine::Bundle& b = e.bd();
    const idx badb = e.eval_bundle(b, dX.get(), du.get(), dY.get(), dZ.get(), obj_weight);
    if (bad_block) *bad_block = badb;
    auto dl = [&](const DArr<double>& a, double* dst) {
      if (dst) a.download(dst, a.size(), e.st);
    };
    dl(b.f, out->f);
    dl(b.g, out->g);
    dl(b.h, out->h);
    dl(b.gx, out->gx);
    dl(b.gu, out->gu);
    dl(b.hx, out->hx);
    dl(b.hu, out->hu);
    dl(b.wxx, out->wxx);
    dl(b.wxu, out->wxu);
    dl(b.wuu, out->wuu);
    dl(b.grad, out->grad_lag);
    e.sync();
    if (badb >= 0) throw Error(kNonFinite, "non-finite basis output (block " + std::to_string(badb) + ")", badb);
  });
}

int bipm_eval_values(bipm_ctx* c, const double* X, const double* u, double* f, double* g,
                     double* h, int32_t* bad_block) {
  return guarded([&] {
    Engine& e = *c->eng;
    const OpfModel& M = e.pb.M;
    const size_t Ms = size_t(e.M);
    DArr<double> dX, du, df(Ms), dg(Ms * M.n_x), dh(Ms * M.m);
    dX.upload(X, Ms * M.n_x, e.st);
    du.upload(u, size_t(M.n_u), e.st);
    const idx badb = e.eval_values(dX.get(), du.get(), df.get(), dg.get(), dh.get());
    if (bad_block) *bad_block = badb;
    df.download(f, df.size(), e.st);
    dg.download(g, dg.size(), e.st);
    dh.download(h, dh.size(), e.st);
    e.sync();
    if (badb >= 0) throw Error(kNonFinite, "non-finite basis output (block " + std::to_string(badb) + ")", badb);
  });
}

namespace {
SolverOptions to_options(const bipm_solve_options* o) {
  SolverOptions so;
  if (o) {
    if (o->tol > 0) so.tol = o->tol;
    if (o->mu0 > 0) so.mu0 = o->mu0;
    if (o->max_iter > 0) so.max_iter = o->max_iter;
  }
  return so;
}
void fill_result(Solver& s, bipm_solve_result* r, double* u) {
  if (r) {
    r->status = s.status;
    r->iterations = int32_t(s.logs.size());
    r->objective = s.logs.empty() ? 0.0 : s.logs.back().objective;
    r->t_total = s.t_total;
    r->t_ad = s.t_ad;
    r->t_kkt = s.t_kkt;
    r->reductions = s.reductions;
  }
  if (u) {
    const auto h = s.host_u();
    std::copy(h.begin(), h.end(), u);
  }
}
}  // namespace

int bipm_solver_create(bipm_ctx* c, const bipm_solve_options* opts, bipm_solver** out) {
  return guarded([&] {
    auto sv = std::make_unique<bipm_solver>();
    sv->ctx = c;
    sv->s = std::make_unique<Solver>(*c->eng, to_options(opts));
    *out = sv.release();
  });
}

void bipm_solver_destroy(bipm_solver* s) { delete s; }

int bipm_solver_start(bipm_solver* s) {
  return guarded([&] { s->s->start(); });
}

int bipm_solver_step(bipm_solver* s, int32_t* status) {
  return guarded([&] {
    const int st = s->s->step();
    if (status) *status = st;
  });
}

int bipm_solver_result(bipm_solver* s, bipm_solve_result* r, double* u) {
  return guarded([&] { fill_result(*s->s, r, u); });
}

int bipm_solver_iterate(bipm_solver* s, const bipm_iterate* out) {
  return guarded([&] {
    if (!out) throw Error(kInvalidArgument, "null argument");
    double* const dst[11] = {out->x,        out->u,        out->s,     out->y,
                             out->z,        out->kappa_lo, out->kappa_up, out->nu_lo,
                             out->nu_up,    out->lambda_lo, out->lambda_up};
    s->s->host_iterate(dst);
  });
}

int bipm_solver_log(bipm_solver* s, int32_t k, double rec[15]) {
  return guarded([&] {
    const auto& L = s->s->logs;
    if (k < 0 || size_t(k) >= L.size()) throw Error(kInvalidArgument, "log index out of range");
    const IterRecord& l = L[size_t(k)];
    const double v[15] = {double(l.iter), l.objective,    l.inf_pr,         l.inf_du,
                          l.complementarity, l.mu,         l.alpha_primal,   l.alpha_dual,
                          l.t_ad,            l.t_kkt,      l.t_total,        double(l.corrections),
                          double(l.refinements), l.delta_w, l.full_step ? 1.0 : 0.0};
    std::copy(v, v + 15, rec);
  });
}

int bipm_solver_step_timed(bipm_solver* s, int32_t* status, double* device_ms) {
  return guarded([&] {
    int st = 0;
    const double ms = s->s->step_timed(&st);
    if (status) *status = st;
    if (device_ms) *device_ms = ms;
  });
}

int bipm_counters(int64_t out[3]) {
  return guarded([&] {
    out[0] = stats().launches.load();
    out[1] = stats().h2d_bytes.load();
    out[2] = stats().d2h_bytes.load();
  });
}

int bipm_ctx_profile(bipm_ctx* c, int32_t enable) {
  return guarded([&] {
    c->eng->resolve_timers();
    if (enable && !c->eng->profiling) c->eng->ktimers.clear();  // a new profiling window
    c->eng->profiling = enable != 0;
  });
}

int bipm_ctx_kernel_time(bipm_ctx* c, const char* name, double* ms, int64_t* count) {
  return guarded([&] {
    c->eng->resolve_timers();
    auto it = c->eng->ktimers.find(name);
    *ms = it == c->eng->ktimers.end() ? 0.0 : it->second.ms;
    *count = it == c->eng->ktimers.end() ? 0 : it->second.n;
  });
}

int bipm_ctx_phase_stamps(bipm_ctx* c, int32_t enable, int64_t out[16]) {
  return guarded([&] {
    Engine& e = *c->eng;
    if (out && e.phase.size()) {  // stamps of the previous reduction
      e.phase.download(reinterpret_cast<long long*>(out), 16, e.st);
      e.sync();
    }
    if (enable) {
      if (!e.phase.size()) e.phase.resize(16);
      e.phase.zero(e.st);
    } else {
      e.phase.resize(0);
    }
  });
}

int bipm_ctx_step_stamps(bipm_ctx* c, int32_t enable, int64_t* out, int32_t cap,
                         int32_t* n_out) {
  return guarded([&] {
    Engine& e = *c->eng;
    const int P = e.use_stream ? e.sprog.steps : 0;
    if (n_out) *n_out = 0;
    if (out && e.phase.size() && P > 0) {
      // (kind, clock64 before the data wait, clock64 after it) per step, then the end stamp
      std::vector<long long> st(e.phase.size());
      e.phase.download(st.data(), st.size(), e.st);
      e.sync();
      const int n = std::min<int>(cap / 3, P + 1);
      for (int j = 0; j < n; ++j) {
        out[3 * j] = j < P ? e.sprog.pat[size_t(e.sprog.issue[size_t(j)].pat_off)] : -1;
        out[3 * j + 1] = st[size_t(2 * j)];
        out[3 * j + 2] = j < P ? st[size_t(2 * j + 1)] : st[size_t(2 * j)];
      }
      if (n_out) *n_out = n;
    }
    if (enable) {
      e.phase.resize(size_t(std::max(16, 2 * P + 2 + 60000)));
      e.phase.zero(e.st);
    } else {
      e.phase.resize(0);
    }
  });
}

int bipm_problem_stream_check(const bipm_problem* bp, int32_t K, int32_t consumers,
                              int32_t ring_bytes, int64_t out[10]) {
  return bipm_problem_stream_check_ex(bp, K, consumers, ring_bytes, 0, out);
}

int bipm_problem_stream_check_ex(const bipm_problem* bp, int32_t K, int32_t consumers,
                                 int32_t ring_bytes, int32_t mode, int64_t out[10]) {
  return guarded([&] {
    const Problem& P = *bp->p;
    const LuPlan& L = P.LU;
    const bool presolved = (mode & 1) != 0, identity = presolved && (mode & 2) != 0;
    const ReachPlan R = build_reach_plan(L, P.D.g.u, P.M.n_u);
    const StreamProgram S = build_stream_program(
        L, P.D.g.u, P.D.kxx.out, P.D.kxu.out, P.M.n_u, K, consumers, ring_bytes,
        kStreamLookahead, presolved ? &R : nullptr, identity, (mode & 4) != 0);
    int64_t bad = 0;
    // (1) every factor entry a sweep reads appears in VS, once per sweep: each
    // L slot twice (L, L'), each U slot twice (U, U'), less the entries the
    // dense tail covers (both row and column in the tail).  The presolved
    // program has no L sweep (the reach solve reads L), the adjoint identity
    // no L' sweep
    std::vector<int> seen(size_t(L.nnz_f), 0);
    for (idx v : S.vs_src) {
      if (v < -1 || v >= L.nnz_f) ++bad;
      if (v >= 0) ++seen[size_t(v)];
    }
    const int l_sweeps = 2 - (presolved ? 1 : 0) - (identity ? 1 : 0);
    auto row_of_l = [&](idx t) { return idx(std::upper_bound(L.l_ptr.begin(), L.l_ptr.end(), t) - L.l_ptr.begin()) - 1; };
    for (idx t = 0; t < L.nnz_l; ++t) {
      const bool in_tail = row_of_l(t) >= L.t0 && L.l_col[size_t(t)] >= L.t0;
      if (seen[size_t(t)] != (in_tail ? 0 : l_sweeps)) ++bad;
    }
    for (idx i = 0; i < L.n; ++i) {
      const int want = i >= L.t0 ? 0 : 2;  // U rows of the tail live in W
      if (seen[size_t(L.diag[size_t(i)])] != want) ++bad;
      for (idx q = L.u_ptr[size_t(i)]; q < L.u_ptr[size_t(i) + 1]; ++q)
        if (seen[size_t(L.u_slot[size_t(q)])] != want) ++bad;
    }
    // (2) ring placement: a step's region never overlaps a step the producer
    // may still be ahead of (within its wait distance), cyclically
    const int n = S.steps;
    auto size_of = [&](const StepIssue& is) {
      auto va = [](int c) { return c > 0 ? ((c + 1) * 8 + 15) & ~15 : 0; };
      return is.pat_bytes + va(is.val_count) + va(is.x_count);
    };
    for (int j = 0; j < n; ++j) {
      const StepIssue& a = S.issue[size_t(j)];
      if (a.ring_off < 0 || a.ring_off + size_of(a) > ring_bytes) ++bad;
      for (int d = 1; d < a.wait_delta; ++d) {
        const StepIssue& b = S.issue[size_t(((j - d) % n + n) % n)];
        if (a.ring_off < b.ring_off + size_of(b) && b.ring_off < a.ring_off + size_of(a)) ++bad;
      }
    }
    out[0] = bad;
    out[1] = S.steps;
    out[2] = S.nnz_vs;
    out[3] = S.n_sweep_steps;
    out[4] = S.n_dense_steps;
    out[5] = S.n_acc_steps;
    out[6] = S.n_spmv_steps;
    out[7] = S.nq;
    out[8] = L.t0;
    out[9] = L.tl;
  });
}

int bipm_ctx_debug_buffer(bipm_ctx* c, int64_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&] {
    Engine& e = *c->eng;
    const size_t n = std::min<size_t>(size_t(cap), e.phase.size());
    if (n) e.phase.download(reinterpret_cast<long long*>(out), n, e.st);
    e.sync();
    *n_out = int64_t(n);
  });
}

int bipm_ctx_info(bipm_ctx* c, int64_t out[12]) {
  return guarded([&] {
    const Engine& e = *c->eng;
    out[0] = e.use_stream ? e.sl.K : e.red.kc;
    out[1] = e.use_stream ? e.sl.chunk : e.red.chunk;
    out[2] = e.use_stream ? e.sl.nchunks : e.red.nchunks;
    out[3] = e.use_stream ? 1 : (e.red.panel_in_smem ? 1 : 0);
    out[4] = e.pb.LU.nnz_l;
    out[5] = e.pb.LU.nnz_f;
    out[6] = (int64_t)e.pb.LU.mul_l.size();
    out[7] = e.sm_count;
    out[8] = e.use_stream ? 1 | (e.presolve ? 2 : 0) | (e.adj_identity ? 4 : 0) : 0;
    out[9] = e.use_stream ? e.sprog.steps : 0;
    out[10] = e.use_stream ? e.sl.ring_bytes : 0;
    out[11] = e.use_stream ? e.sprog.nnz_vs : 0;
  });
}

namespace {
// BK factor (+ inertia) of the shifted K; solves rhs when the factor is
// nonsingular.  inertia = {pos, neg, zero}
void bk_factor_solve(int32_t n, const double* k_colmajor, double* rhs, int32_t inertia[3],
                     cudaStream_t st) {
  DArr<double> K, b;
  DArr<int> ipiv{size_t(n)}, in{size_t(4)};
  DArr<unsigned char> state{bk_work_bytes(n)};
  K.upload(k_colmajor, size_t(n) * n, st);
  launch_bk_factor(K.get(), n, ipiv.get(), state.get(), in.get(), st);
  in.download(inertia, 3, st);
  cuda_check(cudaStreamSynchronize(st), "sync");
  if (rhs && inertia[2] == 0) {
    b.upload(rhs, size_t(n), st);
    launch_bk_solve(K.get(), n, ipiv.get(), b.get(), st);
    b.download(rhs, size_t(n), st);
    cuda_check(cudaStreamSynchronize(st), "sync");
  }
}
}  // namespace

int bipm_dense_factor_solve(int32_t n, const double* k_colmajor, double* rhs, int32_t* pd) {
  return guarded([&] {
    if (n < 1 || !k_colmajor || !pd) throw Error(kInvalidArgument, "null argument");
    cudaStream_t st;
    cuda_check(cudaStreamCreate(&st), "stream");
    DArr<double> K, b;
    DArr<int> info(8);
    K.upload(k_colmajor, size_t(n) * n, st);
    launch_shift_cholesky(K.get(), n, info.get(), nullptr, st);
    int inf[8] = {0};
    info.download(inf, 6, st);
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (inf[0] == 0) {
      *pd = 1;
      if (rhs) {
        b.upload(rhs, size_t(n), st);
        launch_cholesky_solve(K.get(), n, b.get(), st);
        b.download(rhs, size_t(n), st);
        cuda_check(cudaStreamSynchronize(st), "sync");
      }
    } else {
      // the same borderline rule as the engine (Engine::factor_khat)
      double kinf = 0.0, piv = 0.0;
      std::memcpy(&kinf, inf + 2, sizeof(double));
      std::memcpy(&piv, inf + 4, sizeof(double));
      const double tol = 4.0 * n * 2.220446049250313e-16 * std::max(1.0, kinf);
      *pd = 0;
      if (piv > -tol) {
        int32_t in3[3];
        std::vector<double> x(rhs ? rhs : k_colmajor, rhs ? rhs + n : k_colmajor);
        bk_factor_solve(n, k_colmajor, rhs ? x.data() : nullptr, in3, st);
        if (in3[1] == 0 && in3[2] == 0) {
          *pd = 1;
          if (rhs) std::copy(x.begin(), x.end(), rhs);
        }
      }
    }
    cudaStreamDestroy(st);
  });
}

int bipm_dense_inertia(int32_t n, const double* k_colmajor, double* rhs, int32_t inertia[3]) {
  return guarded([&] {
    if (n < 1 || !k_colmajor || !inertia) throw Error(kInvalidArgument, "null argument");
    cudaStream_t st;
    cuda_check(cudaStreamCreate(&st), "stream");
    bk_factor_solve(n, k_colmajor, rhs, inertia, st);
    cudaStreamDestroy(st);
  });
}

int bipm_ctx_factor_stats(bipm_ctx* c, int64_t out[2]) {
  return guarded([&] {
    out[0] = c->eng->bk_fallbacks;
    out[1] = c->eng->khat_bk ? 1 : 0;
  });
}

int bipm_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] { nccl_unique_id(out); });
}

int bipm_ctx_set_nccl(bipm_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank) {
  return guarded([&] { c->eng->comm = make_nccl_comm(id, nranks, rank, c->eng->device); });
}

int bipm_ctx_set_host_comm(bipm_ctx* c, bipm_allreduce_fn fn, void* user, int32_t nranks,
                           int32_t rank) {
  return guarded([&] {
    if (!fn) throw Error(kInvalidArgument, "null all-reduce callback");
    c->eng->comm = make_host_comm(fn, user, nranks, rank);
  });
}

int bipm_ctx_comm(const bipm_ctx* c, int32_t out[3]) {
  return guarded([&] {
    const Engine& e = *c->eng;
    out[0] = e.comm ? e.comm->kind() : 0;
    out[1] = e.comm ? e.comm->size() : 1;
    out[2] = e.comm ? e.comm->rank() : 0;
  });
}

int bipm_partition(int32_t N, int32_t G, int32_t* ranges) {
  return guarded([&] {
    if (G < 1 || G > N) throw Error(kInvalidArgument, "partition: need 1 <= G <= N");
    const int32_t base = N / G, rem = N % G;
    int32_t lo = 0;
    for (int32_t g = 0; g < G; ++g) {
      const int32_t sz = base + (g < rem ? 1 : 0);
      ranges[2 * g] = lo;
      ranges[2 * g + 1] = lo + sz;
      lo += sz;
    }
  });
}

int bipm_solve(bipm_ctx* c, const bipm_solve_options* opts, bipm_solve_result* r, double* u) {
  return guarded([&] {
    Solver s(*c->eng, to_options(opts));
    s.solve();
    fill_result(s, r, u);
  });
}

}  // extern "C"
