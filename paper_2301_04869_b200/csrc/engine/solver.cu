#include "solver.hpp"

#include <algorithm>
#include <cmath>

namespace bipm {

namespace {

double project_start(double start, double lo, double up) {  // ipm.cpp:28-36
  if (std::isfinite(lo) && std::isfinite(up)) {
    const double span = up - lo;
    return std::max(lo + 0.1 * span, std::min(up - 0.1 * span, start));
  }
  if (std::isfinite(lo)) return std::max(start, lo + 0.1 * std::max(1.0, std::abs(lo)));
  if (std::isfinite(up)) return std::min(start, up - 0.1 * std::max(1.0, std::abs(up)));
  return start;
}

double update_mu(double mu, const SolverOptions& o) {  // ipm.cpp:21-24
  return std::max(o.tol / 10.0, std::min(o.kappa_mu * mu, std::pow(mu, o.theta_mu)));
}

}  // namespace

DevIter Solver::IterStore::view() {
  return DevIter{x.get(),   u.get(),   s.get(),   y.get(),   z.get(),  klo.get(),
                 kup.get(), nlo.get(), nup.get(), llo.get(), lup.get()};
}

Solver::Solver(Engine& eng, const SolverOptions& opt)
    : e(eng), o(opt), io(eng), kkt(eng, opt.refine_rounds) {
  const OpfModel& M = e.pb.M;
  if (!e.pb.has_model())
    throw Error(kInvalidArgument,
                "the interior-point driver needs the OPF model (a problem built from patterns "
                "only serves the KKT operators)");
  d = IpmDims{e.M, M.n_x, M.n_u, M.m, M.n_d()};
  xlo.upload(M.x_lo);
  xup.upload(M.x_up);
  ulo.upload(M.u_lo);
  uup.upload(M.u_up);
  slo.upload(M.s_lo);
  sup.upload(M.s_up);
  b = DevBounds{xlo.get(), xup.get(), ulo.get(), uup.get(), slo.get(), sup.get()};
  const size_t nx = size_t(d.M) * d.n_x, nm = size_t(d.M) * d.m, nu = size_t(d.n_u);
  for (IterStore& s : its) {
    for (DArr<double>* a : {&s.x, &s.y, &s.klo, &s.kup}) a->resize(nx);
    for (DArr<double>* a : {&s.s, &s.z, &s.nlo, &s.nup}) a->resize(nm);
    for (DArr<double>* a : {&s.u, &s.llo, &s.lup}) a->resize(nu);
  }
  bsv[0].resize(nx);
  bsv[1].resize(nx);
  bsv[2].resize(nm);
  bsv[3].resize(nm);
  bsv[4].resize(nu);
  bsv[5].resize(nu);
  gsum_u.resize(nu);
  ft.resize(size_t(d.M));
  gt.resize(nx);
  ht.resize(nm);
  partial.resize(600 * 16);  // up to 592 blocks x 16 reduction slots
  scal.resize(32);
  flag.resize(1);
  eval_counter.resize(1);
  eval_counter.zero(e.st);
  // multiplier count of the scaled error (ipm.cpp:345-379): structural
  double fin_x = 0, fin_s = 0, fin_u = 0;
  for (idx i = 0; i < M.n_x; ++i) fin_x += std::isfinite(M.x_lo[size_t(i)]) + std::isfinite(M.x_up[size_t(i)]);
  for (idx i = 0; i < M.m; ++i) fin_s += std::isfinite(M.s_lo[size_t(i)]) + std::isfinite(M.s_up[size_t(i)]);
  for (idx i = 0; i < M.n_u; ++i) fin_u += std::isfinite(M.u_lo[size_t(i)]) + std::isfinite(M.u_up[size_t(i)]);
  const double N = M.N;
  mult_count = N * (M.n_x + fin_x) + N * (M.m + fin_s) + fin_u;
}

double Solver::now() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Solver::ErrEval Solver::kkt_eval(const DevIter& it, Engine::Bundle& bd, const double mus[4],
                                 bool check_bad) {
  double* sc = scal.get();
  launch_grad_u_sum(d, bd.grad.get(), gsum_u.get(), e.st);
  allred(gsum_u.get(), size_t(d.n_u), RedOpKind::kSum);
  launch_kkt_eval(d, it, b, bd.grad.get(), bd.g.get(), bd.h.get(), bd.f.get(),
                  check_bad ? e.bad.get() : nullptr, e.lo, gsum_u.get(), mus, partial.get(),
                  eval_counter.get(), sc, e.st);
  allred(sc, 8, RedOpKind::kMax);      // x/s norms and complementarities
  allred(sc + 8, 2, RedOpKind::kSum);  // multiplier sum, objective
  allred(sc + 10, 1, RedOpKind::kMin); // lowest non-finite scenario
  const auto v = fetch<17>(sc);
  ErrEval E;
  E.stat = std::max({v[0], v[1], v[11]});
  E.primal = std::max(v[2], v[3]);
  for (int k = 0; k < 4; ++k) E.comp[k] = std::max(v[4 + k], v[12 + k]);
  E.mult = v[8] + v[16];
  E.obj = v[9];
  E.bad = v[10] < 1e299 ? idx(v[10]) : -1;
  return E;
}

// IPOPT-style scaled error (ipm.cpp:345-379) at barrier parameter k of E
Solver::Scaled Solver::scaled_of(const ErrEval& E, int k) const {
  const double avg = mult_count > 0 ? E.mult / mult_count : 0.0;
  const double s_d = std::max(100.0, avg) / 100.0;
  Scaled r;
  r.stationarity = E.stat / s_d;
  r.primal = E.primal;
  r.comp = E.comp[k] / s_d;
  r.comp_raw = E.comp[k];
  r.total = std::max({r.stationarity, r.primal, r.comp});
  return r;
}

void Solver::start() {
  const OpfModel& M = e.pb.M;
  std::vector<double> x0(size_t(M.n_x)), u0(size_t(M.n_u)), llo(size_t(M.n_u)), lup(size_t(M.n_u));
  for (idx i = 0; i < M.n_x; ++i)
    x0[size_t(i)] = project_start(M.x_start.empty() ? 0.0 : M.x_start[size_t(i)],
                                  M.x_lo[size_t(i)], M.x_up[size_t(i)]);
  for (idx i = 0; i < M.n_u; ++i) {
    const double lo = M.u_lo[size_t(i)], up = M.u_up[size_t(i)];
    const double u = project_start(M.u_start.empty() ? 0.0 : M.u_start[size_t(i)], lo, up);
    u0[size_t(i)] = u;
    llo[size_t(i)] = std::isfinite(lo) ? o.mu0 / (u - lo) : 0.0;
    lup[size_t(i)] = std::isfinite(up) ? o.mu0 / (up - u) : 0.0;
  }
  icur = 0;
  IterStore& s = its[0];
  DArr<double> dx0;
  // stream-ordered: kernels of an earlier solve may still use these buffers
  dx0.upload(x0.data(), x0.size(), e.st);
  s.u.upload(u0.data(), u0.size(), e.st);
  s.llo.upload(llo.data(), llo.size(), e.st);
  s.lup.upload(lup.data(), lup.size(), e.st);
  launch_init_x(d, cur(), b, dx0.get(), o.mu0, e.st);
  if (d.m > 0) {
    const idx bad = global_first_bad(e.eval_values(s.x.get(), s.u.get(), ft.get(), gt.get(), ht.get()));
    if (bad >= 0) throw Error(kNonFinite, "non-finite basis output at the start point", bad);
    launch_init_slacks(d, cur(), b, ht.get(), o.mu0, e.st);
  }
  e.sync();
  mu = o.mu0;
  delta_w_last = 0;
  iter = 0;
  bundle_fresh = false;
  status = kRunning;
  logs.clear();
  t_ad = t_kkt = 0;
  t0_ = std::chrono::steady_clock::now();
}

void Solver::compute_step(const DevIter& it) {
  Engine::Bundle& bd = e.bd();
  flag.zero(e.st);
  launch_grad_u_sum(d, bd.grad.get(), gsum_u.get(), e.st);
  allred(gsum_u.get(), size_t(d.n_u), RedOpKind::kSum);
  launch_assemble_xs(d, it, b, bd.grad.get(), bd.h.get(), mu, e.sigma_x.get(), kkt.r1x.get(),
                     e.sigma_s.get(), e.r2.get(), e.r4.get(), flag.get(), e.st);
  launch_assemble_u(d, it, b, gsum_u.get(), mu, e.sigma_u.get(), kkt.r1u.get(), flag.get(), e.st);
  kkt.condense_begin();  // per-scenario condensation beside the refactor (side stream)
  kkt.factor_launch();
  kkt.condense_end();
  kkt.check_factor(&flag);  // one round trip: interiority flag + refactor statuses
  kkt.solve(delta_w_last, o.reg);
  reductions = kkt.reductions;
}

int Solver::step() {
  if (status == kNotStarted)
    throw Error(kInvalidArgument, "solver: step() before start()");
  if (status != kRunning) return status;
  IterRecord log;
  log.iter = iter;
  const double t_iter = now();
  DevIter it = cur();
  bool evaluated = false;
  if (!bundle_fresh) {
    const double ta = now();
    e.eval_bundle(e.bd(), it.x, it.u, it.y, it.z, 1.0, /*check=*/false);
    evaluated = true;
    log.t_ad += now() - ta;
  }
  bundle_fresh = false;
  // residuals at mu = 0 and at the next barrier parameters in one pass
  double mus[4] = {0.0, mu, update_mu(mu, o), update_mu(update_mu(mu, o), o)};
  ErrEval E = kkt_eval(it, e.bd(), mus, evaluated);
  if (E.bad >= 0) throw Error(kNonFinite, "non-finite basis output", E.bad);
  const Scaled e0 = scaled_of(E, 0);
  log.objective = objective = E.obj;
  log.inf_pr = e0.primal;
  log.inf_du = e0.stationarity;
  log.complementarity = e0.comp_raw;
  auto finish = [&](int st_code) {
    log.t_total = now() - t_iter;
    t_ad += log.t_ad;
    t_kkt += log.t_kkt;
    logs.push_back(log);
    t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    if (st_code == kRunning && iter == o.max_iter - 1) st_code = kMaxIter;
    ++iter;
    status = st_code;
    return status;
  };
  if (e0.total <= o.tol) {
    log.mu = mu;
    return finish(kOptimal);
  }
  // barrier subproblem test and monotone mu decrease (ipm.cpp:484-492)
  double theta0 = 0.0;
  for (int k = 1;;) {
    if (k > 3) {  // beyond the precomputed candidates: another pass
      mus[1] = mu, mus[2] = update_mu(mu, o), mus[3] = update_mu(mus[2], o);
      E = kkt_eval(it, e.bd(), mus, false);
      k = 1;
    }
    const Scaled emu = scaled_of(E, k);
    if (emu.total <= o.kappa_eps * mu && mu > o.tol / 10.0) {
      mu = update_mu(mu, o);
      ++k;
      continue;
    }
    theta0 = emu.total;  // = the reference's fresh residual at the final mu
    break;
  }
  log.mu = mu;
  const double tk = now();
  compute_step(it);
  log.t_kkt = now() - tk;
  log.corrections = kkt.corrections;
  log.refinements = kkt.refinements;
  log.delta_w = kkt.last_dw;

  DevBoundStep bs{bsv[0].get(), bsv[1].get(), bsv[2].get(), bsv[3].get(), bsv[4].get(), bsv[5].get()};
  const DevStep ps = kkt.step_view();
  launch_bound_steps(d, it, b, ps, mu, o.tau, bs, partial.get(), scal.get(), e.st);
  allred(scal.get(), 2, RedOpKind::kMin);
  const auto caps = fetch<2>(scal.get());
  const double ap = std::min(1.0, caps[0]), ad = std::min(1.0, caps[1]);

  // full-step primal-dual acceptance (ipm.cpp:518-563)
  {
    DevIter tr = alt();
    launch_apply_step(d, it, tr, b, ps, bs, ap, ad, mu, e.st);
    const double ta = now();
    e.eval_bundle(e.trial(), tr.x, tr.u, tr.y, tr.z, 1.0, /*check=*/false);
    const double tmus[4] = {mu, mu, mu, mu};
    const ErrEval E1 = kkt_eval(tr, e.trial(), tmus, true);
    log.t_ad += now() - ta;
    const bool ok = E1.bad < 0;
    const double theta1 = ok ? scaled_of(E1, 0).total : kInf;
    if (ok && theta1 <= 0.99 * theta0) {
      icur = 1 - icur;
      e.swap_bundles();
      bundle_fresh = true;
      log.alpha_primal = ap;
      log.alpha_dual = ad;
      log.full_step = true;
      return finish(kRunning);
    }
  }

  // l1-merit Armijo backtracking (ipm.cpp:566-627)
  Engine::Bundle& bd = e.bd();
  launch_merit(d, it, b, ps, bd.grad.get(), bd.f.get(), bd.g.get(), bd.h.get(), e.gx_p.v,
               e.gu_p.v, e.hx_p.v, e.hu_p.v, bd.gx.get(), bd.gu.get(), bd.hx.get(), bd.hu.get(),
               mu, partial.get(), scal.get(), e.st);
  allred(scal.get(), 1, RedOpKind::kSum);
  allred(scal.get() + 1, 2, RedOpKind::kMax);
  allred(scal.get() + 3, 5, RedOpKind::kSum);
  launch_merit_u(d, it, b, ps.pu, mu, scal.get() + 8, e.st);
  const auto mv = fetch<10>(scal.get());
  const double viol0 = mv[0];
  const double penalty = 1.2 * std::max(mv[1], mv[2]) + 0.1;
  const double bar0 = mu * (mv[3] + mv[8]);
  const double phi0 = mv[6] + bar0 + penalty * viol0;
  const double dird = mv[5] + (mv[4] + mv[9]) - penalty * viol0;
  const double phi_scale = 1.0 + std::abs(bar0) + penalty * viol0 + mv[7];
  const double relax = 1e-13 * phi_scale;
  const double c1 = 1e-4;
  double alpha = ap;
  bool accepted = false;
  DevIter tr = alt();
  for (int ls = 0; ls < 60; ++ls) {
    launch_primal_trial(d, it, tr, ps, alpha, e.st);
    const double ta = now();
    const idx bad = global_first_bad(e.eval_values(tr.x, tr.u, ft.get(), gt.get(), ht.get()));
    if (bad < 0) {
      launch_ls_values(d, tr, b, ft.get(), gt.get(), ht.get(), partial.get(), scal.get() + 12,
                       e.st);
      allred(scal.get() + 12, 3, RedOpKind::kSum);
      launch_merit_u(d, tr, b, nullptr, mu, scal.get() + 15, e.st);
      const auto w = fetch<5>(scal.get() + 12);
      log.t_ad += now() - ta;
      const double phi = w[0] + mu * (w[1] + w[3]) + penalty * w[2];
      if (phi <= phi0 + c1 * alpha * std::min(dird, 0.0) + relax) {
        accepted = true;
        break;
      }
    } else {
      log.t_ad += now() - ta;
    }
    alpha *= 0.5;
    if (alpha < 1e-12) break;
  }
  if (!accepted) {
    message = "step too small (restoration not implemented, as in the reference)";
    return finish(kInfeasible);
  }
  launch_apply_step(d, it, tr, b, ps, bs, alpha, ad, mu, e.st);
  icur = 1 - icur;
  log.alpha_primal = alpha;
  log.alpha_dual = ad;
  return finish(kRunning);
}

double Solver::step_timed(int* st_out) {
  if (status != kRunning) start();
  cudaEvent_t a, z;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&z), "event");
  cudaEventRecord(a, e.st);
  const int s = step();
  cudaEventRecord(z, e.st);
  cudaEventSynchronize(z);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, z);
  cudaEventDestroy(a);
  cudaEventDestroy(z);
  if (st_out) *st_out = s;
  return ms;
}

int Solver::solve() {
  start();
  while (status == kRunning) step();
  return status;
}

std::vector<double> Solver::host_u() {
  std::vector<double> h(its[icur].u.size());
  its[icur].u.download(h.data(), h.size(), e.st);
  e.sync();
  return h;
}

std::vector<double> Solver::host_x() {
  std::vector<double> h(its[icur].x.size());
  its[icur].x.download(h.data(), h.size(), e.st);
  e.sync();
  return h;
}

void Solver::host_iterate(double* const out[11]) {
  IterStore& s = its[icur];
  DArr<double>* a[11] = {&s.x, &s.u, &s.s, &s.y, &s.z, &s.klo, &s.kup, &s.nlo, &s.nup, &s.llo, &s.lup};
  for (int k = 0; k < 11; ++k)
    if (out[k]) a[k]->download(out[k], a[k]->size(), e.st);
  e.sync();
}

}  // namespace bipm
