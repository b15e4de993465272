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

Solver::Solver(Engine& eng, const SolverOptions& opt) : e(eng), o(opt) {
  const OpfModel& M = e.pb.M;
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
  for (DArr<double>* s : {p, q}) {
    s[0].resize(nx);
    s[1].resize(nu);
    s[2].resize(nm);
    s[3].resize(nm);
    s[4].resize(nx);
  }
  bsv[0].resize(nx);
  bsv[1].resize(nx);
  bsv[2].resize(nm);
  bsv[3].resize(nm);
  bsv[4].resize(nu);
  bsv[5].resize(nu);
  r1x.resize(nx);
  r1u.resize(nu);
  gsum_u.resize(nu);
  rhat2_part.resize(size_t(d.M) * nu);
  o1x.resize(nx);
  o1u.resize(nu);
  o2.resize(nm);
  o3.resize(nx);
  o4.resize(nm);
  o1u_part.resize(size_t(d.M) * nu * 2);
  c_rhat1.resize(nx);
  c_rhat2.resize(nu);
  rhs_sum.resize(nu);
  pu_rhs.resize(nu);
  red_u.resize(nu);
  dd_u.resize(2 * nu);
  ft.resize(size_t(d.M));
  gt.resize(nx);
  ht.resize(nm);
  partial.resize(600 * 16);  // up to 592 blocks x 16 reduction slots
  scal.resize(32);
  flag.resize(1);
  eval_counter.resize(1);
  eval_counter.zero(e.st);
  cuda_check(cudaMallocHost(&pinned, 64 * sizeof(double)), "cudaMallocHost");
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

template <int K>
std::array<double, K> Solver::fetch(const double* dptr) {
  cuda_check(cudaMemcpyAsync(pinned, dptr, K * sizeof(double), cudaMemcpyDeviceToHost, e.st),
             "fetch");
  stats().d2h_bytes += K * (long long)sizeof(double);
  e.sync();
  std::array<double, K> r;
  std::copy(pinned, pinned + K, r.begin());
  return r;
}

double Solver::fetch1(const double* dptr) { return fetch<1>(dptr)[0]; }

void Solver::allred(double* dptr, size_t n, RedOpKind op) {
  if (e.multi()) e.comm->allreduce(dptr, n, op, e.st);
}

double Solver::host_all(double v, RedOpKind op) {
  if (!e.multi()) return v;
  double* slot = scal.get() + 30;
  cuda_check(cudaMemcpyAsync(slot, &v, sizeof(double), cudaMemcpyHostToDevice, e.st), "h2d");
  e.comm->allreduce(slot, 1, op, e.st);
  return fetch1(slot);
}

idx Solver::global_first_bad(idx local_bad) {
  if (!e.multi()) return local_bad;
  const double v = host_all(local_bad >= 0 ? double(local_bad) : 1e300, RedOpKind::kMin);
  return v < 1e299 ? idx(v) : -1;
}

DevStep Solver::step_view(DArr<double>* s) {
  return DevStep{s[0].get(), s[1].get(), s[2].get(), s[3].get(), s[4].get()};
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
  dx0.upload(x0);
  s.u.upload(u0);
  s.llo.upload(llo);
  s.lup.upload(lup);
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

bool Solver::attempt(double dw, const DevIter& it) {
  (void)it;
  Engine::Bundle& bd = e.bd();
  ++reductions;
  // the rhs reduction only reads the factors and the condensed blocks: it runs
  // on a side stream beside the Schur reduction (filling the SMs of its last
  // wave) and joins before the rhs is used
  e.reduce_rhs_fork(dw, rhs_sum.get());
  e.reduce_local(dw);
  e.finish_reduce(dw);
  e.reduce_rhs_join(rhs_sum.get());
  // refinement scale (independent of the factor) rides on the Cholesky sync
  launch_rhs_scale(d, r1x.get(), r1u.get(), e.r2.get(), bd.g.get(), e.r4.get(), partial.get(),
                   scal.get() + 20, e.st);
  allred(scal.get() + 20, 1, RedOpKind::kMax);
  cudaMemcpyAsync(pinned + 40, scal.get() + 20, sizeof(double), cudaMemcpyDeviceToHost, e.st);
  if (!e.factor_khat()) return false;
  const double scale = pinned[40];
  // solve_with(c, first_sum): p_u, then state/adjoint and slack/dual recovery
  launch_pu_rhs(d.n_u, rhs_sum.get(), e.rhat2.get(), p[1].get(), true, e.st);
  e.solve_khat(p[1].get());
  e.recover(dw, p[1].get(), p[0].get(), p[4].get(), p[3].get(), p[2].get());
  // refinement against the unreduced augmented system (kkt.cpp:988-999)
  const DerivPlan& D = e.pb.D;
  (void)D;
  for (int round = 0; round < o.refine_rounds; ++round) {
    AugResidualArgs a{};
    a.d = d;
    a.gx = e.gx_p.v;
    a.gu = e.gu_p.v;
    a.hx = e.hx_p.v;
    a.hu = e.hu_p.v;
    a.wxx = e.wxx_p.v;
    a.wxu = e.wxu_p.v;
    a.wuu = e.wuu_p.v;
    a.gx_v = bd.gx.get();
    a.gu_v = bd.gu.get();
    a.hx_v = bd.hx.get();
    a.hu_v = bd.hu.get();
    a.wxx_v = bd.wxx.get();
    a.wxu_v = bd.wxu.get();
    a.wuu_v = bd.wuu.get();
    a.sigma_x = e.sigma_x.get();
    a.sigma_s = e.sigma_s.get();
    a.sigma_u = e.sigma_u.get();
    a.r1x = r1x.get();
    a.r1u = r1u.get();
    a.r2 = e.r2.get();
    a.r3 = bd.g.get();
    a.r4 = e.r4.get();
    a.p = step_view(p);
    a.dw = dw;
    a.o1x = o1x.get();
    a.o2 = o2.get();
    a.o3 = o3.get();
    a.o4 = o4.get();
    a.o1u_part = o1u_part.get();
    launch_aug_residual(a, partial.get(), scal.get() + 21, e.st);
    if (e.multi()) {
      allred(scal.get() + 21, 1, RedOpKind::kMax);
      launch_aug_residual_u_local(a, dd_u.get(), e.st);
      allred(dd_u.get(), 2 * size_t(d.n_u), RedOpKind::kSum);
      launch_aug_residual_u_finish(a, dd_u.get(), o1u.get(), scal.get() + 22, e.st);
    } else {
      launch_aug_residual_u(a, dd_u.get(), o1u.get(), scal.get() + 22, e.st);
    }
    const auto v = fetch<2>(scal.get() + 21);
    const double rel = std::max(v[0], v[1]) / scale;
    if (rel <= 1e-12) break;
    ++refinements;
    // substitute_rhs (kkt.cpp:342-358): re-condense only the rhs from rho
    launch_condensed_rhs(d, e.hx_p.v, e.hu_p.v, bd.hx.get(), bd.hu.get(), e.sigma_s.get(),
                         o4.get(), o2.get(), o1x.get(), c_rhat1.get(), rhat2_part.get(), e.st);
    condensed_u_sum(rhat2_part.get(), o1u.get(), c_rhat2.get());
    e.reduce_rhs_local(dw, rhs_sum.get(), c_rhat1.get(), o3.get());
    launch_pu_rhs(d.n_u, rhs_sum.get(), c_rhat2.get(), q[1].get(), false, e.st);
    e.solve_khat(q[1].get());
    e.recover(dw, q[1].get(), q[0].get(), q[4].get(), q[3].get(), q[2].get(), c_rhat1.get(),
              o3.get(), o2.get(), o4.get());
    launch_axpy_step(d, step_view(p), step_view(q), e.st);
  }
  return true;
}

void Solver::compute_step(const DevIter& it) {
  Engine::Bundle& bd = e.bd();
  flag.zero(e.st);
  launch_grad_u_sum(d, bd.grad.get(), gsum_u.get(), e.st);
  allred(gsum_u.get(), size_t(d.n_u), RedOpKind::kSum);
  launch_assemble_xs(d, it, b, bd.grad.get(), bd.h.get(), mu, e.sigma_x.get(), r1x.get(),
                     e.sigma_s.get(), e.r2.get(), e.r4.get(), flag.get(), e.st);
  launch_assemble_u(d, it, b, gsum_u.get(), mu, e.sigma_u.get(), r1u.get(), flag.get(), e.st);
  cuda_check(cudaMemcpyAsync(e.rhat3.get(), bd.g.get(), e.rhat3.size() * sizeof(double),
                             cudaMemcpyDeviceToDevice, e.st),
             "rhat3");
  e.condense_blocks();
  launch_condensed_rhs(d, e.hx_p.v, e.hu_p.v, bd.hx.get(), bd.hu.get(), e.sigma_s.get(),
                       e.r4.get(), e.r2.get(), r1x.get(), e.rhat1.get(), rhat2_part.get(), e.st);
  condensed_u_sum(rhat2_part.get(), r1u.get(), e.rhat2.get());
  e.factor_gx_launch();
  // one round trip for the interiority flag and the refactor statuses
  std::vector<int> st_host(static_cast<size_t>(d.M) + 1);
  flag.download(st_host.data(), 1, e.st);
  e.lu_status.download(st_host.data() + 1, size_t(d.M), e.st);
  e.sync();
  if (host_all(double(st_host[0]), RedOpKind::kMax) > 0)
    throw Error(kNonInterior, "iterate not strictly interior");
  idx local_sing = -1;
  for (idx k = 0; k < d.M; ++k)
    if (st_host[size_t(k) + 1]) {
      local_sing = e.lo + k;
      break;
    }
  const idx sing = global_first_bad(local_sing);
  if (sing >= 0)
    throw Error(kSingularBlock,
                "singular block " + std::to_string(sing) +
                    " (the reference falls back to the augmented strategy, which is not on the "
                    "GPU path)",
                sing);
  corrections = 0;
  refinements = 0;
  double dw = 0.0;
  if (!attempt(0.0, it)) {
    dw = delta_w_last == 0 ? o.reg.delta_w0
                           : std::max(o.reg.delta_w_min, delta_w_last * o.reg.kappa_minus);
    for (;;) {
      ++corrections;
      if (attempt(dw, it)) {
        delta_w_last = dw;
        break;
      }
      dw *= delta_w_last == 0 ? o.reg.kappa_plus_emergency : o.reg.kappa_plus;
      if (dw > o.reg.delta_w_max)
        throw Error(kLinearSolve, "inertia correction: regularization budget exhausted");
    }
  }
  last_dw = dw;
}

int Solver::step() {
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
  log.corrections = corrections;
  log.refinements = refinements;
  log.delta_w = last_dw;

  DevBoundStep bs{bsv[0].get(), bsv[1].get(), bsv[2].get(), bsv[3].get(), bsv[4].get(), bsv[5].get()};
  const DevStep ps = step_view(p);
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
  launch_merit_u(d, it, b, p[1].get(), mu, scal.get() + 8, e.st);
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

// base + sum over scenarios of part (and over ranks when sharded)
void Solver::condensed_u_sum(const double* part, const double* base, double* out) {
  if (!e.multi()) {
    launch_scenario_sum(d.M, d.n_u, part, base, out, e.st);
    return;
  }
  launch_scenario_sum(d.M, d.n_u, part, nullptr, red_u.get(), e.st);
  allred(red_u.get(), size_t(d.n_u), RedOpKind::kSum);
  launch_scenario_sum(1, d.n_u, red_u.get(), base, out, e.st);
}

int Solver::solve() {
  start();
  while (status == kRunning) step();
  return status;
}

std::vector<double> Solver::host_u() const {
  return const_cast<Solver*>(this)->its[icur].u.to_host();
}

std::vector<double> Solver::host_x() const {
  return const_cast<Solver*>(this)->its[icur].x.to_host();
}

}  // namespace bipm
