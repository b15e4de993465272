#include "kkt_step.hpp"

#include <cstdlib>
#include <string>
#include <vector>

namespace bipm {

KktStep::KktStep(Engine& eng, int rounds) : refine_rounds(rounds), e(eng), io(eng) {
  const OpfModel& M = e.pb.M;
  d = IpmDims{e.M, M.n_x, M.n_u, M.m, M.n_d()};
  const size_t nx = size_t(d.M) * d.n_x, nm = size_t(d.M) * d.m, nu = size_t(d.n_u);
  for (DArr<double>* s : {p, q}) {
    s[0].resize(nx);
    s[1].resize(nu);
    s[2].resize(nm);
    s[3].resize(nm);
    s[4].resize(nx);
  }
  r1x.resize(nx);
  r1u.resize(nu);
  o1x.resize(nx);
  o1u.resize(nu);
  o2.resize(nm);
  o3.resize(nx);
  o4.resize(nm);
  o1u_part.resize(size_t(d.M) * nu * 2);
  c_rhat1.resize(nx);
  c_rhat2.resize(nu);
  rhs_sum.resize(nu);
  red_u.resize(nu);
  dd_u.resize(2 * nu);
  rhat2_part.resize(size_t(d.M) * nu);
  partial.resize(600 * 16);  // up to 592 blocks x 16 reduction slots
  scal.resize(32);
  khat0.resize(nu * nu);
  khat1.resize(nu * nu);
  rhs0.resize(nu);
  rhs1.resize(nu);
  if (const char* v = std::getenv("BIPM_RETRY_EXACT")) exact_retries = std::atoi(v) != 0;
}

// base + sum over scenarios of part (and over ranks when sharded)
void KktStep::condensed_u_sum(const double* part, const double* base, double* out) {
  if (!e.multi()) {
    launch_scenario_sum(d.M, d.n_u, part, base, out, e.st);
    return;
  }
  launch_scenario_sum(d.M, d.n_u, part, nullptr, red_u.get(), e.st);
  io.allred(red_u.get(), size_t(d.n_u), RedOpKind::kSum);
  launch_scenario_sum(1, d.n_u, red_u.get(), base, out, e.st);
}

void KktStep::condense() {
  Engine::Bundle& bd = e.bd();
  cuda_check(cudaMemcpyAsync(e.rhat3.get(), bd.g.get(), e.rhat3.size() * sizeof(double),
                             cudaMemcpyDeviceToDevice, e.st),
             "rhat3");
  e.condense_blocks();
  launch_condensed_rhs(d, e.hx_p.v, e.hu_p.v, bd.hx.get(), bd.hu.get(), e.sigma_s.get(),
                       e.r4.get(), e.r2.get(), r1x.get(), e.rhat1.get(), rhat2_part.get(), e.st);
  condensed_u_sum(rhat2_part.get(), r1u.get(), e.rhat2.get());
}

void KktStep::condense_begin() {
  if (!e.overlap_rhs || !e.st_rhs) {
    cond_forked = false;
    return;
  }
  if (!ev_cond0) {
    cuda_check(cudaEventCreateWithFlags(&ev_cond0, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_cond1, cudaEventDisableTiming), "event");
  }
  Engine::Bundle& bd = e.bd();
  cudaStream_t s = e.st_rhs;
  cuda_check(cudaEventRecord(ev_cond0, e.st), "fork");
  cuda_check(cudaStreamWaitEvent(s, ev_cond0, 0), "fork");
  cuda_check(cudaMemcpyAsync(e.rhat3.get(), bd.g.get(), e.rhat3.size() * sizeof(double),
                             cudaMemcpyDeviceToDevice, s),
             "rhat3");
  e.condense_blocks(s);
  launch_condensed_rhs(d, e.hx_p.v, e.hu_p.v, bd.hx.get(), bd.hu.get(), e.sigma_s.get(),
                       e.r4.get(), e.r2.get(), r1x.get(), e.rhat1.get(), rhat2_part.get(), s);
  cuda_check(cudaEventRecord(ev_cond1, s), "join");
  cond_forked = true;
}

void KktStep::condense_end() {
  if (!cond_forked) {
    condense();
    return;
  }
  cuda_check(cudaStreamWaitEvent(e.st, ev_cond1, 0), "join");
  condensed_u_sum(rhat2_part.get(), r1u.get(), e.rhat2.get());
  cond_forked = false;
}

void KktStep::factor_launch() { e.factor_gx_launch(); }

void KktStep::check_factor(const DArr<int>* interior_flag) {
  std::vector<int> st_host(static_cast<size_t>(d.M) + 1, 0);
  if (interior_flag) interior_flag->download(st_host.data(), 1, e.st);
  e.lu_status.download(st_host.data() + 1, size_t(d.M), e.st);
  e.sync();
  if (interior_flag && io.host_all(double(st_host[0]), RedOpKind::kMax) > 0)
    throw Error(kNonInterior, "iterate not strictly interior");
  idx local_sing = -1;
  int why = 0;
  for (idx k = 0; k < d.M; ++k)
    if (st_host[size_t(k) + 1]) {
      local_sing = e.lo + k;
      why = st_host[size_t(k) + 1];
      break;
    }
  const idx sing = io.global_first_bad(local_sing);
  if (sing >= 0)
    throw Error(kSingularBlock,
                "singular block " + std::to_string(sing) +
                    (why == 2 && sing == local_sing
                         ? " (pivot growth of the shared static pivot order)"
                         : "") +
                    " (the reference falls back to the augmented strategy, which is not on the "
                    "GPU path)",
                sing);
}

bool KktStep::attempt(double dw, int k) {
  Engine::Bundle& bd = e.bd();
  const size_t nn = size_t(d.n_u) * d.n_u;
  auto copy = [&](DArr<double>& dst, const double* src, size_t n) {
    cuda_check(cudaMemcpyAsync(dst.get(), src, n * sizeof(double), cudaMemcpyDeviceToDevice, e.st),
               "copy");
  };
  const bool mix = k >= 2 && !exact_retries && dw1 != dw0;
  const double t = mix ? (dw - dw0) / (dw1 - dw0) : 0.0;
  auto mix_khat = [&] {
    launch_affine_mix(khat0.get(), khat1.get(), t, (long long)nn, e.khat.get(), e.st);
  };
  if (mix) {
    // K_hat(dw), rhs(dw) on the line through the first two attempts
    mix_khat();
    launch_affine_mix(rhs0.get(), rhs1.get(), t, d.n_u, rhs_sum.get(), e.st);
    ++mixed;
  } else {
    ++reductions;
    // the rhs reduction only reads the factors and the condensed blocks: it
    // runs on a side stream beside the Schur reduction (filling the SMs of
    // its last wave) and joins before the rhs is used
    e.reduce_rhs_fork(dw, rhs_sum.get());
    e.reduce_local(dw);
    e.finish_reduce(dw);
    e.reduce_rhs_join(rhs_sum.get());
    if (k <= 1 && !exact_retries) {  // the factor overwrites K_hat: keep it
      copy(k == 0 ? khat0 : khat1, e.khat.get(), nn);
      copy(k == 0 ? rhs0 : rhs1, rhs_sum.get(), size_t(d.n_u));
      (k == 0 ? dw0 : dw1) = dw;
    }
  }
  // refinement scale (independent of the factor) rides on the Cholesky sync
  launch_rhs_scale(d, r1x.get(), r1u.get(), e.r2.get(), bd.g.get(), e.r4.get(), partial.get(),
                   scal.get() + 20, e.st);
  io.allred(scal.get() + 20, 1, RedOpKind::kMax);
  io.fetch_async(scal.get() + 20, 40);
  if (!e.factor_khat(dw, mix ? std::function<void()>(mix_khat) : std::function<void()>()))
    return false;
  const double scale = io.pinned(40);
  // solve_with(c, first_sum): p_u, then state/adjoint and slack/dual recovery
  launch_pu_rhs(d.n_u, rhs_sum.get(), e.rhat2.get(), p[1].get(), true, e.st);
  e.solve_khat(p[1].get());
  e.recover(dw, p[1].get(), p[0].get(), p[4].get(), p[3].get(), p[2].get());
  // refinement against the unreduced augmented system (kkt.cpp:988-999)
  for (int round = 0; round < refine_rounds; ++round) {
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
    a.p = view(p);
    a.dw = dw;
    a.o1x = o1x.get();
    a.o2 = o2.get();
    a.o3 = o3.get();
    a.o4 = o4.get();
    a.o1u_part = o1u_part.get();
    launch_aug_residual(a, partial.get(), scal.get() + 21, e.st);
    if (e.multi()) {
      io.allred(scal.get() + 21, 1, RedOpKind::kMax);
      launch_aug_residual_u_local(a, dd_u.get(), e.st);
      io.allred(dd_u.get(), 2 * size_t(d.n_u), RedOpKind::kSum);
      launch_aug_residual_u_finish(a, dd_u.get(), o1u.get(), scal.get() + 22, e.st);
    } else {
      launch_aug_residual_u(a, dd_u.get(), o1u.get(), scal.get() + 22, e.st);
    }
    const auto v = io.fetch<2>(scal.get() + 21);
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
    launch_axpy_step(d, view(p), view(q), e.st);
  }
  return true;
}

void KktStep::solve(double& delta_w_last, const RegOptions& reg) {
  corrections = 0;
  refinements = 0;
  double dw = 0.0;
  int k = 0;
  if (!attempt(0.0, k++)) {
    dw = delta_w_last == 0 ? reg.delta_w0
                           : std::max(reg.delta_w_min, delta_w_last * reg.kappa_minus);
    for (;;) {
      ++corrections;
      if (attempt(dw, k++)) {
        delta_w_last = dw;
        break;
      }
      dw *= delta_w_last == 0 ? reg.kappa_plus_emergency : reg.kappa_plus;
      if (dw > reg.delta_w_max)
        throw Error(kLinearSolve, "inertia correction: regularization budget exhausted");
    }
  }
  last_dw = dw;
}

}  // namespace bipm
