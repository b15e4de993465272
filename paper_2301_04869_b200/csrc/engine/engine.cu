#include "engine.hpp"

#include <algorithm>

namespace bipm {

std::unique_ptr<Problem> Problem::from_parts(GridCase cs, ScenarioDraw sc) {
  auto p = std::make_unique<Problem>();
  p->cs = std::move(cs);
  p->sc = std::move(sc);
  p->M = build_opf_model(p->cs, p->sc);
  p->deps = basis_deps(p->M);
  p->D = make_deriv_plan(p->M, p->deps);
  p->LU = make_lu_plan(p->D.g.x);
  return p;
}

std::unique_ptr<Problem> Problem::from_case_file(const std::string& path, idx N, double sigma,
                                                 std::uint64_t seed) {
  GridCase cs = read_matpower_file(path);
  ScenarioDraw sc = draw_scenarios(cs, N, sigma, {}, seed);
  return from_parts(std::move(cs), std::move(sc));
}

void DevPattern::upload(const Csr& p) {
  ptr.upload(p.ptr);
  ind.upload(p.ind);
  const Csr t = p.transpose_pattern();
  std::vector<int> slot(t.val.size());
  for (size_t k = 0; k < slot.size(); ++k) slot[k] = int(t.val[k]);
  t_ptr.upload(t.ptr);
  t_row.upload(t.ind);
  t_slot.upload(slot);
  v = DevCsr{p.rows, p.cols, p.nnz(), ptr.get(), ind.get(), t_ptr.get(), t_row.get(), t_slot.get()};
}

void DevCondense::upload(const CondenseProgram& p) {
  w_of.upload(p.w_of);
  ptr.upload(p.ptr);
  ka.upload(p.ka);
  kb.upload(p.kb);
  r.upload(p.r);
  v = CondenseDev{p.out.nnz(), w_of.get(), ptr.get(), ka.get(), kb.get(), r.get()};
}

Engine::Engine(const Problem& problem, int dev, idx lo_, idx hi_)
    : pb(problem), lo(lo_), hi(hi_), M(hi_ - lo_), device(dev) {
  if (lo < 0 || hi > pb.M.N || M < 1) throw Error(kInvalidArgument, "engine: bad scenario range");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  cuda_check(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device), "attr");
  const DerivPlan& D = pb.D;
  const LuPlan& L = pb.LU;
  const OpfModel& Mo = pb.M;

  gx_p.upload(D.g.x);
  gu_p.upload(D.g.u);
  hx_p.upload(D.h.x);
  hu_p.upload(D.h.u);
  kxx_p.upload(D.kxx.out);
  kxu_p.upload(D.kxu.out);
  kuu_p.upload(D.kuu.out);
  cxx.upload(D.kxx);
  cxu.upload(D.kxu);
  cuu.upload(D.kuu);

  auto up = [&](const std::vector<idx>& v) -> const int* {
    lu_arrays.emplace_back();
    lu_arrays.back().upload(v);
    return lu_arrays.back().get();
  };
  lu_arrays.reserve(40);
  lu.n = L.n;
  lu.nnz_l = L.nnz_l;
  lu.nnz_f = L.nnz_f;
  lu.n_fwd = idx(L.fwd_ptr.size()) - 1;
  lu.n_bwd = idx(L.bwd_ptr.size()) - 1;
  lu.perm = up(L.perm);
  lu.iperm = up(L.iperm);
  lu.l_ptr = up(L.l_ptr);
  lu.l_col = up(L.l_col);
  lu.u_ptr = up(L.u_ptr);
  lu.u_col = up(L.u_col);
  lu.u_slot = up(L.u_slot);
  lu.diag = up(L.diag);
  lu.ut_ptr = up(L.ut_ptr);
  lu.ut_row = up(L.ut_row);
  lu.ut_slot = up(L.ut_slot);
  lu.lt_ptr = up(L.lt_ptr);
  lu.lt_row = up(L.lt_row);
  lu.lt_slot = up(L.lt_slot);
  lu.fwd_ptr = up(L.fwd_ptr);
  lu.fwd_rows = up(L.fwd_rows);
  lu.bwd_ptr = up(L.bwd_ptr);
  lu.bwd_rows = up(L.bwd_rows);
  lu.lvl_u_ptr = up(L.lvl_u_ptr);
  lu.lvl_u_slot = up(L.lvl_u_slot);
  lu.lvl_l_ptr = up(L.lvl_l_ptr);
  lu.lvl_l_slot = up(L.lvl_l_slot);
  lu.a_src = up(L.a_src);
  lu.piv_of = up(L.piv_of);
  lu.mul_ptr = up(L.mul_ptr);
  lu.mul_l = up(L.mul_l);
  lu.mul_u = up(L.mul_u);

  const size_t Ms = size_t(M);
  gx.resize(Ms * nnz(D.g.x));
  gu.resize(Ms * nnz(D.g.u));
  hx.resize(Ms * nnz(D.h.x));
  hu.resize(Ms * nnz(D.h.u));
  wxx.resize(Ms * nnz(D.wxx));
  wxu.resize(Ms * nnz(D.wxu));
  wuu.resize(Ms * nnz(D.wuu));
  kxx.resize(Ms * nnz(D.kxx.out));
  kxu.resize(Ms * nnz(D.kxu.out));
  kuu.resize(Ms * nnz(D.kuu.out));
  sigma_x.resize(Ms * size_t(Mo.n_x));
  rhat1.resize(Ms * size_t(Mo.n_x));
  rhat3.resize(Ms * size_t(Mo.n_x));
  sigma_s.resize(Ms * size_t(Mo.m));
  r2.resize(Ms * size_t(Mo.m));
  r4.resize(Ms * size_t(Mo.m));
  sigma_u.resize(size_t(Mo.n_u));
  rhat2.resize(size_t(Mo.n_u));
  F.resize(Ms * size_t(L.nnz_f));
  lu_status.resize(Ms);
  khat.resize(size_t(Mo.n_u) * Mo.n_u);
  rhs.resize(size_t(Mo.n_u));
  rhs_part.resize(Ms * size_t(Mo.n_u));
  chol_info.resize(1);

  red.lu = lu;
  red.gu = gu_p.v;
  red.kxx = kxx_p.v;
  red.kxu = kxu_p.v;
  red.kuu = kuu_p.v;
  red.n_x = Mo.n_x;
  red.n_u = Mo.n_u;
  red.M = M;
  plan_reduce_launch(red, 200 * 1024, sm_count);
  red_partial.resize(size_t(red.nchunks) * Mo.n_u * Mo.n_u);
  red_scratch.resize(reduce_scratch_doubles(red));
}

Engine::~Engine() {
  if (st) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
}

void Engine::sync() { cuda_check(cudaStreamSynchronize(st), "stream sync"); }

idx Engine::factor_gx() {
  launch_lu_refactor(lu, M, gx.get(), pb.D.g.x.nnz(), F.get(), lu_status.get(), 1e-12, st);
  std::vector<int> s(static_cast<size_t>(M));
  lu_status.download(s.data(), s.size(), st);
  sync();
  for (idx b = 0; b < M; ++b)
    if (s[size_t(b)]) return lo + b;
  return -1;
}

void Engine::condense_blocks() {
  const DerivPlan& D = pb.D;
  const int m = pb.M.m;
  launch_condense(cxx.v, M, wxx.get(), D.wxx.nnz(), hx.get(), D.h.x.nnz(), hx.get(), D.h.x.nnz(),
                  sigma_s.get(), m, kxx.get(), st);
  launch_condense(cxu.v, M, wxu.get(), D.wxu.nnz(), hx.get(), D.h.x.nnz(), hu.get(), D.h.u.nnz(),
                  sigma_s.get(), m, kxu.get(), st);
  launch_condense(cuu.v, M, wuu.get(), D.wuu.nnz(), hu.get(), D.h.u.nnz(), hu.get(), D.h.u.nnz(),
                  sigma_s.get(), m, kuu.get(), st);
}

void Engine::reduce_local(double dw) {
  red.F = F.get();
  red.gu_v = gu.get();
  red.kxx_v = kxx.get();
  red.kxu_v = kxu.get();
  red.kuu_v = kuu.get();
  red.sigma_x = sigma_x.get();
  red.dw = dw;
  red.partial = red_partial.get();
  red.scratch = red_scratch.get();
  launch_reduce_tiles(red, st);
}

void Engine::reduce_rhs_local(double dw, double* d_out) {
  RhsLaunch a{};
  a.lu = lu;
  a.gu = gu_p.v;
  a.kxx = kxx_p.v;
  a.kxu = kxu_p.v;
  a.n_x = pb.M.n_x;
  a.n_u = pb.M.n_u;
  a.M = M;
  a.F = F.get();
  a.gu_v = gu.get();
  a.kxx_v = kxx.get();
  a.kxu_v = kxu.get();
  a.sigma_x = sigma_x.get();
  a.rhat1 = rhat1.get();
  a.rhat3 = rhat3.get();
  a.dw = dw;
  a.part = rhs_part.get();
  launch_reduce_rhs(a, st);
  launch_sum_parts(rhs_part.get(), M, pb.M.n_u, d_out, nullptr, 0.0, 0, nullptr, st);
}

void Engine::finish_reduce(double dw) {
  const int n_u = pb.M.n_u;
  launch_sum_parts(red_partial.get(), red.nchunks, (long long)n_u * n_u, khat.get(),
                   sigma_u.get(), dw, n_u, nullptr, st);
}

bool Engine::factor_khat() {
  launch_shift_cholesky(khat.get(), pb.M.n_u, chol_info.get(), nullptr, st);
  int info = 0;
  chol_info.download(&info, 1, st);
  sync();
  return info == 0;
}

void Engine::solve_khat(double* d_vec) { launch_cholesky_solve(khat.get(), pb.M.n_u, d_vec, st); }

void Engine::recover(double dw, const double* d_pu, double* d_px, double* d_py, double* d_pz,
                     double* d_ps) {
  RecoverLaunch a{};
  a.lu = lu;
  a.gu = gu_p.v;
  a.kxx = kxx_p.v;
  a.kxu = kxu_p.v;
  a.n_x = pb.M.n_x;
  a.n_u = pb.M.n_u;
  a.M = M;
  a.F = F.get();
  a.gu_v = gu.get();
  a.kxx_v = kxx.get();
  a.kxu_v = kxu.get();
  a.sigma_x = sigma_x.get();
  a.rhat1 = rhat1.get();
  a.rhat3 = rhat3.get();
  a.pu = d_pu;
  a.dw = dw;
  a.px = d_px;
  a.py = d_py;
  launch_recover_state(a, st);
  launch_recover_slack(hx_p.v, hu_p.v, pb.M.m, pb.M.n_x, M, hx.get(), hu.get(), d_px, d_pu,
                       sigma_s.get(), r2.get(), r4.get(), d_pz, d_ps, st);
}

}  // namespace bipm
