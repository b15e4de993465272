#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace bipm {

std::unique_ptr<Problem> Problem::from_parts(GridCase cs, ScenarioDraw sc) {
  auto p = std::make_unique<Problem>();
  p->cs = std::move(cs);
  p->sc = std::move(sc);
  p->M = build_opf_model(p->cs, p->sc);
  p->deps = basis_deps(p->M);
  p->D = make_deriv_plan(p->M, p->deps);
  p->LU = make_lu_plan(p->D.g.x);
  p->AD = make_ad_program(p->M, p->deps, p->D);
  return p;
}

std::unique_ptr<Problem> Problem::from_case_file(const std::string& path, idx N, double sigma,
                                                 std::uint64_t seed,
                                                 const std::vector<idx>& contingencies) {
  GridCase cs = read_matpower_file(path);
  ScenarioDraw sc = draw_scenarios(cs, N, sigma, contingencies, seed);
  return from_parts(std::move(cs), std::move(sc));
}

std::unique_ptr<Problem> Problem::from_patterns(idx N, Csr gx, Csr gu, Csr hx, Csr hu, Csr wxx,
                                                Csr wxu, Csr wuu) {
  const idx n_x = gx.rows, n_u = gu.cols, m = hx.rows;
  auto need = [](bool ok, const char* what) {
    if (!ok) throw Error(kInvalidArgument, std::string("patterns: ") + what);
  };
  need(N >= 1 && n_x >= 1 && n_u >= 1, "need N, n_x, n_u >= 1");
  need(gx.cols == n_x && gu.rows == n_x, "G_x must be n_x x n_x and G_u n_x x n_u");
  need(hu.rows == m && hx.cols == n_x && hu.cols == n_u, "H_x / H_u shapes");
  need(wxx.rows == n_x && wxx.cols == n_x && wxu.rows == n_x && wxu.cols == n_u &&
           wuu.rows == n_u && wuu.cols == n_u,
       "W_xx / W_xu / W_uu shapes");
  for (const Csr* c : {&gx, &gu, &hx, &hu, &wxx, &wxu, &wuu}) {
    need(c->ptr.size() == size_t(c->rows) + 1 && c->ptr.front() == 0 &&
             c->ptr.back() == c->nnz(),
         "row pointers");
    for (idx i = 0; i < c->rows; ++i)
      for (idx k = c->ptr[size_t(i)]; k < c->ptr[size_t(i) + 1]; ++k)
        need(c->ind[size_t(k)] >= 0 && c->ind[size_t(k)] < c->cols &&
                 (k == c->ptr[size_t(i)] || c->ind[size_t(k)] > c->ind[size_t(k) - 1]),
             "column indices must be in range and strictly increasing per row");
  }
  auto p = std::make_unique<Problem>();
  p->model = false;
  p->M.N = N;
  p->M.n_x = n_x;
  p->M.n_u = n_u;
  p->M.m = m;
  p->M.name = "patterns";
  DerivPlan& D = p->D;
  D.g.x = std::move(gx);
  D.g.u = std::move(gu);
  D.h.x = std::move(hx);
  D.h.u = std::move(hu);
  D.wxx = std::move(wxx);
  D.wxu = std::move(wxu);
  D.wuu = std::move(wuu);
  // the reference's make_condense_work (kkt.cpp:111-117)
  D.kxx = plan_condense_program(D.wxx, D.h.x, D.h.x);
  D.kxu = plan_condense_program(D.wxu, D.h.x, D.h.u);
  D.kuu = plan_condense_program(D.wuu, D.h.u, D.h.u);
  p->LU = make_lu_plan(D.g.x);
  return p;
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
  cuda_check(cudaStreamCreateWithFlags(&st_rhs, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_levels, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_reach, cudaEventDisableTiming), "event");
  if (const char* e = std::getenv("BIPM_NO_OVERLAP")) overlap_rhs = std::atoi(e) == 0;
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
  wxx_p.upload(D.wxx);
  wxu_p.upload(D.wxu);
  wuu_p.upload(D.wuu);
  cxx.upload(D.kxx);
  cxu.upload(D.kxu);
  cuu.upload(D.kuu);

  auto up = [&](const std::vector<idx>& v) -> const int* {
    lu_arrays.emplace_back();
    lu_arrays.back().upload(v);
    return lu_arrays.back().get();
  };
  lu_arrays.reserve(120);
  lu.n = L.n;
  lu.growth = 1e10;  // ~10 of 16 digits lost to growth: the refinement cannot recover them
  if (const char* e = std::getenv("BIPM_GROWTH_LIMIT")) lu.growth = std::atof(e);
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
  auto up0 = [&](const std::vector<idx>& v) { return up(v.empty() ? std::vector<idx>{0} : v); };
  lu.n_nt = idx(L.nt_lvl_u_ptr.size()) - 1;
  lu.n_tail_ent = idx(L.tail_slot.size());
  lu.nt_lvl_u_ptr = up(L.nt_lvl_u_ptr);
  lu.nt_lvl_u_slot = up0(L.nt_lvl_u_slot);
  lu.nt_lvl_l_ptr = up(L.nt_lvl_l_ptr);
  lu.nt_lvl_l_slot = up0(L.nt_lvl_l_slot);
  lu.tail_slot = up0(L.tail_slot);
  lu.tail_mul_ptr = up(L.tail_mul_ptr);
  lu.tail_mul_l = up0(L.tail_mul_l);
  lu.tail_mul_u = up0(L.tail_mul_u);
  lu.rf_nphase = idx(L.rf_phase_ptr.size()) - 1;
  lu.rf_phase_ptr = up(L.rf_phase_ptr);
  lu.rf_rec = reinterpret_cast<const int4*>(up(L.rf_rec.empty() ? std::vector<idx>{0, 0, 0, -1} : L.rf_rec));
  lu.rf_piv = up0(L.rf_piv);
  lu.rf_pair = reinterpret_cast<const int2*>(up(L.rf_pair.empty() ? std::vector<idx>{0, 0} : L.rf_pair));
  lu.t0 = L.t0;
  lu.tl = L.tl;
  lu.ft_src = up(L.ft_src);
  {
    std::vector<idx> ds;
    for (const auto& v : L.dense_src) ds.insert(ds.end(), v.begin(), v.end());
    if (ds.empty()) ds.push_back(-1);
    lu.dense_src = up(ds);
  }
  auto sweep = [&](const SweepPlan& S) {
    DevSweep d{};
    d.col = up(S.col.empty() ? std::vector<idx>{0} : S.col);
    d.items = up(S.items.empty() ? std::vector<idx>{0, 0, 0, 0} : S.items);
    d.lvl_ptr = up(S.lvl_ptr);
    d.n_lvl = idx(S.lvl_ptr.size()) - 1;
    d.tail_items = up(S.tail_items.empty() ? std::vector<idx>{0, 0, 0, 0} : S.tail_items);
    d.n_tail = idx(S.tail_items.size() / 4);
    return d;
  };
  lu.sL = sweep(L.sL);
  lu.sU = sweep(L.sU);
  lu.sUt = sweep(L.sUt);
  lu.sLt = sweep(L.sLt);

  const size_t Ms = size_t(M);
  for (Bundle& b : bundles) {
    b.f.resize(Ms);
    b.g.resize(Ms * size_t(Mo.n_x));
    b.h.resize(Ms * size_t(Mo.m));
    b.gx.resize(Ms * nnz(D.g.x));
    b.gu.resize(Ms * nnz(D.g.u));
    b.hx.resize(Ms * nnz(D.h.x));
    b.hu.resize(Ms * nnz(D.h.u));
    b.wxx.resize(Ms * nnz(D.wxx));
    b.wxu.resize(Ms * nnz(D.wxu));
    b.wuu.resize(Ms * nnz(D.wuu));
    b.grad.resize(Ms * size_t(Mo.n_d()));
  }
  if (pb.has_model()) upload_ad();
  // +2: the streamed reduction's bulk copies start on a 16-byte boundary
  kxx.resize(Ms * nnz(D.kxx.out) + 2);
  kxu.resize(Ms * nnz(D.kxu.out));
  kuu.resize(Ms * nnz(D.kuu.out));
  sigma_x.resize(Ms * size_t(Mo.n_x) + 2);
  rhat1.resize(Ms * size_t(Mo.n_x));
  rhat3.resize(Ms * size_t(Mo.n_x));
  sigma_s.resize(Ms * size_t(Mo.m));
  r2.resize(Ms * size_t(Mo.m));
  r4.resize(Ms * size_t(Mo.m));
  sigma_u.resize(size_t(Mo.n_u));
  rhat2.resize(size_t(Mo.n_u));
  F.resize(Ms * size_t(L.nnz_f));
  FT.resize(Ms * size_t(L.nnz_f));
  Dt.resize(std::max<size_t>(1, Ms * 2 * size_t(L.tl) * size_t(L.tl)) + 2);
  lu_status.resize(Ms);
  lu_scale.resize(Ms);
  if (!single_rhs_smem(int(Mo.n_x))) rhs_scratch.resize(Ms * 2 * size_t(Mo.n_x));
  khat.resize(size_t(Mo.n_u) * Mo.n_u);
  rhs.resize(size_t(Mo.n_u));
  rhs_part.resize(Ms * size_t(Mo.n_u));
  chol_info.resize(8);  // status, |K|_inf, rejected pivot (kkt_kernels.hpp)
  bk_ipiv.resize(size_t(Mo.n_u));
  bk_inertia.resize(4);
  bk_state.resize(bk_work_bytes(Mo.n_u));
  if (const char* e = std::getenv("BIPM_FORCE_BK")) force_bk = std::atoi(e) != 0;

  red.lu = lu;
  red.gu = gu_p.v;
  red.kxx = kxx_p.v;
  red.kxu = kxu_p.v;
  red.kuu = kuu_p.v;
  red.n_x = Mo.n_x;
  red.n_u = Mo.n_u;
  red.M = M;
  plan_reduce_launch(red, 200 * 1024, sm_count);
  if (const char* e = std::getenv("BIPM_REDUCE")) use_stream = std::strcmp(e, "tiles") != 0;
  if (const char* e = std::getenv("BIPM_FORCE_COMM")) force_comm = std::atoi(e) != 0;
  if (use_stream) setup_stream();
  if (use_stream) {
    red_parts = sl.nchunks + 1 + tail_splits;  // + the K_uu slab + the tail GEMM's
    red_partial.resize(size_t(red_parts) * Mo.n_u * Mo.n_u);
    red_partial.zero(st);
  } else {
    red_parts = red.nchunks;
    red_partial.resize(size_t(red.nchunks) * Mo.n_u * Mo.n_u);
    red_scratch.resize(reduce_scratch_doubles(red));
  }
}

void Engine::setup_stream() {
  const DerivPlan& D = pb.D;
  const LuPlan& L = pb.LU;
  const int n_x = pb.M.n_x, n_u = pb.M.n_u;
  // Configuration: tile width K, consumers C per CTA and CTAs per SM.  Among
  // the configurations with a useful ring (>= 16 KB) keep the most panel
  // columns in flight per SM (K x CTAs), then the widest tile: measured at
  // 1354/256, one CTA of 512 consumers with K = 8 (47.8 ms) beats two CTAs
  // with K = 4 (62 ms) and four with K = 1 (100 ms) -- each level step costs
  // the same latency whatever its width, and smaller rings mean more steps.
  int cap = 1;
  while (cap < 32 && cap < n_u) cap *= 2;
  if (const char* e = std::getenv("BIPM_PRESOLVE")) presolve = std::atoi(e) != 0;
  if (presolve) rplan = build_reach_plan(L, D.g.u, n_u);
  const Csr gut = D.g.u.transpose_pattern(), kxut = D.kxu.out.transpose_pattern();
  if (const char* e = std::getenv("BIPM_STREAM_K")) cap = std::max(1, std::min(cap, std::atoi(e)));
  int force_c = 0;
  if (const char* e = std::getenv("BIPM_STREAM_C")) force_c = std::atoi(e);
  auto list_cap_of = [&](int K) {
    int lc = 0;
    for (int j0 = 0; j0 < n_u; j0 += K) {
      const int j1 = std::min(n_u, j0 + K);
      const int a = presolve ? rplan.yn_ptr[size_t(j1)] - rplan.yn_ptr[size_t(j0)]
                             : gut.ptr[size_t(j1)] - gut.ptr[size_t(j0)];
      const int b = kxut.ptr[size_t(j1)] - kxut.ptr[size_t(j0)];
      lc = std::max(lc, ((a + 1) & ~1) + ((b + 1) & ~1));
    }
    return lc;
  };
  struct Cfg { int K, C, ctas, ring, list_cap; };
  Cfg best{0, 0, 0, 0, 0};
  for (int C : {512, 256, 128}) {
    if (force_c && C != force_c) continue;
    const int ctas = 512 / C;
    for (int K = cap; K >= 1; K /= 2) {
      if (C < 512 && K > (C == 256 ? 8 : 4)) continue;  // instantiated kernels
      if ((size_t(n_u) * K + C - 1) / C > size_t(kStreamMaxQ)) continue;
      const int lc = list_cap_of(K);
      const int ring = stream_ring_capacity(n_x, K, L.tl, 4096, lc, ctas);
      if (ring < 16 * 1024) continue;
      const bool better = K * ctas > best.K * best.ctas ||
                          (K * ctas == best.K * best.ctas && K > best.K);
      if (better) best = Cfg{K, C, ctas, ring, lc};
      break;  // widest K that fits for this C
    }
  }
  if (best.K < 1) {
    use_stream = false;  // panel does not fit: tile kernel with a global panel
    return;
  }
  const int K = best.K, ring = best.ring, list_cap = best.list_cap;
  // adjoint identity (stream_plan.hpp): the L' sweep and W' product give way
  // to a y_N' z_N accumulation and an n_u x tl product against X_T -- a win
  // while n_u x tl stays small against the sweep it removes
  // (BIPM_ADJ_IDENTITY=0/1 overrides)
  bool adj = false;
  if (presolve) {
    long long lt_ent = 0;
    for (idx i = 0; i < L.t0; ++i) lt_ent += L.lt_ptr[size_t(i) + 1] - L.lt_ptr[size_t(i)];
    adj = rplan.nnz_yn < lt_ent;  // measured: 1354 and 2869 gain, 9241 loses
    if (const char* e = std::getenv("BIPM_ADJ_IDENTITY")) adj = std::atoi(e) != 0;
  }
  adj_identity = adj;
  if (const char* e = std::getenv("BIPM_TAIL_DEFER")) defer_tail = std::atoi(e) != 0;
  defer_tail = defer_tail && adj && L.tl > 0;
  // producer lookahead in steps (< the kernel's 32 mbarrier slots;
  // BIPM_LOOKAHEAD for experiments)
  int lookahead = kStreamLookahead;
  if (const char* e = std::getenv("BIPM_LOOKAHEAD")) lookahead = std::max(1, std::min(31, std::atoi(e)));
  sprog = build_stream_program(L, D.g.u, D.kxx.out, D.kxu.out, n_u, K, best.C, ring,
                               lookahead, presolve ? &rplan : nullptr, adj, defer_tail);
  if (presolve) {
    rp_op_ptr.upload(rplan.op_ptr);
    rp_ops.upload(rplan.ops.empty() ? std::vector<idx>(4, 0) : rplan.ops);
    rp_ent.upload(rplan.ent.empty() ? std::vector<idx>(2, 0) : rplan.ent);
    rp_yn_ptr.upload(rplan.yn_ptr);
    rp_yn_row.upload(rplan.yn_row.empty() ? std::vector<idx>{0} : rplan.yn_row);
    rp_yt_ptr.upload(rplan.yt_ptr);
    rp_yt_row.upload(rplan.yt_row.empty() ? std::vector<idx>{0} : rplan.yt_row);
    // the sparse product wins while y_T is sparse enough (measured: 1354 with
    // 307 tail rows, 8.7 % dense: 1.42 -> 1.29 ms per reduce_pre at 256
    // scenarios; 272 rows, ~10 %: 1.36 -> 1.32; 2869 with 314 rows (11 %) and
    // 9241 (17.5 %) lose against the DMMA GEMM)
    // (2869 with the 506-row tail is 8.6 % dense but the GEMM, on larger
    // operands, wins: 1.62 against 2.01 ms -- and the staged W' column block
    // leaves one CTA per SM; so only short tails)
    xt_sparse = L.tl <= 320 &&
                double(rplan.yt_row.size()) < 0.12 * double(n_u) * double(std::max<idx>(1, L.tl));
    if (const char* e = std::getenv("BIPM_XT_SPARSE")) xt_sparse = std::atoi(e) != 0;
    int ymax = 1;
    for (idx u = 0; u < n_u; ++u)
      ymax = std::max(ymax, int(rplan.yn_ptr[size_t(u) + 1] - rplan.yn_ptr[size_t(u)]));
    // lanes per column ~ the mean entries per op (1354: 4.5 -> 4, 9241: 42 -> 32)
    const double per_op = double(rplan.fmas) / std::max<size_t>(1, rplan.ops.size() / 4);
    // (1354, 4.5 entries per op: 8 lanes 1.31 against 4 lanes 1.36 ms per reduce_pre)
    int grp = per_op <= 3 ? 4 : per_op <= 14 ? 8 : per_op <= 28 ? 16 : 32;
    if (const char* e = std::getenv("BIPM_REACH_GROUP")) grp = std::atoi(e);  // experiments
    const idx nnz_yt = idx(rplan.yt_row.size());
    rdev = ReachDev{int(n_u), int(L.tl), int(rplan.ldy), int(rplan.nnz_yn), ymax, grp,
                    rp_op_ptr.get(), reinterpret_cast<const int4*>(rp_ops.get()),
                    reinterpret_cast<const int2*>(rp_ent.get()), rp_yn_ptr.get(),
                    xt_sparse ? 1 : 0, int(nnz_yt), rp_yt_ptr.get()};
    const size_t Ms = size_t(M);
    YN.resize(Ms * size_t(std::max<idx>(1, rplan.nnz_yn)) + 2);  // + the bulk copies' 16-byte rounding
    // the sparse product reads y_T packed (its pattern only); the GEMM dense
    YT.resize(Ms * (xt_sparse ? size_t(std::max<idx>(1, nnz_yt)) : size_t(n_u) * size_t(rplan.ldy)));
    XT.resize(Ms * size_t(n_u) * size_t(rplan.ldy));
    XT.zero(st);
    if (defer_tail) {
      ZT.resize(Ms * size_t(n_u) * size_t(rplan.ldy));
      ZT.zero(st);
      // about sixteen CTAs per SM over the lower 64 x 64 tiles of K_hat (up
      // to five are co-resident; measured reduce_post, same box: 1354/256
      // 10 -> 32 splits 1.13 -> 0.85 ms, 2869/512 3 -> 16-64 splits 13.8 ->
      // 9.0-9.3 ms -- three CTAs per SM left the FP64 pipe idle)
      const long long tt = (n_u + 63) / 64, t = tt * (tt + 1) / 2;
      tail_splits = int(std::max(1LL, std::min<long long>(M, (16LL * sm_count + t / 2) / t)));
      if (const char* e = std::getenv("BIPM_TAIL_SPLITS"))
        tail_splits = std::max(1, std::min(int(M), std::atoi(e)));
    }
  }
  sp_pat.upload(sprog.pat);
  {
    std::vector<int> iss;
    iss.reserve(sprog.issue.size() * 12);
    for (const StepIssue& is : sprog.issue) {
      const int r[12] = {is.pat_off, is.pat_bytes, is.ring_off, is.val_arr, is.val_off,
                         is.val_count, is.x_arr, is.x_off, is.x_count, is.val_ring, is.x_ring,
                         is.wait_delta};
      iss.insert(iss.end(), r, r + 12);
    }
    sp_issue.upload(iss);
  }
  {
    // ring words: offset | accumulation-step skip control (reduce_stream.cu kRw*)
    // (BIPM_ACC_SKIP=0: no step skipped, for A/B runs)
    const char* ev = std::getenv("BIPM_ACC_SKIP");
    const bool acc_skip = !ev || std::atoi(ev) != 0;
    std::vector<int> rw(sprog.ring_off.size());
    for (size_t j = 0; j < rw.size(); ++j) {
      const unsigned off = unsigned(sprog.ring_off[j]);
      if (off > 0x3ffffu) throw Error(kInvalidArgument, "stream program: ring offset exceeds 18 bits");
      const int sk = sprog.skip[j];
      const unsigned hi = acc_skip ? unsigned(std::min(sk >> 4, 4095)) : 4095u;
      const unsigned fl = ((sk & kFlagBarrier) ? 1u << 18 : 0u) | ((sk & kFlagPre) ? 1u << 19 : 0u);
      rw[j] = int(off | fl | (hi << 20));
    }
    sp_ring.upload(rw);
  }
  sp_vs_src.upload(sprog.vs_src);
  sp_kxu_slot.upload(sprog.kxu_t_slot.empty() ? std::vector<idx>{0} : sprog.kxu_t_slot);
  sp_gu_slot.upload(sprog.gu_t_slot.empty() ? std::vector<idx>{0} : sprog.gu_t_slot);
  {
    const Csr& ku = D.kuu.out;
    std::vector<idx> r(size_t(ku.nnz())), c(ku.ind.begin(), ku.ind.end());
    for (idx i = 0; i < ku.rows; ++i)
      for (idx k = ku.ptr[size_t(i)]; k < ku.ptr[size_t(i) + 1]; ++k) r[size_t(k)] = i;
    if (r.empty()) r.push_back(0), c.push_back(0);
    kuu_row.upload(r);
    kuu_col.upload(c);
  }
  const size_t Ms = size_t(M);
  VS.resize(Ms * size_t(sprog.nnz_vs) + 2);
  Dp.resize(std::max<size_t>(1, Ms * size_t(sprog.stride[kArrDense])));
  kxu_t.resize(Ms * nnz(D.kxu.out) + 2);
  gu_t.resize(Ms * nnz(D.g.u) + 2);

  sl.n_x = n_x;
  sl.n_u = n_u;
  sl.M = M;
  sl.K = K;
  sl.nq = sprog.nq;
  sl.steps = sprog.steps;
  sl.ring_bytes = ring;
  sl.t0 = L.t0;
  sl.tl = L.tl;
  sl.list_cap = list_cap;
  sl.consumers = best.C;
  sl.ctas_per_sm = best.ctas;
  plan_stream_chunks(sl, sm_count);
  sl.pat = sp_pat.get();
  sl.issue = sp_issue.get();
  sl.ring_off = sp_ring.get();
  for (int k = 0; k < kStreamArrays; ++k) sl.stride[k] = sprog.stride[k];
  sl.gu = gu_p.v;
  sl.kxu = kxu_p.v;
  sl.kuu = kuu_p.v;
  sl.iperm = lu.iperm;
  sl.presolved = presolve ? 1 : 0;
  sl.ldy = int(rplan.ldy);
  sl.nnz_yn = int(rplan.nnz_yn);
  sl.yn_ptr = presolve ? rp_yn_ptr.get() : nullptr;
  sl.yn_row = presolve ? rp_yn_row.get() : nullptr;
  sl.yn_v = presolve ? YN.get() : nullptr;
  sl.xt = presolve ? XT.get() : nullptr;
  sl.zt = defer_tail ? ZT.get() : nullptr;
  const int tiles = (n_u + K - 1) / K;
  sp_scratch.resize(size_t(tiles) * sl.nchunks * (size_t(n_x) * K + size_t(list_cap)));
}

Engine::~Engine() {
  if (st_rhs) {
    cudaStreamSynchronize(st_rhs);
    cudaStreamDestroy(st_rhs);
  }
  for (auto& t : pending_timers) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_levels) cudaEventDestroy(ev_levels);
  if (ev_reach) cudaEventDestroy(ev_reach);
  if (st) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
}

void Engine::sync() { cuda_check(cudaStreamSynchronize(st), "stream sync"); }

// the padded dense slot the streamed reduction reads: both without the
// adjoint identity (W for the first dense product, W' for the second); with
// it, W for the X_T GEMM or W' for the sparse X_T product
int Engine::dp_slot() const {
  if (!use_stream || !presolve || !adj_identity) return -1;
  return xt_sparse ? 1 : 0;
}

bool Engine::reach_overlap() const { return use_stream && presolve && overlap_rhs && st_rhs; }

void Engine::invalidate_reach() {
  // a stale reach still in flight on st_rhs must not overlap what st does
  // next with G_u, y_N, y_T
  if (reach_ready) cuda_check(cudaStreamWaitEvent(st, ev_reach, 0), "reach join");
  reach_ready = false;
}

void Engine::launch_reach_async() {
  invalidate_reach();
  if (!reach_overlap()) return;
  cuda_check(cudaStreamWaitEvent(st_rhs, ev_levels, 0), "reach wait");
  timed("reduce_pre", [&] {
    launch_reach_solve(rdev, M, F.get(), pb.LU.nnz_f, bd().gu.get(), nnz(pb.D.g.u), YN.get(),
                       YT.get(), st_rhs);
  }, st_rhs);
  cuda_check(cudaEventRecord(ev_reach, st_rhs), "reach record");
  reach_ready = true;
}

void Engine::factor_gx_launch() {
  timed("lu_refactor", [&] {
    launch_lu_refactor(lu, M, bd().gx.get(), pb.D.g.x.nnz(), F.get(), FT.get(), Dt.get(),
                       lu_status.get(), 1e-12, use_stream ? sp_vs_src.get() : nullptr,
                       int(sprog.nnz_vs), use_stream ? VS.get() : nullptr,
                       use_stream ? Dp.get() : nullptr, lu_scale.get(), st, dp_slot(),
                       reach_overlap() ? ev_levels : nullptr);
  });
  launch_reach_async();
}

idx Engine::factor_gx() {
  timed("lu_refactor", [&] {
    launch_lu_refactor(lu, M, bd().gx.get(), pb.D.g.x.nnz(), F.get(), FT.get(), Dt.get(),
                       lu_status.get(), 1e-12, use_stream ? sp_vs_src.get() : nullptr,
                       int(sprog.nnz_vs), use_stream ? VS.get() : nullptr,
                       use_stream ? Dp.get() : nullptr, lu_scale.get(), st, dp_slot(),
                       reach_overlap() ? ev_levels : nullptr);
  });
  launch_reach_async();
  std::vector<int> s(static_cast<size_t>(M));
  lu_status.download(s.data(), s.size(), st);
  sync();
  for (idx b = 0; b < M; ++b)
    if (s[size_t(b)]) return lo + b;
  return -1;
}

void Engine::condense_blocks(cudaStream_t on) {
  timed("condense", [&] { condense_launch(on); }, on);
}

void Engine::condense_launch(cudaStream_t on) {
  cudaStream_t st = on ? on : this->st;
  const DerivPlan& D = pb.D;
  const int m = pb.M.m;
  launch_condense(cxx.v, M, bd().wxx.get(), D.wxx.nnz(), bd().hx.get(), D.h.x.nnz(), bd().hx.get(), D.h.x.nnz(),
                  sigma_s.get(), m, kxx.get(), st);
  launch_condense(cxu.v, M, bd().wxu.get(), D.wxu.nnz(), bd().hx.get(), D.h.x.nnz(), bd().hu.get(), D.h.u.nnz(),
                  sigma_s.get(), m, kxu.get(), st);
  launch_condense(cuu.v, M, bd().wuu.get(), D.wuu.nnz(), bd().hu.get(), D.h.u.nnz(), bd().hu.get(), D.h.u.nnz(),
                  sigma_s.get(), m, kuu.get(), st);
}

void Engine::reduce_local(double dw) {
  if (use_stream) {
    const DerivPlan& D = pb.D;
    const int n_u = pb.M.n_u;
    double* kuu_part = red_partial.get() + size_t(sl.nchunks) * n_u * n_u;
    if (presolve) {
      // forward half for all columns: y_N, y_T (reach_solve, already issued
      // beside the refactor's dense tail when reach_ready), X_T = W y_T
      if (reach_ready) cuda_check(cudaStreamWaitEvent(st, ev_reach, 0), "reach join");
      timed("reduce_pre", [&] {
        if (!reach_ready)
          launch_reach_solve(rdev, M, F.get(), pb.LU.nnz_f, bd().gu.get(), nnz(D.g.u), YN.get(),
                             YT.get(), st);
        const int tl = int(pb.LU.tl);
        if (xt_sparse) {
          // W' = W transposed is Dp's second slot (rows padded to dense_ld)
          launch_xt_sparse(Dp.get() + size_t(tl) * dense_ld(tl), dense_ld(tl),
                           sprog.stride[kArrDense], YT.get(), rdev.nnz_yt, rp_yt_ptr.get(),
                           rp_yt_row.get(), n_u, tl, int(M), XT.get(), rplan.ldy, st);
        } else {
          GemmTN g{tl, n_u, tl, int(M), 0, 1.0, 0, Dp.get(), dense_ld(tl), sprog.stride[kArrDense],
                   YT.get(), rplan.ldy, (long long)n_u * rplan.ldy,
                   XT.get(), rplan.ldy, (long long)n_u * rplan.ldy};
          launch_gemm_tn(g, st);
        }
      });
    }
    timed("reduce_tiles", [&] {
      launch_gather_values(kxu.get(), nnz(D.kxu.out), sp_kxu_slot.get(), int(nnz(D.kxu.out)),
                           kxu_t.get(), nnz(D.kxu.out), M, st);
      if (!adj_identity)  // the G_u' Y accumulation reads column-order G_u
        launch_gather_values(bd().gu.get(), nnz(D.g.u), sp_gu_slot.get(), int(nnz(D.g.u)),
                             gu_t.get(), nnz(D.g.u), M, st);
      launch_kuu_sum(kuu.get(), nnz(D.kuu.out), kuu_row.get(), kuu_col.get(),
                     int(nnz(D.kuu.out)), M, n_u, kuu_part, st);
      sl.arr[kArrSweep] = VS.get();
      sl.arr[kArrDense] = Dp.get();
      sl.arr[kArrKxx] = kxx.get();
      sl.arr[kArrKxuT] = kxu_t.get();
      sl.arr[kArrGuT] = gu_t.get();
      sl.arr[kArrSigma] = sigma_x.get();
      sl.arr[kArrYN] = presolve ? YN.get() : nullptr;
      sl.gu_v = bd().gu.get();
      sl.kxu_v = kxu.get();
      sl.kuu_v = kuu.get();
      sl.dw = dw;
      sl.partial = red_partial.get();
      sl.scratch = sp_scratch.get();
      sl.phase = phase.size() ? phase.get() : nullptr;
      static const int dbg = [] {
        const char* e = std::getenv("BIPM_STREAM_DEBUG");
        return e ? std::atoi(e) : 0;
      }();
      sl.debug = dbg;
      launch_reduce_stream(sl, st);
    });
    if (defer_tail) {
      // -sum_s X_T' Z_T into the tail slabs (after the K_uu slab)
      timed("reduce_post", [&] {
        const int tl = int(pb.LU.tl);
        const long long nn = (long long)n_u * n_u;
        GemmTN g{n_u, n_u, tl, int(M), tail_splits, -1.0, /*lower=*/1,
                 XT.get(), rplan.ldy, (long long)n_u * rplan.ldy,
                 ZT.get(), rplan.ldy, (long long)n_u * rplan.ldy,
                 red_partial.get() + size_t(sl.nchunks + 1) * nn, n_u, nn};
        launch_gemm_tn(g, st);
      });
    }
    return;
  }
  red.F = F.get();
  red.FT = FT.get();
  red.D = Dt.get();
  red.gu_v = bd().gu.get();
  red.kxx_v = kxx.get();
  red.kxu_v = kxu.get();
  red.kuu_v = kuu.get();
  red.sigma_x = sigma_x.get();
  red.dw = dw;
  red.partial = red_partial.get();
  red.scratch = red_scratch.get();
  red.phase = phase.size() ? phase.get() : nullptr;
  timed("reduce_tiles", [&] { launch_reduce_tiles(red, st); });
}

void Engine::reduce_rhs_local(double dw, double* d_out, const double* d_rhat1,
                              const double* d_rhat3) {
  RhsLaunch a{};
  a.lu = lu;
  a.gu = gu_p.v;
  a.kxx = kxx_p.v;
  a.kxu = kxu_p.v;
  a.n_x = pb.M.n_x;
  a.n_u = pb.M.n_u;
  a.M = M;
  a.F = F.get();
  a.FT = FT.get();
  a.D = Dt.get();
  a.gu_v = bd().gu.get();
  a.kxx_v = kxx.get();
  a.kxu_v = kxu.get();
  a.sigma_x = sigma_x.get();
  a.rhat1 = d_rhat1 ? d_rhat1 : rhat1.get();
  a.rhat3 = d_rhat3 ? d_rhat3 : rhat3.get();
  a.dw = dw;
  a.part = rhs_part.get();
  a.scratch = rhs_scratch.size() ? rhs_scratch.get() : nullptr;
  // step-stamp debug mode: the last 64 entries of the buffer
  a.phase = phase.size() > 1000 ? phase.get() + phase.size() - 64 : nullptr;
  timed("reduce_rhs", [&] { launch_reduce_rhs(a, st); });
  launch_sum_parts(rhs_part.get(), M, pb.M.n_u, d_out, nullptr, 0.0, 0, nullptr, st);
  if (multi()) comm->allreduce(d_out, size_t(pb.M.n_u), RedOpKind::kSum, st);
}

void Engine::reduce_rhs_fork(double dw, double* d_out) {
  if (!overlap_rhs) {
    reduce_rhs_local(dw, d_out);
    return;
  }
  RhsLaunch a{};
  a.lu = lu;
  a.gu = gu_p.v;
  a.kxx = kxx_p.v;
  a.kxu = kxu_p.v;
  a.n_x = pb.M.n_x;
  a.n_u = pb.M.n_u;
  a.M = M;
  a.F = F.get();
  a.FT = FT.get();
  a.D = Dt.get();
  a.gu_v = bd().gu.get();
  a.kxx_v = kxx.get();
  a.kxu_v = kxu.get();
  a.sigma_x = sigma_x.get();
  a.rhat1 = rhat1.get();
  a.rhat3 = rhat3.get();
  a.dw = dw;
  a.part = rhs_part.get();
  a.scratch = rhs_scratch.size() ? rhs_scratch.get() : nullptr;
  a.phase = phase.size() > 1000 ? phase.get() + phase.size() - 64 : nullptr;
  cuda_check(cudaEventRecord(ev_fork, st), "fork");
  cuda_check(cudaStreamWaitEvent(st_rhs, ev_fork, 0), "fork");
  timed("reduce_rhs", [&] { launch_reduce_rhs(a, st_rhs); }, st_rhs);
  launch_sum_parts(rhs_part.get(), M, pb.M.n_u, d_out, nullptr, 0.0, 0, nullptr, st_rhs);
  cuda_check(cudaEventRecord(ev_join, st_rhs), "join");
}

void Engine::reduce_rhs_join(double* d_out) {
  if (!overlap_rhs) return;
  cuda_check(cudaStreamWaitEvent(st, ev_join, 0), "join");
  if (multi()) comm->allreduce(d_out, size_t(pb.M.n_u), RedOpKind::kSum, st);
}

cudaEvent_t Engine::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cuda_check(cudaEventCreate(&e), "event");
  return e;
}

void Engine::resolve_timers() {
  for (auto& t : pending_timers) {
    cudaEventSynchronize(t.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, t.a, t.b);
    KTimer& k = ktimers[t.name];
    k.ms += ms;
    ++k.n;
    event_pool.push_back(t.a);
    event_pool.push_back(t.b);
  }
  pending_timers.clear();
}

void Engine::finish_reduce(double dw) {
  const int n_u = pb.M.n_u;
  const long long nn = (long long)n_u * n_u;
  // the lower triangles of the slabs, mirrored (the tail GEMM computes the
  // lower tiles only; the Cholesky and Bunch-Kaufman read the lower triangle)
  if (!multi()) {
    launch_sum_parts(red_partial.get(), red_parts, nn, khat.get(), sigma_u.get(), dw, n_u,
                     nullptr, st, n_u);
    return;
  }
  // local sum -> all-reduce over the scenario groups -> diagonal terms once
  launch_sum_parts(red_partial.get(), red_parts, nn, khat.get(), nullptr, 0.0, 0, nullptr, st,
                   n_u);
  comm->allreduce(khat.get(), size_t(nn), RedOpKind::kSum, st);
  launch_sum_parts(khat.get(), 1, nn, khat.get(), sigma_u.get(), dw, n_u, nullptr, st, n_u);
}

bool Engine::factor_khat(double dw, const std::function<void()>& regenerate) {
  const int n = pb.M.n_u;
  timed("cholesky", [&] { launch_shift_cholesky(khat.get(), n, chol_info.get(), nullptr, st); });
  int info[8] = {0};
  chol_info.download(info, 6, st);
  sync();
  khat_bk = false;
  if (info[0] == 0) return true;
  double kinf = 0.0, piv = 0.0;
  std::memcpy(&kinf, info + 2, sizeof(double));
  std::memcpy(&piv, info + 4, sizeof(double));
  // dpotrf rejects a pivot that is not > 0; a clearly negative (or NaN) one
  // means K_hat is indefinite, which the reference's Bunch-Kaufman inertia
  // reports too (neg > 0): reject without factoring again
  const double tol = 4.0 * n * 2.220446049250313e-16 * std::max(1.0, kinf);
  if (!(piv > -tol) && !force_bk) return false;
  if (regenerate)  // K_hat again: the Cholesky overwrote it
    regenerate();
  else
    finish_reduce(dw);
  timed("cholesky", [&] {
    launch_bk_factor(khat.get(), n, bk_ipiv.get(), bk_state.get(), bk_inertia.get(), st);
  });
  int in[3] = {0, 0, 0};
  bk_inertia.download(in, 3, st);
  sync();
  ++bk_fallbacks;
  if (in[1] == 0 && in[2] == 0) {
    khat_bk = true;
    return true;
  }
  return false;
}

void Engine::solve_khat(double* d_vec) {
  const int n = pb.M.n_u;
  timed("khat_solve", [&] {
    if (khat_bk)
      launch_bk_solve(khat.get(), n, bk_ipiv.get(), d_vec, st);
    else
      launch_cholesky_solve(khat.get(), n, d_vec, st);
  });
}

void Engine::recover(double dw, const double* d_pu, double* d_px, double* d_py, double* d_pz,
                     double* d_ps, const double* d_rhat1, const double* d_rhat3,
                     const double* d_r2, const double* d_r4) {
  RecoverLaunch a{};
  a.lu = lu;
  a.gu = gu_p.v;
  a.kxx = kxx_p.v;
  a.kxu = kxu_p.v;
  a.n_x = pb.M.n_x;
  a.n_u = pb.M.n_u;
  a.M = M;
  a.F = F.get();
  a.FT = FT.get();
  a.D = Dt.get();
  a.gu_v = bd().gu.get();
  a.kxx_v = kxx.get();
  a.kxu_v = kxu.get();
  a.sigma_x = sigma_x.get();
  a.rhat1 = d_rhat1 ? d_rhat1 : rhat1.get();
  a.rhat3 = d_rhat3 ? d_rhat3 : rhat3.get();
  a.pu = d_pu;
  a.dw = dw;
  a.px = d_px;
  a.py = d_py;
  a.scratch = rhs_scratch.size() ? rhs_scratch.get() : nullptr;
  timed("recover_state", [&] { launch_recover_state(a, st); });
  launch_recover_slack(hx_p.v, hu_p.v, pb.M.m, pb.M.n_x, M, bd().hx.get(), bd().hu.get(), d_px, d_pu,
                       sigma_s.get(), d_r2 ? d_r2 : r2.get(), d_r4 ? d_r4 : r4.get(), d_pz, d_ps, st);
}

}  // namespace bipm

namespace bipm {

namespace {

template <typename T>
const T* keep(std::vector<DArr<T>>& store, const std::vector<T>& v) {
  store.emplace_back();
  store.back().upload(v);
  return store.back().get();
}

}  // namespace

void Engine::upload_ad() {
  const OpfModel& Mo = pb.M;
  const AdProgram& P = pb.AD;
  ad_i.reserve(64);
  ad_d.reserve(32);
  DevAd& A = ad;
  A.M = M;
  A.nbus = Mo.nbus;
  A.nbr = Mo.nbr;
  A.ngen = Mo.ngen;
  A.n_x = Mo.n_x;
  A.n_u = Mo.n_u;
  A.m = Mo.m;
  A.n_b = Mo.n_b();
  A.n_d = Mo.n_d();
  A.ref_bus = Mo.ref_bus;
  A.slack_gen = Mo.slack_gen;
  A.vv = Mo.lay.vv;
  A.br = Mo.lay.br;
  A.sq = Mo.lay.sq;
  A.pd = Mo.lay.pd;
  A.qd = Mo.lay.qd;
  A.pg = Mo.lay.pg;
  A.pg2 = Mo.lay.pg2;
  A.vmag_in = keep(ad_i, Mo.vmag_in);
  A.pgen_in = keep(ad_i, Mo.pgen_in);
  std::vector<idx> th(2 * size_t(Mo.nbr)), vm(2 * size_t(Mo.nbr));
  std::vector<double> brc(8 * size_t(Mo.nbr));
  for (idx l = 0; l < Mo.nbr; ++l) {
    const auto& c = Mo.br[size_t(l)];
    th[2 * size_t(l)] = Mo.theta_in[size_t(c.from)];
    th[2 * size_t(l) + 1] = Mo.theta_in[size_t(c.to)];
    vm[2 * size_t(l)] = Mo.vmag_in[size_t(c.from)];
    vm[2 * size_t(l) + 1] = Mo.vmag_in[size_t(c.to)];
    const double v[8] = {c.gff, c.bff, c.gft, c.bft, c.gtf, c.btf, c.gtt, c.btt};
    std::copy(v, v + 8, brc.begin() + 8 * long(l));
  }
  A.br_th = keep(ad_i, th);
  A.br_v = keep(ad_i, vm);
  A.brc = keep(ad_d, brc);
  A.gs_ref = Mo.gs_ref;
  A.br_ref = keep(ad_i, P.branch_ref);
  A.gen_ref_other = keep(ad_i, P.gen_ref_other);
  // the owned scenarios' constants, element-major ([width][M]) for the
  // scenario-fastest AD kernels
  auto slice = [&](const std::vector<double>& all, idx width) {
    std::vector<double> t(size_t(width) * size_t(M));
    for (idx s = 0; s < M; ++s)
      for (idx k = 0; k < width; ++k)
        t[size_t(k) * size_t(M) + size_t(s)] = all[size_t(lo + s) * size_t(width) + size_t(k)];
    return t;
  };
  pd_v.upload(slice(Mo.pd, Mo.nbus));
  qd_v.upload(slice(Mo.qd, Mo.nbus));
  status_v.upload(slice(Mo.status, Mo.nbr));
  A.pd_v = pd_v.get();
  A.qd_v = qd_v.get();
  A.status = status_v.get();
  A.Lf_ptr = keep(ad_i, Mo.L_f.ptr);
  A.Lf_ind = keep(ad_i, Mo.L_f.ind);
  A.Lf_val = keep(ad_d, Mo.L_f.val);
  A.Lg_ptr = keep(ad_i, Mo.L_g.ptr);
  A.Lg_ind = keep(ad_i, Mo.L_g.ind);
  A.Lg_val = keep(ad_d, Mo.L_g.val);
  A.Lh_ptr = keep(ad_i, Mo.L_h.ptr);
  A.Lh_ind = keep(ad_i, Mo.L_h.ind);
  A.Lh_val = keep(ad_d, Mo.L_h.val);
  A.n_dp = P.n_dp;
  A.n_c = P.n_c;
  A.c_bus = P.c_bus;
  A.c_gen = P.c_gen;
  A.c_slack = P.c_slack;
  A.nsd = idx(P.sd.size());
  A.dp_off = keep(ad_i, P.dp_off);
  A.sd = keep(ad_i, P.sd);
  auto gat = [&](const Gather& G) {
    DevGather d{};
    d.n = G.outputs();
    d.ptr = keep(ad_i, G.ptr);
    d.src = keep(ad_i, G.src);
    d.coef = G.coef.empty() ? nullptr : keep(ad_d, G.coef);
    return d;
  };
  A.slack_val = gat(P.slack_val);
  A.slack_grad = gat(P.slack_grad);
  A.w = gat(P.w);
  A.gx = gat(P.gx);
  A.gu = gat(P.gu);
  A.hx = gat(P.hx);
  A.hu = gat(P.hu);
  A.grad = gat(P.grad);
  A.wxx = gat(P.wxx);
  A.wxu = gat(P.wxu);
  A.wuu = gat(P.wuu);
  xt.resize(size_t(M) * size_t(Mo.n_x));
  yt.resize(size_t(M) * size_t(Mo.n_x));
  zt.resize(size_t(M) * size_t(std::max(1, Mo.m)));
  psi.resize(size_t(M) * size_t(A.n_b));
  dpart.resize(size_t(M) * size_t(std::max(1, A.n_dp)));
  wlane.resize(size_t(M) * size_t(A.n_b));
  contrib.resize(size_t(M) * size_t(std::max(1, A.n_c)));
  bad.resize(size_t(M));
}

idx Engine::eval_bundle(Bundle& out, const double* dX, const double* du, const double* dY,
                        const double* dZ, double obj_w, bool check) {
  if (!pb.has_model())
    throw Error(kInvalidArgument, "eval_bundle: the problem was built from patterns only");
  // a reach solve still reading a bundle's G_u must finish before any bundle
  // is rewritten (the async one reads bd(); a trial bundle becomes bd() on swap)
  invalidate_reach();
  AdBuffers b{};
  b.X = dX;
  b.u = du;
  b.Y = dY;
  b.Z = dZ;
  b.obj_w = obj_w;
  b.Xt = xt.get();
  b.Yt = yt.get();
  b.Zt = zt.get();
  b.psi = psi.get();
  b.dp = dpart.get();
  b.w = wlane.get();
  b.c = contrib.get();
  b.f = out.f.get();
  b.g = out.g.get();
  b.h = out.h.get();
  b.gx = out.gx.get();
  b.gu = out.gu.get();
  b.hx = out.hx.get();
  b.hu = out.hu.get();
  b.wxx = out.wxx.get();
  b.wxu = out.wxu.get();
  b.wuu = out.wuu.get();
  b.grad = out.grad.get();
  b.bad = bad.get();
  bad.zero(st);
  timed("ad_bundle", [&] { launch_ad_bundle(ad, b, st); });
  return check ? first_bad() : -1;
}

idx Engine::eval_values(const double* dX, const double* du, double* df, double* dg,
                        double* dh) {
  if (!pb.has_model())
    throw Error(kInvalidArgument, "eval_values: the problem was built from patterns only");
  AdBuffers b{};
  b.X = dX;
  b.u = du;
  b.Xt = xt.get();
  b.psi = psi.get();
  b.dp = dpart.get();
  b.f = df;
  b.g = dg;
  b.h = dh;
  b.bad = bad.get();
  bad.zero(st);
  timed("ad_values", [&] { launch_ad_values(ad, b, st); });
  return first_bad();
}

idx Engine::first_bad() {
  std::vector<int> flags(static_cast<size_t>(M));
  bad.download(flags.data(), flags.size(), st);
  sync();
  for (idx s = 0; s < M; ++s)
    if (flags[size_t(s)]) return lo + s;
  return -1;
}

}  // namespace bipm
