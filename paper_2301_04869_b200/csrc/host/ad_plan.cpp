#include "ad_plan.hpp"

#include <algorithm>

namespace bipm {

namespace {

idx pos_in(const std::vector<idx>& v, idx d) {
  auto it = std::find(v.begin(), v.end(), d);
  return it == v.end() ? -1 : idx(it - v.begin());
}

// slot lists of (coef, dp) for one Jacobian output entry (row i, input d)
void jac_entry(Gather& G, const Csr& L, idx i, idx d, const LaneDeps& deps,
               const std::vector<idx>& dp_off) {
  for (idx e = L.ptr[size_t(i)]; e < L.ptr[size_t(i) + 1]; ++e) {
    const idx lane = L.ind[size_t(e)];
    const idx p = pos_in(deps.jac[size_t(lane)], d);
    if (p >= 0) G.push(dp_off[size_t(lane)] + p, L.val[size_t(e)]);
  }
  G.close();
}

}  // namespace

AdProgram make_ad_program(const OpfModel& M, const LaneDeps& deps, const DerivPlan& D) {
  AdProgram A;
  const BasisLayout& lay = M.lay;
  const idx n_b = lay.n_b, n_x = M.n_x, n_d = M.n_d();

  A.dp_off.assign(size_t(n_b) + 1, 0);
  for (idx j = 0; j < n_b; ++j)
    A.dp_off[size_t(j) + 1] = A.dp_off[size_t(j)] + idx(deps.jac[size_t(j)].size());
  A.n_dp = A.dp_off.back();

  // ---- slack lane: p = Pd_ref + gs_ref vv_ref + ref branch flows - other gens
  A.sd = deps.jac[size_t(lay.pg + M.slack_gen)];
  std::vector<std::pair<double, idx>> terms;  // (coef, lane), reference order
  terms.push_back({M.gs_ref, lay.vv + M.ref_bus});
  for (idx l : M.ref_from) {
    const auto& c = M.br[size_t(l)];
    terms.push_back({c.gff, lay.cff(l)});
    terms.push_back({c.gft, lay.wc(l)});
    terms.push_back({c.bft, lay.ws(l)});
  }
  for (idx l : M.ref_to) {
    const auto& c = M.br[size_t(l)];
    terms.push_back({c.gtt, lay.ctt(l)});
    terms.push_back({c.gtf, lay.wc(l)});
    terms.push_back({-c.btf, lay.ws(l)});
  }
  for (idx g : M.ref_other_gens) terms.push_back({-1.0, lay.pg + g});
  for (const auto& [c, lane] : terms) A.slack_val.push(lane, c);
  A.slack_val.close();
  for (idx d : A.sd) {
    for (const auto& [c, lane] : terms) {
      const idx p = pos_in(deps.jac[size_t(lane)], d);
      if (p >= 0) A.slack_grad.push(A.dp_off[size_t(lane)] + p, c);
    }
    A.slack_grad.close();
  }

  A.branch_ref.assign(size_t(M.nbr), 0);
  for (idx l : M.ref_from) A.branch_ref[size_t(l)] |= 1;
  for (idx l : M.ref_to) A.branch_ref[size_t(l)] |= 2;
  A.gen_ref_other.assign(size_t(M.ngen), 0);
  for (idx g : M.ref_other_gens) A.gen_ref_other[size_t(g)] = 1;

  // ---- lane weights w = obj_w L_f' + L_g' y + L_h' z
  {
    const Csr ft = M.L_f.transpose_pattern(), gt = M.L_g.transpose_pattern(),
              ht = M.L_h.transpose_pattern();
    for (idx j = 0; j < n_b; ++j) {
      for (idx q = ft.ptr[size_t(j)]; q < ft.ptr[size_t(j) + 1]; ++q)
        A.w.push(-1, M.L_f.val[size_t(ft.val[size_t(q)])]);
      for (idx q = gt.ptr[size_t(j)]; q < gt.ptr[size_t(j) + 1]; ++q)
        A.w.push(gt.ind[size_t(q)], M.L_g.val[size_t(gt.val[size_t(q)])]);
      for (idx q = ht.ptr[size_t(j)]; q < ht.ptr[size_t(j) + 1]; ++q)
        A.w.push(n_x + ht.ind[size_t(q)], M.L_h.val[size_t(ht.val[size_t(q)])]);
      A.w.close();
    }
  }

  // ---- Jacobian blocks
  auto jac_block = [&](Gather& G, const Csr& pat, const Csr& L, idx col_off) {
    for (idx i = 0; i < pat.rows; ++i)
      for (idx k = pat.ptr[size_t(i)]; k < pat.ptr[size_t(i) + 1]; ++k)
        jac_entry(G, L, i, col_off + pat.ind[size_t(k)], deps, A.dp_off);
  };
  jac_block(A.gx, D.g.x, M.L_g, 0);
  jac_block(A.gu, D.g.u, M.L_g, n_x);
  jac_block(A.hx, D.h.x, M.L_h, 0);
  jac_block(A.hu, D.h.u, M.L_h, n_x);

  // ---- contributions to the Lagrangian gradient and Hessian
  A.c_bus = 14 * M.nbr;
  A.c_gen = A.c_bus + 2 * M.nbus;
  A.c_slack = A.c_gen + 2 * M.ngen;
  const idx nsd = idx(A.sd.size());
  A.n_c = A.c_slack + nsd * nsd;
  const Csr& H = D.hess;
  std::vector<std::vector<idx>> hc(static_cast<size_t>(H.nnz())), gc(static_cast<size_t>(n_d));
  auto add_h = [&](idx a, idx b, idx c) {
    const idx s = H.find(a, b);
    if (s >= 0) hc[size_t(s)].push_back(c);
  };
  for (idx b = 0; b < M.nbus; ++b) {
    const idx v = M.vmag_in[size_t(b)];
    gc[size_t(v)].push_back(A.c_bus + 2 * b);
    add_h(v, v, A.c_bus + 2 * b + 1);
  }
  static const int pair_index[4][4] = {{0, 1, 2, 3}, {1, 4, 5, 6}, {2, 5, 7, 8}, {3, 6, 8, 9}};
  for (idx l = 0; l < M.nbr; ++l) {
    const auto& c = M.br[size_t(l)];
    const idx loc[4] = {M.theta_in[size_t(c.from)], M.theta_in[size_t(c.to)],
                        M.vmag_in[size_t(c.from)], M.vmag_in[size_t(c.to)]};
    const idx base = 14 * l;
    for (int a = 0; a < 4; ++a)
      if (loc[a] >= 0) gc[size_t(loc[a])].push_back(base + a);
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
        if (loc[a] >= 0 && loc[b] >= 0) add_h(loc[a], loc[b], base + 4 + pair_index[a][b]);
  }
  for (idx g = 0; g < M.ngen; ++g) {
    if (g == M.slack_gen) continue;
    const idx p = M.pgen_in[size_t(g)];
    gc[size_t(p)].push_back(A.c_gen + 2 * g);
    add_h(p, p, A.c_gen + 2 * g + 1);
  }
  for (idx i = 0; i < nsd; ++i)
    for (idx j = 0; j < nsd; ++j) add_h(A.sd[size_t(i)], A.sd[size_t(j)], A.c_slack + i * nsd + j);

  for (idx d = 0; d < n_d; ++d) {
    for (idx c : gc[size_t(d)]) A.grad.push(c);
    A.grad.close();
  }
  auto hblock = [&](Gather& G, const std::vector<idx>& src) {
    for (idx s : src) {
      for (idx c : hc[size_t(s)]) G.push(c);
      G.close();
    }
  };
  hblock(A.wxx, D.wxx_src);
  hblock(A.wxu, D.wxu_src);
  hblock(A.wuu, D.wuu_src);
  return A;
}

}  // namespace bipm
