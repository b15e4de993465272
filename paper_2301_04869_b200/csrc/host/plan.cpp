#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <set>

namespace bipm {

namespace {

std::vector<idx> branch_support(const OpfModel& M, idx l) {
  const auto& c = M.br[size_t(l)];
  std::vector<idx> v;
  if (M.theta_in[size_t(c.from)] >= 0) v.push_back(M.theta_in[size_t(c.from)]);
  if (M.theta_in[size_t(c.to)] >= 0) v.push_back(M.theta_in[size_t(c.to)]);
  v.push_back(M.vmag_in[size_t(c.from)]);
  v.push_back(M.vmag_in[size_t(c.to)]);
  return v;
}

SplitMap split_columns(const Csr& p, idx n_x) {
  SplitMap s;
  std::vector<std::pair<idx, idx>> xc, uc;
  for (idx i = 0; i < p.rows; ++i)
    for (idx k = p.ptr[size_t(i)]; k < p.ptr[size_t(i) + 1]; ++k) {
      const idx c = p.ind[size_t(k)];
      (c < n_x ? xc : uc).push_back(c < n_x ? std::pair{i, c} : std::pair{i, c - n_x});
    }
  s.x = Csr::pattern(p.rows, n_x, xc);
  s.u = Csr::pattern(p.rows, p.cols - n_x, uc);
  s.x_src.assign(size_t(s.x.nnz()), -1);
  s.u_src.assign(size_t(s.u.nnz()), -1);
  for (idx i = 0; i < p.rows; ++i)
    for (idx k = p.ptr[size_t(i)]; k < p.ptr[size_t(i) + 1]; ++k) {
      const idx c = p.ind[size_t(k)];
      if (c < n_x)
        s.x_src[size_t(s.x.find(i, c))] = k;
      else
        s.u_src[size_t(s.u.find(i, c - n_x))] = k;
    }
  return s;
}

// Sorted-list intersection: calls f(pos_a, pos_b) for every common value.
template <typename F>
void intersect(const idx* a, idx na, const idx* b, idx nb, F&& f) {
  idx i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j])
      ++i;
    else if (b[j] < a[i])
      ++j;
    else
      f(i++, j++);
  }
}

}  // namespace

LaneDeps basis_deps(const OpfModel& M) {
  const BasisLayout& lay = M.lay;
  LaneDeps d;
  d.jac.assign(size_t(lay.n_b), {});
  for (idx b = 0; b < M.nbus; ++b) d.jac[size_t(lay.vv + b)] = {M.vmag_in[size_t(b)]};
  for (idx l = 0; l < M.nbr; ++l) {
    const auto& c = M.br[size_t(l)];
    d.jac[size_t(lay.cff(l))] = {M.vmag_in[size_t(c.from)]};
    d.jac[size_t(lay.ctt(l))] = {M.vmag_in[size_t(c.to)]};
    const auto all = branch_support(M, l);
    for (idx lane : {lay.wc(l), lay.ws(l), lay.sqf(l), lay.sqt(l)}) d.jac[size_t(lane)] = all;
  }
  for (idx g = 0; g < M.ngen; ++g) {
    if (g == M.slack_gen) continue;
    d.jac[size_t(lay.pg + g)] = {M.pgen_in[size_t(g)]};
    d.jac[size_t(lay.pg2 + g)] = {M.pgen_in[size_t(g)]};
  }
  std::vector<idx> sd = {M.vmag_in[size_t(M.ref_bus)]};
  for (const auto* list : {&M.ref_from, &M.ref_to})
    for (idx l : *list)
      for (idx i : branch_support(M, l)) sd.push_back(i);
  for (idx g : M.ref_other_gens) sd.push_back(M.pgen_in[size_t(g)]);
  std::sort(sd.begin(), sd.end());
  sd.erase(std::unique(sd.begin(), sd.end()), sd.end());
  d.jac[size_t(lay.pg + M.slack_gen)] = sd;
  d.jac[size_t(lay.pg2 + M.slack_gen)] = sd;

  d.hess = d.jac;
  for (idx g = 0; g < M.ngen; ++g)
    if (g != M.slack_gen) d.hess[size_t(lay.pg + g)].clear();
  // the slack lane is linear in the other reference-bus generators
  auto& sl = d.hess[size_t(lay.pg + M.slack_gen)];
  std::vector<idx> keep;
  for (idx i : sl) {
    bool other = false;
    for (idx g : M.ref_other_gens) other |= M.pgen_in[size_t(g)] == i;
    if (!other) keep.push_back(i);
  }
  sl = keep;
  return d;
}

CondenseProgram plan_condense_program(const Csr& W, const Csr& A, const Csr& B) {
  if (W.rows != A.cols || W.cols != B.cols || A.rows != B.rows)
    throw Error(kInvalidArgument, "condense plan: shapes not conformable");
  std::vector<std::pair<idx, idx>> coords;
  for (idx i = 0; i < W.rows; ++i)
    for (idx k = W.ptr[size_t(i)]; k < W.ptr[size_t(i) + 1]; ++k) coords.push_back({i, W.ind[size_t(k)]});
  for (idx r = 0; r < A.rows; ++r)
    for (idx ka = A.ptr[size_t(r)]; ka < A.ptr[size_t(r) + 1]; ++ka)
      for (idx kb = B.ptr[size_t(r)]; kb < B.ptr[size_t(r) + 1]; ++kb)
        coords.push_back({A.ind[size_t(ka)], B.ind[size_t(kb)]});
  CondenseProgram p;
  p.out = Csr::pattern(W.rows, W.cols, std::move(coords));
  const idx no = p.out.nnz();
  p.w_of.assign(size_t(no), -1);
  for (idx i = 0; i < W.rows; ++i)
    for (idx k = W.ptr[size_t(i)]; k < W.ptr[size_t(i) + 1]; ++k)
      p.w_of[size_t(p.out.find(i, W.ind[size_t(k)]))] = k;
  // triples grouped by output slot, keeping the (r, ka, kb) loop order
  std::vector<idx> cnt(size_t(no) + 1, 0);
  struct T { idx ka, kb, r, slot; };
  std::vector<T> all;
  for (idx r = 0; r < A.rows; ++r)
    for (idx ka = A.ptr[size_t(r)]; ka < A.ptr[size_t(r) + 1]; ++ka)
      for (idx kb = B.ptr[size_t(r)]; kb < B.ptr[size_t(r) + 1]; ++kb) {
        const idx s = p.out.find(A.ind[size_t(ka)], B.ind[size_t(kb)]);
        all.push_back({ka, kb, r, s});
        ++cnt[size_t(s) + 1];
      }
  for (idx s = 0; s < no; ++s) cnt[size_t(s) + 1] += cnt[size_t(s)];
  p.ptr = cnt;
  p.ka.resize(all.size());
  p.kb.resize(all.size());
  p.r.resize(all.size());
  std::vector<idx> fill(cnt.begin(), cnt.end() - 1);
  for (const T& t : all) {
    const idx pos = fill[size_t(t.slot)]++;
    p.ka[size_t(pos)] = t.ka;
    p.kb[size_t(pos)] = t.kb;
    p.r[size_t(pos)] = t.r;
  }
  return p;
}

DerivPlan make_deriv_plan(const OpfModel& M, const LaneDeps& deps) {
  DerivPlan P;
  const idx n_d = M.n_d();
  auto jac_of = [&](const Csr& L) {
    std::vector<std::pair<idx, idx>> c;
    for (idx i = 0; i < L.rows; ++i)
      for (idx e = L.ptr[size_t(i)]; e < L.ptr[size_t(i) + 1]; ++e)
        for (idx d : deps.jac[size_t(L.ind[size_t(e)])]) c.push_back({i, d});
    return Csr::pattern(L.rows, n_d, std::move(c));
  };
  P.jac_g = jac_of(M.L_g);
  P.jac_h = jac_of(M.L_h);
  std::vector<char> used(size_t(M.n_b()), 0);
  for (const Csr* L : {&M.L_f, &M.L_g, &M.L_h})
    for (idx j : L->ind) used[size_t(j)] = 1;
  std::vector<std::pair<idx, idx>> hc;
  for (idx j = 0; j < M.n_b(); ++j)
    if (used[size_t(j)])
      for (idx a : deps.hess[size_t(j)])
        for (idx b : deps.hess[size_t(j)]) hc.push_back({a, b});
  P.hess = Csr::pattern(n_d, n_d, std::move(hc));

  P.g = split_columns(P.jac_g, M.n_x);
  P.h = split_columns(P.jac_h, M.n_x);
  {
    const idx nx = M.n_x, nu = M.n_u;
    std::vector<std::pair<idx, idx>> xx, xu, uu;
    const Csr& H = P.hess;
    for (idx i = 0; i < H.rows; ++i)
      for (idx k = H.ptr[size_t(i)]; k < H.ptr[size_t(i) + 1]; ++k) {
        const idx c = H.ind[size_t(k)];
        if (i < nx && c < nx) xx.push_back({i, c});
        if (i < nx && c >= nx) xu.push_back({i, c - nx});
        if (i >= nx && c >= nx) uu.push_back({i - nx, c - nx});
      }
    P.wxx = Csr::pattern(nx, nx, xx);
    P.wxu = Csr::pattern(nx, nu, xu);
    P.wuu = Csr::pattern(nu, nu, uu);
    P.wxx_src.assign(size_t(P.wxx.nnz()), -1);
    P.wxu_src.assign(size_t(P.wxu.nnz()), -1);
    P.wuu_src.assign(size_t(P.wuu.nnz()), -1);
    for (idx i = 0; i < H.rows; ++i)
      for (idx k = H.ptr[size_t(i)]; k < H.ptr[size_t(i) + 1]; ++k) {
        const idx c = H.ind[size_t(k)];
        if (i < nx && c < nx) P.wxx_src[size_t(P.wxx.find(i, c))] = k;
        if (i < nx && c >= nx) P.wxu_src[size_t(P.wxu.find(i, c - nx))] = k;
        if (i >= nx && c >= nx) P.wuu_src[size_t(P.wuu.find(i - nx, c - nx))] = k;
      }
  }
  P.kxx = plan_condense_program(P.wxx, P.h.x, P.h.x);
  P.kxu = plan_condense_program(P.wxu, P.h.x, P.h.u);
  P.kuu = plan_condense_program(P.wuu, P.h.u, P.h.u);
  return P;
}

// Exact minimum degree on the elimination graph of a symmetric pattern;
// ties go to the lowest index, so the order is deterministic.
std::vector<idx> min_degree_order(const Csr& S) {
  const idx n = S.rows;
  std::vector<std::vector<idx>> nbr(static_cast<size_t>(n));
  for (idx i = 0; i < n; ++i)
    for (idx k = S.ptr[size_t(i)]; k < S.ptr[size_t(i) + 1]; ++k) {
      const idx j = S.ind[size_t(k)];
      if (j == i) continue;
      nbr[size_t(i)].push_back(j);
      nbr[size_t(j)].push_back(i);
    }
  for (auto& v : nbr) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  std::set<std::pair<idx, idx>> heap;
  for (idx i = 0; i < n; ++i) heap.insert({idx(nbr[size_t(i)].size()), i});
  std::vector<char> done(static_cast<size_t>(n), 0);
  std::vector<idx> order, merged;
  order.reserve(size_t(n));
  while (!heap.empty()) {
    const idx v = heap.begin()->second;
    heap.erase(heap.begin());
    done[size_t(v)] = 1;
    order.push_back(v);
    const std::vector<idx> clique = std::move(nbr[size_t(v)]);
    for (idx u : clique) {
      auto& nu = nbr[size_t(u)];
      heap.erase({idx(nu.size()), u});
      merged.clear();
      std::set_union(nu.begin(), nu.end(), clique.begin(), clique.end(),
                     std::back_inserter(merged));
      nu.clear();
      for (idx w : merged)
        if (w != u && !done[size_t(w)]) nu.push_back(w);
      heap.insert({idx(nu.size()), u});
    }
  }
  return order;
}

namespace {

// symbolic factorisation of B = P A P' by row subtrees of the etree: the
// sorted strict-lower column pattern of every row
std::vector<std::vector<idx>> symbolic_rows(const Csr& A, const std::vector<idx>& perm,
                                            const std::vector<idx>& iperm) {
  const idx n = A.rows;
  std::vector<std::vector<idx>> lrow(static_cast<size_t>(n));
  std::vector<idx> parent(size_t(n), -1), mark(size_t(n), -1);
  for (idx i = 0; i < n; ++i) {
    mark[size_t(i)] = i;
    const idx oi = perm[size_t(i)];
    for (idx k = A.ptr[size_t(oi)]; k < A.ptr[size_t(oi) + 1]; ++k) {
      idx j = iperm[size_t(A.ind[size_t(k)])];
      if (j >= i) continue;
      while (mark[size_t(j)] != i) {
        lrow[size_t(i)].push_back(j);
        mark[size_t(j)] = i;
        if (parent[size_t(j)] < 0) parent[size_t(j)] = i;
        j = parent[size_t(j)];
      }
    }
    std::sort(lrow[size_t(i)].begin(), lrow[size_t(i)].end());
  }
  return lrow;
}

// Dense tail: the rows of the top forward levels of the elimination tree,
// from the first level after which every level holds at most `width` rows,
// capped at `max_rows`.  The set is closed under etree ancestors (levels grow
// towards the root), so moving it to the end of the order keeps the fill.
// Each level it absorbs is one dependent step less in every triangular sweep;
// its cost is the dense W = (L_TT U_TT)^{-1} product.
std::vector<char> choose_tail_rows(const std::vector<std::vector<idx>>& lrow, idx width,
                                   idx max_rows) {
  const idx n = idx(lrow.size());
  std::vector<idx> fl(size_t(n), 0);
  idx nlev = 0;
  for (idx i = 0; i < n; ++i) {
    idx lv = 0;
    for (idx j : lrow[size_t(i)]) lv = std::max(lv, fl[size_t(j)] + 1);
    fl[size_t(i)] = lv;
    nlev = std::max(nlev, lv + 1);
  }
  std::vector<idx> cnt(size_t(nlev) + 1, 0);
  for (idx v : fl) ++cnt[size_t(v)];
  idx ls = nlev, rows = 0;
  for (idx l = nlev - 1; l >= 0; --l) {
    if (cnt[size_t(l)] > width || rows + cnt[size_t(l)] > max_rows) break;
    rows += cnt[size_t(l)];
    ls = l;
  }
  std::vector<char> tail(size_t(n), 0);
  if (rows < 8) return tail;
  for (idx i = 0; i < n; ++i) tail[size_t(i)] = fl[size_t(i)] >= ls;
  return tail;
}

}  // namespace

void build_sweeps(LuPlan& P, const std::vector<std::vector<idx>>& lrow,
                  const std::vector<std::vector<idx>>& urow, const std::vector<idx>& fl) {
  const idx n = P.n;
  (void)fl;
  P.tl = n - P.t0;
  const idx t0 = P.t0;
  // --- CSR layouts with direct value indexing
  SweepPlan& L = P.sL;
  SweepPlan& U = P.sU;
  SweepPlan& Ut = P.sUt;
  SweepPlan& Lt = P.sLt;
  L.has_diag = false, L.forward = true;
  U.has_diag = true, U.forward = false;
  Ut.has_diag = true, Ut.forward = true;
  Lt.has_diag = false, Lt.forward = false;
  for (SweepPlan* S : {&L, &U, &Ut, &Lt}) S->ptr.assign(1, 0);
  for (idx i = 0; i < n; ++i) {
    for (idx j : lrow[size_t(i)]) L.col.push_back(j);  // F[t] for t < nnz_l
    L.ptr.push_back(idx(L.col.size()));
    U.col.push_back(i);  // diag first; F[nnz_l + t]
    for (idx c : urow[size_t(i)]) U.col.push_back(c);
    U.ptr.push_back(idx(U.col.size()));
  }
  // FT: U' rows then L' rows
  P.ft_src.clear();
  auto u_slot_of = [&](idx r, idx c) {
    if (r == c) return P.diag[size_t(r)];
    const auto b = P.u_col.begin() + P.u_ptr[size_t(r)], e = P.u_col.begin() + P.u_ptr[size_t(r) + 1];
    return P.u_slot[size_t(std::lower_bound(b, e, c) - P.u_col.begin())];
  };
  auto l_slot_of = [&](idx r, idx c) {
    const auto b = P.l_col.begin() + P.l_ptr[size_t(r)], e = P.l_col.begin() + P.l_ptr[size_t(r) + 1];
    return idx(std::lower_bound(b, e, c) - P.l_col.begin());
  };
  for (idx i = 0; i < n; ++i) {
    Ut.col.push_back(i);
    P.ft_src.push_back(P.diag[size_t(i)]);
    for (idx k : lrow[size_t(i)]) {  // U(k, i), k < i
      Ut.col.push_back(k);
      P.ft_src.push_back(u_slot_of(k, i));
    }
    Ut.ptr.push_back(idx(Ut.col.size()));
  }
  for (idx i = 0; i < n; ++i) {
    for (idx r : urow[size_t(i)]) {  // L(r, i), r > i
      Lt.col.push_back(r);
      P.ft_src.push_back(l_slot_of(r, i));
    }
    Lt.ptr.push_back(idx(Lt.col.size()));
  }
  // --- level schedules over the non-tail rows
  std::vector<idx> lev(size_t(n), 0);
  auto fill_items = [&](SweepPlan& S, const std::vector<std::vector<idx>>& dep, bool forward) {
    std::fill(lev.begin(), lev.end(), -1);
    idx nlev = 0;
    if (forward) {
      for (idx i = 0; i < t0; ++i) {
        idx v = 0;
        for (idx j : dep[size_t(i)])
          if (j < t0) v = std::max(v, lev[size_t(j)] + 1);
        lev[size_t(i)] = v;
        nlev = std::max(nlev, v + 1);
      }
    } else {
      for (idx i = t0 - 1; i >= 0; --i) {
        idx v = 0;
        for (idx j : dep[size_t(i)])
          if (j < t0) v = std::max(v, lev[size_t(j)] + 1);
        lev[size_t(i)] = v;
        nlev = std::max(nlev, v + 1);
      }
    }
    std::vector<std::vector<idx>> by(static_cast<size_t>(nlev));
    for (idx i = 0; i < t0; ++i) by[size_t(lev[size_t(i)])].push_back(i);
    S.lvl_ptr.assign(1, 0);
    S.items.clear();
    for (const auto& rows : by) {
      for (idx r : rows) {
        S.items.insert(S.items.end(), {r, S.ptr[size_t(r)], S.ptr[size_t(r) + 1], 0});
      }
      S.lvl_ptr.push_back(idx(S.items.size() / 4));
    }
    S.tail_items.clear();
    if (forward)
      for (idx r = t0; r < n; ++r) {
        idx split = S.ptr[size_t(r)] + (S.has_diag ? 1 : 0);
        while (split < S.ptr[size_t(r) + 1] && S.col[size_t(split)] < t0) ++split;
        S.tail_items.insert(S.tail_items.end(), {r, S.ptr[size_t(r)], split, 0});
      }
  };
  fill_items(L, lrow, true);
  fill_items(U, urow, false);
  fill_items(Ut, lrow, true);
  fill_items(Lt, urow, false);
  // --- dense tail blocks (column-major tl x tl)
  const idx tl = P.tl;
  for (auto& v : P.dense_src) v.assign(size_t(tl) * size_t(tl), -1);
  for (idx a = 0; a < tl; ++a)
    for (idx b = 0; b < tl; ++b) {
      const idx r = t0 + a, c = t0 + b;  // entry (r, c) of the tail block
      idx lslot = -1, uslot = -1;
      if (r > c) {
        const auto& lr = lrow[size_t(r)];
        if (std::binary_search(lr.begin(), lr.end(), c)) lslot = l_slot_of(r, c);
      } else {
        const auto& ur = urow[size_t(r)];
        if (r == c || std::binary_search(ur.begin(), ur.end(), c)) uslot = u_slot_of(r, c);
      }
      // column-major position of (a, b) is b * tl + a
      P.dense_src[0][size_t(b) * tl + a] = lslot;  // L_TT
      P.dense_src[1][size_t(b) * tl + a] = uslot;  // U_TT
    }
}

LuPlan make_lu_plan(const Csr& A) {
  if (A.rows != A.cols) throw Error(kInvalidArgument, "lu plan: matrix not square");
  const idx n = A.rows;
  // structural symmetry is what makes one static symmetric ordering valid
  for (idx i = 0; i < n; ++i) {
    if (A.find(i, i) < 0) throw Error(kSingularBlock, "lu plan: structurally zero diagonal");
    for (idx k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k)
      if (A.find(A.ind[size_t(k)], i) < 0)
        throw Error(kUnsupported, "lu plan: G_x pattern is not structurally symmetric");
  }
  LuPlan P;
  P.n = n;
  P.perm = min_degree_order(A);
  P.iperm.assign(size_t(n), 0);
  for (idx k = 0; k < n; ++k) P.iperm[size_t(P.perm[size_t(k)])] = k;
  std::vector<std::vector<idx>> lrow = symbolic_rows(A, P.perm, P.iperm);
  // dense tail: move the top levels of the etree to the end of the order
  // (same elimination tree, same fill) and redo the symbolic pass
  {
    // large grids (n >= kWideTailN): the wide tail (measured, round 2, with the
    // presolved reduction: 9241/16 345 -> 300 ms and 2869/64 40.5 -> 35.6 ms per
    // reduction + refactor; at 1354 the tl^3 Gauss-Jordan outgrows the gain)
    idx width = n >= kWideTailN ? 32 : kTailWidth, max_rows = n >= kWideTailN ? kMaxTailLimit : kMaxTail;
    if (const char* e = std::getenv("BIPM_TAIL_WIDTH")) width = std::atoi(e);
    if (const char* e = std::getenv("BIPM_TAIL_MAX"))
      max_rows = std::max<idx>(0, std::min<idx>(kMaxTailLimit, std::atoi(e)));
    const std::vector<char> tail = choose_tail_rows(lrow, width, max_rows);
    std::vector<idx> perm2;
    perm2.reserve(size_t(n));
    for (idx k = 0; k < n; ++k)
      if (!tail[size_t(k)]) perm2.push_back(P.perm[size_t(k)]);
    P.t0 = idx(perm2.size());
    for (idx k = 0; k < n; ++k)
      if (tail[size_t(k)]) perm2.push_back(P.perm[size_t(k)]);
    if (perm2 != P.perm) {
      P.perm = perm2;
      for (idx k = 0; k < n; ++k) P.iperm[size_t(P.perm[size_t(k)])] = k;
      lrow = symbolic_rows(A, P.perm, P.iperm);
    }
  }
  // U strict upper rows = transpose of the L pattern
  std::vector<std::vector<idx>> urow(static_cast<size_t>(n));
  for (idx r = 0; r < n; ++r)
    for (idx j : lrow[size_t(r)]) urow[size_t(j)].push_back(r);  // ascending r

  P.l_ptr.assign(1, 0);
  for (idx i = 0; i < n; ++i) {
    for (idx j : lrow[size_t(i)]) {
      P.l_col.push_back(j);
      P.l_slot.push_back(idx(P.l_slot.size()));
    }
    P.l_ptr.push_back(idx(P.l_col.size()));
  }
  P.nnz_l = idx(P.l_col.size());
  idx next = P.nnz_l;
  P.u_ptr.assign(1, 0);
  P.diag.assign(size_t(n), -1);
  for (idx i = 0; i < n; ++i) {
    P.diag[size_t(i)] = next++;
    for (idx c : urow[size_t(i)]) {
      P.u_col.push_back(c);
      P.u_slot.push_back(next++);
    }
    P.u_ptr.push_back(idx(P.u_col.size()));
  }
  P.nnz_f = next;
  // slot lookup helpers
  auto l_slot_of = [&](idx r, idx c) {  // r > c
    const auto b = P.l_col.begin() + P.l_ptr[size_t(r)], e = P.l_col.begin() + P.l_ptr[size_t(r) + 1];
    auto it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? idx(it - P.l_col.begin()) : -1;
  };
  auto u_slot_of = [&](idx r, idx c) {  // r <= c
    if (r == c) return P.diag[size_t(r)];
    const auto b = P.u_col.begin() + P.u_ptr[size_t(r)], e = P.u_col.begin() + P.u_ptr[size_t(r) + 1];
    auto it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? P.u_slot[size_t(it - P.u_col.begin())] : idx(-1);
  };
  // column access for the transposed sweeps
  P.ut_ptr.assign(1, 0);
  P.lt_ptr.assign(1, 0);
  for (idx i = 0; i < n; ++i) {
    for (idx k : lrow[size_t(i)]) {  // U(k, i), k < i
      P.ut_row.push_back(k);
      P.ut_slot.push_back(u_slot_of(k, i));
    }
    P.ut_ptr.push_back(idx(P.ut_row.size()));
    for (idx r : urow[size_t(i)]) {  // L(r, i), r > i
      P.lt_row.push_back(r);
      P.lt_slot.push_back(l_slot_of(r, i));
    }
    P.lt_ptr.push_back(idx(P.lt_row.size()));
  }
  // level schedules
  std::vector<idx> fl(size_t(n), 0), bl(size_t(n), 0);
  idx nf = 0, nbk = 0;
  for (idx i = 0; i < n; ++i) {
    idx lv = 0;
    for (idx j : lrow[size_t(i)]) lv = std::max(lv, fl[size_t(j)] + 1);
    fl[size_t(i)] = lv;
    nf = std::max(nf, lv + 1);
  }
  for (idx i = n - 1; i >= 0; --i) {
    idx lv = 0;
    for (idx j : urow[size_t(i)]) lv = std::max(lv, bl[size_t(j)] + 1);
    bl[size_t(i)] = lv;
    nbk = std::max(nbk, lv + 1);
  }
  auto bucket = [&](const std::vector<idx>& lev, idx nlev, std::vector<idx>& ptr,
                    std::vector<idx>& rows) {
    ptr.assign(size_t(nlev) + 1, 0);
    for (idx i = 0; i < n; ++i) ++ptr[size_t(lev[size_t(i)]) + 1];
    for (idx l = 0; l < nlev; ++l) ptr[size_t(l) + 1] += ptr[size_t(l)];
    rows.assign(size_t(n), 0);
    std::vector<idx> fill(ptr.begin(), ptr.end() - 1);
    for (idx i = 0; i < n; ++i) rows[size_t(fill[size_t(lev[size_t(i)])]++)] = i;
  };
  bucket(fl, nf, P.fwd_ptr, P.fwd_rows);
  bucket(bl, nbk, P.bwd_ptr, P.bwd_rows);

  // G_x slot -> factor slot
  P.a_src.assign(size_t(P.nnz_f), -1);
  for (idx i = 0; i < n; ++i)
    for (idx k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k) {
      const idx pi = P.iperm[size_t(i)], pj = P.iperm[size_t(A.ind[size_t(k)])];
      const idx s = pi > pj ? l_slot_of(pi, pj) : u_slot_of(pi, pj);
      P.a_src[size_t(s)] = k;
    }
  // Crout refactor program, level by level
  P.piv_of.assign(size_t(P.nnz_f), -1);
  P.mul_ptr.assign(size_t(P.nnz_f) + 1, 0);
  std::vector<std::vector<std::pair<idx, idx>>> prog(static_cast<size_t>(P.nnz_f));
  for (idx j = 0; j < n; ++j) {
    const auto& Lj = lrow[size_t(j)];
    // U(j, c) for c = j and c in urow(j): sum over k in Lrow(j) n Lrow(c)
    auto u_entry = [&](idx c, idx slot) {
      const auto& Lc = lrow[size_t(c)];
      intersect(Lj.data(), idx(Lj.size()), Lc.data(), idx(Lc.size()), [&](idx pa, idx) {
        const idx k = Lj[size_t(pa)];
        prog[size_t(slot)].push_back({P.l_ptr[size_t(j)] + pa, u_slot_of(k, c)});
      });
    };
    u_entry(j, P.diag[size_t(j)]);
    for (idx t = P.u_ptr[size_t(j)]; t < P.u_ptr[size_t(j) + 1]; ++t)
      u_entry(P.u_col[size_t(t)], P.u_slot[size_t(t)]);
    // L(r, j) for r in urow(j): sum over k in Lrow(r) n Lrow(j)
    for (idx r : urow[size_t(j)]) {
      const idx slot = l_slot_of(r, j);
      P.piv_of[size_t(slot)] = P.diag[size_t(j)];
      const auto& Lr = lrow[size_t(r)];
      intersect(Lr.data(), idx(Lr.size()), Lj.data(), idx(Lj.size()), [&](idx pa, idx pb) {
        const idx k = Lj[size_t(pb)];
        prog[size_t(slot)].push_back({P.l_ptr[size_t(r)] + pa, u_slot_of(k, j)});
      });
    }
  }
  for (idx s = 0; s < P.nnz_f; ++s) P.mul_ptr[size_t(s) + 1] = P.mul_ptr[size_t(s)] + idx(prog[size_t(s)].size());
  P.mul_l.reserve(size_t(P.mul_ptr.back()));
  P.mul_u.reserve(size_t(P.mul_ptr.back()));
  for (idx s = 0; s < P.nnz_f; ++s)
    for (auto [a, b] : prog[size_t(s)]) {
      P.mul_l.push_back(a);
      P.mul_u.push_back(b);
    }
  build_sweeps(P, lrow, urow, fl);
  P.lvl_u_ptr.assign(1, 0);
  P.lvl_l_ptr.assign(1, 0);
  for (idx l = 0; l < nf; ++l) {
    for (idx t = P.fwd_ptr[size_t(l)]; t < P.fwd_ptr[size_t(l) + 1]; ++t) {
      const idx j = P.fwd_rows[size_t(t)];
      P.lvl_u_slot.push_back(P.diag[size_t(j)]);
      for (idx q = P.u_ptr[size_t(j)]; q < P.u_ptr[size_t(j) + 1]; ++q)
        P.lvl_u_slot.push_back(P.u_slot[size_t(q)]);
      for (idx r : urow[size_t(j)]) P.lvl_l_slot.push_back(l_slot_of(r, j));
    }
    P.lvl_u_ptr.push_back(idx(P.lvl_u_slot.size()));
    P.lvl_l_ptr.push_back(idx(P.lvl_l_slot.size()));
  }
  // split at the dense tail
  const idx t0 = P.t0;
  P.nt_lvl_u_ptr.assign(1, 0);
  P.nt_lvl_l_ptr.assign(1, 0);
  for (idx l = 0; l < nf; ++l) {
    bool any = false;
    for (idx t = P.fwd_ptr[size_t(l)]; t < P.fwd_ptr[size_t(l) + 1]; ++t) {
      const idx j = P.fwd_rows[size_t(t)];
      if (j >= t0) continue;
      any = true;
      P.nt_lvl_u_slot.push_back(P.diag[size_t(j)]);
      for (idx q = P.u_ptr[size_t(j)]; q < P.u_ptr[size_t(j) + 1]; ++q)
        P.nt_lvl_u_slot.push_back(P.u_slot[size_t(q)]);
      for (idx r : urow[size_t(j)]) P.nt_lvl_l_slot.push_back(l_slot_of(r, j));
    }
    if (!any) continue;
    P.nt_lvl_u_ptr.push_back(idx(P.nt_lvl_u_slot.size()));
    P.nt_lvl_l_ptr.push_back(idx(P.nt_lvl_l_slot.size()));
  }
  P.tail_mul_ptr.assign(1, 0);
  auto add_tail = [&](idx slot) {
    P.tail_slot.push_back(slot);
    for (idx t = P.mul_ptr[size_t(slot)]; t < P.mul_ptr[size_t(slot) + 1]; ++t)
      if (P.l_col[size_t(P.mul_l[size_t(t)])] < t0) {
        P.tail_mul_l.push_back(P.mul_l[size_t(t)]);
        P.tail_mul_u.push_back(P.mul_u[size_t(t)]);
      }
    P.tail_mul_ptr.push_back(idx(P.tail_mul_l.size()));
  };
  for (idx i = t0; i < n; ++i) {
    for (idx q = P.l_ptr[size_t(i)]; q < P.l_ptr[size_t(i) + 1]; ++q)
      if (P.l_col[size_t(q)] >= t0) add_tail(q);  // L(i, j), t0 <= j < i
    add_tail(P.diag[size_t(i)]);
    for (idx q = P.u_ptr[size_t(i)]; q < P.u_ptr[size_t(i) + 1]; ++q) add_tail(P.u_slot[size_t(q)]);
  }
  // flattened phases
  P.rf_phase_ptr.assign(1, 0);
  auto rec = [&](idx slot, idx mb, idx me, bool divide) {
    P.rf_rec.insert(P.rf_rec.end(), {slot, idx(P.rf_pair.size() / 2) + 0, 0, P.a_src[size_t(slot)]});
    const size_t at = P.rf_rec.size() - 4;
    for (idx t = mb; t < me; ++t) P.rf_pair.insert(P.rf_pair.end(), {P.mul_l[size_t(t)], P.mul_u[size_t(t)]});
    P.rf_rec[at + 2] = idx(P.rf_pair.size() / 2);
    P.rf_piv.push_back(divide ? P.piv_of[size_t(slot)] : -1);
  };
  for (size_t lv = 0; lv + 1 < P.nt_lvl_u_ptr.size(); ++lv) {
    for (idx q = P.nt_lvl_u_ptr[lv]; q < P.nt_lvl_u_ptr[lv + 1]; ++q) {
      const idx slot = P.nt_lvl_u_slot[size_t(q)];
      rec(slot, P.mul_ptr[size_t(slot)], P.mul_ptr[size_t(slot) + 1], false);
    }
    P.rf_phase_ptr.push_back(idx(P.rf_piv.size()));
    for (idx q = P.nt_lvl_l_ptr[lv]; q < P.nt_lvl_l_ptr[lv + 1]; ++q) {
      const idx slot = P.nt_lvl_l_slot[size_t(q)];
      rec(slot, P.mul_ptr[size_t(slot)], P.mul_ptr[size_t(slot) + 1], true);
    }
    P.rf_phase_ptr.push_back(idx(P.rf_piv.size()));
  }
  for (size_t it = 0; it < P.tail_slot.size(); ++it) {
    const idx slot = P.tail_slot[it];
    P.rf_rec.insert(P.rf_rec.end(), {slot, idx(P.rf_pair.size() / 2), 0, P.a_src[size_t(slot)]});
    for (idx t = P.tail_mul_ptr[it]; t < P.tail_mul_ptr[it + 1]; ++t)
      P.rf_pair.insert(P.rf_pair.end(), {P.tail_mul_l[size_t(t)], P.tail_mul_u[size_t(t)]});
    P.rf_rec[P.rf_rec.size() - 2] = idx(P.rf_pair.size() / 2);
    P.rf_piv.push_back(-1);
  }
  if (!P.tail_slot.empty()) P.rf_phase_ptr.push_back(idx(P.rf_piv.size()));
  return P;
}

}  // namespace bipm
