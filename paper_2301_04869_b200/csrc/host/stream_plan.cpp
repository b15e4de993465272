#include "stream_plan.hpp"

#include <stdexcept>

#include <algorithm>
#include <cstdlib>
#include <queue>

namespace bipm {

namespace {

int round16(int bytes) { return (bytes + 15) & ~15; }
int val_alloc(int count) { return count > 0 ? round16((count + 1) * 8) : 0; }

struct Builder {
  StreamProgram& S;
  const int max_bytes;
  std::vector<int> group;  // row -> warp of its subtree (-1: team levels); empty: none
  int warp_rr = 0;  // round-robin position of the next unit chunk (all-warp steps)
  int last_team = 16;  // reset to the all-consumer team (consumers / 32) by build_stream_program
  struct Pending {
    int kind, flags, aux0, aux1;
    std::vector<int> items;  // 4 ints per item
    std::vector<int> col;
    int val_arr = -1, val_off = 0, val_count = 0;
    int x_arr = -1, x_off = 0, x_count = 0;
    std::vector<int> levels;  // sweep steps: 4 ints per level (unit_begin, unit_end, lg, barrier)
    std::vector<int> dir;     // warp-local sweeps: level range per consumer warp
  };

  // column entries are 16-bit panel rows, padded to 16 bytes
  static int pat_bytes(int n_items, int n_ent, int n_lev = 0, int dir_ints = 0) {
    return 4 * kStepHeaderInts + round16(4 * dir_ints) + 16 * n_lev + 16 * n_items +
           2 * ((n_ent + 7) & ~7);
  }
  // lanes per work unit: all units in one pass of `lanes` threads, and at
  // least ~3 entries per lane
  static int lanes_log2(int units, int max_ent, int lanes) {
    static const int per_lane = [] {
      const char* e = std::getenv("BIPM_LANE_ENT");
      return e ? std::max(1, std::atoi(e)) : 3;
    }();
    int lg = 0;
    while (lg < 5 && units * (2 << lg) <= lanes && (2 << lg) * per_lane <= max_ent) ++lg;
    return lg;
  }
  static int step_bytes(int n_items, int n_ent, int vcount, int xcount, int n_lev = 0) {
    return pat_bytes(n_items, n_ent, n_lev) + val_alloc(vcount) + val_alloc(xcount);
  }

  void emit(Pending p) {
    const int K = S.K, NG = K > kStreamUnitCols ? K / kStreamUnitCols : 1;
    const int n_items = int(p.items.size() / 4);
    const int n_lev = int(p.levels.size() / 4);
    const int n_col = (int(p.col.size()) + 7) & ~7;  // 16-bit entries
    StepIssue is{};
    is.pat_off = int(S.pat.size());
    is.pat_bytes = pat_bytes(n_items, int(p.col.size()), n_lev, int(p.dir.size()));
    const int par = (p.val_count > 0 ? ((p.val_off & 1) | (int(S.stride[p.val_arr] & 1) << 1)) : 0) |
                    (p.x_count > 0 ? (((p.x_off & 1) << 2) | (int(S.stride[p.x_arr] & 1) << 3)) : 0);
    // work units and lanes of the all-warp steps; rows become panel words
    int units = 0, lg = 0, max_ent = 0;
    for (int it = 0; it < n_items; ++it)
      max_ent = std::max(max_ent, p.items[size_t(it) * 4 + 2] - p.items[size_t(it) * 4 + 1]);
    if (p.kind == kStepSpmv) {
      units = n_items * NG;
      static const int spmv_lanes = [] {
        const char* e = std::getenv("BIPM_SPMV_LANES");
        return e ? std::max(32, std::atoi(e)) : 0;
      }();
      lg = lanes_log2(units, max_ent, spmv_lanes > 0 ? spmv_lanes : S.consumers);
    } else if (p.kind == kStepDense) {
      units = p.aux1 * NG;
      lg = lanes_log2(units, p.val_count / std::max(1, p.aux1), S.consumers);
    }
    if (p.kind == kStepSweep || p.kind == kStepSweepW || p.kind == kStepSpmv)
      for (int it = 0; it < n_items; ++it)
        p.items[size_t(it) * 4] = panel_word(p.items[size_t(it) * 4], K);
    // column entries are 16 bits: the panel word / 16 for K >= 2 (the word of
    // row r is a multiple of 16; r K / 2 + sw(r) < 2^16 whenever the panel
    // fits in shared memory), the panel row for K = 1 (word = 8 r)
    for (int& c : p.col) {
      if (c < 0) throw std::runtime_error("stream program: negative panel row");
      if (K >= 2) c = panel_word(c, K) >> 4;
      if (c > 0xffff) throw std::runtime_error("stream program: column entry exceeds 16 bits");
    }
    const int warp0 = warp_rr;
    if (units > 0) {
      const int upw = 32 >> lg;
      warp_rr = (warp_rr + (units + upw - 1) / upw) % (S.consumers / 32);
    }
    int hdr[kStepHeaderInts] = {p.kind, p.flags, n_items, n_col, p.aux0, p.aux1, p.val_count,
                                par, lg, units, warp0, n_lev};
    S.pat.insert(S.pat.end(), hdr, hdr + kStepHeaderInts);
    if (!p.dir.empty()) {
      S.pat.insert(S.pat.end(), p.dir.begin(), p.dir.end());
      while (S.pat.size() & 3) S.pat.push_back(0);  // 16-byte alignment
    }
    S.pat.insert(S.pat.end(), p.levels.begin(), p.levels.end());
    S.pat.insert(S.pat.end(), p.items.begin(), p.items.end());
    for (int i = 0; i < n_col; i += 2) {
      const int c0 = i < int(p.col.size()) ? p.col[size_t(i)] : 0;
      const int c1 = i + 1 < int(p.col.size()) ? p.col[size_t(i) + 1] : 0;
      S.pat.push_back(int(unsigned(c0) | (unsigned(c1) << 16)));
    }
    is.val_arr = p.val_count > 0 ? p.val_arr : 0;
    is.val_off = p.val_off;
    is.val_count = p.val_count;
    is.x_arr = p.x_count > 0 ? p.x_arr : 0;
    is.x_off = p.x_off;
    is.x_count = p.x_count;
    S.issue.push_back(is);
    S.skip.push_back(p.kind == kStepAcc && n_items > 0
                         ? ((p.aux1 + n_items - 1) << 4) | (p.flags & (kFlagPre | kFlagBarrier))
                         : (0x7ffffff << 4));
  }

  // One triangular sweep (its levels, then optionally the tail gather as one
  // more level).  Each level gets a team: the lowest T warps, T a power of two
  // sized to its units x lanes; consecutive levels with the same team and
  // diagonal mode share a step and are separated by team barriers (named
  // barrier, or __syncwarp for one warp).  Values are appended to VS.
  // pre_t0 >= 0 (backward sweeps U, L', whose tail rows are final before the
  // sweep starts): every row's entries in the tail columns (>= pre_t0, the
  // end of each row) form one independent level ahead of the schedule, so
  // the dependent levels carry only the non-tail entries (1354: half of the
  // U sweep's off-diagonal entries, all of its first level's)
  void sweep(const SweepPlan& sw, const std::vector<idx>& slot_of_t, bool diag, bool with_tail,
             int tail_skip, idx pre_t0 = -1) {
    const int K = S.K, NG = K > kStreamUnitCols ? K / kStreamUnitCols : 1;
    struct Unit { idx row, b, e; };
    std::vector<std::vector<Unit>> levels;
    std::vector<char> level_diag;
    std::vector<Unit> pre;
    const idx nl = idx(sw.lvl_ptr.size()) - 1;
    for (idx l = 0; l < nl; ++l) {
      std::vector<Unit> us;
      for (idx it = sw.lvl_ptr[size_t(l)]; it < sw.lvl_ptr[size_t(l) + 1]; ++it) {
        const idx row = sw.items[size_t(it) * 4], b = sw.items[size_t(it) * 4 + 1];
        idx e = sw.items[size_t(it) * 4 + 2];
        if (pre_t0 >= 0) {
          idx sp = e;
          for (idx t = b + (diag ? 1 : 0); t < e; ++t)
            if (sw.col[size_t(t)] >= pre_t0) {
              sp = t;
              break;
            }
          if (sp < e) pre.push_back({row, sp, e});
          e = sp;
        }
        if (!diag && e <= b) continue;  // nothing to subtract
        us.push_back({row, b, e});
      }
      if (!us.empty()) {
        levels.push_back(std::move(us));
        level_diag.push_back(diag);
      }
    }
    if (!pre.empty()) {
      levels.insert(levels.begin(), std::move(pre));
      level_diag.insert(level_diag.begin(), 0);
    }
    // the subtree rows leave the team levels for the warp-local part: per
    // warp, its rows grouped by level (rows of one level are independent)
    const int nw = S.consumers / 32;
    const size_t nws = static_cast<size_t>(nw);
    std::vector<std::vector<std::vector<Unit>>> wl(nws);
    if (!group.empty()) {
      std::vector<std::vector<Unit>> upper;
      for (auto& us : levels) {
        std::vector<std::vector<Unit>> per(nws);
        std::vector<Unit> up;
        for (const Unit& u : us) {
          const int g = group[size_t(u.row)];
          (g >= 0 ? per[size_t(g)] : up).push_back(u);
        }
        for (int w = 0; w < nw; ++w)
          if (!per[size_t(w)].empty()) wl[size_t(w)].push_back(std::move(per[size_t(w)]));
        if (!up.empty()) upper.push_back(std::move(up));
      }
      levels = std::move(upper);
      level_diag.assign(levels.size(), diag);
    }
    bool any_wl = false;
    for (const auto& v : wl) any_wl = any_wl || !v.empty();
    // forward sweeps (L, U'): the subtrees first, the levels above them after;
    // backward sweeps (U, L'): the other way round
    if (any_wl && sw.forward) warp_local(wl, diag, sw, slot_of_t);
    if (with_tail) {  // the tail rows are independent of each other
      std::vector<Unit> us;
      for (size_t it = 0; it < sw.tail_items.size() / 4; ++it) {
        const idx row = sw.tail_items[it * 4], b = sw.tail_items[it * 4 + 1] + tail_skip,
                  e = sw.tail_items[it * 4 + 2];
        if (e > b) us.push_back({row, b, e});
      }
      if (!us.empty()) {
        levels.push_back(std::move(us));
        level_diag.push_back(false);
      }
    }
    Pending p{kStepSweep, 0, 0, 0, {}, {}};
    std::vector<idx> slots;
    int cur_team = -1;
    bool cur_diag = false;
    auto flush = [&] {
      if (p.items.empty()) return;
      p.flags = (cur_diag ? kFlagDiag : 0) | (cur_team != last_team ? kFlagPre : 0);
      p.aux0 = cur_team;
      last_team = cur_team;
      if (S.vs_src.size() & 1) S.vs_src.push_back(-1);
      p.val_arr = kArrSweep;
      p.val_off = int(S.vs_src.size());
      p.val_count = int(p.col.size());
      S.vs_src.insert(S.vs_src.end(), slots.begin(), slots.end());
      emit(p);
      ++S.n_sweep_steps;
      p.items.clear();
      p.col.clear();
      p.levels.clear();
      slots.clear();
    };
    for (size_t l = 0; l < levels.size(); ++l) {
      const auto& us = levels[l];
      const bool dg = level_diag[l];
      int max_ent = 0;
      for (const Unit& u : us) max_ent = std::max(max_ent, int(u.e - u.b) - (dg ? 1 : 0));
      const int units = int(us.size()) * NG;
      static const int max_lanes = [] {
        const char* e = std::getenv("BIPM_MAX_LANES");
        return e ? std::atoi(e) : 0;
      }();
      int lg = lanes_log2(units, max_ent, max_lanes > 0 ? max_lanes : S.consumers);
      // a level whose units fit one warp runs on that warp alone (no team
      // barrier, __syncwarp between levels): fewer lanes per unit if needed
      static const int solo_max = [] {
        const char* e = std::getenv("BIPM_SOLO_UNITS");
        return e ? std::atoi(e) : 0;
      }();
      if (units <= solo_max)
        while (lg > 0 && units * (1 << lg) > 32) --lg;
      static const int min_team = [] {
        const char* e = std::getenv("BIPM_MIN_TEAM");
        return e ? std::max(1, std::atoi(e)) : 1;
      }();
      int team = min_team;
      while (team < S.consumers / 32 && team * 32 < units * (1 << lg)) team *= 2;
      if (!p.items.empty() && (team != cur_team || dg != cur_diag)) flush();
      cur_team = team;
      cur_diag = dg;
      size_t u = 0;
      while (u < us.size()) {
        // as many of the level's units as fit in this step
        const int ub = int(p.items.size() / 4);
        while (u < us.size()) {
          const int n_new = int(us[u].e - us[u].b);
          if (!p.items.empty() &&
              step_bytes(int(p.items.size() / 4) + 1, int(p.col.size()) + n_new,
                         int(p.col.size()) + n_new, 0, int(p.levels.size() / 4) + 1) > max_bytes)
            break;
          const int beg = int(p.col.size());
          for (idx t = us[u].b; t < us[u].e; ++t) {
            p.col.push_back(sw.col[size_t(t)]);
            slots.push_back(slot_of_t[size_t(t)]);
          }
          p.items.insert(p.items.end(), {us[u].row, beg, int(p.col.size()), 0});
          ++u;
        }
        const int ue = int(p.items.size() / 4);
        if (ue > ub)  // barrier after the level's last part
          p.levels.insert(p.levels.end(), {ub * NG, ue * NG, lg, u == us.size() ? 1 : 0});
        if (u < us.size()) flush();  // the step is full: the level continues in the next
      }
    }
    flush();
    if (any_wl && !sw.forward) warp_local(wl, diag, sw, slot_of_t);
    last_team = S.consumers / 32;  // the steps after a sweep start with an all-consumer barrier
  }

  // Warp-local part of a sweep: kStepSweepW steps, each holding the next
  // levels of every warp (round robin, one level per warp per round, while
  // the step fits).  The first step synchronises all consumers (the rows it
  // reads were written by other warps); the warps then run without barriers.
  template <typename Unit>
  void warp_local(const std::vector<std::vector<std::vector<Unit>>>& wl, bool diag,
                  const SweepPlan& sw, const std::vector<idx>& slot_of_t) {
    const int K = S.K, NG = K > kStreamUnitCols ? K / kStreamUnitCols : 1;
    const int nw = S.consumers / 32;
    std::vector<size_t> pos(size_t(nw), 0);
    bool first = true;
    for (;;) {
      struct WB {
        std::vector<std::vector<int>> lev_items;  // per level: row, local col begin, end
        std::vector<std::vector<int>> lev_col;
        std::vector<std::vector<idx>> lev_slot;
        std::vector<int> lev_lg;
      };
      std::vector<WB> wb(static_cast<size_t>(nw));
      int n_items = 0, n_ent = 0, n_lev = 0;
      for (bool progress = true; progress;) {
        progress = false;
        for (int w = 0; w < nw; ++w) {
          if (pos[size_t(w)] >= wl[size_t(w)].size()) continue;
          const auto& us = wl[size_t(w)][pos[size_t(w)]];
          int ents = 0, max_ent = 0;
          for (const Unit& u : us) {
            ents += int(u.e - u.b);
            max_ent = std::max(max_ent, int(u.e - u.b) - (diag ? 1 : 0));
          }
          const int bytes = pat_bytes(n_items + int(us.size()), n_ent + ents, n_lev + 1, 2 * nw) +
                            val_alloc(n_ent + ents);
          if (n_lev > 0 && bytes > max_bytes) continue;
          WB& b = wb[size_t(w)];
          std::vector<int> it, col;
          std::vector<idx> sl;
          for (const Unit& u : us) {
            const int beg = int(col.size());
            for (idx t = u.b; t < u.e; ++t) {
              col.push_back(sw.col[size_t(t)]);
              sl.push_back(slot_of_t[size_t(t)]);
            }
            it.insert(it.end(), {u.row, beg, int(col.size()), 0});
          }
          b.lev_items.push_back(std::move(it));
          b.lev_col.push_back(std::move(col));
          b.lev_slot.push_back(std::move(sl));
          b.lev_lg.push_back(lanes_log2(int(us.size()) * NG, max_ent, 32));
          ++pos[size_t(w)];
          ++n_lev;
          n_items += int(us.size());
          n_ent += ents;
          progress = true;
        }
      }
      if (n_lev == 0) break;
      Pending p{kStepSweepW, (diag ? kFlagDiag : 0) | (first ? kFlagPre : 0), 0, 0, {}, {}};
      p.dir.assign(size_t(2 * nw), 0);
      std::vector<idx> slots;
      for (int w = 0; w < nw; ++w) {
        const WB& b = wb[size_t(w)];
        p.dir[size_t(2 * w)] = int(p.levels.size() / 4);
        for (size_t L = 0; L < b.lev_items.size(); ++L) {
          const int ub = int(p.items.size() / 4), c0 = int(p.col.size());
          const auto& it = b.lev_items[L];
          for (size_t q = 0; q < it.size(); q += 4)
            p.items.insert(p.items.end(), {it[q], c0 + it[q + 1], c0 + it[q + 2], 0});
          p.col.insert(p.col.end(), b.lev_col[L].begin(), b.lev_col[L].end());
          slots.insert(slots.end(), b.lev_slot[L].begin(), b.lev_slot[L].end());
          const int ue = int(p.items.size() / 4);
          p.levels.insert(p.levels.end(), {ub * NG, ue * NG, b.lev_lg[L], 0});
        }
        p.dir[size_t(2 * w + 1)] = int(p.levels.size() / 4);
      }
      if (S.vs_src.size() & 1) S.vs_src.push_back(-1);
      p.val_arr = kArrSweep;
      p.val_off = int(S.vs_src.size());
      p.val_count = int(p.col.size());
      S.vs_src.insert(S.vs_src.end(), slots.begin(), slots.end());
      emit(p);
      ++S.n_sweep_steps;
      first = false;
    }
    last_team = -1;  // the team levels after the subtrees start with a barrier
  }
};

}  // namespace

std::vector<int> subtree_groups(const LuPlan& L, int nwarps) {
  const idx n = L.n, t0 = L.t0;
  std::vector<int> group(size_t(n), -1);
  if (nwarps <= 0 || t0 <= 0) return group;
  // elimination forest of the non-tail rows: parent(j) = first row i > j with
  // L(i, j) != 0 (rows in the tail end the forest)
  std::vector<idx> parent(size_t(t0), -1);
  for (idx i = 0; i < n; ++i)
    for (idx q = L.l_ptr[size_t(i)]; q < L.l_ptr[size_t(i) + 1]; ++q) {
      const idx j = L.l_col[size_t(q)];
      if (j < t0 && (parent[size_t(j)] < 0 || i < parent[size_t(j)])) parent[size_t(j)] = i;
    }
  const size_t t0s = static_cast<size_t>(t0);
  std::vector<std::vector<idx>> kids(t0s);
  std::vector<idx> roots;
  for (idx j = 0; j < t0; ++j) {
    if (parent[size_t(j)] >= 0 && parent[size_t(j)] < t0)
      kids[size_t(parent[size_t(j)])].push_back(j);
    else
      roots.push_back(j);
  }
  // work of a row: its entries in the four sweeps (L, U each twice) + 1
  std::vector<double> sub(size_t(t0), 0.0);
  double total = 0.0;
  for (idx j = 0; j < t0; ++j) {  // children precede parents
    sub[size_t(j)] += 1.0 + (L.l_ptr[size_t(j) + 1] - L.l_ptr[size_t(j)]) +
                      (L.u_ptr[size_t(j) + 1] - L.u_ptr[size_t(j)]);
    total += 1.0 + (L.l_ptr[size_t(j) + 1] - L.l_ptr[size_t(j)]) +
             (L.u_ptr[size_t(j) + 1] - L.u_ptr[size_t(j)]);
    if (parent[size_t(j)] >= 0 && parent[size_t(j)] < t0) sub[size_t(parent[size_t(j)])] += sub[size_t(j)];
  }
  // split the heaviest subtree (its root joins the team levels) until the
  // pieces are small enough to balance over the warps
  static const double pieces_per_warp = [] {
    const char* e = std::getenv("BIPM_SUBTREE_PIECES");
    return e ? std::max(1.0, std::atof(e)) : 4.0;
  }();
  const double cap = total / (nwarps * pieces_per_warp);
  auto cmp = [&](idx a, idx b) { return sub[size_t(a)] < sub[size_t(b)]; };
  std::priority_queue<idx, std::vector<idx>, decltype(cmp)> heap(cmp);
  for (idx r : roots) heap.push(r);
  std::vector<idx> pieces;
  while (!heap.empty()) {
    const idx r = heap.top();
    heap.pop();
    if (sub[size_t(r)] <= cap || kids[size_t(r)].empty()) {
      pieces.push_back(r);
      continue;
    }
    for (idx c : kids[size_t(r)]) heap.push(c);  // r stays with the team levels
  }
  // longest processing time first onto the least loaded warp
  std::sort(pieces.begin(), pieces.end(),
            [&](idx a, idx b) { return sub[size_t(a)] > sub[size_t(b)]; });
  std::vector<double> load(size_t(nwarps), 0.0);
  std::vector<int> owner(size_t(t0), -1);
  for (idx r : pieces) {
    const int w = int(std::min_element(load.begin(), load.end()) - load.begin());
    load[size_t(w)] += sub[size_t(r)];
    owner[size_t(r)] = w;
  }
  // every row of a piece belongs to the piece root's warp (top-down: parents
  // have larger indices, so walk rows from the top)
  for (idx j = t0 - 1; j >= 0; --j) {
    if (owner[size_t(j)] >= 0) {
      group[size_t(j)] = owner[size_t(j)];
      continue;
    }
    const idx pj = parent[size_t(j)];
    if (pj >= 0 && pj < t0 && group[size_t(pj)] >= 0) group[size_t(j)] = group[size_t(pj)];
  }
  return group;
}

ReachPlan build_reach_plan(const LuPlan& L, const Csr& gu, idx n_u) {
  ReachPlan R;
  const idx n = L.n, t0 = L.t0;
  R.n_u = n_u;
  R.t0 = t0;
  R.tl = L.tl;
  R.ldy = dense_ld(L.tl);
  const Csr gut = gu.transpose_pattern();  // column u -> (state row, G_u slot)
  R.yn_ptr.assign(size_t(n_u) + 1, 0);
  R.op_ptr.assign(size_t(n_u) + 1, 0);
  R.yt_ptr.assign(size_t(n_u) + 1, 0);
  std::vector<idx> local(size_t(n), -1), b_of(size_t(n), -1);
  std::vector<std::vector<std::pair<idx, idx>>> in(static_cast<size_t>(n));  // row -> (col, slot)
  std::vector<idx> reach, touched_tail;
  for (idx u = 0; u < n_u; ++u) {
    reach.clear();
    touched_tail.clear();
    for (idx k = gut.ptr[size_t(u)]; k < gut.ptr[size_t(u) + 1]; ++k) {
      const idx r = L.iperm[size_t(gut.ind[size_t(k)])];
      b_of[size_t(r)] = idx(gut.val[size_t(k)]);
      if (r < t0 && local[size_t(r)] < 0) {
        local[size_t(r)] = 0;
        reach.push_back(r);
      }
      if (r >= t0) touched_tail.push_back(r);
    }
    // reach of the G_u rows in the graph of L (column c feeds rows r > c with
    // L(r, c) != 0), the non-tail part only; ascending order is a topological
    // order of the lower-triangular dependencies
    for (size_t h = 0; h < reach.size(); ++h) {
      const idx c = reach[h];
      for (idx q = L.lt_ptr[size_t(c)]; q < L.lt_ptr[size_t(c) + 1]; ++q) {
        const idx r = L.lt_row[size_t(q)];
        if (r < t0 && local[size_t(r)] < 0) {
          local[size_t(r)] = 0;
          reach.push_back(r);
        }
      }
    }
    std::sort(reach.begin(), reach.end());
    for (size_t k = 0; k < reach.size(); ++k) local[size_t(reach[k])] = idx(k);
    for (idx c : reach)
      for (idx q = L.lt_ptr[size_t(c)]; q < L.lt_ptr[size_t(c) + 1]; ++q) {
        const idx r = L.lt_row[size_t(q)];
        if (r >= t0 && in[size_t(r)].empty() && b_of[size_t(r)] < 0) touched_tail.push_back(r);
        in[size_t(r)].push_back({c, L.lt_slot[size_t(q)]});
      }
    std::sort(touched_tail.begin(), touched_tail.end());
    touched_tail.erase(std::unique(touched_tail.begin(), touched_tail.end()), touched_tail.end());
    auto emit_op = [&](idx r, idx dest) {
      auto& e = in[size_t(r)];
      std::sort(e.begin(), e.end());  // row order of L, like the full sweep
      const idx eb = idx(R.ent.size() / 2);
      for (const auto& [c, slot] : e) R.ent.insert(R.ent.end(), {local[size_t(c)], slot});
      R.ops.insert(R.ops.end(), {dest, b_of[size_t(r)], eb, idx(R.ent.size() / 2)});
      R.fmas += idx(e.size());
      e.clear();
    };
    for (size_t k = 0; k < reach.size(); ++k) {
      emit_op(reach[k], idx(k));
      R.yn_row.push_back(reach[k]);
    }
    for (idx t : touched_tail) {
      emit_op(t, -1 - (t - t0));
      R.yt_row.push_back(t - t0);
    }
    R.yt_ptr[size_t(u) + 1] = idx(R.yt_row.size());
    R.yn_ptr[size_t(u) + 1] = idx(R.yn_row.size());
    R.op_ptr[size_t(u) + 1] = idx(R.ops.size() / 4);
    for (idx r : reach) local[size_t(r)] = -1;
    for (idx k = gut.ptr[size_t(u)]; k < gut.ptr[size_t(u) + 1]; ++k)
      b_of[size_t(L.iperm[size_t(gut.ind[size_t(k)])])] = -1;
  }
  R.nnz_yn = idx(R.yn_row.size());
  return R;
}

StreamProgram build_stream_program(const LuPlan& L, const Csr& gu, const Csr& kxx, const Csr& kxu,
                                   idx n_u, int K, int consumers, int ring_bytes,
                                   int lookahead_max, const ReachPlan* reach,
                                   bool adjoint_identity, bool defer_tail) {
  const bool presolved = reach != nullptr;
  adjoint_identity = adjoint_identity && presolved;
  StreamProgram S;
  S.K = K;
  S.consumers = consumers;
  S.ring_bytes = ring_bytes;
  // fewer, larger steps win: the per-step overhead outweighs the lookahead
  // (measured at 1354/256: ring/2 47.8 ms, ring/4 55.2 ms per reduction)
  static const double step_div = [] {
    const char* e = std::getenv("BIPM_STEP_DIV");
    return e ? std::max(1.0, std::atof(e)) : 2.0;
  }();
  S.max_step_bytes = std::max(4096, std::min(int(ring_bytes / step_div) & ~15, 64 * 1024));
  const idx n = L.n, t0 = L.t0, tl = L.tl;
  S.stride[kArrDense] = 2LL * tl * dense_ld(tl);
  S.stride[kArrKxx] = kxx.nnz();
  S.stride[kArrKxuT] = kxu.nnz();
  S.stride[kArrGuT] = gu.nnz();
  S.stride[kArrSigma] = n;
  S.stride[kArrYN] = presolved ? reach->nnz_yn : 0;
  // stride[kArrSweep] is fixed after the program is built (nnz_vs, even)
  Builder B{S, S.max_step_bytes, {}};
  B.last_team = consumers / 32;
  // warp-local subtree sweeps: correct, measured no faster at 1354/256
  // (23.5 -> 24.1 ms per reduction: the per-warp level chains, not the team
  // barriers, bound the sweeps), so off unless BIPM_SUBTREE=1
  static const int subtree_on = [] {
    const char* e = std::getenv("BIPM_SUBTREE");
    return e ? std::atoi(e) : 0;
  }();
  if (subtree_on) B.group = subtree_groups(L, consumers / 32);
  using P = Builder::Pending;

  // factor slot of every entry of the four sweeps' direct value arrays
  std::vector<idx> slot_L(size_t(L.nnz_l)), slot_U(size_t(L.nnz_f - L.nnz_l)),
      slot_Ut(size_t(L.nnz_f - L.nnz_l)), slot_Lt(size_t(L.nnz_l));
  for (idx t = 0; t < L.nnz_l; ++t) slot_L[size_t(t)] = t;
  for (idx t = 0; t < L.nnz_f - L.nnz_l; ++t) slot_U[size_t(t)] = L.nnz_l + t;
  for (idx t = 0; t < L.nnz_f - L.nnz_l; ++t) slot_Ut[size_t(t)] = L.ft_src[size_t(t)];
  for (idx t = 0; t < L.nnz_l; ++t) slot_Lt[size_t(t)] = L.ft_src[size_t(L.nnz_f - L.nnz_l + t)];

  // the dense tail product: one all-warp step; W (tl x tl per scenario) is
  // read straight from global memory (L2: the 65 column tiles of a scenario
  // run close together), not staged through the ring
  auto dense = [&](int which) {
    if (tl == 0) return;
    P p{kStepDenseG, kFlagPre | kFlagCommit | kFlagBarrier, which, 0, {}, {}};
    B.emit(p);
    ++S.n_dense_steps;
  };
  // accumulator rows: control u belongs to register q = (u K + c) / consumers
  const int R = consumers / K;
  S.nq = int((size_t(n_u) * K + consumers - 1) / consumers);
  auto acc = [&](const Csr& A, std::vector<idx>& t_slot) {
    bool first_acc = true;  // the accumulation reads the finished sweep
    const Csr t = A.transpose_pattern();  // column u -> (state row, slot)
    t_slot.resize(t.val.size());
    for (size_t k = 0; k < t.val.size(); ++k) t_slot[k] = idx(t.val[k]);
    // a step spans as many controls as fit (several accumulator registers
    // q = u / R: the kernel loops over them), fewer steps than one per q
    {
      const int ue = int(n_u);
      int u0 = 0;
      const int q = 0;  // header aux0, unused by the kernel
      while (u0 < ue) {
        // grow the step while it fits
        int u1 = u0;
        int ents = 0;
        while (u1 < ue) {
          const int add = t.ptr[size_t(u1) + 1] - t.ptr[size_t(u1)];
          if (u1 > u0 && Builder::step_bytes(u1 - u0 + 1, ents + add, ents + add, 0) > S.max_step_bytes)
            break;
          ents += add;
          ++u1;
        }
        P p{kStepAcc, first_acc ? kFlagPre : 0, q, u0, {}, {}};
        for (int u = u0; u < u1; ++u) {
          const int beg = int(p.col.size());
          for (idx k = t.ptr[size_t(u)]; k < t.ptr[size_t(u) + 1]; ++k)
            p.col.push_back(L.iperm[size_t(t.ind[size_t(k)])]);
          p.items.insert(p.items.end(), {u, beg, int(p.col.size()), 0});  // u: not a panel row
        }
        p.val_arr = (&t_slot == &S.kxu_t_slot) ? kArrKxuT : kArrGuT;
        p.val_off = t.ptr[size_t(u0)];
        p.val_count = t.ptr[size_t(u1)] - t.ptr[size_t(u0)];
        if (p.val_count > 0) {  // an empty range contributes nothing
          B.emit(p);
          ++S.n_acc_steps;
          first_acc = false;
        }
        u0 = u1;
      }
    }
  };
  auto spmv = [&] {
    idx i0 = 0;
    while (i0 < n) {
      idx i1 = i0;
      int ents = 0;
      while (i1 < n) {
        const int add = kxx.ptr[size_t(i1) + 1] - kxx.ptr[size_t(i1)];
        if (i1 > i0 && Builder::step_bytes(int(i1 - i0) + 1, ents + add, ents + add,
                                           int(i1 - i0) + 1) > S.max_step_bytes)
          break;
        ents += add;
        ++i1;
      }
      P p{kStepSpmv, 0, 0, 0, {}, {}};
      const idx e0 = kxx.ptr[size_t(i0)];
      for (idx i = i0; i < i1; ++i) {
        const int beg = int(p.col.size());
        for (idx k = kxx.ptr[size_t(i)]; k < kxx.ptr[size_t(i) + 1]; ++k)
          p.col.push_back(L.iperm[size_t(kxx.ind[size_t(k)])]);
        p.items.insert(p.items.end(), {L.iperm[size_t(i)], beg, int(p.col.size()), int(i - i0)});
      }
      p.val_arr = kArrKxx;
      p.val_off = e0;
      p.val_count = kxx.ptr[size_t(i1)] - e0;
      p.x_arr = kArrSigma;
      p.x_off = i0;
      p.x_count = i1 - i0;
      B.emit(p);
      ++S.n_spmv_steps;
      i0 = i1;
    }
  };

  // scatter and copy-back synchronise internally (before) and after
  if (presolved) {
    B.emit(P{kStepScatterY, kFlagPre | kFlagBarrier, 0, 0, {}, {}});
  } else {
    B.emit(P{kStepScatter, kFlagPre | kFlagBarrier, 0, 0, {}, {}});
    B.sweep(L.sL, slot_L, false, true, 0);
    dense(0);
  }
  static const int pre_tail = [] {
    const char* e = std::getenv("BIPM_PRE_TAIL");
    return e ? std::atoi(e) : 1;
  }();
  // measured (same box): 1354/256 -0.7 %, 2869/64 -0.4 % per tile kernel with
  // the adjoint identity; +1 % at 9241 (K = 1, no identity): there off
  const idx pre_t0 = pre_tail && tl > 0 && adjoint_identity ? t0 : -1;
  B.sweep(L.sU, slot_U, true, false, 0, pre_t0);
  acc(kxu, S.kxu_t_slot);
  spmv();
  B.emit(P{kStepCopyBack, kFlagPre | kFlagBarrier, 0, 0, {}, {}});
  B.sweep(L.sUt, slot_Ut, true, true, 1);  // the diagonal is not part of the tail gather
  if (adjoint_identity) {
    // acc -= y_N' z_N: items per control u = its reach rows (panel rows),
    // values y_N[yn_ptr[u] ..] (kArrYN)
    bool first_acc = true;
    int u0 = 0;
    while (u0 < n_u) {
      int u1 = u0, ents = 0;
      while (u1 < n_u) {
        const int add = reach->yn_ptr[size_t(u1) + 1] - reach->yn_ptr[size_t(u1)];
        if (u1 > u0 &&
            Builder::step_bytes(u1 - u0 + 1, ents + add, ents + add, 0) > S.max_step_bytes)
          break;
        ents += add;
        ++u1;
      }
      P p{kStepAcc, first_acc ? kFlagPre : 0, 0, u0, {}, {}};
      for (int u = u0; u < u1; ++u) {
        const int beg = int(p.col.size());
        for (idx k = reach->yn_ptr[size_t(u)]; k < reach->yn_ptr[size_t(u) + 1]; ++k)
          p.col.push_back(reach->yn_row[size_t(k)]);
        p.items.insert(p.items.end(), {u, beg, int(p.col.size()), 0});
      }
      p.val_arr = kArrYN;
      p.val_off = reach->yn_ptr[size_t(u0)];
      p.val_count = reach->yn_ptr[size_t(u1)] - reach->yn_ptr[size_t(u0)];
      if (p.val_count > 0) {
        B.emit(p);
        ++S.n_acc_steps;
        first_acc = false;
      }
      u0 = u1;
    }
    // acc -= X_T' z_T (reads the tail rows the U' sweep's gather finished)
    if (tl > 0)
      B.emit(P{defer_tail ? kStepStoreTail : kStepAccTail, kFlagPre | kFlagBarrier, 0, 0, {}, {}});
  } else {
    dense(1);
    B.sweep(L.sLt, slot_Lt, false, false, 0, pre_t0);
    acc(gu, S.gu_t_slot);
  }

  if (S.vs_src.size() & 1) S.vs_src.push_back(-1);
  if (S.vs_src.empty()) S.vs_src.assign(2, -1);
  S.nnz_vs = idx(S.vs_src.size());
  S.stride[kArrSweep] = S.nnz_vs;
  // the VS parity bits were emitted with stride 0: VS offsets are even and its
  // stride is even, so they are correct as written
  S.steps = int(S.issue.size());

  // ---- ring placement (sequential with wrap; every scenario starts at 0)
  std::vector<int> beg(size_t(S.steps)), end(size_t(S.steps));
  int off = 0;
  for (int j = 0; j < S.steps; ++j) {
    StepIssue& is = S.issue[size_t(j)];
    const int bytes = is.pat_bytes + val_alloc(is.val_count) + val_alloc(is.x_count);
    if (bytes > ring_bytes) throw Error(kInvalidArgument, "stream plan: step larger than the ring");
    if (j == 0 || off + bytes > ring_bytes) off = 0;
    is.ring_off = off;
    is.val_ring = off + is.pat_bytes;
    is.x_ring = is.val_ring + val_alloc(is.val_count);
    beg[size_t(j)] = off;
    end[size_t(j)] = off + bytes;
    off += bytes;
  }
  // ---- producer waits: the latest earlier step (cyclically: the previous
  // scenario's program) whose region overlaps; capped by the lookahead
  S.ring_off.resize(size_t(S.steps));
  for (int j = 0; j < S.steps; ++j) {
    S.ring_off[size_t(j)] = S.issue[size_t(j)].ring_off;
    int d = 1;
    for (; d <= lookahead_max; ++d) {
      const int k = ((j - d) % S.steps + S.steps) % S.steps;
      if (beg[size_t(k)] < end[size_t(j)] && beg[size_t(j)] < end[size_t(k)]) break;
    }
    S.issue[size_t(j)].wait_delta = std::min(d, lookahead_max);
  }
  return S;
}

}  // namespace bipm
