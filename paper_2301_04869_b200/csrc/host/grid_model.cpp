#include "grid_model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <numeric>
#include <random>
#include <sstream>

namespace bipm {

namespace {

constexpr double kPi = 3.14159265358979323846;

[[noreturn]] void parse_fail(const std::string& what, int line = 0) {
  throw Error(kParseError, what + (line > 0 ? " (line " + std::to_string(line) + ")" : ""));
}

struct NumericTable {
  std::vector<std::vector<double>> rows;
  std::vector<int> lines;
};

// Locate `mpc.<name> = [ ... ]` and split its body into rows: a row ends at
// ';' or a newline, '%' comments to end of line, blanks/tabs/commas separate.
bool find_table(const std::string& text, const std::string& name, NumericTable& out) {
  const std::string key = "mpc." + name;
  size_t at = 0;
  for (;;) {
    at = text.find(key, at);
    if (at == std::string::npos) return false;
    size_t q = at + key.size();
    while (q < text.size() && (text[q] == ' ' || text[q] == '\t')) ++q;
    if (q < text.size() && text[q] == '=') break;
    at += key.size();
  }
  const size_t lb = text.find('[', at);
  if (lb == std::string::npos) parse_fail("missing '[' after " + key);
  const size_t rb = text.find(']', lb);
  if (rb == std::string::npos) parse_fail("missing ']' for " + key);
  int line = 1 + int(std::count(text.begin(), text.begin() + long(lb), '\n'));
  std::vector<double> row;
  auto end_row = [&](int ln) {
    if (row.empty()) return;
    out.rows.push_back(std::move(row));
    out.lines.push_back(ln);
    row.clear();
  };
  size_t i = lb + 1;
  while (i < rb) {
    const char c = text[i];
    if (c == '\n') {
      end_row(line);
      ++line;
      ++i;
    } else if (c == ';') {
      end_row(line);
      ++i;
    } else if (c == '%') {
      while (i < rb && text[i] != '\n') ++i;
    } else if (c == ' ' || c == '\t' || c == '\r' || c == ',') {
      ++i;
    } else {
      size_t j = i;
      while (j < rb && std::string(" \t;\n,%\r").find(text[j]) == std::string::npos) ++j;
      const std::string tok = text.substr(i, j - i);
      char* endp = nullptr;
      const double v = std::strtod(tok.c_str(), &endp);
      if (endp != tok.c_str() + tok.size()) parse_fail("malformed number '" + tok + "'", line);
      row.push_back(v);
      i = j;
    }
  }
  end_row(line);
  return true;
}

void need_cols(const std::vector<double>& r, size_t n, int line, const char* table) {
  if (r.size() < n)
    parse_fail(std::string("row of mpc.") + table + " has " + std::to_string(r.size()) +
                   " columns, need " + std::to_string(n),
               line);
}

// Union-find connectivity of the live network minus `down`.
bool network_connected(const GridCase& cs, const std::vector<idx>& down) {
  const idx nb = idx(cs.bus.size());
  std::map<int, idx> of_id;
  for (idx b = 0; b < nb; ++b) of_id[cs.bus[size_t(b)].id] = b;
  std::vector<idx> up(static_cast<size_t>(nb));
  std::iota(up.begin(), up.end(), 0);
  auto root = [&](idx a) {
    while (up[size_t(a)] != a) a = up[size_t(a)] = up[size_t(up[size_t(a)])];
    return a;
  };
  for (idx l = 0; l < idx(cs.branch.size()); ++l) {
    if (!cs.branch[size_t(l)].status) continue;
    if (std::find(down.begin(), down.end(), l) != down.end()) continue;
    const idx a = root(of_id.at(cs.branch[size_t(l)].from));
    const idx b = root(of_id.at(cs.branch[size_t(l)].to));
    if (a != b) up[size_t(a)] = b;
  }
  for (idx b = 1; b < nb; ++b)
    if (root(b) != root(0)) return false;
  return true;
}

BranchAdmittance admittance(const CaseBranch& br, const std::map<int, idx>& of_id,
                            double baseMVA) {
  BranchAdmittance a;
  a.from = of_id.at(br.from);
  a.to = of_id.at(br.to);
  const double z2 = br.r * br.r + br.x * br.x;
  const double gser = br.r / z2, bser = -br.x / z2;
  const double t = br.tap == 0.0 ? 1.0 : br.tap;
  const double phi = br.shift * kPi / 180.0;
  const double cphi = std::cos(phi), sphi = std::sin(phi);
  a.gff = gser / (t * t);
  a.bff = (bser + br.b / 2.0) / (t * t);
  a.gft = -(gser * cphi - bser * sphi) / t;
  a.bft = -(gser * sphi + bser * cphi) / t;
  a.gtf = -(gser * cphi + bser * sphi) / t;
  a.btf = -(-gser * sphi + bser * cphi) / t;
  a.gtt = gser;
  a.btt = bser + br.b / 2.0;
  const double rate = br.rateA / baseMVA;
  a.rate2 = br.rateA > 0 ? rate * rate : 0.0;
  return a;
}

}  // namespace

int GridCase::ref_bus() const {
  int r = -1;
  for (size_t i = 0; i < bus.size(); ++i)
    if (bus[i].type == 3) {
      if (r >= 0) parse_fail("multiple reference buses");
      r = int(i);
    }
  if (r < 0) parse_fail("no reference bus");
  return r;
}

GridCase read_matpower_text(const std::string& text) {
  GridCase cs;
  if (size_t f = text.find("function"); f != std::string::npos) {
    if (size_t eq = text.find('=', f); eq != std::string::npos) {
      size_t b = eq + 1;
      while (b < text.size() && std::isspace(static_cast<unsigned char>(text[b]))) ++b;
      size_t e = b;
      while (e < text.size() && !std::isspace(static_cast<unsigned char>(text[e]))) ++e;
      cs.name = text.substr(b, e - b);
    }
  }
  {
    const size_t p = text.find("mpc.baseMVA");
    if (p == std::string::npos) parse_fail("missing mpc.baseMVA");
    const size_t eq = text.find('=', p);
    const size_t sc = eq == std::string::npos ? eq : text.find(';', eq);
    if (eq == std::string::npos || sc == std::string::npos) parse_fail("malformed mpc.baseMVA");
    cs.baseMVA = std::strtod(text.substr(eq + 1, sc - eq - 1).c_str(), nullptr);
    if (!(cs.baseMVA > 0)) parse_fail("baseMVA must be positive");
  }
  NumericTable tb, tg, tl, tc;
  if (!find_table(text, "bus", tb)) parse_fail("missing table mpc.bus");
  if (!find_table(text, "gen", tg)) parse_fail("missing table mpc.gen");
  if (!find_table(text, "branch", tl)) parse_fail("missing table mpc.branch");
  if (!find_table(text, "gencost", tc)) parse_fail("missing table mpc.gencost");

  for (size_t r = 0; r < tb.rows.size(); ++r) {
    const auto& v = tb.rows[r];
    need_cols(v, 13, tb.lines[r], "bus");
    CaseBus b;
    b.id = int(v[0]);
    b.type = int(v[1]);
    b.Pd = v[2];
    b.Qd = v[3];
    b.Gs = v[4];
    b.Bs = v[5];
    b.Vm = v[7];
    b.Va = v[8];
    b.Vmax = v[11];
    b.Vmin = v[12];
    cs.bus.push_back(b);
  }
  for (size_t r = 0; r < tg.rows.size(); ++r) {
    const auto& v = tg.rows[r];
    need_cols(v, 10, tg.lines[r], "gen");
    CaseGen g;
    g.bus = int(v[0]);
    g.Pg = v[1];
    g.Qg = v[2];
    g.Qmax = v[3];
    g.Qmin = v[4];
    g.Vg = v[5];
    g.status = int(v[7]);
    g.Pmax = v[8];
    g.Pmin = v[9];
    cs.gen.push_back(g);
  }
  for (size_t r = 0; r < tl.rows.size(); ++r) {
    const auto& v = tl.rows[r];
    need_cols(v, 11, tl.lines[r], "branch");
    CaseBranch br;
    br.from = int(v[0]);
    br.to = int(v[1]);
    br.r = v[2];
    br.x = v[3];
    br.b = v[4];
    br.rateA = v[5];
    br.tap = v[8];
    br.shift = v[9];
    br.status = int(v[10]);
    cs.branch.push_back(br);
  }
  for (size_t r = 0; r < tc.rows.size(); ++r) {
    const auto& v = tc.rows[r];
    need_cols(v, 4, tc.lines[r], "gencost");
    CaseCost c;
    c.model = int(v[0]);
    c.ncost = int(v[3]);
    if (c.model != 2) parse_fail("only polynomial gencost (model 2) supported", tc.lines[r]);
    if (v.size() < size_t(4 + c.ncost)) parse_fail("gencost row shorter than ncost", tc.lines[r]);
    if (c.ncost > 3) parse_fail("cost polynomials above degree 2 not supported", tc.lines[r]);
    c.coef.assign(v.begin() + 4, v.begin() + 4 + c.ncost);
    cs.cost.push_back(c);
  }
  for (const auto& br : cs.branch) {
    bool f = false, t = false;
    for (const auto& b : cs.bus) {
      f |= b.id == br.from;
      t |= b.id == br.to;
    }
    if (!f || !t) parse_fail("branch endpoint references unknown bus");
  }
  cs.ref_bus();
  if (!cs.cost.empty() && cs.cost.size() != cs.gen.size())
    parse_fail("gencost rows do not match gen rows");
  return cs;
}

GridCase read_matpower_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) parse_fail("cannot open case file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return read_matpower_text(ss.str());
}

ScenarioDraw draw_scenarios(const GridCase& cs, idx N, double sigma,
                            const std::vector<idx>& contingencies, std::uint64_t seed) {
  if (N < 1) throw Error(kInvalidArgument, "draw_scenarios: N must be >= 1");
  if (sigma < 0) throw Error(kInvalidArgument, "draw_scenarios: sigma must be >= 0");
  const idx nb = idx(cs.bus.size());
  ScenarioDraw d;
  d.N = N;
  d.sigma = sigma;
  d.seed = seed;
  d.mult.assign(size_t(N) * size_t(nb), 1.0);
  d.outages.assign(size_t(N), {});
  if (sigma > 0) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> normal(1.0, sigma);
    for (size_t k = 0; k < d.mult.size(); ++k) d.mult[k] = std::clamp(normal(gen), 0.5, 1.5);
  }
  for (size_t k = 0; k < contingencies.size(); ++k) {
    const idx l = contingencies[k];
    if (l < 0 || l >= idx(cs.branch.size()) || !cs.branch[size_t(l)].status)
      throw Error(kInvalidArgument, "contingency names an unknown or out-of-service branch");
    d.outages[k % size_t(N)].push_back(l);
  }
  for (idx s = 0; s < N; ++s)
    if (!network_connected(cs, d.outages[size_t(s)]))
      throw Error(kInvalidArgument,
                  "scenario " + std::to_string(s) + ": contingency disconnects the network");
  return d;
}

OpfModel build_opf_model(const GridCase& cs, const ScenarioDraw& sc) {
  OpfModel M;
  const idx nbus = idx(cs.bus.size());
  const idx N = sc.N;
  if (N < 1) throw Error(kInvalidArgument, "build_opf_model: need at least one scenario");
  if (sc.mult.size() != size_t(N) * size_t(nbus))
    throw Error(kInvalidArgument, "build_opf_model: scenario multipliers shape");
  const double base = cs.baseMVA;
  const idx ref = idx(cs.ref_bus());
  std::map<int, idx> of_id;
  for (idx b = 0; b < nbus; ++b) of_id[cs.bus[size_t(b)].id] = b;

  // live generators and branches
  std::vector<idx> live_gen, live_br;
  std::vector<char> gen_at(size_t(nbus), 0);
  for (idx g = 0; g < idx(cs.gen.size()); ++g)
    if (cs.gen[size_t(g)].status) {
      live_gen.push_back(g);
      M.gen_bus.push_back(of_id.at(cs.gen[size_t(g)].bus));
      gen_at[size_t(M.gen_bus.back())] = 1;
    }
  for (idx l = 0; l < idx(cs.branch.size()); ++l)
    if (cs.branch[size_t(l)].status) live_br.push_back(l);
  const idx ngen = idx(live_gen.size()), L = idx(live_br.size());

  M.slack_gen = -1;
  for (idx g = 0; g < ngen && M.slack_gen < 0; ++g)
    if (M.gen_bus[size_t(g)] == ref) M.slack_gen = g;
  if (M.slack_gen < 0) parse_fail("reference bus has no in-service generator");

  // variables: x = [theta of non-ref buses | v of non-gen buses],
  //            u = [p of non-slack gens | v of gen buses]
  std::vector<idx> th_x(size_t(nbus), -1), v_x(size_t(nbus), -1), v_u(size_t(nbus), -1),
      p_u(size_t(ngen), -1);
  idx nx = 0, nu = 0;
  for (idx b = 0; b < nbus; ++b)
    if (b != ref) th_x[size_t(b)] = nx++;
  for (idx b = 0; b < nbus; ++b)
    if (!gen_at[size_t(b)]) v_x[size_t(b)] = nx++;
  for (idx g = 0; g < ngen; ++g)
    if (g != M.slack_gen) p_u[size_t(g)] = nu++;
  for (idx b = 0; b < nbus; ++b)
    if (gen_at[size_t(b)]) v_u[size_t(b)] = nu++;

  M.name = cs.name + "_N" + std::to_string(N);
  M.N = N;
  M.nbus = nbus;
  M.nbr = L;
  M.ngen = ngen;
  M.n_x = nx;
  M.n_u = nu;
  M.ref_bus = ref;
  M.theta_in = th_x;
  M.vmag_in.assign(size_t(nbus), -1);
  for (idx b = 0; b < nbus; ++b)
    M.vmag_in[size_t(b)] = v_x[size_t(b)] >= 0 ? v_x[size_t(b)] : nx + v_u[size_t(b)];
  M.pgen_in.assign(size_t(ngen), -1);
  for (idx g = 0; g < ngen; ++g)
    if (p_u[size_t(g)] >= 0) M.pgen_in[size_t(g)] = nx + p_u[size_t(g)];

  BasisLayout& lay = M.lay;
  lay.vv = 1;
  lay.br = lay.vv + nbus;
  lay.sq = lay.br + 4 * L;
  lay.pd = lay.sq + 2 * L;
  lay.qd = lay.pd + nbus;
  lay.pg = lay.qd + nbus;
  lay.pg2 = lay.pg + ngen;
  lay.n_b = lay.pg2 + ngen;

  for (idx l : live_br) M.br.push_back(admittance(cs.branch[size_t(l)], of_id, base));

  M.pd.resize(size_t(N) * size_t(nbus));
  M.qd.resize(size_t(N) * size_t(nbus));
  for (idx s = 0; s < N; ++s)
    for (idx b = 0; b < nbus; ++b) {
      const double k = sc.mult[size_t(s) * size_t(nbus) + size_t(b)];
      M.pd[size_t(s) * size_t(nbus) + size_t(b)] = cs.bus[size_t(b)].Pd / base * k;
      M.qd[size_t(s) * size_t(nbus) + size_t(b)] = cs.bus[size_t(b)].Qd / base * k;
    }
  M.status.assign(size_t(N) * size_t(L), 1.0);
  for (idx s = 0; s < N && s < idx(sc.outages.size()); ++s)
    for (idx l : sc.outages[size_t(s)]) {
      auto it = std::find(live_br.begin(), live_br.end(), l);
      if (it == live_br.end())
        throw Error(kInvalidArgument, "scenario outage names an out-of-service branch");
      M.status[size_t(s) * size_t(L) + size_t(it - live_br.begin())] = 0.0;
    }
  M.gs.resize(size_t(nbus));
  M.bs.resize(size_t(nbus));
  for (idx b = 0; b < nbus; ++b) {
    M.gs[size_t(b)] = cs.bus[size_t(b)].Gs / base;
    M.bs[size_t(b)] = cs.bus[size_t(b)].Bs / base;
  }
  M.gs_ref = M.gs[size_t(ref)];
  for (idx l = 0; l < L; ++l) {
    if (M.br[size_t(l)].from == ref) M.ref_from.push_back(l);
    if (M.br[size_t(l)].to == ref) M.ref_to.push_back(l);
  }
  for (idx g = 0; g < ngen; ++g)
    if (M.gen_bus[size_t(g)] == ref && g != M.slack_gen) M.ref_other_gens.push_back(g);

  // ---- linear maps of the basis ----
  using Entry = std::pair<std::pair<idx, idx>, double>;
  std::vector<Entry> eg, eh, ef;
  std::vector<idx> prow(size_t(nbus), -1), qrow(size_t(nbus), -1);
  idx r = 0;
  for (idx b = 0; b < nbus; ++b)
    if (b != ref) prow[size_t(b)] = r++;
  for (idx b = 0; b < nbus; ++b)
    if (v_u[size_t(b)] < 0) qrow[size_t(b)] = r++;
  if (r != nx) throw Error(kInvalidArgument, "opf model: g row count mismatch");

  // branch-end injections (from side uses cff/ctt's own-voltage lane)
  auto p_terms = [&](std::vector<Entry>& e, idx row, idx l, bool from, double sgn) {
    const auto& c = M.br[size_t(l)];
    if (from) {
      e.push_back({{row, lay.cff(l)}, sgn * c.gff});
      e.push_back({{row, lay.wc(l)}, sgn * c.gft});
      e.push_back({{row, lay.ws(l)}, sgn * c.bft});
    } else {
      e.push_back({{row, lay.ctt(l)}, sgn * c.gtt});
      e.push_back({{row, lay.wc(l)}, sgn * c.gtf});
      e.push_back({{row, lay.ws(l)}, sgn * -c.btf});
    }
  };
  auto q_terms = [&](std::vector<Entry>& e, idx row, idx l, bool from, double sgn) {
    const auto& c = M.br[size_t(l)];
    if (from) {
      e.push_back({{row, lay.cff(l)}, sgn * -c.bff});
      e.push_back({{row, lay.wc(l)}, sgn * -c.bft});
      e.push_back({{row, lay.ws(l)}, sgn * c.gft});
    } else {
      e.push_back({{row, lay.ctt(l)}, sgn * -c.btt});
      e.push_back({{row, lay.wc(l)}, sgn * -c.btf});
      e.push_back({{row, lay.ws(l)}, sgn * -c.gtf});
    }
  };
  for (idx b = 0; b < nbus; ++b) {
    if (const idx pr = prow[size_t(b)]; pr >= 0) {
      for (idx g = 0; g < ngen; ++g)
        if (M.gen_bus[size_t(g)] == b) eg.push_back({{pr, lay.pg + g}, 1.0});
      eg.push_back({{pr, lay.pd + b}, -1.0});
      eg.push_back({{pr, lay.vv + b}, -M.gs[size_t(b)]});
    }
    if (const idx qr = qrow[size_t(b)]; qr >= 0) {
      eg.push_back({{qr, lay.qd + b}, -1.0});
      eg.push_back({{qr, lay.vv + b}, M.bs[size_t(b)]});
    }
  }
  for (idx l = 0; l < L; ++l) {
    const auto& c = M.br[size_t(l)];
    if (prow[size_t(c.from)] >= 0) p_terms(eg, prow[size_t(c.from)], l, true, -1.0);
    if (prow[size_t(c.to)] >= 0) p_terms(eg, prow[size_t(c.to)], l, false, -1.0);
    if (qrow[size_t(c.from)] >= 0) q_terms(eg, qrow[size_t(c.from)], l, true, -1.0);
    if (qrow[size_t(c.to)] >= 0) q_terms(eg, qrow[size_t(c.to)], l, false, -1.0);
  }

  // h rows: squared flows at both ends (2L), reactive generation at each
  // generator bus, slack active power; limits live in the slack bounds.
  idx ngb = 0;
  for (idx b = 0; b < nbus; ++b) ngb += v_u[size_t(b)] >= 0;
  const idx m = 2 * L + ngb + 1;
  M.m = m;
  M.s_lo.assign(size_t(m), -kInf);
  M.s_up.assign(size_t(m), kInf);
  for (idx l = 0; l < L; ++l) {
    eh.push_back({{l, lay.sqf(l)}, 1.0});
    eh.push_back({{L + l, lay.sqt(l)}, 1.0});
    if (M.br[size_t(l)].rate2 > 0) {
      M.s_lo[size_t(l)] = -M.br[size_t(l)].rate2;
      M.s_lo[size_t(L + l)] = -M.br[size_t(l)].rate2;
    }
  }
  idx hr = 2 * L;
  for (idx b = 0; b < nbus; ++b) {
    if (v_u[size_t(b)] < 0) continue;
    eh.push_back({{hr, lay.qd + b}, 1.0});
    eh.push_back({{hr, lay.vv + b}, -M.bs[size_t(b)]});
    for (idx l = 0; l < L; ++l) {
      if (M.br[size_t(l)].from == b) q_terms(eh, hr, l, true, 1.0);
      if (M.br[size_t(l)].to == b) q_terms(eh, hr, l, false, 1.0);
    }
    double qlo = 0, qhi = 0;
    for (idx g = 0; g < ngen; ++g)
      if (M.gen_bus[size_t(g)] == b) {
        qlo += cs.gen[size_t(live_gen[size_t(g)])].Qmin / base;
        qhi += cs.gen[size_t(live_gen[size_t(g)])].Qmax / base;
      }
    M.s_lo[size_t(hr)] = -qhi;
    M.s_up[size_t(hr)] = -qlo;
    ++hr;
  }
  eh.push_back({{hr, lay.pg + M.slack_gen}, 1.0});
  {
    const CaseGen& g = cs.gen[size_t(live_gen[size_t(M.slack_gen)])];
    M.s_lo[size_t(hr)] = -g.Pmax / base;
    M.s_up[size_t(hr)] = -g.Pmin / base;
  }
  if (++hr != m) throw Error(kInvalidArgument, "opf model: h row count mismatch");

  // averaged polynomial cost
  const double avg = 1.0 / double(N);
  for (idx g = 0; g < ngen; ++g) {
    const idx gi = live_gen[size_t(g)];
    double c2 = 0, c1 = 0, c0 = 0;
    if (size_t(gi) < cs.cost.size()) {
      const CaseCost& gc = cs.cost[size_t(gi)];
      if (gc.ncost >= 3) {
        c2 = gc.coef[size_t(gc.ncost - 3)];
        c1 = gc.coef[size_t(gc.ncost - 2)];
        c0 = gc.coef[size_t(gc.ncost - 1)];
      } else if (gc.ncost == 2) {
        c1 = gc.coef[0];
        c0 = gc.coef[1];
      } else if (gc.ncost == 1) {
        c0 = gc.coef[0];
      }
    }
    if (c2 != 0) ef.push_back({{0, lay.pg2 + g}, avg * c2 * base * base});
    if (c1 != 0) ef.push_back({{0, lay.pg + g}, avg * c1 * base});
    if (c0 != 0) ef.push_back({{0, 0}, avg * c0});
  }
  M.L_f = Csr::assemble(1, lay.n_b, std::move(ef));
  M.L_g = Csr::assemble(nx, lay.n_b, std::move(eg));
  M.L_h = Csr::assemble(m, lay.n_b, std::move(eh));

  // bounds and start point
  M.x_lo.assign(size_t(nx), -kInf);
  M.x_up.assign(size_t(nx), kInf);
  M.u_lo.assign(size_t(nu), -kInf);
  M.u_up.assign(size_t(nu), kInf);
  M.x_start.assign(size_t(nx), 0.0);
  M.u_start.assign(size_t(nu), 0.0);
  for (idx b = 0; b < nbus; ++b) {
    const CaseBus& bus = cs.bus[size_t(b)];
    if (th_x[size_t(b)] >= 0) M.x_start[size_t(th_x[size_t(b)])] = bus.Va * kPi / 180.0;
    if (const idx i = v_x[size_t(b)]; i >= 0) {
      M.x_lo[size_t(i)] = bus.Vmin;
      M.x_up[size_t(i)] = bus.Vmax;
      M.x_start[size_t(i)] = bus.Vm > 0 ? bus.Vm : 1.0;
    }
    if (const idx i = v_u[size_t(b)]; i >= 0) {
      M.u_lo[size_t(i)] = bus.Vmin;
      M.u_up[size_t(i)] = bus.Vmax;
      M.u_start[size_t(i)] = 1.0;
    }
  }
  for (idx g = 0; g < ngen; ++g) {
    const CaseGen& gen = cs.gen[size_t(live_gen[size_t(g)])];
    if (const idx i = p_u[size_t(g)]; i >= 0) {
      M.u_lo[size_t(i)] = gen.Pmin / base;
      M.u_up[size_t(i)] = gen.Pmax / base;
      M.u_start[size_t(i)] = gen.Pg / base;
    }
    if (const idx i = v_u[size_t(M.gen_bus[size_t(g)])]; i >= 0 && gen.Vg > 0)
      M.u_start[size_t(i)] = gen.Vg;
  }
  return M;
}

}  // namespace bipm
