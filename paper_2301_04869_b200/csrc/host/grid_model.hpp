// Power-grid input side of the solver: MATPOWER case reading, scenario
// draws and the block-structured OPF model the GPU kernels evaluate.
//
// Semantics follow the reference so a user's case files, seeds and options
// produce the same problem:
//   reading      proj/core/src/opf_parse.cpp:19-214
//   scenarios    proj/core/src/scenarios.cpp:44-80
//   variables    proj/core/src/opf_model.cpp:580-622
//   model        proj/core/src/opf_model.cpp:624-875 (basis layout :65-76,
//                branch admittances :13-45)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace bipm {

struct CaseBus {
  int id = 0, type = 1;
  double Pd = 0, Qd = 0, Gs = 0, Bs = 0, Vm = 1, Va = 0, Vmax = 1.1, Vmin = 0.9;
};
struct CaseGen {
  int bus = 0, status = 1;
  double Pg = 0, Qg = 0, Qmax = 0, Qmin = 0, Vg = 1, Pmax = 0, Pmin = 0;
};
struct CaseBranch {
  int from = 0, to = 0, status = 1;
  double r = 0, x = 0, b = 0, rateA = 0, tap = 0, shift = 0;
};
struct CaseCost {
  int model = 2, ncost = 0;
  std::vector<double> coef;  // highest order first
};

struct GridCase {
  std::string name;
  double baseMVA = 100;
  std::vector<CaseBus> bus;
  std::vector<CaseGen> gen;
  std::vector<CaseBranch> branch;
  std::vector<CaseCost> cost;
  int ref_bus() const;  // index of the single type-3 bus (throws kParseError)
};

GridCase read_matpower_text(const std::string& text);
GridCase read_matpower_file(const std::string& path);

// Load multipliers N(1, sigma^2) clamped to [0.5, 1.5] drawn with
// std::mt19937_64(seed) scenario-major; outages round-robin.
struct ScenarioDraw {
  idx N = 0;
  double sigma = 0;
  std::uint64_t seed = 0;
  std::vector<double> mult;               // [N][nbus]
  std::vector<std::vector<idx>> outages;  // per scenario, branch indices
};
ScenarioDraw draw_scenarios(const GridCase& cs, idx N, double sigma,
                            const std::vector<idx>& contingencies, std::uint64_t seed);

struct BranchAdmittance {
  idx from = 0, to = 0;
  double gff = 0, bff = 0, gft = 0, bft = 0, gtf = 0, btf = 0, gtt = 0, btt = 0;
  double rate2 = 0;  // squared per-unit flow limit (0: unlimited)
};

// Basis lane layout: [1 | v^2 per bus | 4 monomials per branch | 2 squared
// flows per branch | Pd, Qd per bus | Pg, Pg^2 per live generator].
struct BasisLayout {
  idx vv = 1, br = 0, sq = 0, pd = 0, qd = 0, pg = 0, pg2 = 0, n_b = 0;
  idx cff(idx l) const { return br + 4 * l; }
  idx ctt(idx l) const { return br + 4 * l + 1; }
  idx wc(idx l) const { return br + 4 * l + 2; }
  idx ws(idx l) const { return br + 4 * l + 3; }
  idx sqf(idx l) const { return sq + 2 * l; }
  idx sqt(idx l) const { return sq + 2 * l + 1; }
};

// The block-structured OPF: per scenario b,
//   min f_b(x_b, u)  s.t.  g_b = L_g psi(x_b, u) = 0,  h_b = L_h psi + s_b = 0,
// with f_b = L_f psi and psi the shared polar power-flow basis.
struct OpfModel {
  std::string name;
  idx N = 0, nbus = 0, nbr = 0, ngen = 0;
  idx n_x = 0, n_u = 0, m = 0;
  idx ref_bus = -1, slack_gen = -1;
  BasisLayout lay;
  // input maps (index into [x | u] of length n_x + n_u)
  std::vector<idx> theta_in;  // bus -> input, -1 at the reference bus
  std::vector<idx> vmag_in;   // bus -> input
  std::vector<idx> pgen_in;   // live gen -> input, -1 for the slack
  std::vector<idx> gen_bus;   // live gen -> bus
  std::vector<BranchAdmittance> br;  // live branches
  std::vector<double> gs, bs;        // per-bus shunts (pu)
  std::vector<double> pd, qd;        // [N][nbus] scenario loads (pu)
  std::vector<double> status;        // [N][nbr] branch status (1 / 0)
  double gs_ref = 0;
  std::vector<idx> ref_from, ref_to, ref_other_gens;
  Csr L_f, L_g, L_h;
  std::vector<double> x_lo, x_up, u_lo, u_up, s_lo, s_up, x_start, u_start;

  idx n_d() const { return n_x + n_u; }
  idx n_b() const { return lay.n_b; }
};

OpfModel build_opf_model(const GridCase& cs, const ScenarioDraw& sc);

}  // namespace bipm
