// Reference-oracle driver: runs the UNMODIFIED reference solver
// (/root/reference/proj/core, compiled by oracle/Makefile into oracle/_ref/)
// and dumps fixtures from its public API.
//
// TEST INFRASTRUCTURE (oracle/).  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg and --impl reference) execute this binary.
//
//   bipm_ref solve --case F --N n --sigma s --seed k [--groups G --workers W
//                  --max-iter I --batch B --tol t] [--iterate-out DIR]
//                  [--contingencies l1,l2,...]
//       full reference solve (proj/core/src/ipm.cpp:435-664); prints one JSON
//       object: status, iterations, objective, per-iteration logs, timers.
//   bipm_ref dump --case F --N n --sigma s --seed k --iter K --out DIR
//       iterate after K reference iterations (solve with max_iter=K), then at
//       that iterate: the model, the derivative bundle
//       (autodiff.cpp:484-516), the augmented system (kkt.cpp:67-109), the
//       condensed system (kkt.cpp:123-170), the reduced system at delta_w=0
//       (kkt.cpp:492-505) and the reduced-strategy Newton step
//       (kkt.cpp:945-1006 via ipm.cpp:174-192).  Arrays are raw little-endian
//       files listed in DIR/manifest.json.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "blockipm/ipm.hpp"
#include "blockipm/kkt.hpp"
#include "blockipm/opf.hpp"
#ifdef BIPM_WITH_GPU_SHIM
// bipm_ref_gpu: the same driver linked with integration/bipm_reference_shim.cpp
// (--gpu kkt | ad | kkt,ad routes the reference's solve_reduced and/or its
// AD calls to the B200 engine through the C-ABI)
#include "bipm_reference_shim.hpp"
#endif

using namespace blockipm;

namespace {

struct Args {
  std::map<std::string, std::string> kv;
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
};

Args parse_args(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::invalid_argument("bad argument " + k);
    k = k.substr(2);
    if (i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0)
      a.kv[k] = argv[++i];
    else
      a.kv[k] = "1";
  }
  return a;
}

struct Dumper {
  std::string dir;
  nlohmann::json manifest = nlohmann::json::object();

  void raw(const std::string& name, const std::string& dtype, std::vector<long> shape,
           const void* data, size_t bytes) {
    std::ofstream f(dir + "/" + name + ".bin", std::ios::binary);
    f.write(static_cast<const char*>(data), std::streamsize(bytes));
    manifest[name] = {{"dtype", dtype}, {"shape", shape}};
  }
  // Matrix(rows, cols) column-major == numpy (cols, rows) row-major.
  void mat(const std::string& name, const Matrix& m) {
    raw(name, "f8", {m.cols(), m.rows()}, m.data(), m.size() * sizeof(double));
  }
  void vec(const std::string& name, const Vector& v) {
    raw(name, "f8", {long(v.size())}, v.data(), v.size() * sizeof(double));
  }
  void ivec(const std::string& name, const std::vector<index_t>& v) {
    raw(name, "i4", {long(v.size())}, v.data(), v.size() * sizeof(index_t));
  }
  void pat(const std::string& name, const SparsityPattern& p) {
    ivec(name + "_rowptr", p.row_ptr);
    ivec(name + "_colind", p.col_ind);
    manifest[name + "_shape"] = {p.rows, p.cols};
  }
  void spm(const std::string& name, const SparseMatrix& m) {
    ivec(name + "_rowptr", m.row_ptr);
    ivec(name + "_colind", m.col_ind);
    vec(name + "_val", m.val);
    manifest[name + "_shape"] = {m.rows, m.cols};
  }
  void scalar(const std::string& name, double v) { manifest[name] = v; }
  void finish() {
    std::ofstream f(dir + "/manifest.json");
    f << manifest.dump(1);
  }
};

IpmOptions options_from(const Args& a) {
  IpmOptions o;
  o.tol = std::stod(a.get("tol", "1e-6"));
  o.max_iter = std::stoi(a.get("max-iter", "300"));
  o.groups = std::stoi(a.get("groups", "1"));
  o.n_batch = std::stoi(a.get("batch", "32"));
  o.exec.worker_count = std::stoi(a.get("workers", a.get("groups", "1")));
  o.exec.order = a.get("fast", "0") == "1" ? ReduceOrder::fast : ReduceOrder::deterministic;
  o.check_step_residual = a.get("check-residual", "0") == "1";
  return o;
}

BlockNlp load(const Args& a, opf::CaseData* cs_out = nullptr, opf::ScenarioSet* sc_out = nullptr) {
  opf::CaseData cs = opf::parse_matpower_file(a.get("case"));
  const index_t N = std::stoi(a.get("N", "1"));
  const double sigma = std::stod(a.get("sigma", "0"));
  const std::uint64_t seed = std::stoull(a.get("seed", "0"));
  std::vector<index_t> cont;  // --contingencies 4,7,...: branch indices, round-robin
  {
    std::stringstream ss(a.get("contingencies"));
    for (std::string tok; std::getline(ss, tok, ',');)
      if (!tok.empty()) cont.push_back(index_t(std::stoi(tok)));
  }
  opf::ScenarioSet sc = opf::generate_scenarios(cs, N, sigma, cont, seed);
  if (cs_out) *cs_out = cs;
  if (sc_out) *sc_out = sc;
  return opf::build_block_opf(cs, sc);
}

void dump_iterate(Dumper& d, const std::string& pre, const Iterate& it) {
  d.mat(pre + "x", it.x);
  d.vec(pre + "u", it.u);
  d.mat(pre + "s", it.s);
  d.mat(pre + "y", it.y);
  d.mat(pre + "z", it.z);
  d.mat(pre + "kappa_lo", it.kappa_lo);
  d.mat(pre + "kappa_up", it.kappa_up);
  d.mat(pre + "nu_lo", it.nu_lo);
  d.mat(pre + "nu_up", it.nu_up);
  d.vec(pre + "lambda_lo", it.lambda_lo);
  d.vec(pre + "lambda_up", it.lambda_up);
}

int cmd_solve(const Args& a) {
  opf::CaseData cs;
  opf::ScenarioSet sc;
  const BlockNlp nlp = load(a, &cs, &sc);
#ifdef BIPM_WITH_GPU_SHIM
  const std::string gpu = a.get("gpu");
  if (gpu.find("kkt") != std::string::npos) bipm_shim::enable_kkt(true);
  if (gpu.find("ad") != std::string::npos) bipm_shim::enable_ad(cs, sc);
#endif
  IpmOptions o = options_from(a);
  Executor exec(o.exec);
  const auto t0 = std::chrono::steady_clock::now();
  SolveResult r = solve(nlp, exec, o);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  nlohmann::json j;
  j["status"] = to_string(r.status);
  j["iterations"] = r.logs.size();
  j["objective"] = r.objective;
  j["t_total"] = r.t_total;
  j["t_ad"] = r.t_ad;
  j["t_kkt"] = r.t_kkt;
  j["wall"] = wall;
  j["n_x"] = nlp.dims.n_x;
  j["n_u"] = nlp.dims.n_u;
  j["m"] = nlp.dims.m;
  j["N"] = nlp.dims.N;
  j["counters"] = {r.counters.spsm, r.counters.spmm, r.counters.tiles};
  j["max_step_residual"] = r.max_step_residual;
  nlohmann::json logs = nlohmann::json::array();
  for (const auto& l : r.logs)
    logs.push_back({{"iter", l.iter},         {"objective", l.objective}, {"inf_pr", l.inf_pr},
                    {"inf_du", l.inf_du},     {"mu", l.mu},               {"alpha_p", l.alpha_primal},
                    {"alpha_d", l.alpha_dual}, {"t_ad", l.t_ad},          {"t_kkt", l.t_kkt},
                    {"t_total", l.t_total},   {"corr", l.corrections},    {"fallback", l.fallback}});
  j["logs"] = logs;
  j["u"] = r.iterate.u;
#ifdef BIPM_WITH_GPU_SHIM
  j["gpu_kkt_calls"] = bipm_shim::kkt_calls();
  j["gpu_ad_calls"] = bipm_shim::ad_calls();
#endif
  std::printf("%s\n", j.dump().c_str());
  if (!a.get("iterate-out").empty()) {
    Dumper d{a.get("iterate-out")};
    dump_iterate(d, "", r.iterate);
    d.scalar("objective", r.objective);
    d.finish();
  }
  return 0;
}

int cmd_dump(const Args& a) {
  const BlockNlp nlp = load(a);
  const BlockDims& dm = nlp.dims;
  const int K = std::stoi(a.get("iter", "0"));
  IpmOptions o = options_from(a);
  Executor exec(o.exec);

  // Iterate at the start of iteration K and the mu used by iteration K.
  Iterate it = initial_iterate(nlp, o);
  double mu = o.mu0;
  if (K > 0) {
    IpmOptions ok = o;
    ok.max_iter = K;
    SolveResult rk = solve(nlp, exec, ok);
    if (int(rk.logs.size()) != K) throw std::runtime_error("solve ended before the dump iterate");
    it = rk.iterate;
  }
  {
    IpmOptions o1 = o;
    o1.max_iter = K + 1;
    SolveResult r1 = solve(nlp, exec, o1);
    if (int(r1.logs.size()) != K + 1) throw std::runtime_error("no iteration K to dump");
    mu = r1.logs.back().mu;
  }

  AdPlan plan = make_ad_plan(nlp);
  DerivativeBundle bd = make_bundle(nlp, plan);
  AdWorkspace ws(nlp, plan, dm.N);
  eval_bundle_range(nlp, plan, ws, it.x, it.u, it.y, it.z, 1.0, 0, bd);

  Dumper d{a.get("out")};
  d.manifest["dims"] = {dm.N, dm.n_x, dm.n_u, dm.m, dm.n_b};
  d.manifest["p_jac"] = plan.p_jac;
  d.manifest["p_hess"] = plan.p_hess;
  d.scalar("mu", mu);
  d.scalar("iter", K);
  // model
  d.spm("L_f", nlp.L_f);
  d.spm("L_g", nlp.L_g);
  d.spm("L_h", nlp.L_h);
  d.vec("x_lo", nlp.x_bounds.lower);
  d.vec("x_up", nlp.x_bounds.upper);
  d.vec("u_lo", nlp.u_bounds.lower);
  d.vec("u_up", nlp.u_bounds.upper);
  d.vec("s_lo", nlp.s_bounds.lower);
  d.vec("s_up", nlp.s_bounds.upper);
  d.vec("x_start", nlp.x_start);
  d.vec("u_start", nlp.u_start);
  // patterns
  d.pat("gx_p", plan.g_split.x_pat);
  d.pat("gu_p", plan.g_split.u_pat);
  d.pat("hx_p", plan.h_split.x_pat);
  d.pat("hu_p", plan.h_split.u_pat);
  d.pat("wxx_p", plan.w_split.xx);
  d.pat("wxu_p", plan.w_split.xu);
  d.pat("wuu_p", plan.w_split.uu);
  d.pat("hess_p", plan.patterns.hess);
  // iterate + bundle
  dump_iterate(d, "it_", it);
  d.vec("f", bd.f);
  d.mat("g", bd.g);
  d.mat("h", bd.h);
  d.mat("gx", bd.gx);
  d.mat("gu", bd.gu);
  d.mat("hx", bd.hx);
  d.mat("hu", bd.hu);
  d.mat("wxx", bd.wxx);
  d.mat("wxu", bd.wxu);
  d.mat("wuu", bd.wuu);
  d.mat("grad_lag", bd.grad_lag);
  // augmented + condensed
  AugmentedSystem sys = assemble_augmented(nlp, it, mu, bd);
  d.mat("sigma_x", sys.sigma_x);
  d.vec("sigma_u", sys.sigma_u);
  d.mat("sigma_s", sys.sigma_s);
  d.mat("r1x", sys.r1x);
  d.vec("r1u", sys.r1u);
  d.mat("r2", sys.r2);
  d.mat("r3", sys.r3);
  d.mat("r4", sys.r4);
  CondenseWork work = make_condense_work(plan);
  CondensedSystem c = condense(sys, work);
  d.pat("kxx_p", c.kxx_p);
  d.pat("kxu_p", c.kxu_p);
  d.pat("kuu_p", c.kuu_p);
  d.mat("kxx", c.kxx);
  d.mat("kxu", c.kxu);
  d.mat("kuu", c.kuu);
  d.mat("rhat1", c.rhat1);
  d.vec("rhat2", c.rhat2);
  d.mat("rhat3", c.rhat3);
  // reduced system at delta_w = 0 (and at a positive delta_w)
  Partition part = partition(dm.N, 1);
  std::vector<BlockDiagFactor> facts;
  facts.push_back(factor_gx_range(c, 0, dm.N));
  for (double dw : {0.0, 1e-4}) {
    c.delta_w = dw;
    ReducedSystem red = reduce(c, part, facts, o.n_batch, exec);
    const std::string sfx = dw == 0.0 ? "0" : "dw";
    d.mat("khat_" + sfx, red.khat);
    d.vec("rhs_" + sfx, red.rhs);
    if (dw == 0.0) d.manifest["counters"] = {red.counters.spsm, red.counters.spmm, red.counters.tiles};
  }
  d.scalar("dw_probe", 1e-4);
  // reduced-strategy step (fresh warm start)
  double dwl = 0;
  StepInfo info;
  Step st = compute_step(nlp, it, mu, bd, KktStrategy::reduced, o, exec, dwl, &info);
  d.mat("px", st.px);
  d.vec("pu", st.pu);
  d.mat("ps", st.ps);
  d.mat("pz", st.pz);
  d.mat("py", st.py);
  d.scalar("step_delta_w", info.delta_w);
  d.scalar("step_corrections", info.corrections);
  {
    AugmentedSystem s2 = assemble_augmented(nlp, it, mu, bd);
    s2.delta_w = info.delta_w;
    d.scalar("step_residual", augmented_step_residual(s2, st));
  }
  d.finish();
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: bipm_ref solve|dump --case F --N n ...\n");
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    Args a = parse_args(argc, argv, 2);
    if (cmd == "solve") return cmd_solve(a);
    if (cmd == "dump") return cmd_dump(a);
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "bipm_ref: %s\n", e.what());
    return 1;
  }
}
