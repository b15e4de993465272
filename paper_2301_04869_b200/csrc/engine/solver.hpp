// Device-resident interior-point solver on the reduced KKT path.
//
// Control flow restates the reference driver (proj/core/src/ipm.cpp:435-664)
// and the reduced strategy (kkt.cpp:742-772 inertia loop, kkt.cpp:945-1006
// solve_reduced with up to three refinement rounds).  Every N-sized vector
// lives in HBM; the host only sees the scalars that steer control flow
// (norms, step sizes, merit values, factorisation status).
#pragma once

#include <array>
#include <chrono>
#include <string>
#include <vector>

#include "../kernels/ipm_kernels.hpp"
#include "engine.hpp"
#include "host_link.hpp"
#include "kkt_step.hpp"

namespace bipm {

struct SolverOptions {  // IpmOptions (ipm.hpp:7-25)
  double tol = 1e-6, mu0 = 1e-1, kappa_mu = 0.2, theta_mu = 1.5, tau = 0.995, kappa_eps = 10.0;
  int max_iter = 300;
  RegOptions reg;
  int refine_rounds = 3;
};

struct IterRecord {  // IterationLog (ipm.hpp:27-36)
  int iter = 0;
  double objective = 0, inf_pr = 0, inf_du = 0, complementarity = 0, mu = 0;
  double alpha_primal = 0, alpha_dual = 0;
  double t_ad = 0, t_kkt = 0, t_total = 0;
  int corrections = 0, refinements = 0;
  double delta_w = 0;
  bool full_step = false;
};

enum SolveStatusCode : int {
  kNotStarted = -2,
  kRunning = -1,
  kOptimal = 0,
  kMaxIter = 1,
  kInfeasible = 2,
  kLinFail = 3
};

class Solver {
 public:
  Solver(Engine& e, const SolverOptions& o);

  void start();      // initial_iterate (ipm.cpp:59-105)
  int step();        // one IPM iteration; returns a SolveStatusCode
  int solve();       // start + steps until done
  // one step bracketed by CUDA events on the engine stream (restarts the
  // solve first when it already terminated); returns the device ms
  double step_timed(int* st_out);

  int status = kNotStarted;  // step() before start() is an error
  int iter = 0;
  double mu = 0, delta_w_last = 0, objective = 0;
  std::vector<IterRecord> logs;
  double t_ad = 0, t_kkt = 0, t_total = 0;
  long long reductions = 0;  // K_hat assemblies (every inertia attempt)
  std::string message;

  // host copies of the current iterate (stream-ordered after the queued work)
  std::vector<double> host_u();
  std::vector<double> host_x();
  // every array of the current primal-dual point (Iterate, model.hpp:41-55):
  // x, u, s, y, z, kappa_lo, kappa_up, nu_lo, nu_up, lambda_lo, lambda_up
  void host_iterate(double* const out[11]);

 private:
  struct Scaled {
    double total, stationarity, primal, comp, comp_raw;
  };
  struct IterStore {
    DArr<double> x, u, s, y, z, klo, kup, nlo, nup, llo, lup;
    DevIter view();
  };
  // one fused residual pass at mus[0..3]; bad flags of the last bundle
  // evaluation are folded in when check_bad (lowest non-finite scenario)
  struct ErrEval {
    double stat, primal, comp[4], mult, obj;
    idx bad;
  };
  ErrEval kkt_eval(const DevIter& it, Engine::Bundle& bd, const double mus[4], bool check_bad);
  Scaled scaled_of(const ErrEval& E, int k) const;
  // assemble_augmented on the device, then solve_reduced (kkt.cpp:945-1006)
  void compute_step(const DevIter& it);
  double fetch1(const double* d) { return io.fetch1(d); }
  template <int K>
  std::array<double, K> fetch(const double* d) {
    return io.fetch<K>(d);
  }
  void allred(double* d, size_t n, RedOpKind op) { io.allred(d, n, op); }
  idx global_first_bad(idx local_bad) { return io.global_first_bad(local_bad); }
  double now() const;

  Engine& e;
  SolverOptions o;
  HostLink io;
  KktStep kkt;
  IpmDims d{};
  DevBounds b{};
  DArr<double> xlo, xup, ulo, uup, slo, sup;
  IterStore its[2];
  int icur = 0;
  DevIter cur() { return its[icur].view(); }
  DevIter alt() { return its[1 - icur].view(); }
  bool bundle_fresh = false;
  double mult_count = 0;
  DArr<double> gsum_u;
  DArr<double> bsv[6];
  DArr<double> ft, gt, ht;  // line-search trial values
  DArr<double> partial, scal;
  DArr<int> flag;
  DArr<unsigned int> eval_counter;
  std::chrono::steady_clock::time_point t0_;
};

}  // namespace bipm
