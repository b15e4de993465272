// Device engine: one GPU owning scenarios [lo, hi) of a problem.
//
// Host plans (patterns, gather programs, the LU plan) are uploaded once; the
// per-scenario values (bundle, condensed blocks, factors) stay resident in
// HBM in the reference's scenario-major layout.  The operator methods mirror
// the reference's reduced-strategy operators (kkt.hpp:110-162,
// linalg.hpp:116) and run entirely on the device stream.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../host/ad_plan.hpp"
#include "../host/grid_model.hpp"
#include "../host/plan.hpp"
#include "../host/stream_plan.hpp"
#include "../kernels/ad_launch.hpp"
#include "../kernels/kkt_kernels.hpp"
#include "../kernels/reach_gemm.hpp"
#include "../kernels/reduce_stream.hpp"
#include "comm.hpp"
#include "device_array.hpp"

namespace bipm {

// Host model + symbolic plans.  Two ways in:
//  * from an OPF case (file or the reference's CaseData / ScenarioSet tables):
//    everything, including the basis kernel's data the AD needs;
//  * from the derivative patterns alone (from_patterns): the KKT operators
//    only (condense, refactor, reduce, recover, solve_reduced) -- what a
//    reference solve needs when its own AD and IPM call the GPU for
//    solve_reduced.
struct Problem {
  GridCase cs;
  ScenarioDraw sc;
  OpfModel M;  // dims only when built from patterns
  LaneDeps deps;
  DerivPlan D;
  LuPlan LU;
  AdProgram AD;
  bool model = true;
  bool has_model() const { return model; }
  static std::unique_ptr<Problem> from_case_file(const std::string& path, idx N, double sigma,
                                                 std::uint64_t seed,
                                                 const std::vector<idx>& contingencies = {});
  static std::unique_ptr<Problem> from_parts(GridCase cs, ScenarioDraw sc);
  // N scenarios sharing G_x | G_u (n_x x n_x | n_x x n_u), H_x | H_u (m x .)
  // and the Lagrangian Hessian blocks W_xx, W_xu, W_uu
  static std::unique_ptr<Problem> from_patterns(idx N, Csr gx, Csr gu, Csr hx, Csr hu, Csr wxx,
                                                Csr wxu, Csr wuu);
};

struct DevPattern {
  DArr<int> ptr, ind, t_ptr, t_row, t_slot;
  DevCsr v{};
  void upload(const Csr& p);
};

struct DevCondense {
  DArr<int> w_of, ptr, ka, kb, r;
  CondenseDev v{};
  void upload(const CondenseProgram& p);
};

class Engine {
 public:
  Engine(const Problem& pb, int device, idx lo, idx hi);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Problem& pb;
  const idx lo, hi, M;
  std::unique_ptr<Comm> comm;  // null: single GPU (no exchange)
  // exchange through comm; BIPM_FORCE_COMM=1 also routes a one-rank
  // communicator through it (tests the NCCL path on a single GPU)
  bool force_comm = false;
  bool multi() const { return comm && (comm->size() > 1 || force_comm); }
  int device = 0, sm_count = 148;
  cudaStream_t st = nullptr;

  // ---- uploaded plans
  DevPattern gx_p, gu_p, hx_p, hu_p, kxx_p, kxu_p, kuu_p, wxx_p, wxu_p, wuu_p;
  DevCondense cxx, cxu, cuu;
  std::vector<DArr<int>> lu_arrays;
  DevLu lu{};

  // ---- derivative bundles ([M][len]); the IPM keeps the iterate's and a
  // trial point's and swaps them on acceptance (ipm.cpp:204-205, 545)
  struct Bundle {
    DArr<double> f, g, h, gx, gu, hx, hu, wxx, wxu, wuu, grad;
  };
  Bundle bundles[2];
  int cur = 0;
  Bundle& bd() { return bundles[cur]; }
  Bundle& trial() { return bundles[1 - cur]; }
  void swap_bundles() {
    cur = 1 - cur;
    invalidate_reach();
  }
  // AD program + scratch
  std::vector<DArr<int>> ad_i;
  std::vector<DArr<double>> ad_d;
  DevAd ad{};
  DArr<double> psi, dpart, wlane, contrib;  // element-major AD scratch
  DArr<double> xt, yt, zt;                   // element-major copies of the AD inputs
  DArr<int> bad;
  DArr<double> pd_v, qd_v, status_v;
  DArr<double> kxx, kxu, kuu;                  // condensed blocks
  DArr<double> sigma_x, sigma_s, rhat1, rhat3, r2, r4;
  DArr<double> sigma_u, rhat2;                 // n_u (replicated)
  DArr<double> F, FT, Dt;                      // LU factors [M][nnz_f], transposed, dense tails
  DArr<double> lu_scale, rhs_scratch;         // refactor guard scale [M]; single-RHS [M][2 n_x]
  DArr<int> lu_status;
  // ---- streamed reduction (reduce_stream.cu): step program, sweep-ordered
  // factor values, column-order K_xu / G_u copies
  bool use_stream = true;
  StreamProgram sprog;
  StreamLaunch sl{};
  DArr<int> sp_pat, sp_issue, sp_ring, sp_vs_src, sp_kxu_slot, sp_gu_slot, kuu_row, kuu_col;
  DArr<double> VS, Dp, kxu_t, gu_t, sp_scratch;  // Dp: W, W' with padded rows
  // presolved forward half (host/stream_plan.hpp ReachPlan, reach_gemm.cu):
  // y_N [M][nnz_yn], y_T and X_T = W y_T [M][n_u][ldy]; BIPM_PRESOLVE=0 runs
  // the L sweep and the first dense product inside every column tile instead
  bool presolve = true;
  bool adj_identity = false;  // adjoint half via y_N' z_N + X_T' z_T (stream_plan.hpp)
  ReachPlan rplan;
  ReachDev rdev{};
  DArr<int> rp_op_ptr, rp_ops, rp_ent, rp_yn_ptr, rp_yn_row, rp_yt_ptr, rp_yt_row;
  bool xt_sparse = true;  // X_T = W y_T over y_T's pattern (BIPM_XT_SPARSE=0: dense DMMA GEMM)
  int dp_slot() const;    // which of Dp's W / W' slots the reduction reads (-1: both)
  // the reach solve (y_N, y_T) of the current factor and G_u, issued on
  // st_rhs right after the refactor's non-tail levels so it runs beside the
  // dense-tail Gauss-Jordan (whose second wave leaves SMs idle); reduce_local
  // waits on ev_reach.  Invalidated when G_u changes (operator uploads,
  // bundle swap) -- reduce_local then solves it on st itself.
  bool reach_ready = false;
  cudaEvent_t ev_levels = nullptr, ev_reach = nullptr;
  void launch_reach_async();
  void invalidate_reach();
  bool reach_overlap() const;
  DArr<double> YN, YT, XT, ZT;
  // adjoint identity with a deferred tail: -sum_s X_T' Z_T by one batch-sum
  // GEMM into tail_splits slabs after the kuu slab (BIPM_TAIL_DEFER=0: the
  // product runs inside every tile instead)
  bool defer_tail = true;
  int tail_splits = 0;
  int red_parts = 0;  // partial K_hat slabs summed by finish_reduce
  // ---- reduction workspace (tile kernel, BIPM_REDUCE=tiles)
  ReduceLaunch red{};
  DArr<double> red_partial, red_scratch, rhs_part;
  DArr<double> khat, rhs;   // n_u x n_u (column-major), n_u
  DArr<long long> phase;    // optional reduction phase stamps (debug)
  DArr<int> chol_info;

  // ---- operators (device-resident inputs/outputs)
  // eval_bundle_range (autodiff.cpp:484-516) into `out`; returns the lowest
  // global scenario index with a non-finite basis / derivative, or -1.
  // check=false only launches: the per-scenario flags stay in `bad` for a
  // later fused reduction (Solver::kkt_eval) and -1 is returned
  idx eval_bundle(Bundle& out, const double* dX, const double* du, const double* dY,
                  const double* dZ, double obj_w, bool check = true);
  // batch_eval (autodiff.cpp:256-281): f, g, h only
  idx eval_values(const double* dX, const double* du, double* df, double* dg, double* dh);
  // factor_gx_range (kkt.cpp:190-196): returns the lowest singular global
  // scenario index or -1.
  idx factor_gx();
  void factor_gx_launch();  // refactor only; statuses stay in lu_status
  // condense (kkt.cpp:123-170) of the K blocks from the bundle and sigma_s
  void condense_blocks(cudaStream_t on = nullptr);
  void condense_launch(cudaStream_t on = nullptr);
  // local part of reduce (kkt.cpp:371-466): khat/rhs partial sums over the
  // owned scenarios, without the sigma_u / rhat2 terms.
  void reduce_local(double delta_w);
  // rhs of the reduced system from (rhat1, rhat3) (defaults: the engine's)
  void reduce_rhs_local(double delta_w, double* d_rhs_out, const double* d_rhat1 = nullptr,
                        const double* d_rhat3 = nullptr);
  // the same with the engine's rhat1/rhat3, issued on st_rhs after everything
  // already queued on st (fork) so it runs beside the next launches on st
  // (the Schur reduction); reduce_rhs_join orders st after it and does the
  // cross-rank sum.  Without overlap_rhs: reduce_rhs_local.
  void reduce_rhs_fork(double delta_w, double* d_rhs_out);
  void reduce_rhs_join(double* d_rhs_out);
  // finish_reduce (kkt.cpp:468-488): K_hat = sum of the partial tiles (all
  // ranks) + diag(sigma_u + delta_w)
  void finish_reduce(double delta_w);
  // shift + Cholesky (kkt.cpp:965-971); true when the reference would accept
  // the attempt.  A Cholesky failure at a pivot within rounding of zero is
  // decided by the Bunch-Kaufman inertia of K_hat instead (linalg.cpp:136-145,
  // dense_bk.cu): K_hat is re-summed from the partial slabs (finish_reduce at
  // dw) and the attempt is accepted, and later solved with the LDL' factors,
  // iff BK reports neg = 0 and zero = 0.  BIPM_FORCE_BK=1 takes that path on
  // every Cholesky failure (tests).
  // regenerate: writes K_hat again for the Bunch-Kaufman factorisation
  // (default: finish_reduce(dw) from the partial slabs)
  bool factor_khat(double dw, const std::function<void()>& regenerate = {});
  void solve_khat(double* d_vec);
  bool khat_bk = false;       // the accepted factor is Bunch-Kaufman (else Cholesky)
  bool force_bk = false;
  long long bk_fallbacks = 0;  // borderline attempts decided by the BK inertia
  DArr<int> bk_ipiv, bk_inertia;
  DArr<unsigned char> bk_state;
  // recover_state_adjoint + recover_slack_dual (kkt.cpp:507-532, :172-188)
  void recover(double delta_w, const double* d_pu, double* d_px, double* d_py, double* d_pz,
               double* d_ps, const double* d_rhat1 = nullptr, const double* d_rhat3 = nullptr,
               const double* d_r2 = nullptr, const double* d_r4 = nullptr);

  void sync();
  void upload_ad();
  void setup_stream();

  // optional CUDA-event timing of named kernel groups: an event pair around
  // each launch, no host synchronisation (the GPU keeps its queue); pairs are
  // resolved into ktimers when read (resolve_timers)
  struct KTimer {
    double ms = 0;
    long long n = 0;
  };
  bool profiling = false;
  std::map<std::string, KTimer> ktimers;
  struct PendingTimer {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<PendingTimer> pending_timers;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t take_event();
  void resolve_timers();
  template <typename F>
  void timed(const char* name, F&& launch, cudaStream_t on = nullptr) {
    if (!profiling) {
      launch();
      return;
    }
    if (!on) on = st;
    cudaEvent_t a = take_event(), b = take_event();
    cudaEventRecord(a, on);
    launch();
    cudaEventRecord(b, on);
    pending_timers.push_back({name, a, b});
    if (pending_timers.size() >= 256) resolve_timers();
  }
  // side stream for the reduced rhs, overlapped with the Schur reduction
  cudaStream_t st_rhs = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool overlap_rhs = true;
  idx first_bad();
  size_t nnz(const Csr& c) const { return size_t(c.nnz()); }
};

}  // namespace bipm
