// Host-only dump of the streamed-reduction step program (sizes, ring waits).
// g++ -std=c++20 -O2 -I paper_2301_04869_b200/csrc tools/stream_plan_dump.cpp \
//   paper_2301_04869_b200/_lib/obj/host/*.o -o /tmp/spd
#include <cstdio>
#include <cstdlib>
#include <map>

#include "host/grid_model.hpp"
#include "host/plan.hpp"
#include "host/stream_plan.hpp"

using namespace bipm;

int main(int argc, char** argv) {
  GridCase cs = read_matpower_file(argv[1]);
  ScenarioDraw sc = draw_scenarios(cs, 2, 0.05, {}, 0);
  OpfModel M = build_opf_model(cs, sc);
  LaneDeps deps = basis_deps(M);
  DerivPlan D = make_deriv_plan(M, deps);
  LuPlan L = make_lu_plan(D.g.x);
  const int K = argc > 2 ? atoi(argv[2]) : 8, ring = argc > 3 ? atoi(argv[3]) : 51616;
  StreamProgram S = build_stream_program(L, D.g.u, D.kxx.out, D.kxu.out, M.n_u, K, 512, ring, 24);
  std::map<int, int> wd;
  long long bytes = 0;
  for (auto& is : S.issue) {
    wd[is.wait_delta]++;
    bytes += is.pat_bytes + (is.val_count ? ((is.val_count + 1) * 8 + 15) / 16 * 16 : 0) +
             (is.x_count ? ((is.x_count + 1) * 8 + 15) / 16 * 16 : 0);
  }
  printf("steps %d ring %d max_step %d bytes/scenario %lld nnz_vs %d nq %d\n", S.steps, ring,
         S.max_step_bytes, bytes, S.nnz_vs, S.nq);
  printf("sweep %d dense %d acc %d spmv %d\nwait_delta histogram:", S.n_sweep_steps,
         S.n_dense_steps, S.n_acc_steps, S.n_spmv_steps);
  for (auto [k, v] : wd) printf(" %d:%d", k, v);
  printf("\n");
}
