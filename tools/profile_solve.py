"""Full GPU solve with per-kernel-group CUDA-event timing.
Usage: python tools/profile_solve.py case N [sigma] [max_iter]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_04869_b200 import _native as nat  # noqa: E402

case, N = sys.argv[1], int(sys.argv[2])
sigma = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
max_iter = int(sys.argv[4]) if len(sys.argv) > 4 else 300
t0 = time.time()
p = nat.Problem(os.path.join(ROOT, "paper_2301_04869_b200/data", case + ".m"), N, sigma, 0)
t1 = time.time()
ctx = nat.Context(p)
t2 = time.time()
info = ctx.info()
s = nat.Solver(ctx, max_iter=max_iter)
r = s.solve()  # warm (first solve includes lazy CUDA init)
ctx.profile(True)
t3 = time.time()
r = s.solve()
t4 = time.time()
groups = ["ad_bundle", "ad_values", "condense", "lu_refactor", "reduce_pre", "reduce_tiles", "reduce_post", "reduce_rhs",
          "cholesky", "khat_solve", "recover_state"]
kt = {g: ctx.kernel_time(g) for g in groups}
it = r["iterations"]
out = {"case": case, "N": N, "n_x": p.n_x, "n_u": p.n_u, "m": p.m, "status": r["status_name"],
       "iterations": it, "objective": r["objective"], "solve_s": t4 - t3,
       "ms_per_iter": 1e3 * (t4 - t3) / it, "problem_setup_s": t1 - t0, "ctx_setup_s": t2 - t1,
       "reductions": r["reductions"], "info": info,
       "kernels_ms_total": {g: round(v[0], 3) for g, v in kt.items()},
       "kernels_count": {g: v[1] for g, v in kt.items()}}
print(json.dumps(out))
