"""Side-by-side per-iteration log of the GPU solver and the reference's
(committed in tests/golden/solves.json).  Usage:
  python tools/compare_solve.py case9 8 0.05 [max_rows]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_04869_b200 import _native as nat  # noqa: E402

case, N, sigma = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
rows = int(sys.argv[4]) if len(sys.argv) > 4 else 400
ref = json.load(open(os.path.join(ROOT, "tests/golden/solves.json")))[f"{case}_N{N}_s{sigma}_seed0"]
p = nat.Problem(os.path.join(ROOT, "paper_2301_04869_b200/data", case + ".m"), N, sigma, 0)
ctx = nat.Context(p)
r = nat.Solver(ctx).solve()
print("GPU:", r["status_name"], r["iterations"], repr(r["objective"]), "t_total", r["t_total"])
print("REF:", ref["status"], ref["iterations"], repr(ref["objective"]))
for k in range(min(rows, max(len(r["logs"]), len(ref["logs"])))):
    a = r["logs"][k] if k < len(r["logs"]) else None
    b = ref["logs"][k] if k < len(ref["logs"]) else None
    fa = f"{a['objective']:.10e} pr {a['inf_pr']:.2e} du {a['inf_du']:.2e} mu {a['mu']:.1e} a {a['alpha_p']:.3e} c{int(a['corr'])} r{int(a['refinements'])} fs{int(a['full_step'])}" if a else "-"
    fb = f"{b['objective']:.10e} pr {b['inf_pr']:.2e} du {b['inf_du']:.2e} mu {b['mu']:.1e} a {b['alpha_p']:.3e} c{b['corr']}" if b else "-"
    print(f"{k:3d} | {fa} | {fb}")
import numpy as np
print("max |u - u_ref| / max(1,|u_ref|):", np.abs(r["u"] - np.array(ref["u"])).max() / max(1, np.abs(ref["u"]).max()))
