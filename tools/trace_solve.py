"""Step a GPU solve and print its log next to a reference log until the end or
the first error.  Usage: python tools/trace_solve.py case N [golden_file]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_04869_b200 import _native as nat  # noqa: E402

case, N = sys.argv[1], int(sys.argv[2])
gold = sys.argv[3] if len(sys.argv) > 3 else "solves_large.json"
ref = json.load(open(os.path.join(ROOT, "tests/golden", gold)))[f"{case}_N{N}_s0.05_seed0"]["logs"]
p = nat.Problem(os.path.join(ROOT, "paper_2301_04869_b200/data", case + ".m"), N, 0.05, 0)
s = nat.Solver(nat.Context(p))
s.start()
k = 0
while True:
    try:
        st = s.step()
    except nat.BipmError as e:
        print("ERROR at iteration", k, e)
        break
    a, b = s.log(k), ref[k] if k < len(ref) else None
    print(f"{k:3d} obj {a['objective']:.10e} pr {a['inf_pr']:.2e} du {a['inf_du']:.2e} mu {a['mu']:.1e} "
          f"a {a['alpha_p']:.3e} c{int(a['corr'])} fs{int(a['full_step'])} | "
          + (f"{b['objective']:.10e} pr {b['inf_pr']:.2e} du {b['inf_du']:.2e} mu {b['mu']:.1e} a {b['alpha_p']:.3e} c{b['corr']}" if b else "-"))
    k += 1
    if st != -1:
        print("status", st)
        break
