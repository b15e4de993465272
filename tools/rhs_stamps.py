"""Phase breakdown (clock64, scenario 0) of the single-RHS reduced rhs kernel
on a case's real patterns with seeded synthetic values (debug).
Usage: python tools/rhs_stamps.py case N"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2301_04869_b200 import _native as nat  # noqa: E402
from test_gpu_kkt import synthetic_condensed  # noqa: E402

case, N = sys.argv[1], int(sys.argv[2])
p = nat.Problem(os.path.join(ROOT, "paper_2301_04869_b200/data", case + ".m"), N, 0.05, 0)
v = synthetic_condensed(p, N, seed=7)
ctx = nat.Context(p)
ctx.factor_gx(v["gx"])
args = {k: v[k] for k in v if k != "gx"}
ctx.reduce(0.5, **args)
ctx.step_stamps(True)
ctx.reduce(0.5, **args)
buf = ctx.debug_buffer()
st = [x for x in buf[-64:] if x > 0]
names = ["init", "L", "tail+W", "U", "spmv", "U'", "tail+W'", "L'", "acc"]
d = {names[i]: st[i + 1] - st[i] for i in range(min(len(names), len(st) - 1))}
print(json.dumps({"case": case, "N": N, "cycles": d, "total": st[-1] - st[0] if st else 0}))
