"""Per-event trace of the streamed reduction (CTA (0,0), thread 0, first
scenario).  Usage: python tools/trace_reduce.py case N"""
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
P = ctx.info()["steps"]
buf = ctx.debug_buffer()
n = buf[2 * P + 1]
ev = [(buf[2 * P + 2 + 2 * i], buf[2 * P + 3 + 2 * i]) for i in range(n)]
t0 = ev[0][1]
print(json.dumps({"P": P, "events": [(c, t - t0) for c, t in ev]}))
