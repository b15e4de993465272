"""Micro-benchmark of the Schur reduction alone (CUDA-event kernel time) on a
case's real patterns with seeded synthetic values.
Usage: python tools/micro_reduce.py case N [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2301_04869_b200 import _native as nat  # noqa: E402
from test_gpu_kkt import synthetic_condensed  # noqa: E402

case, N = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = nat.Problem(os.path.join(ROOT, "paper_2301_04869_b200/data", case + ".m"), N, 0.05, 0)
v = synthetic_condensed(p, N, seed=7)
ctx = nat.Context(p)
ctx.factor_gx(v["gx"])
args = {k: v[k] for k in v if k != "gx"}
ctx.reduce(0.5, **args)  # warm
ctx.profile(True)
for _ in range(reps):
    ctx.reduce(0.5, **args)
ctx.factor_gx(v["gx"])
out = {g: ctx.kernel_time(g) for g in ("reduce_pre", "reduce_tiles", "reduce_post", "reduce_rhs", "lu_refactor")}
ctx.profile(False)
print(json.dumps({"case": case, "N": N, "info": ctx.info(), "tl": int(p.array("lu_shape")[4]),
                  "ms_per_call": {g: (t / max(1, n)) for g, (t, n) in out.items()}}))

# per-step-kind breakdown of CTA (0,0), first scenario (clock64 cycles)
info = ctx.info()
if info.get("streamed"):
    ctx.step_stamps(True)
    ctx.reduce(0.5, **args)
    st = ctx.step_stamps(False)
    names = {0: "scatter", 1: "sweep", 2: "dense", 3: "acc", 4: "spmv", 5: "copyback"}
    by, cnt, wait = {}, {}, {}
    for (k, t0, w0), (_, t1, _) in zip(st[:-1], st[1:]):
        nm = names.get(k, k)
        by[nm] = by.get(nm, 0) + (t1 - t0)
        wait[nm] = wait.get(nm, 0) + (w0 - t0)
        cnt[nm] = cnt.get(nm, 0) + 1
    print(json.dumps({"step_cycles": by, "wait_cycles": wait, "steps": cnt,
                      "total": st[-1][1] - st[0][1],
                      "cycles_per_step": {k: round(by[k] / cnt[k]) for k in by}}))
    print(json.dumps({"per_step": [(k, t1 - t0, w0 - t0) for (k, t0, w0), (_, t1, _) in
                                   zip(st[:-1], st[1:])]}))
else:
    ctx.phase_stamps(True)
    ctx.reduce(0.5, **args)
    st = ctx.phase_stamps(True)
    names = ["scatter", "L-levels", "L-tailgather", "tail L+U", "U-levels", "spmv", "Ut-levels",
             "Ut-tailgather", "tail Ut+Lt", "Lt-levels", "GuY"]
    d = [st[i + 1] - st[i] for i in range(len(names)) if st[i + 1] > 0]
    print(json.dumps({"phase_cycles": dict(zip(names, d)), "total": st[len(d)] - st[0]}))
