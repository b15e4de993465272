#!/usr/bin/env python3
"""ms per IPM iteration of the stochastic AC-OPF interior-point solve on the
reduced-space KKT path, B200 (this repo) vs the reference CPU implementation.

A *step* is one interior-point iteration of the solve (AD of the bundle,
condensation, batched G_x refactor, Schur reduction + inertia loop, dense
Cholesky, recovery, refinement, globalisation), iterations warmup..warmup+steps-1
of a fresh solve (a converged solve restarts).  Workload: case1354pegase with
256 scenarios, the configuration north_star's target is stated on (BASELINE.json
configs[2]); it fits one B200 (~0.6 GB resident), so N=1 runs it whole and
--gpus N shards its scenarios (override with --case/--scenarios, e.g. configs[1]
= case118 / 64).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--comm nccl|gloo]

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).  Rank r drives GPU
r mod device_count; --comm gloo exchanges through host-staged gloo all-reduces
instead of NCCL, so N ranks can share one GPU (the two-rank strong-scaling
path on a one-GPU box).

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per IPM iteration & total solve time (case, N scenarios) at 1/2/4/8 B200"
DATA_DIR = os.path.join(ROOT, "paper_2301_04869_b200", "data")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "bipm_ref")
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def run_reference_solve(case, N, sigma, seed, max_iter, threads):
    """The reference's own solver (oracle/_ref: reference sources compiled
    unchanged; Eigen SparseLU restated, see oracle/stubs) on host cores."""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    cmd = [REF_BIN, "solve", "--case", os.path.join(DATA_DIR, case + ".m"), "--N", str(N),
           "--sigma", str(sigma), "--seed", str(seed), "--groups", str(min(threads, N)),
           "--workers", str(threads), "--max-iter", str(max_iter)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, check=True)
    return json.loads(r.stdout)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        time.sleep(0.25)
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def algorithmic_bytes(p, info, group, M):
    """Algorithmic bytes per launch of a kernel group (SURVEY.md §8(d) model;
    DESIGN.md 'Roofline')."""
    nnz = {k: len(p.array(k + "_p_colind")) for k in ("gx", "gu", "hx", "hu", "wxx", "wxu", "wuu",
                                                       "kxx", "kxu", "kuu")}
    n_x, n_u, m = p.n_x, p.n_u, p.m
    nnz_f = info["nnz_f"]
    if group == "reduce_tiles":
        per = 7 * n_x * n_u * 8 + 2 * nnz_f * 12 + (nnz["gu"] + nnz["kxx"] + nnz["kxu"] +
                                                     nnz["kuu"]) * 12
        return M * per + n_u * n_u * 8  # one K_hat per GPU (G n_u^2 8)
    if group == "lu_refactor":
        return M * (nnz["gx"] + nnz_f) * 8
    if group in ("reduce_rhs", "recover_state"):
        return M * (2 * nnz_f * 8 + (nnz["kxx"] + nnz["kxu"] + nnz["gu"]) * 12 + 6 * n_x * 8)
    if group == "cholesky":
        return 2 * n_u * n_u * 8
    if group == "condense":
        return M * 8 * (nnz["wxx"] + nnz["wxu"] + nnz["wuu"] + nnz["hx"] + nnz["hu"] + m +
                        nnz["kxx"] + nnz["kxu"] + nnz["kuu"])
    if group in ("ad_bundle", "ad_values"):
        outs = sum(nnz[k] for k in ("gx", "gu", "hx", "hu", "wxx", "wxu", "wuu"))
        return M * 8 * (outs + n_x + m + (n_x + n_u) + 1 + 2 * n_x + m + 2 * p.nbus + p.nbranch)
    return 0


def ncu_traffic(workload, group):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return j.get(workload, {}).get(group, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


def bench_ours(a, rank, world):
    import torch
    from paper_2301_04869_b200 import _native as nat

    ndev = max(1, torch.cuda.device_count())
    dev = int(os.environ.get("LOCAL_RANK", "0")) % ndev
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if a.comm == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    from paper_2301_04869_b200.distributed import sharded_context

    def max_over_ranks(v: float) -> float:
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64,
                         device="cuda" if a.comm == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    case_file = os.path.join(DATA_DIR, a.case + ".m")
    workload = f"{a.case}_N{a.scenarios}"
    p = nat.Problem(case_file, a.scenarios, a.sigma, a.seed)
    # one scenario group per rank; K_hat / rhs / norms all-reduced (NCCL over
    # NVLink, or host-staged gloo)
    ctx = sharded_context(p, world, rank, device=dev, backend=a.comm)
    comm = ctx.comm_info()
    info = ctx.info()
    solver = nat.Solver(ctx)
    solver.start()
    for _ in range(a.warmup):
        solver.step_timed()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    ctx.profile(True)
    c0 = nat.counters()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(dev) as clk:
        for k in range(a.steps):
            flush.fill_(float(k))  # L2 flush between timed iterations (untimed)
            torch.cuda.synchronize()
            _, ms = solver.step_timed()
            times.append(ms)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    c1 = nat.counters()
    groups = ["ad_bundle", "ad_values", "condense", "lu_refactor", "reduce_pre", "reduce_tiles", "reduce_post", "reduce_rhs",
              "cholesky", "recover_state"]
    kt = {g: ctx.kernel_time(g) for g in groups}
    ctx.profile(False)
    total_ms = max_over_ranks(sum(times))
    ms_per_step = total_ms / a.steps

    # end to end through the public C-ABI with host buffers: context upload
    # (H2D of model + plans), full solve, result download (D2H).  The timed
    # context is released first (its device memory is recycled, as a user's
    # next solve would)
    info_keep, M_local = info, ctx.hi - ctx.lo
    del solver, ctx
    import gc
    gc.collect()
    torch.cuda.synchronize()
    # a.e2e_runs full solves, each with a fresh context; the median is
    # reported (single runs vary by ~10 % on the host side), all are listed
    runs = []
    for r in range(max(1, a.e2e_runs)):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        h0_r = nat.counters()
        t0 = time.perf_counter()
        ctx2 = sharded_context(p, world, rank, device=dev, backend=a.comm)
        torch.cuda.synchronize()
        t_ctx_r = time.perf_counter() - t0
        t_s = time.perf_counter()
        sol2 = nat.Solver(ctx2)
        t_setup_r = time.perf_counter() - t_s
        res = sol2.solve()
        torch.cuda.synchronize()
        e2e_r = time.perf_counter() - t0
        del sol2
        h1_r = nat.counters()
        e2e_r = max_over_ranks(e2e_r)
        # each run keeps its own iteration count and result
        runs.append((e2e_r, t_ctx_r, h0_r, h1_r, t_setup_r, res))
        del ctx2
        gc.collect()
    e2e_s, t_ctx, h0, h1, t_setup, res = sorted(runs, key=lambda x: x[0])[len(runs) // 2]
    iters = max(1, res["iterations"])

    # the Schur reduction is three kernels since round 2: reduce_pre
    # (reach_solve + gemm_tn, the forward half for all columns) and the
    # streamed tile kernel; its roofline covers both (one launch of each per
    # reduction, SURVEY §8(d) model for the whole reduction)
    kr = dict(kt)
    for extra in ("reduce_pre", "reduce_post"):
        if kr.get(extra, (0.0, 0))[1] > 0:
            x_ms, _ = kr.pop(extra)
            kr["reduce_tiles"] = (kr["reduce_tiles"][0] + x_ms, kr["reduce_tiles"][1])
        else:
            kr.pop(extra, None)
    dom = max(kr, key=lambda g: kr[g][0])
    dom_ms, dom_n = kr[dom]
    peak, peak_kind = peaks()
    algo = algorithmic_bytes(p, info_keep, dom, M_local)
    achieved = (algo / (dom_ms / dom_n * 1e-3)) / 1e9 if dom_n else 0.0
    line = {
        "metric": METRIC, "value": round(ms_per_step, 4), "unit": "ms/iteration",
        "n_gpus": world, "devices_used": min(world, ndev), "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(ms_per_step, 4), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic MATPOWER replica {a.case} (reference proj/data, gen_cases.py), "
                f"N={a.scenarios} load scenarios N(1,{a.sigma}^2) seed {a.seed}",
        "config": {"workload": workload, "case": a.case, "scenarios": a.scenarios,
                   "sigma": a.sigma, "seed": a.seed,
                   "parallelism": "1 GPU" if world == 1 else
                   f"dp{world}: scenario groups per rank, {a.comm} all-reduce of K_hat/rhs/norms"
                   + ("" if world <= ndev else f", {world} ranks on {ndev} GPU(s)"),
                   "step": "one IPM iteration (iterations warmup.. of a fresh solve)",
                   "l2": "flushed (256 MiB write) before every timed iteration"},
        "total_solve_s": round(res["t_total"], 5), "iterations": res["iterations"],
        "objective": res["objective"], "status": res["status_name"],
        "clocks": clk.summary(),
        "e2e": {"value": round(1e3 * e2e_s / iters, 4), "unit": "ms/iteration",
                "total_s": round(e2e_s, 5), "context_upload_s": round(t_ctx, 5),
                "solver_setup_s": round(t_setup, 5), "solver_t_total_s": round(res["t_total"], 5),
                "runs_s": [round(x[0], 4) for x in runs], "reported": "median",
                "h2d_bytes_per_step": int((h1["h2d_bytes"] - h0["h2d_bytes"]) / iters),
                "d2h_bytes_per_step": int((h1["d2h_bytes"] - h0["d2h_bytes"]) / iters)},
        "gpu_launches": int(c1["launches"] - c0["launches"]),
        "comm": comm,
        "roofline": {"kernel": dom + ("".join(f" + {x}" for x in ("reduce_pre", "reduce_post")
                                              if dom == "reduce_tiles" and kt.get(x, (0, 0))[1])),
                     "bound": "hbm", "achieved": round(achieved, 2),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 5),
                     "peak_kind": peak_kind, "traffic": ncu_traffic(workload, dom),
                     "algorithmic_bytes_per_launch": algo,
                     "avg_launch_ms": round(dom_ms / max(1, dom_n), 5)},
        "kernel_ms_per_step": {g: round(v[0] / a.steps, 4) for g, v in kt.items()},
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline and os.path.exists(REF_BIN):
        # the same iteration window as the GPU value (iterations warmup..),
        # bounded to cpu_iters timed iterations (~10-30 s of host work)
        cores = cpu_cores()
        n_cpu = max(1, min(a.cpu_iters, a.steps))
        j = run_reference_solve(a.case, a.scenarios, a.sigma, a.seed, a.warmup + n_cpu, cores)
        logs = j["logs"][a.warmup:a.warmup + n_cpu] or j["logs"][-1:]
        ms = 1e3 * sum(l["t_total"] for l in logs) / len(logs)
        line["cpu_baseline"] = {
            "value": round(ms, 3), "unit": "ms/iteration", "cores": cores, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"iterations {a.warmup}..{a.warmup + len(logs) - 1} of the reference "
                      f"solve of {workload} (IterationLog.t_total; {j['iterations']} run), "
                      f"--groups/--workers {cores}; Eigen SparseLU restated in oracle/stubs",
            "iterations_timed": len(logs)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_reference(a, rank, world):
    if rank != 0:
        return
    workload = f"{a.case}_N{a.scenarios}"
    cores = cpu_cores()
    j = run_reference_solve(a.case, a.scenarios, a.sigma, a.seed, a.warmup + a.steps, cores)
    logs = j["logs"][a.warmup:a.warmup + a.steps] or j["logs"]
    ms = 1e3 * sum(l["t_total"] for l in logs) / len(logs)
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/iteration", "n_gpus": world,
        "steps": len(logs), "warmup": a.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": f"synthetic MATPOWER replica {a.case}, N={a.scenarios}, sigma {a.sigma}, seed {a.seed}",
        "config": {"workload": workload, "case": a.case, "scenarios": a.scenarios,
                   "sigma": a.sigma, "seed": a.seed, "parallelism": f"{cores} host threads",
                   "step": "one IPM iteration (reference IterationLog.t_total)"},
        "cpu_baseline": {"value": round(ms, 4), "unit": "ms/iteration", "cores": cores,
                         "kind": "reference", "cpu_model": cpu_model(),
                         "sample": f"iterations {a.warmup}..{a.warmup + len(logs) - 1} of the "
                                   f"reference solve (--groups/--workers {cores}); Eigen "
                                   "SparseLU restated in oracle/stubs"},
        "e2e": {"value": round(ms, 4), "unit": "ms/iteration", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "status": j["status"], "iterations_run": j["iterations"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--case", default="case1354pegase")
    ap.add_argument("--scenarios", type=int, default=256)
    ap.add_argument("--sigma", type=float, default=0.05)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-iters", type=int, default=3,
                    help="timed iterations of the CPU baseline sample, after the same warm-up "
                         "iterations as the GPU value (bounded: ~10-30 s of host work)")
    ap.add_argument("--comm", choices=["nccl", "gloo"], default="nccl",
                    help="cross-rank exchange: NCCL (one GPU per rank) or host-staged gloo "
                         "(ranks may share a GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-runs", type=int, default=3,
                    help="end-to-end solves (fresh context each); the median is reported")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        # --gpus N outside torchrun: re-launch under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl == "reference":
        bench_reference(a, rank, world)
    else:
        bench_ours(a, rank, world)


if __name__ == "__main__":
    main()
