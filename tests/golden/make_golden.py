"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference (oracle/_ref/bipm_ref, built by oracle/Makefile
from /root/reference) and stores compressed fixtures:

  case9_N8_s005_it3.npz     case9, 8 scenarios, sigma 0.05, seed 0, iterate 3
  case118_N4_s005_it5.npz   case118, 4 scenarios, sigma 0.05, seed 0, iterate 5
  case118_N4_s005_it20.npz  same problem, iterate 20 (near convergence)
  solves.json               full reference solves (iterations, objective, logs)
  solves_large.json         case1354pegase / 256 full solve; case2869pegase / 512
                            capped at 4 iterations (per-iteration logs), 8 threads

Each .npz holds the model maps, patterns, the iterate, the derivative bundle,
the augmented and condensed systems, K_hat / rhs at delta_w in {0, 1e-4}
and the reduced-strategy step (see oracle/ref_driver.cpp).

Round-2 fixtures (``--iterates``, ``--dumps2``, ``--long``):

  iterates_*.npz            final primal/dual iterate of a full reference solve
                            (x, u, s, y, z, kappa_lo/up, nu_lo/up, lambda_lo/up;
                            Iterate, model.hpp:41-55): whole arrays for small
                            problems; for the pegase configs every array's
                            per-scenario inf-norm and +-1 projection checksum,
                            plus the full rows of a few sample scenarios
  case1354pegase_N4_s005_it40.npz   reduced-KKT fixture near convergence
  case9241pegase_N2_s005_it2.npz    reduced-KKT fixture at the largest config
  solves_large.json         adds case2869pegase / 512 (full solve) and
                            case9241pegase / 128 capped at 3 iterations

Usage: python tests/golden/make_golden.py   (needs /root/reference; run in
the build container, not on the GPU box)
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.fixtures import load_dump, save_npz  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "bipm_ref")
DATA = os.path.join(ROOT, "oracle", "_ref", "data")

DUMPS = [
    ("case9", 8, 0.05, 0, 3),
    ("case118", 4, 0.05, 0, 5),
    ("case118", 4, 0.05, 0, 20),
]
SOLVES = [
    ("case9", 8, 0.0, 0),
    ("case9", 8, 0.05, 0),
    ("case118", 4, 0.05, 0),
    ("case118", 64, 0.05, 0),
]


LARGE = [  # (case, N, sigma, seed, max_iter); run with --large (hours of CPU)
    ("case1354pegase", 256, 0.05, 0, 300),
    ("case2869pegase", 512, 0.05, 0, 4),
]


def large():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    path = os.path.join(HERE, "solves_large.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    threads = str(min(8, os.cpu_count() or 1))
    for case, N, sigma, seed, max_iter in LARGE:
        key = f"{case}_N{N}_s{sigma}_seed{seed}" + (f"_it{max_iter}" if max_iter < 300 else "")
        if key in out:
            continue
        r = subprocess.run([REF, "solve", "--case", f"{DATA}/{case}.m", "--N", str(N), "--sigma",
                            str(sigma), "--seed", str(seed), "--groups", threads, "--workers",
                            threads, "--max-iter", str(max_iter)],
                           check=True, env=env, capture_output=True, text=True)
        j = json.loads(r.stdout)
        out[key] = j
        print(key, j["status"], j["iterations"], j["objective"])
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


ITERATE_NAMES = ("x", "u", "s", "y", "z", "kappa_lo", "kappa_up", "nu_lo", "nu_up",
                 "lambda_lo", "lambda_up")
FULL_LIMIT = 400_000  # store whole arrays when the iterate is this small


def projection_signs(n: int) -> np.ndarray:
    """Deterministic +-1 weights of the per-scenario projection checksum."""
    return np.where(np.random.default_rng(12345).random(n) < 0.5, -1.0, 1.0)


def iterate_fixture(d: str) -> dict:
    """Compress a `bipm_ref solve --iterate-out` directory (see module doc)."""
    fx = load_dump(d)
    total = sum(fx[k].size for k in ITERATE_NAMES)
    out = {"objective": np.array([fx.meta["objective"]])}
    for k in ITERATE_NAMES:
        a = fx[k]
        if total <= FULL_LIMIT or a.ndim == 1:
            out[k] = a
            continue
        N = a.shape[0]
        rows = np.unique(np.array([0, 1, N // 2, N - 1]))
        w = projection_signs(a.shape[1])
        out[k + "__rows"] = rows
        out[k + "__sample"] = a[rows]
        out[k + "__absmax"] = np.abs(a).max(axis=1)
        out[k + "__proj"] = a @ w
        out[k + "__projabs"] = np.abs(a) @ np.ones(a.shape[1])
    return out


def ref_solve(case, N, sigma, seed, threads=1, max_iter=300, iterate_dir=None, cont=()):
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    cmd = [REF, "solve", "--case", f"{DATA}/{case}.m", "--N", str(N), "--sigma", str(sigma),
           "--seed", str(seed), "--groups", str(threads), "--workers", str(threads),
           "--max-iter", str(max_iter)]
    if cont:
        cmd += ["--contingencies", ",".join(str(c) for c in cont)]
    if iterate_dir:
        cmd += ["--iterate-out", iterate_dir]
    r = subprocess.run(cmd, check=True, env=env, capture_output=True, text=True)
    return json.loads(r.stdout)


ITERATES = [  # (case, N, sigma, seed): full solves whose final iterate is kept
    ("case9", 8, 0.0, 0),
    ("case9", 8, 0.05, 0),
    ("case118", 4, 0.05, 0),
    ("case118", 64, 0.05, 0),
    ("case1354pegase", 256, 0.05, 0),
]


def iterates():
    threads = min(8, os.cpu_count() or 1)
    for case, N, sigma, seed in ITERATES:
        name = f"iterates_{case}_N{N}_s{str(sigma).replace('.', '')}.npz"
        path = os.path.join(HERE, name)
        if os.path.exists(path):
            continue
        with tempfile.TemporaryDirectory() as d:
            j = ref_solve(case, N, sigma, seed, threads if N >= 64 else 1, iterate_dir=d)
            out = iterate_fixture(d)
        out["iterations"] = np.array([j["iterations"]])
        np.savez_compressed(path, **out)
        print("wrote", name, j["status"], j["iterations"], j["objective"], flush=True)


CONTINGENCY = [  # (case, N, sigma, seed, outaged branches, round-robin over scenarios)
    ("case9", 4, 0.05, 0, (4, 7)),
    ("case118", 64, 0.05, 0, (10, 20, 30, 40)),
]


def contingency_key(case, N, sigma, seed, cont):
    return f"{case}_N{N}_s{sigma}_seed{seed}_c" + "-".join(str(c) for c in cont)


def contingencies():
    """solves_contingency.json + iterates_<key>.npz: outage scenarios
    (generate_scenarios contingencies, scenarios.cpp:44-80)."""
    path = os.path.join(HERE, "solves_contingency.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for case, N, sigma, seed, cont in CONTINGENCY:
        key = contingency_key(case, N, sigma, seed, cont)
        if key in out:
            continue
        with tempfile.TemporaryDirectory() as d:
            j = ref_solve(case, N, sigma, seed, 4 if N >= 64 else 1, iterate_dir=d, cont=cont)
            it = iterate_fixture(d)
        it["iterations"] = np.array([j["iterations"]])
        np.savez_compressed(os.path.join(HERE, f"iterates_{key}.npz"), **it)
        for k in ("t_total", "t_ad", "t_kkt", "wall"):
            j.pop(k, None)
        for log in j["logs"]:
            for k in ("t_ad", "t_kkt", "t_total"):
                log.pop(k, None)
        j["contingencies"] = list(cont)
        out[key] = j
        print(key, j["status"], j["iterations"], j["objective"], flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


DUMPS2 = [
    ("case1354pegase", 4, 0.05, 0, 40),
    ("case9241pegase", 2, 0.05, 0, 2),
]


def dumps2():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    for case, N, sigma, seed, it in DUMPS2:
        name = f"{case}_N{N}_s{str(sigma).replace('.', '')}_it{it}.npz"
        if os.path.exists(os.path.join(HERE, name)):
            continue
        with tempfile.TemporaryDirectory() as d:
            subprocess.run([REF, "dump", "--case", f"{DATA}/{case}.m", "--N", str(N), "--sigma",
                            str(sigma), "--seed", str(seed), "--iter", str(it), "--out", d],
                           check=True, env=env)
            fx = load_dump(d)
            fx.meta.update(case=case, N=N, sigma=sigma, seed=seed)
            save_npz(fx, os.path.join(HERE, name))
        print("wrote", name, flush=True)


LONG = [  # (case, N, sigma, seed, max_iter, keep the iterate)
    ("case9241pegase", 128, 0.05, 0, 3, False),
    ("case2869pegase", 512, 0.05, 0, 300, True),
    ("case9241pegase", 128, 0.05, 0, 10, False),  # ~75 min on 8 threads
    ("case9241pegase", 128, 0.05, 0, 30, False),  # ~3.8 h on 8 threads
]


def long_runs():
    path = os.path.join(HERE, "solves_large.json")
    threads = min(8, os.cpu_count() or 1)
    for case, N, sigma, seed, max_iter, keep in LONG:
        out = json.load(open(path)) if os.path.exists(path) else {}
        key = f"{case}_N{N}_s{sigma}_seed{seed}" + (f"_it{max_iter}" if max_iter < 300 else "")
        if key in out:
            continue
        with tempfile.TemporaryDirectory() as d:
            j = ref_solve(case, N, sigma, seed, threads, max_iter, iterate_dir=d if keep else None)
            if keep:
                it = iterate_fixture(d)
                it["iterations"] = np.array([j["iterations"]])
                np.savez_compressed(os.path.join(
                    HERE, f"iterates_{case}_N{N}_s{str(sigma).replace('.', '')}.npz"), **it)
        j["note"] = f"reference CPU, {threads} threads (--groups/--workers), this container"
        out = json.load(open(path)) if os.path.exists(path) else {}
        out[key] = j
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(key, j["status"], j["iterations"], j["objective"], flush=True)


def main():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    for case, N, sigma, seed, it in DUMPS:
        with tempfile.TemporaryDirectory() as d:
            subprocess.run([REF, "dump", "--case", f"{DATA}/{case}.m", "--N", str(N), "--sigma",
                            str(sigma), "--seed", str(seed), "--iter", str(it), "--out", d],
                           check=True, env=env)
            fx = load_dump(d)
            fx.meta.update(case=case, N=N, sigma=sigma, seed=seed)
            name = f"{case}_N{N}_s{str(sigma).replace('.', '')}_it{it}.npz"
            save_npz(fx, os.path.join(HERE, name))
            print("wrote", name)
    out = {}
    for case, N, sigma, seed in SOLVES:
        r = subprocess.run([REF, "solve", "--case", f"{DATA}/{case}.m", "--N", str(N), "--sigma",
                            str(sigma), "--seed", str(seed)], check=True, env=env,
                           capture_output=True, text=True)
        j = json.loads(r.stdout)
        for k in ("t_total", "t_ad", "t_kkt", "wall"):
            j.pop(k, None)
        for log in j["logs"]:
            for k in ("t_ad", "t_kkt", "t_total"):
                log.pop(k, None)
        out[f"{case}_N{N}_s{sigma}_seed{seed}"] = j
        print(case, N, sigma, j["status"], j["iterations"], j["objective"])
    with open(os.path.join(HERE, "solves.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    if "--large" in sys.argv:
        large()
    elif "--iterates" in sys.argv:
        iterates()
    elif "--dumps2" in sys.argv:
        dumps2()
    elif "--long" in sys.argv:
        long_runs()
    elif "--contingency" in sys.argv:
        contingencies()
    else:
        main()
