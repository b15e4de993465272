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

Usage: python tests/golden/make_golden.py   (needs /root/reference; run in
the build container, not on the GPU box)
"""
import json
import os
import subprocess
import sys
import tempfile

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
    large() if "--large" in sys.argv else main()
