"""The drop-in demonstrated: the reference's OWN interior-point driver
(ipm.cpp, compiled unchanged into oracle/_ref/libblockipm_ref.a) running with
its solve_reduced -- and optionally its AD (eval_bundle_range, batch_eval) --
served by the B200 engine through the C-ABI.

oracle/_ref/bipm_ref_gpu is oracle/ref_driver.cpp linked with
integration/bipm_reference_shim.cpp and -Wl,--wrap on those three symbols
(oracle/Makefile); nothing of the reference is modified.  The hybrid runs
must reproduce the pure reference solve (tests/golden/solves*.json): same
iteration count and per-iteration corrections, objective and controls within
1e-6 relative.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, case_path

pytestmark = pytest.mark.gpu

HYBRID = os.path.join(ROOT, "oracle", "_ref", "bipm_ref_gpu")
SOLVES = json.load(open(os.path.join(GOLDEN, "solves.json")))
LARGE = json.load(open(os.path.join(GOLDEN, "solves_large.json")))


def hybrid_solve(case, N, sigma, gpu, extra=()):
    assert os.path.exists(HYBRID), f"{HYBRID} missing: run __graft_entry__.build() where " \
                                   "/root/reference is mounted"
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    r = subprocess.run([HYBRID, "solve", "--case", case_path(case), "--N", str(N), "--sigma",
                        str(sigma), "--seed", "0", "--gpu", gpu, *extra],
                       capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


def check_against(ref, j):
    assert j["status"] == ref["status"] == "Optimal"
    assert j["iterations"] == ref["iterations"]
    assert abs(j["objective"] - ref["objective"]) <= 1e-6 * abs(ref["objective"])
    u_ref = np.array(ref["u"])
    assert np.abs(np.array(j["u"]) - u_ref).max() <= 1e-6 * max(1.0, np.abs(u_ref).max())
    for a, b in zip(j["logs"], ref["logs"]):
        assert a["corr"] == b["corr"]
        assert a["objective"] == pytest.approx(b["objective"], rel=1e-6)


@pytest.mark.parametrize("case,N,sigma", [("case9", 8, 0.05), ("case118", 64, 0.05)])
@pytest.mark.parametrize("gpu", ["kkt", "kkt,ad"])
def test_reference_ipm_with_gpu_operators(case, N, sigma, gpu):
    j = hybrid_solve(case, N, sigma, gpu)
    check_against(SOLVES[f"{case}_N{N}_s{sigma}_seed0"], j)
    # every Newton step went through bipm_solve_reduced (one per iteration
    # that computed a step: all but the converged last one)
    assert j["gpu_kkt_calls"] == j["iterations"] - 1
    if "ad" in gpu:
        assert j["gpu_ad_calls"] >= j["iterations"]
    else:
        assert j["gpu_ad_calls"] == 0


def test_reference_ipm_with_gpu_operators_case1354_N256():
    """The north-star configuration: the reference's driver on 1354pegase /
    256 scenarios with the B200 solve_reduced and AD."""
    j = hybrid_solve("case1354pegase", 256, 0.05, "kkt,ad")
    check_against(LARGE["case1354pegase_N256_s0.05_seed0"], j)
    assert j["gpu_kkt_calls"] == j["iterations"] - 1
