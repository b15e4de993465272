"""Dense reduced-matrix factorisation on the GPU (rows a13-a14 of SURVEY §8(a)):
shift 1e-13 max(1,|K|_inf) + Cholesky + solve against numpy, and the
not-positive-definite verdict (LAPACK dpotrf semantics) that drives the
inertia loop (kkt.cpp:965-971)."""
import numpy as np
import pytest

from conftest import case_path
from paper_2301_04869_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [5, 37, 107, 150, 151, 300, 519, 1019, 2047])
def test_shift_cholesky_solve(n):
    rng = np.random.default_rng(n)
    A = rng.normal(size=(n, n))
    K = A @ A.T + n * np.eye(n)
    b = rng.normal(size=n)
    pd, x = nat.dense_factor_solve(K, b)
    assert pd
    Ks = K + 1e-13 * max(1.0, np.abs(K).max()) * np.eye(n)
    ref = np.linalg.solve(Ks, b)
    assert np.abs(x - ref).max() <= 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("n", [37, 151, 519])
def test_indefinite_is_rejected(n):
    rng = np.random.default_rng(1)
    A = rng.normal(size=(n, n))
    K = A @ A.T + np.eye(n)
    K[n // 2, n // 2] = -1e3
    pd, _ = nat.dense_factor_solve(K, np.ones(n))
    assert not pd


@pytest.mark.parametrize("n,where", [(519, 0), (519, 31), (519, 32), (519, 518), (700, 650)])
def test_indefinite_pivot_position(n, where):
    """the blocked (DMMA) factor must fail wherever the bad pivot sits:
    first column, panel edges, last column"""
    rng = np.random.default_rng(where)
    A = rng.normal(size=(n, n))
    K = A @ A.T / n + np.eye(n)
    K[where, where] = -1.0
    pd, _ = nat.dense_factor_solve(K, np.ones(n))
    assert not pd


def _ldl_inertia(K):
    """LAPACK dsytrf (scipy.linalg.ldl, Bunch-Kaufman) inertia with the
    reference's 2x2 rule (lapack.cpp:55-97)."""
    import scipy.linalg as sl
    _, d, _ = sl.ldl(K, lower=True)
    n, k, pos, neg, zero = len(d), 0, 0, 0, 0
    while k < n:
        if k + 1 < n and d[k + 1, k] != 0.0:
            a, c, b = d[k, k], d[k + 1, k + 1], d[k + 1, k]
            det = a * c - b * b
            if det < 0:
                pos, neg = pos + 1, neg + 1
            elif det > 0:
                pos, neg = (pos + 2, neg) if a + c > 0 else (pos, neg + 2)
            k += 2
        else:
            pos, neg, zero = pos + (d[k, k] > 0), neg + (d[k, k] < 0), zero + (d[k, k] == 0)
            k += 1
    return pos, neg, zero


@pytest.mark.parametrize("n,n_neg", [(5, 2), (107, 1), (200, 37), (519, 3), (519, 0), (700, 250)])
def test_bunch_kaufman_inertia_and_solve(n, n_neg):
    """bipm_dense_inertia = DenseSymFactor's Bunch-Kaufman branch
    (linalg.cpp:136-145): inertia equal to the eigenvalue signs and to
    LAPACK dsytrf's, and the LDL' solve equal to a dense solve."""
    rng = np.random.default_rng(n + n_neg)
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = rng.uniform(0.5, 4.0, size=n)
    lam[:n_neg] *= -1.0
    K = (Q * lam) @ Q.T
    K = 0.5 * (K + K.T)
    b = rng.normal(size=n)
    (pos, neg, zero), x = nat.dense_inertia(K, b)
    assert (pos, neg, zero) == (n - n_neg, n_neg, 0)
    Ks = K + 1e-13 * max(1.0, np.abs(K).max()) * np.eye(n)
    assert (pos, neg, zero) == _ldl_inertia(Ks)
    ref = np.linalg.solve(Ks, b)
    assert np.abs(x - ref).max() <= 1e-9 * np.abs(ref).max()


def test_bunch_kaufman_two_by_two_pivots():
    """a matrix whose diagonal is zero forces 2x2 pivots (dsytf2's kstep 2)"""
    n = 64
    rng = np.random.default_rng(3)
    A = rng.normal(size=(n // 2, n // 2))
    K = np.block([[np.zeros((n // 2, n // 2)), A], [A.T, np.zeros((n // 2, n // 2))]])
    (pos, neg, zero), x = nat.dense_inertia(K, np.ones(n))
    assert (pos, neg, zero) == (n // 2, n // 2, 0) == _ldl_inertia(K + 1e-13 * max(1.0, np.abs(K).max()) * np.eye(n))
    Ks = K + 1e-13 * max(1.0, np.abs(K).max()) * np.eye(n)
    ref = np.linalg.solve(Ks, np.ones(n))
    assert np.abs(x - ref).max() <= 1e-8 * np.abs(ref).max()


def test_inertia_loop_with_bunch_kaufman_verdicts(monkeypatch):
    """BIPM_FORCE_BK=1: every Cholesky failure of the inertia loop is decided
    by the Bunch-Kaufman inertia (the reference's rule, kkt.cpp:969-971); the
    solve must follow the reference trajectory exactly as the Cholesky-only
    verdicts do (tests/golden/solves.json)."""
    import json
    import os
    from conftest import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "solves.json")))["case118_N64_s0.05_seed0"]
    monkeypatch.setenv("BIPM_FORCE_BK", "1")
    ctx = nat.Context(nat.Problem(case_path("case118"), 64, 0.05, 0))
    r = nat.Solver(ctx).solve()
    assert r["iterations"] == ref["iterations"]
    assert abs(r["objective"] - ref["objective"]) <= 1e-6 * abs(ref["objective"])
    assert [int(l["corr"]) for l in r["logs"]] == [l["corr"] for l in ref["logs"]]
    assert ctx.factor_stats()["bk_fallbacks"] > 0  # the BK path ran
