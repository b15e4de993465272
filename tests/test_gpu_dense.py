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
