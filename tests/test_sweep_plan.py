"""Host-side check of the static-pivot LU plan and its solve layouts (no GPU):
the plan's level schedules, tail split, transposed copy and dense tail maps,
executed in numpy exactly as the CUDA sweeps execute them
(paper_2301_04869_b200/csrc/kernels/sweeps.cuh), solve with random factors of
the plan's own pattern to machine precision against dense triangular solves."""
import numpy as np
import pytest
import scipy.linalg as sl

from conftest import case_path
from paper_2301_04869_b200 import _native as nat


def emulate(p, F):
    n, nnz_l, nnz_f, t0, tl = p.array("lu_shape")
    FT = F[p.array("lu_ft_src")]
    dense = []
    for b in range(2):
        src = p.array(f"lu_dense_src{b}")
        d = np.where(src >= 0, F[np.maximum(src, 0)], 0.0)
        dense.append(d.reshape(tl, tl).T if tl else np.zeros((0, 0)))  # column-major -> [i, j]
    # what the refactor forms: W = (L_TT U_TT)^{-1}
    if tl:
        LT = np.tril(dense[0], -1) + np.eye(tl)
        UT = np.triu(dense[1])
        W = np.linalg.solve(UT, np.linalg.solve(LT, np.eye(tl)))

    def level(name, V, x, diag):
        lp, items, col = p.array(f"lu_{name}_lvl_ptr"), p.array(f"lu_{name}_items"), \
            p.array(f"lu_{name}_col")
        items = items.reshape(-1, 4)
        for lv in range(len(lp) - 1):
            upd = {}
            for row, b, e, _ in items[lp[lv]:lp[lv + 1]]:
                bb = b + (1 if diag else 0)
                acc = np.dot(V[bb:e], x[col[bb:e]])
                upd[row] = (x[row] - acc) / V[b] if diag else x[row] - acc
            for r, v in upd.items():
                x[r] = v

    def gather(name, V, x, diag):
        items, col = p.array(f"lu_{name}_tail_items").reshape(-1, 4), p.array(f"lu_{name}_col")
        for row, b, split, _ in items:
            bb = b + (1 if diag else 0)
            x[row] -= np.dot(V[bb:split], x[col[bb:split]])

    def solve_LU(x):  # sweeps.cuh solve_LU
        level("sL", F, x, False); gather("sL", F, x, False)
        if tl:
            x[t0:] = W @ x[t0:]
        level("sU", F[nnz_l:], x, True)

    def solve_LUt(x):  # sweeps.cuh solve_LUt
        level("sUt", FT, x, True); gather("sUt", FT, x, True)
        if tl:
            x[t0:] = W.T @ x[t0:]
        level("sLt", FT[nnz_f - nnz_l:], x, False)

    return solve_LU, solve_LUt


@pytest.mark.parametrize("case", ["case9", "case118", "case1354pegase"])
def test_sweeps_solve_the_factor_pattern(case):
    p = nat.Problem(case_path(case), 2, 0.05, 0)
    n, nnz_l, nnz_f, t0, tl = p.array("lu_shape")
    rng = np.random.default_rng(3)
    F = rng.uniform(-0.2, 0.2, nnz_f) / 8
    diag = p.array("lu_diag")
    F[diag] = rng.uniform(1.0, 2.0, n) * np.sign(rng.uniform(-1, 1, n))
    # dense L and U from the plan's row layouts
    L = np.eye(n)
    lp, lc = p.array("lu_l_ptr"), p.array("lu_l_col")
    for i in range(n):
        L[i, lc[lp[i]:lp[i + 1]]] = F[lp[i]:lp[i + 1]]
    U = np.zeros((n, n))
    sp, sc = p.array("lu_sU_ptr"), p.array("lu_sU_col")
    for i in range(n):
        U[i, sc[sp[i]:sp[i + 1]]] = F[nnz_l + sp[i]:nnz_l + sp[i + 1]]
    solve_LU, solve_LUt = emulate(p, F)
    b = rng.normal(size=n)
    A = L @ U
    for fn, M in ((solve_LU, A), (solve_LUt, A.T)):
        x = b.copy()
        fn(x)
        ref = np.linalg.solve(M, b)
        assert np.abs(x - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())
    if case == "case1354pegase":
        assert tl >= 64  # the separator chain goes to the dense tail


@pytest.mark.parametrize("case", ["case9", "case118", "case1354pegase"])
@pytest.mark.parametrize("K", [1, 8])
def test_stream_program_is_valid(case, K):
    """The streamed reduction's static step program (host/stream_plan.cpp):
    every factor entry a sweep reads is staged exactly once per sweep, the
    dense tail's entries never, and no step's ring region overlaps a region the
    producer may still be refilling (checked on the host, bipm_problem_stream_check)."""
    p = nat.Problem(case_path(case), 2, 0.05, 0)
    for ring in (24 * 1024, 48 * 1024):
        st = p.stream_check(K, 512, ring)
        assert st["violations"] == 0, st
        assert st["dense_steps"] == (2 if st["tl"] else 0)
        assert st["t0"] + st["tl"] == p.n_x


def test_dense_tail_keeps_the_fill(monkeypatch):
    """Moving the top etree levels to the end of the order (the dense tail)
    keeps the elimination tree, hence the factor's fill, and cuts the levels
    every triangular sweep walks (make_lu_plan)."""
    case = case_path("case1354pegase")
    monkeypatch.setenv("BIPM_TAIL_WIDTH", "0")
    p0 = nat.Problem(case, 2, 0.05, 0)
    monkeypatch.delenv("BIPM_TAIL_WIDTH")
    p1 = nat.Problem(case, 2, 0.05, 0)
    s0, s1 = p0.array("lu_shape"), p1.array("lu_shape")
    assert s0[1] == s1[1] and s0[2] == s1[2]  # nnz_l, nnz_f
    assert s0[4] == 0 and s1[4] > 100          # tail rows
    lev0 = len(p0.array("lu_sL_lvl_ptr")) - 1
    lev1 = len(p1.array("lu_sL_lvl_ptr")) - 1
    assert lev1 < lev0 / 3, (lev0, lev1)
    assert sorted(p1.array("lu_perm")) == list(range(p1.n_x))
