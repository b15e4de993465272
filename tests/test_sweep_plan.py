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
        # round-2 variants: presolved forward half (no L sweep, no first dense
        # step), + adjoint identity (no L' sweep, no second dense step), +
        # deferred tail; the factor coverage check adapts to the sweeps left
        for mode, dense in ((1, 1), (3, 0), (7, 0)):
            sv = p.stream_check(K, 512, ring, mode)
            assert sv["violations"] == 0, (mode, sv)
            assert sv["dense_steps"] == (dense if st["tl"] else 0), (mode, sv)
            assert sv["steps"] < st["steps"] or not st["tl"], (mode, sv, st)


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


@pytest.mark.parametrize("case", ["case118", "case1354pegase"])
def test_split_refactor_program_factors_the_pattern(case):
    """The flattened refactor program (refactor_levels_kernel: Crout phases of
    the pivots before the dense tail, then the tail block's partial sums)
    followed by a dense LU of the tail block (refactor_tail_* kernels),
    executed in numpy on a random diagonally dominant matrix with G_x's
    pattern, reproduces P A P' = L U."""
    p = nat.Problem(case_path(case), 2, 0.05, 0)
    n, nnz_l, nnz_f, t0, tl = p.array("lu_shape")
    rp, ci = p.array("gx_p_rowptr"), p.array("gx_p_colind")
    rng = np.random.default_rng(5)
    A = np.zeros((n, n))
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            A[i, ci[k]] = rng.normal()
        A[i, i] = 10.0 + abs(A[i]).sum()
    vals = np.array([A[i, ci[k]] for i in range(n) for k in range(rp[i], rp[i + 1])])
    phase = p.array("lu_rf_phase_ptr")
    rec = p.array("lu_rf_rec").reshape(-1, 4)
    piv = p.array("lu_rf_piv")
    pair = p.array("lu_rf_pair").reshape(-1, 2)
    F = np.zeros(nnz_f)
    for ph in range(len(phase) - 1):
        new = {}
        for it in range(phase[ph], phase[ph + 1]):
            slot, b, e, src = rec[it]
            acc = sum(F[pair[t, 0]] * F[pair[t, 1]] for t in range(b, e))
            v = (vals[src] if src >= 0 else 0.0) - acc
            if piv[it] >= 0:
                v /= F[piv[it]]
            new[slot] = v
        for k, v in new.items():  # a phase's entries are independent
            F[k] = v
    # dense LU of the tail block (what the tail kernels do), written back
    src0, src1 = p.array("lu_dense_src0"), p.array("lu_dense_src1")
    T = np.zeros((tl, tl))
    for q in range(tl * tl):
        a, b = q % tl, q // tl
        s = src0[q] if a > b else src1[q]
        T[a, b] = F[s] if s >= 0 else 0.0
    for k in range(tl - 1):
        T[k + 1:, k] /= T[k, k]
        T[k + 1:, k + 1:] -= np.outer(T[k + 1:, k], T[k, k + 1:])
    for q in range(tl * tl):
        a, b = q % tl, q // tl
        s = src0[q] if a > b else src1[q]
        if s >= 0:
            F[s] = T[a, b]
    # assemble L, U and compare with P A P'
    perm = p.array("lu_perm")
    l_ptr, l_col = p.array("lu_l_ptr"), p.array("lu_l_col")
    u_ptr, u_col, u_slot, diag = (p.array("lu_u_ptr"), p.array("lu_u_col"), p.array("lu_u_slot"),
                                  p.array("lu_diag"))
    L = np.eye(n)
    U = np.zeros((n, n))
    for i in range(n):
        for t in range(l_ptr[i], l_ptr[i + 1]):
            L[i, l_col[t]] = F[t]
        U[i, i] = F[diag[i]]
        for t in range(u_ptr[i], u_ptr[i + 1]):
            U[i, u_col[t]] = F[u_slot[t]]
    PA = A[np.ix_(perm, perm)]
    assert np.abs(L @ U - PA).max() <= 1e-10 * np.abs(PA).max()


def _gj_folded_inverse(S, kB=16):
    """numpy restatement of refactor_tail_gj_kernel's pass (kkt_kernels.cu):
    each block of kB pivots is one rank-kB update W <- W' - C' R2 with
    C' = W[:, P] (pivot rows -e_p), R2 = A11^{-1} W[P, :] (pivot columns
    A11^{-1}) and W' = W with the pivot rows and columns zeroed."""
    W = S.astype(np.float64).copy()
    n = W.shape[0]
    for k0 in range(0, n, kB):
        P = np.arange(k0, min(n, k0 + kB))
        Ai = np.linalg.inv(W[np.ix_(P, P)])
        C = W[:, P].copy()
        C[P, :] = -np.eye(len(P))
        R2 = Ai @ W[P, :]
        R2[:, P] = Ai
        Wp = W.copy()
        Wp[P, :] = 0.0
        Wp[:, P] = 0.0
        W = Wp - C @ R2
    return W


@pytest.mark.parametrize("n", [5, 16, 37, 233])
def test_gauss_jordan_folded_update_inverts(n):
    rng = np.random.default_rng(n)
    S = rng.standard_normal((n, n)) + n * np.eye(n)  # static pivots stay nonzero
    W = _gj_folded_inverse(S)
    assert np.allclose(W @ S, np.eye(n), atol=1e-10)
