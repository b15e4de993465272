"""Host-side check of the presolved forward half of the Schur reduction
(host/stream_plan.hpp ReachPlan, executed by reach_solve_kernel in
paper_2301_04869_b200/csrc/kernels/reach_gemm.cu): the per-column op program,
run in numpy exactly as the kernel runs it, against a dense triangular solve
of L y = P G_u with random factor values on the plan's own pattern.  The
reach must be complete (y is exactly zero off it) and the tail rows must
equal (P G_u)_T - L_TN y_N (the input of X_T = W y_T)."""
import numpy as np
import pytest
import scipy.linalg as sla

from conftest import case_path
from paper_2301_04869_b200 import _native as nat


@pytest.mark.parametrize("case", ["case9", "case118", "case1354pegase"])
def test_reach_plan_matches_dense_forward_solve(case):
    p = nat.Problem(case_path(case), 1, 0.0, 0)
    n, nnz_l, nnz_f, t0, tl = p.array("lu_shape")
    l_ptr, l_col = p.array("lu_l_ptr"), p.array("lu_l_col")
    perm = p.array("lu_perm")
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(n)
    gptr, gcol = p.array("gu_p_rowptr"), p.array("gu_p_colind")
    n_u = int(gcol.max()) + 1 if len(gcol) else 0
    rng = np.random.default_rng(3)
    F = rng.uniform(-0.5, 0.5, nnz_f)  # L strict lower values at slots [0, nnz_l)
    gu = rng.uniform(-1.0, 1.0, len(gcol))
    # dense unit lower L (permuted) and B = P G_u
    L = np.eye(n)
    for r in range(n):
        for q in range(l_ptr[r], l_ptr[r + 1]):
            L[r, l_col[q]] = F[q]
    B = np.zeros((n, n_u))
    for r in range(len(gptr) - 1):
        for q in range(gptr[r], gptr[r + 1]):
            B[iperm[r], gcol[q]] = gu[q]
    yN = sla.solve_triangular(L[:t0, :t0], B[:t0], lower=True, unit_diagonal=True)
    yT = B[t0:] - L[t0:, :t0] @ yN

    yn_ptr, yn_row = p.array("reach_yn_ptr"), p.array("reach_yn_row")
    op_ptr = p.array("reach_op_ptr")
    ops, ent = p.array("reach_ops").reshape(-1, 4), p.array("reach_ent").reshape(-1, 2)
    yt_ptr, yt_row = p.array("reach_yt_ptr"), p.array("reach_yt_row")
    assert len(yn_ptr) == n_u + 1 and len(yt_ptr) == n_u + 1
    scale = np.abs(yN).max(initial=0.0) + np.abs(yT).max(initial=0.0)
    for u in range(n_u):
        rows = yn_row[yn_ptr[u]:yn_ptr[u + 1]]
        assert np.all(np.diff(rows) > 0) and np.all(rows < t0)
        off = np.ones(t0, bool)
        off[rows] = False
        assert np.all(yN[off, u] == 0.0), "reach incomplete"
        y = np.zeros(len(rows))
        t = np.zeros(tl)
        for dest, bslot, eb, ee in ops[op_ptr[u]:op_ptr[u + 1]]:
            v = (gu[bslot] if bslot >= 0 else 0.0) - np.dot(F[ent[eb:ee, 1]], y[ent[eb:ee, 0]])
            if dest >= 0:
                y[dest] = v
            else:
                t[-1 - dest] = v
        assert np.abs(y - yN[rows, u]).max(initial=0.0) <= 1e-13 * scale
        assert np.abs(t - yT[:, u]).max(initial=0.0) <= 1e-13 * scale
        # y_T's pattern (the sparse X_T = W y_T product): exactly the rows the ops write
        pat = yt_row[yt_ptr[u]:yt_ptr[u + 1]]
        assert np.all(np.diff(pat) > 0)
        off_t = np.ones(tl, bool)
        off_t[pat] = False
        assert np.all(yT[off_t, u] == 0.0), "y_T pattern incomplete"
