"""CPU restatement of the reference's reduced-KKT operators (numpy / scipy).

TEST INFRASTRUCTURE (oracle/).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may use this module, and only as the checker.

Restated from /root/reference/proj/core/src/kkt.cpp:
  reduce             reduce_group + finish_reduce       kkt.cpp:371-488
  reduce_rhs         reduce_rhs_group                   kkt.cpp:209-239
  recover            recover_state_adjoint + recover_slack_dual
                                                        kkt.cpp:507-532, 172-188
  condense           condense / run_condense            kkt.cpp:123-170, sparse.cpp:208-214
The per-scenario G_x factor is scipy's SuperLU with COLAMD ordering and
partial pivoting (diag_pivot_thresh=1.0), the same algorithm family as the
reference's Eigen::SparseLU defaults (linalg.cpp:76-104; Eigen is absent
from this image).  Pinned against the reference itself by
tests/test_oracle.py on the golden fixtures in tests/golden/.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla


def csr(rowptr, colind, shape, values) -> sp.csr_matrix:
    return sp.csr_matrix((np.asarray(values, dtype=np.float64), colind, rowptr), shape=shape)


class ScenarioFactor:
    """G_x = P^-1 L U Q^-1 of one scenario (BlockDiagFactor::solve_block, linalg.cpp:91-104)."""

    def __init__(self, G: sp.csr_matrix):
        self.lu = sla.splu(G.tocsc(), permc_spec="COLAMD", diag_pivot_thresh=1.0)

    def solve(self, B: np.ndarray, transpose: bool = False) -> np.ndarray:
        return self.lu.solve(np.asarray(B, dtype=np.float64), trans="T" if transpose else "N")


def reduce(pats: dict, vals: dict, dw: float):
    """K_hat and rhs of the reduced system (kkt.cpp:371-488).

    pats: name -> (rowptr, colind, shape) for gx, gu, kxx, kxu, kuu.
    vals: gx, gu, kxx, kxu, kuu ([N, nnz]); sigma_x, rhat1, rhat3 ([N, n_x]);
          sigma_u, rhat2 ([n_u]).
    Returns (khat [n_u, n_u], rhs [n_u]).
    """
    N = vals["gx"].shape[0]
    n_u = len(vals["sigma_u"])
    khat = np.zeros((n_u, n_u))
    rhs = np.zeros(n_u)
    for b in range(N):
        G = csr(*pats["gx"][:2], pats["gx"][2], vals["gx"][b])
        Gu = csr(*pats["gu"][:2], pats["gu"][2], vals["gu"][b]).toarray()
        Kxx = csr(*pats["kxx"][:2], pats["kxx"][2], vals["kxx"][b])
        Kxu = csr(*pats["kxu"][:2], pats["kxu"][2], vals["kxu"][b]).toarray()
        Kuu = csr(*pats["kuu"][:2], pats["kuu"][2], vals["kuu"][b]).toarray()
        ktil = Kxx + sp.diags(vals["sigma_x"][b] + dw)
        f = ScenarioFactor(G)
        T = -f.solve(Gu)                         # kkt.cpp:388-404
        Lx = ktil @ T + Kxu                      # kkt.cpp:406-423
        Y = f.solve(Lx, transpose=True)          # kkt.cpp:427
        khat += Kxu.T @ T - Gu.T @ Y + Kuu       # kkt.cpp:430-447
        a = f.solve(vals["rhat3"][b])            # kkt.cpp:217-229
        t = vals["rhat1"][b] - ktil @ a
        t = f.solve(t, transpose=True)
        rhs += Gu.T @ t + Kxu.T @ a
    khat[np.diag_indices(n_u)] += vals["sigma_u"] + dw   # kkt.cpp:483-486
    rhs -= vals["rhat2"]
    return khat, rhs


def recover(pats: dict, vals: dict, dw: float, pu: np.ndarray):
    """p_x, p_y (kkt.cpp:507-532) and p_z, p_s (kkt.cpp:172-188) per scenario."""
    N = vals["gx"].shape[0]
    out = {k: [] for k in ("px", "py", "pz", "ps")}
    for b in range(N):
        G = csr(*pats["gx"][:2], pats["gx"][2], vals["gx"][b])
        Gu = csr(*pats["gu"][:2], pats["gu"][2], vals["gu"][b])
        Kxx = csr(*pats["kxx"][:2], pats["kxx"][2], vals["kxx"][b])
        Kxu = csr(*pats["kxu"][:2], pats["kxu"][2], vals["kxu"][b])
        Hx = csr(*pats["hx"][:2], pats["hx"][2], vals["hx"][b])
        Hu = csr(*pats["hu"][:2], pats["hu"][2], vals["hu"][b])
        f = ScenarioFactor(G)
        px = -f.solve(vals["rhat3"][b] + Gu @ pu)
        t = vals["rhat1"][b] + Kxx @ px + (vals["sigma_x"][b] + dw) * px + Kxu @ pu
        py = -f.solve(t, transpose=True)
        hp = Hx @ px + Hu @ pu
        ss = vals["sigma_s"][b]
        pz = ss * (hp + vals["r4"][b]) - vals["r2"][b]
        ps = -(vals["r2"][b] + pz) / ss
        for k, v in (("px", px), ("py", py), ("pz", pz), ("ps", ps)):
            out[k].append(v)
    return {k: np.array(v) for k, v in out.items()}


def condense(pats: dict, vals: dict):
    """K_xx, K_xu, K_uu values on the condensed patterns (kkt.cpp:156-162).

    pats needs wxx, wxu, wuu, hx, hu and the output patterns kxx, kxu, kuu.
    """
    N = vals["hx"].shape[0]
    res = {"kxx": [], "kxu": [], "kuu": []}
    for b in range(N):
        S = sp.diags(vals["sigma_s"][b])
        Hx = csr(*pats["hx"][:2], pats["hx"][2], vals["hx"][b])
        Hu = csr(*pats["hu"][:2], pats["hu"][2], vals["hu"][b])
        for name, W, A, B in (("kxx", "wxx", Hx, Hx), ("kxu", "wxu", Hx, Hu),
                              ("kuu", "wuu", Hu, Hu)):
            Wm = csr(*pats[W][:2], pats[W][2], vals[W][b])
            K = (Wm + A.T @ S @ B).tocsr()
            rp, ci, shape = pats[name]
            dense = K.toarray()
            rows = np.repeat(np.arange(shape[0]), np.diff(rp))
            res[name].append(dense[rows, ci])
    return {k: np.array(v) for k, v in res.items()}


def rhat(pats: dict, vals: dict):
    """rhat1 (per scenario) and rhat2 of the condensed rhs (kkt.cpp:163-168)."""
    N = vals["hx"].shape[0]
    r1, r2 = [], np.array(vals["r1u"], dtype=np.float64).copy()
    for b in range(N):
        Hx = csr(*pats["hx"][:2], pats["hx"][2], vals["hx"][b])
        Hu = csr(*pats["hu"][:2], pats["hu"][2], vals["hu"][b])
        t = vals["sigma_s"][b] * vals["r4"][b] - vals["r2"][b]
        r1.append(vals["r1x"][b] + Hx.T @ t)
        r2 += Hu.T @ t
    return np.array(r1), r2
