"""ctypes binding of the C-ABI in ``include/bipm_gpu.h``.

The shared library is built in-tree (``paper_2301_04869_b200/_lib``) by
``__graft_entry__.build()``.  There is no fallback: if the library is missing
or a CUDA call fails, the call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BIPM_LIB: A/B experiments against another build (tools/); default the in-tree one
LIB_PATH = os.environ.get("BIPM_LIB") or os.path.join(_HERE, "_lib", "libbipm_gpu.so")

STATUS = {
    0: "OK",
    1: "SINGULAR_BLOCK",
    2: "NONFINITE",
    3: "NOT_PD",
    4: "CUDA_ERROR",
    5: "INVALID_ARGUMENT",
    6: "NON_INTERIOR",
    7: "LINEAR_SOLVE",
    8: "PARSE_ERROR",
    9: "UNSUPPORTED",
}


class BipmError(RuntimeError):
    def __init__(self, code: int, msg: str, block: int = -1):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.block = block


class SingularBlockError(BipmError):
    """Mirror of blockipm::SingularBlockError (types.hpp:99-103)."""


class NonFiniteError(BipmError):
    """Mirror of blockipm::NonFiniteError (types.hpp:105-109)."""


class NonInteriorError(BipmError):
    """Mirror of blockipm::NonInteriorError (kkt.hpp:31-33)."""


class LinearSolveError(BipmError):
    """Mirror of blockipm::LinearSolveError (kkt.hpp:34-36)."""


_EXC = {1: SingularBlockError, 2: NonFiniteError, 6: NonInteriorError, 7: LinearSolveError}

_lib = None
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int32)

# exported symbol -> (restype, argtypes); also the list the CPU tests check
SIGNATURES = {
    "bipm_last_error": (ctypes.c_char_p, []),
    "bipm_last_error_block": (ctypes.c_int32, []),
    "bipm_version": (ctypes.c_int, []),
    "bipm_problem_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int32, ctypes.c_double,
                                           ctypes.c_uint64, ctypes.POINTER(_P)]),
    "bipm_problem_destroy": (None, [_P]),
    "bipm_problem_dims": (ctypes.c_int, [_P, _I]),
    "bipm_problem_array": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(_P),
                                          ctypes.POINTER(ctypes.c_int64), _I]),
    "bipm_ctx_create": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(_P)]),
    "bipm_ctx_destroy": (None, [_P]),
    "bipm_factor_gx": (ctypes.c_int, [_P, _D, _I]),
    "bipm_reduce": (ctypes.c_int, [_P, _P, ctypes.c_double, _D, _D]),
    "bipm_eval_bundle": (ctypes.c_int, [_P, _D, _D, _D, _D, ctypes.c_double, _P, _I]),
    "bipm_eval_values": (ctypes.c_int, [_P, _D, _D, _D, _D, _D, _I]),
    "bipm_solver_create": (ctypes.c_int, [_P, _P, ctypes.POINTER(_P)]),
    "bipm_solver_destroy": (None, [_P]),
    "bipm_solver_start": (ctypes.c_int, [_P]),
    "bipm_solver_step": (ctypes.c_int, [_P, _I]),
    "bipm_solver_result": (ctypes.c_int, [_P, _P, _D]),
    "bipm_solver_log": (ctypes.c_int, [_P, ctypes.c_int32, _D]),
    "bipm_solve": (ctypes.c_int, [_P, _P, _P, _D]),
    "bipm_solver_step_timed": (ctypes.c_int, [_P, _I, _D]),
    "bipm_counters": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int64)]),
    "bipm_ctx_profile": (ctypes.c_int, [_P, ctypes.c_int32]),
    "bipm_ctx_kernel_time": (ctypes.c_int, [_P, ctypes.c_char_p, _D,
                                            ctypes.POINTER(ctypes.c_int64)]),
    "bipm_ctx_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "bipm_dense_factor_solve": (ctypes.c_int, [ctypes.c_int32, _D, _D, _I]),
    "bipm_partition": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _I]),
    "bipm_nccl_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
    "bipm_ctx_set_nccl": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int32,
                                         ctypes.c_int32]),
    "bipm_ctx_set_host_comm": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, ctypes.c_int32]),
    "bipm_ctx_phase_stamps": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
    "bipm_problem_stream_check": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
    "bipm_problem_stream_check_ex": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32,
                                                    ctypes.c_int32, ctypes.c_int32,
                                                    ctypes.POINTER(ctypes.c_int64)]),
    "bipm_ctx_debug_buffer": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                             ctypes.POINTER(ctypes.c_int64)]),
    "bipm_ctx_step_stamps": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.c_int32, _I]),
    "bipm_problem_create_ex": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int32, ctypes.c_double,
                                              ctypes.c_uint64, _I, ctypes.c_int32,
                                              ctypes.POINTER(_P)]),
    "bipm_problem_create_tables": (ctypes.c_int, [_P, _P, ctypes.POINTER(_P)]),
    "bipm_problem_create_patterns": (ctypes.c_int, [ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P,
                                                    ctypes.POINTER(_P)]),
    "bipm_condense": (ctypes.c_int, [_P, _P, _P]),
    "bipm_reduce_rhs": (ctypes.c_int, [_P, _P, ctypes.c_double, _D]),
    "bipm_recover": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, _D, _D, _D, _D, _D]),
    "bipm_solve_reduced": (ctypes.c_int, [_P, _P, _P, _D, _P, _P]),
    "bipm_solver_iterate": (ctypes.c_int, [_P, _P]),
    "bipm_ctx_comm": (ctypes.c_int, [_P, _I]),
    "bipm_dense_inertia": (ctypes.c_int, [ctypes.c_int32, _D, _D, _I]),
    "bipm_ctx_factor_stats": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
}

BUNDLE_FIELDS = ("f", "g", "h", "gx", "gu", "hx", "hu", "wxx", "wxu", "wuu", "grad_lag")


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _destroy(obj, fn_name: str) -> None:
    """Release a C-ABI handle; quiet at interpreter shutdown (module globals gone)."""
    h = getattr(obj, "_h", None)
    if not h:
        return
    obj._h = None
    try:
        getattr(_lib, fn_name)(h)
    except Exception:  # noqa: BLE001
        pass


def check(code: int) -> None:
    if code != 0:
        msg = lib().bipm_last_error().decode()
        raise _EXC.get(code, BipmError)(code, msg, lib().bipm_last_error_block())


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


class _Condensed(ctypes.Structure):
    _fields_ = [(n, _D) for n in ("gu", "kxx", "kxu", "kuu", "sigma_x", "rhat1", "rhat3",
                                  "sigma_u", "rhat2")]


class _Bundle(ctypes.Structure):
    _fields_ = [(n, _D) for n in BUNDLE_FIELDS]


AUGMENTED_FIELDS = ("gx", "gu", "hx", "hu", "wxx", "wxu", "wuu", "sigma_x", "r1x", "r3",
                    "sigma_s", "r2", "r4", "sigma_u", "r1u")
CONDENSED_OUT_FIELDS = ("kxx", "kxu", "kuu", "rhat1", "rhat3", "rhat2")
STEP_FIELDS = ("px", "pu", "ps", "pz", "py")
ITERATE_FIELDS = ("x", "u", "s", "y", "z", "kappa_lo", "kappa_up", "nu_lo", "nu_up",
                  "lambda_lo", "lambda_up")


class _Augmented(ctypes.Structure):
    _fields_ = [(n, _D) for n in AUGMENTED_FIELDS]


class _CondensedOut(ctypes.Structure):
    _fields_ = [(n, _D) for n in CONDENSED_OUT_FIELDS]


class _SlackRows(ctypes.Structure):
    _fields_ = [(n, _D) for n in ("hx", "hu", "sigma_s", "r2", "r4")]


class _RegSchedule(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("delta_w0", "delta_w_min", "delta_w_max",
                                               "kappa_minus", "kappa_plus",
                                               "kappa_plus_emergency")]


class _Step(ctypes.Structure):
    _fields_ = [(n, _D) for n in STEP_FIELDS]


class _StepInfo(ctypes.Structure):
    _fields_ = [("delta_w", ctypes.c_double), ("corrections", ctypes.c_int32),
                ("refinements", ctypes.c_int32), ("reductions", ctypes.c_int64)]


class _Iterate(ctypes.Structure):
    _fields_ = [(n, _D) for n in ITERATE_FIELDS]


class _Csr(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("row_ptr", _I),
                ("col_ind", _I)]


class _CaseTables(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("base_mva", ctypes.c_double),
                ("nbus", ctypes.c_int32), ("ngen", ctypes.c_int32), ("nbranch", ctypes.c_int32),
                ("ngencost", ctypes.c_int32), ("bus", _D), ("gen", _D), ("branch", _D),
                ("gencost", _D), ("gencost_coef", _D)]


class _ScenarioTables(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("sigma", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("multipliers", _D), ("outage_ptr", _I), ("outage_branch", _I)]


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


ALLREDUCE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, _D, ctypes.c_int64, ctypes.c_int32)


def partition(N: int, G: int):
    """Contiguous scenario groups (executor.cpp:7-19) as [(lo, hi)] * G."""
    out = (ctypes.c_int32 * (2 * G))()
    check(lib().bipm_partition(N, G, out))
    return [(out[2 * g], out[2 * g + 1]) for g in range(G)]


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(lib().bipm_nccl_unique_id(buf))
    return bytes(buf)


class _SolveOptions(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("mu0", ctypes.c_double), ("max_iter", ctypes.c_int32)]


class _SolveResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("objective", ctypes.c_double), ("t_total", ctypes.c_double),
                ("t_ad", ctypes.c_double), ("t_kkt", ctypes.c_double),
                ("reductions", ctypes.c_int64)]


SOLVE_STATUS = {-2: "NotStarted", -1: "Running", 0: "Optimal", 1: "MaxIter", 2: "Infeasible"}
LOG_FIELDS = ("iter", "objective", "inf_pr", "inf_du", "complementarity", "mu", "alpha_p",
              "alpha_d", "t_ad", "t_kkt", "t_total", "corr", "refinements", "delta_w",
              "full_step")


class Problem:
    """Host model + symbolic plans (no GPU): bipm_problem_create[_ex].

    ``contingencies``: branch indices outaged round-robin over the scenarios
    (generate_scenarios, scenarios.cpp:44-80)."""

    def __init__(self, case_path: str | None, N: int, sigma: float = 0.0, seed: int = 0,
                 contingencies=(), _handle=None):
        h = _P()
        if _handle is not None:
            h = _handle
        elif contingencies:
            c = np.ascontiguousarray(contingencies, dtype=np.int32)
            check(lib().bipm_problem_create_ex(case_path.encode(), N, sigma, seed, iptr(c),
                                               len(c), ctypes.byref(h)))
        else:
            check(lib().bipm_problem_create(case_path.encode(), N, sigma, seed, ctypes.byref(h)))
        self._init(h)

    @classmethod
    def from_tables(cls, base_mva: float, bus, gen, branch, gencost_rows, gencost_coef,
                    multipliers, outages=None, sigma: float = 0.0, seed: int = 0,
                    name: str = "tables"):
        """bipm_problem_create_tables: the reference's CaseData / ScenarioSet as
        tables (columns in include/bipm_gpu.h)."""
        keep = [_f64(bus), _f64(gen), _f64(branch), _f64(gencost_rows), _f64(gencost_coef),
                _f64(multipliers)]
        t = _CaseTables(name.encode(), base_mva, keep[0].shape[0], keep[1].shape[0],
                        keep[2].shape[0], keep[3].shape[0], *[dptr(a) for a in keep[:5]])
        N = keep[5].shape[0]
        sc = _ScenarioTables(N, sigma, seed, dptr(keep[5]), None, None)
        if outages is not None:
            ptr = np.zeros(N + 1, dtype=np.int32)
            ptr[1:] = np.cumsum([len(o) for o in outages])
            idx = np.ascontiguousarray(np.concatenate([np.asarray(o, dtype=np.int32)
                                                       for o in outages] + [np.zeros(0, np.int32)]),
                                       dtype=np.int32)
            keep += [ptr, idx]
            sc.outage_ptr, sc.outage_branch = iptr(ptr), iptr(idx)
        h = _P()
        check(lib().bipm_problem_create_tables(ctypes.byref(t), ctypes.byref(sc),
                                               ctypes.byref(h)))
        return cls(None, N, _handle=h)

    @classmethod
    def from_patterns(cls, N: int, pats: dict):
        """bipm_problem_create_patterns: pats[name] = (row_ptr, col_ind, (rows, cols))
        for gx, gu, hx, hu, wxx, wxu, wuu (KKT operators only)."""
        keep, cs = [], []
        for k in ("gx", "gu", "hx", "hu", "wxx", "wxu", "wuu"):
            rp, ci, shape = pats[k]
            rp = np.ascontiguousarray(rp, dtype=np.int32)
            ci = np.ascontiguousarray(ci, dtype=np.int32)
            keep += [rp, ci]
            cs.append(_Csr(shape[0], shape[1], iptr(rp), iptr(ci)))
        h = _P()
        check(lib().bipm_problem_create_patterns(N, *[ctypes.byref(c) for c in cs],
                                                 ctypes.byref(h)))
        return cls(None, N, _handle=h)

    def _init(self, h):
        self._h = h
        d = (ctypes.c_int32 * 10)()
        check(lib().bipm_problem_dims(h, d))
        (self.N, self.n_x, self.n_u, self.m, self.n_b, self.nbus, self.nbranch, self.ngen,
         self.nnz_factor, self.levels) = list(d)

    def array(self, name: str) -> np.ndarray:
        data, n, is_int = _P(), ctypes.c_int64(), ctypes.c_int32()
        check(lib().bipm_problem_array(self._h, name.encode(), ctypes.byref(data),
                                       ctypes.byref(n), ctypes.byref(is_int)))
        if n.value == 0:
            return np.zeros(0, dtype=np.int32 if is_int.value else np.float64)
        ct = ctypes.c_int32 if is_int.value else ctypes.c_double
        buf = (ct * n.value).from_address(data.value)
        return np.array(buf, copy=True)

    def stream_check(self, K: int, consumers: int = 512, ring_bytes: int = 48 * 1024,
                     mode: int = 0) -> dict:
        """Host-only build + validation of the streamed reduction's step program
        (mode: 1 presolved, 2 adjoint identity, 4 deferred tail; include/bipm_gpu.h)."""
        out = (ctypes.c_int64 * 10)()
        check(lib().bipm_problem_stream_check_ex(self._h, K, consumers, ring_bytes, mode, out))
        keys = ("violations", "steps", "nnz_vs", "sweep_steps", "dense_steps", "acc_steps",
                "spmv_steps", "nq", "t0", "tl")
        return dict(zip(keys, list(out)))

    def csr(self, name: str):
        return self.array(name + "_rowptr"), self.array(name + "_colind")

    def __del__(self):
        _destroy(self, "bipm_problem_destroy")


class Context:
    """One GPU owning scenarios [lo, hi): bipm_ctx_create."""

    def __init__(self, problem: Problem, device: int = 0, lo: int = 0, hi: int | None = None):
        self.problem = problem
        self.lo, self.hi = lo, problem.N if hi is None else hi
        h = _P()
        check(lib().bipm_ctx_create(problem._h, device, self.lo, self.hi, ctypes.byref(h)))
        self._h = h

    def factor_gx(self, gx: np.ndarray) -> None:
        gx = np.ascontiguousarray(gx, dtype=np.float64)
        bad = ctypes.c_int32(-1)
        check(lib().bipm_factor_gx(self._h, dptr(gx), ctypes.byref(bad)))

    def reduce(self, delta_w: float, **arrays):
        keep = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in arrays.items()}
        c = _Condensed(**{k: dptr(v) for k, v in keep.items()})
        n_u = self.problem.n_u
        khat = np.zeros(n_u * n_u)
        rhs = np.zeros(n_u)
        check(lib().bipm_reduce(self._h, ctypes.byref(c), delta_w, dptr(khat), dptr(rhs)))
        return khat.reshape(n_u, n_u).T.copy(), rhs  # column-major -> numpy

    def _augmented(self, a: dict):
        keep = {k: _f64(a[k]) for k in AUGMENTED_FIELDS}
        return keep, _Augmented(**{k: dptr(v) for k, v in keep.items()})

    def condense(self, **aug):
        """condense (kkt.cpp:123-170) through bipm_condense."""
        keep, a = self._augmented(aug)
        p, M = self.problem, self.hi - self.lo
        nnz = {k: len(p.array(k + "_p_colind")) for k in ("kxx", "kxu", "kuu")}
        out = {k: np.zeros((M, v)) for k, v in nnz.items()}
        out.update(rhat1=np.zeros((M, p.n_x)), rhat3=np.zeros((M, p.n_x)), rhat2=np.zeros(p.n_u))
        o = _CondensedOut(**{k: dptr(v) for k, v in out.items()})
        check(lib().bipm_condense(self._h, ctypes.byref(a), ctypes.byref(o)))
        return out

    def _condensed(self, arrays: dict):
        keep = {k: _f64(arrays[k]) for k, _ in _Condensed._fields_}
        return keep, _Condensed(**{k: dptr(v) for k, v in keep.items()})

    def reduce_rhs(self, delta_w: float, **arrays):
        """reduce_rhs_group (kkt.cpp:209-239), summed over the ctx's scenarios."""
        keep, c = self._condensed(arrays)
        rhs = np.zeros(self.problem.n_u)
        check(lib().bipm_reduce_rhs(self._h, ctypes.byref(c), delta_w, dptr(rhs)))
        return rhs

    def recover(self, delta_w: float, pu, hx, hu, sigma_s, r2, r4, **arrays):
        """recover_state_adjoint + recover_slack_dual (kkt.cpp:507-532, 172-188)."""
        keep, c = self._condensed(arrays)
        srk = [_f64(v) for v in (hx, hu, sigma_s, r2, r4)]
        sr = _SlackRows(*[dptr(v) for v in srk])
        p, M = self.problem, self.hi - self.lo
        pu = _f64(pu)
        px, py = np.zeros((M, p.n_x)), np.zeros((M, p.n_x))
        pz, ps = np.zeros((M, p.m)), np.zeros((M, p.m))
        check(lib().bipm_recover(self._h, ctypes.byref(c), ctypes.byref(sr), delta_w, dptr(pu),
                                 dptr(px), dptr(py), dptr(pz), dptr(ps)))
        return {"px": px, "py": py, "pz": pz, "ps": ps}

    def solve_reduced(self, delta_w_last: float = 0.0, reg: dict | None = None, **aug):
        """solve_reduced (kkt.cpp:945-1006) through bipm_solve_reduced.
        Returns (step dict, info dict, delta_w_last)."""
        keep, a = self._augmented(aug)
        p, M = self.problem, self.hi - self.lo
        out = {"px": np.zeros((M, p.n_x)), "pu": np.zeros(p.n_u), "ps": np.zeros((M, p.m)),
               "pz": np.zeros((M, p.m)), "py": np.zeros((M, p.n_x))}
        st = _Step(**{k: dptr(v) for k, v in out.items()})
        r = _RegSchedule(**(reg or {}))
        dwl = ctypes.c_double(delta_w_last)
        info = _StepInfo()
        check(lib().bipm_solve_reduced(self._h, ctypes.byref(a), ctypes.byref(r),
                                       ctypes.byref(dwl), ctypes.byref(st), ctypes.byref(info)))
        return out, {k: getattr(info, k) for k, _ in _StepInfo._fields_}, dwl.value

    def bundle_shapes(self):
        p, M = self.problem, self.hi - self.lo
        nnz = {k: len(p.array(k + "_p_colind")) for k in ("gx", "gu", "hx", "hu", "wxx", "wxu",
                                                           "wuu")}
        shapes = {"f": (M,), "g": (M, p.n_x), "h": (M, p.m), "grad_lag": (M, p.n_x + p.n_u)}
        shapes.update({k: (M, v) for k, v in nnz.items()})
        return shapes

    def eval_bundle(self, X, u, y, z, obj_weight=1.0):
        """eval_bundle_range (autodiff.cpp:484-516) through bipm_eval_bundle."""
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (X, u, y, z)]
        out = {k: np.zeros(s) for k, s in self.bundle_shapes().items()}
        b = _Bundle(**{k: dptr(v) for k, v in out.items()})
        bad = ctypes.c_int32(-1)
        check(lib().bipm_eval_bundle(self._h, *[dptr(a) for a in arrs], obj_weight,
                                     ctypes.byref(b), ctypes.byref(bad)))
        return out

    def eval_values(self, X, u):
        """batch_eval (autodiff.cpp:256-281) through bipm_eval_values."""
        p, M = self.problem, self.hi - self.lo
        X = np.ascontiguousarray(X, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        f, g, h = np.zeros(M), np.zeros((M, p.n_x)), np.zeros((M, p.m))
        bad = ctypes.c_int32(-1)
        check(lib().bipm_eval_values(self._h, dptr(X), dptr(u), dptr(f), dptr(g), dptr(h),
                                     ctypes.byref(bad)))
        return f, g, h

    def set_nccl(self, uid: bytes, nranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        check(lib().bipm_ctx_set_nccl(self._h, buf, nranks, rank))

    def set_host_comm(self, allreduce, nranks: int, rank: int):
        """allreduce(np.ndarray view, op) with op 0 sum / 1 max / 2 min, in place."""
        def cb(_user, buf, n, op):
            allreduce(np.ctypeslib.as_array(buf, shape=(n,)), op)
        self._cb = ALLREDUCE_FN(cb)  # keep alive
        check(lib().bipm_ctx_set_host_comm(self._h, ctypes.cast(self._cb, ctypes.c_void_p), None,
                                           nranks, rank))

    def profile(self, enable: bool = True):
        check(lib().bipm_ctx_profile(self._h, 1 if enable else 0))

    def kernel_time(self, name: str):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib().bipm_ctx_kernel_time(self._h, name.encode(), ctypes.byref(ms),
                                         ctypes.byref(n)))
        return ms.value, n.value

    def phase_stamps(self, enable: bool):
        out = (ctypes.c_int64 * 16)()
        check(lib().bipm_ctx_phase_stamps(self._h, 1 if enable else 0, out))
        return list(out)

    def step_stamps(self, enable: bool, cap: int = 8192):
        """(kind, clock64 before the step's data wait, after it) per step of the
        streamed reduction (debug)."""
        out = (ctypes.c_int64 * cap)()
        n = ctypes.c_int32(0)
        check(lib().bipm_ctx_step_stamps(self._h, 1 if enable else 0, out, cap, ctypes.byref(n)))
        return [(out[3 * j], out[3 * j + 1], out[3 * j + 2]) for j in range(n.value)]

    def debug_buffer(self, cap: int = 200000):
        out = (ctypes.c_int64 * cap)()
        n = ctypes.c_int64(0)
        check(lib().bipm_ctx_debug_buffer(self._h, out, cap, ctypes.byref(n)))
        return list(out[:n.value])

    def factor_stats(self) -> dict:
        out = (ctypes.c_int64 * 2)()
        check(lib().bipm_ctx_factor_stats(self._h, out))
        return {"bk_fallbacks": out[0], "khat_bk": bool(out[1])}

    def comm_info(self) -> dict:
        """The context's exchange: kind (none / nccl / host), ranks, rank."""
        out = (ctypes.c_int32 * 3)()
        check(lib().bipm_ctx_comm(self._h, out))
        return {"kind": {0: "none", 1: "nccl", 2: "host"}.get(out[0], str(out[0])),
                "nranks": out[1], "rank": out[2]}

    def info(self) -> dict:
        out = (ctypes.c_int64 * 12)()
        check(lib().bipm_ctx_info(self._h, out))
        keys = ("tile_cols", "chunk", "nchunks", "panel_in_smem", "nnz_l", "nnz_f", "lu_madds",
                "sm_count", "streamed", "steps", "ring_bytes", "nnz_vs")
        d = dict(zip(keys, list(out)))
        # streamed bits: 1 streamed reduction, 2 presolved forward half,
        # 4 adjoint identity (host/stream_plan.hpp)
        d["presolve"], d["adj_identity"] = int(bool(d["streamed"] & 2)), int(bool(d["streamed"] & 4))
        d["streamed"] &= 1
        return d

    def __del__(self):
        _destroy(self, "bipm_ctx_destroy")


class Solver:
    """The GPU interior-point driver (ipm.cpp:435-664) through bipm_solver_*."""

    def __init__(self, ctx: Context, tol: float = 1e-6, mu0: float = 0.1, max_iter: int = 300):
        self.ctx = ctx
        self._opts = _SolveOptions(tol, mu0, max_iter)
        h = _P()
        check(lib().bipm_solver_create(ctx._h, ctypes.byref(self._opts), ctypes.byref(h)))
        self._h = h

    def start(self):
        check(lib().bipm_solver_start(self._h))

    def step(self) -> int:
        st = ctypes.c_int32(-1)
        check(lib().bipm_solver_step(self._h, ctypes.byref(st)))
        return st.value

    def result(self):
        r = _SolveResult()
        u = np.zeros(self.ctx.problem.n_u)
        check(lib().bipm_solver_result(self._h, ctypes.byref(r), dptr(u)))
        out = {k: getattr(r, k) for k, _ in _SolveResult._fields_}
        out["status_name"] = SOLVE_STATUS.get(r.status, str(r.status))
        out["u"] = u
        out["logs"] = [self.log(k) for k in range(r.iterations)]
        return out

    def iterate(self) -> dict:
        """The current primal-dual point (Iterate, model.hpp:41-55)."""
        p, M = self.ctx.problem, self.ctx.hi - self.ctx.lo
        shapes = {"x": (M, p.n_x), "y": (M, p.n_x), "kappa_lo": (M, p.n_x),
                  "kappa_up": (M, p.n_x), "s": (M, p.m), "z": (M, p.m), "nu_lo": (M, p.m),
                  "nu_up": (M, p.m), "u": (p.n_u,), "lambda_lo": (p.n_u,),
                  "lambda_up": (p.n_u,)}
        out = {k: np.zeros(shapes[k]) for k in ITERATE_FIELDS}
        it = _Iterate(**{k: dptr(v) for k, v in out.items()})
        check(lib().bipm_solver_iterate(self._h, ctypes.byref(it)))
        return out

    def log(self, k: int) -> dict:
        rec = np.zeros(15)
        check(lib().bipm_solver_log(self._h, k, dptr(rec)))
        return dict(zip(LOG_FIELDS, rec.tolist()))

    def step_timed(self):
        st, ms = ctypes.c_int32(-1), ctypes.c_double()
        check(lib().bipm_solver_step_timed(self._h, ctypes.byref(st), ctypes.byref(ms)))
        return st.value, ms.value

    def solve(self):
        self.start()
        st = -1
        while st == -1:
            st = self.step()
        return self.result()

    def __del__(self):
        _destroy(self, "bipm_solver_destroy")


def counters() -> dict:
    out = (ctypes.c_int64 * 3)()
    check(lib().bipm_counters(out))
    return {"launches": out[0], "h2d_bytes": out[1], "d2h_bytes": out[2]}


def dense_inertia(K: np.ndarray, b: np.ndarray | None = None):
    """Bunch-Kaufman LDL' of the shifted K on the GPU: ((pos, neg, zero), K^{-1} b)."""
    K = np.ascontiguousarray(np.asarray(K, dtype=np.float64).T)  # column-major
    x = None if b is None else np.array(b, dtype=np.float64)
    out = (ctypes.c_int32 * 3)()
    check(lib().bipm_dense_inertia(len(K), dptr(K), None if x is None else dptr(x), out))
    return (out[0], out[1], out[2]), x


def dense_factor_solve(K: np.ndarray, b: np.ndarray):
    """factor_dense_sym + solve on the GPU: (positive_definite, K^{-1} b)."""
    K = np.ascontiguousarray(np.asarray(K, dtype=np.float64).T)  # column-major
    x = np.array(b, dtype=np.float64)
    pd = ctypes.c_int32(0)
    check(lib().bipm_dense_factor_solve(len(x), dptr(K), dptr(x), ctypes.byref(pd)))
    return bool(pd.value), x
