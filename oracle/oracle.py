"""ctypes/numpy wrapper over the C oracle (oracle/sdc_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Matrices are passed as
Fortran-ordered float64 numpy arrays (column-major, as the C code expects).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

STOP_FIXED, STOP_RTEST, STOP_E21 = 0, 1, 2
REGION_UNIT_DISK, REGION_DISK, REGION_HALFPLANE = 0, 1, 2
FLAG_SYMMETRIC, FLAG_PLATEAU, FLAG_ONESIDED, FLAG_QL_ORTH = 1, 2, 4, 8
STATUS_SPLIT, STATUS_NO_SPLIT, STATUS_NONFINITE = 0, 1, 2
SPLIT_ACCEPT = 1e-8


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, -O2 -ffp-contract=off -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sdc_oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Result(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int), ("r", ctypes.c_int), ("metric", ctypes.c_double),
                ("metric_fro", ctypes.c_double), ("iters", ctypes.c_int),
                ("converged", ctypes.c_int), ("status", ctypes.c_int), ("side", ctypes.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
            P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
            _lib.orc_split.restype = I
            _lib.orc_split.argtypes = [I, P, I, P, I, P, I, P, I, I, D, I, P, I, P, I, P, I, P, I,
                                       ctypes.POINTER(_Result)]
            _lib.orc_split_region.restype = I
            _lib.orc_split_region.argtypes = [I, P, I, P, I, P, I, P, I, I, D, I, I, D, I, P, I, P, I,
                                              P, I, P, I, ctypes.POINTER(_Result)]
            _lib.orc_svd_split.restype = I
            _lib.orc_svd_split.argtypes = [I, I, P, I, D, P, I, I, D, I, P, I, P, I, P, I,
                                           ctypes.POINTER(_Result)]
            U64 = ctypes.c_ulonglong
            _lib.orc_haar.restype = None
            _lib.orc_haar.argtypes = [I, U64, U64, P, I]
            _lib.orc_schur.restype = I
            _lib.orc_schur.argtypes = [I, P, I, I, U64, I, D, P, I, P, I, P, P, P, P, P]
            _lib.orc_schur_keyed.restype = I
            _lib.orc_schur_keyed.argtypes = [I, P, I, I, I, U64, I, D, P, I, P, I, P, P, P, P, P]
            _lib.orc_schur_node.restype = I
            _lib.orc_schur_node.argtypes = [I, P, I, I, I, U64, I, D, P, I, P, P]
            _lib.orc_split_select.restype = D
            _lib.orc_split_select.argtypes = [I, P, I, D, P, I, D, ctypes.POINTER(I), P]
            _lib.orc_norm1.restype = D
            _lib.orc_norm1.argtypes = [I, I, P, I]
            for name, args in {
                "orc_geqr2": [I, I, P, I, P],
                "orc_apply_qt": [I, I, P, I, P, I, P, I],
                "orc_org2r_signed": [I, P, I, P, P, I],
                "orc_complement": [I, P, I, P, P, I],
                "orc_gerq2": [I, P, I, P],
                "orc_orgr2_signed": [I, P, I, P, P, I],
                "orc_geql2": [I, P, I, P],
                "orc_org2l_signed": [I, P, I, P, P, I],
                "orc_gemm": [I, I, I, I, I, P, I, P, I, P, I],
                "orc_irs_pass": [I, P, I, P, I, P, I, P, I, P],
                "orc_grurv_right": [I, P, I, P, I, P, I, P, I, P, P],
                "orc_grurv_left": [I, P, I, P, I, P, I, P, I],
                "orc_trevc": [I, P, I, P, I, P, I],
                "orc_trevc_cols": [I, P, I, I, I, P, I],
            }.items():
                f = getattr(_lib, name)
                f.restype = None
                f.argtypes = args
    return _lib


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ---- building blocks (each mirrors one C routine) ------------------------------------
def geqr2(a):
    """Householder QR (dgeqr2). Returns (factored array, tau)."""
    a = _f(a).copy(order="F")
    m, n = a.shape
    tau = np.zeros(min(m, n))
    lib().orc_geqr2(m, n, _p(a), m, _p(tau))
    return a, tau


def qr_signed(a):
    """Q (m x n thin, explicit) and R (n x n) with diag(R) >= 0, via the oracle's geqr2.

    For square a uses orc_org2r_signed; for tall a, Q = H_0..H_{n-1} [I;0] D."""
    y, tau = geqr2(a)
    m, n = y.shape
    d = np.where(np.diag(y)[:n] < 0, -1.0, 1.0)
    r = d[:, None] * np.triu(y[:n, :n])
    if m == n:
        q = np.zeros((n, n), order="F")
        lib().orc_org2r_signed(n, _p(y), m, _p(tau), _p(q), n)
        return q, r
    # thin Q of a tall matrix: Q^T applied to identity columns, transposed back
    e = np.asfortranarray(np.eye(m))
    lib().orc_apply_qt(m, n, _p(y), m, _p(tau), m, _p(e), m)   # e = Q^T (full m x m)
    q = np.ascontiguousarray(e.T)[:, :n] * d[None, :]
    return np.asfortranarray(q), r


def complement(y, tau):
    """[Q12; Q22] = H_0..H_{n-1} [0; I] for a 2n x n geqr2 factorisation."""
    m, n = y.shape
    c = np.zeros((m, n), order="F")
    lib().orc_complement(n, _p(_f(y)), m, _p(np.ascontiguousarray(tau)), _p(c), m)
    return c


def rq_signed(a):
    """RQ (dgerq2) of square a: returns (R upper, diag >= 0; Q orthogonal) with a = R Q."""
    y = _f(a).copy(order="F")
    n = y.shape[0]
    tau = np.zeros(n)
    lib().orc_gerq2(n, _p(y), n, _p(tau))
    q = np.zeros((n, n), order="F")
    lib().orc_orgr2_signed(n, _p(y), n, _p(tau), _p(q), n)
    d = np.where(np.diag(y) < 0, -1.0, 1.0)
    r = np.triu(y) * d[None, :]
    return r, q


def ql_signed(a):
    """QL (dgeql2) of square a: returns (Q orthogonal, L lower, diag >= 0) with a = Q L."""
    y = _f(a).copy(order="F")
    n = y.shape[0]
    tau = np.zeros(n)
    lib().orc_geql2(n, _p(y), n, _p(tau))
    q = np.zeros((n, n), order="F")
    lib().orc_org2l_signed(n, _p(y), n, _p(tau), _p(q), n)
    d = np.where(np.diag(y) < 0, -1.0, 1.0)
    l = d[:, None] * np.tril(y)
    return q, l


def gemm(a, b, ta=False, tb=False):
    a, b = _f(a), _f(b)
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    c = np.zeros((m, n), order="F")
    lib().orc_gemm(int(ta), int(tb), m, n, k, _p(a), a.shape[0], _p(b), b.shape[0], _p(c), m)
    return c


def irs_pass(a, b):
    """One IRS pass; returns (A_{j+1}, B_{j+1}, R_j with diag >= 0)."""
    a, b = _f(a), _f(b)
    n = a.shape[0]
    ao = np.zeros((n, n), order="F")
    bo = np.zeros((n, n), order="F")
    r = np.zeros((n, n), order="F")
    lib().orc_irs_pass(n, _p(a), n, _p(b), n, _p(ao), n, _p(bo), n, _p(r))
    return ao, bo, r


def irs(a, b, passes):
    hist = []
    for _ in range(passes):
        a, b, r = irs_pass(a, b)
        hist.append(r)
    return a, b, hist


def grurv_right(ap, bp, v):
    """Q = GRURV(2, A_p+B_p, A_p; -1,+1); also returns R1, R2 (diag >= 0)."""
    ap, bp, v = _f(ap), _f(bp), _f(v)
    n = ap.shape[0]
    q = np.zeros((n, n), order="F")
    r1 = np.zeros((n, n), order="F")
    r2 = np.zeros((n, n), order="F")
    lib().orc_grurv_right(n, _p(ap), n, _p(bp), n, _p(v), n, _p(q), n, _p(r1), _p(r2))
    return q, r1, r2


def grurv_left(ap, bp, vl):
    ap, bp, vl = _f(ap), _f(bp), _f(vl)
    n = ap.shape[0]
    q = np.zeros((n, n), order="F")
    lib().orc_grurv_left(n, _p(ap), n, _p(bp), n, _p(vl), n, _p(q), n)
    return q


def split_select(ahat, norm_a, bhat=None, norm_b=1.0):
    """Returns (r, metric, m[1..n-1])."""
    ahat = _f(ahat)
    n = ahat.shape[0]
    bb = None if bhat is None else _f(bhat)
    r = ctypes.c_int(0)
    mv = np.zeros(max(n - 1, 0))
    met = lib().orc_split_select(n, _p(ahat), n, float(norm_a), _p(bb), n, float(norm_b),
                                 ctypes.byref(r), _p(mv))
    return r.value, met, mv


def norm1(a):
    a = _f(a)
    return lib().orc_norm1(a.shape[0], a.shape[1], _p(a), a.shape[0])


@dataclass
class SplitResult:
    Q: np.ndarray
    QL: np.ndarray | None
    Ahat: np.ndarray
    k: int
    r: int
    metric: float
    metric_fro: float
    iters: int
    converged: int
    status: int
    hist: np.ndarray


def split(A, B=None, V=None, VL=None, max_iters=12, tol=0.0, stop=STOP_FIXED,
          hist_cap=None, region=REGION_UNIT_DISK, param=1.0, flags=0) -> SplitResult:
    """The whole step (RNEP if B is None, RGNEP otherwise), mirroring sdc_split /
    sdc_split_region (region: unit disk, disk of radius param, half plane Re z < param)."""
    A = _f(A)
    n = A.shape[0]
    Bf = None if B is None else _f(B)
    V = _f(V)
    VLf = None if VL is None else _f(VL)
    hist_cap = max_iters if hist_cap is None else hist_cap
    Q = np.zeros((n, n), order="F")
    QL = np.zeros((n, n), order="F") if Bf is not None else None
    Ah = np.zeros((n, n), order="F")
    hist = np.full((hist_cap, 3), np.nan)
    res = _Result()
    rc = lib().orc_split_region(n, _p(A), n, _p(Bf), n, _p(V), n, _p(VLf), n, int(region),
                                float(param), int(flags), max_iters, float(tol), int(stop), _p(Q),
                                n, _p(QL), n, _p(Ah), n, _p(hist), hist_cap, ctypes.byref(res))
    if rc != 0:
        raise ValueError(f"orc_split returned {rc}")
    return SplitResult(Q, QL, Ah, res.k, res.r, res.metric, res.metric_fro, res.iters,
                       res.converged, res.status, hist)


def svd_split(A, rho, V, max_iters=12, tol=0.0, stop=STOP_FIXED, hist_cap=None) -> SplitResult:
    """Singular values of the m x n A below rho: RSEP step on [[0, A], [A^T, 0]]
    (PAPER.md:453); mirrors sdc_svd_split.  Q and Ahat are (m+n) x (m+n)."""
    A = _f(A)
    m, n = A.shape
    N = m + n
    V = _f(V)
    hist_cap = max_iters if hist_cap is None else hist_cap
    Q = np.zeros((N, N), order="F")
    Ah = np.zeros((N, N), order="F")
    hist = np.full((hist_cap, 3), np.nan)
    res = _Result()
    rc = lib().orc_svd_split(m, n, _p(A), m, float(rho), _p(V), N, max_iters, float(tol), int(stop),
                             _p(Q), N, _p(Ah), N, _p(hist), hist_cap, ctypes.byref(res))
    if rc != 0:
        raise ValueError(f"orc_svd_split returned {rc}")
    return SplitResult(Q, None, Ah, res.k, res.r, res.metric, res.metric_fro, res.iters,
                       res.converged, res.status, hist)


def trevc(T, Q=None):
    """Eigenvectors X (upper triangular, X_jj = 1) of the upper triangular T, TX = XD
    (PAPER.md:1018-1027); Q X when Q is given (eigenvectors of A = Q T Q^T)."""
    T = _f(T)
    n = T.shape[0]
    Qf = None if Q is None else _f(Q)
    X = np.zeros((n, n), order="F")
    lib().orc_trevc(n, _p(T), n, _p(Qf), n, _p(X), n)
    return X


def trevc_cols(T, j0, j1):
    """Columns j0..j1-1 of TREVC's X (n x (j1-j0)), same arithmetic as trevc."""
    T = _f(T)
    n = T.shape[0]
    X = np.zeros((n, n), order="F")
    lib().orc_trevc_cols(n, _p(T), n, int(j0), int(j1), _p(X), n)
    return X[:, j0:j1]


def haar_stream(m, seed, key):
    """Haar V of order m from the counter-based Gaussian stream (seed, key)."""
    V = np.zeros((m, m), order="F")
    lib().orc_haar(int(m), int(seed), int(key), _p(V), int(m))
    return V


@dataclass
class SchurResult:
    Q: np.ndarray
    T: np.ndarray
    blocks: list          # [(offset, size)] in processing order
    splits: int
    failed_attempts: int
    unsplit: int
    passes: int
    max_metric: float


def schur(A, leaf=1, seed=1, max_iters=60, tol=1e-13, key_off=0) -> SchurResult:
    """Recursive divide-and-conquer A = Q T Q^T, T block upper triangular;
    key_off: global offset of A's first row (a subproblem's random draws are keyed by it)."""
    A = _f(A)
    n = A.shape[0]
    Q = np.zeros((n, n), order="F")
    T = np.zeros((n, n), order="F")
    off = np.zeros(n, dtype=np.int32)
    size = np.zeros(n, dtype=np.int32)
    nb = ctypes.c_int(0)
    stats = np.zeros(4, dtype=np.int32)
    mm = ctypes.c_double(0.0)
    rc = lib().orc_schur_keyed(n, _p(A), n, int(key_off), int(leaf), int(seed), int(max_iters),
                               float(tol), _p(Q), n, _p(T), n, off.ctypes.data_as(ctypes.c_void_p),
                         size.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nb),
                         stats.ctypes.data_as(ctypes.c_void_p), ctypes.byref(mm))
    if rc != 0:
        raise ValueError(f"orc_schur returned {rc}")
    blocks = [(int(off[i]), int(size[i])) for i in range(nb.value)]
    return SchurResult(Q, T, blocks, int(stats[0]), int(stats[1]), int(stats[2]), int(stats[3]),
                       mm.value)


def schur_node(Tb, o, leaf=1, seed=1, max_iters=60, tol=1e-13):
    """One node of the recursion on the diagonal block Tb at global offset o (in place:
    Tb <- Ahat with E21 = 0 when split).  Returns (r, Qb or None, stats[4], max_metric);
    r = 0: leaf or unsplit block."""
    m = Tb.shape[0]
    assert Tb.flags.f_contiguous and Tb.dtype == np.float64
    Qb = np.zeros((m, m), order="F")
    stats = np.zeros(4, dtype=np.int32)
    mm = ctypes.c_double(0.0)
    r = lib().orc_schur_node(m, _p(Tb), m, int(o), int(leaf), int(seed), int(max_iters), float(tol),
                             _p(Qb), m, stats.ctypes.data_as(ctypes.c_void_p), ctypes.byref(mm))
    if r < 0:
        raise ValueError(f"orc_schur_node returned {r}")
    return r, (Qb if r > 0 else None), stats, mm.value
