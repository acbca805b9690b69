"""Python binding of libsdc.so over torch CUDA tensors (argument marshalling only).

Every step of the split runs in libsdc's sm_100a kernels; this module only turns torch
tensors into (device pointer, leading dimension) pairs, passes the current CUDA stream,
and converts the C result struct.  Matrices are column-major fp64: a tensor `X` with
`X.stride() == (1, ld)` (e.g. `X.t().contiguous().t()`, or `colmajor(X)`).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import SdcResult, check, load

STOPS = {"fixed": _lib.STOP_FIXED, "rtest": _lib.STOP_RTEST, "e21": _lib.STOP_E21}


def colmajor(x: torch.Tensor) -> torch.Tensor:
    """Column-major (Fortran-ordered) fp64 view/copy of a 2-D tensor."""
    if x.dim() != 2:
        raise ValueError("expected a matrix")
    if x.dtype != torch.float64:
        x = x.to(torch.float64)
    if x.stride(0) == 1 and x.stride(1) >= max(1, x.shape[0]):
        return x
    return x.t().contiguous().t()


def empty_colmajor(m: int, n: int, device) -> torch.Tensor:
    return torch.empty((n, m), dtype=torch.float64, device=device).t()


def _ptr_ld(x: torch.Tensor | None):
    if x is None:
        return None, 1
    if not x.is_cuda or x.dtype != torch.float64 or (x.stride(0) != 1 and x.shape[0] > 1):
        raise ValueError("expected a column-major float64 CUDA tensor")
    ld = x.stride(1) if x.shape[1] > 1 else x.shape[0]
    return ctypes.c_void_p(x.data_ptr()), max(1, ld, x.shape[0])


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class SplitInfo:
    k: int
    r: int
    metric: float
    metric_fro: float
    iters: int
    converged: int
    status: int
    hist: np.ndarray


class Handle:
    """Owns libsdc workspace for matrices up to n_max on one device."""

    def __init__(self, n_max: int, pencil: bool = False, device: int | None = None):
        self.lib = load()
        self.device = torch.cuda.current_device() if device is None else device
        self.n_max = n_max
        self.pencil = pencil
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.sdc_create(ctypes.byref(h), self.device, n_max, int(pencil)), "sdc_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self.lib.sdc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.sdc_kernel_launches(self._h))

    def schedule_counters(self, reset: bool = False) -> dict:
        """sdc_schedule_counters: how often each schedule path was enqueued (evidence)."""
        out = (ctypes.c_longlong * len(_lib.SCHED_NAMES))()
        check(self.lib.sdc_schedule_counters(self._h, out, len(_lib.SCHED_NAMES), int(reset)),
              "sdc_schedule_counters")
        return dict(zip(_lib.SCHED_NAMES, (int(v) for v in out)))

    def profile(self, enable: bool = True):
        check(self.lib.sdc_profile(self._h, int(enable)), "sdc_profile")

    def profile_read(self, cls: int):
        ms, n, w = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        check(self.lib.sdc_profile_read(self._h, cls, ctypes.byref(ms), ctypes.byref(n),
                                        ctypes.byref(w)), "sdc_profile_read")
        return ms.value, n.value, w.value

    # ---- the step ---------------------------------------------------------------------
    def split(self, A, B=None, V=None, VL=None, max_iters=12, tol=0.0, stop="fixed",
              Q=None, QL=None, want_ahat=False, hist_cap=None, region="unit_disk", param=1.0,
              symmetric=False, ql_orth=False):
        """sdc_split_region: returns (Q, QL or None, Ahat or None, SplitInfo).
        region: "unit_disk" | "disk" (|z| < param) | "halfplane" (Re z < param)."""
        n = A.shape[0]
        dev = A.device
        A, V = colmajor(A), colmajor(V)
        B = None if B is None else colmajor(B)
        VL = None if VL is None else colmajor(VL)
        Q = empty_colmajor(n, n, dev) if Q is None else Q
        if B is not None and QL is None:
            QL = empty_colmajor(n, n, dev)
        Ah = empty_colmajor(n, n, dev) if want_ahat else None
        hist_cap = max_iters if hist_cap is None else hist_cap
        hist = np.full((hist_cap, 3), np.nan)
        res = SdcResult()
        pa, la = _ptr_ld(A)
        pb, lb = _ptr_ld(B)
        pv, lv = _ptr_ld(V)
        pvl, lvl = _ptr_ld(VL)
        pq, lq = _ptr_ld(Q)
        pql, lql = _ptr_ld(QL)
        pah, lah = _ptr_ld(Ah)
        reg = {"unit_disk": _lib.REGION_UNIT_DISK, "disk": _lib.REGION_DISK,
               "halfplane": _lib.REGION_HALFPLANE}[region]
        rc = self.lib.sdc_split_region(self._h, _stream(dev), n, pa, la, pb, lb, pv, lv, pvl, lvl,
                                       reg, float(param),
                                       (_lib.FLAG_SYMMETRIC if symmetric else 0) |
                                       (_lib.FLAG_QL_ORTH if ql_orth else 0),
                                       max_iters, float(tol), STOPS[stop], pq, lq, pql, lql, pah,
                                       lah, hist.ctypes.data_as(ctypes.c_void_p), hist_cap,
                                       ctypes.byref(res))
        check(rc, "sdc_split")
        info = SplitInfo(res.k, res.r, res.metric, res.metric_fro, res.iters, res.converged,
                         res.status, hist)
        return Q, QL, Ah, info

    def svd_split(self, A, rho, V, max_iters=12, tol=0.0, stop="fixed", Q=None, want_ahat=False,
                  hist_cap=None):
        """sdc_svd_split: singular values of the m x n A below rho.
        Returns (Q (m+n)x(m+n), Ahat or None, SplitInfo); info.k = 2 #{sigma < rho} + |m-n|."""
        m, n = A.shape
        N = m + n
        dev = A.device
        A, V = colmajor(A), colmajor(V)
        Q = empty_colmajor(N, N, dev) if Q is None else Q
        Ah = empty_colmajor(N, N, dev) if want_ahat else None
        hist_cap = max_iters if hist_cap is None else hist_cap
        hist = np.full((hist_cap, 3), np.nan)
        res = SdcResult()
        pa, la = _ptr_ld(A)
        pv, lv = _ptr_ld(V)
        pq, lq = _ptr_ld(Q)
        pah, lah = _ptr_ld(Ah)
        rc = self.lib.sdc_svd_split(self._h, _stream(dev), m, n, pa, la, float(rho), pv, lv,
                                    max_iters, float(tol), STOPS[stop], pq, lq, pah, lah,
                                    hist.ctypes.data_as(ctypes.c_void_p), hist_cap, ctypes.byref(res))
        check(rc, "sdc_svd_split")
        return Q, Ah, SplitInfo(res.k, res.r, res.metric, res.metric_fro, res.iters, res.converged,
                                res.status, hist)

    def split_batched(self, A, V, max_iters=12, Q=None):
        """sdc_split_batched: A, V of shape (batch, n, n) with each A[b] column-major (e.g.
        A = X.transpose(1, 2).contiguous().transpose(1, 2)); returns (Q, [SplitInfo])."""
        if A.dim() != 3 or A.shape[1] != A.shape[2]:
            raise ValueError("A must be (batch, n, n)")
        batch, n, _ = A.shape
        if Q is None:
            Q = torch.empty((batch, n, n), dtype=torch.float64, device=A.device).transpose(1, 2)
        # the C ABI cannot see buffer sizes: V and Q must match A's batch and order
        for name, x in (("A", A), ("V", V), ("Q", Q)):
            if tuple(x.shape) != (batch, n, n):
                raise ValueError(f"{name} must have shape {(batch, n, n)}, got {tuple(x.shape)}")
            if (x.dtype != torch.float64 or not x.is_cuda or x.device != A.device or
                    (n > 1 and x.stride(1) != 1) or x.stride(2) < n or
                    (batch > 1 and x.stride(0) < x.stride(2) * n)):
                raise ValueError(f"{name}: expected (batch, n, n) column-major float64 CUDA tensors")
        res = (SdcResult * max(1, batch))()
        check(self.lib.sdc_split_batched(self._h, _stream(A.device), batch, n,
                                         ctypes.c_void_p(A.data_ptr()), A.stride(2), A.stride(0),
                                         ctypes.c_void_p(V.data_ptr()), V.stride(2), V.stride(0),
                                         max_iters, ctypes.c_void_p(Q.data_ptr()), Q.stride(2),
                                         Q.stride(0), res), "sdc_split_batched")
        infos = [SplitInfo(r.k, r.r, r.metric, r.metric_fro, r.iters, r.converged, r.status, None)
                 for r in res[:batch]]
        return Q, infos

    def schur(self, A, leaf=1, seed=1, max_iters=60, tol=1e-13, Q=None, T=None, key_off=0):
        """sdc_schur_keyed: recursive divide-and-conquer A = Q T Q^T; key_off
        is the global offset of A in a larger recursion (draws keyed by it).
        Returns (Q, T, blocks [(offset, size)], stats dict)."""
        n = A.shape[0]
        A = colmajor(A)
        Q = empty_colmajor(n, n, A.device) if Q is None else Q
        T = empty_colmajor(n, n, A.device) if T is None else T
        off = np.zeros(n, dtype=np.int32)
        size = np.zeros(n, dtype=np.int32)
        nb = ctypes.c_int(0)
        stats = np.zeros(4, dtype=np.int32)
        mm = ctypes.c_double(0.0)
        pa, la = _ptr_ld(A)
        pq, lq = _ptr_ld(Q)
        pt, lt = _ptr_ld(T)
        check(self.lib.sdc_schur_keyed(self._h, _stream(A.device), n, pa, la, int(key_off), int(leaf),
                                       int(seed), int(max_iters), float(tol), pq, lq, pt, lt,
                                 off.ctypes.data_as(ctypes.c_void_p), size.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(nb), stats.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(mm)), "sdc_schur")
        blocks = [(int(off[i]), int(size[i])) for i in range(nb.value)]
        info = {"splits": int(stats[0]), "failed_attempts": int(stats[1]), "unsplit": int(stats[2]),
                "passes": int(stats[3]), "max_metric": mm.value}
        return Q, T, blocks, info

    def schur_node(self, Tb, key_off, leaf=1, seed=1, max_iters=60, tol=1e-13, Qb=None, stats=None):
        """sdc_schur_node: one node of the recursion on the diagonal block Tb (in place).
        Returns (r, Qb); r = 0: leaf / unsplit.  stats: optional int32[4] + [max_metric]
        accumulators (numpy), updated in place."""
        m = Tb.shape[0]
        pt, lt = _ptr_ld(Tb)
        if Tb.shape != (m, m):
            raise ValueError("Tb must be square")
        Qb = empty_colmajor(m, m, Tb.device) if Qb is None else Qb
        pq, lq = _ptr_ld(Qb)
        st = np.zeros(4, dtype=np.int32) if stats is None else stats[0]
        mm = ctypes.c_double(0.0 if stats is None else float(stats[1][0]))
        r = ctypes.c_int(0)
        check(self.lib.sdc_schur_node(self._h, _stream(Tb.device), m, pt, lt, int(key_off), int(leaf),
                                      int(seed), int(max_iters), float(tol), pq, lq, ctypes.byref(r),
                                      st.ctypes.data_as(ctypes.c_void_p), ctypes.byref(mm)),
              "sdc_schur_node")
        if stats is not None:
            stats[1][0] = mm.value
        return r.value, Qb

    def trevc(self, T, Q=None, X=None):
        """sdc_trevc: eigenvectors X (X_jj = 1, TX = XD) of the upper triangular T, or Q X
        when Q is given.  Enqueued on the current stream."""
        n = T.shape[0]
        T = colmajor(T)
        Q = None if Q is None else colmajor(Q)
        X = empty_colmajor(n, n, T.device) if X is None else X
        pt, lt = _ptr_ld(T)
        pq, lq = _ptr_ld(Q)
        px, lx = _ptr_ld(X)
        check(self.lib.sdc_trevc(self._h, _stream(T.device), n, pt, lt, pq, lq, px, lx), "sdc_trevc")
        return X

    def split_host(self, A: np.ndarray, B=None, V=None, VL=None, max_iters=12, tol=0.0,
                   stop="fixed", Q=None, QL=None, want_ahat=False, stream=None):
        """sdc_split_host on host (numpy, Fortran-ordered fp64) buffers: the end-to-end path."""
        n = A.shape[0]

        def f(x):
            return None if x is None else np.asfortranarray(x, dtype=np.float64)

        A, B, V, VL = f(A), f(B), f(V), f(VL)
        Q = np.empty((n, n), order="F") if Q is None else Q
        if B is not None and QL is None:
            QL = np.empty((n, n), order="F")
        # host buffers are read / written as n x n column-major fp64
        for name, x in (("A", A), ("B", B), ("V", V), ("VL", VL), ("Q", Q), ("QL", QL)):
            if x is None:
                continue
            if x.shape != (n, n):
                raise ValueError(f"{name} must be {n} x {n}, got {x.shape}")
            if x.dtype != np.float64 or not x.flags.f_contiguous:
                raise ValueError(f"{name} must be a Fortran-ordered float64 array")
        if B is not None and VL is None:
            raise ValueError("a pencil (B given) needs VL")
        Ah = np.empty((n, n), order="F") if want_ahat else None
        hist = np.full((max_iters, 3), np.nan)
        res = SdcResult()

        def p(x):
            return None if x is None else x.ctypes.data_as(ctypes.c_void_p)

        st = _stream(torch.device("cuda", self.device)) if stream is None else stream
        rc = self.lib.sdc_split_host(self._h, st, n, p(A), p(B), p(V), p(VL), max_iters,
                                     float(tol), STOPS[stop], p(Q), p(QL), p(Ah), p(hist),
                                     max_iters, ctypes.byref(res))
        check(rc, "sdc_split_host")
        return Q, QL, Ah, SplitInfo(res.k, res.r, res.metric, res.metric_fro, res.iters,
                                    res.converged, res.status, hist)

    # ---- building blocks (kernel-level parity tests) ------------------------------------
    def dgemm(self, A, B, transa=False, transb=False, alpha=1.0, beta=0.0, C=None):
        A, B = colmajor(A), colmajor(B)
        M = A.shape[1] if transa else A.shape[0]
        K = A.shape[0] if transa else A.shape[1]
        N = B.shape[0] if transb else B.shape[1]
        C = empty_colmajor(M, N, A.device) if C is None else C
        pa, la = _ptr_ld(A)
        pb, lb = _ptr_ld(B)
        pc, lc = _ptr_ld(C)
        check(self.lib.sdc_dgemm(self._h, _stream(A.device), int(transa), int(transb), M, N, K,
                                 float(alpha), pa, la, pb, lb, float(beta), pc, lc), "sdc_dgemm")
        return C

    def qr(self, A, want_q=True):
        """Blocked Householder QR; returns (Q thin with diag(R)>=0, R with diag>=0)."""
        A = colmajor(A).clone().t().contiguous().t()
        m, n = A.shape
        Q = empty_colmajor(m, n, A.device) if want_q else None
        pa, la = _ptr_ld(A)
        pq, lq = _ptr_ld(Q)
        check(self.lib.sdc_qr(self._h, _stream(A.device), m, n, pa, la, pq, lq), "sdc_qr")
        return Q, torch.triu(A[:n, :n])   # sdc_qr leaves R with diag >= 0 in the upper triangle

    def irs_pass(self, A, B):
        A, B = colmajor(A), colmajor(B)
        n = A.shape[0]
        Ao, Bo, R = (empty_colmajor(n, n, A.device) for _ in range(3))
        args = []
        for x in (A, B, Ao, Bo, R):
            args += list(_ptr_ld(x))
        check(self.lib.sdc_irs_pass(self._h, _stream(A.device), n, *args), "sdc_irs_pass")
        return Ao, Bo, R

    def split_select(self, Ahat, normA, Bhat=None, normB=1.0):
        Ahat = colmajor(Ahat)
        Bhat = None if Bhat is None else colmajor(Bhat)
        n = Ahat.shape[0]
        mv = torch.zeros(n, dtype=torch.float64, device=Ahat.device)
        r = ctypes.c_int(0)
        met = ctypes.c_double(0)
        pa, la = _ptr_ld(Ahat)
        pb, lb = _ptr_ld(Bhat)
        check(self.lib.sdc_split_select(self._h, _stream(Ahat.device), n, pa, la, float(normA), pb,
                                        lb, float(normB), ctypes.byref(r), ctypes.byref(met),
                                        ctypes.c_void_p(mv.data_ptr())), "sdc_split_select")
        return r.value, met.value, mv
