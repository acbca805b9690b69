"""ctypes declarations of libsdc.so (include/sdc.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsdc.so")

STOP_FIXED, STOP_RTEST, STOP_E21 = 0, 1, 2
STATUS_SPLIT, STATUS_NO_SPLIT, STATUS_NONFINITE = 0, 1, 2
REGION_UNIT_DISK, REGION_DISK, REGION_HALFPLANE = 0, 1, 2
FLAG_SYMMETRIC, FLAG_PLATEAU, FLAG_ONESIDED, FLAG_QL_ORTH = 1, 2, 4, 8
PROF_GEMM, PROF_PANEL, PROF_WYRED, PROF_SELECT, PROF_GEMM_W0, PROF_GEMM_UPD, PROF_GEMM_OTHER = 0, 1, 2, 3, 4, 5, 6
SPLIT_ACCEPT = 1e-8
SCHED_NAMES = ("lookahead_forks", "xpass_forks", "ctx_forks", "panel_cluster", "panel_mcluster",
               "panel_grid", "graph_captures", "graph_replays", "panel_mcluster_capped", "panel_cqr_tried",
               "panel_cqr_done", "panel_cqr_fallback", "gemm_cpasync", "max_clusters16",
               "panel_mcluster8", "gemm_tma", "schur_batch_launches", "schur_batch_blocks",
               "panel_cq_split", "cq_split_breakdowns")


class SdcResult(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int), ("r", ctypes.c_int), ("metric", ctypes.c_double),
                ("metric_fro", ctypes.c_double), ("iters", ctypes.c_int),
                ("converged", ctypes.c_int), ("status", ctypes.c_int), ("side", ctypes.c_double)]


_lib = None
P, I, D, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong

_SIGS = {
    "sdc_create": (I, [ctypes.POINTER(P), I, I, I]),
    "sdc_destroy": (None, [P]),
    "sdc_split": (I, [P, P, I, P, I, P, I, P, I, P, I, I, I, D, I, P, I, P, I, P, I, P, I,
                      ctypes.POINTER(SdcResult)]),
    "sdc_split_region": (I, [P, P, I, P, I, P, I, P, I, P, I, I, D, I, I, D, I, P, I, P, I, P, I, P, I,
                             ctypes.POINTER(SdcResult)]),
    "sdc_trevc": (I, [P, P, I, P, I, P, I, P, I]),
    "sdc_split_batched": (I, [P, P, I, I, P, I, LL, P, I, LL, I, P, I, LL, P]),
    "sdc_schur": (I, [P, P, I, P, I, I, ctypes.c_ulonglong, I, D, P, I, P, I, P, P,
                      ctypes.POINTER(I), P, ctypes.POINTER(D)]),
    "sdc_schur_keyed": (I, [P, P, I, P, I, I, I, ctypes.c_ulonglong, I, D, P, I, P, I, P, P,
                            ctypes.POINTER(I), P, ctypes.POINTER(D)]),
    "sdc_schur_node": (I, [P, P, I, P, I, I, I, ctypes.c_ulonglong, I, D, P, I, ctypes.POINTER(I), P,
                           ctypes.POINTER(D)]),
    "sdc_svd_split": (I, [P, P, I, I, P, I, D, P, I, I, D, I, P, I, P, I, P, I,
                          ctypes.POINTER(SdcResult)]),
    "sdc_split_host": (I, [P, P, I, P, P, P, P, I, D, I, P, P, P, P, I, ctypes.POINTER(SdcResult)]),
    "sdc_dgemm": (I, [P, P, I, I, I, I, I, D, P, I, P, I, D, P, I]),
    "sdc_qr": (I, [P, P, I, I, P, I, P, I]),
    "sdc_irs_pass": (I, [P, P, I, P, I, P, I, P, I, P, I, P, I]),
    "sdc_split_select": (I, [P, P, I, P, I, D, P, I, D, ctypes.POINTER(I), ctypes.POINTER(D), P]),
    "sdc_kernel_launches": (LL, [P]),
    "sdc_schedule_counters": (I, [P, P, I, I]),
    "sdc_profile": (I, [P, I]),
    "sdc_debug_counters": (I, [P, P, I, I]),
    "sdc_profile_read": (I, [P, I, ctypes.POINTER(D), ctypes.POINTER(LL), ctypes.POINTER(D)]),
    "sdc_last_error": (ctypes.c_char_p, []),
}
EXPORTS = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load libsdc.so.  There is no fallback: a missing library is an error."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_1011_3077_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class SdcError(RuntimeError):
    pass


def check(rc: int, what: str):
    if rc != 0:
        msg = load().sdc_last_error().decode(errors="replace")
        raise SdcError(f"{what} failed with {rc}: {msg}")
