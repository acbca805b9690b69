"""B200-native (sm_100a) inverse-free split step of randomized spectral divide-and-conquer
(arXiv 1011.3077).  The compute path is libsdc.so (hand-written CUDA behind the C ABI in
include/sdc.h); `api.Handle` is the thin torch binding.  Importing this package does not
load the library; `Handle(...)` does, and fails loudly if it is missing (no CPU fallback).
"""
__all__ = ["Handle", "colmajor", "empty_colmajor", "inputs"]


def __getattr__(name):
    if name in ("Handle", "colmajor", "empty_colmajor", "SplitInfo"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
