"""CPU-side checks of the C ABI boundary (-m "not gpu"): libsdc.so builds, loads and
exports every function include/sdc.h declares; without a GPU it fails loudly (no CPU
fallback).  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sdc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(sdc_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1011_3077_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for n in ("sdc_create", "sdc_destroy", "sdc_split", "sdc_split_host", "sdc_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1011_3077_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTS, f"{name} missing from the Python binding"


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = lib.sdc_create(ctypes.byref(h), 0, 64, 0)
    assert rc == -100
    assert b"no CPU fallback" in lib.sdc_last_error()


def test_sm100a_only_cubin():
    # the library carries sm_100a SASS (and no other architecture)
    import subprocess
    from paper_1011_3077_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_dmma_in_sass():
    # FP64 tensor-core instructions really are in the GEMM kernels
    import subprocess
    from paper_1011_3077_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB],
                         capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out


def test_schedule_counter_names_match_header():
    # the binding's counter names (api.Handle.schedule_counters) follow the enum of include/sdc.h
    import os
    import re
    from paper_1011_3077_b200 import _lib
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "sdc.h")).read()
    enum = dict((m.group(1), int(m.group(2))) for m in re.finditer(r"SDC_SCHED_([A-Z0-9_]+) = (\d+)", hdr))
    assert enum.pop("COUNTERS") == len(_lib.SCHED_NAMES) == len(enum)
    for name, idx in enum.items():
        assert _lib.SCHED_NAMES[idx].upper() == name, (name, idx, _lib.SCHED_NAMES[idx])
