"""The C-ABI library loads and exports every entry point include/rbe_cuda.h
declares; without a GPU the compute entry points fail loudly (no fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from tests.helpers import HAS_GPU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rbe_cuda.h")
LIB = os.path.join(ROOT, "paper_1802_06466_b200", "_lib", "librbe_cuda.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rbe_cuda_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("rbe_cuda_index_create", "rbe_cuda_index_upload_partition", "rbe_cuda_index_fill_synthetic",
                 "rbe_cuda_index_destroy", "rbe_cuda_search", "rbe_cuda_search_device", "rbe_cuda_merge_device",
                 "rbe_cuda_search_multi", "rbe_cuda_last_error", "rbe_cuda_version",
                 "rbe_cuda_index_last_batch_ms"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run python -m paper_1802_06466_b200.build"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(\w+)$", out, re.M))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    lib = C.CDLL(LIB)
    for n in declared():
        assert hasattr(lib, n)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(HAS_GPU, reason="CPU-only behaviour")
def test_no_gpu_fails_loudly():
    lib = C.CDLL(LIB)
    lib.rbe_cuda_last_error.restype = C.c_char_p

    class Shape(C.Structure):
        _fields_ = [("dim", C.c_uint32), ("kp", C.c_uint32), ("rw", C.c_uint32)]

    h = C.c_void_p()
    ords = (C.c_uint32 * 1)(0)
    counts = (C.c_uint64 * 1)(10)
    rc = lib.rbe_cuda_index_create(C.byref(Shape(64, 2, 1)), 1, ords, counts, 0, C.byref(h))
    assert rc == 3  # RBE_CUDA_ERUNTIME
    assert b"no CPU fallback" in lib.rbe_cuda_last_error()
    rc = lib.rbe_cuda_index_create(C.byref(Shape(0, 2, 1)), 1, ords, counts, 0, C.byref(h))
    assert rc == 1  # EINVAL checked before touching the device


def test_ctypes_binding_declares_only_exported_symbols():
    """The reference-side ctypes binding (tests/rbe_ctypes.py, shown in INTEGRATION.md)
    loads on CPU and every function it types is exported and declared in the header."""
    from tests import rbe_ctypes

    lib = rbe_ctypes.load()
    typed = [n for n in dir(lib) if n.startswith("rbe_cuda_")]
    names = set(declared())
    for n in ("rbe_cuda_index_create", "rbe_cuda_index_upload_partition", "rbe_cuda_search",
              "rbe_cuda_index_destroy", "rbe_cuda_last_error"):
        assert n in names
        assert getattr(lib, n).argtypes is not None
    assert all(n in names for n in typed)
