"""The C ABI driven directly through ctypes with declared argtypes (the binding
INTEGRATION.md shows, tests/rbe_ctypes.py): create / upload_partition / search /
destroy, results equal to the compiled reference, errors as status codes."""
import numpy as np
import pytest

from oracle.oracle import gen_queries, synthetic_partitions
from tests import rbe_ctypes

pytestmark = pytest.mark.gpu


def test_ctypes_binding_matches_reference(ref, port):
    lib = rbe_ctypes.load()
    assert lib.rbe_cuda_version().startswith(b"rbe_cuda")
    dim, kp, qp, P, N, n = 128, 3, 3, 3, 300_007, 250
    parts = synthetic_partitions(61, N, dim, kp, P, True, port)
    ix = rbe_ctypes.Index(lib, dim, kp, True, parts)
    qs = gen_queries(62, 5, dim, qp)
    geo = (2, 256, 256, 1)
    got, st = ix.search(qs, geo, n)
    want, scored = ref.index(dim, kp, True, parts).search(qs, geo, n)
    assert got == want
    assert st.scored == scored == 5 * N and st.variant == 2  # RBE_VARIANT_TENSOR
    dev, scan = rbe_ctypes.C.c_uint64(), rbe_ctypes.C.c_uint64()
    assert lib.rbe_cuda_index_bytes(ix.h, rbe_ctypes.C.byref(dev), rbe_ctypes.C.byref(scan)) == 0
    assert scan.value == N * (kp * 2 * 8 + 4)
    # reference error semantics through status codes
    with pytest.raises(ValueError, match="geometry does not cover partition"):
        ix.search(qs, (1, 16, 16, 1), n)
    with pytest.raises(ValueError, match="queue_length must be positive"):
        ix.search(qs, (2, 256, 256, 0), n)
    with pytest.raises(IndexError):
        ix._ck(lib.rbe_cuda_index_upload_partition(ix.h, 7, parts[0][0].reshape(-1), parts[0][1], parts[0][2]))
    ix.close()


def test_ctypes_open_rbei_matches_reference(ref, port, tmp_path):
    """rbe_cuda_index_open_rbei through ctypes on a file the reference wrote (save_index)."""
    lib = rbe_ctypes.load()
    dim, kp, qp, P, N, n = 128, 3, 3, 2, 100_003, 100
    parts = synthetic_partitions(63, N, dim, kp, P, True, port)
    r = ref.index(dim, kp, True, parts)
    r.save(tmp_path / "ix.rbei")
    ix = rbe_ctypes.Index.open_rbei(lib, tmp_path / "ix.rbei")
    assert ix.stats.file_bytes_read == N * (kp * 2 * 8 + 12)
    qs = gen_queries(64, 4, dim, qp)
    geo = (1, 256, 256, 1)
    got, _ = ix.search(qs, geo, n)
    want, _ = r.search(qs, geo, n)
    assert got == want
    ix.close()
