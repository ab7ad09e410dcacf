"""queue_length >= items_per_thread (the lossless regime): BoundedQueue keeps every
item of a logical thread (reference src/search.cpp:32-48), so the search is the exact top n under
(score desc, id asc).  The tensor scan serves it by emitting every pair >= theta directly; results
must equal the compiled reference and the CUDA-core exact kernel."""
import numpy as np
import pytest

from oracle.oracle import gen_queries, synthetic_partitions
from tests.test_gpu_parity import gpu_search

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("geo_tail,P,N", [
    ((256, 256, 256), 1, 300_007),
    ((256, 16, 16), 2, 200_003),
    ((128, 32, 1000), 3, 150_001),
    ((256, 256, 256), 1, 10_000_000),
])
def test_lossless_tensor_matches_reference(rbe, ref, port, geo_tail, P, N):
    dim, kp, qp, Q, n = 128, 3, 3, 8, 500
    tpb, ipt, ql = geo_tail
    per = -(-N // P)
    geo = (-(-per // (tpb * ipt)), tpb, ipt, ql)
    dix = rbe.DeviceIndex.synthetic(dim, kp, True, N, P, 0xD0C5)
    qs = gen_queries(0x0E1 + ql, Q, dim, qp)
    got, accs, counts, st = gpu_search(rbe, dix, qs, geo, n, "tensor")
    assert st["variant"] == "tensor" and st["scored"] == Q * N
    parts = [dix.download_partition(p) for p in range(P)]
    want, _ = ref.index(dim, kp, True, parts).search(qs, geo, n, threads=8)
    assert got == want
    if N <= 1_000_000:
        ex, _, _, _ = gpu_search(rbe, dix, qs, geo, n, "exact")
        assert ex == got
