"""GPU parity: the B200 path (through the C ABI: DeviceIndex.search_words ->
rbe_cuda_search) against the compiled reference (oracle/_ref) and the golden
fixtures, bit-exact: same ids, same order/tie-breaks, identical double scores,
exact integer accumulators, SearchStats.scored == Q * N."""
import json
import math
import os

import numpy as np
import pytest

from oracle.oracle import Ref, gen_queries, synthetic_partitions

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def geometry(rbe, g):
    s = rbe.ScanGeometry()
    s.blocks, s.threads_per_block, s.items_per_thread, s.queue_length = g
    return s


def device_index(rbe, dim, kp, rw, parts):
    return rbe.DeviceIndex(rbe.index_from_arrays(dim, kp, rw, [tuple(p) for p in parts]))


def gpu_search(rbe, dix, qs, geo, n, variant="auto"):
    scores, ids, parts, accs, counts, stats = dix.search_words(qs, geometry(rbe, geo), n, variant)
    out = []
    for q in range(qs.shape[0]):
        c = int(counts[q])
        out.append([(float(scores[q, k]), int(ids[q, k]), int(parts[q, k])) for k in range(c)])
    return out, accs, counts, stats


def check_accs(res, accs, parts_by_id, qp, kp, rw):
    L = qp + kp - 2 if rw else 0
    for q, r in enumerate(res):
        for k, (s, i, p) in enumerate(r):
            mag = parts_by_id[i]
            assert s == math.ldexp(float(accs[q, k]), -L) / float(mag)


def mags_by_id(parts):
    d = {}
    for planes, mags, ids in parts:
        d.update(zip(ids.tolist(), mags.tolist()))
    return d


def test_synthetic_generator_bit_exact(rbe, port):
    for dim, kp, rw, P, N in ((64, 2, True, 1, 5000), (65, 3, True, 3, 4001), (128, 3, False, 2, 3000),
                              (1, 1, True, 1, 100), (200, 4, True, 5, 2222), (512, 6, True, 2, 300)):
        dix = rbe.DeviceIndex.synthetic(dim, kp, rw, N, P, 0xD0C5)
        want = synthetic_partitions(0xD0C5, N, dim, kp, P, rw, port)
        assert dix.total_keywords == N
        for p in range(P):
            planes, mags, ids = dix.download_partition(p)
            wp, wm, wi = want[p]
            assert np.array_equal(planes.reshape(-1), wp.reshape(-1))
            assert np.array_equal(mags, wm), (dim, kp, rw, p)
            assert np.array_equal(ids, wi)


def test_golden_cases(rbe):
    for c in json.load(open(os.path.join(GOLD, "search_cases.json"))):
        parts = synthetic_partitions(c["seed"], c["n_docs"], c["dim"], c["kp"], c["partitions"],
                                     c["residual_weights"])
        qs = gen_queries(c["query_seed"], c["n_queries"], c["dim"], c["qp"])
        dix = device_index(rbe, c["dim"], c["kp"], c["residual_weights"], parts)
        for variant in ("exact", "auto"):
            res, accs, counts, stats = gpu_search(rbe, dix, qs, tuple(c["geometry"]), c["n"], variant)
            assert stats["scored"] == c["n_queries"] * c["n_docs"]
            got = [[[s.hex(), i, p] for s, i, p in r] for r in res]
            assert got == c["results"], (c["name"], variant)
            check_accs(res, accs, mags_by_id(parts), c["qp"], c["kp"], c["residual_weights"])


SWEEP = [
    # N, dim, kp, qp, P, geometry, n, rw
    (4000, 1, 1, 1, 1, (1, 16, 256, 1), 20, True),
    (4000, 63, 2, 2, 2, (2, 32, 32, 2), 30, True),
    (4000, 64, 1, 4, 1, (1, 64, 64, 1), 30, True),
    (4000, 65, 4, 2, 3, (1, 128, 16, 3), 100, True),
    (3000, 128, 3, 3, 8, (1, 8, 64, 1), 50, False),
    (2000, 512, 2, 3, 1, (3, 32, 32, 16), 40, True),
    (3000, 100, 3, 1, 2, (6, 33, 9, 1), 70, True),
    (5000, 128, 3, 3, 1, (1, 256, 256, 1), 1000, True),
    (5000, 128, 4, 4, 1, (1, 256, 256, 1), 5000, True),
    (3000, 64, 2, 2, 1, (1, 1, 3000, 3000), 3000, True),   # lossless single thread
    (6000, 96, 3, 2, 2, (1, 128, 32, 1), 9000, True),      # n > survivors
]


@pytest.mark.parametrize("case", SWEEP)
def test_matches_reference(rbe, port, case):
    N, dim, kp, qp, P, geo, n, rw = case
    ref = Ref()
    parts = synthetic_partitions(11, N, dim, kp, P, rw, port)
    ri = ref.index(dim, kp, rw, parts)
    qs = gen_queries(13, 4, dim, qp)
    want, scored = ri.search(qs, geo, n)
    dix = device_index(rbe, dim, kp, rw, parts)
    for variant in ("exact", "auto"):
        got, accs, counts, stats = gpu_search(rbe, dix, qs, geo, n, variant)
        assert stats["scored"] == scored == 4 * N
        assert got == want, (case, variant)
        check_accs(got, accs, mags_by_id(parts), qp, kp, rw)


def test_tie_heavy(rbe, port):
    """Many identical docs: ties broken by lower slot inside a logical thread
    (search.cpp:39) and by lower id across threads (search.cpp:50-53)."""
    ref = Ref()
    rng = np.random.default_rng(3)
    dim, kp, qp, N = 64, 2, 2, 6000
    patterns = rng.integers(0, 2 ** 63, size=(8, kp), dtype=np.uint64)
    pick = rng.integers(0, 8, N)
    words = patterns[pick]  # [N][kp]
    ids = rng.permutation(N * 3)[:N].astype(np.uint64)
    for P, geo, n in ((1, (1, 32, 256, 1), 200), (3, (1, 16, 128, 2), 500), (2, (2, 64, 32, 4), 1000)):
        parts = []
        for p in range(P):
            sel = np.arange(p, N, P)
            planes = np.ascontiguousarray(words[sel].T)  # [kp][count]
            mags = port.magnitudes(planes, len(sel), dim, kp, True)
            parts.append((planes, mags, ids[sel]))
        ri = ref.index(dim, kp, True, parts)
        qs = gen_queries(5, 3, dim, qp)
        want, _ = ri.search(qs, geo, n)
        dix = device_index(rbe, dim, kp, True, parts)
        for variant in ("exact", "auto"):
            got, _, _, _ = gpu_search(rbe, dix, qs, geo, n, variant)
            assert got == want, (P, geo, variant)


def test_drop_in_search_and_errors(rbe):
    ref = Ref()
    parts = synthetic_partitions(21, 3000, 64, 2, 2, True)
    kix = rbe.index_from_arrays(64, 2, True, parts)
    qs = gen_queries(22, 2, 64, 2)
    q_emb = rbe.make_embedding([rbe.pack([1 if (int(qs[0, s, 0]) >> b) & 1 else -1 for b in range(64)])
                                for s in range(2)])
    g = geometry(rbe, (1, 64, 64, 1))
    got = rbe.search(q_emb, kix, g, 25)
    want, _ = ref.index(64, 2, True, parts).search(qs[:1], (1, 64, 64, 1), 25)
    assert got == want[0]
    batch = rbe.search_batch([q_emb, q_emb], kix, g, 25)
    assert batch[0] == batch[1] == got
    with pytest.raises(ValueError, match="queue_length must be positive"):
        rbe.search(q_emb, kix, geometry(rbe, (1, 64, 64, 0)), 5)
    with pytest.raises(ValueError, match="geometry does not cover partition"):
        rbe.search(q_emb, kix, geometry(rbe, (1, 4, 4, 1)), 5)
    with pytest.raises(ValueError, match="query dimension mismatch"):
        rbe.search(rbe.make_embedding([rbe.pack([1, -1])]), kix, g, 5)
    assert rbe.search(q_emb, kix, g, 0) == []
    many = rbe.make_embedding([rbe.pack([1] * 64)] * 33)
    with pytest.raises(ValueError, match="too many planes"):
        rbe.search(many, kix, g, 5)
    bad = list(parts[0])
    bad[1] = bad[1].copy()
    bad[1][5] = 0.0
    with pytest.raises(ValueError, match="magnitudes must be finite"):
        rbe.DeviceIndex(rbe.index_from_arrays(64, 2, True, [tuple(bad)]))


def test_upload_roundtrip(rbe, port):
    parts = synthetic_partitions(31, 5000, 130, 3, 3, True, port)
    dix = device_index(rbe, 130, 3, True, parts)
    for p in range(3):
        planes, mags, ids = dix.download_partition(p)
        assert np.array_equal(planes.reshape(-1), parts[p][0].reshape(-1))
        assert np.array_equal(mags, parts[p][1]) and np.array_equal(ids, parts[p][2])


def test_config1_full_scale(rbe):
    """BASELINE config 1: 1M docs, 64-dim, 2+2 planes, 16 queries, k=100, P=1,
    default geometry with auto blocks -- GPU == compiled reference for all 16."""
    ref = Ref()
    N, dim, kp, qp, Q, n = 1_000_000, 64, 2, 2, 16, 100
    blocks = -(-N // 65536)
    geo = (blocks, 256, 256, 1)
    dix = rbe.DeviceIndex.synthetic(dim, kp, True, N, 1, 0xD0C5)
    parts = [dix.download_partition(0)]
    qs = gen_queries(0x0E1, Q, dim, qp)
    want, scored = ref.index(dim, kp, True, parts).search(qs, geo, n, threads=8)
    for variant in ("exact", "auto"):
        got, accs, counts, stats = gpu_search(rbe, dix, qs, geo, n, variant)
        assert stats["scored"] == scored == Q * N
        assert got == want, variant


def test_tensor_matches_exact_at_scale(rbe):
    """Config-2 shape at reduced N (8M docs, 128-dim, 3+3 planes, k=1000):
    the tensor-core variant equals the exact CUDA-core variant bit for bit."""
    N = 8_000_000
    blocks = -(-N // 65536)
    geo = (blocks, 256, 256, 1)
    dix = rbe.DeviceIndex.synthetic(128, 3, True, N, 1, 0xD0C5)
    qs = gen_queries(0x0E1, 8, 128, 3)
    a = gpu_search(rbe, dix, qs, geo, 1000, "exact")
    b = gpu_search(rbe, dix, qs, geo, 1000, "auto")
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1])


TENSOR_SWEEP = [
    # N, dim, kp, qp, P, geometry, n, rw, Q
    (20000, 64, 2, 2, 1, (1, 256, 256, 1), 100, True, 4),
    (30000, 128, 3, 3, 1, (1, 256, 256, 1), 1000, True, 4),
    (30000, 128, 3, 3, 3, (1, 128, 128, 1), 300, True, 3),
    (20000, 65, 4, 2, 2, (2, 256, 64, 1), 200, True, 5),
    (20000, 200, 1, 6, 1, (1, 384, 64, 1), 50, True, 2),
    (20000, 100, 3, 2, 2, (1, 256, 64, 1), 100, False, 4),
    (20000, 128, 5, 3, 1, (1, 256, 128, 1), 100, True, 3),
    (40000, 128, 3, 3, 1, (1, 256, 256, 1), 5000, True, 2),   # n > threads: no bound, every pair rescored
    (30000, 64, 2, 2, 1, (1, 256, 256, 1), 64, True, 70),     # two 64-query passes
    (30000, 128, 3, 3, 1, (1, 256, 256, 1), 10, True, 1),
]


@pytest.mark.parametrize("case", TENSOR_SWEEP)
def test_tensor_matches_reference(rbe, port, case):
    N, dim, kp, qp, P, geo, n, rw, Q = case
    ref = Ref()
    parts = synthetic_partitions(17, N, dim, kp, P, rw, port)
    ri = ref.index(dim, kp, rw, parts)
    qs = gen_queries(19, Q, dim, qp)
    want, scored = ri.search(qs, geo, n, threads=8)
    dix = device_index(rbe, dim, kp, rw, parts)
    got, accs, counts, stats = gpu_search(rbe, dix, qs, geo, n, "tensor")
    assert stats["variant"] == "tensor"
    assert stats["scored"] == scored == Q * N
    assert got == want, case
    check_accs(got, accs, mags_by_id(parts), qp, kp, rw)


SMALL_BATCH = [
    # N, kp, qp, P, geometry, n, rw, Q -- dim 128, 256-wide strips: <= 2 live queries take the
    # CUDA-core scoring body of the tensor scan (kCCMaxQ, scan_tensor.cu)
    (200000, 3, 3, 1, (4, 256, 256, 1), 100, True, 1),
    (200000, 3, 3, 1, (4, 256, 256, 1), 1000, True, 2),
    (150000, 1, 3, 3, (2, 256, 128, 1), 50, True, 2),
    (150000, 2, 2, 2, (1, 512, 256, 1), 200, True, 1),
    (150000, 4, 3, 1, (3, 256, 256, 1), 100, False, 2),
    (100000, 7, 2, 1, (2, 256, 256, 1), 300, True, 1),
    (100000, 3, 3, 2, (2, 256, 256, 256), 500, True, 2),   # lossless (queue_length >= items_per_thread)
]


@pytest.mark.parametrize("case", SMALL_BATCH)
def test_small_batch_matches_reference(rbe, port, case):
    """Batches of one or two queries (the latency path): the CUDA-core scoring body computes the
    same F as the tensor core, so results equal the reference bit for bit."""
    N, kp, qp, P, geo, n, rw, Q = case
    ref = Ref()
    parts = synthetic_partitions(31, N, 128, kp, P, rw, port)
    qs = gen_queries(37, Q, 128, qp)
    want, scored = ref.index(128, kp, rw, parts).search(qs, geo, n, threads=8)
    dix = device_index(rbe, 128, kp, rw, parts)
    got, accs, counts, stats = gpu_search(rbe, dix, qs, geo, n, "tensor")
    assert stats["scored"] == scored == Q * N
    assert got == want, case
    check_accs(got, accs, mags_by_id(parts), qp, kp, rw)


def test_small_batch_matches_exact_at_scale(rbe):
    """8M docs, 1 and 2 queries: the CUDA-core body of the tensor scan == the exact kernel."""
    N = 8_000_000
    geo = (-(-N // 65536), 256, 256, 1)
    dix = rbe.DeviceIndex.synthetic(128, 3, True, N, 1, 0xD0C5)
    for Q in (1, 2):
        qs = gen_queries(0x0E1 + Q, Q, 128, 3)
        a = gpu_search(rbe, dix, qs, geo, 1000, "exact")
        b = gpu_search(rbe, dix, qs, geo, 1000, "auto")
        assert a[0] == b[0]
        assert np.array_equal(a[1], b[1])


def test_tensor_state_table_overflow(rbe, port):
    """n above the survivor count (theta stays -inf): every (query, logical thread)
    state entry of a strip is set -- 40 queries x 256 threads > the 4096-entry
    touched list, so the strip end scans the whole table.  Tensor == reference."""
    N, dim, kp, qp, geo, n, Q = 40000, 128, 3, 3, (1, 256, 256, 1), 60000, 40
    ref = Ref()
    parts = synthetic_partitions(17, N, dim, kp, 1, True, port)
    qs = gen_queries(19, Q, dim, qp)
    want, scored = ref.index(dim, kp, True, parts).search(qs, geo, n)
    dix = device_index(rbe, dim, kp, True, parts)
    got, accs, counts, stats = gpu_search(rbe, dix, qs, geo, n, "tensor")
    assert stats["variant"] == "tensor"
    assert got == want


def test_search_words_out_buffers(rbe, port):
    """search_words(out=...) writes into the caller's arrays (reused across batches) and
    returns them; results equal the freshly allocated ones."""
    N, dim, kp, qp, geo, n = 20000, 128, 3, 3, (1, 256, 256, 1), 200
    parts = synthetic_partitions(23, N, dim, kp, 1, True, port)
    dix = device_index(rbe, dim, kp, True, parts)
    qs = gen_queries(29, 5, dim, qp)
    g = geometry(rbe, geo)
    want = dix.search_words(qs, g, n, "auto")
    out = (np.full((5, n), 7.0), np.zeros((5, n), np.uint64), np.zeros((5, n), np.uint32),
           np.zeros((5, n), np.int64), np.zeros(5, np.uint64))
    for _ in range(2):
        got = dix.search_words(qs, g, n, "auto", 0, False, out)
        for a, b, o in zip(got[:5], want[:5], out):
            assert a is o
            assert np.array_equal(a, b)
    # page-locked out arrays: results are DMA'd straight into them
    pe = rbe.pinned_empty
    pinned = (pe((5, n), np.float64), pe((5, n), np.uint64), pe((5, n), np.uint32), pe((5, n), np.int64),
              pe(5, np.uint64))
    for arr in pinned:
        arr.fill(3)
    got = dix.search_words(qs, g, n, "auto", 0, False, pinned)
    for a, b in zip(got[:5], want[:5]):
        assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        dix.search_words(qs, g, n, "auto", 0, False, out[:4])
    with pytest.raises(ValueError):
        dix.search_words(qs, g, n, "auto", 0, False, (out[0].astype(np.float32),) + out[1:])
