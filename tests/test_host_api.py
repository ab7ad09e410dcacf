"""Host side of the drop-in surface (paper_1802_06466_b200._core) against the
compiled reference: same values, same exception types/messages, RBEI byte
compatibility.  CPU only; search itself is GPU-only (no CPU fallback)."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import synthetic_partitions
from tests.helpers import HAS_GPU

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rand_pm(rng, n):
    return [int(v) for v in rng.choice([-1, 1], n)]


def test_pack_unpack_dot(rbe, ref):
    rng = np.random.default_rng(1)
    for dim in (1, 63, 64, 65, 128, 512):
        for _ in range(20):
            a, b = rand_pm(rng, dim), rand_pm(rng, dim)
            va, vb = rbe.pack(a), rbe.pack(b)
            assert va.words == [int(w) for w in ref.pack(a)[0]]
            assert rbe.unpack(va) == a
            assert rbe.binary_dot(va, vb) == sum(x * y for x, y in zip(a, b))
    with pytest.raises(ValueError, match="pack: empty input"):
        rbe.pack([])
    with pytest.raises(ValueError, match="pack: values must be -1 or \\+1"):
        rbe.pack([1, 0])
    with pytest.raises(ValueError, match="binary_dot: dimension mismatch"):
        rbe.binary_dot(rbe.pack([1]), rbe.pack([1, 1]))


def test_kats(rbe):
    k = json.load(open(os.path.join(GOLD, "spec_kats.json")))
    for c in k["pack"]:
        assert rbe.pack(c["values"]).words == c["words"]
    for c in k["magnitude"]:
        e = rbe.make_embedding([rbe.pack(p) for p in c["planes"]], c["rw"])
        assert e.magnitude == c["magnitude"]
        assert rbe.refined_vector(e, c["rw"]) == c["refined"]
    for c in k["thread_assignment"]:
        g = rbe.ScanGeometry()
        g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length = c["geometry"]
        assert rbe.thread_assignment(g, c["count"], c["block"], c["thread"]) == c["items"]
    cfg = rbe.SimilarityConfig()
    cfg.query_planes = cfg.keyword_planes = 1
    cfg.normalize_query = False
    c = k["rbe_score"][0]
    assert rbe.rbe_score(rbe.make_embedding([rbe.pack(c["q"])]), rbe.make_embedding([rbe.pack(c["k"])]), cfg) == 0.0
    m = k["memory"]
    e = rbe.make_embedding([rbe.pack([1] * 64), rbe.pack([-1] * 64)])
    idx = rbe.build_index([(i, e) for i in range(1000)])
    assert idx.plane_bytes_per_keyword == m["bytes_per_keyword"]
    assert idx.plane_payload_bytes == 1000 * m["bytes_per_keyword"]


def test_magnitude_and_score_bit_exact(rbe, ref):
    rng = np.random.default_rng(2)
    for dim in (3, 64, 100, 128):
        for np_ in (1, 2, 3, 4):
            for rw in (True, False):
                planes = [rbe.pack(rand_pm(rng, dim)) for _ in range(np_)]
                e = rbe.make_embedding(planes, rw)
                w = np.array([p.words for p in planes], np.uint64)
                assert e.magnitude == ref.magnitude(w, np_, dim, rw)
                q = [rbe.pack(rand_pm(rng, dim)) for _ in range(2)]
                qe = rbe.make_embedding(q, rw)
                cfg = rbe.SimilarityConfig()
                cfg.query_planes, cfg.keyword_planes, cfg.residual_weights = 2, np_, rw
                for norm in (True, False):
                    cfg.normalize_query = norm
                    qw = np.array([p.words for p in q], np.uint64)
                    try:
                        want = ref.rbe_score(qw, 2, w, np_, dim, rw, norm)
                    except ValueError as ex:
                        with pytest.raises(ValueError, match=str(ex)):
                            rbe.rbe_score(qe, e, cfg)
                        continue
                    assert rbe.rbe_score(qe, e, cfg) == want


def _embeddings(rbe, n, dim, kp, seed, rw=True):
    rng = np.random.default_rng(seed)
    return [(int(i * 7 + 3), rbe.make_embedding([rbe.pack(rand_pm(rng, dim)) for _ in range(kp)], rw))
            for i in range(n)]


def test_build_index_matches_reference(rbe, ref):
    for dim, kp, P, rw in ((64, 2, 3, True), (65, 3, 1, False), (130, 1, 4, True)):
        embs = _embeddings(rbe, 50, dim, kp, dim, rw)
        ours = rbe.build_index(embs, P, rw)
        words = np.array([[p.words for p in e.planes] for _, e in embs], np.uint64)
        ids = np.array([i for i, _ in embs], np.uint64)
        theirs = ref.build_index(dim, kp, rw, P, words, ids)
        assert ours.total_keywords == 50 and ours.partition_count == P
        for p in range(P):
            a = ours.partition_arrays(p)
            b = theirs.partition(p)
            for x, y in zip(a, b):
                assert np.array_equal(np.asarray(x).reshape(-1), np.asarray(y).reshape(-1))


def test_builder_errors(rbe):
    e1 = rbe.make_embedding([rbe.pack([1, -1])])
    e2 = rbe.make_embedding([rbe.pack([1, -1, 1])])
    with pytest.raises(ValueError, match="need at least one partition"):
        rbe.build_index([(1, e1)], 0)
    with pytest.raises(ValueError, match="inconsistent dim or plane count"):
        rbe.build_index([(1, e1), (2, e2)])
    with pytest.raises(ValueError, match="duplicate keyword id"):
        rbe.build_index([(1, e1), (1, e1)])


def test_rbei_byte_compatible(rbe, ref, tmp_path):
    embs = _embeddings(rbe, 40, 65, 3, 9)
    ours = rbe.build_index(embs, 3, True)
    words = np.array([[p.words for p in e.planes] for _, e in embs], np.uint64)
    ids = np.array([i for i, _ in embs], np.uint64)
    theirs = ref.build_index(65, 3, True, 3, words, ids)
    rbe.save_index(ours, str(tmp_path / "ours.rbei"))
    theirs.save(tmp_path / "theirs.rbei")
    assert (tmp_path / "ours.rbei").read_bytes() == (tmp_path / "theirs.rbei").read_bytes()
    back = rbe.load_index(str(tmp_path / "theirs.rbei"))
    for p in range(3):
        for x, y in zip(back.partition_arrays(p), ours.partition_arrays(p)):
            assert np.array_equal(x, y)
    with pytest.raises(RuntimeError, match="not an RBEI index file"):
        (tmp_path / "bad").write_bytes(b"XXXX")
        rbe.load_index(str(tmp_path / "bad"))
    with pytest.raises(RuntimeError, match="truncated index file"):
        (tmp_path / "trunc").write_bytes((tmp_path / "ours.rbei").read_bytes()[:100])
        rbe.load_index(str(tmp_path / "trunc"))


def test_search_arg_errors_without_gpu(rbe):
    embs = _embeddings(rbe, 20, 64, 2, 3)
    idx = rbe.build_index(embs)
    q = embs[0][1]
    g = rbe.ScanGeometry()
    with pytest.raises(ValueError, match="query dimension mismatch"):
        rbe.search(rbe.make_embedding([rbe.pack([1, 1])]), idx, g, 5)
    empty = rbe.build_index([], 2)
    with pytest.raises(ValueError, match="search: empty index"):
        rbe.search(q, empty, g, 5)
    with pytest.raises(ValueError, match="thread_assignment: block or thread out of range"):
        rbe.thread_assignment(g, 10, 1, 0)


@pytest.mark.skipif(HAS_GPU, reason="CPU-only behaviour")
def test_search_fails_loudly_without_gpu(rbe):
    embs = _embeddings(rbe, 20, 64, 2, 4)
    idx = rbe.build_index(embs)
    with pytest.raises(RuntimeError, match="no usable CUDA device"):
        rbe.search(embs[0][1], idx, rbe.ScanGeometry(), 5)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rbe.DeviceIndex.synthetic(64, 2, True, 1000)
