"""RBEE bulk embeddings -> index build on the device: DeviceIndex.build_rbee
must hold what the reference's `rbe build` (EmbeddingReader + IndexBuilder,
src/embedding_io.cpp:48-95, src/index.cpp:36-78) builds from the same file -- round-robin
partitions, record magnitudes kept when > 0 and recomputed by make_embedding otherwise -- and
raise the reference's errors."""
import struct

import numpy as np
import pytest

from tests.helpers import HAS_GPU


def write_rbee(path, dim, kp, rw, ids, words, mags):
    """RBEE v1 (embedding_io.cpp:15-45): header, then (u64 id, [kp][wpp] u64 words, f32 magnitude)."""
    wpp = (dim + 63) // 64
    rec = np.zeros(len(ids), dtype=[("id", "<u8"), ("w", "<u8", (kp * wpp,)), ("m", "<f4")])
    rec["id"] = ids
    rec["w"] = words.reshape(len(ids), kp * wpp)
    rec["m"] = mags
    with open(path, "wb") as f:
        f.write(b"RBEE" + struct.pack("<4I", 1, dim, kp, 1 if rw else 0))
        f.write(rec.tobytes())


def corpus(dim, kp, n, seed):
    rng = np.random.default_rng(seed)
    wpp = (dim + 63) // 64
    words = rng.integers(0, 2**63, size=(n, kp, wpp), dtype=np.uint64) * 2 + rng.integers(0, 2, size=(n, kp, wpp),
                                                                                          dtype=np.uint64)
    if dim % 64:
        words[:, :, -1] &= np.uint64((1 << (dim % 64)) - 1)
    ids = rng.permutation(np.arange(10 * n, dtype=np.uint64))[:n] + np.uint64(7)
    mags = rng.uniform(0.5, 3.0, size=n).astype(np.float32)
    mags[::3] = 0.0  # recomputed by the builder
    mags[1::7] = np.nan  # not > 0 either: recomputed
    return ids, words, mags


def expected(ref, dim, kp, rw, P, ids, words, mags):
    """IndexBuilder::add, record k -> partition k % P, slot k // P."""
    n = len(ids)
    out = []
    for p in range(P):
        sel = np.arange(p, n, P)
        planes = np.ascontiguousarray(words[sel].transpose(1, 0, 2)).reshape(kp, -1)
        m = mags[sel].copy()
        for j, k in enumerate(sel):
            if not (float(m[j]) > 0.0):
                m[j] = np.float32(ref.magnitude(words[k], kp, dim, rw))
        out.append((planes, m, ids[sel]))
    return out


def test_rbee_header(rbe, tmp_path):
    ids, words, mags = corpus(65, 3, 11, 1)
    write_rbee(tmp_path / "e.rbee", 65, 3, True, ids, words, mags)
    h = rbe.rbee_header(str(tmp_path / "e.rbee"))
    assert h == {"dim": 65, "plane_count": 3, "residual_weights": True, "count": 11}
    data = (tmp_path / "e.rbee").read_bytes()
    with pytest.raises(RuntimeError, match="cannot open embeddings file"):
        rbe.rbee_header(str(tmp_path / "missing"))
    (tmp_path / "m").write_bytes(b"RBEX" + data[4:])
    with pytest.raises(RuntimeError, match="not an RBEE embeddings file"):
        rbe.rbee_header(str(tmp_path / "m"))
    (tmp_path / "v").write_bytes(data[:4] + struct.pack("<I", 9) + data[8:])
    with pytest.raises(RuntimeError, match="unsupported embeddings version"):
        rbe.rbee_header(str(tmp_path / "v"))
    (tmp_path / "s").write_bytes(data[:8] + struct.pack("<I", 0) + data[12:])
    with pytest.raises(RuntimeError, match="embeddings file has empty shape"):
        rbe.rbee_header(str(tmp_path / "s"))
    (tmp_path / "t").write_bytes(data[:-3])
    with pytest.raises(RuntimeError, match="embeddings file has truncated records"):
        rbe.rbee_header(str(tmp_path / "t"))


@pytest.mark.skipif(HAS_GPU, reason="CPU-only behaviour")
def test_build_rbee_without_gpu_fails_loudly(rbe, tmp_path):
    ids, words, mags = corpus(64, 2, 5, 2)
    write_rbee(tmp_path / "e.rbee", 64, 2, True, ids, words, mags)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rbe.DeviceIndex.build_rbee(str(tmp_path / "e.rbee"), 2)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,kp,rw,P,n,devices", [
    (128, 3, True, 3, 20_001, [0]),
    (65, 2, True, 4, 1_003, [0, 0]),
    (200, 4, False, 1, 999, [0]),
    (64, 1, True, 5, 3, [0, 0, 0]),
])
def test_build_rbee_matches_index_builder(rbe, ref, tmp_path, dim, kp, rw, P, n, devices):
    ids, words, mags = corpus(dim, kp, n, dim + n)
    path = str(tmp_path / "e.rbee")
    write_rbee(path, dim, kp, rw, ids, words, mags)
    dix = rbe.DeviceIndex.build_rbee(path, P, devices)
    assert dix.total_keywords == n and dix.partition_count == P
    want = expected(ref, dim, kp, rw, P, ids, words, mags)
    for p in range(P):
        got = dix.download_partition(p)
        for x, y in zip(got, want[p]):
            assert np.array_equal(np.asarray(x).reshape(-1), np.asarray(y).reshape(-1)), p
    # the RBEI written from the device equals save_index of the same KeywordIndex
    dix.save_index(str(tmp_path / "dev.rbei"))
    host = rbe.index_from_arrays(dim, kp, rw, [tuple(w) for w in want])
    rbe.save_index(host, str(tmp_path / "host.rbei"))
    assert (tmp_path / "dev.rbei").read_bytes() == (tmp_path / "host.rbei").read_bytes()


@pytest.mark.gpu
def test_build_rbee_equals_reference_builder(rbe, ref, tmp_path):
    """All record magnitudes 0: every magnitude comes from make_embedding, exactly what the
    reference's build_index (its own IndexBuilder) produces from the same words and ids."""
    dim, kp, rw, P, n = 128, 3, True, 8, 40_000
    ids, words, _ = corpus(dim, kp, n, 5)
    write_rbee(tmp_path / "e.rbee", dim, kp, rw, ids, words, np.zeros(n, np.float32))
    dix = rbe.DeviceIndex.build_rbee(str(tmp_path / "e.rbee"), P)
    theirs = ref.build_index(dim, kp, rw, P, words, ids)
    theirs.save(tmp_path / "ref.rbei")
    dix.save_index(str(tmp_path / "dev.rbei"))
    assert (tmp_path / "dev.rbei").read_bytes() == (tmp_path / "ref.rbei").read_bytes()


@pytest.mark.gpu
def test_build_rbee_errors(rbe, tmp_path):
    ids, words, mags = corpus(64, 2, 100, 9)
    dup = ids.copy()
    dup[77] = dup[3]
    write_rbee(tmp_path / "d.rbee", 64, 2, True, dup, words, mags)
    with pytest.raises(ValueError, match="duplicate keyword id"):
        rbe.DeviceIndex.build_rbee(str(tmp_path / "d.rbee"), 3)
    with pytest.raises(ValueError, match="duplicate keyword id"):  # the two copies on different devices
        rbe.DeviceIndex.build_rbee(str(tmp_path / "d.rbee"), 2, [0, 0])
    with pytest.raises(ValueError, match="need at least one partition"):
        rbe.DeviceIndex.build_rbee(str(tmp_path / "d.rbee"), 0)
    # unweighted, complementary planes: every refined value is 0 -> zero magnitude
    z = words.copy()
    z[:, 1, :] = ~z[:, 0, :]
    m = mags.copy()
    m[10] = 0.0
    write_rbee(tmp_path / "z.rbee", 64, 2, False, ids, z, m)
    with pytest.raises(ValueError, match="keyword has zero magnitude"):
        rbe.DeviceIndex.build_rbee(str(tmp_path / "z.rbee"), 1)
