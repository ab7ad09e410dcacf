"""RBEI v1 ingest straight into HBM: DeviceIndex.from_rbei must hold
exactly what the reference's load_index (src/index.cpp:170-208) reads from the same file,
and answer searches identically; the header reader raises the reference's errors."""
import struct

import numpy as np
import pytest

from oracle.oracle import gen_queries, synthetic_partitions
from tests.helpers import HAS_GPU


def _write_ref_file(rbe, ref, tmp_path, dim, kp, rw, P, N, name="x.rbei"):
    from oracle.oracle import Port

    parts = synthetic_partitions(0xD0C5, N, dim, kp, P, rw, Port())
    path = tmp_path / name
    ref.index(dim, kp, rw, [tuple(p) for p in parts]).save(path)  # the reference's own save_index
    return str(path), parts


def test_rbei_header_reads_reference_file(rbe, ref, tmp_path):
    path, parts = _write_ref_file(rbe, ref, tmp_path, 65, 3, True, 3, 1001)
    h = rbe.rbei_header(path)
    assert (h["dim"], h["keyword_planes"], h["residual_weights"]) == (65, 3, True)
    assert h["counts"] == [len(p[2]) for p in parts]


def test_rbei_header_errors(rbe, ref, tmp_path):
    path, _ = _write_ref_file(rbe, ref, tmp_path, 64, 2, True, 2, 100)
    data = open(path, "rb").read()
    with pytest.raises(RuntimeError, match="cannot open index"):
        rbe.rbei_header(str(tmp_path / "missing.rbei"))
    (tmp_path / "bad").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(RuntimeError, match="not an RBEI index file"):
        rbe.rbei_header(str(tmp_path / "bad"))
    (tmp_path / "v2").write_bytes(data[:4] + struct.pack("<I", 2) + data[8:])
    with pytest.raises(RuntimeError, match="unsupported index version"):
        rbe.rbei_header(str(tmp_path / "v2"))
    (tmp_path / "trunc").write_bytes(data[:-1])
    with pytest.raises(RuntimeError, match="truncated index file"):
        rbe.rbei_header(str(tmp_path / "trunc"))


@pytest.mark.skipif(HAS_GPU, reason="CPU-only behaviour")
def test_from_rbei_without_gpu_fails_loudly(rbe, ref, tmp_path):
    path, _ = _write_ref_file(rbe, ref, tmp_path, 64, 2, True, 1, 50)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rbe.DeviceIndex.from_rbei(path)


def _geometry(rbe, count):
    g = rbe.ScanGeometry()
    g.blocks = max(1, -(-count // 65536))
    return g


@pytest.mark.gpu
@pytest.mark.parametrize("dim,kp,rw,P,N,devices", [
    (128, 3, True, 3, 200_003, [0]),
    (128, 3, True, 8, 100_000, [0, 0]),
    (65, 2, True, 4, 3, [0]),          # partitions with no documents
    (200, 4, False, 2, 5000, [0, 0, 0]),
])
def test_from_rbei_equals_load_index(rbe, ref, tmp_path, dim, kp, rw, P, N, devices):
    path, parts = _write_ref_file(rbe, ref, tmp_path, dim, kp, rw, P, N)
    dix = rbe.DeviceIndex.from_rbei(path, devices)
    st = dix.load_stats
    assert st["file_bytes"] == sum(len(i) * (kp * ((dim + 63) // 64) * 8 + 12) for _, _, i in parts)
    host = rbe.load_index(path)
    assert dix.total_keywords == N and dix.partition_count == P
    for p in range(P):
        got = dix.download_partition(p)
        want = host.partition_arrays(p)
        for x, y in zip(got, want):
            assert np.array_equal(np.asarray(x).reshape(-1), np.asarray(y).reshape(-1)), p
    if N >= 100:
        qs = gen_queries(0x0E1, 8, dim, kp)
        g = _geometry(rbe, max(len(i) for _, _, i in parts))
        a = dix.search_words(qs, g, 100)
        b = rbe.DeviceIndex(host, devices).search_words(qs, g, 100)
        for x, y in zip(a[:5], b[:5]):
            assert np.array_equal(x, y)


@pytest.mark.gpu
def test_from_rbei_rejects_zero_magnitude(rbe, ref, tmp_path):
    path, parts = _write_ref_file(rbe, ref, tmp_path, 64, 2, True, 1, 1000)
    data = bytearray(open(path, "rb").read())
    mags_off = 4 + 5 * 4 + 8 + 1000 * 2 * 8  # header, one count, 2 planes x 1000 words
    data[mags_off + 4 * 17:mags_off + 4 * 18] = struct.pack("<f", 0.0)
    (tmp_path / "zero.rbei").write_bytes(bytes(data))
    with pytest.raises(ValueError, match="magnitudes must be finite and > 0"):
        rbe.DeviceIndex.from_rbei(str(tmp_path / "zero.rbei"))
    with pytest.raises(RuntimeError, match="truncated index file"):
        (tmp_path / "t.rbei").write_bytes(bytes(data[:-8]))
        rbe.DeviceIndex.from_rbei(str(tmp_path / "t.rbei"))
