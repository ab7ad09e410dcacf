"""GPU tests of the device-resident entry points the bench and the multi-GPU path
use (rbe_cuda_search_device, rbe_cuda_merge_device, rbe_cuda_search_multi), the
reference's local_select / global_select on the device, stream ordering, the
sticky internal-consistency flag, and steady-state memory (no per-call
allocations)."""
import numpy as np
import pytest

from oracle.oracle import gen_queries, synthetic_partitions

pytestmark = pytest.mark.gpu

REC = np.dtype([("score", "<f8"), ("id", "<u8"), ("acc", "<i8"), ("partition", "<u4"), ("valid", "<u4")])


def geometry(rbe, g):
    s = rbe.ScanGeometry()
    s.blocks, s.threads_per_block, s.items_per_thread, s.queue_length = g
    return s


def decode(buf, Q, n):
    rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=REC).reshape(Q, n)
    return [[(float(r["score"]), int(r["id"]), int(r["partition"]), int(r["acc"])) for r in row if r["valid"]]
            for row in rec]


def words_result(dix, qs, g, n, variant="auto"):
    scores, ids, parts, accs, counts, _ = dix.search_words(qs, g, n, variant)
    return [[(float(scores[q, k]), int(ids[q, k]), int(parts[q, k]), int(accs[q, k])) for k in range(int(counts[q]))]
            for q in range(qs.shape[0])]


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def test_search_device_and_merge_device(rbe, torch):
    """Two single-partition indexes (ranks 0 and 1 of a 2-way split) searched with
    search_device, merged with merge_device == the 2-partition index searched whole."""
    N, dim, kp, qp, Q, n = 2_000_000, 128, 3, 3, 16, 500
    g = geometry(rbe, (-(-N // 2 // 65536), 256, 256, 1))
    qs = gen_queries(41, Q, dim, qp)
    whole = rbe.DeviceIndex.synthetic(dim, kp, True, N, 2, 0xD0C5)
    want = words_result(whole, qs, g, n)
    shards = [rbe.DeviceIndex.synthetic(dim, kp, True, N, 2, 0xD0C5, [0], r, 2) for r in range(2)]
    d_words = torch.from_numpy(qs.view(np.int64).copy()).cuda()
    stream = torch.cuda.Stream()
    outs = [torch.empty(Q * n * rbe.RESULT_RECORD_BYTES, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for with_stats in (True, False):
        for r in range(2):
            st = rbe.search_device(shards[r].handle(0), d_words.data_ptr(), Q, qp, g, n, outs[r].data_ptr(),
                                   stream.cuda_stream, "auto", with_stats)
            if with_stats:
                assert st["scored"] == Q * N // 2 and st["variant"] == "tensor"
        cat = torch.cat(outs)
        merged = torch.empty_like(outs[0])
        rbe.merge_device(0, cat.data_ptr(), 2, Q, n, merged.data_ptr(), stream.cuda_stream)
        stream.synchronize()
        assert decode(merged, Q, n) == want
        # each shard's own list equals its partition's results
        for r in range(2):
            assert all(e[2] == r for row in decode(outs[r], Q, n) for e in row)


def test_multi_handle_search_on_one_gpu(rbe, port):
    """DeviceIndex(k, devices=[0, 0]): two handles on one GPU, each scanning its
    partitions concurrently, lists peer-copied and merged on the first -- identical to
    the single-handle index; a handle with no partitions (P=1 on two devices) is skipped."""
    dim, kp, qp, n = 128, 3, 3, 300
    qs = gen_queries(43, 6, dim, qp)
    for P, N in ((4, 400_000), (3, 300_001), (1, 200_000)):
        kix = rbe.index_from_arrays(dim, kp, True, [tuple(p) for p in synthetic_partitions(44, N, dim, kp, P, True, port)])
        g = geometry(rbe, (-(-(-(-N // P)) // 65536), 256, 256, 1))
        single = rbe.DeviceIndex(kix, [0])
        multi = rbe.DeviceIndex(kix, [0, 0])
        assert multi.devices == [0, 0]
        for variant in ("auto", "exact"):
            a = single.search_words(qs, g, n, variant)
            b = multi.search_words(qs, g, n, variant)
            for x, y in zip(a[:5], b[:5]):
                assert np.array_equal(x, y), (P, variant)
            assert b[5]["scored"] == 6 * N


def test_device_local_and_global_select(rbe, ref, port):
    """local_select (per-thread lists incl. queue_length > 1 and ragged tails) and
    global_select on the device == the reference's own functions."""
    dim, kp, qp = 96, 3, 2
    parts = synthetic_partitions(45, 50_003, dim, kp, 3, True, port)
    kix = rbe.index_from_arrays(dim, kp, True, [tuple(p) for p in parts])
    dix = rbe.DeviceIndex(kix, [0])
    ri = ref.index(dim, kp, True, parts)
    qs = gen_queries(46, 3, dim, qp)
    for geo in ((2, 128, 80, 1), (1, 256, 70, 3), (3, 40, 200, 8), (1, 1, 20000, 5)):
        for p in range(3):
            for q in range(3):
                s, z, c, scored = rbe.local_select_arrays(dix, qs[q], p, geometry(rbe, geo))
                ws, wz, wc, wscored = ri.local_select(qs[q], p, geo)
                assert scored == wscored == len(parts[p][2])
                assert np.array_equal(c, wc)
                mask = np.arange(s.shape[1])[None, :] < c[:, None]
                assert np.array_equal(s[mask], ws[mask]) and np.array_equal(z[mask], wz[mask]), (geo, p, q)
                # global_select of the same candidates on the device
                n = 150
                sel_s, sel_i = rbe.select_topn(s[mask], parts[p][2][z[mask].astype(np.int64)], p, n)
                want, _ = ri.partition_select(qs[q], p, geo, n)
                assert list(zip(sel_s.tolist(), sel_i.tolist())) == [(a, b) for a, b, _ in want]
    # the drop-in list-of-lists form
    emb = rbe.make_embedding([rbe.pack([1 if (int(qs[0, s, w]) >> b) & 1 else -1
                                        for w in range(2) for b in range(64)][:dim]) for s in range(qp)])
    lists = rbe.local_select(emb, kix, 1, geometry(rbe, (1, 256, 70, 3)))
    ws, wz, wc, _ = ri.local_select(qs[0], 1, (1, 256, 70, 3))
    assert [len(l) for l in lists] == wc.tolist()
    assert lists[7] == [(float(ws[7, k]), int(wz[7, k])) for k in range(int(wc[7]))]


def test_streams_are_ordered(rbe, torch):
    """Back-to-back asynchronous batches of one index on two different streams share its
    scratch safely (the second waits for the first): every batch's result is intact."""
    N, dim, kp, qp, Q, n = 3_000_000, 128, 3, 3, 8, 200
    g = geometry(rbe, (-(-N // 65536), 256, 256, 1))
    dix = rbe.DeviceIndex.synthetic(dim, kp, True, N, 1, 0xD0C5)
    qa, qb = gen_queries(47, Q, dim, qp), gen_queries(48, Q, dim, qp)
    want_a, want_b = words_result(dix, qa, g, n), words_result(dix, qb, g, n)
    da = torch.from_numpy(qa.view(np.int64).copy()).cuda()
    db = torch.from_numpy(qb.view(np.int64).copy()).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for k in range(6):
        o = torch.empty(Q * n * rbe.RESULT_RECORD_BYTES, dtype=torch.uint8, device="cuda")
        st, d = (s1, da) if k % 2 == 0 else (s2, db)
        o.record_stream(st)
        rbe.search_device(dix.handle(0), d.data_ptr(), Q, qp, g, n, o.data_ptr(), st.cuda_stream, "auto", False)
        outs.append(o)
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        got = decode(o, Q, n)
        assert got == (want_a if k % 2 == 0 else want_b), k


def test_sticky_error_surfaces_on_async_path(rbe, torch):
    """An accumulator-recovery failure flagged during an asynchronous batch is not lost:
    the next synchronous call on the index raises, once, and the index stays usable."""
    N, dim, kp, qp, Q, n = 500_000, 128, 3, 3, 4, 100
    g = geometry(rbe, (-(-N // 65536), 256, 256, 1))
    dix = rbe.DeviceIndex.synthetic(dim, kp, True, N, 1, 0xD0C5)
    qs = gen_queries(49, Q, dim, qp)
    d = torch.from_numpy(qs.view(np.int64).copy()).cuda()
    o = torch.empty(Q * n * rbe.RESULT_RECORD_BYTES, dtype=torch.uint8, device="cuda")
    h = dix.handle(0)
    rbe.index_check(h)  # clean
    rbe.index_inject_error(h)
    rbe.search_device(h, d.data_ptr(), Q, qp, g, n, o.data_ptr(), 0, "auto", False)  # async: no report yet
    with pytest.raises(RuntimeError, match="accumulator recovery failed"):
        rbe.last_batch_ms(h)
    rbe.last_batch_ms(h)  # reported once, then cleared
    rbe.index_inject_error(h)
    with pytest.raises(RuntimeError, match="accumulator recovery failed"):
        dix.search_words(qs, g, n, "auto", 0, False)  # rbe_cuda_search reads it with the results
    rbe.index_inject_error(h)
    with pytest.raises(RuntimeError, match="accumulator recovery failed"):
        rbe.search_device(h, d.data_ptr(), Q, qp, g, n, o.data_ptr(), 0, "auto", True)
    assert words_result(dix, qs, g, n) == words_result(dix, qs, g, n)


def test_no_device_memory_growth(rbe, torch):
    """100 rounds of search_device + merge_device + search_words + multi-handle search:
    free device memory is flat after the first round (no per-call allocations or leaks)."""
    N, dim, kp, qp, Q, n = 1_000_000, 128, 3, 3, 16, 1000
    g = geometry(rbe, (-(-N // 2 // 65536), 256, 256, 1))
    shards = [rbe.DeviceIndex.synthetic(dim, kp, True, N, 2, 0xD0C5, [0], r, 2) for r in range(2)]
    multi = rbe.DeviceIndex(rbe.index_from_arrays(dim, kp, True, [shards[0].download_partition(0),
                                                                 shards[1].download_partition(1)]), [0, 0])
    qs = gen_queries(50, Q, dim, qp)
    d = torch.from_numpy(qs.view(np.int64).copy()).cuda()
    outs = [torch.empty(Q * n * rbe.RESULT_RECORD_BYTES, dtype=torch.uint8, device="cuda") for _ in range(2)]
    cat = torch.empty(2 * Q * n * rbe.RESULT_RECORD_BYTES, dtype=torch.uint8, device="cuda")
    merged = torch.empty_like(outs[0])
    stream = torch.cuda.current_stream()

    def round_():
        for r in range(2):
            rbe.search_device(shards[r].handle(0), d.data_ptr(), Q, qp, g, n, outs[r].data_ptr(), stream.cuda_stream,
                              "auto", False)
        torch.cat(outs, out=cat)
        rbe.merge_device(0, cat.data_ptr(), 2, Q, n, merged.data_ptr(), stream.cuda_stream)
        shards[0].search_words(qs, g, n, "auto", 0, False)
        multi.search_words(qs, g, n, "auto", 0, False)

    for _ in range(2):
        round_()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(100):
        round_()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (2 << 20), (free0, free1)
    want = words_result(multi, qs, g, n)
    assert decode(merged, Q, n) == want
