"""Multi-rank orchestration of the sharded search (paper_1802_06466_b200.distributed)
on CPU: world_size 2 over gloo.

Each rank owns partitions p % world == rank (src/index.cpp:53's round-robin rule
applied to partitions), computes its per-query top-n with the CPU oracle (the
device scan's stand-in here; the GPU path is covered by tests/test_gpu_parity.py),
encodes the lists as the C ABI's 32-byte rbe_result records, and
gather_and_merge() collects them on rank 0, which merges under entry_less
(score desc, id asc; src/search.cpp:50-53, 160-167).  The merged lists must equal
the oracle's search over the whole partitioned index -- the property that makes
results identical for any GPU count with the partition count fixed.
"""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Port, gen_queries, synthetic_partitions

REC = np.dtype([("score", "<f8"), ("id", "<u8"), ("acc", "<i8"), ("partition", "<u4"), ("valid", "<u4")])


def encode(lists, n):
    rec = np.zeros((len(lists), n), dtype=REC)
    for q, entries in enumerate(lists):
        for k, (s, i, p, a) in enumerate(entries[:n]):
            rec[q, k] = (s, i, a, p, 1)
    return rec


def merge_cpu(blocks, n_queries, n):
    """entry_less merge of per-rank [Q][n] record blocks (CPU stand-in for rbe_cuda_merge_device)."""
    recs = [np.frombuffer(b.numpy().tobytes(), dtype=REC).reshape(n_queries, n) for b in blocks]
    out = np.zeros((n_queries, n), dtype=REC)
    for q in range(n_queries):
        cat = np.concatenate([r[q][r[q]["valid"] == 1] for r in recs])
        order = np.lexsort((cat["id"], -cat["score"]))
        m = min(n, len(order))
        out[q, :m] = cat[order[:m]]
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, result_path):
    import torch
    import torch.distributed as dist

    from paper_1802_06466_b200.distributed import RESULT_BYTES, gather_and_merge, owned_partitions

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n_docs, dim, kp, qp, P, geo, n, Q = case
        oracle = Port()
        parts = synthetic_partitions(0xD0C5, n_docs, dim, kp, P, True, oracle)
        qs = gen_queries(0x0E1, Q, dim, qp)
        mine = set(owned_partitions(P, rank, world))
        assert sorted(mine) == [p for p in range(P) if p % world == rank]
        # non-owned partitions are empty here, so partition ordinals stay global
        local = [pt if p in mine else (pt[0][:, :0], pt[1][:0], pt[2][:0]) for p, pt in enumerate(parts)]
        lists = [oracle.search(qs[q], dim, kp, True, local, geo, n)[0] for q in range(Q)]
        block = torch.from_numpy(encode(lists, n).view(np.uint8).reshape(-1).copy())
        assert block.numel() == Q * n * RESULT_BYTES
        merged = gather_and_merge(block, rank, world, lambda bl: merge_cpu(bl, Q, n), dist)
        if rank == 0:
            want = [oracle.search(qs[q], dim, kp, True, parts, geo, n)[0] for q in range(Q)]
            got = [[(float(r["score"]), int(r["id"]), int(r["partition"]), int(r["acc"]))
                    for r in merged[q] if r["valid"]] for q in range(Q)]
            ok = got == [[(s, i, p, a) for s, i, p, a in w] for w in want]
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
        else:
            assert merged is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (6000, 128, 3, 3, 4, (1, 256, 256, 256), 40, 3),   # lossless queue: invariant to the sharding
    (9000, 64, 2, 2, 8, (1, 256, 16, 1), 25, 2),        # rbeKNN queue length 1, eight partitions
])
def test_two_rank_gather_merge_equals_whole_index(tmp_path, case):
    import torch.multiprocessing as mp

    out = tmp_path / "result"
    mp.spawn(_worker, args=(2, _free_port(), case, str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"


def test_owned_partitions_round_robin():
    from paper_1802_06466_b200.distributed import owned_partitions

    assert owned_partitions(8, 0, 1) == list(range(8))
    assert owned_partitions(8, 1, 4) == [1, 5]
    assert sorted(sum((owned_partitions(10, r, 3) for r in range(3)), [])) == list(range(10))
