"""Run one small tensor-scan case against the compiled reference (GPU box debugging):
python tools/dbg_case.py N DIM KP QP P BLOCKS TPB IPT QL n [rw]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1802_06466_b200 as rbe  # noqa: E402
from oracle.oracle import Ref, gen_queries, synthetic_partitions  # noqa: E402

N, dim, kp, qp, P, B, T, I, QL, n = map(int, sys.argv[1:11])
rw = len(sys.argv) <= 11 or sys.argv[11] != "0"
parts = synthetic_partitions(0xD0C5, N, dim, kp, P, rw)
qs = gen_queries(0x0E1, 3, dim, qp)
dix = rbe.DeviceIndex(rbe.index_from_arrays(dim, kp, rw, [tuple(p) for p in parts]))
g = rbe.ScanGeometry()
g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length = B, T, I, QL
want, _ = Ref().index(dim, kp, rw, parts).search(qs, (B, T, I, QL), n)
for variant in ("exact", "tensor"):
    scores, ids, pp, accs, counts, stats = dix.search_words(qs, g, n, variant)
    print(variant, stats, flush=True)
    got = [[(float(scores[q, k]), int(ids[q, k]), int(pp[q, k])) for k in range(int(counts[q]))]
           for q in range(qs.shape[0])]
    print(variant, "parity", got == want, flush=True)
