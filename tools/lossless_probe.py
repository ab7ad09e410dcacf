"""Device time of one 64-query batch at 100M docs in the lossless regime (queue_length >=
items_per_thread) on the tensor variant, next to queue_length 1 (tensor and CUDA-core exact variants).
The exact kernel cannot hold 256-entry queues for 390K threads x 64 queries (153 GB of scratch)."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dix = rbe.DeviceIndex.synthetic(128, 3, True, N, 1, 0xD0C5, [0])
qs = gen_queries(0x0E1, 64, 128, 3)
for ql, variant in ((1, "tensor"), (256, "tensor"), (1, "exact")):
    g = rbe.ScanGeometry(); g.blocks = -(-N // 65536); g.queue_length = ql
    for _ in range(2):
        st = dix.search_words(qs, g, 1000, variant)[5]
    print(f"queue_length={ql} variant={variant}:", {k: st[k] for k in ("device_ms", "candidates", "survivors")}, flush=True)
