"""Device time of the C2 batch (100M docs, Q=64, k=1000): best of 7 (quick A/B of kernel builds)."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dix = rbe.DeviceIndex.synthetic(128, 3, True, N, P, 0xD0C5, [0])
g = rbe.ScanGeometry(); g.blocks = -(-(-(-N // P)) // 65536)
qs = gen_queries(0x0E1, 64, 128, 3)
for _ in range(2):
    dix.search_words(qs, g, 1000)
ts = [dix.search_words(qs, g, 1000)[5] for _ in range(7)]
print("device_ms best", round(min(t["device_ms"] for t in ts), 4), "median", round(sorted(t["device_ms"] for t in ts)[3], 4))
