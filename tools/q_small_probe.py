import sys; sys.path.insert(0, "/root/repo")
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries
N = 100_000_000
dix = rbe.DeviceIndex.synthetic(128, 3, True, N, 1, 0xD0C5, [0])
g = rbe.ScanGeometry(); g.blocks = -(-N // 65536)
for Q in (1, 8, 16, 32, 63, 64):
    qs = gen_queries(0x0E1 + Q, Q, 128, 3)
    for _ in range(2): st = dix.search_words(qs, g, 1000)[5]
    print(Q, {k: st[k] for k in ("device_ms", "candidates", "survivors")}, flush=True)
