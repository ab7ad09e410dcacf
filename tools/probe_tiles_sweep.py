import sys; sys.path.insert(0, "/root/repo")
import paper_1802_06466_b200 as rbe
from oracle.oracle import gen_queries
N = 1_000_000_000
dix = rbe.DeviceIndex.synthetic(128, 3, True, N, 8, 0xD0C5, [0])
g = rbe.ScanGeometry(); g.blocks = -(-(N // 8) // 65536)
qs = gen_queries(0x0E1, 64, 128, 3)
for pt in [int(x) for x in sys.argv[1:]] or (8, 4, 2, 1, 16):
    for _ in range(2): st = dix.search_words(qs, g, 1000, "auto", pt)[5]
    ts = [dix.search_words(qs, g, 1000, "auto", pt)[5]["device_ms"] for _ in range(3)]
    print(pt, round(min(ts), 3), st["candidates"], st["survivors"], flush=True)
