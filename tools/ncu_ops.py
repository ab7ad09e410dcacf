"""Opcode histogram (thread-instructions per doc) and top stall lines of the
captured main scan kernel: python tools/ncu_ops.py <tag> [n_docs]"""
import csv
import io
import subprocess
import sys
from collections import Counter

tag = sys.argv[1]
n_docs = float(sys.argv[2]) if len(sys.argv) > 2 else 1e8
out = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{tag}.ncu-rep", "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ai, si = hdr.index("Address"), hdr.index("Source")
st, ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
c = Counter()
for r in data:
    e = int(r[ex] or 0)
    if not e:
        continue
    t = r[si].strip().split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += e
tot = sum(c.values())
print(f"total warp-instr {tot}  thread-instr/doc {tot * 32 / n_docs:.1f}")
print("  ".join(f"{k}:{v * 32 / n_docs:.1f}" for k, v in c.most_common(24)))
tot_st = sum(int(r[st] or 0) for r in data)
for r in sorted(data, key=lambda r: -int(r[st] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 16]:
    print(f"{int(r[st]) / tot_st * 100:5.1f}% {int(r[ex] or 0):11d} {r[ai][-5:]} {r[si].strip()[:90]}")
