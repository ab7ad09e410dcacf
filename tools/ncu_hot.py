"""Hot SASS instructions by stall samples, with context: python tools/ncu_hot.py REP [pct] [ctx]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pct = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
hdr, data = rows[0], rows[1:]
iE, iS, iW = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iW] or 0) for r in data if len(r) > iW)
print("total samples", tot)
shown = set()
for k, r in enumerate(data):
    if len(r) <= iW:
        continue
    if int(r[iW] or 0) > tot * pct / 100:
        for kk in range(max(0, k - ctx), min(len(data), k + 1)):
            if kk in shown:
                continue
            shown.add(kk)
            rr = data[kk]
            print(f"{kk:5d} {int(rr[iW] or 0):7d} {int(rr[iE] or 0):10d}  {rr[iS][:100]}")
        print("   ...")
