"""Per-instruction execution counts and stall samples of an ncu capture, grouped into
straight-line runs of equal count (run here, no GPU):
python tools/sass_regions.py REP [min_pct] [dump_path]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
hdr, data = rows[0], rows[1:]
iE, iS, iW = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        for k, r in enumerate(data):
            f.write(f"{k:5d} {int(r[iW] or 0):6d} {int(r[iE] or 0):10d} {r[iS]}\n")
tot = sum(int(r[iE] or 0) for r in data)
tots = sum(int(r[iW] or 0) for r in data)
print("total exec", tot, "samples", tots)
grp, cur = [], None
for k, r in enumerate(data):
    e = int(r[iE] or 0)
    w = int(r[iW] or 0)
    if cur and cur[2] == e:
        cur[1] = k
        cur[3] += w
    else:
        cur = [k, k, e, w]
        grp.append(cur)
for g in sorted(grp, key=lambda g: -g[2] * (g[1] - g[0] + 1)):
    n = g[1] - g[0] + 1
    if g[2] * n < tot * min_pct / 100:
        break
    print(f"{g[0]:5d}-{g[1]:5d} n={n:4d} exec/inst={g[2]:10d} exec%={100 * g[2] * n / tot:5.1f} "
          f"stall%={100 * g[3] / tots:5.1f}  {data[g[0]][iS][:50]}")
