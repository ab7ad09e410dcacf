"""Quick summary of an ncu --set full capture (run here, no GPU):
python tools/ncu_quick.py gpurun_out/prof_TAG.ncu-rep [n_subtiles]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 781250.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
pat = re.compile(r"dram__bytes_(read|write)\.sum$|gpu__time_duration.sum|sm__inst_executed_pipe_(alu|fma|lsu|uniform|xu|tmem|tc)\.sum.pct_of_peak_sustained_active|"
                 r"sm__pipe_(alu|fma|shared|tensor)_cycles_active.avg.pct_of_peak_sustained_active|sm__issue_active.avg.pct|"
                 r"launch__registers_per_thread$|sm__cycles_elapsed.avg$|smsp__inst_executed.sum$|dram__throughput.avg.pct_of_peak_sustained_elapsed|"
                 r"smsp__average_warps_issue_stalled_.*_per_issue_active")
for h, u, v in zip(rows[0], rows[1], rows[2]):
    if pat.search(h):
        try:
            if float(v) == 0:
                continue
        except ValueError:
            pass
        print(f"{h:90s} {u:8s} {v}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
lines = sass.splitlines()
r2 = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = r2[0]
iE, iS, iW = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ops, st = collections.Counter(), collections.Counter()
tot = 0
for r in r2[1:]:
    if len(r) <= iW:
        continue
    n = int(r[iE] or 0)
    tot += n
    toks = r[iS].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += n
    st[op.split(".")[0]] += int(r[iW] or 0)
print(f"total warp-instr {tot}  per unit {tot / units:.1f}")
for k, v in ops.most_common(25):
    print(f"  {k:12s} {v / units:8.1f} per unit   stall-samples {st[k]}")
