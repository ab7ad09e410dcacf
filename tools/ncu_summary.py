"""Summarise ncu outputs brought back by tools/profile_tensor.sh (run here)."""
import csv
import re
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = defaultdict(list)
    for r in rows:
        name = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("rbe_dev::", "")
        name = re.sub(r"\(.*\)$", "", name.replace("void ", "")).replace("unnamed>::", "")
        agg[name].append(float(r["Metric Value"]) / 1e3)
    return agg


def raw(rep, keys):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr) if any(h.startswith(k) for k in keys)}


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    agg = launches(f"gpurun_out/launches_{tag}.csv")
    print("kernel                                         launches  median_us")
    for k, v in agg.items():
        v = sorted(v)
        print(f"{k[:48]:48s} {len(v):6d} {v[len(v) // 2]:10.1f}")
    r = raw(f"gpurun_out/prof_{tag}.ncu-rep",
            ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct",
             "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct",
             "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
             "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_selected",
             "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
             "smsp__pcsamp_warps_issue_stalled_math_pipe", "smsp__pcsamp_warps_issue_stalled_no_instruction",
             "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_lg_throttle"])
    for k in sorted(r):
        print(f"{k:70s} {r[k][0]:>16s} {r[k][1]}")
