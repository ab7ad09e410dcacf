"""Summarise the ncu outputs of tools/profile_tensor.sh into profiles/ (run here):
python tools/ncu_summary.py TAG [ALGORITHMIC_BYTES_PER_LAUNCH] [CONFIG]  ->  profiles/TAG_ncu_launches.txt, profiles/TAG_ncu_scan.txt,
                                     profiles/scan_traffic.json (dram bytes per main-scan launch)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

tag = sys.argv[1]
lines = open(f"gpurun_out/launches_{tag}.csv").read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
agg = collections.defaultdict(list)
for r in rows:
    name = re.sub(r"\(.*$", "", r["Kernel Name"].replace("void ", "")).replace("rbe_dev::", "")
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    agg[name].append(float(r["Metric Value"]) / 1e3)
out = ["# ncu --metrics gpu__time_duration.sum --clock-control none, one bench step (cold-cache, serialised:",
       "# compare shares, not absolutes).  kernel  launches  mean_us  share_of_search_step", ""]
search = {k: v for k, v in agg.items() if not any(x in k for x in ("fill_", "mag_range"))}
tot = sum(sum(v) / len(v) for v in search.values())
for k, v in sorted(search.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
    m = sum(v) / len(v)
    out.append(f"{k:45s} {len(v):4d} {m:10.1f}  {100 * m / tot:5.1f}%")
open(f"profiles/{tag}_ncu_launches.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))

raw = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{tag}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
pat = re.compile(r"dram__bytes_(read|write)\.sum$|gpu__time_duration.sum|sm__inst_executed_pipe_(alu|fma|lsu|tmem|tc|uniform|xu)\.sum.pct_of_peak_sustained_active|"
                 r"sm__pipe_(alu|fma|shared|tensor)_cycles_active.avg.pct_of_peak_sustained_active|sm__issue_active.avg.pct|"
                 r"launch__registers_per_thread$|launch__grid_size|launch__block_size|sm__cycles_elapsed.avg$|smsp__inst_executed.sum$|"
                 r"dram__throughput.avg.pct_of_peak_sustained_elapsed|smsp__average_warps_issue_stalled_.*_per_issue_active|Kernel Name|"
                 r"sm__warps_active.avg.pct_of_peak_sustained_active|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$")
lines = [f"# ncu --set full --clock-control none, main tensor_scan_kernel launch (gpurun_out/prof_{tag}.ncu-rep)", ""]
vals = {}
for h, u, v in zip(r[0], r[1], r[2]):
    if pat.search(h):
        lines.append(f"{h:90s} {u:10s} {v}")
        vals[h] = (u, v)
open(f"profiles/{tag}_ncu_scan.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:12]))


def to_bytes(uv):
    u, v = uv
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


traffic = to_bytes(vals["dram__bytes_read.sum"]) + to_bytes(vals["dram__bytes_write.sum"])
algo = float(sys.argv[2]) if len(sys.argv) > 2 else 52e9
config = sys.argv[3] if len(sys.argv) > 3 else "bench default: 1B docs, P=8, Q=64, k=1000 (one launch scans all partitions)"
json.dump({"dram_bytes_per_launch": traffic, "kernel": "tensor_scan_kernel (main pass)", "source": f"profiles/{tag}_ncu_scan.txt",
           "algorithmic_bytes_per_launch": algo, "config": config}, open("profiles/scan_traffic.json", "w"), indent=1)
print("traffic", traffic)
