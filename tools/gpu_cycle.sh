#!/bin/bash
# One GPU iteration (run under gpurun): GPU parity tests, smoke, the bench line (with
# the CPU baseline), the reference arm, the ncu launch list and one full capture of
# the main scan launch.  Outputs under gpurun_out/ (tag = $1).
TAG=${1:-r01}
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"], 3), "scan_ms", round(d["roofline"]["scan_ms"], 3),
      "frac", round(d["roofline"]["frac"], 3), "cands", d["candidates_per_batch"], "surv", d["survivors_per_batch"],
      "e2e", round(d["e2e"]["value"]), "cpu", d["cpu_baseline"] and d["cpu_baseline"].get("value"), "clk", d["clocks"])
r = json.load(open("gpurun_out/bench_ref_$TAG.json"))
print("reference arm", r.get("value"), r.get("unit"), r.get("cpu_baseline", {}).get("cores"))
PY
[ "$2" = "noprof" ] || ./tools/profile_tensor.sh $TAG
