#!/bin/bash
# One GPU iteration (run under gpurun): GPU parity tests, a bench line, the
# ncu launch list + full capture of the main scan kernel.
TAG=${1:-r01}
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"], 3), "scan_ms", round(d["roofline"]["scan_ms"], 3),
      "frac", round(d["roofline"]["frac"], 3), "cands", d["candidates_per_batch"], "surv", d["survivors_per_batch"],
      "e2e", round(d["e2e"]["value"]), "clk", d["clocks"])
PY
[ "$2" = "noprof" ] || ./tools/profile_tensor.sh $TAG
