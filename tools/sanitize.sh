#!/bin/bash
# Run under gpurun: compute-sanitizer memcheck / racecheck / synccheck over smoke()
# (exact scan, tensor scan with its tensor-core and CUDA-core bodies, probe, theta, select on 40K docs) and the device merge test.
# Logs: gpurun_out/sanitizer_<tool>.log
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 \
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer_$tool.log)"
done
