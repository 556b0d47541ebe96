#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/build_trace.sh > gpurun_out/trace_build.log 2>&1 || { tail gpurun_out/trace_build.log; exit 1; }
for n in ${NS:-2048}; do
  N=$n timeout 300 python tools/step_timeline.py > gpurun_out/timeline_$n.log 2>&1
  echo "N=$n"; head -30 gpurun_out/timeline_$n.log
done
