#!/bin/bash
cd "$(dirname "$0")/.."
for n in 2048 16384; do
  for v in wl nowl; do
    if [ $v = nowl ]; then export LAPSSD_NO_WAITLIST=1; else unset LAPSSD_NO_WAITLIST; fi
    timeout 300 python bench.py --steps 200 --warmup 20 --n-per-gpu $n --no-e2e --no-cpu-baseline > gpurun_out/wl_${n}_$v.log 2>&1
    echo "N=$n $v"; python tools/bench_summary.py gpurun_out/wl_${n}_$v.log
  done
done
unset LAPSSD_NO_WAITLIST
[ -n "$TIMELINE" ] && NS="2048 16384" bash tools/timeline_run.sh 2>&1 | grep -v "merge passes" | head -40
