#!/bin/bash
# configs[3] driver-window A/B of verify-kernel knobs (diagnostic builds under tools/variants/), alternating fresh processes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in $VARS; do
    LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-profile > gpurun_out/wv_${v}_$i.log 2>&1
    echo "$v $i $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/wv_${v}_$i.log)"
  done
done
