#!/bin/bash
# f1 speculation-depth variants, A/B in one session (diagnostic builds under tools/variants/)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in $VARS; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_logits.py -x -q 2>&1 | tail -1
done
for i in 1 2; do
for v in $VARS; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python bench.py --workload logits --steps 400 --warmup 5 --no-cpu-baseline > gpurun_out/sv_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sv_$v.log)"
done
done
