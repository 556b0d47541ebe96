#!/bin/bash
# tree kernel: CTAs-per-tree (cluster size) variants, diagnostic builds under tools/variants/ (never the product).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_f4.py -x -q > gpurun_out/pytest_f4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f4.log
tail -2 gpurun_out/pytest_f4.log
timeout 600 python bench.py --workload tree --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/f4_tree.log 2>&1
echo "product $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/f4_tree.log)"
for v in $TREE_VARIANTS; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_f4.py -x -q 2>&1 | tail -1
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 600 python bench.py --workload tree --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/f4_tree_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/f4_tree_$v.log)"
done
