#!/bin/bash
# f1 lazy kernel: CTA size / residency variants (diagnostic builds under tools/variants/, never the product)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_logits.py -x -q 2>&1 | tail -1
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python bench.py --workload logits --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/lz_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/lz_$v.log)"
done
timeout 300 python bench.py --workload logits --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/lz_product.log 2>&1
echo "product $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/lz_product.log)"
