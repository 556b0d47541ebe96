#!/bin/bash
# configs[4] MC engine variants (diagnostic builds under tools/variants/, never the product)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mc.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --workload mc --steps 100 --warmup 10 --no-cpu-baseline --mc-policies "" > gpurun_out/mcv_product.log 2>&1
echo "product $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mcv_product.log)"
for v in $MC_VARIANTS; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_mc.py -x -q 2>&1 | tail -1
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 600 python bench.py --workload mc --steps 100 --warmup 10 --no-cpu-baseline --mc-policies "" > gpurun_out/mcv_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mcv_$v.log)"
done
timeout 600 python bench.py --workload mc --steps 100 --warmup 10 --no-cpu-baseline --mc-policies "" > gpurun_out/mcv_product2.log 2>&1
echo "product $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/mcv_product2.log)"
