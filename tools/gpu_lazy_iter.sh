#!/bin/bash
# f1 lazy kernel iteration: parity tests, bench line, per-unit timeline (trace build).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_logits.py -x -q > gpurun_out/pytest_logits.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_logits.log
tail -3 gpurun_out/pytest_logits.log
timeout 300 python bench.py --workload logits --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_logits.log 2>&1; echo "rc=$?" >> gpurun_out/bench_logits.log
grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_logits.log
timeout 300 python tools/lazy_timeline.py > gpurun_out/lazy_timeline.log 2>&1; echo "rc=$?" >> gpurun_out/lazy_timeline.log
tail -c 3000 gpurun_out/lazy_timeline.log
for v in $LAZY_VARIANTS; do
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_logits.py -x -q 2>&1 | tail -1
  LAPSSD_LIBRARY=tools/variants/lib_$v.so timeout 300 python bench.py --workload logits --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/lz_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/lz_$v.log)"
done
