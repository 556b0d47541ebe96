#!/bin/bash
# The driver's bench window (--steps 20 --warmup 5) in fresh processes, vs later windows.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/win_$i.log 2>&1
  python tools/bench_summary.py gpurun_out/win_$i.log
done
for w in 50 200; do
  timeout 300 python bench.py --steps 20 --warmup $w --no-e2e --no-cpu-baseline > gpurun_out/win_w$w.log 2>&1
  echo "warmup $w"; python tools/bench_summary.py gpurun_out/win_w$w.log
done
timeout 300 python bench.py --steps 400 --warmup 20 --no-e2e --no-cpu-baseline > gpurun_out/win_400.log 2>&1
echo "400 steps"; python tools/bench_summary.py gpurun_out/win_400.log
