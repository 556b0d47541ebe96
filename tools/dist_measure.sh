#!/bin/bash
cd "$(dirname "$0")/.."
for n in 2048 16384; do
  timeout 300 python bench.py --dist-path --steps 200 --warmup 20 --n-per-gpu $n --no-e2e --no-cpu-baseline > gpurun_out/dist_$n.log 2>&1
  timeout 300 python bench.py --peer-path --steps 200 --warmup 20 --n-per-gpu $n --no-e2e --no-cpu-baseline > gpurun_out/peer_$n.log 2>&1
  echo "peer N=$n"; python tools/bench_summary.py gpurun_out/peer_$n.log
  echo "dist N=$n"; python tools/bench_summary.py gpurun_out/dist_$n.log
done
