#!/bin/bash
# GPU tests, then the default bench N times back to back (tooling: stability / variance).
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
if [ -z "$NO_TESTS" ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi
for i in $(seq 1 ${N:-4}); do
  timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 2000 > gpurun_out/rep_$i.log 2>&1
  python tools/bench_summary.py gpurun_out/rep_$i.log
done
