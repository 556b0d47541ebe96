#!/bin/bash
# Iteration check on one GPU: GPU tests, smoke, bench (summary), per-CTA timeline.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
if [ -z "$NO_TESTS" ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5; fi
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
python tools/bench_summary.py gpurun_out/bench_iter.log
if [ -z "$NO_TIMELINE" ]; then timeout 200 python tools/cta_timeline.py 2>&1 | grep -A20 "rep 2" | grep -v "Exception\|Traceback\|File\|Attribute"; fi
