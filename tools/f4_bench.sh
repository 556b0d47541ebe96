#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python bench.py --workload draft --steps 60 --warmup 5 > gpurun_out/f4_draft.log 2>&1
python tools/bench_summary.py gpurun_out/f4_draft.log
timeout 600 python bench.py --workload tree --steps 60 --warmup 5 > gpurun_out/f4_tree.log 2>&1
python tools/bench_summary.py gpurun_out/f4_tree.log
tail -c 1500 gpurun_out/f4_tree.log
