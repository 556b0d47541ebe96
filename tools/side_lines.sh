#!/bin/bash
# The secondary workloads' bench lines (logits, draft, tree, mc) -> gpurun_out/lines_*.log
cd "$(dirname "$0")/.."
for w in logits draft tree mc; do
  timeout 900 python bench.py --workload $w --steps 60 --warmup 5 > gpurun_out/lines_$w.log 2>&1
  echo "== $w"; python tools/bench_summary.py gpurun_out/lines_$w.log | cut -c 1-220
  grep -o '"roofline": {[^}]*}' gpurun_out/lines_$w.log | cut -c 1-400
done
