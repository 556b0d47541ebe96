#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/gpu_tests.sh logits | tail -2
for v in split two; do
  if [ $v = two ]; then export LAPSSD_NORM_TWO_PASS=1; else unset LAPSSD_NORM_TWO_PASS; fi
  timeout 600 python bench.py --workload logits --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/logits_$v.log 2>&1
  echo "== $v"; python tools/bench_summary.py gpurun_out/logits_$v.log | cut -c 1-160
done
unset LAPSSD_NORM_TWO_PASS
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"logits_norm" -s 4 -c 2 --csv \
  --log-file gpurun_out/r02_logits_split_counts.csv python bench.py --workload logits --steps 4 --warmup 3 --graph-steps 1 --no-cpu-baseline > /dev/null 2>&1
grep -i "norm" gpurun_out/r02_logits_split_counts.csv | cut -c 1-250 | tail -6
