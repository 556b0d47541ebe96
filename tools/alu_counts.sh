#!/bin/bash
# Executed instructions per launch of the ALU-bound kernels (f1 logits, f4 tree) for the
# bench's "alu" roofline: ncu, one GPU.
cd "$(dirname "$0")/.."
M=smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg
timeout 600 ncu --metrics $M --clock-control none -k regex:"logits_lazy|logits_norm|logits_sample" -s 6 -c 4 --csv \
  --log-file gpurun_out/r02_logits_counts.csv python bench.py --workload logits --steps 4 --warmup 3 --graph-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"tree_verify" -s 3 -c 4 --csv \
  --log-file gpurun_out/r02_tree_counts.csv python bench.py --workload tree --steps 4 --warmup 3 --graph-steps 1 --no-cpu-baseline > /dev/null 2>&1
echo done
