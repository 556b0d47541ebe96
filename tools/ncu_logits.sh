#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"logits_norm|logits_sample" -s 4 -c 2 \
  -o gpurun_out/r02_logits_full python bench.py --workload logits --steps 2 --warmup 3 --graph-steps 1 --no-cpu-baseline > gpurun_out/r02_logits_ncu.log 2>&1
ncu -i gpurun_out/r02_logits_full.ncu-rep --page details --csv > gpurun_out/r02_logits_details.csv 2>/dev/null
ncu -i gpurun_out/r02_logits_full.ncu-rep --page raw --csv > gpurun_out/r02_logits_raw.csv 2>/dev/null
echo done
