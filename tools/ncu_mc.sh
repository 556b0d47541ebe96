#!/bin/bash
# configs[4] Monte-Carlo step: one full ncu capture each of verify_kernel and mc_step_kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=(python bench.py --workload mc --steps 6 --warmup 10 --graph-steps 1 --no-cpu-baseline --mc-policies "")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify_kernel" -s 30 -c 1 \
  -o gpurun_out/mc_verify_full "${B[@]}" > gpurun_out/mc_ncu1.log 2>&1
ncu -i gpurun_out/mc_verify_full.ncu-rep --page details --csv > gpurun_out/mc_verify_details.csv 2>/dev/null
ncu -i gpurun_out/mc_verify_full.ncu-rep --page raw --csv > gpurun_out/mc_verify_raw.csv 2>/dev/null
ncu -i gpurun_out/mc_verify_full.ncu-rep --page source --csv --print-source sass > gpurun_out/mc_verify_sass.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_step_kernel" -s 15 -c 1 \
  -o gpurun_out/mc_step_full "${B[@]}" > gpurun_out/mc_ncu2.log 2>&1
ncu -i gpurun_out/mc_step_full.ncu-rep --page details --csv > gpurun_out/mc_step_details.csv 2>/dev/null
ncu -i gpurun_out/mc_step_full.ncu-rep --page raw --csv > gpurun_out/mc_step_raw.csv 2>/dev/null
ncu -i gpurun_out/mc_step_full.ncu-rep --page source --csv --print-source sass > gpurun_out/mc_step_sass.csv 2>/dev/null
timeout 600 python bench.py --workload mc --steps 60 --warmup 10 --no-cpu-baseline --mc-policies "" > gpurun_out/mc_bench.log 2>&1
grep -o '"ms_per_step": [0-9.]*' gpurun_out/mc_bench.log
echo done
