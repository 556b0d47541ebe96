#!/bin/bash
# ncu evidence for profiles/: per-launch list of the bench command (configs[3] and the
# configs[4] MC mode), and one full capture of the verify kernel.  Never multi-rank.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"verify_kernel|select_side_kernel|accept_kernel|presort_kernel|select_final_kernel|select_kernel" \
  -s 30 -c 60 --csv --log-file gpurun_out/r01f_launches.csv \
  python bench.py --steps 20 --warmup 10 --graph-steps 0 --no-e2e --no-cpu-baseline > gpurun_out/r01f_launch_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify_kernel|mc_step_kernel" \
  -s 30 -c 30 --csv --log-file gpurun_out/r01f_mc_launches.csv \
  python bench.py --workload mc --steps 20 --warmup 10 --graph-steps 1 --no-cpu-baseline > gpurun_out/r01f_mc_launch_bench.log 2>&1
echo "mc launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify_kernel" -s 12 -c 1 \
  -o gpurun_out/r01f_verify_full python bench.py --steps 4 --warmup 10 --graph-steps 0 --no-e2e --no-cpu-baseline \
  > gpurun_out/r01f_full_bench.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/r01f_verify_full.ncu-rep --page raw --csv > gpurun_out/r01f_verify_raw.csv 2>/dev/null
echo "raw export rc=$?"
ncu -i gpurun_out/r01f_verify_full.ncu-rep --page details --csv > gpurun_out/r01f_verify_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_side_kernel" -s 12 -c 1 \
  -o gpurun_out/r01f_side_full python bench.py --steps 4 --warmup 10 --graph-steps 0 --no-e2e --no-cpu-baseline \
  > gpurun_out/r01f_side_bench.log 2>&1
ncu -i gpurun_out/r01f_side_full.ncu-rep --page raw --csv > gpurun_out/r01f_side_raw.csv 2>/dev/null
echo "side capture rc=$?"
