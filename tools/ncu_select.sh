#!/bin/bash
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
export LAPSSD_CPB=4
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"select_final_kernel" -s 10 -c 1 -o gpurun_out/prof_self python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_self.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_self.log
