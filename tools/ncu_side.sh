#!/bin/bash
# Full ncu capture of the side-stream select kernel (tooling): source-level stall sampling.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on \
  -k regex:"select_side_kernel" -s 12 -c 1 -o gpurun_out/prof_side \
  python bench.py --steps 4 --warmup 10 --graph-steps 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_side.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_side.log
ncu -i gpurun_out/prof_side.ncu-rep --page source --csv --print-source sass > gpurun_out/side_sass.csv 2>&1
ncu -i gpurun_out/prof_side.ncu-rep --page source --csv --print-source cuda > gpurun_out/side_cuda.csv 2>&1
ncu -i gpurun_out/prof_side.ncu-rep --page raw --csv > gpurun_out/side_raw.csv 2>&1
ls -la gpurun_out/
