#!/bin/bash
# full ncu capture of the f4 tree verification kernel (pipe utilisation of its 128-bit chains)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_verify" -s 3 -c 1 \
  -o gpurun_out/r02_tree_full python bench.py --workload tree --steps 2 --warmup 3 --graph-steps 1 --no-cpu-baseline > gpurun_out/r02_tree_ncu.log 2>&1
ncu -i gpurun_out/r02_tree_full.ncu-rep --page details --csv > gpurun_out/r02_tree_details.csv 2>/dev/null
ncu -i gpurun_out/r02_tree_full.ncu-rep --page raw --csv > gpurun_out/r02_tree_raw.csv 2>/dev/null
echo done
