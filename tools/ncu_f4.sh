#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_verify" -s 6 -c 1 \
  -o gpurun_out/f4_tree_full python bench.py --workload tree --steps 4 --warmup 3 --graph-steps 0 --no-cpu-baseline > gpurun_out/f4_ncu.log 2>&1
echo "rc=$?"
ncu -i gpurun_out/f4_tree_full.ncu-rep --page details --csv > gpurun_out/f4_tree_details.csv 2>/dev/null
ncu -i gpurun_out/f4_tree_full.ncu-rep --page raw --csv > gpurun_out/f4_tree_raw.csv 2>/dev/null
ncu -i gpurun_out/f4_tree_full.ncu-rep --page source --csv --print-source sass > gpurun_out/f4_tree_source.csv 2>/dev/null
grep -i "duration\|dram__bytes\|Throughput\|Registers\|Achieved Occupancy\|Issue Slots\|Warp Cycles Per Issued\|No Eligible\|stall" gpurun_out/f4_tree_details.csv | head -40
