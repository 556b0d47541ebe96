#!/bin/bash
# full ncu capture of the f1 lazy kernel (variant library in $1, default: the product)
cd "$(dirname "$0")/.."
lib=${1:-paper_2505_17074_b200/liblapssd.so}
LAPSSD_LIBRARY=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"logits_lazy" -s 4 -c 1 \
  -o gpurun_out/r02_lazy_full python bench.py --workload logits --steps 2 --warmup 3 --graph-steps 1 --no-cpu-baseline > gpurun_out/r02_lazy_ncu.log 2>&1
ncu -i gpurun_out/r02_lazy_full.ncu-rep --page details --csv > gpurun_out/r02_lazy_details.csv 2>/dev/null
ncu -i gpurun_out/r02_lazy_full.ncu-rep --page raw --csv > gpurun_out/r02_lazy_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_lazy_full.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02_lazy_source_cuda.csv 2>/dev/null
echo done
