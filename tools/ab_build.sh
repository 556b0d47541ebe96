#!/bin/bash
# A/B: the product build vs a diagnostic build with extra -D flags ($1), bench windows.
cd "$(dirname "$0")/.."
mkdir -p tools/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false $1 \
  -Xcompiler -fPIC -shared -o tools/variants/lib_ab.so paper_2505_17074_b200/csrc/api.cu paper_2505_17074_b200/csrc/verify.cu \
  paper_2505_17074_b200/csrc/verify_logits.cu paper_2505_17074_b200/csrc/sched.cu paper_2505_17074_b200/csrc/mc.cu \
  paper_2505_17074_b200/csrc/draft_tree.cu -ldl
for rep in 1 2; do
  timeout 300 python bench.py --steps 400 --warmup 20 --no-e2e --no-cpu-baseline > gpurun_out/ab_base_$rep.log 2>&1
  python tools/bench_summary.py gpurun_out/ab_base_$rep.log
  LAPSSD_LIBRARY=tools/variants/lib_ab.so timeout 300 python bench.py --steps 400 --warmup 20 --no-e2e --no-cpu-baseline > gpurun_out/ab_var_$rep.log 2>&1
  python tools/bench_summary.py gpurun_out/ab_var_$rep.log
done
