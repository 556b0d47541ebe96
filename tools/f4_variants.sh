#!/bin/bash
# tree kernel: trees per CTA variants (diagnostic builds under tools/variants/, never the product)
cd "$(dirname "$0")/.."
mkdir -p tools/variants
bash tools/gpu_tests.sh f4 | tail -2
for t in 4 2 8; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -DLAPSSD_TREES_PER_CTA=$t \
    -Xcompiler -fPIC -shared -o tools/variants/lib_g$t.so paper_2505_17074_b200/csrc/api.cu paper_2505_17074_b200/csrc/verify.cu \
    paper_2505_17074_b200/csrc/verify_logits.cu paper_2505_17074_b200/csrc/sched.cu paper_2505_17074_b200/csrc/mc.cu \
    paper_2505_17074_b200/csrc/draft_tree.cu -ldl
  LAPSSD_LIBRARY=tools/variants/lib_g$t.so timeout 600 python bench.py --workload tree --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/f4_tree_g$t.log 2>&1
  echo "trees/CTA $t"; python tools/bench_summary.py gpurun_out/f4_tree_g$t.log | cut -c 1-150
done
