#!/bin/bash
# tree kernel thread-count variants (diagnostic builds under tools/variants/, never the product)
cd "$(dirname "$0")/.."
mkdir -p tools/variants
for t in 256 512 128; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -DLAPSSD_TREE_THREADS=$t \
    -Xcompiler -fPIC -shared -o tools/variants/lib_t$t.so paper_2505_17074_b200/csrc/api.cu paper_2505_17074_b200/csrc/verify.cu \
    paper_2505_17074_b200/csrc/verify_logits.cu paper_2505_17074_b200/csrc/sched.cu paper_2505_17074_b200/csrc/mc.cu \
    paper_2505_17074_b200/csrc/draft_tree.cu -ldl
  LAPSSD_LIBRARY=tools/variants/lib_t$t.so timeout 600 python bench.py --workload tree --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/f4_tree_t$t.log 2>&1
  echo "threads $t"; python tools/bench_summary.py gpurun_out/f4_tree_t$t.log
done
