#!/bin/bash
# Build a product-equivalent library variant with extra -D flags: tools/variants/lib_$1.so (tooling).
cd "$(dirname "$0")/.."
mkdir -p tools/variants
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false "$@" \
  -Xcompiler -fPIC -shared -o tools/variants/lib_$name.so paper_2505_17074_b200/csrc/api.cu \
  paper_2505_17074_b200/csrc/verify.cu paper_2505_17074_b200/csrc/verify_logits.cu paper_2505_17074_b200/csrc/sched.cu paper_2505_17074_b200/csrc/mc.cu paper_2505_17074_b200/csrc/draft_tree.cu -ldl
