#!/bin/bash
# Diagnostic build of liblapssd.so with per-event timestamps (never the product build).
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -DLAPSSD_TRACE $EXTRA \
  -Xcompiler -fPIC -shared -o ${OUT:-tools/liblapssd_trace.so} paper_2505_17074_b200/csrc/api.cu \
  paper_2505_17074_b200/csrc/verify.cu paper_2505_17074_b200/csrc/verify_logits.cu paper_2505_17074_b200/csrc/sched.cu paper_2505_17074_b200/csrc/mc.cu -ldl
