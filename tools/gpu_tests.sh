#!/bin/bash
# GPU parity tests only (optionally a -k filter in $1).  Output under gpurun_out/.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
python paper_2505_17074_b200/build.py > /dev/null 2>&1 || true
if [ -n "$1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
fi
tail -30 gpurun_out/pytest_gpu.log
