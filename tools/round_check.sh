#!/bin/bash
# Full round check on one GPU: smoke, default bench (JSON line), un-profiled bench, GPU tests.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
tail -c 2500 gpurun_out/bench_full.log
timeout 200 python bench.py --no-profile --steps 1000 --no-e2e --no-cpu-baseline > gpurun_out/bench_noprof.log 2>&1
tail -c 600 gpurun_out/bench_noprof.log
timeout 240 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
tail -c 800 gpurun_out/bench_ref.log
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
