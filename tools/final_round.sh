#!/bin/bash
# Round-end evidence for THIS build on one GPU: ncu captures first (their source digests make
# the bench lines report traffic / instruction counts), then smoke, the driver's bench
# commands, every secondary workload's line, and the GPU test suite.  Outputs: gpurun_out/final_*.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/final_profiles.sh > gpurun_out/final_profiles.log 2>&1
cp gpurun_out/verify_dram.json gpurun_out/alu_counts.json profiles/ 2>/dev/null
bash tools/ncu_lazy.sh > /dev/null 2>&1
bash tools/ncu_mc.sh > /dev/null 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 400 python bench.py > gpurun_out/final_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_default.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/final_win_$i.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_reference.log
timeout 300 python bench.py --workload logits > gpurun_out/final_line_logits.log 2>&1
timeout 600 python bench.py --workload logits_step > gpurun_out/final_line_logits_step.log 2>&1
timeout 900 python bench.py --workload mc > gpurun_out/final_line_mc.log 2>&1
timeout 300 python bench.py --workload draft > gpurun_out/final_line_draft.log 2>&1
timeout 300 python bench.py --workload tree > gpurun_out/final_line_tree.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest_gpu.log
for f in gpurun_out/final_*.log; do echo "== $f"; tail -c 400 $f | tail -2; done
