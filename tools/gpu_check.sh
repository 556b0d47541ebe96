#!/bin/bash
# One GPU session: parity tests, then bench variants.  Output under gpurun_out/.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-default}; do
  if [ "$v" = "default" ]; then unset LAPSSD_VERIFY_CTAS_PER_SM; else export LAPSSD_VERIFY_CTAS_PER_SM=$v; fi
  timeout 240 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  echo "variant=$v"; python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_$v.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_$v.log').read()[-3000:]); sys.exit()
d=json.loads(l[-1]); r=d['roofline']
print('value %.4g ms/step %.4f verify %.4f ms select %.4f ms presort_end %.4f ms achieved %.0f GB/s frac %.3f' % (d['value'], d['ms_per_step'], r['verify_ms_avg'], r['select_ms_avg'], r.get('presort_end_ms_avg', 0), r['achieved'], r['frac']))"
done
