#!/bin/bash
# Bench each tools/variants/lib_*.so (or those named in $VARIANTS) back to back (tooling).
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in ${VARIANTS:-$(ls tools/variants | sed 's/lib_//; s/.so//')}; do
  envs=""; [ -f tools/variants/$v.env ] && envs=$(cat tools/variants/$v.env)
  env $envs LAPSSD_LIBRARY=$PWD/tools/variants/lib_$v.so timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 1000 > gpurun_out/var_$v.log 2>&1
  python tools/bench_summary.py gpurun_out/var_$v.log
done
done
