#!/bin/bash
# configs[1] / configs[2] full size: parity + JCT per policy; configs[2] load sweep (LAPS-SD, FCFS, LP-SJF, LAS)
cd "$(dirname "$0")/.."
for pol in 0 1 2 3; do
  timeout 900 python bench.py --workload c2 --policy $pol > gpurun_out/c2_p$pol.log 2>&1; tail -c 600 gpurun_out/c2_p$pol.log | grep -o '"jct": {[^}]*}\|"bit_exact": [a-z]*\|"ms_per_step": [0-9.]*'
done
for rho in 0.5 0.7 0.9 1.0 1.2; do
  for pol in 0 1 2 3; do
    par=""; [ "$rho" != "0.9" ] && par="--no-parity"
    timeout 900 python bench.py --workload c3 --policy $pol --rho $rho $par > gpurun_out/c3_r${rho}_p$pol.log 2>&1
    echo "rho $rho pol $pol: $(grep -o '"mean_ms": [0-9.]*\|"bit_exact": [a-z]*' gpurun_out/c3_r${rho}_p$pol.log | tr '\n' ' ')"
  done
done
