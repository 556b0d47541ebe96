#!/bin/bash
# Per-launch device times of the library's kernels (cold-cache, serialised by ncu).
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/launches.csv}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify_kernel|select_final_kernel|presort_kernel|select_kernel|accept_kernel|merge_kernel|candidates_kernel|update_kernel" -s 20 -c 60 --csv \
  --log-file $OUT python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
python - "$OUT" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); agg[d['Kernel Name'].split('(')[0]].append(float(d['Metric Value'].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items(): print(f"{k:45s} n={len(v):3d} mean={sum(v)/len(v)/1000:8.2f} us share={sum(v)/tot:.3f}")
PY
