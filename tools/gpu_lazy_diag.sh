#!/bin/bash
# f1 lazy kernel diagnostics: per-unit timeline (trace build) + one full ncu capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/lazy_timeline.py > gpurun_out/lazy_timeline.log 2>&1; echo "rc=$?" >> gpurun_out/lazy_timeline.log
tail -c 6000 gpurun_out/lazy_timeline.log
bash tools/ncu_lazy.sh
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/r02_lazy_details.csv")) if r]
hdr=rows[0]
iname=hdr.index("Metric Name"); iv=hdr.index("Metric Value"); iu=hdr.index("Metric Unit"); isec=hdr.index("Section Name")
for r in rows[1:]:
    if r[isec] in ("GPU Speed Of Light Throughput","Compute Workload Analysis","Memory Workload Analysis","Occupancy","Warp State Statistics","Launch Statistics"):
        print(r[isec][:20], r[iname], r[iv], r[iu])
PY
