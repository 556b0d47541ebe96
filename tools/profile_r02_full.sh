#!/bin/bash
# Round-2 ncu evidence for profiles/: launch lists (configs[3] step, configs[4] MC, f4) and
# full captures of the verify kernel and the side select.  One GPU, never multi-rank.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify_kernel" -s 15 -c 1 \
  -o gpurun_out/r02_verify_full python bench.py --steps 4 --warmup 20 --graph-steps 0 --no-e2e --no-cpu-baseline --no-profile \
  > gpurun_out/r02_full_bench.log 2>&1
echo "verify full rc=$?"
ncu -i gpurun_out/r02_verify_full.ncu-rep --page raw --csv > gpurun_out/r02_verify_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_verify_full.ncu-rep --page details --csv > gpurun_out/r02_verify_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_side_kernel" -s 15 -c 1 \
  -o gpurun_out/r02_side_full python bench.py --steps 4 --warmup 20 --graph-steps 0 --no-e2e --no-cpu-baseline --no-profile \
  > gpurun_out/r02_side_bench.log 2>&1
ncu -i gpurun_out/r02_side_full.ncu-rep --page details --csv > gpurun_out/r02_side_details.csv 2>/dev/null
echo "side full rc=$?"
python - <<'PY'
import csv, json, sys
sys.path.insert(0, ".")
import bench
rows = list(csv.reader(open("gpurun_out/r02_verify_raw.csv")))
hdr = rows[0]
def val(name):
    i = hdr.index(name)
    v = rows[2][i].replace(",", "")
    return float(v)
rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
t = val("gpu__time_duration.sum")
out = {"dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "gpu_time_us": t / 1e3 if t > 1e4 else t,
       "source": "ncu --set full --clock-control none, verify_kernel (bf16, launch 16 of bench.py --graph-steps 0, configs[3]), round-2 build; profiles/r02_verify_raw.csv",
       "build_digest": bench.build_digest()}
json.dump(out, open("gpurun_out/verify_dram.json", "w"), indent=1)
print(out)
PY
