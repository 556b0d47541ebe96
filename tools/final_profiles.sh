#!/bin/bash
# Final ncu evidence for THIS build: verify full capture (-> verify_dram.json), launch list,
# side select, instruction counts of the ALU-bound kernels (-> alu_counts.json).
cd "$(dirname "$0")/.."
bash tools/profile_r02.sh
bash tools/alu_counts.sh
python - <<'PY'
import csv, collections, statistics, json, sys
sys.path.insert(0, ".")
import bench
def agg(f):
    rows = [r for r in csv.reader(open(f)) if r]
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]; ik = hdr.index("Kernel Name"); im = hdr.index("Metric Name"); iv = hdr.index("Metric Value")
    iu = hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hi + 1:]:
        try: d[r[ik].split("(")[0]][r[im]].append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1))
        except Exception: pass
    return {k: {m: statistics.mean(v) for m, v in mm.items()} for k, mm in d.items()}
lg = agg("gpurun_out/r02_logits_counts.csv"); tr = agg("gpurun_out/r02_tree_counts.csv")
out = {"build_digest": bench.build_digest(),
       "source": "ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_*,sm__cycles_elapsed.avg --clock-control none (tools/alu_counts.sh), profiles/r02_logits_counts.csv, profiles/r02_tree_counts.csv",
       "peak_note": "B200: 148 SMs x 4 SM sub-partitions x 1 warp instruction issued per clock = 592 warp instructions per clock",
       "logits": {"workload": {"B": 512, "V": 128256, "k": 8}, "warp_inst_per_step": sum(v["smsp__inst_executed.sum"] for v in lg.values()),
                  "dram_bytes_per_step": sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in lg.values()),
                  "per_kernel": {k: v["smsp__inst_executed.sum"] for k, v in lg.items()}},
       "tree": {"workload": {"B": 512, "V": 128256, "nodes": 16, "max_children": 3},
                "warp_inst_per_step": sum(v["smsp__inst_executed.sum"] for v in tr.values())}}
json.dump(out, open("gpurun_out/alu_counts.json", "w"), indent=1)
print(out["logits"]["warp_inst_per_step"], out["tree"]["warp_inst_per_step"])
PY
