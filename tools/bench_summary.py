"""One-line summary of a bench.py JSON log (tooling)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "NO JSON:", open(path).read()[-1500:])
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    err = ("  DEVICE ERROR: " + d["device_error"]) if d.get("device_error") else ""
    print("%s: value %.4g %s  ms/step %.4f  verify %.4f ms  frac %.3f  clocks %s  launches %s  e2e %s  cpu %s%s" % (
        path, d["value"], d.get("unit", ""), d.get("ms_per_step", 0),
        r.get("verify_interval_ms", r.get("verify_ms_avg", 0)) or 0,
        r.get("frac", 0) or 0, d.get("clocks", {}).get("sm_mhz"), d.get("gpu_launches"),
        (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), err))
