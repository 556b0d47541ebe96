"""Per-unit timeline of the f1 lazy logits kernel (diagnostic build: tools/build_variant.sh
lazytr -DLAPSSD_LAZY_TRACE).  Runs the bench's logits workload (B=512, V=128,256, k=8) and
summarises one step: span, units in flight over time, claim waits, unit durations."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib_path = os.environ.setdefault("LAPSSD_LIBRARY", os.path.join(ROOT, "tools", "variants", "lib_lazytr.so"))
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

lib = C.CDLL(lib_path)
dev = torch.device("cuda", 0)
B, k, V = int(os.environ.get("B", 512)), 8, 128256
pool = synth.make_logits_pool(V, k, "bf16", n_buckets=64, variants=16, seed=synth.CONFIGS["c4"]["seed"], device=dev)
gen = torch.Generator(device=dev)
gen.manual_seed(1000)
req = torch.arange(B, device=dev, dtype=torch.int32)
ws = torch.empty(L.spec_verify_logits_workspace_bytes(B, k, V, "bf16"), dtype=torch.uint8, device=dev)
buf = np.zeros((16384, 4), np.uint64)
n = C.c_uint(0)
out = []
for step in range(6):
    slab = torch.randint(0, pool.S, (B,), generator=gen, device=dev, dtype=torch.int32)
    rnd = torch.randint(0, 1 << 12, (B,), generator=gen, device=dev, dtype=torch.int32)
    torch.cuda.synchronize()
    lib.lapssd_lazy_trace_read(buf.ctypes.data_as(C.c_void_p), C.byref(n))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tok, na, z = L.spec_verify_logits(pool.p, pool.q, pool.draft, req, rnd, 0x5D0F1, slab=slab, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    lib.lapssd_lazy_trace_read(buf.ctypes.data_as(C.c_void_p), C.byref(n))
    if step < 3:
        continue
    m = min(n.value, 16384)
    t = buf[:m].copy()
    code = (t[:, 0] & 0x7FFFFFFF).astype(np.int64)
    resid = ((t[:, 0] >> 31) & 1).astype(bool)
    sm = (t[:, 0] >> 32).astype(np.int64)
    t0 = t[:, 1].min()
    claim, got, end = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3
    rows = 2 * k + 1
    ri = code % rows
    pos = np.where(code >= B * rows, -1, np.where(ri <= k, ri, ri - k - 1))   # -1: residual parts
    span = end.max()
    bins = np.arange(0, span + 10, 10.0)
    act = [int(((got < b + 10) & (end > b)).sum()) for b in bins]
    r = na.cpu().numpy()
    rec = {"step": step, "event_ms": e0.elapsed_time(e1), "units": m, "span_us": float(span),
           "rows_needed": int((2 * np.minimum(r + 1, k) + (r == k)).sum()),
           "wait_us_total": float((got - claim).sum()), "busy_us_total": float((end - got).sum()),
           "ctas_sms": int(len(np.unique(sm))),
           "unit_us_mean_norm": float((end - got)[pos >= 0].mean()),
           "unit_us_mean_resid": float((end - got)[pos < 0].mean()) if (pos < 0).any() else None,
           "resid_start_us": [float(got[pos < 0].min()), float(np.median(got[pos < 0])), float(got[pos < 0].max())]
           if (pos < 0).any() else None,
           "pos_start_us": {int(j): [float(got[pos == j].min()), float(np.median(got[pos == j])), float(got[pos == j].max())]
                            for j in range(k + 1) if (pos == j).any()},
           "active_per_10us": act,
           "r_hist": np.bincount(r, minlength=k + 1).tolist()}
    out.append(rec)
    print(json.dumps(rec))
