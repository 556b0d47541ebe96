"""Per-item timeline (producer issue / consumer start / consumer done) of the two traced
CTAs of the diagnostic build (tools/build_trace.sh with EXTRA="-DLAPSSD_TRACE_A=a -DLAPSSD_TRACE_B=b")."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LAPSSD_LIBRARY"] = os.path.join(ROOT, "tools", "liblapssd_trace.so")
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

lib = C.CDLL(os.environ["LAPSSD_LIBRARY"])
tr = synth.make_trace(2048, 7, arrival="zero", length="uniform", len_min=512, len_max=4096, beta_ab=(7, 3))
pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=64, variants=16, seed=7, device="cuda")
tab = synth.slab_table(tr, 64, 16, R=64, seed=7)
cfg = L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9)
h = L.Handle(cfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=512, V=128256)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(512)
for _ in range(10):
    h.laps_step(rows, 512)
torch.cuda.synchronize()
buf = np.zeros((2, 16, 1024), np.uint64)
ct = np.zeros((10, 160), np.uint64)
lib.lapssd_trace_read(buf.ctypes.data_as(C.c_void_p))
lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
h.laps_step(rows, 512)
torch.cuda.synchronize()
lib.lapssd_trace_read(buf.ctypes.data_as(C.c_void_p))
lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
v0 = ct[0, :147].astype(np.int64).min()
for cta in range(2):
    b = buf[cta].astype(np.int64)
    print(f"--- traced CTA slot {cta}")
    rows_out = []
    for k in range(0, 64):
        ev = {e: (b[e, k] - v0) / 1000 for e in (1, 2, 8, 3, 4) if b[e, k] > 0}
        if ev:
            rows_out.append((k, ev))
    prev = None
    for k, ev in rows_out:
        cs = ev.get(3, float("nan"))
        cd = ev.get(4, float("nan"))
        print("k=%2d P-wait %6.2f P-issued %6.2f C-full %6.2f C-done %6.2f  latency(issue->full) %5.2f" % (
            k, ev.get(1, float("nan")), ev.get(8, float("nan")), cs, cd, cs - ev.get(8, float("nan"))))
