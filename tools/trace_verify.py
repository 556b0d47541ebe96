"""Timeline of one verify launch from the diagnostic build (tools/build_trace.sh)."""
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
pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=64, variants=2, seed=7, device="cuda")
tab = synth.slab_table(tr, 64, 2, R=64, seed=7)
cfg = L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9)
h = L.Handle(cfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=512, V=128256)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(512)
for _ in range(8):
    h.laps_step(rows, 512)
torch.cuda.synchronize()
buf = np.zeros((2, 16, 1024), np.uint64)
ct = np.zeros((2, 160), np.uint64)
lib.lapssd_trace_read(buf.ctypes.data_as(C.c_void_p))
lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
h.laps_step(rows, 512)
torch.cuda.synchronize()
lib.lapssd_trace_read(buf.ctypes.data_as(C.c_void_p))
lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
names = {1: "P-wait", 2: "P-free", 8: "P-issued", 3: "C-full", 4: "C-done", 5: "F-pop", 6: "F-ready", 7: "F-done",
         9: "f-Z", 10: "f-seg", 11: "f-y", 12: "f-out", 13: "f-upd"}
for cta in range(2):
    b = buf[cta].astype(np.int64)
    t0 = b[b > 0].min()
    print(f"--- CTA {0 if cta == 0 else 74}")
    for k in range(0, 60):
        row = [(names[e], (b[e, k] - t0) / 1000) for e in (1, 2, 8, 3, 4) if b[e, k] > 0]
        if row:
            print(k, " ".join(f"{n}={t:.2f}" for n, t in row))
    fin = [(names[e], x, round((b[e, x] - t0) / 1000, 2)) for e in (5, 6, 9, 10, 11, 12, 13, 7) for x in range(1024) if b[e, x] > 0]
    print("finisher:", sorted(fin, key=lambda z: z[2])[:40])
allb = buf.astype(np.int64)
t0 = allb[allb > 0].min()
sel = np.zeros(16, np.uint64)
lib.lapssd_sel_trace_read(sel.ctypes.data_as(C.c_void_p))
t = sel.astype(np.int64)
print("select_final phases (us):", [(i, round((t[i] - t[0]) / 1000, 2)) for i in range(6)])
fs = np.zeros(8, np.uint64)
lib.lapssd_fs_trace_read(fs.ctypes.data_as(C.c_void_p))
starts = ct[0][ct[0] < 2**63].astype(np.int64); ends = ct[1][ct[1] > 0].astype(np.int64)
v0 = starts.min()
print("verify CTAs: first start 0, last start %.2f us, first end %.2f, last end %.2f; select_final start %.2f end %.2f" % (
    (starts.max() - v0) / 1000, (ends.min() - v0) / 1000, (ends.max() - v0) / 1000, (t[0] - v0) / 1000, (t[5] - v0) / 1000))
f = fs.astype(np.int64)
print("fused final select phases from verify start (us):", [round((f[i] - v0) / 1000, 2) for i in range(7)])
