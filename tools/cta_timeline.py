"""Per-CTA timeline of one verify launch inside laps_step (diagnostic build, tools/build_trace.sh)."""
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
ct = np.zeros((10, 160), np.uint64)
for rep in range(int(os.environ.get("REPS", "3"))):
    for _ in range(10):
        h.laps_step(rows, 512)
    torch.cuda.synchronize()
    lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
    slt = np.zeros((3, 4096), np.uint64)
    lib.lapssd_slot_trace_read(slt.ctypes.data_as(C.c_void_p))
    si = np.zeros((128, 2), np.uint64)
    ns = C.c_uint(0)
    lib.lapssd_side_trace_read(si.ctypes.data_as(C.c_void_p), C.byref(ns))
    h.laps_step(rows, 512)
    torch.cuda.synchronize()
    lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
    lib.lapssd_side_trace_read(si.ctypes.data_as(C.c_void_p), C.byref(ns))
    lib.lapssd_slot_trace_read(slt.ctypes.data_as(C.c_void_p))
    n = 147
    t = ct[:, :n].astype(np.float64)
    v0 = t[0].min()
    rel = (np.concatenate([t[:5], t[6:9]]) - v0) / 1000.0
    by = t[5] / 1e6

    def q(x):
        return "min %.2f p10 %.2f med %.2f p90 %.2f max %.2f" % (x.min(), np.percentile(x, 10), np.median(x),
                                                               np.percentile(x, 90), x.max())
    print(f"=== rep {rep}")
    sl = slt[:, :512].astype(np.int64)
    v00 = t[0].min()
    for w_, nm in ((0, "update start"), (1, "published"), (2, "sampled")):
        x = (sl[w_][sl[w_] > 0] - v00) / 1000.0
        if len(x):
            print("slot %-13s min %.2f p50 %.2f p90 %.2f p99 %.2f max %.2f (n=%d)" % (nm, x.min(), np.median(x), np.percentile(x, 90), np.percentile(x, 99), x.max(), len(x)))
    late = np.argsort(sl[1])[-8:]
    print("latest published slots:", [(int(b), round((sl[0][b] - v00) / 1000, 2), round((sl[1][b] - v00) / 1000, 2)) for b in late])
    ev = [(round((int(si[x, 0]) - v0) / 1000.0, 2), int(si[x, 1])) for x in range(min(ns.value, 128))]
    print("side events (us from verify start, tag):", ev)
    print("start        ", q(rel[0]))
    print("prod last    ", q(rel[2]))
    print("cons last    ", q(rel[3]))
    print("fin last rdy ", q(rel[4]))
    print("fin y        ", q(rel[5]))
    print("fin upd      ", q(rel[6]))
    print("fin done     ", q(rel[7]))
    print("end          ", q(rel[1]))
    crit = np.argsort(rel[1])[-5:]
    for c in crit:
        print("  late CTA %3d: rdy %.2f y %.2f upd %.2f done %.2f end %.2f cons %.2f" % (c, rel[4][c], rel[5][c], rel[6][c], rel[7][c], rel[1][c], rel[3][c]))
    print("MB per CTA   ", q(by), " total %.1f MB" % by.sum())
    rate = by / np.maximum(rel[3] - rel[0], 1e-3) * 1e3  # GB/s per CTA
    print("GB/s per CTA ", q(rate), " aggregate %.0f GB/s to last consumer" % (by.sum() / rel[3].max() * 1e3))
    smid = ct[9, :n].astype(np.int64)
    order = np.argsort(rate)
    print("slowest CTAs (cta/sm/GB/s):", [(int(c), int(smid[c]), round(float(rate[c]), 1)) for c in order[:20]])
    print("fastest CTAs (cta/sm/GB/s):", [(int(c), int(smid[c]), round(float(rate[c]), 1)) for c in order[-8:]])
    cc = np.corrcoef(by, rel[3])[0, 1]
    print("corr(bytes, cons_last) %.2f" % cc)
