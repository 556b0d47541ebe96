"""Per-step timeline under CUDA-graph replay (trace build): verify first-CTA start / last-CTA
end and side kernel start / end, indexed by the committed-step counter."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LAPSSD_LIBRARY"] = os.environ.get("TRACE_LIB") or os.path.join(ROOT, "tools", "liblapssd_trace.so")
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

lib = C.CDLL(os.environ["LAPSSD_LIBRARY"])
N = int(os.environ.get("N", 2048))
tr = synth.make_trace(N, 7, arrival="zero", length="uniform", len_min=512, len_max=4096, beta_ab=(7, 3))
pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=64, variants=16, seed=7, device="cuda")
tab = synth.slab_table(tr, 64, 16, R=64, seed=7)
h = L.Handle(L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9), tr.arrival_us, tr.L_true, tr.L_pred,
             max_batch=512, V=128256, overlap=True)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(512)
for _ in range(3):
    h.laps_step(rows, 512)
torch.cuda.synchronize()
G = 12
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(G):
        h.laps_step(rows, 512)
vt = np.zeros((64, 2), np.uint64)
stt = np.zeros((64, 10), np.uint64)
for mode in ("graph", "eager"):
    torch.cuda.synchronize()
    lib.lapssd_vstep_trace_read(vt.ctypes.data_as(C.c_void_p))
    lib.lapssd_sstep_trace_read(stt.ctypes.data_as(C.c_void_p))
    vsm = np.zeros((64, 3), np.uint64)
    lib.lapssd_vstep_sm_read(vsm.ctypes.data_as(C.c_void_p))
    sit = np.zeros((64, 8, 3), np.uint64)
    lib.lapssd_siter_read(sit.ctypes.data_as(C.c_void_p))
    v0 = int(h.state()["vstep"]) if "vstep" in h.state() else None
    if mode == "graph":
        g.replay()
    else:
        for _ in range(G):
            h.laps_step(rows, 512)
    torch.cuda.synchronize()
    lib.lapssd_vstep_trace_read(vt.ctypes.data_as(C.c_void_p))
    lib.lapssd_sstep_trace_read(stt.ctypes.data_as(C.c_void_p))
    lib.lapssd_vstep_sm_read(vsm.ctypes.data_as(C.c_void_p))
    lib.lapssd_siter_read(sit.ctypes.data_as(C.c_void_p))
    idx = [i for i in range(64) if vt[i, 1] > 0 and vt[i, 0] < 2**63]
    vs = {i: (int(vt[i, 0]), int(vt[i, 1])) for i in idx}
    ss = {i: [int(x) for x in stt[i]] for i in range(64) if stt[i, 4] > 0}
    order = sorted(idx, key=lambda i: vs[i][0])
    t0 = vs[order[0]][0]
    print(f"--- {mode}: per step (us from first verify start): verify start/end, side start/end")
    prev = None
    for i in order:
        a, b = vs[i]
        s_ = ss.get(i, [0] * 10)
        line = "step %2d verify %7.2f .. %6.2f  side %7.2f adm %5.1f mem %5.1f keys %5.1f top %5.1f presort %5.1f merged %5.1f snap %5.1f end %5.1f" % (
            i, (a - t0) / 1e3, (b - a) / 1e3, (s_[0] - t0) / 1e3, (s_[6] - a) / 1e3, (s_[7] - a) / 1e3,
            (s_[8] - a) / 1e3, (s_[9] - a) / 1e3, (s_[1] - a) / 1e3,
            (s_[2] - a) / 1e3, (s_[3] - a) / 1e3, (s_[4] - a) / 1e3)
        if prev is not None:
            line += "  period %.2f" % ((a - prev) / 1e3)
        smid = s_[5]
        line = line.replace("  period", " | period")
        used = [sm for sm in range(192) if (int(vsm[i, sm >> 6]) >> (sm & 63)) & 1]
        line += "  side SM %d (verify used %d SMs%s)" % (smid, len(used), ", SHARED" if smid in used else "")
        prev = a
        print(line)
        its = [(round((int(sit[i, x, 0]) - a) / 1e3, 1), int(sit[i, x, 1]), int(sit[i, x, 2])) for x in range(8) if sit[i, x, 0] > 0]
        print("      merge passes (us, collected, merged):", its)
