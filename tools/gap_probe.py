"""Inter-step timeline under CUDA-graph replay (trace build): verify start of step t+1
relative to the side kernel's end of step t."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LAPSSD_LIBRARY"] = os.path.join(ROOT, "tools", "liblapssd_trace.so")
import paper_2505_17074_b200 as L, synth
lib = C.CDLL(os.environ["LAPSSD_LIBRARY"])
tr = synth.make_trace(2048, 7, arrival="zero", length="uniform", len_min=512, len_max=4096, beta_ab=(7, 3))
pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=16, variants=2, seed=7, device="cuda")
tab = synth.slab_table(tr, 16, 2, R=64, seed=7)
h = L.Handle(L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=512, V=128256)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(512)
for _ in range(3):
    h.laps_step(rows, 512)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(10):
        h.laps_step(rows, 512)
vs = np.zeros(64, np.uint64); se = np.zeros(64, np.uint64)
for mode in ("graph", "eager"):
    lib.lapssd_vstart_read(vs.ctypes.data_as(C.c_void_p)); lib.lapssd_send_read(se.ctypes.data_as(C.c_void_p))
    torch.cuda.synchronize()
    if mode == "graph":
        g.replay()
    else:
        for _ in range(10):
            h.laps_step(rows, 512)
    torch.cuda.synchronize()
    lib.lapssd_vstart_read(vs.ctypes.data_as(C.c_void_p)); lib.lapssd_send_read(se.ctypes.data_as(C.c_void_p))
    v = vs[:10].astype(np.int64); s = se[:10].astype(np.int64)
    print(mode, "step period (us):", np.round(np.diff(v) / 1e3, 1))
    print(mode, "verify start -> side end (us):", np.round((s - v) / 1e3, 1))
    print(mode, "side end -> next verify start (us):", np.round((v[1:] - s[:-1]) / 1e3, 1))
