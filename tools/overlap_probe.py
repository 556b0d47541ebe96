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
ct = np.zeros((2, 160), np.uint64); sel = np.zeros(16, np.uint64)
lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
for step in range(3):
    h.laps_step(rows, 512)
    torch.cuda.synchronize()
    lib.lapssd_cta_trace_read(ct.ctypes.data_as(C.c_void_p))
    lib.lapssd_sel_trace_read(sel.ctypes.data_as(C.c_void_p))
    st = ct[0][ct[0] < 2**63].astype(np.int64); en = ct[1][ct[1] > 0].astype(np.int64)
    t0 = min(st.min(), int(sel[8]))
    print(f"step {step}: verify CTAs start {(st.min()-t0)/1e3:.1f}..{(st.max()-t0)/1e3:.1f} end {(en.min()-t0)/1e3:.1f}..{(en.max()-t0)/1e3:.1f} us; side kernel {(int(sel[8])-t0)/1e3:.1f}..{(int(sel[9])-t0)/1e3:.1f} us; n_cta={len(st)}")
    it = np.zeros((128, 2), np.uint64); nn = np.zeros(1, np.uint32)
    lib.lapssd_side_trace_read(it.ctypes.data_as(C.c_void_p), nn.ctypes.data_as(C.c_void_p))
    k = min(int(nn[0]), 128)
    print("  side iters (us, m):", [(round((int(it[i][0]) - t0) / 1e3, 1), int(it[i][1])) for i in range(k)])
    try:
        print("  flags", h.check())
    except Exception as e:
        print("  ", e)
