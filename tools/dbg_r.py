import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import oracle, synth
os.environ["LAPSSD_LIBRARY"] = "/root/repo/tools/liblapssd_trace.so"
import ctypes as C
import paper_2505_17074_b200 as L
lib = C.CDLL(os.environ["LAPSSD_LIBRARY"])
from test_gpu_step import workload, BASE
tr, pool, tab = workload(160, 32000, 4, "f32", 0x5D0002, False)
kw = dict(BASE, policy=0, k=4, seed=11)
B = 16
gcfg = L.SchedConfig(**kw); ocfg = oracle.SchedConfig(**kw)
h = L.Handle(gcfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V)
sim = oracle.Sim(ocfg, tr.arrival_us, tr.L_true, tr.L_pred)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, dtype=torch.int32, device="cuda"))
P = pool.numpy(); P["slab_tab"], P["R"] = tab, tab.shape[1]
sel_o, _ = sim.select(B); h.laps_select(B)
nacc = torch.empty(B, dtype=torch.int32, device="cuda")
prev = None
for step in range(4):
    sel_g = h.sel[:B].cpu().numpy()
    sel_o_before = sel_o.copy()
    st = h.state()
    h.laps_step(rows, B, n_accept=nacc)
    cnt, tok_o, na_o, _ = sim.step(P, sel_o)
    g = nacc.cpu().numpy()
    live = sel_g >= 0
    print("step", step, "sel", sel_g, "oracle sel", sel_o_before, "rounds", st["rounds"][sel_g[live]])
    print("   gpu r", g[live], " oracle r", na_o[live], " was in prev batch:", [int(i in (prev if prev is not None else [])) for i in sel_g[live]])
    prev = sel_g[live]
    dr = np.zeros((16, 4), np.uint64)
    torch.cuda.synchronize()
    lib.lapssd_dbg_rec_read(dr.ctypes.data_as(C.c_void_p))
    for b in range(4):
        print("      brec[%d] key %016x desc.i %d desc.r %d sel %d L %016x" % (b, int(dr[b,0]), int(dr[b,1]) >> 32, int(dr[b,1]) & 0xffffffff, int(dr[b,2]) if int(dr[b,2]) < 2**31 else int(dr[b,2]) - 2**32, int(dr[b,3])))
