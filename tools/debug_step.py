import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17074_b200 as L, synth
tr = synth.make_trace(160, 0x5D0002, arrival="poisson", rate_per_s=80.0, len_mu=np.log(40), len_sigma=0.6,
                      len_min=4, len_max=400, beta_ab=(4, 2), drift=False)
pool = synth.make_pool("f2", V=32000, k=4, dtype="f32", n_buckets=8, variants=3, seed=1, device="cuda")
tab = synth.slab_table(tr, 8, 3, R=16, seed=1)
h = L.Handle(L.SchedConfig(k=4, seed=11), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=16, V=32000)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(16)
torch.cuda.synchronize()
print("sel before", h.sel.cpu().numpy())
nacc = torch.full((16,), -7, dtype=torch.int32, device="cuda")
h.laps_step(rows, 16, n_accept=nacc)
torch.cuda.synchronize()
print("nacc", nacc.cpu().numpy())
print("sel after", h.sel.cpu().numpy())
try:
    print("flags", h.check())
except Exception as e:
    print("check:", e)
