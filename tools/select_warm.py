"""Select-kernel time in a tight loop (warm caches) vs. inside the streaming step."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

tr = synth.make_trace(2048, 7, arrival="zero", length="uniform", len_min=512, len_max=4096, beta_ab=(7, 3))
h = L.Handle(L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9), tr.arrival_us, tr.L_true, tr.L_pred,
             max_batch=512, V=128256)
for _ in range(5):
    h.laps_select(512)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    h.laps_select(512)
e1.record()
torch.cuda.synchronize()
print("laps_select warm loop: %.2f us per call" % (e0.elapsed_time(e1) * 1000 / 200))
# same, with an L2-flushing copy between calls
buf = torch.empty(512 * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda")
buf2 = torch.empty_like(buf)
tot = 0.0
for _ in range(50):
    buf2.copy_(buf)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); h.laps_select(512); b.record()
    torch.cuda.synchronize()
    tot += a.elapsed_time(b)
print("laps_select after 1 GB copy (cold L2): %.2f us per call" % (tot * 1000 / 50))
