"""configs[4] readings sweep (tooling): mean JCT of LAPS-SD under alternative readings of
the paper's silent points (AMB-14 placement, AMB-15 pin rule) and queue counts K (the
Fig. 6 axis, no switching cost), against FCFS / LP-SJF / LAS on the same traces.
Usage: python tools/mc_readings.py [n_traces]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048


class A:
    mc_traces, mc_n, mc_variants = T, 512, 256


dev = torch.device("cuda", 0)
w, pool = bench.build_mc(A, 0, 1, dev)
c = synth.CONFIGS["c5"]
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device=dev))


def run(**kw):
    cfg = L.SchedConfig(**dict(bench.MC_SCHED, seed=c["seed"], **kw))
    mc = L.MCHandle(cfg, w.offsets, w.arrival_us, w.L_true, w.L_pred, V=c["V"])
    mc.select(rows)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(64):
            act = mc.step(rows)
    steps = 0
    while True:
        g.replay()
        steps += 64
        if int(act.item()) == 0 or steps > 2_000_000:
            break
    st = mc.state()[0]
    jct = (st["C_us"] - w.arrival_us).astype(np.float64).mean() / 1e3
    del mc
    return float(jct)


out = {}
t0 = time.time()
for name, kw in [("FCFS", dict(policy=1)), ("LP-SJF", dict(policy=2)), ("LAS", dict(policy=3)),
                 ("LAPS-SD", dict(policy=0)), ("LAPS-SD pin_on_stable", dict(policy=0, pin_rule=1)),
                 ("LAPS-SD placement=stay", dict(policy=0, placement=1)),
                 ("LAPS-SD gamma=3", dict(policy=0, gamma=3, delta=0.1))] + \
        [(f"LAPS-SD K={K}", dict(policy=0, K=K)) for K in (1, 2, 3, 6, 8, 10)]:
    out[name] = run(**kw)
    print(f"{name:28s} mean JCT {out[name]:9.1f} ms", flush=True)
print(json.dumps({"traces": T, "requests_per_trace": 512, "mean_jct_ms": out, "seconds": time.time() - t0}))
