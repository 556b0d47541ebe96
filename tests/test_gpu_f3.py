"""SURVEY 8(f) f3 (Fig. 7 analogue) on the GPU: the Monte-Carlo engine runs
configs[4]-shaped traces to completion; for every request that became perceptible, the
estimate fixed at stabilisation (T~_i, Eq. 6 at L_pred) and the service it then
received (E_i) must equal the oracle's bit for bit, and so must the estimator
report bench.py prints in its --workload mc line (MAPE with the predicted length and with
the true length).  The closed-form pin of the estimator itself is
tests/test_oracle_estimator.py."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MS = 1000
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_mc_estimator_accuracy_equals_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import bench
    import paper_2505_17074_b200 as L
    T, n, V, k, R = 16, 40, 4096, 4, 16
    sched = dict(bench.MC_SCHED, policy=0, seed=0xF3F3)
    rate = synth.mc_rate_for_load(0.8, k, sched["t_ssm_us"], sched["t_llm_us"], len_mu=np.log(60))
    w = synth.make_mc_workload(T, n, 0xF3, rate_per_s=rate, len_mu=np.log(60), len_sigma=0.7, len_min=8,
                               len_max=600, n_buckets=16, variants=4, R=R)
    pool = synth.make_pool("f2", V=V, k=k, dtype="bf16", n_buckets=16, variants=4, seed=0xF3, device="cuda")
    mc = L.MCHandle(L.SchedConfig(**sched), w.offsets, w.arrival_us, w.L_true, w.L_pred, V=V)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device="cuda"))
    mc.select(rows)
    for _ in range(100000):
        if int(mc.step(rows).item()) == 0:
            break
    g = mc.state()[0]
    assert g["done"].all() and mc.check() == 0
    P = pool.numpy()
    parts = {f: [] for f in ("T_total_us", "E_us", "perceptible", "done", "rounds")}
    for t in range(T):
        a, lt, lp, tab = w.trace(t)
        sim = oracle.Sim(oracle.SchedConfig(**sched), a, lt, lp, trace=t)
        Pt = dict(P, slab_tab=np.ascontiguousarray(tab), R=R)
        sel, _ = sim.select(1)
        while not sim.state()["done"].all():
            sim.step(Pt, sel)
        o = sim.state()
        for f in parts:
            parts[f].append(np.asarray(o[f]))
    o = {f: np.concatenate(v) for f, v in parts.items()}
    m = g["perceptible"].astype(bool)
    assert m.sum() > T * n // 2                       # most requests stabilise
    for f in parts:
        assert (np.asarray(g[f]) == o[f]).all(), f"{f} differs"
    rep_g = bench.estimator_accuracy(g, w, sched)
    rep_o = bench.estimator_accuracy(o, w, sched)
    assert rep_g == rep_o
    assert 0.0 < rep_g["mape_with_L_true"] < 1.0
