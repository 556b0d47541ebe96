"""the paper's queue-count experiment (Fig. 6 analogue) with the
switching cost of P:73 / P:102 (DESIGN.md AMB-24, AMB-32), on the Monte-Carlo engine.

Workload: T independent traces; each trace is a burst of N requests that all arrive at
t = 0 and are served one at a time (batch 1), as in the paper's "number of requests
varied from 10 to 50".  Two request profiles stand in for the paper's datasets:
"short" (prompt median 64, output lengths lognormal(ln 128, 0.8)) and "long" (prompt
median 512, output lognormal(ln 384, 0.6)) -- the paper attributes the dataset
dependence to "longer average input and output lengths".  Rows: F2 slab pool,
V = 32,000, k = 4, bf16, Beta(4, 2) acceptance (configs[4]'s pool).

Switching cost (AMB-32): c0 = 0 and c1 calibrated to P:102's "switching a request with an
output length of 500 tokens adds a 14.21% overhead to the total LLM inference time":
c1 * 500 = 0.1421 * (500 / tau) * T_LLM, tau = E[tokens per round] at the pool's mean
acceptance, i.e. c1 = 0.1421 * T_LLM / tau; swept at x0, x0.25, x1 of that value.

Thresholds (S_j^up = M^(j-1) S_1^up), two readings of what "changing the number
of queues" keeps fixed (AMB-33): "fixed-M" -- M = 2 and S_1^up = 4 c_round as in every
other run, so queues whose thresholds exceed every request's service stay empty; and
"fixed-span" -- S_1^up = 4 c_round and the last finite threshold S_{K-1}^up = 64 c_round
(~ the mean service of the long profile) fixed, M = 16^(1/(K-2)), so more queues mean
finer demotion steps over the same range.

For every (thresholds, profile, N, c1) the mean JCT (C_i - r_i) of LAPS-SD at K = 2..10, LAS at
the same K, and FCFS / LP-SJF, on the SAME traces and rows (common random numbers).  Trace
0 of every run is replayed on the oracle and its per-request C_i must match exactly.

Usage: python tools/f2_k_sweep.py [T] [out.json]"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (cross-check of trace 0 only)
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "f2_k_sweep.json")
k, V, T_SSM, T_LLM = 4, 32000, 1000, 10_000
BASE = dict(s1_up_us=4 * (k * T_SSM + T_LLM), M=2.0, gamma=5, delta=0.05, k=k, t_ssm_us=T_SSM,
            t_llm_us=T_LLM, placement=0, pin_rule=0, seed=0x5D00F2)
beta = 4.0 / 6.0
tau = float(synth.tokens_per_round(np.array([beta]), k)[0])
C1_PAPER = 0.1421 * T_LLM / tau                     # us per token of context (AMB-32)
PROFILES = {"short": dict(prompt_median=64, len_mu=math.log(128), len_sigma=0.8),
            "long": dict(prompt_median=512, len_mu=math.log(384), len_sigma=0.6)}

dev = torch.device("cuda", 0)
pool = synth.make_pool("f2", V=V, k=k, dtype="bf16", n_buckets=64, variants=32, seed=0x5D00F2, device=dev)
P = pool.numpy()


def workload(profile, N, seed):
    pr = PROFILES[profile]
    w = synth.make_mc_workload(T, N, seed, rate_per_s=1.0, len_mu=pr["len_mu"], len_sigma=pr["len_sigma"],
                               len_min=8, len_max=4096, n_buckets=64, variants=32, R=16)
    w.arrival_us[:] = 0                              # a burst: all N arrive at t = 0
    prompt = synth.prompt_lengths(T * N, seed, median=pr["prompt_median"], lo=8, hi=8192)
    return w, prompt


def thresholds(mode, K):
    if mode == "fixed-M" or K <= 2:
        return {}
    return dict(M=16.0 ** (1.0 / (K - 2)))


def run(w, prompt, rows, **kw):
    cfg = L.SchedConfig(**dict(BASE, **kw))
    mc = L.MCHandle(cfg, w.offsets, w.arrival_us, w.L_true, w.L_pred, V=V, prompt=prompt)
    mc.select(rows)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(64):
            act = mc.step(rows)
    steps = 0
    while True:
        g.replay()
        steps += 64
        if int(act.item()) == 0 or steps > 4_000_000:
            break
    st = mc.state()[0]
    assert st["done"].all()
    C = st["C_us"].copy()
    jct = (C - w.arrival_us).astype(np.float64)
    assert mc.check() == 0
    del mc
    return float(jct.mean() / 1e3), int(st["switch_total_us"]), C, steps


def oracle_trace0(w, prompt, C_gpu, **kw):
    a, lt, lp, tab = w.trace(0)
    N = len(a)
    sim = oracle.Sim(oracle.SchedConfig(**dict(BASE, **kw)), a, lt, lp, trace=0, prompt=prompt[:N])
    Pt = dict(P, slab_tab=np.ascontiguousarray(tab), R=tab.shape[1])
    sel, _ = sim.select(1)
    while not sim.state()["done"].all():
        sim.step(Pt, sel)
    return bool((sim.state()["C_us"] == C_gpu[:N]).all())


res = {"traces": T, "k": k, "V": V, "T_SSM_us": T_SSM, "T_LLM_us": T_LLM, "tau": tau,
       "c1_paper_us_per_token": C1_PAPER, "profiles": PROFILES, "runs": []}
t0 = time.time()
for mode in ("fixed-M", "fixed-span"):
  for profile in PROFILES:
    for N in (10, 30):
        w, prompt = workload(profile, N, 0x5D00F2 + 7 * N + (0 if profile == "short" else 1))
        rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device=dev))
        for scale in (0.0, 0.25, 1.0):
            c1 = int(round(scale * C1_PAPER))
            sw = dict(switch_c0_us=0, switch_c1_us=c1)
            entry = {"thresholds": mode, "profile": profile, "N": N, "c1_scale": scale, "c1_us": c1,
                     "laps_sd": {}, "las": {}}
            ok = True
            for K in range(2, 11):
                th = thresholds(mode, K)
                j, swt, C, _ = run(w, prompt, rows, policy=0, K=K, **sw, **th)
                entry["laps_sd"][K] = {"mean_jct_ms": j, "switch_ms_per_request": swt / 1e3 / (T * N)}
                if K in (2, 6, 10) or mode == "fixed-span":
                    ok &= oracle_trace0(w, prompt, C, policy=0, K=K, **sw, **th)
                j, swt, C, _ = run(w, prompt, rows, policy=3, K=K, **sw, **th)
                entry["las"][K] = {"mean_jct_ms": j, "switch_ms_per_request": swt / 1e3 / (T * N)}
            for name, pol in (("fcfs", 1), ("lp_sjf", 2)):
                j, swt, C, _ = run(w, prompt, rows, policy=pol, K=4, **sw)
                entry[name] = {"mean_jct_ms": j, "switch_ms_per_request": swt / 1e3 / (T * N)}
            best = min(entry["laps_sd"], key=lambda K: entry["laps_sd"][K]["mean_jct_ms"])
            entry["laps_sd_best_K"] = best
            entry["oracle_trace0_exact"] = ok
            res["runs"].append(entry)
            line = " ".join(f"{K}:{entry['laps_sd'][K]['mean_jct_ms']:.0f}" for K in range(2, 11))
            print(f"{mode:10s} {profile:5s} N={N:2d} c1={c1:5d}us  LAPS-SD K->JCT ms {line}  best K={best}  "
                  f"LAS(K=4) {entry['las'][4]['mean_jct_ms']:.0f}  FCFS {entry['fcfs']['mean_jct_ms']:.0f}  "
                  f"LP-SJF {entry['lp_sjf']['mean_jct_ms']:.0f}  oracle trace0 {'ok' if ok else 'MISMATCH'}",
                  flush=True)
res["seconds"] = time.time() - t0
os.makedirs(os.path.dirname(OUT), exist_ok=True)
json.dump(res, open(OUT, "w"), indent=1)
print(f"wrote {OUT} ({res['seconds']:.0f} s)")
