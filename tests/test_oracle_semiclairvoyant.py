"""Pins for the semi-clairvoyant core of LAPS-SD, run through the token-level simulation
(``orc_sim``: select -> verify -> update -> clock), not the job-level schedule.

* Fig. 1(c) ("if we have information about both the request length and the
  acceptance rate ... leads to the optimal scheduling"): every request perceptible at
  arrival with A = its rate.  The schedule must be the brute-force optimum of Eq. (2)
  (order R3, R1, R2, mean JCT 450 ms); FCFS / LP-SJF through the same simulation give
  the paper's printed 583 / 683 ms.
* within a queue, perceptible requests come first, ordered SJF on the remaining
  estimate (AMB-12); non-perceptible ones follow in FCFS order.
* a request that becomes perceptible is moved to the queue of its estimate
  (AMB-14), up or down; ``placement = STAY`` keeps the attained-service queue.

Deterministic emulation of the Fig. 1 job model: rounds verify ONE candidate (k = 1) on
F1 rows with beta = 0 (draft and target supports are disjoint, so every draft is
rejected and every round emits exactly one token from the residual), each round costs
t_tok = 10 ms (the Fig. 1 cost model, no SSM time).  A request "of L tokens at
rate alpha" then needs L / alpha candidate rounds: L_true = L / alpha, and the
scheduler's estimate is T~ = L_pred t_tok / A with L_pred = L, A = alpha (the Fig. 1
model, AMB-31).  tests/test_oracle_mutants.py checks that a reversed SJF order,
perceptible requests placed after non-perceptible ones, and bottom-queue placement
each fail a test here.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from conftest import golden

MS = 1000


def read_fig1():
    vals = {}
    for line in open(golden("fig1.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        vals[f[0]] = f[1:]
    return vals


def beta0_pool(n, V=16, seed=0):
    """One F1 slab per request with beta = 0 at every position (k = 1)."""
    g = torch.Generator()
    g.manual_seed(seed)
    ps, qs, ds = [], [], []
    for _ in range(n):
        p, q, d = synth.f1_rows(V, 1, [0.0, 0.0], g)
        ps.append(p), qs.append(q), ds.append(d)
    P = dict(p=synth.to_numpy_rows(torch.stack(ps)), q=synth.to_numpy_rows(torch.stack(qs)),
             draft=torch.stack(ds).numpy().astype(np.int32))
    P["slab_tab"] = np.repeat(np.arange(n, dtype=np.int32)[:, None], 4, 1)
    P["R"] = 4
    return P


def fig1_cfg(policy, **kw):
    base = dict(policy=policy, K=1, s1_up_us=1000 * MS, M=2.0, gamma=3, delta=0.0, k=1,
                cost_model=oracle.COST_FIG1, t_tok_us=10 * MS, t_ssm_us=0, t_llm_us=0, seed=5)
    base.update(kw)
    return oracle.SchedConfig(**base)


def run(sim, P, B=1, hook=None):
    """Steps to completion; returns the sequence of batches (lists of ids)."""
    sel, _ = sim.select(B)
    order = [list(sel[sel >= 0])]
    for _ in range(10_000):
        if sim.state()["done"].all():
            return order
        cnt, tok, na, _ = sim.step(P, sel)
        assert (na[sel >= 0] == 0).all() if (sel >= 0).any() else True   # beta = 0: r = 0
        if hook:
            hook(sim)
        order.append(list(sel[sel >= 0]))
    raise AssertionError("simulation did not finish")


def service_order(order):
    seen = []
    for b in order:
        for i in b:
            if not seen or seen[-1] != i:
                seen.append(int(i))
    return seen


def fig1_requests():
    v = read_fig1()
    names = ("R1", "R2", "R3")
    L = np.array([int(v[r][0]) for r in names])
    alpha = np.array([float(v[r][1]) for r in names])
    cand = np.round(L / alpha).astype(np.int32)          # candidates to verify
    return v, L, alpha, cand


def test_fig1_model_estimate_is_candidates_times_t_tok():
    v, L, alpha, cand = fig1_requests()
    assert list(cand) == [20, 50, 15]                    # "20 candidate tokens"
    for l, a, c in zip(L, alpha, cand):
        assert oracle.fig1_est(l, a, 10 * MS) == c * 10 * MS
    assert oracle.fig1_est(10, 0.0, 10 * MS) == 2**64 - 1    # A = 0: no finite estimate


@pytest.mark.parametrize("policy,printed", [(oracle.POL_FCFS, "fcfs_avg_ms"),
                                            (oracle.POL_LPSJF, "sjf_avg_ms")])
def test_fig1_fcfs_lpsjf_token_level_match_paper(policy, printed):
    v, L, alpha, cand = fig1_requests()
    P = beta0_pool(3)
    sim = oracle.Sim(fig1_cfg(policy), np.zeros(3, np.int64), cand, L)
    order = run(sim, P)
    st = sim.state()
    assert (st["acc_tok"] == cand).all()
    want = [0, 1, 2] if policy == oracle.POL_FCFS else [1, 0, 2]
    assert service_order(order) == want
    assert round(st["C_us"].mean() / MS) == int(v[printed][0])    # 583 / 683 ms
    assert st["C_us"].sum() == {oracle.POL_FCFS: 1_750_000, oracle.POL_LPSJF: 2_050_000}[policy]


def test_fig1_clairvoyant_laps_sd_is_optimal_through_the_simulation():
    v, L, alpha, cand = fig1_requests()
    P = beta0_pool(3)
    sim = oracle.Sim(fig1_cfg(oracle.POL_LAPSSD), np.zeros(3, np.int64), cand, L)
    for i in range(3):
        sim.make_perceptible(i, alpha[i])
    st0 = sim.state()
    assert list(st0["T_total_us"]) == [200 * MS, 500 * MS, 150 * MS]
    order = run(sim, P)
    st = sim.state()
    assert service_order(order) == [2, 0, 1]                      # R3, R1, R2
    assert list(st["C_us"]) == [350 * MS, 850 * MS, 150 * MS]
    best, best_order, _ = oracle.brute_force(cand.astype(np.int64) * 10 * MS)
    assert st["C_us"].sum() == best == 1_350_000                  # 450 ms: the optimum
    assert list(best_order) == [2, 0, 1]
    assert st["pinned"].all()                                     # selected while perceptible
    # no preemption: each request runs in one contiguous stretch
    assert [i for b in order for i in b] == [2] * 15 + [0] * 20 + [1] * 50


def test_perceptible_first_then_fcfs_within_a_queue():
    """one queue holding two non-perceptible requests (ids 0, 1) and two
    perceptible ones (ids 2, 3, estimates 300 ms and 100 ms): perceptible first,
    shortest estimate first, then the non-perceptible ones in arrival order."""
    P = beta0_pool(4)
    L = np.array([5, 5, 30, 10], np.int32)
    sim = oracle.Sim(fig1_cfg(oracle.POL_LAPSSD), np.zeros(4, np.int64), L, L)
    sim.make_perceptible(2, 1.0)
    sim.make_perceptible(3, 1.0)
    keys = sim.state()["key"]
    order = run(sim, P)
    assert service_order(order) == [3, 2, 0, 1]
    st = sim.state()
    assert list(st["C_us"]) == [450 * MS, 500 * MS, 400 * MS, 100 * MS]
    del keys


def test_perceptible_preempts_running_non_perceptible_in_same_queue():
    """AMB-16 / P:202: a non-perceptible request runs; once a same-queue request becomes
    perceptible it is served next (perceptible first), the running one waits."""
    P = beta0_pool(2)
    L = np.array([10, 4], np.int32)
    sim = oracle.Sim(fig1_cfg(oracle.POL_LAPSSD), np.zeros(2, np.int64), L, L)
    state = {"t": 0}

    def hook(s):
        state["t"] += 1
        if state["t"] == 3:
            s.make_perceptible(1, 1.0)

    order = run(sim, P, hook=hook)
    flat = [int(i) for b in order for i in b]
    # the hook runs after the 3rd step's select, so request 0 has 4 rounds when the
    # next select sees request 1 perceptible
    assert flat == [0] * 4 + [1] * 4 + [0] * 6
    assert list(sim.state()["C_us"]) == [140 * MS, 80 * MS]


def test_sjf_uses_the_remaining_estimate():
    """AMB-12: two perceptible requests, keyed on T~(L_pred - tokens so far): request 0
    (12 predicted, 8 already emitted: 40 ms left) goes before request 1 (6 predicted,
    60 ms), although its total estimate (120 ms) is the larger."""
    P = beta0_pool(2)
    L = np.array([12, 6], np.int32)
    sim = oracle.Sim(fig1_cfg(oracle.POL_LAPSSD), np.zeros(2, np.int64), L, L)
    sel, _ = sim.select(1)
    assert list(sel) == [0]
    for _ in range(8):                              # request 0 runs 8 rounds non-perceptible
        sim.step(P, sel)
        assert list(sel) == [0]
    sim.make_perceptible(0, 1.0)
    sim.make_perceptible(1, 1.0)
    st = sim.state()
    assert list(st["T_total_us"]) == [120 * MS, 60 * MS]
    # the keys of the coming select: secondary field = T~_rem
    sim.step(P, sel)
    assert list(sel) == [0]
    st = sim.state()
    sec = (st["key"].astype(np.uint64) >> np.uint64(24)) & np.uint64(0xFFFFFFFF)
    assert list(sec) == [30 * MS, 60 * MS]           # 3 left for 0 after this round, 6 for 1
    flat = []
    while not sim.state()["done"].all():
        sim.step(P, sel)
        flat += [int(i) for i in sel if i >= 0]
    assert flat == [0] * 2 + [1] * 6      # batches chosen after rounds 10..17
    assert list(sim.state()["C_us"]) == [120 * MS, 180 * MS]


@pytest.mark.parametrize("placement", [0, 1])
def test_placement_moves_to_the_queue_of_the_estimate(placement):
    """P:148 / AMB-14.  Thresholds 50 / 100 / 200 ms (K = 4).  A request that has run
    70 ms (attained-service queue 1) and stabilises with estimate 46.666 ms moves UP to
    queue 0 (by estimate); with placement = STAY it stays in queue 1.  Natural
    stabilisation: constant rate 0.5 for gamma = 5 rounds (Eq. 6)."""
    cfg = oracle.SchedConfig(policy=oracle.POL_LAPSSD, K=4, s1_up_us=50 * MS, M=2.0, gamma=5,
                             delta=0.05, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS,
                             placement=placement)
    sim = oracle.Sim(cfg, [0], [10**6], [10])
    sim.select(1)
    levels = []
    for t in range(5):
        sim.update([0], [2])
        levels.append(int(sim.state()["level"][0]))
        sim.select(1)
    st = sim.state()
    assert st["perceptible"][0] and st["A"][0] == 0.5
    assert st["T_total_us"][0] == 46_666                    # Eq. 6: 10 * 14 / 3 ms
    assert levels[:4] == [0, 0, 0, 1]                       # E = 56 ms >= 50 ms at round 4
    assert levels[4] == (0 if placement == 0 else 1)


def test_placement_of_clairvoyant_requests_by_estimate():
    """P:148 with estimates spanning the queues: 40 ms -> queue 0, 70 -> 1, 150 -> 2,
    900 ms -> 3 (the unbounded bottom queue)."""
    cfg = fig1_cfg(oracle.POL_LAPSSD, K=4, s1_up_us=50 * MS)
    L = np.array([4, 7, 15, 90], np.int32)
    sim = oracle.Sim(cfg, np.zeros(4, np.int64), L, L)
    for i in range(4):
        sim.make_perceptible(i, 1.0)
    st = sim.state()
    assert list(st["T_total_us"]) == [40 * MS, 70 * MS, 150 * MS, 900 * MS]
    assert list(st["level"]) == [0, 1, 2, 3]
    # inter-queue order: higher queue first, whatever the estimate order
    P = beta0_pool(4)
    assert service_order(run(sim, P)) == [0, 1, 2, 3]
