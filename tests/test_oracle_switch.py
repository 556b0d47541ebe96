"""Pins for the switching-cost model (AMB-24): a request that enters the
batch without having run in the previous step has its KV cache switched in, costing
c0 + c1 (prompt + generated tokens) of SYSTEM time (the step lasts c_round + the
batch's switch-ins; attained service E_i is not charged, S:... "speculation and
verification operations" only).  P:73 / P:102: "frequent preemption introduces
significant overhead ... switching the KV caches"; Fig. 2 ties the cost to length.

Expected values: a hand-evaluated two-request LAS preemption, the zero-cost identity,
work conservation, monotonicity in c1, non-preemptive policies paying exactly one
switch-in per request, and the sharded (G = 2) selection equal to the single rank.
"""
import numpy as np
import pytest

import oracle
from test_oracle_semiclairvoyant import beta0_pool, fig1_cfg
from test_oracle_sched import random_workload

MS = 1000


def test_two_request_las_preemption_hand_values():
    """LAS, K = 2 queues split at 20 ms, one candidate per 10 ms round (beta = 0 rows:
    one token per round), L = (3, 3), prompts (100, 200), c0 = 1 ms, c1 = 10 us/token.
    Hand schedule: R0 (switch 2.00 ms), R0, [R0 demoted at E = 20 ms] R1 (3.00 ms), R1,
    [R1 demoted] R0 (1 + 0.01*(100+2) = 2.02 ms), [done at 57.02 ms] R1 (3.02 ms), done
    at 70.04 ms."""
    P = beta0_pool(2)
    cfg = fig1_cfg(oracle.POL_LAS, K=2, s1_up_us=20 * MS, switch_c0_us=1 * MS, switch_c1_us=10)
    sim = oracle.Sim(cfg, np.zeros(2, np.int64), [3, 3], [3, 3], prompt=[100, 200])
    sel, _ = sim.select(1)
    flat = [int(sel[0])]
    costs = [sim.state()["step_cost_us"]]
    while not sim.state()["done"].all():
        sim.step(P, sel)
        flat += [int(i) for i in sel if i >= 0]
        costs.append(sim.state()["step_cost_us"])
    st = sim.state()
    assert flat == [0, 0, 1, 1, 0, 1]
    assert costs[:6] == [12_000, 10_000, 13_000, 10_000, 12_020, 13_020]
    assert list(st["C_us"]) == [57_020, 70_040]
    assert list(st["switch_us"]) == [4_020, 6_020]
    assert st["switch_total_us"] == 10_040
    assert list(st["E_us"]) == [30 * MS, 30 * MS]               # not charged to E_i
    assert st["C_us"].max() == 6 * 10 * MS + st["switch_total_us"]  # work conservation


def run_all(cfg, tr, P, B, prompt):
    sim = oracle.Sim(cfg, tr.arrival_us, tr.L_true, tr.L_pred, prompt=prompt)
    sel, _ = sim.select(B)
    n_steps = 0
    while not sim.state()["done"].all():
        sim.step(P, sel)
        n_steps += 1
        assert n_steps < 100_000
    return sim.state()


def prompts(n, seed):
    rng = np.random.default_rng(seed)
    return np.clip(np.round(np.exp(rng.normal(np.log(150), 0.7, n))), 4, 2048).astype(np.int32)


@pytest.mark.parametrize("policy", [oracle.POL_LAPSSD, oracle.POL_LAS, oracle.POL_FCFS])
def test_zero_cost_is_the_plain_simulation(policy):
    tr, P = random_workload(30, 41)
    base = dict(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4, t_ssm_us=1 * MS,
                t_llm_us=10 * MS, seed=4)
    a = run_all(oracle.SchedConfig(**base), tr, P, 3, None)
    b = run_all(oracle.SchedConfig(**base, switch_c0_us=0, switch_c1_us=0), tr, P, 3, prompts(30, 1))
    for f in ("C_us", "x_us", "acc_draft", "rounds", "level", "perceptible", "key"):
        assert (a[f] == b[f]).all(), f
    assert b["switch_total_us"] == 0


def test_non_preemptive_policies_pay_one_switch_in_per_request():
    tr, P = random_workload(30, 42)
    pr = prompts(30, 2)
    for pol in (oracle.POL_FCFS, oracle.POL_LPSJF):
        cfg = oracle.SchedConfig(policy=pol, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=2,
                                 switch_c0_us=500, switch_c1_us=7)
        st = run_all(cfg, tr, P, 2, pr)
        assert (st["switch_us"] == 500 + 7 * pr).all()      # entered once, at 0 tokens
        assert st["switch_total_us"] == st["switch_us"].sum()


def test_las_jct_rises_with_c1_and_conserves_work():
    """B = 1 and every arrival at 0: the server is never idle, so the last completion
    equals every round's service plus every switch-in (conservation), and the mean JCT
    cannot fall when the per-token switching cost rises (same schedule: LAS keys do not
    depend on the cost; every completion moves later)."""
    tr, P = random_workload(16, 43)
    tr.arrival_us[:] = 0
    pr = prompts(16, 3)
    c_round = 4 * MS + 10 * MS
    prev = None
    for c1 in (0, 5, 20, 80):
        cfg = oracle.SchedConfig(policy=oracle.POL_LAS, K=6, s1_up_us=20 * MS, gamma=3, k=4,
                                 t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=9, switch_c0_us=200,
                                 switch_c1_us=c1)
        st = run_all(cfg, tr, P, 1, pr)
        assert st["C_us"].max() == st["rounds"].sum() * c_round + st["switch_total_us"]
        assert st["switch_total_us"] == st["switch_us"].sum()
        jct = st["C_us"].mean()
        if prev is not None:
            assert jct > prev
        prev = jct


@pytest.mark.parametrize("policy", [oracle.POL_LAPSSD, oracle.POL_LAS])
def test_sharded_selection_with_switch_costs_equals_single_rank(policy):
    """PIN-G with switching costs: each rank sends every candidate's switch-in cost with
    its key; the merged step duration (global batch) equals the single rank's."""
    tr, P = random_workload(40, 44)
    pr = prompts(40, 4)
    B, G = 4, 2
    cfg = oracle.SchedConfig(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4,
                             t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=8, switch_c0_us=300,
                             switch_c1_us=11)
    ref = oracle.Sim(cfg, tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    sims = [oracle.Sim(cfg, tr.arrival_us[g::G], tr.L_true[g::G], tr.L_pred[g::G], rank=g, world=G,
                       prompt=pr[g::G]) for g in range(G)]
    tab = P["slab_tab"]

    def dist_select():
        cands = [s.candidates(B, with_switch=True) for s in sims]
        keys = np.concatenate([c[0] for c in cands])
        sw = np.concatenate([c[1] for c in cands])
        nxt = np.array([c[2] for c in cands])
        return [s.merge(keys, B, nxt, B, all_switch=sw) for s in sims]

    sel_ref, _ = ref.select(B)
    res = dist_select()
    for _ in range(400):
        if ref.state()["done"].all():
            break
        _, _, na_ref, _ = ref.step(P, sel_ref)
        # each rank verifies its own slots (same Philox counters: global id, round)
        for g, s in enumerate(sims):
            sel = res[g][0]
            na = np.full(B, -1, np.int32)
            stg = s.state()
            for b, i in enumerate(sel):
                if i < 0:
                    continue
                gid, rnd = i * G + g, stg["rounds"][i]
                slab = tab[gid, rnd if rnd < 16 else 8 + (rnd - 8) % 8]
                _, o = oracle.verify_request(P["p"][slab], P["q"][slab], P["draft"][slab], gid, rnd,
                                             cfg.seed)
                na[b] = o.r
            s.update(sel, na)
        res = dist_select()
        got = sorted(int(i) * G + g for g in range(G) for i in res[g][0] if i >= 0)
        assert got == sorted(int(i) for i in sel_ref if i >= 0)
        assert all(s.state()["now_us"] == ref.state()["now_us"] for s in sims)
        assert all(s.state()["step_cost_us"] == ref.state()["step_cost_us"] for s in sims)
    st = ref.state()
    assert st["done"].all() and st["switch_total_us"] > 0
    for g, s in enumerate(sims):
        sg = s.state()
        assert (sg["C_us"] == st["C_us"][g::G]).all()
        assert (sg["switch_us"] == st["switch_us"][g::G]).all()
