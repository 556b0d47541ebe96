"""Pins for the oracle's LAPS-SD scheduler and Fig. 1.

Expected values come from the paper's printed numbers, hand evaluation of its
formulas, exhaustive enumeration, an exact renewal DP for expected
step counts, the 1/t bound on cumulative-rate movement, and the algorithm's own
degeneracies (LAPS-SD with one queue and no stabilisation is FCFS; with delta = 0
it is LAS).
"""
import itertools
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from conftest import golden

MS = 1000  # microseconds per millisecond


def read_fig1():
    vals = {}
    for line in open(golden("fig1.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        vals[f[0]] = f[1:]
    return vals


# ---------------------------------------------------------------- P:169 thresholds (PIN-T)
def test_thresholds_exponential():
    assert list(oracle.thresholds(4, 50 * MS, 2.0)) == [50 * MS, 100 * MS, 200 * MS]
    assert list(oracle.thresholds(3, 10 * MS, 3.0)) == [10 * MS, 30 * MS]
    assert list(oracle.thresholds(1, 50 * MS, 2.0)) == []
    with pytest.raises(ValueError):
        oracle.thresholds(0, 50, 2.0)
    with pytest.raises(ValueError):
        oracle.thresholds(4, 0, 2.0)
    with pytest.raises(ValueError):
        oracle.thresholds(4, 50, 1.0)


# ---------------------------------------------------------------- Eq. (6) (PIN-E)
def test_eq6_hand_values():
    # L=100, A=0.5, n=4, T_SSM=1 ms, T_LLM=10 ms: 4*100*1/3 + 100*10/3 = 466.67 ms
    assert oracle.eq6(100, 0.5, 4, 1 * MS, 10 * MS) == 466_666
    # L=5, A=1, n=4, T_SSM=0, T_LLM=10 ms: 5*10/5 = 10 ms
    assert oracle.eq6(5, 1.0, 4, 0, 10 * MS) == 10_000
    # L=10, A=0: bonus-token-only progress, 40 + 100 = 140 ms
    assert oracle.eq6(10, 0.0, 4, 1 * MS, 10 * MS) == 140_000
    # remaining 60 tokens of the first case: 280 ms
    assert oracle.eq6(60, 0.5, 4, 1 * MS, 10 * MS) == 280_000
    assert oracle.eq6(0, 0.5, 4, 1 * MS, 10 * MS) == 0


# ---------------------------------------------------------------- Fig. 1 (PIN-F1)
def fig1_jobs():
    v = read_fig1()
    L = np.array([int(v[r][0]) for r in ("R1", "R2", "R3")])
    alpha = np.array([float(v[r][1]) for r in ("R1", "R2", "R3")])
    t_tok = int(v["t_tok_ms"][0]) * MS
    service = np.round(L / alpha).astype(np.int64) * t_tok   # L / alpha candidates
    return v, L, alpha, service


def test_fig1_candidates():
    v, L, alpha, service = fig1_jobs()
    assert L[0] / alpha[0] == 20                              # "20 candidate tokens"
    assert list(service) == [200 * MS, 500 * MS, 150 * MS]


def test_fig1_fcfs_and_sjf_averages_match_paper():
    v, L, alpha, service = fig1_jobs()
    arr = np.zeros(3, np.int64)
    tot, order, _ = oracle.jobs_schedule(1, arr, service)
    assert list(order) == [0, 1, 2]                           # "FCFS first schedules R1 and R2"
    assert round(tot / 3 / MS) == int(v["fcfs_avg_ms"][0])   # 583 ms
    assert tot == 1_750_000
    tot, order, _ = oracle.jobs_schedule(2, arr, service, L_pred=L)
    assert order[0] == 1                                      # "R2 is scheduled first"
    assert round(tot / 3 / MS) == int(v["sjf_avg_ms"][0])    # 683 ms
    assert tot == 2_050_000


def test_fig1_optimal_is_laps_sd_with_known_rates():
    v, L, alpha, service = fig1_jobs()
    est = (np.round(L / alpha) * 10 * MS).astype(np.int64)     # T~ = L/A * 10 ms
    tot, order, _ = oracle.jobs_schedule(0, np.zeros(3, np.int64), service, est_us=est)
    best, best_order, sums = oracle.brute_force(service)
    assert tot == best == 1_350_000                           # 450 ms
    assert list(order) == [2, 0, 1] == list(best_order)       # R3, R1, R2 -- R2 last
    assert list(sums) == [1_750_000, 1_400_000, 2_050_000, 2_000_000, 1_350_000, 1_650_000]
    assert sums.max() == 2_050_000                             # LP-SJF is the worst order


def test_sjf_on_estimates_equals_brute_force_optimum():
    """Immediate stabilisation + exact estimates = SJF = the optimum of Eq. (2) with
    simultaneous arrivals (checked exhaustively, 200 instances of <= 7 requests)."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 8))
        service = rng.integers(1, 60, size=n).astype(np.int64) * MS
        tot, _, _ = oracle.jobs_schedule(0, np.zeros(n, np.int64), service, est_us=service)
        best, _, sums = oracle.brute_force(service)
        assert tot == best == sums.min()
        assert len(sums) == math.factorial(n)


# ---------------------------------------------------------------- helpers for token-level runs
def tiny_pool(betas, V=16, k=4, dtype=torch.float32, seed=0):
    """One F1 slab per request; slab i has acceptance betas[i] at every position."""
    g = torch.Generator()
    g.manual_seed(seed)
    ps, qs, ds = [], [], []
    for b in betas:
        p, q, d = synth.f1_rows(V, k, [b] * (k + 1), g, dtype=dtype)
        ps.append(p), qs.append(q), ds.append(d)
    P = dict(p=synth.to_numpy_rows(torch.stack(ps)), q=synth.to_numpy_rows(torch.stack(qs)),
             draft=torch.stack(ds).numpy().astype(np.int32))
    n = len(betas)
    P["slab_tab"] = np.repeat(np.arange(n, dtype=np.int32)[:, None], 4, 1)
    P["R"] = 4
    return P


def run_sim(cfg, arrival, L_true, L_pred, pools, B, max_steps=100_000):
    sim = oracle.Sim(cfg, arrival, L_true, L_pred)
    sel, _ = sim.select(B)
    steps = 0
    orders = [sel.copy()]
    while True:
        st = sim.state()
        if st["done"].all():
            break
        sim.step(pools, sel)
        orders.append(sel.copy())
        steps += 1
        assert steps < max_steps
    return sim, sim.state(), orders


def expected_steps(L, beta, k):
    """Exact E[number of rounds to emit L tokens] by the renewal DP
    E[S(l)] = 1 + sum_e P(e) E[S(l - e)], P(e = j+1) = b^j (1-b) (j < k),
    P(e = k+1) = b^k."""
    pe = [beta ** j * (1 - beta) for j in range(k)] + [beta ** k]
    S = [0.0] * (L + 1)
    for l in range(1, L + 1):
        S[l] = 1 + sum(pe[e - 1] * S[max(l - e, 0)] for e in range(1, k + 2))
    return S[L]


def test_fig1_token_level_expectations():
    """Fig. 1 with real rejection sampling (V=16, k=4, 4 candidates x 10 ms per
    round): E[avg JCT] from the exact DP, against the oracle's Monte-Carlo
    mean (PIN-F2)."""
    L = [10, 5, 15]
    betas = [0.5, 0.1, 1.0]
    k = 4
    ES = [expected_steps(l, b, k) for l, b in zip(L, betas)]
    assert ES[0] == pytest.approx(5.59375) and ES[1] == pytest.approx(4.6)
    assert ES[2] == pytest.approx(3.0)
    c = 40 * MS
    want = {oracle.POL_FCFS: (3 * ES[0] + 2 * ES[1] + ES[2]) * c / 3,
            oracle.POL_LPSJF: (3 * ES[1] + 2 * ES[0] + ES[2]) * c / 3}
    assert want[oracle.POL_FCFS] / MS == pytest.approx(386.4167, abs=1e-3)
    assert want[oracle.POL_LPSJF] / MS == pytest.approx(373.1667, abs=1e-3)
    pools = tiny_pool(betas)
    n_seeds = 6000
    for pol, target in want.items():
        jct = []
        for seed in range(n_seeds):
            cfg = oracle.SchedConfig(policy=pol, K=4, s1_up_us=4 * c, k=k, t_ssm_us=0,
                                     t_llm_us=c, seed=seed)
            _, st, _ = run_sim(cfg, np.zeros(3, np.int64), L, L, pools, B=1)
            assert (st["acc_tok"] == L).all()
            jct.append(st["C_us"].mean())
        jct = np.array(jct)
        assert abs(jct.mean() - target) < 5 * jct.std() / np.sqrt(n_seeds)


# ---------------------------------------------------------------- stability (PIN-ST)
def drive_one(cfg, accepts, L=10**6):
    sim = oracle.Sim(cfg, [0], [L], [L])
    sel, _ = sim.select(1)
    became = None
    for t, a in enumerate(accepts, start=1):
        sim.update([0], [a])
        st = sim.state()
        if st["perceptible"][0] and became is None:
            became = t
        sim.select(1)
    return sim, became


def test_cumulative_rate_history():
    """per-round (proposed, accepted) = (4,4), (4,2) -> rates 1.0, 0.75;
    the ring stores cumulative accepted drafts a_t and proposed is k t."""
    cfg = oracle.SchedConfig(k=4, gamma=5)
    sim, _ = drive_one(cfg, [4, 2])
    st = sim.state()
    assert st["ring"][0][1] == 4 and st["ring"][0][2] == 6
    assert st["ring"][0][1] / (4 * 1) == 1.0 and st["ring"][0][2] / (4 * 2) == 0.75


def test_constant_rate_stabilises_at_gamma_with_exact_mean():
    cfg = oracle.SchedConfig(k=4, gamma=5, delta=0.05, t_ssm_us=1 * MS, t_llm_us=10 * MS)
    sim, t = drive_one(cfg, [2] * 10, L=100)
    st = sim.state()
    assert t == 5
    assert st["A"][0] == 0.5
    assert st["T_total_us"][0] == 466_666          # Eq. (6) at L=100, A=0.5


def test_delta_zero_never_stabilises():
    cfg = oracle.SchedConfig(k=4, gamma=3, delta=0.0)
    _, t = drive_one(cfg, [2] * 60)
    assert t is None


def deadline(gamma, delta, tmax=1000):
    """First t with sum_{s=t-gamma+2..t} 1/s < delta: |rate_t - rate_{t-1}| <= 1/t."""
    for t in range(gamma, tmax):
        if sum(1.0 / s for s in range(t - gamma + 2, t + 1)) < delta:
            return t


def test_stability_deadline_any_draws():
    assert deadline(5, 0.05) == 82 and deadline(3, 0.05) == 41
    rng = np.random.default_rng(1)
    k = 4
    seqs = [[0, k] * 60, [k] * 40 + [0] * 80, [0] * 40 + [k] * 80,
            list(rng.integers(0, k + 1, 120))]
    seqs += [list(rng.choice([0, k], 120)) for _ in range(300)]
    worst = 0
    for gamma in (3, 5):
        bound = deadline(gamma, 0.05)
        for s in seqs:
            cfg = oracle.SchedConfig(k=k, gamma=gamma, delta=0.05)
            _, t = drive_one(cfg, s)
            assert t is not None and t <= bound
            worst = max(worst, t)
    assert worst > 10


# ---------------------------------------------------------------- degeneracies (PIN-DG)
def random_workload(n, seed, V=64, k=4, dtype="f32"):
    tr = synth.make_trace(n, seed, arrival="poisson", rate_per_s=60.0, len_mu=np.log(40),
                          len_sigma=0.6, len_min=4, len_max=200, beta_ab=(3, 2), drift=True)
    pool = synth.make_pool("f2", V=V, k=k, dtype=dtype, n_buckets=8, variants=3, seed=seed)
    P = pool.numpy()
    P["slab_tab"] = synth.slab_table(tr, 8, 3, R=16, seed=seed)
    P["R"] = 16
    return tr, P


@pytest.mark.parametrize("B", [1, 3])
def test_one_queue_no_stabilisation_is_fcfs(B):
    for seed in range(4):
        tr, P = random_workload(24, seed)
        base = dict(K=1, gamma=3, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=seed)
        a = run_sim(oracle.SchedConfig(policy=oracle.POL_LAPSSD, delta=0.0, **base),
                    tr.arrival_us, tr.L_true, tr.L_pred, P, B)
        b = run_sim(oracle.SchedConfig(policy=oracle.POL_FCFS, delta=0.0, **base),
                    tr.arrival_us, tr.L_true, tr.L_pred, P, B)
        assert len(a[2]) == len(b[2])
        for x, y in zip(a[2], b[2]):
            assert (x == y).all()
        assert (a[1]["C_us"] == b[1]["C_us"]).all()


@pytest.mark.parametrize("B", [1, 4])
def test_delta_zero_is_las(B):
    for seed in range(4):
        tr, P = random_workload(24, 100 + seed)
        base = dict(K=4, s1_up_us=30 * MS, gamma=3, delta=0.0, k=4, t_ssm_us=1 * MS,
                    t_llm_us=10 * MS, seed=seed)
        a = run_sim(oracle.SchedConfig(policy=oracle.POL_LAPSSD, **base),
                    tr.arrival_us, tr.L_true, tr.L_pred, P, B)
        b = run_sim(oracle.SchedConfig(policy=oracle.POL_LAS, **base),
                    tr.arrival_us, tr.L_true, tr.L_pred, P, B)
        for x, y in zip(a[2], b[2]):
            assert (x == y).all()
        assert (a[1]["C_us"] == b[1]["C_us"]).all()


# ---------------------------------------------------------------- invariants (PIN-INV)
@pytest.mark.parametrize("policy", [oracle.POL_LAPSSD, oracle.POL_FCFS, oracle.POL_LPSJF,
                                    oracle.POL_LAS])
def test_invariants(policy):
    tr, P = random_workload(40, 7)
    cfg = oracle.SchedConfig(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4,
                             t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=3)
    sim = oracle.Sim(cfg, tr.arrival_us, tr.L_true, tr.L_pred)
    B = 4
    sel, _ = sim.select(B)
    prev = sim.state()
    busy_steps = 0
    while not prev["done"].all():
        nonempty = (sel >= 0).any()
        cnt, tok, na, z = sim.step(P, sel)
        st = sim.state()
        busy_steps += int(nonempty)
        ran = prev["rounds"] != st["rounds"]
        # every verified request gains >= 1 token unless it completed
        grew = st["acc_tok"] - prev["acc_tok"]
        assert ((grew >= 1) | st["done"].astype(bool))[ran].all()
        # perceptibility is one-way, levels never fall for non-perceptible
        assert (st["perceptible"] >= prev["perceptible"]).all()
        np_mask = st["perceptible"] == 0
        assert (st["level"][np_mask] >= prev["level"][np_mask]).all()
        prev = st
    st = prev
    assert (st["acc_tok"] == tr.L_true).all()                     # sum emitted = L
    assert (st["x_us"] >= tr.arrival_us).all()                    # x_i >= r_i (Eq. 3)
    c_round = 4 * MS + 10 * MS
    assert (st["C_us"] >= st["x_us"] + c_round).all()             # C_i >= x_i + round
    assert (st["E_us"] == st["rounds"] * c_round).all()           # E_i
    assert st["rounds"].sum() <= busy_steps * B


def test_fcfs_and_lpsjf_never_preempt():
    tr, P = random_workload(30, 11)
    for pol in (oracle.POL_FCFS, oracle.POL_LPSJF):
        cfg = oracle.SchedConfig(policy=pol, k=4, seed=2)
        _, st, orders = run_sim(cfg, tr.arrival_us, tr.L_true, tr.L_pred, P, B=2)
        # once selected a request stays in every batch until it is done
        seen = {}
        for t, sel in enumerate(orders):
            for i in sel[sel >= 0]:
                seen.setdefault(int(i), []).append(t)
        for i, ts in seen.items():
            assert ts == list(range(ts[0], ts[0] + len(ts)))


# ---------------------------------------------------------------- multi-rank merge (PIN-G, oracle side)
@pytest.mark.parametrize("policy,G", [(oracle.POL_LAPSSD, 2), (oracle.POL_LAS, 2), (oracle.POL_FCFS, 2),
                                      (oracle.POL_LAPSSD, 4), (oracle.POL_LAPSSD, 8), (oracle.POL_LAS, 8)])
def test_sharded_global_topB_equals_single_rank(policy, G):
    """PIN-G: sharding over G = 2, 4, 8 ranks gives every request the single-rank result."""
    tr, P = random_workload(48, 21)
    B = 5
    cfg = oracle.SchedConfig(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4,
                             t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=8)
    ref, st_ref, orders = run_sim(cfg, tr.arrival_us, tr.L_true, tr.L_pred, P, B)
    sims = [oracle.Sim(cfg, *(lambda s: (s.arrival_us, s.L_true, s.L_pred))(tr.shard(g, G)),
                       rank=g, world=G) for g in range(G)]
    pools = []
    for g in range(G):
        Pg = dict(P)
        Pg["slab_tab"] = np.ascontiguousarray(P["slab_tab"][g::G])
        pools.append(Pg)

    def dist_select():
        cands = [s.candidates(B) for s in sims]
        keys = np.concatenate([c[0] for c in cands])
        nxt = np.array([c[1] for c in cands])
        return [s.merge(keys, B, nxt, B) for s in sims]

    res = dist_select()
    for t in range(1, len(orders)):
        # the global batch in key order, mapped back to global ids
        for g, s in enumerate(sims):
            s.update_sel = res[g][0]
        for g, s in enumerate(sims):
            sel = res[g][0]
            # verify + update on each rank's own slots (no select inside)
            k = cfg.k
            na = np.full(B, -1, np.int32)
            for b, i in enumerate(sel):
                if i < 0:
                    continue
                gid = i * G + g
                rnd = s.state()["rounds"][i]
                slab = pools[g]["slab_tab"][i, rnd if rnd < 16 else 8 + (rnd - 8) % 8]
                _, o = oracle.verify_request(P["p"][slab], P["q"][slab], P["draft"][slab],
                                             gid, rnd, cfg.seed)
                na[b] = o.r
            s.update(sel, na)
        res = dist_select()
        got = sorted(int(i) * G + g for g in range(G) for i in res[g][0] if i >= 0)
        want = sorted(int(i) for i in orders[t] if i >= 0)
        assert got == want
        assert res[0][2] == len(want)
    for g, s in enumerate(sims):
        st = s.state()
        assert (st["C_us"] == st_ref["C_us"][g::G]).all()
        assert (st["acc_draft"] == st_ref["acc_draft"][g::G]).all()


def test_openmp_build_equals_plain_oracle():
    """The all-cores CPU baseline (the same source built with -fopenmp: a step's requests
    verified in parallel) computes exactly what the plain single-thread oracle computes."""
    import synth
    tr = synth.make_trace(60, 5, arrival="poisson", rate_per_s=80.0, len_mu=np.log(20), len_sigma=0.5,
                          len_min=4, len_max=80, drift=True)
    pool = synth.make_pool("f2", V=512, k=4, dtype="bf16", n_buckets=4, variants=2, seed=5, device="cpu")
    tab = synth.slab_table(tr, 4, 2, R=8, seed=5)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 8
    out = []
    for parallel in (False, True):
        sim = oracle.Sim(oracle.SchedConfig(k=4, seed=3), tr.arrival_us, tr.L_true, tr.L_pred, parallel=parallel)
        sel, _ = sim.select(12)
        toks = []
        while not sim.state()["done"].all():
            _, tok, na, _ = sim.step(P, sel)
            toks.append(tok.copy())
        out.append((np.concatenate(toks), sim.state()))
    assert (out[0][0] == out[1][0]).all()
    for f in ("C_us", "acc_draft", "E_us", "key"):
        assert (out[0][1][f] == out[1][1][f]).all()


def test_concurrent_simulations_in_threads_equal_sequential():
    """The all-cores Monte-Carlo baseline runs independent traces in Python threads (the
    oracle's C calls release the GIL): each trace's result equals its sequential run."""
    import concurrent.futures as cf

    import synth
    w = synth.make_mc_workload(8, 30, 3, rate_per_s=30.0, len_mu=np.log(20), len_sigma=0.5, len_min=2,
                               len_max=60, n_buckets=4, variants=2, R=8)
    pool = synth.make_pool("f2", V=256, k=4, dtype="bf16", n_buckets=4, variants=2, seed=3, device="cpu")
    P = pool.numpy()
    cfg = oracle.SchedConfig(k=4, seed=9, s1_up_us=40 * MS)

    def run(t):
        a, lt, lp, tab = w.trace(t)
        sim = oracle.Sim(cfg, a, lt, lp, trace=t)
        Pt = dict(P, slab_tab=np.ascontiguousarray(tab), R=8)
        sel, _ = sim.select(1)
        for _ in range(5000):
            if sim.step(Pt, sel)[0] == 0 and sim.state()["done"].all():
                break
        return sim.state()["C_us"]

    seq = [run(t) for t in range(8)]
    with cf.ThreadPoolExecutor(8) as ex:
        par = list(ex.map(run, range(8)))
    for a, b in zip(seq, par):
        assert (a == b).all()
