"""Monte-Carlo replica engine (configs[4], SURVEY §8(a) a6 per-trace top-1) against the
oracle: every trace is an independent batch-1 simulation with Philox trace index t, so
trace t of the GPU engine must equal oracle.Sim(..., trace=t) run alone with B = 1 --
selection, r, emitted tokens every step, and every state field at the end."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MS = 1000


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_17074_b200 as lib
    return lib


FIELDS = ["acc_tok", "acc_draft", "rounds", "E_us", "T_total_us", "C_us", "x_us", "admitted", "done",
          "perceptible", "pinned", "level", "running", "key", "switch_us"]


def run_mc_lockstep(L, kw, T, n, V, k, dtype, seed, R=8, max_steps=4000, prompt=False):
    rate = synth.mc_rate_for_load(0.8, k, kw["t_ssm_us"], kw["t_llm_us"], len_mu=np.log(30))
    w = synth.make_mc_workload(T, n, seed, rate_per_s=rate, len_mu=np.log(30), len_sigma=0.6, len_min=4,
                               len_max=200, n_buckets=8, variants=3, R=R)
    pool = synth.make_pool("f2", V=V, k=k, dtype=dtype, n_buckets=8, variants=3, seed=seed, device="cuda")
    P = pool.numpy()
    cfg = dict(kw, k=k)
    pr = synth.prompt_lengths(T * n, seed) if prompt else None
    sims, sels, Ps = [], [], []
    for t in range(T):
        a, lt, lp, tab = w.trace(t)
        sim = oracle.Sim(oracle.SchedConfig(**cfg), a, lt, lp, trace=t,
                         prompt=pr[t * n:(t + 1) * n] if prompt else None)
        sel, _ = sim.select(1)
        Pt = dict(P)
        Pt["slab_tab"], Pt["R"] = np.ascontiguousarray(tab), R
        sims.append(sim), sels.append(sel), Ps.append(Pt)
    mc = L.MCHandle(L.SchedConfig(**cfg), w.offsets, w.arrival_us, w.L_true, w.L_pred, V=V, prompt=pr)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device="cuda"))
    mc.select(rows)
    tokens = torch.full((T, k + 1), -9, dtype=torch.int32, device="cuda")
    nacc = torch.full((T,), -9, dtype=torch.int32, device="cuda")
    steps = 0
    while True:
        st, now, cur, sel_g = mc.state()
        for t in range(T):
            assert sel_g[t] == sels[t][0], f"step {steps} trace {t}: selection differs"
        if all(s.state()["done"].all() for s in sims):
            break
        active = mc.step(rows, tokens=tokens, n_accept=nacc)
        tok_g, na_g = tokens.cpu().numpy(), nacc.cpu().numpy()
        for t in range(T):
            ran = sels[t][0] >= 0
            _, tok_o, na_o, _ = sims[t].step(Ps[t], sels[t])
            if ran:
                assert na_g[t] == na_o[0], f"step {steps} trace {t}: r differs"
                assert (tok_g[t] == tok_o[0]).all(), f"step {steps} trace {t}: tokens differ"
            else:
                assert na_g[t] == -1
        assert int(active.item()) == sum(int(s[0] >= 0) for s in sels)
        steps += 1
        assert steps < max_steps
    st, now, cur, sel_g = mc.state()
    for t in range(T):
        a, b = int(w.offsets[t]), int(w.offsets[t + 1])
        o = sims[t].state()
        for f in FIELDS:
            assert (np.asarray(st[f][a:b]) == np.asarray(o[f])).all(), f"trace {t}: field {f} differs"
        assert (st["A"][a:b].view(np.uint64) == o["A"].view(np.uint64)).all(), f"trace {t}: A differs"
        assert (st["ring"][a:b] == o["ring"]).all(), f"trace {t}: ring differs"
        assert now[t] == o["now_us"] and cur[t] == o["cursor"], f"trace {t}: clock differs"
    assert st["switch_total_us"] == sum(s.state()["switch_total_us"] for s in sims)
    assert mc.check() == 0
    return steps


BASE = dict(K=4, s1_up_us=56 * MS, M=2.0, gamma=5, delta=0.05, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=7)


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_mc_traces_equal_single_trace_oracle(L, policy):
    steps = run_mc_lockstep(L, dict(BASE, policy=policy), T=6, n=24, V=2048, k=4, dtype="bf16", seed=50 + policy)
    assert steps > 20


def test_mc_fp32_rows_many_traces(L):
    """More traces than one verify sub-launch holds would need >4096; here: many small
    traces, fp32 rows, ragged V (two fp32 chunks)."""
    run_mc_lockstep(L, dict(BASE, policy=0), T=40, n=6, V=8200, k=3, dtype="f32", seed=9)


def test_mc_sub_launch_split(L):
    """T > the verify kernel's per-launch slot capacity: several verify sub-launches."""
    cap = 4096
    T = cap + 37
    w = synth.make_mc_workload(T, 2, 5, rate_per_s=5.0, len_mu=np.log(6), len_sigma=0.3, len_min=2, len_max=12,
                               n_buckets=4, variants=2, R=4)
    pool = synth.make_pool("f2", V=512, k=2, dtype="bf16", n_buckets=4, variants=2, seed=5, device="cuda")
    cfg = dict(BASE, policy=0, k=2)
    mc = L.MCHandle(L.SchedConfig(**cfg), w.offsets, w.arrival_us, w.L_true, w.L_pred, V=512)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device="cuda"))
    mc.select(rows)
    nacc = torch.empty(T, dtype=torch.int32, device="cuda")
    P = pool.numpy()
    picks = [0, 1, cap - 1, cap, T - 1]   # traces on both sides of the split, against the oracle
    sims, sels, Ps = {}, {}, {}
    for t in picks:
        a, lt, lp, tab = w.trace(t)
        sims[t] = oracle.Sim(oracle.SchedConfig(**cfg), a, lt, lp, trace=t)
        sels[t], _ = sims[t].select(1)
        Ps[t] = dict(P, slab_tab=np.ascontiguousarray(tab), R=4)
    for _ in range(30):
        mc.step(rows, n_accept=nacc)
        na = nacc.cpu().numpy()
        for t in picks:
            ran = sels[t][0] >= 0
            _, _, na_o, _ = sims[t].step(Ps[t], sels[t])
            if ran:
                assert na[t] == na_o[0]
    assert mc.check() == 0


@pytest.mark.parametrize("policy", [0, 3])
def test_mc_switching_cost(L, policy):
    """f2 (AMB-24) on the Monte-Carlo engine: batch 1 per trace, a request
    that did not run in the trace's previous step pays c0 + c1 (prompt + tokens)."""
    kw = dict(BASE, policy=policy, switch_c0_us=3 * MS, switch_c1_us=20)
    run_mc_lockstep(L, kw, T=8, n=20, V=2048, k=4, dtype="bf16", seed=70 + policy, prompt=True)


def test_mc_multi_step_no_sync(L):
    """Several laps_mc_step calls back to back without host synchronisation (T fits one
    verify sub-launch, so consecutive steps share its scratch set): mc_step_kernel waits
    for the verify grid it overlaps before it completes, so the results equal
    those of a synchronised run."""
    kw = dict(BASE, policy=0)
    T, n, V, k, R = 64, 16, 4096, 4, 8
    rate = synth.mc_rate_for_load(0.8, k, kw["t_ssm_us"], kw["t_llm_us"], len_mu=np.log(30))
    w = synth.make_mc_workload(T, n, 81, rate_per_s=rate, len_mu=np.log(30), len_sigma=0.6, len_min=4,
                               len_max=200, n_buckets=8, variants=3, R=R)
    pool = synth.make_pool("f2", V=V, k=k, dtype="bf16", n_buckets=8, variants=3, seed=81, device="cuda")
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device="cuda"))
    outs = []
    for sync in (True, False):
        mc = L.MCHandle(L.SchedConfig(**dict(kw, k=k)), w.offsets, w.arrival_us, w.L_true, w.L_pred, V=V)
        mc.select(rows)
        nacc = torch.empty(40, T, dtype=torch.int32, device="cuda")
        for s in range(40):
            mc.step(rows, n_accept=nacc[s])
            if sync:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        st, now, _, _ = mc.state()
        outs.append((nacc.cpu().numpy(), st["acc_tok"], now))
        assert mc.check() == 0
    assert (outs[0][0] == outs[1][0]).all()
    assert (outs[0][1] == outs[1][1]).all() and (outs[0][2] == outs[1][2]).all()
