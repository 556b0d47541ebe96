"""GPU parity of the fused step (laps_select + laps_step through the C-ABI) against the
oracle simulation, step by step on the same seeded workload: the selected batch (in
key order), every priority key, and every field of the per-request state are compared
bit-exactly; A_i (fp64) is compared as bits."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

FIELDS = ["acc_tok", "acc_draft", "rounds", "E_us", "T_total_us", "C_us", "x_us", "admitted",
          "done", "perceptible", "pinned", "level", "running", "key", "ring", "switch_us"]


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_17074_b200 as lib
    return lib


def workload(n, V, k, dtype, seed, drift, R=16, arrival="poisson", rate=80.0, len_mu=np.log(40),
             family="f2", n_buckets=8, variants=3):
    tr = synth.make_trace(n, seed, arrival=arrival, rate_per_s=rate, len_mu=len_mu, len_sigma=0.6,
                          len_min=4, len_max=400, beta_ab=(4, 2), drift=drift)
    pool = synth.make_pool(family, V=V, k=k, dtype=dtype, n_buckets=n_buckets, variants=variants,
                           seed=seed, device="cuda")
    tab = synth.slab_table(tr, n_buckets, variants, R=R, seed=seed)
    return tr, pool, tab


def compare_state(g, o, step):
    for f in FIELDS:
        a, b = np.asarray(g[f]), np.asarray(o[f])
        assert a.shape == b.shape and (a == b).all(), f"step {step}: field {f} differs"
    assert (g["A"].view(np.uint64) == o["A"].view(np.uint64)).all(), f"step {step}: A differs"
    for f in ("now_us", "cursor", "prev_count", "step_cost_us", "switch_total_us"):
        assert g[f] == o[f], f"step {step}: {f} {g[f]} != {o[f]}"


def run_lockstep(L, cfg_kw, tr, pool, tab, B, max_steps=5000, check_every=1, prompt=None, overlap=False):
    gcfg = L.SchedConfig(**cfg_kw)
    ocfg = oracle.SchedConfig(**cfg_kw)
    h = L.Handle(gcfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V, prompt=prompt,
                 overlap=overlap)
    sim = oracle.Sim(ocfg, tr.arrival_us, tr.L_true, tr.L_pred, prompt=prompt)
    rows = L.Rows(pool.p, pool.q, pool.draft,
                  torch.as_tensor(tab, dtype=torch.int32, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, tab.shape[1]
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    tokens = torch.empty(B, cfg_kw["k"] + 1, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    steps = 0
    while True:
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {steps}: batch differs\n{sel_g}\n{sel_o}"
        if steps % check_every == 0:
            compare_state(h.state(), sim.state(), steps)
        if sim.state()["done"].all():
            break
        h.laps_step(rows, B, tokens=tokens, n_accept=nacc)
        cnt, tok_o, na_o, _ = sim.step(P, sel_o)
        live = sel_g >= 0
        assert (nacc.cpu().numpy()[live] == na_o[live]).all(), f"step {steps}: r differs"
        assert (tokens.cpu().numpy()[live] == tok_o[live]).all(), f"step {steps}: tokens differ"
        steps += 1
        assert steps < max_steps
    assert h.check() == 0
    compare_state(h.state(), sim.state(), steps)
    return steps


BASE = dict(K=4, s1_up_us=56_000, M=2.0, gamma=5, delta=0.05, t_ssm_us=1000, t_llm_us=10_000)


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_step_parity_config2_shape(L, policy):
    """configs[1] shape, scaled: Poisson arrivals, Beta acceptance, fp32, V=32000, k=4."""
    tr, pool, tab = workload(160, 32000, 4, "f32", seed=0x5D0002 + policy, drift=False)
    run_lockstep(L, dict(BASE, policy=policy, k=4, seed=11), tr, pool, tab, B=16)


@pytest.mark.parametrize("B", [1, 8])
def test_step_parity_config3_drift(L, B):
    """configs[2] shape, scaled: drifting acceptance, bf16, V=32000, k=6, K=4."""
    tr, pool, tab = workload(96, 32000, 6, "bf16", seed=0x5D0003 + B, drift=True)
    run_lockstep(L, dict(BASE, k=6, seed=5), tr, pool, tab, B=B, check_every=3)


@pytest.mark.parametrize("kw", [dict(placement=1), dict(pin_rule=1), dict(K=1, delta=0.0),
                                dict(gamma=3, delta=0.2), dict(K=16, M=1.5, s1_up_us=5000)])
def test_step_parity_variants(L, kw):
    tr, pool, tab = workload(80, 2048, 4, "bf16", seed=77, drift=True)
    run_lockstep(L, dict(BASE, k=4, seed=3, **kw), tr, pool, tab, B=6)


def test_step_parity_idle_gaps(L):
    """Sparse arrivals: empty batches make the clock jump to the next arrival."""
    tr, pool, tab = workload(40, 1024, 4, "bf16", seed=8, drift=False, rate=2.0,
                             len_mu=np.log(10))
    run_lockstep(L, dict(BASE, k=4, seed=1), tr, pool, tab, B=4)


def test_step_parity_config4_full_size(L):
    """configs[3] at the bench's launch configuration: N=2048 resident, B=512, V=128256,
    k=8, bf16, all arrive at 0.  A few steps, every slot and every request compared."""
    c = synth.CONFIGS["c4"]
    tr = synth.make_trace(2048, c["seed"], arrival="zero", length="uniform", len_min=512,
                          len_max=4096, beta_ab=(7, 3))
    pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=16, variants=2,
                           seed=c["seed"], device="cuda")
    tab = synth.slab_table(tr, 16, 2, R=16, seed=c["seed"])
    gcfg = L.SchedConfig(**dict(BASE, k=8, seed=c["seed"]))
    h = L.Handle(gcfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=512, V=128256)
    sim = oracle.Sim(oracle.SchedConfig(**dict(BASE, k=8, seed=c["seed"])), tr.arrival_us,
                     tr.L_true, tr.L_pred)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 16
    sel_o, _ = sim.select(512)
    h.laps_select(512)
    nacc = torch.empty(512, dtype=torch.int32, device="cuda")
    for step in range(6):
        assert (h.sel.cpu().numpy() == sel_o).all()
        h.laps_step(rows, 512, n_accept=nacc)
        _, _, na_o, _ = sim.step(P, sel_o)
        assert (nacc.cpu().numpy() == na_o).all()
        compare_state(h.state(), sim.state(), step)


def test_step_parity_graph_replay_config4(L):
    """The launch configuration bench.py times: laps_step captured in a CUDA graph
    (consecutive verify launches overlap through programmatic dependent launch, the
    select runs on the side stream) and replayed; configs[3] sizes.  Every step's
    accepted counts and tokens, and the whole state after each replay, bit-exact."""
    c = synth.CONFIGS["c4"]
    B, G, reps, k = 512, 8, 3, 8
    tr = synth.make_trace(2048, c["seed"] + 1, arrival="zero", length="uniform", len_min=512,
                          len_max=4096, beta_ab=(7, 3))
    pool = synth.make_pool("f2", V=128256, k=k, dtype="bf16", n_buckets=16, variants=4,
                           seed=c["seed"] + 1, device="cuda")
    tab = synth.slab_table(tr, 16, 4, R=32, seed=c["seed"] + 1)
    kw = dict(BASE, k=k, seed=c["seed"] + 1)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=128256,
                 overlap=True)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, tab.shape[1]
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    tok = torch.empty(G, B, k + 1, dtype=torch.int32, device="cuda")
    nacc = torch.empty(G, B, dtype=torch.int32, device="cuda")
    # one eager step first (as the bench's warm-up), checked like the rest
    h.laps_step(rows, B, tokens=tok[0], n_accept=nacc[0])
    _, tok_o, na_o, _ = sim.step(P, sel_o)
    assert (nacc[0].cpu().numpy() == na_o).all() and (tok[0].cpu().numpy() == tok_o).all()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for t in range(G):
            h.laps_step(rows, B, tokens=tok[t], n_accept=nacc[t])
    for rep in range(reps):
        g.replay()
        torch.cuda.synchronize()
        T, NA = tok.cpu().numpy(), nacc.cpu().numpy()
        for t in range(G):   # (a different batch would show in r / tokens / the state)
            cnt, tok_o, na_o, _ = sim.step(P, sel_o)   # sel_o becomes the next batch
            assert (NA[t] == na_o).all(), f"replay {rep} step {t}: r differs"
            assert (T[t] == tok_o).all(), f"replay {rep} step {t}: tokens differ"
        compare_state(h.state(), sim.state(), f"replay {rep}")
        assert (h.sel[:B].cpu().numpy() == sel_o).all(), f"replay {rep}: next batch differs"
    assert h.check() == 0


def _slab_round_index(t, R):
    h = R // 2
    return t if t < R else (R - 1 if h == 0 else h + (t - h) % h)


def test_step_parity_batch_layout_rows_per_step(L):
    """Batch layout (no slab table; slot b reads rows b of THIS call): each step the caller
    gathers the rows of the batch's requests from the pool -- the slab the table assigns
    to the request's current round -- so the run must equal the pooled oracle run."""
    tr, pool, tab = workload(80, 4096, 4, "bf16", seed=31, drift=True)
    kw = dict(BASE, k=4, seed=7)
    B, R = 8, tab.shape[1]
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, R
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    tok = torch.empty(B, 5, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(3000):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        rounds = h.state()["rounds"]
        slabs = [int(tab[i, _slab_round_index(int(rounds[i]), R)]) if i >= 0 else 0 for i in sel_g]
        idx = torch.as_tensor(slabs, device="cuda")
        rows = L.Rows(pool.p[idx].contiguous(), pool.q[idx].contiguous(), pool.draft[idx].contiguous(), None)
        h.laps_step(rows, B, tokens=tok, n_accept=nacc)
        _, tok_o, na_o, _ = sim.step(P, sel_o)
        live = sel_g >= 0
        assert (nacc.cpu().numpy()[live] == na_o[live]).all(), f"step {step}: r differs"
        assert (tok.cpu().numpy()[live] == tok_o[live]).all(), f"step {step}: tokens differ"
        if step % 5 == 0:
            compare_state(h.state(), sim.state(), step)
    assert sim.state()["done"].all()
    assert h.check() == 0


def test_step_parity_max_batch_4096(L):
    """The largest batch the incremental step takes (B = 4,096 slots: the verify
    kernel's per-CTA snapshot capacity; the side select then works on 8,192 keys with
    the radix top-B path), a few steps bit-exact against the oracle."""
    n, B = 8192, 4096
    tr = synth.make_trace(n, 0x5D0009, arrival="zero", length="uniform", len_min=64, len_max=512,
                          beta_ab=(7, 3))
    pool = synth.make_pool("f2", V=1024, k=4, dtype="bf16", n_buckets=8, variants=4, seed=9, device="cuda")
    tab = synth.slab_table(tr, 8, 4, R=16, seed=9)
    kw = dict(BASE, k=4, seed=13)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=1024)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 16
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(6):
        assert (h.sel[:B].cpu().numpy() == sel_o).all(), f"step {step}: batch differs"
        h.laps_step(rows, B, n_accept=nacc)
        _, _, na_o, _ = sim.step(P, sel_o)
        assert (nacc.cpu().numpy() == na_o).all(), f"step {step}: r differs"
        compare_state(h.state(), sim.state(), step)
    assert h.check() == 0


# ---------------------------------------------------------------- f2: switching cost, Fig. 1 model
SWITCH = dict(switch_c0_us=2_000, switch_c1_us=15)   # 2 ms + 15 us per (prompt + generated) token


@pytest.mark.parametrize("policy", [0, 1, 3])
def test_step_parity_switching_cost(L, policy):
    """AMB-24: requests entering the batch pay c0 + c1 (prompt + tokens) of
    system time; clock, C_i, per-request switching time and the total, bit-exact."""
    tr, pool, tab = workload(120, 4096, 4, "bf16", seed=0x5F00 + policy, drift=True)
    pr = synth.prompt_lengths(tr.n, 0x5F00 + policy)
    run_lockstep(L, dict(BASE, policy=policy, k=4, seed=21, **SWITCH), tr, pool, tab, B=8, prompt=pr)


def test_step_parity_switching_cost_overlap_batch1(L):
    """Batch 1 (preemption at every round boundary makes switching frequent), the
    overlapped launch configuration."""
    tr, pool, tab = workload(40, 2048, 4, "bf16", seed=0x5F10, drift=True, rate=20.0)
    pr = synth.prompt_lengths(tr.n, 0x5F10)
    run_lockstep(L, dict(BASE, k=4, seed=22, **SWITCH), tr, pool, tab, B=1, prompt=pr, overlap=True)


def test_step_parity_switching_cost_batch_layout(L):
    """Batch layout (presort + final select path) with switching cost."""
    tr, pool, tab = workload(60, 2048, 4, "bf16", seed=0x5F20, drift=True)
    pr = synth.prompt_lengths(tr.n, 0x5F20)
    kw = dict(BASE, k=4, seed=23, **SWITCH)
    B, R = 6, tab.shape[1]
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V, prompt=pr)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, R
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    for step in range(3000):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        rounds = h.state()["rounds"]
        slabs = [int(tab[i, _slab_round_index(int(rounds[i]), R)]) if i >= 0 else 0 for i in sel_g]
        idx = torch.as_tensor(slabs, device="cuda")
        rows = L.Rows(pool.p[idx].contiguous(), pool.q[idx].contiguous(), pool.draft[idx].contiguous(), None)
        h.laps_step(rows, B)
        sim.step(P, sel_o)
        if step % 7 == 0:
            compare_state(h.state(), sim.state(), step)
    compare_state(h.state(), sim.state(), "end")
    assert sim.state()["switch_total_us"] > 0
    assert h.check() == 0


def test_step_parity_fig1_cost_model(L):
    """cost_model FIG1: a round is k candidates at t_tok, T~ = L t_tok / A."""
    tr, pool, tab = workload(80, 2048, 4, "bf16", seed=0x5F30, drift=True)
    kw = dict(BASE, k=4, seed=24, cost_model=1, t_tok_us=10_000, s1_up_us=160_000, t_ssm_us=0, t_llm_us=0)
    run_lockstep(L, kw, tr, pool, tab, B=4)


def test_update_select_standalone_switching_cost(L):
    """laps_update + laps_select as separate calls (stateless spec_verify between them)."""
    tr, pool, tab = workload(50, 2048, 4, "bf16", seed=0x5F40, drift=True)
    pr = synth.prompt_lengths(tr.n, 0x5F40)
    kw = dict(BASE, k=4, seed=25, **SWITCH)
    B, R = 5, tab.shape[1]
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V, prompt=pr)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, R
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    for step in range(3000):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        st = h.state()
        live = sel_g >= 0
        rounds = np.where(live, st["rounds"][np.maximum(sel_g, 0)], 0).astype(np.int32)
        slab = np.array([tab[i, _slab_round_index(int(rounds[b]), R)] if i >= 0 else 0
                         for b, i in enumerate(sel_g)], np.int32)
        req = np.where(live, sel_g, 0).astype(np.int32)
        _, na, _ = L.spec_verify(pool.p, pool.q, pool.draft, torch.as_tensor(req, device="cuda"),
                                 torch.as_tensor(rounds, device="cuda"), kw["seed"],
                                 slab=torch.as_tensor(slab, device="cuda"))
        h.laps_update(h.sel[:B], na)
        h.laps_select(B)
        sim.step(P, sel_o)
        if step % 5 == 0:
            compare_state(h.state(), sim.state(), step)
    compare_state(h.state(), sim.state(), "end")
    assert h.check() == 0


# ---------------------------------------------------------------- the side select's waiting list
def test_step_parity_n16384_resident(L):
    """configs[3]'s literal 16,384 concurrent requests resident on ONE GPU (B=512, V=128256,
    k=8): the side select merges the changed keys into its persistent waiting list instead
    of sorting all N every step.  Every step's batch, r and the whole state bit-exact."""
    c = synth.CONFIGS["c4"]
    n, B = 16384, 512
    tr = synth.make_trace(n, c["seed"] + 2, arrival="zero", length="uniform", len_min=512, len_max=4096,
                          beta_ab=(7, 3))
    pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=16, variants=2, seed=c["seed"],
                           device="cuda")
    tab = synth.slab_table(tr, 16, 2, R=16, seed=c["seed"] + 2)
    kw = dict(BASE, k=8, seed=c["seed"] + 2)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=128256, overlap=True)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, parallel=True)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 16
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(8):
        assert (h.sel.cpu().numpy() == sel_o).all(), f"step {step}: batch differs"
        h.laps_step(rows, B, n_accept=nacc)
        _, _, na_o, _ = sim.step(P, sel_o)
        assert (nacc.cpu().numpy() == na_o).all(), f"step {step}: r differs"
        compare_state(h.state(), sim.state(), step)
    assert h.check() == 0


@pytest.mark.parametrize("burst", [300, 1500])
def test_step_parity_admission_burst(L, burst):
    """Admissions after an idle period: a burst within the waiting list's per-step
    admission buffer (merged) and one beyond it (the list is rebuilt that step)."""
    n0 = 60
    tr = synth.make_trace(n0 + burst, 0xAB + burst, arrival="zero", length="uniform", len_min=6, len_max=40,
                          beta_ab=(4, 2), drift=True)
    tr.arrival_us[n0:] = 900_000          # all at 0.9 s: after the first requests have finished
    pool = synth.make_pool("f2", V=2048, k=4, dtype="bf16", n_buckets=8, variants=3, seed=burst, device="cuda")
    tab = synth.slab_table(tr, 8, 3, R=16, seed=burst)
    run_lockstep(L, dict(BASE, k=4, seed=33), tr, pool, tab, B=32, check_every=2, overlap=True)


def test_unnormalised_rows_set_the_mass_flag(L):
    """Rows that are not probabilities (every entry 0.5: mass V/2) must not wrap silently
    into the uint64 segment sums: lapssd_check reports ESTATE with flag 256 (E_MASS)."""
    tr, pool, tab = workload(20, 4096, 4, "bf16", seed=3, drift=False)
    kw = dict(BASE, k=4, seed=7)
    B = 4
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V)
    h.set_row_check(True)
    h.laps_select(B)
    p = torch.full((B, 5, 4096), 0.5, dtype=torch.bfloat16, device="cuda")
    q = torch.zeros(B, 4, 4096, dtype=torch.bfloat16, device="cuda")
    d = torch.zeros(B, 4, dtype=torch.int32, device="cuda")
    h.laps_step(L.Rows(p, q, d, None), B)
    with pytest.raises(L.LapssdError) as e:
        h.check()
    assert "0x100" in str(e.value) or e.value.status == -4
    # valid rows of the same shape do not set it
    h2 = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=pool.V)
    h2.set_row_check(True)
    h2.laps_select(B)
    h2.laps_step(L.Rows(torch.full_like(p, 1 / 4096), q, d, None), B)
    assert h2.check() == 0


def test_unnormalised_rows_flagged_without_the_row_check(L):
    """Without lapssd_set_row_check the finisher's total-mass check still flags a row
    pair whose residual mass exceeds 2 (rows of 0.25: V/4 per row, no lane wraps)."""
    tr, pool, tab = workload(20, 4096, 4, "bf16", seed=4, drift=False)
    h = L.Handle(L.SchedConfig(**dict(BASE, k=4, seed=7)), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=4,
                 V=4096)
    h.laps_select(4)
    p = torch.full((4, 5, 4096), 1 / 512, dtype=torch.bfloat16, device="cuda")   # mass 8 per row
    h.laps_step(L.Rows(p, torch.zeros(4, 4, 4096, dtype=torch.bfloat16, device="cuda"),
                       torch.zeros(4, 4, dtype=torch.int32, device="cuda"), None), 4)
    with pytest.raises(L.LapssdError):
        h.check()
