"""Randomised parity sweep of the fused step (laps_select + laps_step) against the oracle:
configurations drawn from a fixed seed over every scheduler knob the C-ABI exposes
(policy, K, M, S_1^up, gamma, delta, placement, pin rule, cost model, switching cost,
k, V including ragged vocabularies, bf16 / fp32 rows, batch size, arrival pattern,
overlapped launches, the persistent waiting list's admission paths).  Each configuration
runs in lockstep for up to 150 steps: batch, r, tokens and the whole state bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MS = 1000
FIELDS = ["acc_tok", "acc_draft", "rounds", "E_us", "T_total_us", "C_us", "x_us", "admitted", "done",
          "perceptible", "pinned", "level", "running", "key", "ring", "switch_us"]


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_17074_b200 as lib
    return lib


def draw_config(i):
    rng = np.random.default_rng(0xC0FFEE + i)
    k = int(rng.choice([1, 2, 3, 4, 6, 8]))
    dtype = str(rng.choice(["bf16", "f32"]))
    vq = 8 if dtype == "bf16" else 4                      # V * sizeof must be a multiple of 16
    V = int(rng.choice([512, 1000, 4096, 8200, 20000])) // vq * vq
    cost_model = int(rng.random() < 0.2)
    c_round = k * 1000 + 10_000 if cost_model == 0 else k * 5000
    kw = dict(policy=int(rng.integers(0, 4)), K=int(rng.integers(1, 9)), M=float(rng.choice([1.5, 2.0, 3.0])),
              s1_up_us=int(c_round * rng.choice([1, 2, 4, 8])), gamma=int(rng.integers(2, 7)),
              delta=float(rng.choice([0.0, 0.02, 0.05, 0.1, 0.3])), k=k, t_ssm_us=1000, t_llm_us=10_000,
              placement=int(rng.integers(0, 2)), pin_rule=int(rng.integers(0, 2)), seed=int(rng.integers(1, 2**40)),
              cost_model=cost_model, t_tok_us=5000 if cost_model else 0)
    if rng.random() < 0.5:
        kw.update(switch_c0_us=int(rng.integers(0, 3000)), switch_c1_us=int(rng.integers(0, 40)))
    n = int(rng.integers(20, 160))
    B = int(rng.choice([1, 2, 5, 8, 16, 33]))
    arrival = str(rng.choice(["poisson", "zero", "burst"]))
    return kw, dtype, V, n, B, arrival, bool(rng.random() < 0.5), int(rng.integers(0, 2**31))


@pytest.mark.parametrize("i", range(48))
def test_random_configuration_lockstep(L, i):
    kw, dtype, V, n, B, arrival, overlap, seed = draw_config(i)
    k = kw["k"]
    tr = synth.make_trace(n, seed, arrival="zero" if arrival != "poisson" else "poisson", rate_per_s=60.0,
                          len_mu=np.log(25), len_sigma=0.7, len_min=2, len_max=150, beta_ab=(3, 2), drift=True)
    if arrival == "burst":                               # a second wave after an idle period
        tr.arrival_us[n // 2:] = 3_000_000
    pool = synth.make_pool("f2", V=V, k=k, dtype=dtype, n_buckets=6, variants=2, seed=seed % 1000, device="cuda")
    tab = synth.slab_table(tr, 6, 2, R=12, seed=seed % 1000)
    pr = synth.prompt_lengths(n, seed % 1000)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=V, prompt=pr,
                 overlap=overlap)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, tab.shape[1]
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    tok = torch.empty(B, k + 1, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(150):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"config {i} step {step}: batch differs"
        if sim.state()["done"].all():
            break
        h.laps_step(rows, B, tokens=tok, n_accept=nacc)
        _, tok_o, na_o, _ = sim.step(P, sel_o)
        live = sel_g >= 0
        assert (nacc.cpu().numpy()[live] == na_o[live]).all(), f"config {i} step {step}: r differs"
        assert (tok.cpu().numpy()[live] == tok_o[live]).all(), f"config {i} step {step}: tokens differ"
        if step % 10 == 0:
            g, o = h.state(), sim.state()
            for f in FIELDS:
                assert (np.asarray(g[f]) == np.asarray(o[f])).all(), f"config {i} step {step}: {f}"
            assert (g["A"].view(np.uint64) == o["A"].view(np.uint64)).all()
            for f in ("now_us", "cursor", "prev_count", "step_cost_us", "switch_total_us"):
                assert g[f] == o[f], f"config {i} step {step}: {f}"
    assert h.check() == 0
