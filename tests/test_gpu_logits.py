"""GPU parity of spec_verify_logits (DESIGN.md AMB-30) against the
oracle on the same seeded logits: r, every emitted token and the 128-bit integer
residual mass Z, bit-exactly (every decision is an exact integer comparison)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2505_17074_b200 as lib
    return lib


def run_both(L, pool, B, seed, rng, k):
    S = pool.S
    slab = rng.integers(0, S, B).astype(np.int32)
    req = rng.integers(0, 1 << 20, B).astype(np.int32)
    rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
    dev = pool.p.device
    tok, na, z = L.spec_verify_logits(pool.p, pool.q, pool.draft, torch.as_tensor(req, device=dev),
                                      torch.as_tensor(rnd, device=dev), seed,
                                      slab=torch.as_tensor(slab, device=dev))
    P = pool.numpy()
    tok_o, r_o, z_o = oracle.verify_logits_batch(P["p"], P["q"], P["draft"], slab, req, rnd, seed)
    return tok.cpu().numpy(), na.cpu().numpy(), z.cpu().numpy().view(np.uint64), tok_o, r_o, z_o


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("V,k", [(1024, 4), (8200, 1), (32000, 6), (40008, 8)])
def test_spec_verify_logits_parity(L, dtype, V, k):
    pool = synth.make_logits_pool(V, k, dtype, n_buckets=4, variants=2, seed=V + k, device="cuda")
    rng = np.random.default_rng(V * 7 + k)
    tok, na, z, tok_o, r_o, z_o = run_both(L, pool, 24, 1234 + V, rng, k)
    assert (na == r_o).all()
    assert (z == z_o).all()
    assert (tok == tok_o).all()
    assert (na < k).any() and (k == 1 or len(set(na.tolist())) > 1)   # varied outcomes


def test_spec_verify_logits_config4_size(L):
    """configs[3] dimensions (V=128,256, k=8, bf16) at a batch the oracle finishes."""
    pool = synth.make_logits_pool(128256, 8, "bf16", n_buckets=4, variants=2, seed=44, device="cuda")
    rng = np.random.default_rng(44)
    tok, na, z, tok_o, r_o, z_o = run_both(L, pool, 12, 77, rng, 8)
    assert (na == r_o).all() and (z == z_o).all() and (tok == tok_o).all()


def test_spec_verify_logits_special_rows(L):
    """Equal logits (accept everything, bonus row), disjoint supports (reject at 0,
    residual = target) and a logit range wider than the exp cut-off (-28)."""
    V, k, S = 2048, 3, 3
    rng = np.random.default_rng(3)
    zp = (2 * rng.standard_normal((S, k + 1, V))).astype(np.float32)
    zq = zp[:, :k].copy()
    inA = rng.random(V) < 0.5
    zq[1] = np.where(inA, 0.0, -100.0)[None]
    zp[1] = np.where(inA, -100.0, 0.0)[None]
    zp[2, :, : V // 2] -= 60.0            # half the vocabulary below the cut-off
    draft = np.zeros((S, k), np.int32)
    draft[0] = rng.integers(0, V, k)
    draft[1] = np.flatnonzero(inA)[:k]
    draft[2] = rng.integers(V // 2, V, k)
    dev = "cuda"
    slab = np.array([0, 1, 2, 0, 1, 2], np.int32)
    req = np.arange(6, dtype=np.int32)
    rnd = np.zeros(6, np.int32)
    tok, na, z = L.spec_verify_logits(torch.as_tensor(zp, device=dev), torch.as_tensor(zq, device=dev),
                                      torch.as_tensor(draft, device=dev), torch.as_tensor(req, device=dev),
                                      torch.as_tensor(rnd, device=dev), 5,
                                      slab=torch.as_tensor(slab, device=dev))
    tok_o, r_o, z_o = oracle.verify_logits_batch(zp, zq, draft, slab, req, rnd, 5)
    na = na.cpu().numpy()
    assert (na == r_o).all() and (tok.cpu().numpy() == tok_o).all()
    assert (z.cpu().numpy().view(np.uint64) == z_o).all()
    assert na[0] == k and na[3] == k          # equal logits: every draft accepted
    assert na[1] == 0 and na[4] == 0          # disjoint: rejected at position 0
    assert not inA[tok_o[1, 0]]


def _call(L, pool, slab, req, rnd, seed, ws=None):
    dev = pool.p.device
    return L.spec_verify_logits(pool.p, pool.q, pool.draft, torch.as_tensor(req, device=dev),
                                torch.as_tensor(rnd, device=dev), seed, slab=torch.as_tensor(slab, device=dev),
                                workspace=ws)


def test_lazy_equals_every_row_form_large_batch(L, monkeypatch):
    """The one-launch lazy form (only the rows the tests consult are normalised; a work
    queue over a persistent grid) against the two-launch form that normalises every row,
    at more slots than the grid holds CTAs, and against the oracle on a sample of slots."""
    pool = synth.make_logits_pool(32000, 8, "bf16", n_buckets=8, variants=2, seed=91, device="cuda")
    rng = np.random.default_rng(91)
    B = 700
    slab = rng.integers(0, pool.S, B).astype(np.int32)
    req = rng.integers(0, 1 << 20, B).astype(np.int32)
    rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
    tok, na, z = [x.cpu().numpy() for x in _call(L, pool, slab, req, rnd, 9)]
    monkeypatch.setenv("LAPSSD_LOGITS_EAGER", "1")
    tok_e, na_e, z_e = [x.cpu().numpy() for x in _call(L, pool, slab, req, rnd, 9)]
    monkeypatch.delenv("LAPSSD_LOGITS_EAGER")
    assert (na == na_e).all() and (tok == tok_e).all() and (z == z_e).all()
    assert (na == 8).any() and (na == 0).any()
    P = pool.numpy()
    pick = rng.choice(B, 40, replace=False)
    tok_o, r_o, z_o = oracle.verify_logits_batch(P["p"], P["q"], P["draft"], slab[pick], req[pick], rnd[pick], 9)
    assert (na[pick] == r_o).all() and (tok[pick] == tok_o).all() and (z[pick].view(np.uint64) == z_o).all()


@pytest.mark.parametrize("B,k", [(1, 1), (1, 8), (5, 2), (300, 3)])
def test_lazy_queue_reused_workspace(L, B, k):
    """One workspace over several calls (the queue is re-zeroed per call), small and odd
    batches, and rows with every draft accepted (the bonus row p_k is then the last unit)."""
    V = 4096
    pool = synth.make_logits_pool(V, k, "f32", n_buckets=4, variants=2, seed=B + k, device="cuda")
    ws = torch.empty(L.spec_verify_logits_workspace_bytes(B, k, V, "f32"), dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(B * 31 + k)
    P = pool.numpy()
    for call in range(3):
        slab = rng.integers(0, pool.S, B).astype(np.int32)
        req = rng.integers(0, 1 << 20, B).astype(np.int32)
        rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
        tok, na, z = [x.cpu().numpy() for x in _call(L, pool, slab, req, rnd, 100 + call, ws)]
        pick = np.arange(B) if B <= 40 else rng.choice(B, 40, replace=False)
        tok_o, r_o, z_o = oracle.verify_logits_batch(P["p"], P["q"], P["draft"], slab[pick], req[pick], rnd[pick],
                                                     100 + call)
        assert (na[pick] == r_o).all() and (tok[pick] == tok_o).all()
        assert (z[pick].view(np.uint64) == z_o).all()


# fp32 logit gaps d = z - m for which rint(fl32(d log2e)) != rint(d log2e) (the product
# rounds onto a half-integer) AND E = floor(exphat(d) 2^40) then differs between the two:
# found by walking the ulp neighbourhoods of (h + 1/2) / log2e.  AMB-30 rounds the product
# first; an implementation that fuses d log2e + 1.5 2^23 into one FMA gets other masses.
_TIE_GAPS = [float.fromhex(h) for h in ("-0x1.a56ef8p+2", "-0x1.fe2804p+2", "-0x1.842994p+3")]


def test_logits_rint_of_the_rounded_product(L):
    """AMB-30's exphat takes n = rint(fl32(d log2e)): rows built from gaps where one fused
    rounding would change E must give the oracle's r, tokens and Z bit-exactly."""
    V, k, S = 1024, 2, 4
    rng = np.random.default_rng(17)
    zp = np.full((S, k + 1, V), -40.0, np.float32)
    zq = np.full((S, k, V), -40.0, np.float32)
    for s_ in range(S):
        for j in range(k + 1):
            idx = rng.permutation(V)
            zp[s_, j, idx[0]] = 0.0
            for t, g in enumerate(_TIE_GAPS):
                zp[s_, j, idx[1 + 200 * t:1 + 200 * (t + 1)]] = np.float32(g)
        for j in range(k):
            zq[s_, j] = zp[s_, j]
            zq[s_, j, rng.integers(0, V, 300)] = np.float32(_TIE_GAPS[s_ % 3])
    draft = rng.integers(0, V, (S, k)).astype(np.int32)
    draft[:, 0] = np.argmax(zp[:, 0], axis=1)          # a likely accepted first draft
    B = 16
    slab = np.arange(B, dtype=np.int32) % S
    req = np.arange(B, dtype=np.int32) * 7 + 1
    rnd = np.arange(B, dtype=np.int32)
    dev = "cuda"
    tok, na, z = L.spec_verify_logits(torch.as_tensor(zp, device=dev), torch.as_tensor(zq, device=dev),
                                      torch.as_tensor(draft, device=dev), torch.as_tensor(req, device=dev),
                                      torch.as_tensor(rnd, device=dev), 11, slab=torch.as_tensor(slab, device=dev))
    tok_o, r_o, z_o = oracle.verify_logits_batch(zp, zq, draft, slab, req, rnd, 11)
    assert (na.cpu().numpy() == r_o).all() and (tok.cpu().numpy() == tok_o).all()
    assert (z.cpu().numpy().view(np.uint64) == z_o).all()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_residual_near_ties_exact_path(L, dtype):
    """Draft logits equal to the target's except one unit of the format at the draft token
    (and at a few other entries): every residual entry is a near-tie p^ ~ q^ that the
    split-sum pass's fp32 screen cannot decide, so the exact 128-bit comparison decides it;
    logits span the whole exp range, so the masses E run from 0 to 2^40."""
    V, k, S = 8192, 4, 24
    rng = np.random.default_rng(17 if dtype == "bf16" else 18)
    zp = (rng.random((S, k + 1, V)) * -30.0).astype(np.float32)
    zp[:, :, 0] = 0.0
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    zp = torch.as_tensor(zp).to(tdt)
    zq = zp[:, :k].clone()
    draft = torch.as_tensor(rng.integers(1, V, (S, k)).astype(np.int32))
    step = 1 if dtype == "bf16" else 1 << 15          # units in the last place to move
    view = zq.view(torch.int16) if dtype == "bf16" else zq.view(torch.int32)
    for s in range(S):
        for j in range(k):
            x = int(draft[s, j])
            view[s, j, x] -= step * (1 + s % 3)        # logits are <= 0: a smaller magnitude is larger
            others = rng.integers(1, V, 4)
            view[s, j, others[:2]] += step
            view[s, j, others[2:]] -= step
    B = 384
    slab = np.arange(B, dtype=np.int32) % S
    req = rng.integers(0, 1 << 20, B).astype(np.int32)
    rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
    dev = "cuda"
    tok, na, z = L.spec_verify_logits(zp.to(dev), zq.to(dev), draft.to(dev), torch.as_tensor(req, device=dev),
                                      torch.as_tensor(rnd, device=dev), 23, slab=torch.as_tensor(slab, device=dev))
    zp_o, zq_o = synth.to_numpy_rows(zp), synth.to_numpy_rows(zq)
    tok_o, r_o, z_o = oracle.verify_logits_batch(zp_o, zq_o, draft.numpy(), slab, req, rnd, 23)
    na = na.cpu().numpy()
    assert (na == r_o).all()
    assert (z.cpu().numpy().view(np.uint64) == z_o).all()
    assert (tok.cpu().numpy() == tok_o).all()
    assert (na < k).sum() >= 20                       # enough residual draws


@pytest.mark.parametrize("offset", [7950.0, -7990.0, 9000.0, -30000.0])
def test_large_row_max_bf16(L, offset):
    """Row maxima near and beyond the packed floor's range (|m| <= 8000: the floor
    round_down_bf16(m - 28) is coarse there; beyond it the kernel keeps the fp32 clamp):
    bf16 logits offset by a constant, spread over the exp cut-off."""
    V, k, S = 4096, 3, 6
    rng = np.random.default_rng(int(abs(offset)))
    base = rng.standard_normal((S, k + 1, V)).astype(np.float32) * 12.0
    zp = torch.as_tensor(base + offset).to(torch.bfloat16)
    zq = torch.as_tensor(base[:, :k] + offset + rng.standard_normal((S, k, V)).astype(np.float32) * 2.0).to(
        torch.bfloat16)
    qs = torch.softmax(zq.float(), -1).reshape(S * k, V)
    draft = torch.multinomial(qs, 1, generator=torch.Generator().manual_seed(5)).view(S, k).to(torch.int32)
    B = 48
    slab = (np.arange(B) % S).astype(np.int32)
    req = rng.integers(0, 1 << 20, B).astype(np.int32)
    rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
    dev = "cuda"
    tok, na, z = L.spec_verify_logits(zp.to(dev), zq.to(dev), draft.to(dev), torch.as_tensor(req, device=dev),
                                      torch.as_tensor(rnd, device=dev), 31, slab=torch.as_tensor(slab, device=dev))
    tok_o, r_o, z_o = oracle.verify_logits_batch(synth.to_numpy_rows(zp), synth.to_numpy_rows(zq), draft.numpy(),
                                                 slab, req, rnd, 31)
    na = na.cpu().numpy()
    assert (na == r_o).all()
    assert (z.cpu().numpy().view(np.uint64) == z_o).all()
    assert (tok.cpu().numpy() == tok_o).all()


@pytest.mark.parametrize("policy", [0, 3])
def test_laps_sd_driven_by_logits(L, policy):
    """The LAPS-SD step from LOGITS through the C-ABI: spec_verify_logits on the batch the
    handle selected (request id and round as the Philox counter, the round's slab), then
    laps_update with its r and laps_select -- in lockstep with the oracle (verify_logits ->
    Sim.update -> Sim.select) over whole traces, every state field compared."""
    from test_gpu_step import BASE, compare_state
    V, k, B = 4096, 4, 6
    tr = synth.make_trace(60, 0x10C1 + policy, arrival="poisson", rate_per_s=80.0, len_mu=np.log(24),
                          len_sigma=0.6, len_min=2, len_max=96, drift=True)
    pool = synth.make_logits_pool(V, k, "bf16", n_buckets=8, variants=2, seed=0x10C1, device="cuda")
    R = 8
    tab = synth.slab_table(tr, 8, 2, R=R, seed=0x10C1)
    kw = dict(BASE, k=k, seed=31, policy=policy, switch_c0_us=1_000, switch_c1_us=10)
    pr = synth.prompt_lengths(tr.n, 0x10C1)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=V, prompt=pr)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    zp, zq, dr = synth.to_numpy_rows(pool.p), synth.to_numpy_rows(pool.q), pool.draft.cpu().numpy()
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    seed = 0x5EED
    for step in range(4000):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        st = h.state()
        live = sel_g >= 0
        ids = np.maximum(sel_g, 0)
        rounds = np.where(live, st["rounds"][ids], 0).astype(np.int32)
        slab = np.where(live, tab[ids, rounds % R], 0).astype(np.int32)
        req = ids.astype(np.int32)
        _, na, _ = L.spec_verify_logits(pool.p, pool.q, pool.draft, torch.as_tensor(req, device="cuda"),
                                        torch.as_tensor(rounds, device="cuda"), seed,
                                        slab=torch.as_tensor(slab, device="cuda"))
        _, r_o, _ = oracle.verify_logits_batch(zp, zq, dr, slab, req, rounds, seed)
        assert (na.cpu().numpy()[live] == r_o[live]).all(), f"step {step}: r differs"
        h.laps_update(h.sel[:B], na)
        h.laps_select(B)
        sim.update(sel_o, np.where(live, r_o, 0).astype(np.int32))
        sel_o, _ = sim.select(B)
        if step % 4 == 0:
            compare_state(h.state(), sim.state(), step)
    assert sim.state()["done"].all()
    compare_state(h.state(), sim.state(), "end")
    assert h.check() == 0


@pytest.mark.parametrize("B,dtype", [(1, "bf16"), (3, "f32"), (64, "bf16")])
def test_lazy_speculation_long_chains(L, B, dtype):
    """k = 16 with high-acceptance slabs and few slots: almost every CTA of the persistent
    grid waits for work, so rows are run one and two positions ahead speculatively (and
    many of them turn out not to be needed); results against the oracle, and repeated calls
    on one workspace give identical results."""
    V, k = 2048, 16
    pool = synth.make_logits_pool(V, k, dtype, n_buckets=4, variants=2, seed=300 + B, device="cuda")
    rng = np.random.default_rng(300 + B)
    hi = np.arange(pool.S)[np.arange(pool.S) // 2 >= 2]   # the two high-acceptance buckets
    slab = rng.choice(hi, B).astype(np.int32)
    req = rng.integers(0, 1 << 20, B).astype(np.int32)
    rnd = rng.integers(0, 1 << 12, B).astype(np.int32)
    P = pool.numpy()
    if B == 1:   # a round whose chain is long (the oracle picks it)
        for c in range(4096):
            rnd[0] = c
            if oracle.verify_logits_batch(P["p"], P["q"], P["draft"], slab, req, rnd, 41)[1][0] >= 8:
                break
    ws = torch.empty(L.spec_verify_logits_workspace_bytes(B, k, V, dtype), dtype=torch.uint8, device="cuda")
    outs = [[x.cpu().numpy() for x in _call(L, pool, slab, req, rnd, 41, ws)] for _ in range(3)]
    for o in outs[1:]:
        assert all((a == b).all() for a, b in zip(o, outs[0]))
    tok, na, z = outs[0]
    tok_o, r_o, z_o = oracle.verify_logits_batch(P["p"], P["q"], P["draft"], slab, req, rnd, 41)
    assert (na == r_o).all() and (tok == tok_o).all() and (z.view(np.uint64) == z_o).all()
    assert na.max() >= 4


def _slab_round_index(t, R):
    h = R // 2
    return t if t < R else (R - 1 if h == 0 else h + (t - h) % h)


@pytest.mark.parametrize("policy,dtype", [(0, "bf16"), (3, "bf16"), (0, "f32")])
def test_laps_step_logits_lockstep(L, policy, dtype):
    """laps_step_logits (one C-ABI call: the handle's batch verified from logits with its
    own request ids, rounds and slabs, then update and select) against the oracle
    (verify_logits on the same slots -> Sim.update -> Sim.select) over whole traces."""
    from test_gpu_step import BASE, compare_state
    V, k, B, R = 4096, 4, 6, 8
    tr = synth.make_trace(60, 0x10D1 + policy, arrival="poisson", rate_per_s=80.0, len_mu=np.log(24),
                          len_sigma=0.6, len_min=2, len_max=96, drift=True)
    pool = synth.make_logits_pool(V, k, dtype, n_buckets=8, variants=2, seed=0x10D1, device="cuda")
    tab = synth.slab_table(tr, 8, 2, R=R, seed=0x10D1)
    kw = dict(BASE, k=k, seed=37, policy=policy, switch_c0_us=1_000, switch_c1_us=10)
    pr = synth.prompt_lengths(tr.n, 0x10D1)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=V, prompt=pr)
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    zp, zq, dr = synth.to_numpy_rows(pool.p), synth.to_numpy_rows(pool.q), pool.draft.cpu().numpy()
    ws = torch.empty(L.laps_step_logits_workspace_bytes(B, k, V, dtype), dtype=torch.uint8, device="cuda")
    tok = torch.empty(B, k + 1, dtype=torch.int32, device="cuda")
    na = torch.empty(B, dtype=torch.int32, device="cuda")
    sel_o, _ = sim.select(B)
    h.laps_select(B)
    for step in range(4000):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        rounds_o = sim.state()["rounds"]
        live = sel_o >= 0
        ids = np.maximum(sel_o, 0)
        rnd = np.where(live, rounds_o[ids], 0).astype(np.int32)
        slab = np.array([tab[i, _slab_round_index(int(rnd[b]), R)] if i >= 0 else 0 for b, i in enumerate(sel_o)],
                        np.int32)
        tok_o, r_o, _ = oracle.verify_logits_batch(zp, zq, dr, slab, ids.astype(np.int32), rnd, kw["seed"])
        h.laps_step_logits(rows, B, tokens=tok, n_accept=na, workspace=ws)
        na_g, tok_g = na.cpu().numpy(), tok.cpu().numpy()
        assert (na_g[live] == r_o[live]).all() and (na_g[~live] == -1).all(), f"step {step}: r differs"
        assert (tok_g[live] == tok_o[live]).all(), f"step {step}: tokens differ"
        sim.update(sel_o, np.where(live, r_o, 0).astype(np.int32))
        sel_o, _ = sim.select(B)
        if step % 4 == 0:
            compare_state(h.state(), sim.state(), step)
    assert sim.state()["done"].all()
    compare_state(h.state(), sim.state(), "end")
    assert h.check() == 0
