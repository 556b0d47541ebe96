"""Device side of the multi-GPU step (a8) on ONE GPU: two handles play ranks 0 and 1 of
world 2 (requests sharded by global id mod 2).  Each step every rank verifies its own
slots (spec_verify on its slabs) and updates them (laps_update); then each rank runs
laps_candidates, the candidate blocks are concatenated on the device (the all-gather's
result), and each rank runs laps_merge.  The sharded run must equal the single-rank
oracle request by request (the global top-B of per-rank top-B lists is the global top-B)."""
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


@pytest.mark.parametrize("policy,switch,G", [(0, False, 2), (2, False, 2), (0, True, 2), (3, True, 2),
                                             (0, True, 4), (0, False, 8), (3, True, 8)])
def test_two_handles_candidates_merge_equal_single_rank(L, policy, switch, G):
    """PIN-G on the device: G handles on one GPU as ranks 0..G-1 (G = 2, 4, 8)."""
    seed, B, R = 41, 6, 16
    tr = synth.make_trace(40, seed, arrival="poisson", rate_per_s=50.0, len_mu=np.log(30), len_sigma=0.6,
                          len_min=4, len_max=200, beta_ab=(3, 2), drift=True)
    pool = synth.make_pool("f2", V=2048, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed, device="cuda")
    tab = synth.slab_table(tr, 8, 3, R=R, seed=seed)
    kw = dict(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4, t_ssm_us=1 * MS,
              t_llm_us=10 * MS, seed=12)
    pr = None
    if switch:   # AMB-24: the step lasts one round plus the GLOBAL batch's switch-ins
        kw.update(switch_c0_us=2 * MS, switch_c1_us=12)
        pr = synth.prompt_lengths(tr.n, seed)
    # reference: one rank, oracle
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, R
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    sel_o, _ = sim.select(B)
    ref_steps = [sel_o.copy()]
    while not sim.state()["done"].all():
        sim.step(P, sel_o)
        ref_steps.append(sel_o.copy())
    ref = sim.state()
    # two GPU handles
    hs = []
    for g in range(G):
        sh = tr.shard(g, G)
        hs.append(L.Handle(L.SchedConfig(**kw), sh.arrival_us, sh.L_true, sh.L_pred, max_batch=B, V=2048,
                           rank=g, world=G, prompt=pr[g::G] if pr is not None else None))
    Cn = B
    cand = [torch.zeros(2 * Cn + 1, dtype=torch.int64, device="cuda") for _ in range(G)]
    sels = [torch.full((B,), -1, dtype=torch.int32, device="cuda") for _ in range(G)]

    def exchange():
        for g in range(G):
            hs[g].laps_candidates(Cn, cand[g])
        allc = torch.cat(cand)
        for g in range(G):
            hs[g].laps_merge(allc, Cn, B, sel=sels[g])

    exchange()
    for step in range(len(ref_steps) + 5):
        got = sorted(int(i) * G + g for g in range(G) for i in sels[g].cpu().numpy() if i >= 0)
        want = sorted(int(i) for i in ref_steps[step] if i >= 0) if step < len(ref_steps) else []
        assert got == want, f"step {step}"
        if all(h.state()["done"].all() for h in hs):
            break
        for g in range(G):
            s = sels[g].cpu().numpy()
            st = hs[g].state()
            live = s >= 0
            if not live.any():
                continue
            rounds = np.where(live, st["rounds"][np.maximum(s, 0)], 0)
            idx = np.where(rounds < R, rounds, R // 2 + (rounds - R // 2) % (R // 2))
            shard_tab = tab[g::G]
            slab = np.where(live, shard_tab[np.maximum(s, 0), idx], 0).astype(np.int32)
            req = np.where(live, s * G + g, 0).astype(np.int32)
            tok, na, _ = L.spec_verify(pool.p, pool.q, pool.draft, torch.as_tensor(req, device="cuda"),
                                       torch.as_tensor(rounds.astype(np.int32), device="cuda"), kw["seed"],
                                       slab=torch.as_tensor(slab, device="cuda"))
            hs[g].laps_update(sels[g], na)
        exchange()
    for g in range(G):
        st = hs[g].state()
        assert (st["C_us"] == ref["C_us"][g::G]).all()
        assert (st["acc_draft"] == ref["acc_draft"][g::G]).all()
        assert (st["switch_us"] == ref["switch_us"][g::G]).all()
        assert st["switch_total_us"] == ref["switch_total_us"]
        assert hs[g].check() == 0
    assert (ref["switch_total_us"] > 0) == switch


@pytest.mark.parametrize("switch", [False, True])
def test_laps_step_dist_one_rank_lockstep(L, monkeypatch, switch):
    """laps_step_dist end to end (verify + candidates + ncclAllGather + merge) with a
    one-rank NCCL communicator, step by step against the oracle: batch, r, state."""
    import torch.distributed as dist
    monkeypatch.setenv("MASTER_ADDR", "127.0.0.1")
    monkeypatch.setenv("MASTER_PORT", "29565" if switch else "29561")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = L.nccl_comm()
        seed, B, R = 43, 16, 16
        tr = synth.make_trace(120, seed, arrival="poisson", rate_per_s=60.0, len_mu=np.log(30),
                              len_sigma=0.6, len_min=4, len_max=200, beta_ab=(4, 2), drift=True)
        pool = synth.make_pool("f2", V=4096, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed,
                               device="cuda")
        tab = synth.slab_table(tr, 8, 3, R=R, seed=seed)
        kw = dict(K=4, s1_up_us=56 * MS, gamma=5, delta=0.05, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS,
                  seed=17)
        pr = None
        if switch:
            kw.update(switch_c0_us=2 * MS, switch_c1_us=12)
            pr = synth.prompt_lengths(tr.n, seed)
        P = pool.numpy()
        P["slab_tab"], P["R"] = tab, R
        sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
        h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=4096,
                     rank=0, world=1, prompt=pr, overlap=switch)
        rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
        Cn = B
        W = 2 * Cn + 1
        cand = torch.zeros(2 * W, dtype=torch.int64, device="cuda")
        h.laps_candidates(Cn, cand[:W])
        cand[W:].copy_(cand[:W])
        h.laps_merge(cand[W:], Cn, B)
        tok = torch.empty(B, 5, dtype=torch.int32, device="cuda")
        nacc = torch.empty(B, dtype=torch.int32, device="cuda")
        sel_o, _ = sim.select(B)
        for step in range(400):
            sel_g = h.sel[:B].cpu().numpy()
            assert (sel_g == sel_o).all(), f"step {step}: batch differs"
            if sim.state()["done"].all():
                break
            h.laps_step_dist(comm, rows, B, Cn, cand, tokens=tok, n_accept=nacc)
            _, tok_o, na_o, _ = sim.step(P, sel_o)
            live = sel_g >= 0
            assert (nacc.cpu().numpy()[live] == na_o[live]).all(), f"step {step}: r differs"
            assert (tok.cpu().numpy()[live] == tok_o[live]).all(), f"step {step}: tokens differ"
            if step % 4 == 0:
                g, o = h.state(), sim.state()
                for f in ("acc_tok", "acc_draft", "rounds", "E_us", "C_us", "level", "perceptible",
                          "pinned", "key", "switch_us"):
                    assert (np.asarray(g[f]) == np.asarray(o[f])).all(), f"step {step}: {f}"
                assert g["now_us"] == o["now_us"], f"step {step}: clock"
                assert g["switch_total_us"] == o["switch_total_us"], f"step {step}: switching"
        assert sim.state()["done"].all()
        assert h.check() == 0
        L.nccl_comm_destroy(comm)
    finally:
        dist.destroy_process_group()


def test_laps_step_dist_one_rank_graph_replay(L, monkeypatch):
    """The overlapped laps_step_dist captured in a CUDA graph and replayed (as bench.py
    times it at N > 1): the side stream's candidates -> all-gather -> merge chain and the
    programmatic edge from the merge kernel to the next verify launch; every step's r and
    the whole state after each replay against the oracle."""
    import torch.distributed as dist
    monkeypatch.setenv("MASTER_ADDR", "127.0.0.1")
    monkeypatch.setenv("MASTER_PORT", "29563")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = L.nccl_comm()
        seed, B, R, G, reps = 47, 64, 32, 6, 3
        tr = synth.make_trace(256, seed, arrival="zero", length="uniform", len_min=200, len_max=900,
                              beta_ab=(7, 3))
        pool = synth.make_pool("f2", V=32000, k=8, dtype="bf16", n_buckets=8, variants=4, seed=seed,
                               device="cuda")
        tab = synth.slab_table(tr, 8, 4, R=R, seed=seed)
        kw = dict(K=4, s1_up_us=72 * MS, gamma=5, delta=0.05, k=8, t_ssm_us=1 * MS, t_llm_us=10 * MS,
                  seed=19)
        P = pool.numpy()
        P["slab_tab"], P["R"] = tab, R
        sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred)
        h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=32000,
                     rank=0, world=1, overlap=True)
        rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
        Cn = B
        W = 2 * Cn + 1
        cand = torch.zeros(2 * W, dtype=torch.int64, device="cuda")
        h.laps_candidates(Cn, cand[:W])
        cand[W:].copy_(cand[:W])
        h.laps_merge(cand[W:], Cn, B)
        sel_o, _ = sim.select(B)
        h.laps_step_dist(comm, rows, B, Cn, cand)   # eager warm-up step
        sim.step(P, sel_o)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(G):
                h.laps_step_dist(comm, rows, B, Cn, cand)
        for rep in range(reps):
            g.replay()
            torch.cuda.synchronize()
            for _ in range(G):
                sim.step(P, sel_o)
            gs, os_ = h.state(), sim.state()
            for f in ("acc_tok", "acc_draft", "rounds", "E_us", "level", "perceptible", "pinned", "key"):
                assert (np.asarray(gs[f]) == np.asarray(os_[f])).all(), f"replay {rep}: {f}"
            assert gs["now_us"] == os_["now_us"]
            assert (h.sel[:B].cpu().numpy() == sel_o).all(), f"replay {rep}: next batch"
        assert h.check() == 0
        L.nccl_comm_destroy(comm)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("switch,host", [(False, False), (True, False), (False, True)])
def test_laps_step_peer_one_rank_lockstep(L, switch, host):
    """laps_step_peer (the exchange fused into the select kernel over peer memory) with
    one rank, step by step against the oracle; with host=True the slab pool lives in
    pinned host memory (bench.py's e2e at N > 1)."""
    seed, B, R = 53, 16, 16
    tr = synth.make_trace(120, seed, arrival="poisson", rate_per_s=60.0, len_mu=np.log(30),
                          len_sigma=0.6, len_min=4, len_max=200, beta_ab=(4, 2), drift=True)
    pool = synth.make_pool("f2", V=4096, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed, device="cuda")
    tab = synth.slab_table(tr, 8, 3, R=R, seed=seed)
    kw = dict(K=4, s1_up_us=56 * MS, gamma=5, delta=0.05, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=23)
    pr = None
    if switch:
        kw.update(switch_c0_us=2 * MS, switch_c1_us=12)
        pr = synth.prompt_lengths(tr.n, seed)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, R
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=4096, prompt=pr,
                 overlap=True)
    if host:
        rows = L.Rows(pool.p.cpu().pin_memory(), pool.q.cpu().pin_memory(), pool.draft.cpu().pin_memory(),
                      torch.as_tensor(tab, device="cuda"))
    else:
        rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
    Cn = B
    W = 2 * Cn + 1
    cand = torch.zeros(2 * W, dtype=torch.int64, device="cuda")
    h.laps_candidates(Cn, cand[:W])
    cand[W:].copy_(cand[:W])
    h.laps_merge(cand[W:], Cn, B)
    h.set_peers(Cn)
    tok = torch.empty(B, 5, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    sel_o, _ = sim.select(B)
    for step in range(400):
        sel_g = h.sel[:B].cpu().numpy()
        assert (sel_g == sel_o).all(), f"step {step}: batch differs"
        if sim.state()["done"].all():
            break
        h.laps_step_peer(rows, B, tokens=tok, n_accept=nacc)
        _, tok_o, na_o, _ = sim.step(P, sel_o)
        live = sel_g >= 0
        assert (nacc.cpu().numpy()[live] == na_o[live]).all(), f"step {step}: r differs"
        assert (tok.cpu().numpy()[live] == tok_o[live]).all(), f"step {step}: tokens differ"
        assert (nacc.cpu().numpy()[~live] == -1).all()
        if step % 4 == 0:
            g, o = h.state(), sim.state()
            for f in ("acc_tok", "acc_draft", "rounds", "E_us", "C_us", "level", "perceptible", "pinned", "key",
                      "switch_us"):
                assert (np.asarray(g[f]) == np.asarray(o[f])).all(), f"step {step}: {f}"
            assert g["now_us"] == o["now_us"] and g["switch_total_us"] == o["switch_total_us"]
    assert sim.state()["done"].all()
    assert h.check() == 0
