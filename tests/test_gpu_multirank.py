"""The product's multi-rank step with a REAL exchange between processes (PIN-G):
two processes share cuda:0 as ranks 0 and 1 of a gloo group.  Each rank holds the requests
with global id mod 2 == rank in its own handle and every step runs the library's fused
laps_step_candidates (verify + update of its slots, its candidate block of keys, switch-in
costs and next arrival) through the C-ABI; the blocks are exchanged with
torch.distributed.all_gather (gloo, host tensors) and each rank runs laps_merge.  The
sharded run must equal the single-rank oracle request by request: every step's global
batch, and every request's final state (C_i, tokens, rounds, attained service,
switching time) -- the global top-B of per-rank top-B lists is the global top-B."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MS = 1000
G = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup(seed, switch):
    tr = synth.make_trace(48, seed, arrival="poisson", rate_per_s=40.0, len_mu=np.log(30), len_sigma=0.6,
                          len_min=4, len_max=160, beta_ab=(4, 2), drift=True)
    tab = synth.slab_table(tr, 8, 3, R=16, seed=seed)
    kw = dict(K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=31)
    pr = None
    if switch:
        kw.update(switch_c0_us=2 * MS, switch_c1_us=12)
        pr = synth.prompt_lengths(tr.n, seed)
    return tr, tab, kw, pr


def _step_results(sel, nacc, tok, rank):
    """This rank's live slots of one step: [global id, r, tokens...] rows; every slot past
    the rank's count must report r = -1."""
    r, t = nacc.cpu().numpy(), tok.cpu().numpy()
    live = sel >= 0
    assert (r[~live] == -1).all()
    return np.concatenate([(sel[live].astype(np.int64) * G + rank)[:, None], r[live, None], t[live]], axis=1)


def _pack(rs, B):
    out = np.full((len(rs), B, 7), -2, dtype=np.int64)
    for t, a in enumerate(rs):
        out[t, :len(a)] = a
    return out


def _worker(rank, port, policy, switch, seed, B, out_dir):
    import torch.distributed as dist

    import paper_2505_17074_b200 as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    torch.cuda.set_device(0)
    tr, tab, kw, pr = _setup(seed, switch)
    kw["policy"] = policy
    pool = synth.make_pool("f2", V=2048, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed, device="cuda")
    sh = tr.shard(rank, G)
    h = L.Handle(L.SchedConfig(**kw), sh.arrival_us, sh.L_true, sh.L_pred, max_batch=B, V=2048, rank=rank,
                 world=G, prompt=pr[rank::G] if pr is not None else None)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(np.ascontiguousarray(tab[rank::G]), device="cuda"))
    Cn = B
    W = 2 * Cn + 1
    cand = torch.zeros(W, dtype=torch.int64, device="cuda")

    def exchange():
        parts = [torch.zeros(W, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(parts, cand.cpu())
        h.laps_merge(torch.cat(parts).cuda(), Cn, B)

    h.laps_candidates(Cn, cand)
    exchange()
    batches, rs = [], []
    tok = torch.empty(B, 5, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(5000):
        sel = h.sel[:B].cpu().numpy()
        batches.append(sorted(int(i) * G + rank for i in sel if i >= 0))
        done = torch.tensor([int(h.state()["done"].all())])
        dist.all_reduce(done)
        if int(done) == G:
            break
        h.laps_step_candidates(rows, B, Cn, cand, tokens=tok, n_accept=nacc)
        rs.append(_step_results(sel, nacc, tok, rank))
        exchange()
    st = h.state()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), steps=len(batches), rs=_pack(rs, B),
             batches=np.array([np.array(b + [-1] * (B - len(b))) for b in batches]),
             **{f: st[f] for f in ("C_us", "acc_tok", "rounds", "E_us", "x_us", "switch_us", "level",
                                   "perceptible")},
             now_us=st["now_us"], switch_total_us=st["switch_total_us"], flags=h.check())
    dist.destroy_process_group()


@pytest.mark.parametrize("policy,switch", [(0, True), (3, True), (0, False)])
def test_two_processes_gloo_exchange_equal_single_rank(policy, switch, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    seed, B = 0x6D00 + policy, 6
    mp.start_processes(_worker, args=(_free_port(), policy, switch, seed, B, str(tmp_path)), nprocs=G,
                       start_method="spawn", join=True)
    _compare_with_oracle(tmp_path, policy, switch, seed, B)


def _compare_with_oracle(tmp_path, policy, switch, seed, B):
    tr, tab, kw, pr = _setup(seed, switch)
    kw["policy"] = policy
    pool = synth.make_pool("f2", V=2048, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed, device="cuda")
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 16
    sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, prompt=pr)
    sel, _ = sim.select(B)
    ref = [sorted(int(i) for i in sel if i >= 0)]
    ref_r = []   # per step: global id -> (r, tokens)
    while not sim.state()["done"].all():
        ids = sel.copy()
        _, tok_o, na_o, _ = sim.step(P, sel)
        ref_r.append({int(i): (int(na_o[j]), tok_o[j]) for j, i in enumerate(ids) if i >= 0})
        ref.append(sorted(int(i) for i in sel if i >= 0))
    o = sim.state()
    R = [np.load(os.path.join(tmp_path, f"rank{g}.npz")) for g in range(G)]
    assert all(int(r["flags"]) == 0 for r in R)
    n_steps = min(int(r["steps"]) for r in R)
    assert n_steps == len(ref), (n_steps, len(ref))
    for t in range(n_steps):   # the global batch of every step (PIN-G)
        got = sorted(int(x) for r in R for x in r["batches"][t] if x >= 0)
        assert got == ref[t], f"step {t}: {got} != {ref[t]}"
    for t in range(n_steps - 1):   # every slot's r and tokens (the verify outputs of each rank)
        got = {int(row[0]): (int(row[1]), row[2:]) for r in R for row in r["rs"][t] if row[0] >= 0}
        assert sorted(got) == sorted(ref_r[t]), f"step {t}: slots"
        for i, (rr, tt) in got.items():
            ro, to = ref_r[t][i]
            assert rr == ro and (tt == to).all(), f"step {t} request {i}: r/tokens differ"
    for g, r in enumerate(R):
        for f in ("C_us", "acc_tok", "rounds", "E_us", "x_us", "switch_us", "level", "perceptible"):
            assert (r[f] == np.asarray(o[f])[g::G]).all(), f"rank {g}: {f} differs"
        assert int(r["now_us"]) == o["now_us"]
        assert int(r["switch_total_us"]) == o["switch_total_us"]
    assert (o["switch_total_us"] > 0) == switch


def _peer_worker(rank, port, policy, switch, seed, B, out_dir):
    """As _worker, but every step is laps_step_peer: the candidate blocks travel through
    peer memory (torch CUDA IPC between the two processes) inside the select kernel."""
    import torch.distributed as dist

    import paper_2505_17074_b200 as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    torch.cuda.set_device(0)
    tr, tab, kw, pr = _setup(seed, switch)
    kw["policy"] = policy
    pool = synth.make_pool("f2", V=2048, k=4, dtype="bf16", n_buckets=8, variants=3, seed=seed, device="cuda")
    sh = tr.shard(rank, G)
    h = L.Handle(L.SchedConfig(**kw), sh.arrival_us, sh.L_true, sh.L_pred, max_batch=B, V=2048, rank=rank,
                 world=G, prompt=pr[rank::G] if pr is not None else None)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(np.ascontiguousarray(tab[rank::G]), device="cuda"))
    Cn = B
    W = 2 * Cn + 1
    cand = torch.zeros(W, dtype=torch.int64, device="cuda")
    h.laps_candidates(Cn, cand)
    parts = [torch.zeros(W, dtype=torch.int64) for _ in range(G)]
    dist.all_gather(parts, cand.cpu())
    h.laps_merge(torch.cat(parts).cuda(), Cn, B)
    h.set_peers(Cn)
    batches, rs = [], []
    tok = torch.empty(B, 5, dtype=torch.int32, device="cuda")
    nacc = torch.empty(B, dtype=torch.int32, device="cuda")
    for step in range(5000):
        sel = h.sel[:B].cpu().numpy()
        batches.append(sorted(int(i) * G + rank for i in sel if i >= 0))
        done = torch.tensor([int(h.state()["done"].all())])
        dist.all_reduce(done)
        if int(done) == G:
            break
        h.laps_step_peer(rows, B, tokens=tok, n_accept=nacc)
        rs.append(_step_results(sel, nacc, tok, rank))
    torch.cuda.synchronize()
    st = h.state()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), steps=len(batches), rs=_pack(rs, B),
             batches=np.array([np.array(b + [-1] * (B - len(b))) for b in batches]),
             **{f: st[f] for f in ("C_us", "acc_tok", "rounds", "E_us", "x_us", "switch_us", "level",
                                   "perceptible")},
             now_us=st["now_us"], switch_total_us=st["switch_total_us"], flags=h.check())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("policy,switch", [(0, True), (3, False)])
def test_two_processes_peer_exchange_equal_single_rank(policy, switch, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    seed, B = 0x6E00 + policy, 6
    mp.start_processes(_peer_worker, args=(_free_port(), policy, switch, seed, B, str(tmp_path)), nprocs=G,
                       start_method="spawn", join=True)
    _compare_with_oracle(tmp_path, policy, switch, seed, B)
