"""The multi-GPU exchange protocol (include/lapssd.h laps_step_dist) on CPU:
world_size 2 over gloo, each rank holding its shard of requests (global id mod G),
computing with the oracle, and exchanging C candidate keys + its next arrival per step
with a real torch.distributed all-gather.  The sharded run must reproduce the
single-rank run request by request (PIN-G), because the global top-B of the union of
per-rank top-B lists is the global top-B."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

MS = 1000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload(seed):
    tr = synth.make_trace(40, seed, arrival="poisson", rate_per_s=50.0, len_mu=np.log(30), len_sigma=0.6,
                          len_min=4, len_max=200, beta_ab=(3, 2), drift=True)
    pool = synth.make_pool("f2", V=64, k=4, dtype="f32", n_buckets=8, variants=3, seed=seed)
    P = pool.numpy()
    P["slab_tab"] = synth.slab_table(tr, 8, 3, R=16, seed=seed)
    P["R"] = 16
    return tr, P


def _cfg(policy):
    return oracle.SchedConfig(policy=policy, K=4, s1_up_us=30 * MS, gamma=3, delta=0.05, k=4,
                              t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=12)


def _rank_main(rank, world, port, policy, seed, B, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, P = _workload(seed)
        local = tr.shard(rank, world)
        tab = np.ascontiguousarray(P["slab_tab"][rank::world])
        cfg = _cfg(policy)
        sim = oracle.Sim(cfg, local.arrival_us, local.L_true, local.L_pred, rank=rank, world=world)
        Cn = B  # C = min(B_global, max n_local): same on every rank

        def exchange():
            keys, nxt = sim.candidates(Cn)
            mine = torch.tensor(np.concatenate([keys.view(np.int64), [nxt]]), dtype=torch.int64)
            allw = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(allw, mine)
            all_keys = np.concatenate([a[:Cn].numpy().view(np.uint64) for a in allw])
            all_next = np.array([int(a[Cn]) for a in allw], np.int64)
            sel, own, g = sim.merge(all_keys, Cn, all_next, B)
            return sel

        sel = exchange()
        for _ in range(10_000):
            # verify + update this rank's slots (no select inside)
            na = np.full(B, -1, np.int32)
            for b, i in enumerate(sel):
                if i < 0:
                    continue
                rnd = sim.state()["rounds"][i]
                idx = rnd if rnd < 16 else 8 + (rnd - 8) % 8
                slab = tab[i, idx]
                _, o = oracle.verify_request(P["p"][slab], P["q"][slab], P["draft"][slab],
                                             i * world + rank, rnd, cfg.seed)
                na[b] = o.r
            sim.update(sel, na)
            sel = exchange()
            done = torch.tensor([int(sim.state()["done"].all())])
            dist.all_reduce(done, op=dist.ReduceOp.MIN)
            if int(done):
                break
        st = sim.state()
        out[rank] = (st["C_us"].copy(), st["acc_draft"].copy(), st["rounds"].copy())
    finally:
        dist.destroy_process_group()


def _reference(policy, seed, B):
    tr, P = _workload(seed)
    sim = oracle.Sim(_cfg(policy), tr.arrival_us, tr.L_true, tr.L_pred)
    sel, _ = sim.select(B)
    while not sim.state()["done"].all():
        sim.step(P, sel)
    st = sim.state()
    return st["C_us"], st["acc_draft"], st["rounds"]


@pytest.mark.parametrize("policy", [oracle.POL_LAPSSD, oracle.POL_LPSJF])
def test_two_rank_gloo_equals_single_rank(policy):
    B, seed, world = 6, 31, 2
    ref = _reference(policy, seed, B)
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    mp.spawn(_rank_main, args=(world, port, policy, seed, B, out), nprocs=world, join=True)
    for rank in range(world):
        C_us, acc, rounds = out[rank]
        assert (C_us == ref[0][rank::world]).all()
        assert (acc == ref[1][rank::world]).all()
        assert (rounds == ref[2][rank::world]).all()
