#!/usr/bin/env python
"""bench.py -- the LAPS-SD batched speculative-decoding step on B200.

One STEP = one pass of the whole hot path over one batch: spec_verify of every
selected request (rejection sampling) with the fused LAPS-SD
state update, then admission + priority keys + top-B selection of the
next batch -- the C-ABI call laps_step (laps_step_peer for N>1: the
candidate exchange fused into the select kernel over NVLink peer memory; laps_step_dist,
the NCCL form, with --nccl-exchange).

Workload = BASELINE.json configs[3] ("16,384 concurrent requests, V=128,256, k=8,
bf16, batch 512, sharded over 8 B200"): 2,048 resident requests and B=512 per GPU
(weak scaling, DESIGN.md s.7), all arriving at t=0, acceptance ~ Beta(7,3), output
lengths ~ U[512, 4096], probability rows from a 4.5 GB F2 slab pool (inputs larger than
L2; every step reads ~255 MB of rows it did not read in the previous step).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "verified draft tokens/s at V=128k,k=8 on 1/2/4/8 B200; % of HBM peak"
UNIT = "verified draft tokens/s"
WORKLOAD = ("configs[3]: 16,384 concurrent requests over 8 GPUs -> 2,048 resident + batch 512 "
            "per GPU (weak scaling), V=128,256, k=8, bf16 p/q, Beta(7,3) acceptance, "
            "L~U[512,4096], all arrive at t=0, global top-B exchanged over peer memory for N>1")
SCHED = dict(K=4, s1_up_us=4 * (8 * 1000 + 10_000), M=2.0, gamma=5, delta=0.05, k=8,
             t_ssm_us=1000, t_llm_us=10_000, placement=0, pin_rule=0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-per-gpu", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--V", type=int, default=128256)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--buckets", type=int, default=64)
    ap.add_argument("--variants", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--graph-steps", type=int, default=20, help="steps per captured CUDA graph (0 = eager)")
    ap.add_argument("--no-profile", action="store_true", help="no per-kernel events at all")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-path", action="store_true",
                    help="N=1 only: time the NCCL form of the N>1 step (laps_step_dist) with a one-rank communicator")
    ap.add_argument("--peer-path", action="store_true",
                    help="N=1 only: time the N>1 step (laps_step_peer, exchange fused over peer memory) with one rank")
    ap.add_argument("--nccl-exchange", action="store_true",
                    help="N>1: laps_step_dist (candidates -> ncclAllGather -> merge kernel) instead of laps_step_peer")
    ap.add_argument("--traffic-file", default=os.path.join(ROOT, "profiles", "verify_dram.json"))
    ap.add_argument("--workload", choices=["c4", "mc", "logits", "logits_step", "draft", "tree", "c2", "c3"],
                    default="c4",
                    help="c4 = configs[3] (the headline); mc = configs[4] Monte-Carlo traces; "
                    "logits = SURVEY 8(f) f1, spec_verify_logits at configs[3] dimensions; "
                    "draft / tree = SURVEY 8(f) f4, spec_draft_sample / spec_verify_tree; "
                    "c2 / c3 = configs[1] / configs[2] at full size, run to completion with oracle parity")
    ap.add_argument("--tree-nodes", type=int, default=16, help="f4 tree: nodes per request")
    ap.add_argument("--tree-width", type=int, default=3, help="f4 tree: max children per node")
    ap.add_argument("--mc-traces", type=int, default=8192, help="configs[4]: traces (whole job)")
    ap.add_argument("--mc-n", type=int, default=512, help="configs[4]: requests per trace")
    ap.add_argument("--mc-variants", type=int, default=256, help="configs[4]: slab variants per bucket")
    ap.add_argument("--rho", type=float, default=None, help="c2 / c3: offered load (default: the config's)")
    ap.add_argument("--policy", type=int, default=0, help="c2 / c3: scheduling policy (0 LAPS-SD, 1 FCFS, "
                    "2 LP-SJF, 3 LAS)")
    ap.add_argument("--no-parity", action="store_true", help="c2 / c3: skip the oracle run")
    ap.add_argument("--mc-policies", default="0", help="comma list of policies run to completion "
                    "for mean JCT (e.g. 0,1,2,3; empty: throughput only)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING.md):
    NVML polled every ~1 ms from a thread (nvidia-smi's 100 ms cadence would see a
    few-ms timed region at most once).  Falls back to nvidia-smi if NVML is missing."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.samples, self.stop_flag, self.h = [], False, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.h = None
        self.active = False
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def _poll(self):
        while not self.stop_flag:
            if self.h is not None and self.active:
                try:
                    sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                    rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((sm, rs))
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.001)

    def start(self):
        self.active = True

    def stop(self):
        self.active = False
        self.stop_flag = True
        self.t.join(1.0)
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "NVML, 1 ms poll during the timed region"}


# --------------------------------------------------------------------------- workload
def build_workload(args, rank, world, device, pool_slabs=None):
    n_total = args.n_per_gpu * world
    tr = synth.make_trace(n_total, synth.CONFIGS["c4"]["seed"], arrival="zero", length="uniform",
                          len_min=512, len_max=4096, beta_ab=(7, 3))
    local = tr.shard(rank, world)
    buckets, variants = args.buckets, args.variants
    if pool_slabs is not None:
        variants = max(1, pool_slabs // buckets)
    pool = synth.make_pool("f2", V=args.V, k=args.k, dtype="bf16", n_buckets=buckets,
                           variants=variants, seed=synth.CONFIGS["c4"]["seed"], device=device)
    tab_full = synth.slab_table(tr, buckets, variants, R=64, seed=synth.CONFIGS["c4"]["seed"])
    tab = np.ascontiguousarray(tab_full[rank::world])
    return tr, local, pool, tab


def upload_graphs(graphs):
    """cuGraphUpload every captured graph before the timed region, so the first replay
    does not pay the upload of its executable graph to the device."""
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return False
    s = torch.cuda.current_stream().cuda_stream
    ok = True
    for g in graphs:
        rc = cu.cuGraphUpload(ctypes.c_void_p(g.raw_cuda_graph_exec()), ctypes.c_void_p(s))
        ok &= rc == 0
    torch.cuda.synchronize()
    return ok


def build_digest() -> str:
    """sha256 of liblapssd.so's sources, header and nvcc flags: identifies the build an
    ncu capture under profiles/ belongs to."""
    import hashlib
    sys.path.insert(0, os.path.join(ROOT, "paper_2505_17074_b200"))
    import build as lb
    h = hashlib.sha256(" ".join(lb.FLAGS).encode())
    for f in sorted(lb.sources() + [os.path.join(lb.CSRC, x) for x in ("lapssd_internal.cuh", "select_core.cuh")]
                    + [os.path.join(ROOT, "include", "lapssd.h")]):
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def algorithmic_bytes(n_acc: np.ndarray, V: int, k: int, s: int = 2) -> float:
    """SURVEY s.8(d): per verified slot (r<k ? 2 : 1) V s row bytes + 2 s min(r+1,k)
    gathered scalars + 4k draft bytes.  n_acc holds r per slot (-1 = empty)."""
    r = n_acc[n_acc >= 0].astype(np.int64)
    rows = np.where(r < k, 2, 1) * V * s
    gathers = 2 * s * np.minimum(r + 1, k)
    return float((rows + gathers + 4 * k).sum())


# --------------------------------------------------------------------------- ours
def run_ours(args):
    import paper_2505_17074_b200 as L

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B_local = args.batch
    B = B_local * world                        # global batch (weak scaling)
    tr, local, pool, tab = build_workload(args, rank, world, dev)
    cfg = L.SchedConfig(**SCHED, seed=synth.CONFIGS["c4"]["seed"])
    # the slab pool is static, so consecutive verify launches may overlap (lapssd.h:
    # lapssd_set_step_overlap)
    h = L.Handle(cfg, local.arrival_us, local.L_true, local.L_pred, max_batch=B, V=args.V,
                 rank=rank, world=world, overlap=True)
    tab_d = torch.as_tensor(tab, device=dev)
    rows = L.Rows(pool.p, pool.q, pool.draft, tab_d)
    comm = cand = None
    peer = False
    Cn = min(B, args.n_per_gpu)
    W = 2 * Cn + 1                             # candidate block: keys, switch costs, next arrival
    if world > 1:
        cand = torch.zeros((world + 1) * W, dtype=torch.int64, device=dev)
        h.laps_candidates(Cn, cand[:W])
        dist.all_gather_into_tensor(cand[W:], cand[:W])
        h.laps_merge(cand[W:], Cn, B)
        if not args.nccl_exchange:   # the exchange fused into the select kernel over NVLink peer memory
            h.set_peers(Cn)
            peer = True
            # safety net: if the peer exchange does not complete (device watchdog), every
            # rank falls back to the NCCL form on a fresh handle
            h.laps_step_peer(rows, B)
            torch.cuda.synchronize()
            ok = torch.tensor([1.0 if h.check_flags() == 0 else 0.0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() < 1.0:
                print("bench: peer exchange failed, falling back to laps_step_dist", file=sys.stderr, flush=True)
                peer = False
                h = L.Handle(cfg, local.arrival_us, local.L_true, local.L_pred, max_batch=B, V=args.V,
                             rank=rank, world=world, overlap=True)
                h.laps_candidates(Cn, cand[:W])
                dist.all_gather_into_tensor(cand[W:], cand[:W])
                h.laps_merge(cand[W:], Cn, B)
        if not peer:
            comm = L.nccl_comm()
    elif args.peer_path:
        cand = torch.zeros(2 * W, dtype=torch.int64, device=dev)
        h.laps_candidates(Cn, cand[:W])
        cand[W:].copy_(cand[:W])
        h.laps_merge(cand[W:], Cn, B)
        h.set_peers(Cn)
        peer = True
    elif args.dist_path:
        # the N>1 step (laps_step_dist: candidates + ncclAllGather + merge) on one rank, to
        # time its cost on the one GPU available; a one-rank gloo group only carries the
        # NCCL unique id
        import torch.distributed as tdist
        tdist.init_process_group("gloo", rank=0, world_size=1,
                                 init_method=f"tcp://127.0.0.1:{29500 + os.getpid() % 1000}")
        comm = L.nccl_comm()
        tdist.destroy_process_group()
        cand = torch.zeros(2 * W, dtype=torch.int64, device=dev)
        h.laps_candidates(Cn, cand[:W])
        cand[W:].copy_(cand[:W])
        h.laps_merge(cand[W:], Cn, B)
    else:
        h.laps_select(B)
    G = min(args.graph_steps, args.steps) if args.graph_steps > 0 else 0
    plain = world == 1 and not peer and comm is None   # laps_step: the library's per-kernel events
    # r of every step: rows [0, warmup) warm-up, [warmup, warmup + steps) the timed steps,
    # the last row scratch (the instrumented replay)
    hist = torch.full((args.warmup + args.steps + 1, B), -1, dtype=torch.int32, device=dev)
    scratch_row = args.warmup + args.steps

    def step(t):
        if peer:
            h.laps_step_peer(rows, B, n_accept=hist[t])
        elif comm is not None:
            h.laps_step_dist(comm, rows, B, Cn, cand, n_accept=hist[t])
        else:
            h.laps_step(rows, B, n_accept=hist[t])

    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    for t in range(args.warmup):
        step(t)
    torch.cuda.synchronize()
    graphs = []
    launches_per_step = None
    g_prof = None
    if G:
        # timed steps: replays of UNINSTRUMENTED captured graphs of G steps each (the host
        # enqueue cost is removed; the side stream's fork/join is in the graph), each graph
        # writing its steps' r to their own rows of hist (the roofline's bytes are those of
        # exactly the timed steps)
        if plain:
            h.profile(0)
        c0 = L.launch_count()
        for g0 in range(0, args.steps, G):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for t in range(g0, min(g0 + G, args.steps)):
                    step(args.warmup + t)
            graphs.append(gr)
        launches_per_step = (L.launch_count() - c0) / args.steps
        if plain and not args.no_profile:
            # a second graph of G steps with the library's per-kernel CUDA events,
            # replayed right after the timed region (events add graph nodes, so they are
            # kept out of the timed replays)
            h.profile(G)
            g_prof = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_prof):
                for t in range(G):
                    step(scratch_row)
        torch.cuda.synchronize()
        upload_graphs(graphs + ([g_prof] if g_prof is not None else []))
    elif plain and not args.no_profile:
        h.profile(args.steps)
    st0 = h.state()
    launches0 = L.launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record()
    if G:
        for g in graphs:
            g.replay()
    else:
        for t in range(args.steps):
            step(args.warmup + t)
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = L.launch_count() - launches0
    if G:
        launches = int(round(launches_per_step * args.steps))
    st1 = h.state()  # before the instrumented replay, which advances the state further
    clk = clocks.stop()
    device_error = None
    try:  # a device-side watchdog expiry or contract violation invalidates the run
        h.check()
    except Exception as exc:  # noqa: BLE001 (reported in the JSON line, not swallowed)
        device_error = str(exc)
        print(f"bench: device error in the timed region: {device_error}", file=sys.stderr, flush=True)
    prof_ms = None
    if g_prof is not None:
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        g_prof.replay()
        p1.record()
        torch.cuda.synchronize()
        prof_ms = p0.elapsed_time(p1)
    ms = e0.elapsed_time(e1)
    verified_local = int((st1["rounds"] - st0["rounds"]).sum())
    ms_t = torch.tensor([ms, float(verified_local)], dtype=torch.float64, device=dev)
    if dist:
        mx = ms_t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = ms_t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, verified = float(mx[0]), int(sm[1])
    else:
        ms_max, verified = ms, verified_local
    value = verified * args.k / (ms_max * 1e-3)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16 rows; fp32 residual + exact "
           "Q4.60 integer CDF; fp64 scheduler", "data": "synthetic",
           "config": {"workload": WORKLOAD, "N_resident_per_gpu": args.n_per_gpu,
                      "B_per_gpu": B_local, "B_global": B, "V": args.V, "k": args.k,
                      "pool": f"F2 zipf, {pool.S} slabs x {(2 * args.k + 1) * args.V * 2 / 1e6:.2f} MB",
                      "l2": "inputs larger than L2 (4.5 GB slab pool, ~255 MB of rows per step)",
                      "parallelism": f"dp{world}: requests sharded by id mod {world}"
                      + ("; laps_step_dist path" if comm is not None and world == 1 else "")
                      + ("; laps_step_peer path" if peer and world == 1 else "")
                      + ("; global top-B via NCCL all-gather of candidate keys" if world > 1 and comm is not None else "")
                      + ("; global top-B exchanged inside the select kernel over NVLink peer memory (laps_step_peer)"
                         if world > 1 and peer else "")},
           "verified_per_step": verified / args.steps, "gpu_launches": launches, "clocks": clk}
    if world > 1 or peer or comm is not None:
        # the a8 exchange: each rank's candidate block of 2C+1 words (+ a tag
        # word on the peer path) to every rank, once per step
        blk = (2 * Cn + 2 if peer else 2 * Cn + 1) * 8
        out["exchange"] = {"path": "laps_step_peer (in-kernel, NVLink peer stores)" if peer else "ncclAllGather",
                           "bytes_sent_per_rank_per_step": blk * world, "bytes_received_per_rank_per_step": blk * world,
                           "per_step_at_nvlink5_900GBps_us": blk * world / 900e9 * 1e6,
                           "note": "latency-bound: the bytes need ~0.1 us of NVLink-5 bandwidth; the step time "
                                   "above includes the exchange (it runs beside the verify kernel)"}
    if device_error:
        out["device_error"] = device_error
    if not args.no_profile:
        v_ms = s_ms = p_ms = None
        n_prof = 1
        if plain:
            v_ms, s_ms, p_ms, n_prof = h.profile_read()
        # algorithmic bytes of exactly the timed steps (their r_b rows of hist); at N > 1
        # each rank's verify launch reads its own slots' rows: the mean over ranks
        n_acc = hist[args.warmup:args.warmup + args.steps].cpu().numpy()
        alg = algorithmic_bytes(n_acc, args.V, args.k)
        per_launch = alg / n_acc.shape[0]
        if dist:
            pl = torch.tensor([per_launch], dtype=torch.float64, device=dev)
            dist.all_reduce(pl, op=dist.ReduceOp.SUM)
            per_launch = float(pl[0]) / world
        avg_v = v_ms / n_prof if v_ms is not None else None
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        peak = peaks.get("hbm_gbs")
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback (B200_PROFILING.md)"
        peak = peak or 6650.0
        # One verify launch per step on the launching stream, back to back (programmatic
        # dependent launch; the select runs beside it on the side stream): the launch
        # interval in the UNINSTRUMENTED timed region (CUDA events around it) is the
        # kernel's sustained per-launch duration.  The instrumented replay's per-kernel
        # events serialise consecutive launches, so they are reported beside it.
        interval_ms = ms_max / args.steps
        achieved = per_launch / (interval_ms * 1e-3) / 1e9
        # ncu DRAM bytes of one verify launch, only if captured for THIS build (the
        # digest of the library's sources and flags), else null
        traffic, traffic_note = None, "no ncu capture on file"
        if os.path.exists(args.traffic_file):
            try:
                tf = json.load(open(args.traffic_file))
                if tf.get("build_digest") == build_digest():
                    traffic, traffic_note = tf.get("dram_bytes_per_launch"), tf.get("source")
                else:
                    traffic_note = "ncu capture on file is for another build: not reported"
            except (OSError, ValueError):
                traffic = None
        kern = "laps_step" if world == 1 and not peer and comm is None else (
            "laps_step_peer" if peer else "laps_step_dist")
        out["roofline"] = {"kernel": f"verify_kernel<bf16> ({kern}; per rank)" if world > 1
                           else f"verify_kernel<bf16> ({kern})", "bound": "hbm",
                           "achieved": achieved, "peak": peak, "unit": "GB/s",
                           "frac": achieved / peak, "peak_source": peak_src,
                           "frac_of_8TBs": achieved / 8000.0,
                           "algorithmic_bytes_per_launch": per_launch, "traffic": traffic,
                           "traffic_source": traffic_note,
                           "verify_interval_ms": interval_ms,
                           "verify_ms_avg_instrumented": avg_v,
                           "select_ms_avg": s_ms / n_prof if s_ms is not None else None,
                           "presort_end_ms_avg": p_ms / n_prof if p_ms is not None else None,
                           "timing": (f"achieved = algorithmic bytes per verify launch / launch interval in the "
                                      f"timed region ({args.steps} steps as replays of an uninstrumented "
                                      f"CUDA graph of {G} steps, one verify launch per step, CUDA events "
                                      f"around it); per-kernel CUDA events from a second, "
                                      f"instrumented graph of {G} steps replayed right after "
                                      f"({prof_ms / G * 1e3 if prof_ms else 0:.1f} us/step instrumented)"
                                      if G and plain else
                                      f"achieved = mean over ranks of the algorithmic bytes per verify launch / "
                                      f"launch interval (max over ranks) in the timed region" if not plain
                                      else "eager laps_step calls, events on every step")}
        if not args.no_e2e:
            if plain:
                out["e2e"] = run_e2e(args, L, local, pool, cfg, dev)
            elif world > 1 or peer:
                out["e2e"] = run_e2e_multi(args, L, local, pool, tab, cfg, dev, dist, rank, world, Cn, peer)
        if not args.no_cpu_baseline and plain:
            out["cpu_baseline"] = run_cpu_baseline(args, local, pool, tab, cfg)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        L.nccl_comm_destroy(comm)
    if dist:
        dist.destroy_process_group()


def run_e2e(args, L, local, pool, cfg, dev):
    """The same metric through the C-ABI with HOST buffers: each step's batch rows (batch
    layout p[B,k+1,V], q[B,k,V], draft[B,k]) live in pinned host memory and laps_step
    reads them in place (UVA: the bulk copies and gathers pull only the bytes the step
    needs -- the accepted drafts' probabilities and the residual row pair -- across
    PCIe); the batch, accepted counts and tokens are read back every step."""
    B, k, V = args.batch, args.k, args.V
    h = L.Handle(cfg, local.arrival_us, local.L_true, local.L_pred, max_batch=B, V=V)
    host = []
    for j in range(2):
        idx = (torch.arange(B) + j * B) % pool.S
        hp, hq, hd = (pool.p[idx.to(dev)].cpu().pin_memory(), pool.q[idx.to(dev)].cpu().pin_memory(),
                      pool.draft[idx.to(dev)].cpu().pin_memory())
        host.append((hp, hq, hd, L.Rows(hp, hq, hd, None)))
    tok = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
    nacc = torch.empty(B, dtype=torch.int32, device=dev)
    out_sel = torch.empty(B, dtype=torch.int32).pin_memory()
    out_nacc = torch.empty(B, dtype=torch.int32).pin_memory()
    out_tok = torch.empty(B, k + 1, dtype=torch.int32).pin_memory()
    h.laps_select(B)
    s = torch.cuda.current_stream()
    d2h = out_sel.numel() * 4 + out_nacc.numel() * 4 + out_tok.numel() * 4
    h2d = []

    def one(j):
        h.laps_step(host[j % 2][3], B, tokens=tok, n_accept=nacc)
        out_sel.copy_(h.sel[:B], non_blocking=True)
        out_nacc.copy_(nacc, non_blocking=True)
        out_tok.copy_(tok, non_blocking=True)
        s.synchronize()
        r = out_nacc.numpy()
        live = r >= 0
        # bytes the step read from host memory: the rows it streamed and the gathered
        # draft probabilities (2 per position tested) and drafts
        h2d.append(int((np.where(r[live] < k, 2, 1) * V * 2 + 4 * k + 2 * 2 * np.minimum(r[live] + 1, k)).sum()))

    one(0)
    h2d.clear()
    st0 = h.state()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for j in range(args.e2e_steps):
        one(j + 1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    verified = int((h.state()["rounds"] - st0["rounds"]).sum())
    h.close()
    return {"value": verified * k / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": int(np.mean(h2d)) if h2d else 0,
            "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "ms_per_step": ms / args.e2e_steps,
            "path": "laps_step C-ABI; batch-layout rows in pinned host memory read in place over PCIe "
                    "(UVA zero-copy bulk copies and gathers: only the bytes the step needs); batch, "
                    "accepted counts and tokens read back to pinned host memory every step"}


def run_e2e_multi(args, L, local, pool, tab, cfg, dev, dist, rank, world, Cn, peer, host_slabs=64):
    """e2e at N > 1: every rank runs the multi-GPU step through the C-ABI (laps_step_peer,
    or laps_step_dist on the NCCL form) on a fresh handle of its shard, with the slab pool
    in PINNED HOST memory (the first host_slabs slabs; the table maps every request onto
    them) read in place over PCIe, and reads back its batch, accepted counts and tokens
    every step.  Time: CUDA events per rank, the max over ranks; bytes: summed over ranks."""
    B = args.batch * world
    k, V = args.k, args.V
    S = min(host_slabs, pool.S)
    hp, hq, hd = pool.p[:S].cpu().pin_memory(), pool.q[:S].cpu().pin_memory(), pool.draft[:S].cpu().pin_memory()
    rows = L.Rows(hp, hq, hd, torch.as_tensor(np.ascontiguousarray(tab % S), device=dev))
    h = L.Handle(cfg, local.arrival_us, local.L_true, local.L_pred, max_batch=B, V=V, rank=rank, world=world,
                 overlap=True)
    W = 2 * Cn + 1
    cand = torch.zeros((world + 1) * W, dtype=torch.int64, device=dev)
    h.laps_candidates(Cn, cand[:W])
    if dist:
        dist.all_gather_into_tensor(cand[W:], cand[:W])
    else:
        cand[W:].copy_(cand[:W])
    h.laps_merge(cand[W:], Cn, B)
    comm = None
    if peer:
        h.set_peers(Cn)
    else:
        comm = L.nccl_comm()
    tok = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
    nacc = torch.empty(B, dtype=torch.int32, device=dev)
    out_sel = torch.empty(B, dtype=torch.int32).pin_memory()
    out_nacc = torch.empty(B, dtype=torch.int32).pin_memory()
    out_tok = torch.empty(B, k + 1, dtype=torch.int32).pin_memory()
    s = torch.cuda.current_stream()
    h2d = []

    def one():
        if peer:
            h.laps_step_peer(rows, B, tokens=tok, n_accept=nacc)
        else:
            h.laps_step_dist(comm, rows, B, Cn, cand, tokens=tok, n_accept=nacc)
        out_sel.copy_(h.sel[:B], non_blocking=True)
        out_nacc.copy_(nacc, non_blocking=True)
        out_tok.copy_(tok, non_blocking=True)
        s.synchronize()
        r = out_nacc.numpy()
        r = r[r >= 0]
        h2d.append(int((np.where(r < k, 2, 1) * V * 2 + 4 * k + 2 * 2 * np.minimum(r + 1, k)).sum()))

    one()
    h2d.clear()
    st0 = h.state()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    verified = int((h.state()["rounds"] - st0["rounds"]).sum())
    err = h.check_flags()
    agg = torch.tensor([ms, float(verified), float(np.mean(h2d) if h2d else 0.0), float(err)],
                       dtype=torch.float64, device=dev)
    mx, sm = agg.clone(), agg.clone()
    if dist:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if comm is not None:
        L.nccl_comm_destroy(comm)
    if dist:
        dist.barrier()
    h.close()
    ms_max = float(mx[0])
    d2h = (B + B + B * (k + 1)) * 4 * world
    res = {"value": float(sm[1]) * k / (ms_max * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(sm[2]), "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
           "ms_per_step": ms_max / args.e2e_steps,
           "path": f"{'laps_step_peer' if peer else 'laps_step_dist'} C-ABI on every rank; the slab pool "
                   f"({S} slabs) in pinned host memory read in place over PCIe (UVA: only the bytes the step "
                   "needs); each rank's batch, accepted counts and tokens read back every step; max over "
                   "ranks of the CUDA-event time, bytes summed over ranks"}
    if float(mx[3]) != 0:
        res["device_error_flags"] = int(mx[3])
    return res


def host_info():
    """The host the CPU oracle ran on: logical CPUs and the lscpu model name."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def omp_threads():
    return int(os.environ.get("OMP_NUM_THREADS") or os.cpu_count() or 1)


def run_cpu_baseline(args, local, pool, tab, cfg_gpu, budget_s=None, batch=None):
    """The oracle as it stands on a bounded sample of the same workload (the first steps of
    the same request set, same rows, same config): the -fopenmp build of the same source on
    all host cores (a step's requests verified in parallel), and the plain single-thread
    build beside it."""
    import oracle

    budget_s = budget_s or args.cpu_seconds
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, tab.shape[1]
    ocfg = oracle.SchedConfig(**SCHED, seed=cfg_gpu.seed)
    B = batch or args.batch
    res = {}
    for parallel, share in ((True, 0.6), (False, 0.4)):
        sim = oracle.Sim(ocfg, local.arrival_us, local.L_true, local.L_pred, parallel=parallel)
        sel, _ = sim.select(B)
        t0 = time.perf_counter()
        steps = verified = 0
        while time.perf_counter() - t0 < budget_s * share:
            verified += int((sel >= 0).sum())
            sim.step(P, sel)
            steps += 1
        el = time.perf_counter() - t0
        res[parallel] = (verified * args.k / el, steps, el)
    (v_all, n_all, el_all), (v_one, n_one, el_one) = res[True], res[False]
    return {"value": v_all, "unit": UNIT, "cores": omp_threads(), "kind": "oracle",
            "sample": f"first {n_all} steps of the bench workload ({B} verifications per step, "
                      f"V={args.V}, k={args.k}, bf16), oracle/lapssd_oracle.c built with -fopenmp "
                      f"(per-request verify loop on {omp_threads()} threads), {el_all:.1f} s",
            "single_thread": {"value": v_one, "cores": 1, "sample": f"first {n_one} steps, plain build, "
                              f"{el_one:.1f} s"},
            "host": host_info()}



# --------------------------------------------------------------------------- configs[4]
MC_METRIC = METRIC
MC_WORKLOAD = ("configs[4]: Monte-Carlo sweep, 8,192 independent traces x 512 requests, batch 1 per "
               "trace (P:84), V=32,000, k=4, bf16 p/q, Poisson arrivals at rho=0.8, lognormal(ln 128, "
               "0.8) lengths, Beta(4,2) acceptance; traces sharded in contiguous blocks over ranks")
MC_SCHED = dict(K=4, s1_up_us=4 * (4 * 1000 + 10_000), M=2.0, gamma=5, delta=0.05, k=4,
                t_ssm_us=1000, t_llm_us=10_000, placement=0, pin_rule=0)


def build_mc(args, rank, world, dev):
    c = synth.CONFIGS["c5"]
    T_local = args.mc_traces // world
    rate = synth.mc_rate_for_load(c["rho"], c["k"], MC_SCHED["t_ssm_us"], MC_SCHED["t_llm_us"],
                                  len_mu=c["len_mu"], len_sigma=c["len_sigma"], beta_ab=c["beta_ab"])
    w = synth.make_mc_workload(T_local, args.mc_n, c["seed"] + rank, rate_per_s=rate, len_mu=c["len_mu"],
                               len_sigma=c["len_sigma"], len_min=c["len_min"], len_max=c["len_max"],
                               beta_ab=c["beta_ab"], n_buckets=c["n_buckets"], variants=args.mc_variants,
                               R=c["R"])
    pool = synth.make_pool("f2", V=c["V"], k=c["k"], dtype="bf16", n_buckets=c["n_buckets"],
                           variants=args.mc_variants, seed=c["seed"], device=dev)
    return w, pool


def run_mc(args):
    import paper_2505_17074_b200 as L

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    c = synth.CONFIGS["c5"]
    k, V = c["k"], c["V"]
    w, pool = build_mc(args, rank, world, dev)
    T = w.T
    cfg = L.SchedConfig(**MC_SCHED, policy=0, seed=c["seed"])
    mc = L.MCHandle(cfg, w.offsets, w.arrival_us, w.L_true, w.L_pred, V=V)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(w.slab_tab, device=dev))
    mc.select(rows)
    G = max(1, min(args.graph_steps or 20, args.steps))
    hist = torch.full((G, T), -1, dtype=torch.int32, device=dev)
    for t in range(args.warmup):
        mc.step(rows, n_accept=hist[t % G])
    torch.cuda.synchronize()
    c0 = L.launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for t in range(G):
            mc.step(rows, n_accept=hist[t])
    launches_per_step = (L.launch_count() - c0) / G
    reps = max(1, args.steps // G)
    steps = reps * G
    st0 = mc.state()[0]["rounds"].astype(np.int64).sum()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    n_acc = hist.cpu().numpy()
    verified_local = int(mc.state()[0]["rounds"].astype(np.int64).sum() - st0)
    t = torch.tensor([ms, float(verified_local)], dtype=torch.float64, device=dev)
    if dist:
        mx, sm = t.clone(), t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, verified = float(mx[0]), int(sm[1])
    else:
        ms_max, verified = ms, verified_local
    alg_step = algorithmic_bytes(n_acc, V, k) / G
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs") or 6650.0
    achieved = alg_step / (ms / steps * 1e-3) / 1e9
    out = {"metric": MC_METRIC, "value": verified * k / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
           "steps": steps, "warmup": args.warmup, "ms_per_step": ms_max / steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16 rows; fp32 residual + exact Q4.60 "
           "integer CDF; fp64 scheduler", "data": "synthetic",
           "config": {"workload": MC_WORKLOAD, "traces_per_gpu": T, "requests_per_trace": args.mc_n,
                      "V": V, "k": k, "pool": f"F2, {pool.S} slabs x {(2 * k + 1) * V * 2 / 1e6:.2f} MB",
                      "l2": f"inputs larger than L2 ({pool.S * (2 * k + 1) * V * 2 / 1e9:.1f} GB slab pool)",
                      "parallelism": f"dp{world}: traces in contiguous blocks, no collective"},
           "verified_per_step": verified / steps, "gpu_launches": int(round(launches_per_step * steps)),
           "clocks": clk,
           "roofline": {"kernel": "whole MC step (verify sub-launches + warp-per-trace update/select)",
                        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": None,
                        "algorithmic_bytes_per_step": alg_step,
                        "timing": f"{steps} steps as replays of a CUDA graph of {G} steps; step-level "
                                  "bytes / step time (a lower bound for the verify kernel's own rate)"}}
    if args.mc_policies:
        out["jct"] = mc_jct(args, L, w, pool, rows, dev, [int(x) for x in args.mc_policies.split(",")])
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = mc_cpu_baseline(args, w, pool, cfg)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def estimator_accuracy(st, w, sched):
    """SURVEY 8(f) f3 (the paper's Fig. 7 analogue): for every request
    that became perceptible and completed, the Eq. (6) estimate fixed at stabilisation
    (T~_i, from the engine's state) against the service it actually received (E_i =
    rounds x round cost).  Reported twice: as the engine computed it (with the predicted
    length L_pred, lognormal error sigma 0.3) and with the true length (the error of the
    acceptance-rate part alone, T~ rescaled by L_true / L_pred)."""
    m = st["perceptible"].astype(bool) & st["done"].astype(bool)
    est = st["T_total_us"][m].astype(np.float64)
    real = st["E_us"][m].astype(np.float64)
    lp = np.asarray(w.L_pred)[m].astype(np.float64)
    lt = np.asarray(w.L_true)[m].astype(np.float64)
    err = np.abs(est - real) / real
    err_true = np.abs(est * lt / lp - real) / real
    return {"requests": int(m.sum()), "perceptible_frac": float(m.mean()),
            "mape_with_L_pred": float(err.mean()), "mape_with_L_true": float(err_true.mean()),
            "signed_mean_with_L_true": float(((est * lt / lp - real) / real).mean()),
            "paper_context": "6.84 % overall on an L20 with a learned length predictor (P:315)"}


def mc_jct(args, L, w, pool, rows, dev, policies):
    """Run every trace to completion under each policy (same traces, same rows, same
    seeds: common random numbers) and report the mean JCT (C_i - r_i)."""
    res = {}
    c = synth.CONFIGS["c5"]
    for pol in policies:
        cfg = L.SchedConfig(**MC_SCHED, policy=pol, seed=c["seed"])
        mc = L.MCHandle(cfg, w.offsets, w.arrival_us, w.L_true, w.L_pred, V=c["V"])
        mc.select(rows)
        G = 64
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(G):
                act = mc.step(rows)
        steps, t0 = 0, time.perf_counter()
        while True:
            g.replay()
            steps += G
            if int(act.item()) == 0 or steps > 2_000_000:
                break
        el = time.perf_counter() - t0
        st = mc.state()[0]
        jct = (st["C_us"] - w.arrival_us).astype(np.float64)
        r = {"mean_jct_ms": float(jct.mean() / 1e3), "steps": steps, "seconds": el,
             "all_done": bool(st["done"].all())}
        if pol == 0:
            r["estimator"] = estimator_accuracy(st, w, MC_SCHED)
        res[["LAPS-SD", "FCFS", "LP-SJF", "LAS"][pol]] = r
        del mc
    return res


def mc_cpu_baseline(args, w, pool, cfg):
    """The oracle on a bounded sample of the same traces (64 of the 8,192):
    whole traces one after another on one thread, and the same traces spread over all host
    cores (Python threads; the oracle's C step releases the GIL, so traces run in parallel)."""
    import concurrent.futures as cf

    import oracle

    P = pool.numpy()
    ocfg = oracle.SchedConfig(**MC_SCHED, policy=0, seed=cfg.seed)

    def run_trace(t, deadline):
        a, lt, lp, tab = w.trace(t)
        sim = oracle.Sim(ocfg, a, lt, lp, trace=t)
        Pt = dict(P, slab_tab=np.ascontiguousarray(tab), R=tab.shape[1])
        sel, _ = sim.select(1)
        n = 0
        while time.perf_counter() < deadline:
            ran = int(sel[0] >= 0)
            cnt = sim.step(Pt, sel)[0]
            n += ran
            if cnt == 0 and sim.state()["done"].all():
                break
        return n

    budget = args.cpu_seconds
    n_tr = min(64, w.T)
    t0 = time.perf_counter()
    v1 = tr1 = 0
    while tr1 < n_tr and time.perf_counter() - t0 < 0.4 * budget:
        v1 += run_trace(tr1, t0 + 0.4 * budget)
        tr1 += 1
    el1 = time.perf_counter() - t0
    threads = omp_threads()
    t1 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        vs = list(ex.map(lambda t: run_trace(t, t1 + 0.6 * budget), range(n_tr)))
    el = time.perf_counter() - t1
    return {"value": sum(vs) * MC_SCHED["k"] / el, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{n_tr} traces (batch 1 each) of the same workload on {threads} threads "
                      f"(whole traces, or until {0.6 * budget:.0f} s), {sum(vs)} verifications, "
                      f"oracle/lapssd_oracle.c, {el:.1f} s",
            "single_thread": {"value": v1 * MC_SCHED["k"] / el1, "cores": 1,
                              "sample": f"{tr1} traces one after another, {v1} verifications, {el1:.1f} s"},
            "host": host_info()}

# --------------------------------------------------------------------------- reference arm
def run_logits_step(args):
    """f1 inside the LAPS-SD step: Handle.laps_step_logits on the configs[3] workload per GPU
    (2,048 resident, B = 512, V = 128,256, k = 8), the rows a bf16 LOGITS slab pool with the
    same bucket / variant structure as the headline's probability pool.  One GPU (the step's
    select is local; N > 1 would need the global merge)."""
    import paper_2505_17074_b200 as L
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    B, k, V = args.batch, args.k, args.V
    tr = synth.make_trace(args.n_per_gpu, synth.CONFIGS["c4"]["seed"], arrival="zero", length="uniform",
                          len_min=512, len_max=4096, beta_ab=(7, 3))
    pool = synth.make_logits_pool(V, k, "bf16", n_buckets=args.buckets, variants=args.variants,
                                  seed=synth.CONFIGS["c4"]["seed"], device=dev)
    tab = synth.slab_table(tr, args.buckets, args.variants, R=64, seed=synth.CONFIGS["c4"]["seed"])
    cfg = L.SchedConfig(**SCHED, seed=synth.CONFIGS["c4"]["seed"])
    h = L.Handle(cfg, tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=V)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device=dev))
    ws = torch.empty(L.laps_step_logits_workspace_bytes(B, k, V, "bf16"), dtype=torch.uint8, device=dev)
    G = max(1, min(args.graph_steps or 1, args.steps))
    tok = torch.empty(G, B, k + 1, dtype=torch.int32, device=dev)
    na = torch.empty(G, B, dtype=torch.int32, device=dev)
    h.laps_select(B)
    for t in range(max(args.warmup, 3)):
        h.laps_step_logits(rows, B, tokens=tok[t % G], n_accept=na[t % G], workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    lc0 = L.launch_count()
    with torch.cuda.graph(g):
        for t in range(G):
            h.laps_step_logits(rows, B, tokens=tok[t], n_accept=na[t], workspace=ws)
    launches_per_step = (L.launch_count() - lc0) / G
    reps = max(1, args.steps // G)
    g.replay()
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clocks.start()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    steps = reps * G
    r = na.cpu().numpy()
    verified = float((r >= 0).sum()) / G
    value = verified * k * steps / (ms * 1e-3)
    row = V * 2
    rr = r[r >= 0]
    alg = float(((2 * np.minimum(rr + 1, k) + (rr == k)) * row).sum()) / G
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs") or 6650.0
    achieved = alg / (ms / steps * 1e-3) / 1e9
    assert h.check() == 0
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": steps, "warmup": args.warmup,
           "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "bf16 logits; fixed-op fp32 exp, exact 2^40 integer softmax masses; fp64 scheduler",
           "data": "synthetic",
           "config": {"workload": "SURVEY 8(f) f1 inside the step: laps_step_logits on configs[3] per GPU "
                      "(2,048 resident, batch 512, V=128,256, k=8, Beta(7,3) acceptance, L~U[512,4096], all "
                      "arrive at t=0), bf16 logits slab pool", "N_resident_per_gpu": args.n_per_gpu,
                      "B_per_gpu": B, "V": V, "k": k, "pool": f"{pool.S} slabs x {(2 * k + 1) * V * 2 / 1e6:.2f} MB",
                      "l2": "inputs larger than L2 (4.5 GB pool)", "parallelism": "dp1"},
           "verified_per_step": verified, "gpu_launches": int(round(launches_per_step * steps)), "clocks": clk,
           "roofline": {"kernel": "whole step (slot counters, logits_lazy_kernel, mask, update, select)",
                        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "algorithmic_bytes_per_step": alg, "traffic": None,
                        "note": "bytes: the logit rows the acceptance tests consult, once each; the lazy verify "
                                "is issue- and chain-bound (see --workload logits for its ALU roofline); the step "
                                "adds the update and the select, not overlapped"}}
    print(json.dumps(out), flush=True)


def run_logits(args):
    """spec_verify_logits on B=512 slots per GPU per step at configs[3]
    dimensions (V=128,256, k=8, bf16 logits), each step a fresh random draw of slabs from
    a 4.5 GB pool (inputs larger than L2).  Weak scaling: B slots per rank, no collective."""
    import paper_2505_17074_b200 as L
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B, k, V = args.batch, args.k, args.V
    pool = synth.make_logits_pool(V, k, "bf16", n_buckets=args.buckets, variants=args.variants,
                                  seed=synth.CONFIGS["c4"]["seed"] + 17 * rank, device=dev)
    G = max(1, min(args.graph_steps or 1, args.steps))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    slabs = torch.randint(0, pool.S, (G, B), generator=gen, device=dev, dtype=torch.int32)
    req = (torch.arange(B, device=dev, dtype=torch.int32) + rank * B)
    rnds = torch.randint(0, 1 << 12, (G, B), generator=gen, device=dev, dtype=torch.int32)
    tok = torch.empty(G, B, k + 1, dtype=torch.int32, device=dev)
    na = torch.empty(G, B, dtype=torch.int32, device=dev)
    ws = torch.empty(L.spec_verify_logits_workspace_bytes(B, k, V, "bf16"), dtype=torch.uint8, device=dev)
    seed = 0x5D0F1

    def step(t):
        L.spec_verify_logits(pool.p, pool.q, pool.draft, req, rnds[t], seed, slab=slabs[t], tokens=tok[t],
                             n_accept=na[t], z=None, workspace=ws)

    for t in range(max(args.warmup, 3)):
        step(t % G)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    lc0 = L.launch_count()
    with torch.cuda.graph(g):
        for t in range(G):
            step(t)
    launches_per_step = (L.launch_count() - lc0) / G
    reps = max(1, args.steps // G)
    g.replay()
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    steps = reps * G
    if dist:
        t_ = torch.tensor([ms], device=dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_[0])
    value = world * B * k * steps / (ms * 1e-3)
    r = na.cpu().numpy()
    row = V * 2
    eager = bool(os.environ.get("LAPSSD_LOGITS_EAGER"))
    if eager:   # every logit row once (the normalisers)
        alg = float((2 * k + 1) * row * r.size) / G
    else:       # the rows the acceptance tests consult, once each: pairs 0..min(r, k-1), p_k if r = k
        alg = float(((2 * np.minimum(r + 1, k) + (r == k)) * row).sum()) / G
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs") or 6650.0
    achieved = alg / (ms / steps * 1e-3) / 1e9
    traffic = None   # ncu DRAM bytes of one step, only for this build (profiles/alu_counts.json)
    try:
        ac = json.load(open(os.path.join(ROOT, "profiles", "alu_counts.json")))
        if ac.get("build_digest") == build_digest() and not eager:
            traffic = ac.get("logits", {}).get("dram_bytes_per_step")
    except (OSError, ValueError):
        pass
    kern = "logits_norm_kernel + logits_sample_kernel" if eager else "logits_lazy_kernel"
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
           "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16 logits; fixed-op fp32 exp, exact 2^40 integer softmax masses, "
           "128-bit integer acceptance and residual", "data": "synthetic",
           "config": {"workload": "SURVEY 8(f) f1: spec_verify_logits at configs[3] dimensions, B=512 slots "
                      "per GPU per step, V=128,256, k=8, bf16 logits (F2 Zipf, calibrated acceptance buckets), "
                      "slabs drawn at random from a 4.5 GB pool every step", "B_per_gpu": B, "V": V, "k": k,
                      "pool": f"{pool.S} slabs x {(2 * k + 1) * V * 2 / 1e6:.2f} MB",
                      "l2": "inputs larger than L2 (4.5 GB pool)", "parallelism": f"dp{world}: slots per rank"},
           "gpu_launches": int(round(launches_per_step * steps)),
           "clocks": clk,
           "roofline": {"kernel": f"{kern} (spec_verify_logits)",
                        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak,
                        "algorithmic_bytes_per_step": alg, "traffic": traffic,
                        "note": ("algorithmic bytes: every logit row once (2k+1 rows: normalisers)" if eager else
                                 "algorithmic bytes: the logit rows the acceptance tests consult, once each "
                                 "(pairs 0..min(r,k-1), and p_k if r = k); the residual pass re-reads its pair "
                                 "from L2") + "; traffic: ncu DRAM bytes of one step for this build, else null"}}
    if not eager:   # the work the lazy form avoids, against round 1's every-row definition
        every = float((2 * k + 1) * row * r.size) / G
        out["roofline"]["every_row_form"] = {
            "algorithmic_bytes_per_step": every, "rows_consulted_frac": alg / every,
            "equivalent_GBps": every / (ms / steps * 1e-3) / 1e9,
            "note": "the every-row form (round 1: all 2k+1 rows normalised, 1.00 ms per step) reads "
                    "these bytes; the lazy form reads only the consulted rows, so its fractions are "
                    "of a smaller amount of work, not a slower kernel"}
    alu = alu_roofline("logits", {"B": B, "V": V, "k": k}, ms / steps, clk)
    if alu:   # the binding resource: instruction issue (the fixed-op exp and the 128-bit residual)
        hbm = out["roofline"]
        out["roofline"] = dict(alu, kernel=hbm["kernel"],
                               hbm={x: hbm[x] for x in ("achieved", "peak", "unit", "frac", "algorithmic_bytes_per_step",
                                                        "traffic")})
        if "every_row_form" in hbm:
            out["roofline"]["every_row_form"] = hbm["every_row_form"]
    if not args.no_cpu_baseline and rank == 0:
        import oracle
        sl = slabs[0].cpu().numpy()
        rq = req.cpu().numpy()
        rd = rnds[0].cpu().numpy()
        nb, dt = 0, 0.0
        t0 = time.perf_counter()
        while nb < B and dt < args.cpu_seconds:   # slots of the first timed step, 16 at a time
            c = sl[nb:nb + 16]
            P = {"p": synth.to_numpy_rows(pool.p[c]), "q": synth.to_numpy_rows(pool.q[c]),
                 "draft": pool.draft[c].cpu().numpy()}
            oracle.verify_logits_batch(P["p"], P["q"], P["draft"], np.arange(len(c)), rq[nb:nb + 16],
                                       rd[nb:nb + 16], seed)
            nb += len(c)
            dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": nb * k / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"{nb} slots of the same workload, oracle/lapssd_oracle.c "
                               f"orc_verify_logits_batch single thread, {dt:.1f} s"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def timed_graph(args, step, G, local_rank, dist=None):
    """Warm-up, capture G steps in a CUDA graph, upload it, replay it over the timed
    region (CUDA events, NVML clocks, max over ranks).  Returns (ms_total, steps, clocks,
    launches_per_step)."""
    import paper_2505_17074_b200 as L
    for t in range(max(args.warmup, 3)):
        step(t % G)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    lc0 = L.launch_count()
    with torch.cuda.graph(g):
        for t in range(G):
            step(t)
    launches = (L.launch_count() - lc0) / G
    upload_graphs([g])
    reps = max(1, args.steps // G)
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", local_rank)))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t_ = torch.tensor([ms], device="cuda")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_[0])
    return ms, reps * G, clk, launches


def alu_roofline(key, workload, ms_per_step, clk):
    """Issue-rate roofline of an ALU-bound kernel: its executed warp instructions per step
    (ncu, profiles/alu_counts.json, used only for THIS build and this workload) over the
    step time, against 148 SMs x 4 sub-partitions x 1 warp instruction per clock at the
    median SM clock of the timed region.  None if no matching capture is on file."""
    path = os.path.join(ROOT, "profiles", "alu_counts.json")
    if not os.path.exists(path):
        return None
    try:
        d = json.load(open(path))
    except (OSError, ValueError):
        return None
    e = d.get(key)
    if not e or d.get("build_digest") != build_digest() or e.get("workload") != workload:
        return None
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965
    peak = 148 * 4 * mhz * 1e6 / 1e9                  # G warp instructions / s
    achieved = e["warp_inst_per_step"] / (ms_per_step * 1e-3) / 1e9
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "G warp-instructions/s",
            "frac": achieved / peak, "warp_inst_per_step": e["warp_inst_per_step"],
            "peak_source": f"148 SMs x 4 SMSPs x 1 warp instruction/clock at {mhz} MHz (B200_PROFILING.md unit counts)",
            "inst_source": d.get("source")}


def hbm_peak():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    return peaks.get("hbm_gbs") or 6650.0


def run_f4(args):
    """SURVEY 8(f) f4 at configs[3] dimensions (V=128,256, bf16, 512 requests per GPU per
    step).  draft: spec_draft_sample of the k=8 draft rows of every request (4,096 rows of
    256 KB per step, drawn at random from a 2.1 GB pool of F2 draft rows).  tree:
    spec_verify_tree of 512 token trees of --tree-nodes nodes (at most --tree-width children
    per node, tokens drawn from the parent's draft row), two input sets alternating
    (2 x 4.2 GB).  Weak scaling: requests per rank, no collective."""
    import paper_2505_17074_b200 as L
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B, k, V = args.batch, args.k, args.V
    pool = synth.make_pool("f2", V=V, k=k, dtype="bf16", n_buckets=args.buckets, variants=args.variants,
                           seed=synth.CONFIGS["c4"]["seed"] + 31 * rank, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4000 + rank)
    G = max(1, min(args.graph_steps or 1, args.steps))
    peak = hbm_peak()
    seed = 0x5D0F4
    if args.workload == "draft":
        R = B * k
        qrows = pool.q.view(-1, V)
        rows = torch.randint(0, qrows.shape[0], (G, R), generator=gen, device=dev, dtype=torch.int32)
        req = (torch.arange(B, device=dev, dtype=torch.int32) + rank * B).repeat_interleave(k)
        pos = torch.arange(k, device=dev, dtype=torch.int32).repeat(B)
        rnds = torch.randint(0, 1 << 12, (G, R), generator=gen, device=dev, dtype=torch.int32)
        out = torch.empty(G, R, dtype=torch.int32, device=dev)
        zbuf = torch.empty(G, R, dtype=torch.int64, device=dev)

        def step(t):
            L.spec_draft_sample(qrows, req, rnds[t], pos, seed, row=rows[t], out=out[t], z=zbuf[t])

        ms, steps, clk, lps = timed_graph(args, step, G, local_rank, dist)
        alg = float(R * V * 2)
        unit, value = "drafted tokens/s", world * R * steps / (ms * 1e-3)
        kernel = "draft_sample_kernel<bf16> (spec_draft_sample)"
        cfg = {"workload": f"SURVEY 8(f) f4 drafting: spec_draft_sample of B={B} requests x k={k} draft rows per "
                           f"GPU per step, V={V}, bf16 F2 draft rows drawn at random from a "
                           f"{qrows.shape[0] * V * 2 / 1e9:.1f} GB pool", "rows_per_step": R, "V": V,
               "l2": "inputs larger than L2", "parallelism": f"dp{world}: requests per rank"}
        cpu = None
        if not args.no_cpu_baseline and rank == 0:
            import oracle
            Q = synth.to_numpy_rows(qrows[rows[0][:64].long()])
            t0, n_ = time.perf_counter(), 0
            while n_ < 64 and time.perf_counter() - t0 < args.cpu_seconds:
                oracle.draft_sample(Q[n_], int(req[n_]), int(rnds[0][n_]), int(pos[n_]), seed)
                n_ += 1
            dt = time.perf_counter() - t0
            cpu = {"value": n_ / dt, "unit": unit, "cores": 1, "kind": "oracle",
                   "sample": f"{n_} rows of the first timed step, orc_draft_sample single thread, {dt:.1f} s"}
    else:
        n, wmax = args.tree_nodes, args.tree_width
        sets = []
        for si in range(2):
            idx = torch.randint(0, pool.S, (B,), generator=gen, device=dev)
            # node u's rows: target row u % (k+1) and draft row u % k of the request's slab
            ui = torch.arange(n, device=dev)
            p = pool.p[idx][:, ui % (k + 1)].contiguous()
            q = pool.q[idx][:, ui % k].contiguous()
            rng = np.random.default_rng(100 * rank + si)
            par = np.full((B, n), -1, np.int32)
            kids = np.zeros((B, n), np.int32)
            tok = np.zeros((B, n), np.int32)
            for c in range(1, n):
                for b in range(B):
                    cands = [u for u in range(c) if (u == 0 or par[b, u] >= 0) and kids[b, u] < wmax]
                    u = int(rng.choice(cands))
                    par[b, c] = u
                    kids[b, u] += 1
            # tokens: drawn from the parent's draft row on the GPU (the f4 sampler itself)
            qv = q.view(-1, V)
            rows_ = torch.as_tensor((np.arange(B)[:, None] * n + np.maximum(par, 0)).reshape(-1), device=dev,
                                    dtype=torch.int32)
            rq = torch.arange(B * n, device=dev, dtype=torch.int32)
            tk, _ = L.spec_draft_sample(qv, rq, rq * 0 + si, rq * 0, 77, row=rows_)
            tok = tk.view(B, n).contiguous()
            tok[:, 0] = 0
            sets.append((p, q, torch.as_tensor(par, device=dev), tok, par))
        req = torch.arange(B, device=dev, dtype=torch.int32) + rank * B
        rnds = torch.randint(0, 1 << 12, (G, B), generator=gen, device=dev, dtype=torch.int32)
        outs = [(torch.empty(B, n, dtype=torch.int32, device=dev), torch.empty(B, n, dtype=torch.int32, device=dev),
                 torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int64, device=dev))
                for _ in range(G)]

        def step(t):
            p, q, par_d, tok, _ = sets[t % 2]
            L.spec_verify_tree(p, q, par_d, tok, req, rnds[t], seed, tokens=outs[t][0], path=outs[t][1],
                               n_accept=outs[t][2], z=outs[t][3])

        ms, steps, clk, lps = timed_graph(args, step, G, local_rank, dist)
        # algorithmic bytes from the outcomes: per request, the final node's passes --
        # one over (p_u, q_u) per rejected child (all of its w children), or one over p_u
        # at a leaf -- plus two gathered scalars per tested child
        emitted = alg = 0.0
        for t in range(G):
            par = sets[t % 2][4]
            path = outs[t][1].cpu().numpy()
            na = outs[t][2].cpu().numpy()
            for b in range(B):
                u = 0 if na[b] == 0 else int(path[b, na[b] - 1])
                w = int((par[b] == u).sum())
                alg += (w * 2 if w else 1) * V * 2 + 4 * (na[b] + w)
                emitted += na[b] + 1
        alg /= G
        unit = "emitted tokens/s"
        value = world * emitted / G * steps / (ms * 1e-3)
        kernel = "tree_verify_kernel<bf16> (spec_verify_tree)"
        cfg = {"workload": f"SURVEY 8(f) f4 tree verification: spec_verify_tree of B={B} token trees per GPU "
                           f"per step, {n} nodes (<= {wmax} children per node, draft tokens sampled from the "
                           f"parent's draft row), V={V}, bf16 F2 rows, two input sets of "
                           f"{2 * B * n * V * 2 / 1e9:.1f} GB alternating", "trees_per_step": B, "nodes": n,
               "max_children": wmax, "V": V, "mean_accepted": emitted / G / B - 1,
               "l2": "inputs larger than L2", "parallelism": f"dp{world}: trees per rank"}
        cpu = None
        if not args.no_cpu_baseline and rank == 0:
            import oracle
            p, q, _, tok, par = sets[0]
            t0, n_ = time.perf_counter(), 0
            tk = tok.cpu().numpy()
            while n_ < B and time.perf_counter() - t0 < args.cpu_seconds:
                oracle.verify_tree(synth.to_numpy_rows(p[n_]), synth.to_numpy_rows(q[n_]), par[n_], tk[n_],
                                   int(req[n_]), int(rnds[0][n_]), seed)
                n_ += 1
            dt = time.perf_counter() - t0
            cpu = {"value": n_ * (emitted / G / B) / dt, "unit": unit, "cores": 1, "kind": "oracle",
                   "sample": f"{n_} trees of the first input set, orc_verify_tree single thread, {dt:.1f} s"}
    achieved = alg / (ms / steps * 1e-3) / 1e9
    res = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": steps,
           "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16 rows; exact Q4.60 integer masses, 128-bit residual tests",
           "data": "synthetic", "config": cfg, "gpu_launches": int(round(lps * steps)), "clocks": clk,
           "roofline": {"kernel": kernel, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "algorithmic_bytes_per_step": alg, "traffic": None,
                        "timing": f"{steps} steps as replays of a CUDA graph of {G} steps"}}
    if args.workload == "tree":   # neither bound is reached: the issue rate beside the HBM one
        alu = alu_roofline("tree", {"B": B, "V": V, "nodes": args.tree_nodes, "max_children": args.tree_width},
                           ms / steps, clk)
        if alu:
            res["roofline"]["alu"] = {x: alu[x] for x in ("achieved", "peak", "unit", "frac")}
    if cpu:
        res["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(res), flush=True)
    if dist:
        dist.destroy_process_group()


def run_c23(args):
    """configs[1] (1,024 requests, Poisson, Beta(4,2), V=32,000, k=4, fp32, B=64) or
    configs[2] (4,096 requests, drifting acceptance, V=32,000, k=6, bf16, B=64), full size
    on one GPU: the whole trace through laps_step to completion (eager calls: the run's
    length depends on the outcome), then the same trace through the oracle (its OpenMP
    build) and every request's final state compared bit for bit.  value = verified draft
    tokens per second of the GPU run; the line also carries the mean JCT."""
    import paper_2505_17074_b200 as L
    name = "c2" if args.workload == "c2" else "c3"
    c = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    rho = args.rho or c["rho"]
    tr = synth.make_config_trace(name, rho=rho)
    pool = synth.make_pool("f2", V=c["V"], k=c["k"], dtype=c["dtype"], n_buckets=64, variants=c["variants"],
                           seed=c["seed"], device=dev)
    tab = synth.slab_table(tr, 64, c["variants"], R=32, seed=c["seed"])
    kw = dict(K=c["K"], s1_up_us=4 * (c["k"] * 1000 + 10_000), M=2.0, gamma=5, delta=0.05, k=c["k"],
              t_ssm_us=1000, t_llm_us=10_000, policy=args.policy, seed=c["seed"])
    B = c["B"]
    h = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=c["V"], overlap=True)
    rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device=dev))
    h.laps_select(B)
    cnt = h.count
    # warm-up of the kernels on a throwaway handle (same shapes)
    hw = L.Handle(L.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, max_batch=B, V=c["V"], overlap=True)
    hw.laps_select(B)
    for _ in range(max(args.warmup, 3)):
        hw.laps_step(rows, B)
    torch.cuda.synchronize()
    del hw
    clocks = Clocks(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 0
    clocks.start()
    e0.record()
    while True:
        for _ in range(64):                  # 64 steps between host checks of completion
            h.laps_step(rows, B)
        steps += 64
        done = h.state()["done"]
        if done.all() or steps > 10_000_000:
            break
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    st = h.state()
    assert h.check() == 0
    verified = int(st["rounds"].sum())
    jct = (st["C_us"] - tr.arrival_us).astype(np.float64)
    out = {"metric": METRIC, "value": verified * c["k"] / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
           "steps": steps, "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None,
           "dtype": f"{c['dtype']} rows; fp32 residual + exact Q4.60 integer CDF; fp64 scheduler",
           "data": "synthetic",
           "config": {"workload": f"configs[{1 if name == 'c2' else 2}] at full size: {c['n']} requests, "
                                  f"Poisson arrivals at rho={rho}, B={B}, V={c['V']}, k={c['k']}, {c['dtype']}, "
                                  f"{'drifting ' if c['drift'] else ''}Beta(4,2) acceptance, policy {args.policy}, "
                                  "run to completion (steps include the idle tail's host checks)",
                      "n": c["n"], "B": B, "V": c["V"], "k": c["k"], "rho": rho, "policy": args.policy,
                      "l2": f"{pool.S * (2 * c['k'] + 1) * c['V'] * (2 if c['dtype'] == 'bf16' else 4) / 1e9:.1f} "
                            "GB slab pool"},
           "verified_per_step": verified / steps, "clocks": clk,
           "jct": {"mean_ms": float(jct.mean() / 1e3), "p99_ms": float(np.percentile(jct, 99) / 1e3),
                   "sim_makespan_s": float(st["now_us"] / 1e6), "perceptible_frac": float(st["perceptible"].mean())}}
    if not args.no_parity:
        import oracle
        P = pool.numpy()
        P["slab_tab"], P["R"] = tab, tab.shape[1]
        sim = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred, parallel=True)
        sel, _ = sim.select(B)
        t0 = time.perf_counter()
        n_o = 0
        while not sim.state()["done"].all():
            sim.step(P, sel)
            n_o += 1
        el = time.perf_counter() - t0
        o = sim.state()
        fields = ("acc_tok", "acc_draft", "rounds", "E_us", "T_total_us", "C_us", "x_us", "level", "perceptible",
                  "pinned", "key")
        diff = [f for f in fields if not (np.asarray(st[f]) == np.asarray(o[f])).all()]
        out["parity"] = {"oracle_steps": n_o, "fields_compared": list(fields) + ["A (bits)", "now_us"],
                         "mismatched": diff + ([] if (st["A"].view(np.uint64) == o["A"].view(np.uint64)).all()
                                               else ["A"]) + ([] if st["now_us"] == o["now_us"] else ["now_us"]),
                         "bit_exact": not diff and st["now_us"] == o["now_us"]
                         and bool((st["A"].view(np.uint64) == o["A"].view(np.uint64)).all())}
        # one core: the same trace from the start, for a bounded time
        sim1 = oracle.Sim(oracle.SchedConfig(**kw), tr.arrival_us, tr.L_true, tr.L_pred)
        sel1, _ = sim1.select(B)
        t1, v1, n1 = time.perf_counter(), 0, 0
        while time.perf_counter() - t1 < args.cpu_seconds and n1 < n_o:
            v1 += int((sel1 >= 0).sum())
            sim1.step(P, sel1)
            n1 += 1
        el1 = time.perf_counter() - t1
        out["cpu_baseline"] = {"value": int(o["rounds"].sum()) * c["k"] / el, "unit": UNIT, "cores": omp_threads(),
                               "kind": "oracle", "sample": f"the whole trace ({n_o} steps), oracle/lapssd_oracle.c "
                               f"-fopenmp build, {el:.1f} s", "host": host_info(),
                               "single_thread": {"value": v1 * c["k"] / el1, "cores": 1,
                                                 "sample": f"the first {n1} steps of the same trace, plain build, "
                                                           f"{el1:.1f} s"}}
    print(json.dumps(out), flush=True)


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, timed on this host's cores on the
    same config / metric; each step a bounded sample (a smaller batch) of the workload."""
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return
    import oracle

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    # inputs: same generator and recipe; a 128-slab pool is enough for the oracle
    tr, local, pool, tab = build_workload(args, 0, 1, dev, pool_slabs=128)
    # each step is a bounded sample: pick the batch so the whole run takes ~2 minutes
    probe = oracle.Sim(oracle.SchedConfig(**SCHED, seed=1), local.arrival_us, local.L_true,
                       local.L_pred, parallel=True)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, tab.shape[1]
    nb = 4 * omp_threads()
    sel, _ = probe.select(nb)
    t0 = time.perf_counter()
    probe.step(P, sel)
    per_verify = (time.perf_counter() - t0) / nb
    total_steps = args.warmup + args.steps
    b_ref = int(max(1, min(args.batch, 100.0 / (total_steps * per_verify))))
    sim = oracle.Sim(oracle.SchedConfig(**SCHED, seed=synth.CONFIGS["c4"]["seed"]),
                     local.arrival_us, local.L_true, local.L_pred, parallel=True)
    sel, _ = sim.select(b_ref)
    for _ in range(args.warmup):
        sim.step(P, sel)
    verified = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        verified += int((sel >= 0).sum())
        sim.step(P, sel)
    el = time.perf_counter() - t0
    value = verified * args.k / el
    sample = (f"oracle/lapssd_oracle.c built with -fopenmp ({omp_threads()} threads: a step's requests "
              f"verified in parallel); each step verifies a batch of {b_ref} "
              f"(of {args.batch}) requests of the same workload, V={args.V}, k={args.k}, bf16")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16 rows; fp32/fp64/int128 oracle",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOAD, "N_resident_per_gpu": args.n_per_gpu,
                      "B_per_step": b_ref, "V": args.V, "k": args.k},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": omp_threads(), "kind": "oracle",
                            "sample": sample, "host": host_info()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "logits":
        run_logits(args)
    elif args.workload == "logits_step":
        run_logits_step(args)
    elif args.workload in ("draft", "tree"):
        run_f4(args)
    elif args.workload in ("c2", "c3"):
        run_c23(args)
    elif args.workload == "mc":
        run_mc(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
