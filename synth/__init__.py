"""Seeded synthetic inputs for the LAPS-SD step -- the ONE module both sides use.

This module holds none of the method's arithmetic: no acceptance test, no residual,
no sampling, no scheduler rule.  It only *produces inputs* of the shapes and value
distributions of the paper's workloads:

* probability-row slabs -- for one request-step, target rows p[k+1,V] and draft rows
  q[k,V] plus draft tokens x_j sampled from q_j (the stand-in for the SSM/LLM forward
  passes, which are out of scope);
* request traces -- arrival times (Poisson or all-at-zero), true and predicted
  output lengths (the predictor is an input with lognormal noise), per-request
  acceptance processes (constant Beta-distributed or drifting then stable);
* the slab table that says which slab a request sees in each round.

Row families:
  F1 "mixture": q uniform on a random half A of the vocabulary, rho uniform on the
     complement, p = beta*q + (1-beta)*rho.  Any draft in A is accepted with
     probability exactly beta and the residual is exactly rho (used for pins).
  F2 "zipf": Zipf(1.1)-ranked logits plus N(0, 1.5^2) noise, p = softmax(logits);
     q = softmax(logits + eps * N(0,1)) with eps bisected per acceptance bucket.
     Heavy-tailed, full support (used for parity and the bench).
Probabilities are stored as float32 or bf16 (bf16 as uint16 bit patterns in numpy,
torch.bfloat16 on the device; rounding to bf16 is round-to-nearest-even).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

N_BUCKETS = 64


# ---------------------------------------------------------------------------
# dtype plumbing
def bf16_bits(x: torch.Tensor) -> np.ndarray:
    """bfloat16 tensor (any device) -> numpy uint16 bit patterns."""
    return x.detach().to("cpu").contiguous().view(torch.int16).numpy().view(np.uint16)


def to_numpy_rows(x: torch.Tensor) -> np.ndarray:
    """Stored rows as the oracle consumes them: float32, or bf16 as uint16 bits."""
    if x.dtype == torch.bfloat16:
        return bf16_bits(x)
    return x.detach().to("cpu").contiguous().numpy()


def torch_dtype(name: str):
    return {"bf16": torch.bfloat16, "f32": torch.float32, "fp32": torch.float32}[name]


# ---------------------------------------------------------------------------
# row families
def f1_rows(V: int, k: int, betas, gen: torch.Generator, device="cpu", dtype=torch.float32):
    """F1 mixture family for one slab.  betas: k+1 acceptance values (the last one is
    the bonus row's, irrelevant to acceptance).  Returns p[k+1,V], q[k,V], draft[k]."""
    half = V // 2
    p = torch.empty(k + 1, V, dtype=torch.float32)
    q = torch.empty(k, V, dtype=torch.float32)
    draft = torch.empty(k, dtype=torch.int32)
    for j in range(k + 1):
        perm = torch.randperm(V, generator=gen)
        A, Bc = perm[:half], perm[half:]
        qj = torch.zeros(V)
        qj[A] = 1.0 / half
        rho = torch.zeros(V)
        rho[Bc] = 1.0 / (V - half)
        b = float(betas[j])
        p[j] = b * qj + (1.0 - b) * rho
        if j < k:
            q[j] = qj
            draft[j] = int(A[torch.randint(half, (1,), generator=gen)].item())
    return p.to(device=device, dtype=dtype), q.to(device=device, dtype=dtype), draft.to(device)


def _zipf_logits(n_rows: int, V: int, gen: torch.Generator, device):
    ranks = torch.argsort(torch.rand(n_rows, V, generator=gen, device=device), dim=1).float() + 1.0
    return -1.1 * torch.log(ranks) + 1.5 * torch.randn(n_rows, V, generator=gen, device=device)


def _f2_pair(logits, eps, gen):
    noise = torch.randn(logits.shape, generator=gen, device=logits.device)
    p = torch.softmax(logits, dim=-1)
    q = torch.softmax(logits + eps[:, None] * noise, dim=-1)
    return p, q


def calibrate_eps(V: int, targets, gen: torch.Generator, device="cpu", rows=8, iters=22):
    """Bisection on eps so that mean_j sum_v min(p_j, q_j) hits each target."""
    targets = torch.as_tensor(targets, dtype=torch.float32, device=device)
    nb = targets.numel()
    logits = _zipf_logits(rows, V, gen, device)
    noise = torch.randn(rows, V, generator=gen, device=device)
    p = torch.softmax(logits, -1)
    lo = torch.zeros(nb, device=device)
    hi = torch.full((nb,), 40.0, device=device)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        q = torch.softmax(logits[None] + mid[:, None, None] * noise[None], -1)
        acc = torch.minimum(p[None], q).sum(-1).mean(-1)
        too_similar = acc > targets
        lo = torch.where(too_similar, mid, lo)
        hi = torch.where(too_similar, hi, mid)
    return 0.5 * (lo + hi)


@dataclass
class Pool:
    """A slab pool: p[S,k+1,V], q[S,k,V] (torch, on `device`), draft[S,k] int32,
    slab s belongs to acceptance bucket s // variants."""
    p: torch.Tensor
    q: torch.Tensor
    draft: torch.Tensor
    family: str
    n_buckets: int
    variants: int
    beta_realised: torch.Tensor = field(default=None)

    @property
    def S(self):
        return self.p.shape[0]

    @property
    def V(self):
        return self.p.shape[-1]

    @property
    def k(self):
        return self.q.shape[1]

    def numpy(self):
        return dict(p=to_numpy_rows(self.p), q=to_numpy_rows(self.q),
                    draft=self.draft.to("cpu").numpy().astype(np.int32))


def make_pool(family: str, V: int, k: int, dtype: str, n_buckets: int, variants: int,
              seed: int, device="cpu", chunk_slabs: int = 16) -> Pool:
    """Generate S = n_buckets * variants slabs.  Bucket b targets acceptance
    (b + 0.5) / n_buckets."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    tdt = torch_dtype(dtype)
    S = n_buckets * variants
    p = torch.empty(S, k + 1, V, dtype=tdt, device=device)
    q = torch.empty(S, k, V, dtype=tdt, device=device)
    draft = torch.empty(S, k, dtype=torch.int32, device=device)
    betas = (torch.arange(n_buckets, dtype=torch.float32) + 0.5) / n_buckets
    if family == "f1":
        cg = torch.Generator()
        cg.manual_seed(seed)
        for s in range(S):
            b = float(betas[s // variants])
            ps, qs, ds = f1_rows(V, k, [b] * (k + 1), cg, device=device, dtype=tdt)
            p[s], q[s], draft[s] = ps, qs, ds
    elif family == "f2":
        eps_b = calibrate_eps(V, betas.tolist(), gen, device=device)
        for s0 in range(0, S, chunk_slabs):
            s1 = min(S, s0 + chunk_slabs)
            n = s1 - s0
            eps = eps_b[torch.arange(s0, s1, device=device) // variants]
            logits = _zipf_logits(n * (k + 1), V, gen, device).view(n, k + 1, V)
            pp = torch.softmax(logits, -1)
            noise = torch.randn(n, k, V, generator=gen, device=device)
            qq = torch.softmax(logits[:, :k] + eps[:, None, None] * noise, -1)
            p[s0:s1] = pp.to(tdt)
            q[s0:s1] = qq.to(tdt)
            qs = q[s0:s1].float().reshape(n * k, V)
            draft[s0:s1] = torch.multinomial(qs, 1, generator=gen).view(n, k).to(torch.int32)
            del logits, pp, noise, qq, qs
    else:
        raise ValueError(family)
    return Pool(p=p, q=q, draft=draft, family=family, n_buckets=n_buckets, variants=variants)


def make_logits_pool(V: int, k: int, dtype: str, n_buckets: int, variants: int, seed: int,
                     device="cpu", chunk_slabs: int = 16) -> Pool:
    """F2 as LOGITS (the heads' outputs): zp[S,k+1,V] = Zipf(1.1) +
    N(0,1.5^2) logits, zq[S,k,V] = zp[:, :k] + eps N(0,1) with eps calibrated per
    acceptance bucket as in make_pool; drafts sampled from the fp32 softmax of zq (the
    draft model's sampler, an input to the method).  Returned as Pool(p=zp, q=zq)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    tdt = torch_dtype(dtype)
    S = n_buckets * variants
    zp = torch.empty(S, k + 1, V, dtype=tdt, device=device)
    zq = torch.empty(S, k, V, dtype=tdt, device=device)
    draft = torch.empty(S, k, dtype=torch.int32, device=device)
    betas = (torch.arange(n_buckets, dtype=torch.float32) + 0.5) / n_buckets
    eps_b = calibrate_eps(V, betas.tolist(), gen, device=device)
    for s0 in range(0, S, chunk_slabs):
        s1 = min(S, s0 + chunk_slabs)
        n = s1 - s0
        eps = eps_b[torch.arange(s0, s1, device=device) // variants]
        logits = _zipf_logits(n * (k + 1), V, gen, device).view(n, k + 1, V)
        noise = torch.randn(n, k, V, generator=gen, device=device)
        zp[s0:s1] = logits.to(tdt)
        zq[s0:s1] = (logits[:, :k] + eps[:, None, None] * noise).to(tdt)
        qs = torch.softmax(zq[s0:s1].float(), -1).reshape(n * k, V)
        draft[s0:s1] = torch.multinomial(qs, 1, generator=gen).view(n, k).to(torch.int32)
        del logits, noise, qs
    return Pool(p=zp, q=zq, draft=draft, family="f2-logits", n_buckets=n_buckets, variants=variants)


# ---------------------------------------------------------------------------
# request traces
@dataclass
class Trace:
    arrival_us: np.ndarray       # int64, sorted; index = request id (arrival order)
    L_true: np.ndarray           # int32
    L_pred: np.ndarray           # int32
    alpha_s: np.ndarray          # float64 stable acceptance
    amp: np.ndarray              # drift amplitude (0 = constant)
    decay: np.ndarray
    period: np.ndarray

    @property
    def n(self):
        return len(self.arrival_us)

    def alpha_at(self, t: np.ndarray) -> np.ndarray:
        """alpha_i(t) for every request at rounds t[i] (damped sinusoid)."""
        a = self.alpha_s + self.amp * self.decay ** t * np.sin(2 * np.pi * t / self.period)
        return np.clip(a, 0.0, 1.0)

    def shard(self, rank: int, world: int) -> "Trace":
        sl = slice(rank, None, world)
        return Trace(self.arrival_us[sl].copy(), self.L_true[sl].copy(), self.L_pred[sl].copy(),
                     self.alpha_s[sl].copy(), self.amp[sl].copy(), self.decay[sl].copy(),
                     self.period[sl].copy())


def make_trace(n: int, seed: int, *, arrival="poisson", rate_per_s=35.0,
               length="lognormal", len_mu=math.log(200), len_sigma=0.8, len_min=8,
               len_max=2048, beta_ab=(4.0, 2.0), drift=False, pred_sigma=0.3) -> Trace:
    rng = np.random.default_rng(seed)
    if arrival == "poisson":
        gaps = rng.exponential(1e6 / rate_per_s, size=n)
        arr = np.floor(np.cumsum(gaps)).astype(np.int64)
        arr -= arr[0]
    else:
        arr = np.zeros(n, np.int64)
    if length == "lognormal":
        L = np.exp(rng.normal(len_mu, len_sigma, size=n))
        L = np.clip(np.round(L), len_min, len_max).astype(np.int32)
    else:  # uniform
        L = rng.integers(len_min, len_max + 1, size=n).astype(np.int32)
    Lp = np.maximum(1, np.round(L * np.exp(rng.normal(0, pred_sigma, size=n)))).astype(np.int32)
    a_s = rng.beta(beta_ab[0], beta_ab[1], size=n)
    if drift:
        amp = rng.uniform(0.2, 0.4, size=n)
        dec = rng.uniform(0.8, 0.95, size=n)
        per = rng.integers(4, 13, size=n).astype(np.float64)
    else:
        amp = np.zeros(n)
        dec = np.full(n, 0.5)
        per = np.full(n, 8.0)
    return Trace(arr, L, Lp, a_s, amp, dec, per)


def prompt_lengths(n: int, seed: int, median=150.0, sigma=0.7, lo=4, hi=2048) -> np.ndarray:
    """Prompt lengths for the switching-cost workloads (f2, DESIGN.md AMB-24): lognormal
    around `median` tokens, clipped to [lo, hi], int32."""
    rng = np.random.default_rng(seed ^ 0x9E37)
    return np.clip(np.round(np.exp(rng.normal(math.log(median), sigma, n))), lo, hi).astype(np.int32)


def slab_table(trace: Trace, n_buckets: int, variants: int, R: int, seed: int) -> np.ndarray:
    """tab[i, t] = slab seen by request i in round t (t < R; later rounds reuse the
    stable half).  Bucket = randomised rounding of alpha_i(t)*n_buckets
    so its expectation matches alpha_i(t); variant uniform."""
    rng = np.random.default_rng(seed ^ 0x51AB)
    n = trace.n
    tab = np.zeros((n, R), np.int32)
    for t in range(R):
        a = trace.alpha_at(np.full(n, float(t)))
        x = a * n_buckets - 0.5
        b = np.floor(x + rng.random(n)).astype(np.int64)
        b = np.clip(b, 0, n_buckets - 1)
        v = rng.integers(0, variants, size=n)
        tab[:, t] = (b * variants + v).astype(np.int32)
    return tab


# ---------------------------------------------------------------------------
# BASELINE.json configurations
CONFIGS = {
    # configs[1]: 1,024 requests, Poisson, Beta acceptance, V=32000, k=4, fp32, B=64
    "c2": dict(n=1024, V=32000, k=4, dtype="f32", B=64, arrival="poisson", length="lognormal",
               len_mu=math.log(200), len_sigma=0.8, len_min=8, len_max=2048, beta_ab=(4, 2),
               drift=False, rho=0.8, K=4, family="f2", variants=16, seed=0x5D0002),
    # configs[2]: 4,096 requests with drift, K=4, V=32000, k=6, bf16
    "c3": dict(n=4096, V=32000, k=6, dtype="bf16", B=64, arrival="poisson", length="lognormal",
               len_mu=math.log(200), len_sigma=0.8, len_min=8, len_max=2048, beta_ab=(4, 2),
               drift=True, rho=0.9, K=4, family="f2", variants=16, seed=0x5D0003),
    # configs[3]: 16,384 requests over 8 GPUs, V=128256, k=8, bf16, B=512 per GPU
    "c4": dict(n=16384, V=128256, k=8, dtype="bf16", B=512, arrival="zero", length="uniform",
               len_min=512, len_max=4096, beta_ab=(7, 3), drift=False, rho=None, K=4,
               family="f2", variants=16, seed=0x5D0004, per_gpu=2048),
}


# configs[4]: Monte-Carlo sweep, 8,192 independent traces x 512 requests, batch 1 per
# trace, V=32000, k=4, bf16, per-trace Poisson arrivals at load rho=0.8
CONFIGS["c5"] = dict(T=8192, n=512, V=32000, k=4, dtype="bf16", arrival="poisson", length="lognormal",
                     len_mu=math.log(128), len_sigma=0.8, len_min=8, len_max=2048, beta_ab=(4, 2),
                     drift=False, rho=0.8, K=4, family="f2", n_buckets=64, variants=256, R=16,
                     seed=0x5D0005)


@dataclass
class MCWorkload:
    """T traces concatenated: trace t owns requests offsets[t]..offsets[t+1]."""
    offsets: np.ndarray     # [T+1] int64
    arrival_us: np.ndarray  # [n_total] int64, sorted within each trace
    L_true: np.ndarray      # [n_total] int32
    L_pred: np.ndarray      # [n_total] int32
    slab_tab: np.ndarray    # [n_total, R] int32 (global request index)
    alpha: np.ndarray       # [n_total] acceptance rate behind the slab buckets

    @property
    def T(self) -> int:
        return len(self.offsets) - 1

    def trace(self, t: int):
        a, b = int(self.offsets[t]), int(self.offsets[t + 1])
        return self.arrival_us[a:b], self.L_true[a:b], self.L_pred[a:b], self.slab_tab[a:b]


def make_mc_workload(T: int, n: int, seed: int, *, rate_per_s: float, len_mu=math.log(128), len_sigma=0.8,
                     len_min=8, len_max=2048, beta_ab=(4.0, 2.0), n_buckets=64, variants=256, R=16,
                     pred_sigma=0.3) -> MCWorkload:
    """T independent Poisson traces of n requests (vectorised; same recipe as make_trace +
    slab_table per trace: lognormal lengths, L_pred = L * exp(N(0, 0.3^2)), Beta
    acceptance, slab bucket = randomised rounding of alpha * n_buckets)."""
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(1e6 / rate_per_s, size=(T, n))
    arr = np.floor(np.cumsum(gaps, axis=1)).astype(np.int64)
    arr -= arr[:, :1]
    L = np.clip(np.round(np.exp(rng.normal(len_mu, len_sigma, size=(T, n)))), len_min, len_max).astype(np.int32)
    Lp = np.maximum(1, np.round(L * np.exp(rng.normal(0, pred_sigma, size=(T, n))))).astype(np.int32)
    alpha = rng.beta(beta_ab[0], beta_ab[1], size=(T, n))
    tab = np.empty((T * n, R), np.int32)
    for t in range(R):
        x = alpha.reshape(-1) * n_buckets - 0.5
        b = np.clip(np.floor(x + rng.random(T * n)).astype(np.int64), 0, n_buckets - 1)
        v = rng.integers(0, variants, size=T * n)
        tab[:, t] = (b * variants + v).astype(np.int32)
    return MCWorkload(np.arange(T + 1, dtype=np.int64) * n, arr.reshape(-1), L.reshape(-1), Lp.reshape(-1),
                      tab, alpha.reshape(-1))


def mc_rate_for_load(rho: float, k: int, t_ssm_us: int, t_llm_us: int, len_mu=math.log(128), len_sigma=0.8,
                     beta_ab=(4.0, 2.0)) -> float:
    """Arrivals per second giving load rho on one server (batch 1): rho / E[service],
    E[service] = E[L] / E[tokens per round] * c_round (workload sizing only)."""
    EL = math.exp(len_mu + len_sigma ** 2 / 2)
    beta = beta_ab[0] / (beta_ab[0] + beta_ab[1])
    per_round = float(tokens_per_round(np.array([beta]), k)[0])
    c_round_s = (k * t_ssm_us + t_llm_us) * 1e-6
    return rho / (EL / per_round * c_round_s)


def tokens_per_round(beta: np.ndarray, k: int) -> np.ndarray:
    """Workload sizing only (arrival rate for a target load): the textbook expected
    tokens per round (1 - b^(k+1)) / (1 - b) of the cited SD papers."""
    b = np.clip(beta, 1e-9, 1 - 1e-9)
    return (1 - b ** (k + 1)) / (1 - b)


def make_config_trace(name: str, n: int | None = None, rho: float | None = None,
                      t_ssm_us=1000, t_llm_us=10000, G: int = 1) -> Trace:
    c = CONFIGS[name]
    n = n or c["n"]
    rate = 1.0
    if c["arrival"] == "poisson":
        tmp = make_trace(n, c["seed"], arrival="zero", length=c["length"],
                         len_mu=c.get("len_mu", 0), len_sigma=c.get("len_sigma", 1),
                         len_min=c["len_min"], len_max=c["len_max"], beta_ab=c["beta_ab"],
                         drift=c["drift"])
        c_round_s = (c["k"] * t_ssm_us + t_llm_us) * 1e-6
        rounds = tmp.L_true.mean() / tokens_per_round(tmp.alpha_s, c["k"]).mean()
        rate = (rho or c["rho"]) * c["B"] * G / (rounds * c_round_s)
    return make_trace(n, c["seed"], arrival=c["arrival"], rate_per_s=rate, length=c["length"],
                      len_mu=c.get("len_mu", 0), len_sigma=c.get("len_sigma", 1),
                      len_min=c["len_min"], len_max=c["len_max"], beta_ab=c["beta_ab"],
                      drift=c["drift"])
