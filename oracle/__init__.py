"""CPU oracle for the LAPS-SD batched speculative-decoding step (arXiv 2505.17074).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
It wraps ``oracle/liblapssd_oracle.so`` (plain sequential C, ``lapssd_oracle.c``) with
ctypes and numpy marshalling; it shares no code with ``paper_2505_17074_b200``.

Every function cites the PAPER.md passage it follows (``P:NN`` = PAPER.md line NN) in
``lapssd_oracle.c``; the pins that fix each one are listed in ``lapssd_oracle.h`` and
DESIGN.md section 4.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblapssd_oracle.so")
_SRC = os.path.join(_HERE, "lapssd_oracle.c")

F32, BF16 = 0, 1
POL_LAPSSD, POL_FCFS, POL_LPSJF, POL_LAS = 0, 1, 2, 3
COST_EQ6, COST_FIG1 = 0, 1
POLICIES = {"laps-sd": POL_LAPSSD, "fcfs": POL_FCFS, "lp-sjf": POL_LPSJF, "las": POL_LAS}


_SO_OMP = os.path.join(_HERE, "liblapssd_oracle_omp.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FP contraction), and the same source
    with -fopenmp (the all-cores CPU baseline: only the per-request verify loop of a step
    runs in parallel)."""
    deps = max(os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "lapssd_oracle.h")))
    for so, extra in ((_SO, []), (_SO_OMP, ["-fopenmp"])):
        if force or not os.path.exists(so) or os.path.getmtime(so) < deps:
            subprocess.check_call(
                ["gcc", "-O2", "-std=c11", "-Wall", "-Wno-unknown-pragmas", "-ffp-contract=off", "-fPIC", "-shared", *extra,
                 "-o", so, _SRC, "-lm"]
            )
    return _SO


class VerifyOut(C.Structure):
    _fields_ = [("r", C.c_int32), ("y", C.c_int32), ("fallback", C.c_int32),
                ("invalid", C.c_int32), ("Z", C.c_uint64), ("t", C.c_uint64),
                ("z_real", C.c_double), ("z_rel_err", C.c_double), ("margin_rel", C.c_double)]


class LogitsOut(C.Structure):
    _fields_ = [("r", C.c_int32), ("y", C.c_int32), ("fallback", C.c_int32), ("pad", C.c_int32),
                ("Z_lo", C.c_uint64), ("Z_hi", C.c_uint64), ("Sp", C.c_uint64), ("Sq", C.c_uint64)]


class TreeOut(C.Structure):
    _fields_ = [("n_accept", C.c_int32), ("y", C.c_int32), ("final_node", C.c_int32),
                ("n_rejected", C.c_int32), ("fallback", C.c_int32), ("invalid", C.c_int32),
                ("Z", C.c_uint64)]


class OrcConfig(C.Structure):
    _fields_ = [("policy", C.c_int32), ("K", C.c_int32), ("s1_up_us", C.c_int64),
                ("M", C.c_double), ("gamma", C.c_int32), ("delta", C.c_double),
                ("k", C.c_int32), ("t_ssm_us", C.c_int64), ("t_llm_us", C.c_int64),
                ("placement", C.c_int32), ("pin_rule", C.c_int32), ("seed", C.c_uint64),
                ("cost_model", C.c_int32), ("t_tok_us", C.c_int64), ("switch_c0_us", C.c_int64),
                ("switch_c1_us", C.c_int64)]


class StateView(C.Structure):
    _fields_ = [("now_us", C.c_int64), ("cursor", C.c_int32), ("prev_count", C.c_int32),
                ("acc_tok", C.POINTER(C.c_int32)), ("acc_draft", C.POINTER(C.c_int32)),
                ("rounds", C.POINTER(C.c_int32)),
                ("E_us", C.POINTER(C.c_int64)), ("T_total_us", C.POINTER(C.c_int64)),
                ("C_us", C.POINTER(C.c_int64)), ("x_us", C.POINTER(C.c_int64)),
                ("admitted", C.POINTER(C.c_uint8)), ("done", C.POINTER(C.c_uint8)),
                ("perceptible", C.POINTER(C.c_uint8)), ("pinned", C.POINTER(C.c_uint8)),
                ("level", C.POINTER(C.c_uint8)), ("running", C.POINTER(C.c_uint8)),
                ("A", C.POINTER(C.c_double)), ("key", C.POINTER(C.c_uint64)),
                ("ring", C.POINTER(C.c_int32)), ("switch_us", C.POINTER(C.c_int64)),
                ("in_batch", C.POINTER(C.c_uint8)), ("step_cost_us", C.c_int64),
                ("switch_total_us", C.c_int64)]


_libs = {}


def lib(parallel: bool = False):
    """The oracle library; parallel=True: the -fopenmp build of the same source."""
    if parallel not in _libs:
        # LAPSSD_ORACLE_LIB: a mutated build of the same source (tests/test_oracle_mutants.py
        # checks that the pins reject it); default: the oracle itself
        build()
        path = _SO_OMP if parallel else (os.environ.get("LAPSSD_ORACLE_LIB") or _SO)
        _libs[parallel] = L = C.CDLL(path)
        vp, i32, i64, u32, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_verify_request.argtypes = [vp, vp, i32, i64, i32, vp, u32, u32, u64, u32, vp,
                                         C.POINTER(VerifyOut)]
        L.orc_verify_request.restype = i32
        L.orc_verify_many.argtypes = [vp, vp, i32, i64, i32, i32, vp, vp, vp, u64, vp, vp]
        L.orc_exp_hat.argtypes = [C.c_float]
        L.orc_exp_hat.restype = C.c_float
        L.orc_logits_row.argtypes = [vp, i32, i64, vp, vp]
        L.orc_logits_row.restype = u64
        L.orc_verify_logits_request.argtypes = [vp, vp, i32, i64, i32, vp, u32, u32, u64, u32, vp,
                                                C.POINTER(LogitsOut)]
        L.orc_verify_logits_request.restype = i32
        L.orc_verify_logits_many.argtypes = [vp, vp, i32, i64, i32, i32, vp, vp, vp, u64, vp, vp]
        L.orc_verify_logits_batch.argtypes = [vp, vp, i32, i64, i32, i32, vp, vp, vp, vp, u64, vp, vp, vp]
        L.orc_draft_sample.argtypes = [vp, i32, i64, u32, u32, u32, u64, u32, vp, vp]
        L.orc_draft_sample.restype = i32
        L.orc_verify_tree.argtypes = [vp, vp, i32, i64, i32, vp, vp, u32, u32, u64, u32, vp, vp,
                                      C.POINTER(TreeOut)]
        L.orc_verify_tree.restype = i32
        L.orc_thresholds.argtypes = [i32, i64, C.c_double, vp]
        L.orc_thresholds.restype = i32
        L.orc_eq6.argtypes = [i64, C.c_double, i32, i64, i64]
        L.orc_eq6.restype = u64
        L.orc_fig1_est.argtypes = [i64, C.c_double, i64]
        L.orc_fig1_est.restype = u64
        L.orc_sim_make_perceptible.argtypes = [vp, i32, C.c_double]
        L.orc_sim_make_perceptible.restype = i32
        L.orc_sim_create.argtypes = [C.POINTER(OrcConfig), i32, vp, vp, vp, vp, i32, i32]
        L.orc_sim_create.restype = vp
        L.orc_sim_destroy.argtypes = [vp]
        L.orc_sim_set_trace.argtypes = [vp, u32]
        L.orc_sim_select.argtypes = [vp, i32, vp]
        L.orc_sim_select.restype = i32
        L.orc_sim_candidates.argtypes = [vp, i32, vp, vp, vp]
        L.orc_sim_merge.argtypes = [vp, vp, vp, i32, vp, i32, vp, vp]
        L.orc_sim_merge.restype = i32
        L.orc_sim_update.argtypes = [vp, vp, vp, i32]
        L.orc_sim_step.argtypes = [vp, vp, vp, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp]
        L.orc_sim_step.restype = i32
        L.orc_sim_view.argtypes = [vp, C.POINTER(StateView)]
        L.orc_jobs_schedule.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp]
        L.orc_jobs_schedule.restype = i64
        L.orc_brute_force.argtypes = [i32, vp, vp, vp]
        L.orc_brute_force.restype = i64
    return _libs[parallel]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def _dtype_code(rows: np.ndarray) -> int:
    if rows.dtype == np.float32:
        return F32
    if rows.dtype == np.uint16:  # bf16 bit patterns
        return BF16
    raise TypeError("rows must be float32 or uint16 (bf16 bits)")


def verify_request(p_rows, q_rows, draft, req_id, round_idx, seed, trace=0):
    """P:57-64 / P:200 for one request.  p_rows [k+1,V], q_rows [k,V] (float32 or
    uint16 bf16 bits).  Returns (tokens[k+1], VerifyOut)."""
    p = np.ascontiguousarray(p_rows)
    q = np.ascontiguousarray(q_rows)
    k = q.shape[0]
    V = p.shape[1]
    assert p.shape == (k + 1, V) and q.shape == (k, V) and p.dtype == q.dtype
    d = _c(draft, np.int32)
    tok = np.zeros(k + 1, np.int32)
    out = VerifyOut()
    lib().orc_verify_request(_ptr(p), _ptr(q), _dtype_code(p), V, k, _ptr(d), int(req_id),
                             int(round_idx), int(seed) & (2**64 - 1), int(trace), _ptr(tok),
                             C.byref(out))
    return tok, out


def verify_many(p_rows, q_rows, drafts, req_ids, rounds, seed):
    """n independent trials over the same rows; drafts [n,k].  Returns (tokens, r)."""
    p = np.ascontiguousarray(p_rows)
    q = np.ascontiguousarray(q_rows)
    k, V = q.shape
    d = _c(drafts, np.int32)
    n = d.shape[0]
    ri = _c(req_ids, np.uint32)
    ro = _c(rounds, np.uint32)
    tok = np.zeros((n, k + 1), np.int32)
    r = np.zeros(n, np.int32)
    lib().orc_verify_many(_ptr(p), _ptr(q), _dtype_code(p), V, k, n, _ptr(d), _ptr(ri), _ptr(ro),
                          int(seed) & (2**64 - 1), _ptr(tok), _ptr(r))
    return tok, r


def exp_hat(d) -> float:
    """AMB-30: e^d on [-28, 0] by the fixed fp32 operation sequence."""
    return float(lib().orc_exp_hat(float(d)))


def logits_row(z_row):
    """AMB-30's quantised softmax of one row: (E [V] uint64, S, m)."""
    z = np.ascontiguousarray(z_row)
    V = z.shape[-1]
    E = np.zeros(V, np.uint64)
    m = np.zeros(1, np.float32)
    S = lib().orc_logits_row(_ptr(z), _dtype_code(z), V, _ptr(m), _ptr(E))
    return E, int(S), float(m[0])


def verify_logits_request(zp_rows, zq_rows, draft, req_id, round_idx, seed, trace=0):
    """f1: P:57-64 / P:200 with p = softmax(zp), q = softmax(zq), quantised
    as AMB-30.  zp_rows [k+1,V], zq_rows [k,V] logits (float32 or uint16 bf16 bits)."""
    p = np.ascontiguousarray(zp_rows)
    q = np.ascontiguousarray(zq_rows)
    k = q.shape[0]
    V = p.shape[1]
    assert p.shape == (k + 1, V) and q.shape == (k, V) and p.dtype == q.dtype
    d = _c(draft, np.int32)
    tok = np.zeros(k + 1, np.int32)
    out = LogitsOut()
    lib().orc_verify_logits_request(_ptr(p), _ptr(q), _dtype_code(p), V, k, _ptr(d), int(req_id),
                                    int(round_idx), int(seed) & (2**64 - 1), int(trace), _ptr(tok),
                                    C.byref(out))
    return tok, out


def verify_logits_many(zp_rows, zq_rows, drafts, req_ids, rounds, seed):
    p = np.ascontiguousarray(zp_rows)
    q = np.ascontiguousarray(zq_rows)
    k, V = q.shape
    d = _c(drafts, np.int32)
    n = d.shape[0]
    tok = np.zeros((n, k + 1), np.int32)
    r = np.zeros(n, np.int32)
    lib().orc_verify_logits_many(_ptr(p), _ptr(q), _dtype_code(p), V, k, n, _ptr(d),
                                 _ptr(_c(req_ids, np.uint32)), _ptr(_c(rounds, np.uint32)),
                                 int(seed) & (2**64 - 1), _ptr(tok), _ptr(r))
    return tok, r


def verify_logits_batch(zp, zq, drafts, slab, req_ids, rounds, seed):
    """B slots; slot b reads slab slab[b] of zp [S,k+1,V], zq [S,k,V], drafts [S,k].
    Returns (tokens [B,k+1], r [B], Z [B,2] = (lo, hi) of the integer residual mass)."""
    p = np.ascontiguousarray(zp)
    q = np.ascontiguousarray(zq)
    S, k, V = q.shape
    sl = _c(slab, np.int32)
    B = sl.shape[0]
    tok = np.zeros((B, k + 1), np.int32)
    r = np.zeros(B, np.int32)
    z = np.zeros((B, 2), np.uint64)
    lib().orc_verify_logits_batch(_ptr(p), _ptr(q), _dtype_code(p), V, k, B, _ptr(sl),
                                  _ptr(_c(drafts, np.int32)), _ptr(_c(req_ids, np.uint32)),
                                  _ptr(_c(rounds, np.uint32)), int(seed) & (2**64 - 1), _ptr(tok),
                                  _ptr(r), _ptr(z))
    return tok, r, z


def draft_sample(q_row, req_id, round_idx, pos, seed, trace=0):
    """one draft token from the row q_row by the exact integer inverse CDF
    (lapssd_oracle.h orc_draft_sample).  Returns (x, Z, invalid)."""
    q = np.ascontiguousarray(q_row)
    Z = np.zeros(1, np.uint64)
    inv = np.zeros(1, np.int32)
    x = lib().orc_draft_sample(_ptr(q), _dtype_code(q), q.shape[-1], int(req_id), int(round_idx), int(pos),
                               seed & (2**64 - 1), trace, _ptr(Z), _ptr(inv))
    return int(x), int(Z[0]), bool(inv[0])


def verify_tree(p_rows, q_rows, parent, token, req_id, round_idx, seed, trace=0):
    """token-tree verification (lapssd_oracle.h orc_verify_tree).
    p_rows / q_rows [n_nodes, V]; parent / token [n_nodes].  Returns (n_accept, tokens,
    path, TreeOut)."""
    p = np.ascontiguousarray(p_rows)
    q = np.ascontiguousarray(q_rows)
    par = _c(parent, np.int32)
    tok = _c(token, np.int32)
    n = len(par)
    toks = np.zeros(n, np.int32)
    path = np.zeros(n, np.int32)
    o = TreeOut()
    na = lib().orc_verify_tree(_ptr(p), _ptr(q), _dtype_code(p), p.shape[-1], n, _ptr(par), _ptr(tok),
                               int(req_id), int(round_idx), seed & (2**64 - 1), trace, _ptr(toks),
                               _ptr(path), C.byref(o))
    return int(na), toks, path, o


def thresholds(K, s1_up_us, M):
    out = np.zeros(max(K - 1, 1), np.int64)
    rc = lib().orc_thresholds(K, s1_up_us, M, _ptr(out))
    if rc != 0:
        raise ValueError("invalid thresholds (K, s1_up, M)")
    return out[: K - 1]


def eq6(L, A, k, t_ssm_us, t_llm_us) -> int:
    return int(lib().orc_eq6(int(L), float(A), int(k), int(t_ssm_us), int(t_llm_us)))


def fig1_est(L, A, t_tok_us) -> int:
    """Fig. 1 model: floor(L t_tok / A) us."""
    return int(lib().orc_fig1_est(int(L), float(A), int(t_tok_us)))


def jobs_schedule(policy, arrival_us, service_us, L_pred=None, est_us=None):
    """Non-preemptive job-level schedule (Fig. 1 semantics).  policy: 0 SJF-by-est,
    1 FCFS, 2 LP-SJF.  Returns (sum of C_i - r_i, order, C)."""
    a = _c(arrival_us, np.int64)
    n = len(a)
    s = _c(service_us, np.int64)
    lp = _c(L_pred if L_pred is not None else np.zeros(n), np.int64)
    e = _c(est_us if est_us is not None else np.zeros(n), np.int64)
    order = np.zeros(n, np.int32)
    Cc = np.zeros(n, np.int64)
    tot = lib().orc_jobs_schedule(policy, n, _ptr(a), _ptr(s), _ptr(lp), _ptr(e), _ptr(order),
                                  _ptr(Cc))
    return int(tot), order, Cc


def brute_force(service_us):
    s = _c(service_us, np.int64)
    n = len(s)
    best = np.zeros(n, np.int32)
    import math
    sums = np.zeros(math.factorial(n), np.int64)
    tot = lib().orc_brute_force(n, _ptr(s), _ptr(best), _ptr(sums))
    return int(tot), best, sums


@dataclass
class SchedConfig:
    """LAPS-SD parameters; defaults are DESIGN.md readings."""
    policy: int = POL_LAPSSD
    K: int = 4
    s1_up_us: int = 56_000
    M: float = 2.0
    gamma: int = 5
    delta: float = 0.05
    k: int = 4
    t_ssm_us: int = 1_000
    t_llm_us: int = 10_000
    placement: int = 0
    pin_rule: int = 0
    seed: int = 0
    cost_model: int = COST_EQ6
    t_tok_us: int = 0
    switch_c0_us: int = 0
    switch_c1_us: int = 0

    def c(self) -> OrcConfig:
        return OrcConfig(self.policy, self.K, self.s1_up_us, self.M, self.gamma, self.delta,
                         self.k, self.t_ssm_us, self.t_llm_us, self.placement, self.pin_rule,
                         self.seed & (2**64 - 1), self.cost_model, self.t_tok_us,
                         self.switch_c0_us, self.switch_c1_us)


class Sim:
    """The resident-request simulation: admit / select / verify / update / clock."""

    def __init__(self, cfg: SchedConfig, arrival_us, L_true, L_pred, rank=0, world=1, trace=0,
                 prompt=None, parallel=False):
        """parallel: the -fopenmp build (the all-cores CPU baseline; same source)."""
        self.cfg = cfg
        self._L = lib(parallel)
        self._a = _c(arrival_us, np.int64)
        self._lt = _c(L_true, np.int32)
        self._lp = _c(L_pred, np.int32)
        self._pr = _c(prompt, np.int32) if prompt is not None else None
        self.n = len(self._a)
        self._cc = cfg.c()
        self.h = self._L.orc_sim_create(C.byref(self._cc), self.n, _ptr(self._a), _ptr(self._lt),
                                      _ptr(self._lp), _ptr(self._pr) if self._pr is not None else None,
                                      rank, world)
        if not self.h:
            raise ValueError("orc_sim_create rejected the configuration")
        if trace:
            self._L.orc_sim_set_trace(self.h, trace)
        self.rank, self.world = rank, world

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self._L.orc_sim_destroy(h)
            self.h = None

    def select(self, B):
        sel = np.full(B, -1, np.int32)
        cnt = self._L.orc_sim_select(self.h, B, _ptr(sel))
        return sel, cnt

    def make_perceptible(self, i, A):
        """Test hook (Fig. 1(c) clairvoyant case): request i perceptible with rate A."""
        rc = self._L.orc_sim_make_perceptible(self.h, int(i), float(A))
        if rc != 0:
            raise ValueError("make_perceptible rejected")

    def candidates(self, Cn, with_switch=False):
        keys = np.zeros(Cn, np.uint64)
        sw = np.zeros(Cn, np.int64)
        nxt = np.zeros(1, np.int64)
        self._L.orc_sim_candidates(self.h, Cn, _ptr(keys), _ptr(sw), _ptr(nxt))
        if with_switch:
            return keys, sw, int(nxt[0])
        return keys, int(nxt[0])

    def merge(self, all_keys, Cn, all_next, B, all_switch=None):
        k = _c(all_keys, np.uint64)
        nx = _c(all_next, np.int64)
        sw = _c(all_switch, np.int64) if all_switch is not None else None
        sel = np.full(B, -1, np.int32)
        g = np.zeros(1, np.int32)
        own = self._L.orc_sim_merge(self.h, _ptr(k), _ptr(sw) if sw is not None else None, Cn,
                                  _ptr(nx), B, _ptr(sel), _ptr(g))
        return sel, own, int(g[0])

    def update(self, sel, n_accept):
        s = _c(sel, np.int32)
        na = _c(n_accept, np.int32)
        self._L.orc_sim_update(self.h, _ptr(s), _ptr(na), len(s))

    def step(self, pools, sel):
        """pools: dict(p, q, draft, slab_tab, R) from synth.  sel is updated in place."""
        p, q, d, tab = pools["p"], pools["q"], pools["draft"], pools["slab_tab"]
        k = self.cfg.k
        V = p.shape[-1]
        B = len(sel)
        tok = np.zeros((B, k + 1), np.int32)
        na = np.zeros(B, np.int32)
        z = np.zeros(B, np.uint64)
        cnt = self._L.orc_sim_step(self.h, _ptr(p), _ptr(q), _ptr(d), _dtype_code(p), V, _ptr(tab),
                                 int(pools["R"]), B, _ptr(sel), _ptr(tok), _ptr(na), _ptr(z))
        return cnt, tok, na, z

    def state(self) -> dict:
        v = StateView()
        self._L.orc_sim_view(self.h, C.byref(v))
        n, g = self.n, self.cfg.gamma

        def arr(ptr, m=n):
            return np.ctypeslib.as_array(ptr, shape=(m,)).copy() if m else np.zeros(0)

        return dict(now_us=v.now_us, cursor=v.cursor, prev_count=v.prev_count,
                    acc_tok=arr(v.acc_tok), acc_draft=arr(v.acc_draft), rounds=arr(v.rounds),
                    E_us=arr(v.E_us), T_total_us=arr(v.T_total_us), C_us=arr(v.C_us),
                    x_us=arr(v.x_us), admitted=arr(v.admitted), done=arr(v.done),
                    perceptible=arr(v.perceptible), pinned=arr(v.pinned), level=arr(v.level),
                    running=arr(v.running), A=arr(v.A), key=arr(v.key),
                    ring=arr(v.ring, n * g).reshape(n, g) if n else np.zeros((0, g)),
                    switch_us=arr(v.switch_us), in_batch=arr(v.in_batch),
                    step_cost_us=v.step_cost_us, switch_total_us=v.switch_total_us)
