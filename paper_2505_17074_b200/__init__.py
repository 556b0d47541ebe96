"""paper_2505_17074_b200 -- B200-native LAPS-SD batched speculative-decoding step.

Thin Python binding of ``liblapssd.so`` (C-ABI in ``include/lapssd.h``): argument
marshalling only.  Every step of the hot path -- verification by rejection sampling
(PAPER.md P:57-64), the LAPS-SD state update and the top-B
selection -- runs in the library's sm_100a kernels.  PyTorch
supplies device memory, streams and process groups.  There is no CPU fallback: if
the library cannot be loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("LAPSSD_LIBRARY") or os.path.join(_HERE, "liblapssd.so")  # override: diagnostic builds

F32, BF16 = 0, 1
POL_LAPSSD, POL_FCFS, POL_LPSJF, POL_LAS = 0, 1, 2, 3
COST_EQ6, COST_FIG1 = 0, 1
STATUS = {0: "OK", -1: "EINVAL", -2: "ECUDA", -3: "ENCCL", -4: "ESTATE", -5: "ENOMEM"}


class LapssdError(RuntimeError):
    def __init__(self, call, status, msg):
        super().__init__(f"{call}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("K", C.c_int32), ("s1_up_us", C.c_int64),
                ("M", C.c_double), ("gamma", C.c_int32), ("delta", C.c_double),
                ("k", C.c_int32), ("t_ssm_us", C.c_int64), ("t_llm_us", C.c_int64),
                ("placement", C.c_int32), ("pin_rule", C.c_int32), ("seed", C.c_uint64),
                ("cost_model", C.c_int32), ("t_tok_us", C.c_int64), ("switch_c0_us", C.c_int64),
                ("switch_c1_us", C.c_int64)]


class _Requests(C.Structure):
    _fields_ = [("arrival_us", C.c_void_p), ("L_true", C.c_void_p), ("L_pred", C.c_void_p),
                ("n", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("prompt", C.c_void_p)]


class _Rows(C.Structure):
    _fields_ = [("p", C.c_void_p), ("q", C.c_void_p), ("draft", C.c_void_p),
                ("dtype", C.c_int32), ("k", C.c_int32), ("V", C.c_int64),
                ("slab_tab", C.c_void_p), ("R", C.c_int32), ("n_slabs", C.c_int64)]


class _StateView(C.Structure):
    _fields_ = [("now_us", C.c_int64), ("cursor", C.c_int32), ("prev_count", C.c_int32)] + [
        (n, C.c_void_p) for n in ("acc_tok", "acc_draft", "rounds", "E_us", "T_total_us", "C_us",
                                  "x_us", "admitted", "done", "perceptible", "pinned", "level",
                                  "running", "A", "key", "ring", "switch_us")] + [
        ("step_cost_us", C.c_int64), ("switch_total_us", C.c_int64)]

_VIEW_ARRAYS = [f for f, t in _StateView._fields_[3:] if t is C.c_void_p]


def _load():
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (nvcc sm_100a build).  There is no CPU fallback.")
    lib = C.CDLL(_SO)
    vp, i32, i64, u32, u64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_size_t
    sigs = {
        "spec_verify_workspace_bytes": ([i32, i64], sz),
        "spec_verify": ([vp, vp, i32, i64, i32, vp, vp, vp, vp, i32, u64, u32, vp, vp, vp, vp, sz, vp], i32),
        "spec_verify_logits_workspace_bytes": ([i32, i32, i64, i32], sz),
        "spec_verify_logits": ([vp, vp, i32, i64, i32, vp, vp, vp, vp, i32, u64, u32, vp, vp, vp, vp, sz, vp], i32),
        "spec_draft_sample": ([vp, i32, i64, vp, vp, vp, vp, i32, u64, u32, vp, vp, vp], i32),
        "spec_verify_tree": ([vp, vp, i32, i64, i32, vp, vp, vp, vp, i32, u64, u32, vp, vp, vp, vp, vp], i32),
        "lapssd_workspace_bytes": ([vp, i32, i32, i64, i32], sz),
        "lapssd_create": ([vp, vp, i32, i64, vp, sz, vp, vp], i32),
        "lapssd_destroy": ([vp], i32),
        "laps_update": ([vp, vp, vp, i32, vp], i32),
        "laps_select": ([vp, i32, vp, vp, vp], i32),
        "laps_step": ([vp, vp, i32, vp, vp, vp, vp, vp], i32),
        "laps_step_logits_workspace_bytes": ([i32, i32, i64, i32], sz),
        "laps_step_logits": ([vp, vp, i32, vp, vp, vp, vp, vp, sz, vp], i32),
        "lapssd_set_step_overlap": ([vp, i32], i32),
        "lapssd_set_row_check": ([vp, i32], i32),
        "laps_candidates": ([vp, i32, vp, vp], i32),
        "laps_merge": ([vp, vp, i32, i32, vp, vp, vp], i32),
        "laps_step_dist": ([vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp], i32),
        "laps_step_candidates": ([vp, vp, i32, i32, vp, vp, vp, vp, vp], i32),
        "lapssd_peer_buffer_bytes": ([i32, i32], sz),
        "lapssd_set_peers": ([vp, vp, i32, vp], i32),
        "laps_step_peer": ([vp, vp, i32, vp, vp, vp, vp, vp], i32),
        "lapssd_nccl_unique_id": ([vp], i32),
        "lapssd_nccl_comm_init": ([vp, i32, vp, i32], i32),
        "lapssd_nccl_comm_destroy": ([vp], i32),
        "lapssd_read_state": ([vp, vp, vp], i32),
        "lapssd_check": ([vp, vp], i32),
        "lapssd_profile": ([vp, i32], i32),
        "lapssd_profile_read": ([vp, vp, vp, vp, vp], i32),
        "lapssd_mc_workspace_bytes": ([vp, i32, i64, i64], sz),
        "lapssd_mc_create": ([vp, i32, vp, vp, vp, vp, vp, i64, vp, sz, vp, vp], i32),
        "lapssd_mc_destroy": ([vp], i32),
        "laps_mc_select": ([vp, vp, vp], i32),
        "laps_mc_step": ([vp, vp, vp, vp, vp, vp], i32),
        "lapssd_mc_read": ([vp, vp, vp, vp, vp, vp], i32),
        "lapssd_mc_check": ([vp, vp], i32),
        "lapssd_last_error": ([], C.c_char_p),
        "lapssd_launch_count": ([], u64),
    }
    for name, (args, res) in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load()


def library_path() -> str:
    return _SO


def launch_count() -> int:
    """Kernel launches the library has enqueued in this process."""
    return int(_lib.lapssd_launch_count())


def _check(call, rc):
    if rc != 0:
        raise LapssdError(call, rc, _lib.lapssd_last_error().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dptr(t: torch.Tensor | None):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return C.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"rows must be bf16 or fp32, got {t.dtype}")


# --------------------------------------------------------------------------- stateless
def spec_verify_workspace_bytes(B: int, V: int) -> int:
    return int(_lib.spec_verify_workspace_bytes(B, V))


def spec_verify(p, q, draft, req_id, round_idx, seed, *, slab=None, trace=0, tokens=None,
                n_accept=None, z=None, workspace=None, stream=None):
    """Batched verification (include/lapssd.h spec_verify).  p [S,k+1,V], q [S,k,V]
    (bf16/fp32), draft [S,k] int32, req_id / round_idx [B] int32 (uint32 values);
    slab [B] int32 selects rows (None: slot b reads rows b).  Returns
    (tokens [B,k+1], n_accept [B], z [B] uint64-as-int64)."""
    k, V = q.shape[-2], q.shape[-1]
    B = req_id.numel()
    dev = p.device
    if tokens is None:
        tokens = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
    if n_accept is None:
        n_accept = torch.empty(B, dtype=torch.int32, device=dev)
    if z is None:
        z = torch.empty(B, dtype=torch.int64, device=dev)
    ws_bytes = spec_verify_workspace_bytes(B, V)
    if workspace is None:
        workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    rc = _lib.spec_verify(_dptr(p), _dptr(q), _dtype_code(p), V, k, _dptr(draft), _dptr(slab),
                          _dptr(req_id), _dptr(round_idx), B, seed & (2**64 - 1), trace,
                          _dptr(tokens), _dptr(n_accept), _dptr(z), _dptr(workspace),
                          workspace.numel(), _stream(stream))
    _check("spec_verify", rc)
    return tokens, n_accept, z


def laps_step_logits_workspace_bytes(B, k, V, dtype) -> int:
    """Workspace bytes of Handle.laps_step_logits; dtype "bf16" / "f32" or the lapssd code."""
    code = {"bf16": BF16, "f32": F32}.get(dtype, dtype)
    return int(_lib.laps_step_logits_workspace_bytes(B, k, V, code))


def spec_verify_logits_workspace_bytes(B, k, V, dtype) -> int:
    """Workspace bytes of spec_verify_logits; dtype "bf16" / "f32" or the lapssd code."""
    code = {"bf16": BF16, "f32": F32}.get(dtype, dtype)
    return int(_lib.spec_verify_logits_workspace_bytes(B, k, V, code))


def spec_verify_logits(zp, zq, draft, req_id, round_idx, seed, *, slab=None, trace=0, tokens=None,
                       n_accept=None, z=None, workspace=None, stream=None):
    """Batched verification from logits (include/lapssd.h spec_verify_logits, SURVEY
    8(f) f1).  zp [S,k+1,V], zq [S,k,V] logits (bf16/fp32), draft [S,k] int32,
    req_id / round_idx [B]; slab [B] int32 (None: slot b reads slab b).  Returns
    (tokens [B,k+1], n_accept [B], z [B,2] = (lo, hi) of the integer residual mass)."""
    k, V = zq.shape[-2], zq.shape[-1]
    B = req_id.numel()
    dev = zp.device
    if tokens is None:
        tokens = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
    if n_accept is None:
        n_accept = torch.empty(B, dtype=torch.int32, device=dev)
    if z is None:
        z = torch.empty(B, 2, dtype=torch.int64, device=dev)
    ws_bytes = int(_lib.spec_verify_logits_workspace_bytes(B, k, V, _dtype_code(zp)))
    if workspace is None:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    rc = _lib.spec_verify_logits(_dptr(zp), _dptr(zq), _dtype_code(zp), V, k, _dptr(draft), _dptr(slab),
                                 _dptr(req_id), _dptr(round_idx), B, seed & (2**64 - 1), trace,
                                 _dptr(tokens), _dptr(n_accept), _dptr(z), _dptr(workspace),
                                 workspace.numel(), _stream(stream))
    _check("spec_verify_logits", rc)
    return tokens, n_accept, z


def spec_draft_sample(q, req_id, round_idx, pos, seed, *, row=None, trace=0, out=None, z=None, stream=None):
    """Drafting-side sampling (include/lapssd.h spec_draft_sample): one
    token per row.  q [..., V] rows (bf16 / fp32; row r = q.view(-1, V)[row[r] if row is
    given else r]); req_id / round_idx / pos [R] int32.  Returns (draft [R], z [R])."""
    V = q.shape[-1]
    R = req_id.numel()
    dev = q.device
    if out is None:
        out = torch.empty(R, dtype=torch.int32, device=dev)
    if z is None:
        z = torch.empty(R, dtype=torch.int64, device=dev)
    rc = _lib.spec_draft_sample(_dptr(q), _dtype_code(q), V, _dptr(row), _dptr(req_id), _dptr(round_idx),
                                _dptr(pos), R, seed & (2**64 - 1), trace, _dptr(out), _dptr(z), _stream(stream))
    _check("spec_draft_sample", rc)
    return out, z


def spec_verify_tree(p, q, parent, token, req_id, round_idx, seed, *, trace=0, tokens=None, path=None,
                     n_accept=None, z=None, stream=None):
    """Token-tree verification (include/lapssd.h spec_verify_tree).  p, q
    [B, n_nodes, V]; parent / token [B, n_nodes] int32; req_id / round_idx [B].  Returns
    (tokens [B, n_nodes], path [B, n_nodes], n_accept [B], z [B])."""
    B, n, V = p.shape
    dev = p.device
    tokens = torch.empty(B, n, dtype=torch.int32, device=dev) if tokens is None else tokens
    path = torch.empty(B, n, dtype=torch.int32, device=dev) if path is None else path
    n_accept = torch.empty(B, dtype=torch.int32, device=dev) if n_accept is None else n_accept
    z = torch.empty(B, dtype=torch.int64, device=dev) if z is None else z
    rc = _lib.spec_verify_tree(_dptr(p), _dptr(q), _dtype_code(p), V, n, _dptr(parent), _dptr(token),
                               _dptr(req_id), _dptr(round_idx), B, seed & (2**64 - 1), trace, _dptr(tokens),
                               _dptr(path), _dptr(n_accept), _dptr(z), _stream(stream))
    _check("spec_verify_tree", rc)
    return tokens, path, n_accept, z


# --------------------------------------------------------------------------- handle
@dataclass
class SchedConfig:
    """lapssd_config; defaults are DESIGN.md readings (K=4, M=2, gamma=5, delta=.05)."""
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

    def c(self):
        return _Config(self.policy, self.K, self.s1_up_us, self.M, self.gamma, self.delta,
                       self.k, self.t_ssm_us, self.t_llm_us, self.placement, self.pin_rule,
                       self.seed & (2**64 - 1), self.cost_model, self.t_tok_us,
                       self.switch_c0_us, self.switch_c1_us)


class Rows:
    """lapssd_rows: pooled (slab_tab given) or batch layout; p, q, draft device or pinned host
    tensors (read in place over UVA), slab_tab a device tensor."""

    def __init__(self, p, q, draft, slab_tab=None):
        self.p, self.q, self.draft, self.slab_tab = p, q, draft, slab_tab
        self.k, self.V = q.shape[-2], q.shape[-1]
        self.c = _Rows(p.data_ptr(), q.data_ptr(), draft.data_ptr(), _dtype_code(p), self.k, self.V,
                       slab_tab.data_ptr() if slab_tab is not None else None,
                       slab_tab.shape[1] if slab_tab is not None else 0, p.shape[0])


class Handle:
    """A LAPS-SD resident-request state on one GPU (lapssd_create)."""

    def __init__(self, cfg: SchedConfig, arrival_us, L_true, L_pred, *, max_batch: int, V: int,
                 rank: int = 0, world: int = 1, prompt=None, overlap: bool = False, device="cuda",
                 stream=None):
        self.cfg = cfg
        self._cc = cfg.c()
        a = np.ascontiguousarray(arrival_us, np.int64)
        lt = np.ascontiguousarray(L_true, np.int32)
        lp = np.ascontiguousarray(L_pred, np.int32)
        pr = np.ascontiguousarray(prompt, np.int32) if prompt is not None else None
        self.n = len(a)
        self.max_batch, self.V, self.rank, self.world = max_batch, V, rank, world
        req = _Requests(a.ctypes.data, lt.ctypes.data, lp.ctypes.data, self.n, rank, world,
                        pr.ctypes.data if pr is not None else None)
        nbytes = int(_lib.lapssd_workspace_bytes(C.byref(self._cc), self.n, max_batch, V, world))
        if nbytes == 0:
            raise LapssdError("lapssd_workspace_bytes", -1, "invalid sizes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        h = C.c_void_p()
        rc = _lib.lapssd_create(C.byref(self._cc), C.byref(req), max_batch, V,
                                _dptr(self.workspace), nbytes, _stream(stream), C.byref(h))
        _check("lapssd_create", rc)
        self.h = h
        self.sel = torch.full((max_batch,), -1, dtype=torch.int32, device=device)
        self.count = torch.zeros(1, dtype=torch.int32, device=device)
        if overlap:
            self.set_step_overlap(True)

    def set_row_check(self, enable: bool):
        """lapssd_set_row_check: validate the streamed rows' masses (device flag 256)."""
        _check("lapssd_set_row_check", _lib.lapssd_set_row_check(self.h, 1 if enable else 0))

    def set_step_overlap(self, enable: bool):
        """lapssd_set_step_overlap: consecutive verify launches overlap (the caller does not
        write the step's rows between laps_step calls on the stream)."""
        _check("lapssd_set_step_overlap", _lib.lapssd_set_step_overlap(self.h, 1 if enable else 0))

    def close(self):
        if getattr(self, "h", None):
            _lib.lapssd_destroy(self.h)
            self.h = None

    __del__ = close

    # -- the four hot-path calls --------------------------------------------------
    def laps_update(self, sel, n_accept, stream=None):
        _check("laps_update", _lib.laps_update(self.h, _dptr(sel), _dptr(n_accept), sel.numel(),
                                               _stream(stream)))

    def laps_select(self, B, sel=None, count=None, stream=None):
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        _check("laps_select", _lib.laps_select(self.h, B, _dptr(sel), _dptr(count), _stream(stream)))
        return sel, count

    def laps_step_logits(self, rows: Rows, B, sel=None, count=None, tokens=None, n_accept=None, workspace=None,
                         stream=None):
        """The LAPS-SD step from logits (include/lapssd.h laps_step_logits): rows.p / rows.q
        hold target / draft LOGITS.  workspace: a uint8 device tensor of at least
        laps_step_logits_workspace_bytes(B, k, V, dtype) bytes (allocated if None)."""
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        nbytes = int(_lib.laps_step_logits_workspace_bytes(B, rows.k, rows.V, _dtype_code(rows.p)))
        if workspace is None:
            workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=sel.device)
        _check("laps_step_logits", _lib.laps_step_logits(self.h, C.byref(rows.c), B, _dptr(sel), _dptr(count),
                                                         _dptr(tokens), _dptr(n_accept), _dptr(workspace),
                                                         workspace.numel(), _stream(stream)))
        return sel, count

    def laps_step(self, rows: Rows, B, sel=None, count=None, tokens=None, n_accept=None, stream=None):
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        _check("laps_step", _lib.laps_step(self.h, C.byref(rows.c), B, _dptr(sel), _dptr(count),
                                           _dptr(tokens), _dptr(n_accept), _stream(stream)))
        return sel, count

    # -- multi-GPU halves ------------------------------------------------------
    def laps_candidates(self, Cn, cand_out, stream=None):
        _check("laps_candidates", _lib.laps_candidates(self.h, Cn, _dptr(cand_out), _stream(stream)))

    def laps_merge(self, all_cand, Cn, B, sel=None, count=None, stream=None):
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        _check("laps_merge", _lib.laps_merge(self.h, _dptr(all_cand), Cn, B, _dptr(sel),
                                             _dptr(count), _stream(stream)))
        return sel, count

    def laps_step_dist(self, comm, rows: Rows, B_global, Cn, cand_scratch, sel=None, count=None,
                       tokens=None, n_accept=None, stream=None):
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        _check("laps_step_dist", _lib.laps_step_dist(self.h, comm, C.byref(rows.c), B_global, Cn,
                                                     _dptr(sel), _dptr(count), _dptr(tokens), _dptr(n_accept),
                                                     _dptr(cand_scratch), _stream(stream)))
        return sel, count

    def laps_step_candidates(self, rows: Rows, B_global, Cn, cand_out, sel=None, tokens=None, n_accept=None,
                             stream=None):
        """verify + update of this rank's slots, then its candidate block (2 Cn + 1 words)
        into cand_out; the caller all-gathers the blocks and calls laps_merge."""
        sel = self.sel if sel is None else sel
        _check("laps_step_candidates", _lib.laps_step_candidates(self.h, C.byref(rows.c), B_global, Cn,
                                                                 _dptr(sel), _dptr(tokens), _dptr(n_accept),
                                                                 _dptr(cand_out), _stream(stream)))
        return sel

    def set_peers(self, Cn, group=None, stream=None):
        """Peer-memory exchange for laps_step_peer: a zero-filled buffer of
        lapssd_peer_buffer_bytes(world, Cn) per rank, mapped into every process with torch's
        CUDA IPC (torch.multiprocessing.reductions over torch.distributed), then
        lapssd_set_peers.  world == 1 needs no process group."""
        nbytes = int(_lib.lapssd_peer_buffer_bytes(self.world, Cn))
        own = torch.zeros((nbytes + 7) // 8, dtype=torch.int64, device=self.sel.device)
        bufs = [own]
        if self.world > 1:
            import torch.distributed as dist
            from torch.multiprocessing.reductions import reduce_tensor
            objs = [None] * self.world
            dist.all_gather_object(objs, reduce_tensor(own), group=group)
            bufs = [own if g == self.rank else fn(*args) for g, (fn, args) in enumerate(objs)]
            dist.barrier(group=group)
        self._peer_bufs = bufs                    # keep the mappings alive
        ptrs = (C.c_void_p * self.world)(*[b.data_ptr() for b in bufs])
        _check("lapssd_set_peers", _lib.lapssd_set_peers(self.h, ptrs, Cn, _stream(stream)))

    def laps_step_peer(self, rows: Rows, B_global, sel=None, count=None, tokens=None, n_accept=None,
                       stream=None):
        sel = self.sel if sel is None else sel
        count = self.count if count is None else count
        _check("laps_step_peer", _lib.laps_step_peer(self.h, C.byref(rows.c), B_global, _dptr(sel), _dptr(count),
                                                     _dptr(tokens), _dptr(n_accept), _stream(stream)))
        return sel, count

    # -- snapshot -----------------------------------------------------------------
    def state(self, stream=None) -> dict:
        arrs = _state_arrays(self.n, self.cfg.gamma)
        v = _StateView(0, 0, 0, *[arrs[f].ctypes.data for f in _VIEW_ARRAYS], 0, 0)
        _check("lapssd_read_state", _lib.lapssd_read_state(self.h, C.byref(v), _stream(stream)))
        arrs.update(now_us=v.now_us, cursor=v.cursor, prev_count=v.prev_count,
                    step_cost_us=v.step_cost_us, switch_total_us=v.switch_total_us)
        return arrs

    def profile(self, max_steps: int):
        """Record verify / select kernel times for the next max_steps laps_step calls."""
        _check("lapssd_profile", _lib.lapssd_profile(self.h, max_steps))

    def profile_read(self):
        """(verify_ms, select_ms, presort_ms, steps) summed over the profiled steps."""
        v, s, p, n = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
        _check("lapssd_profile_read", _lib.lapssd_profile_read(self.h, C.byref(v), C.byref(s),
                                                               C.byref(p), C.byref(n)))
        return v.value, s.value, p.value, n.value

    def check(self):
        flags = C.c_uint32()
        rc = _lib.lapssd_check(self.h, C.byref(flags))
        _check("lapssd_check", rc)
        return flags.value

    def check_flags(self) -> int:
        """The device flags (0: none), without raising."""
        flags = C.c_uint32()
        _lib.lapssd_check(self.h, C.byref(flags))
        return flags.value


def _state_arrays(n, gamma):
    return dict(acc_tok=np.zeros(n, np.int32), acc_draft=np.zeros(n, np.int32),
                rounds=np.zeros(n, np.int32), E_us=np.zeros(n, np.int64),
                T_total_us=np.zeros(n, np.int64), C_us=np.zeros(n, np.int64),
                x_us=np.zeros(n, np.int64), admitted=np.zeros(n, np.uint8),
                done=np.zeros(n, np.uint8), perceptible=np.zeros(n, np.uint8),
                pinned=np.zeros(n, np.uint8), level=np.zeros(n, np.uint8),
                running=np.zeros(n, np.uint8), A=np.zeros(n, np.float64),
                key=np.zeros(n, np.uint64), ring=np.zeros((n, gamma), np.int32),
                switch_us=np.zeros(n, np.int64))


# --------------------------------------------------------------------------- Monte-Carlo replicas
class MCHandle:
    """T independent traces, batch 1 each (lapssd_mc_create): configs[4]'s engine.
    Requests are concatenated trace by trace; offsets[t]..offsets[t+1] belong to trace t."""

    def __init__(self, cfg: SchedConfig, offsets, arrival_us, L_true, L_pred, *, V: int, prompt=None,
                 device="cuda", stream=None):
        self.cfg = cfg
        self._cc = cfg.c()
        off = np.ascontiguousarray(offsets, np.int64)
        a = np.ascontiguousarray(arrival_us, np.int64)
        lt = np.ascontiguousarray(L_true, np.int32)
        lp = np.ascontiguousarray(L_pred, np.int32)
        pr = np.ascontiguousarray(prompt, np.int32) if prompt is not None else None
        self.T, self.n, self.V = len(off) - 1, int(off[-1]), V
        self.offsets = off
        nbytes = int(_lib.lapssd_mc_workspace_bytes(C.byref(self._cc), self.T, self.n, V))
        if nbytes == 0:
            raise LapssdError("lapssd_mc_workspace_bytes", -1, "invalid sizes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        h = C.c_void_p()
        rc = _lib.lapssd_mc_create(C.byref(self._cc), self.T, off.ctypes.data, a.ctypes.data, lt.ctypes.data,
                                   lp.ctypes.data, pr.ctypes.data if pr is not None else None, V,
                                   _dptr(self.workspace), nbytes, _stream(stream), C.byref(h))
        _check("lapssd_mc_create", rc)
        self.h = h
        self.active = torch.zeros(1, dtype=torch.int32, device=device)

    def close(self):
        if getattr(self, "h", None):
            _lib.lapssd_mc_destroy(self.h)
            self.h = None

    __del__ = close

    def select(self, rows: Rows, stream=None):
        _check("laps_mc_select", _lib.laps_mc_select(self.h, C.byref(rows.c), _stream(stream)))

    def step(self, rows: Rows, tokens=None, n_accept=None, active=None, stream=None):
        active = self.active if active is None else active
        _check("laps_mc_step", _lib.laps_mc_step(self.h, C.byref(rows.c), _dptr(tokens), _dptr(n_accept),
                                                 _dptr(active), _stream(stream)))
        return active

    def state(self, stream=None):
        """(per-request state dict over all traces, now_us[T], cursor[T], sel[T])."""
        arrs = _state_arrays(self.n, self.cfg.gamma)
        v = _StateView(0, 0, 0, *[arrs[f].ctypes.data for f in _VIEW_ARRAYS], 0, 0)
        now = np.zeros(self.T, np.int64)
        cur = np.zeros(self.T, np.int32)
        sel = np.zeros(self.T, np.int32)
        _check("lapssd_mc_read", _lib.lapssd_mc_read(self.h, C.byref(v), now.ctypes.data, cur.ctypes.data,
                                                      sel.ctypes.data, _stream(stream)))
        arrs["switch_total_us"] = v.switch_total_us
        return arrs, now, cur, sel

    def check(self):
        flags = C.c_uint32()
        _check("lapssd_mc_check", _lib.lapssd_mc_check(self.h, C.byref(flags)))
        return flags.value


# --------------------------------------------------------------------------- NCCL plumbing
def nccl_comm(group=None):
    """Create a NCCL communicator for the library's all-gather: rank 0 draws the
    unique id, torch.distributed broadcasts it, every rank initialises."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = (C.c_uint8 * 128)()
    if rank == 0:
        _check("lapssd_nccl_unique_id", _lib.lapssd_nccl_unique_id(buf))
    t = torch.tensor(list(bytes(buf)), dtype=torch.uint8,
                     device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    dist.broadcast(t, 0, group=group)
    ids = (C.c_uint8 * 128)(*t.cpu().tolist())
    comm = C.c_void_p()
    _check("lapssd_nccl_comm_init", _lib.lapssd_nccl_comm_init(C.byref(comm), world, ids, rank))
    return comm


def nccl_comm_destroy(comm):
    _check("lapssd_nccl_comm_destroy", _lib.lapssd_nccl_comm_destroy(comm))
