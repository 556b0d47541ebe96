"""Probe (tooling): spec_verify reading its rows in place from pinned host memory (UVA
zero-copy) -- same results as from device memory, and its speed."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402
import ctypes as C  # noqa: E402

L._dptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())   # allow pinned host tensors

B, V, k = 64, 128256, 8
pool = synth.make_pool("f2", V=V, k=k, dtype="bf16", n_buckets=8, variants=8, seed=3, device="cuda")
req = torch.arange(B, dtype=torch.int32, device="cuda")
rnd = torch.zeros(B, dtype=torch.int32, device="cuda")
tok_d, na_d, z_d = L.spec_verify(pool.p, pool.q, pool.draft, req, rnd, 11)
hp, hq, hd = pool.p.cpu().pin_memory(), pool.q.cpu().pin_memory(), pool.draft.cpu().pin_memory()
torch.cuda.synchronize()
outs = dict(tokens=torch.empty_like(tok_d), n_accept=torch.empty_like(na_d), z=torch.empty_like(z_d),
            workspace=torch.zeros(L.spec_verify_workspace_bytes(B, V), dtype=torch.uint8, device="cuda"))
tok_h, na_h, z_h = L.spec_verify(hp, hq, hd, req, rnd, 11, **outs)
torch.cuda.synchronize()
print("same r", bool((na_h == na_d).all()), "same tokens", bool((tok_h == tok_d).all()), "same Z", bool((z_h == z_d).all()))
for name, (p, q, d) in {"device": (pool.p, pool.q, pool.draft), "host": (hp, hq, hd)}.items():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        L.spec_verify(p, q, d, req, rnd, 11, **outs)
    torch.cuda.synchronize()
    print(name, "%.3f ms per call" % ((time.perf_counter() - t0) / 5 * 1e3))
