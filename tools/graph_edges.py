"""Capture two laps_step calls in a CUDA graph and print its nodes and edge types
(tooling: which dependencies the programmatic-launch attribute turned programmatic)."""
import os
import sys

import torch
from cuda.bindings import runtime as rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_17074_b200 as L  # noqa: E402
import synth  # noqa: E402

tr = synth.make_trace(256, 7, arrival="zero", length="uniform", len_min=512, len_max=4096, beta_ab=(7, 3))
pool = synth.make_pool("f2", V=32000, k=8, dtype="bf16", n_buckets=8, variants=4, seed=7, device="cuda")
tab = synth.slab_table(tr, 8, 4, R=16, seed=7)
h = L.Handle(L.SchedConfig(K=4, s1_up_us=72000, k=8, seed=9), tr.arrival_us, tr.L_true, tr.L_pred,
             max_batch=64, V=32000)
rows = L.Rows(pool.p, pool.q, pool.draft, torch.as_tensor(tab, device="cuda"))
h.laps_select(64)
for _ in range(3):
    h.laps_step(rows, 64)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph(keep_graph=True)
with torch.cuda.graph(g):
    for _ in range(2):
        h.laps_step(rows, 64)
raw = g.raw_cuda_graph()
err, nodes, n = rt.cudaGraphGetNodes(raw, 0)
err, nodes, n = rt.cudaGraphGetNodes(raw, n)
idx = {}
for j, nd in enumerate(nodes):
    err, ty = rt.cudaGraphNodeGetType(nd)
    name = str(ty).split(".")[-1]
    if ty == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
        err, p = rt.cudaGraphKernelNodeGetParams(nd)
        err, fname = rt.cudaFuncGetName(p.func) if hasattr(rt, "cudaFuncGetName") else (0, b"?")
        name += " " + (fname.decode() if isinstance(fname, bytes) else str(fname))[:60]
    idx[int(nd)] = j
    print(j, name)
res = rt.cudaGraphGetEdges_v2(raw, 0)
ne = res[-1]
res = rt.cudaGraphGetEdges_v2(raw, ne)
frm, to, data = res[1], res[2], res[3]
for a, b, d in zip(frm, to, data):
    print("edge %d -> %d  type %s  from_port %s" % (idx[int(a)], idx[int(b)], d.type, d.from_port))
