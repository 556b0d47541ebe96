"""SURVEY 8(f) f4 on the GPU through the C-ABI, bit-exact against the oracle:
spec_draft_sample (drafting-side inverse-CDF sampling) and spec_verify_tree
(token-tree multi-step speculative sampling, SpecInfer at P:322) -- tokens, accepted
paths, counts and the integer mass of every final draw.  The oracle's pins are
tests/test_oracle_f4.py."""
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


def _softmax_rows(n, V, seed, dtype, sharp=2.0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    z = torch.randn(n, V, generator=g, device="cuda") * sharp
    return torch.softmax(z, -1).to(dtype), z


def _pair(n, V, seed, dtype, eps=0.7):
    """Target / draft rows with moderate acceptance: q = softmax(z + eps noise)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    z = torch.randn(n, V, generator=g, device="cuda") * 2.5
    p = torch.softmax(z, -1)
    q = torch.softmax(z + eps * torch.randn(n, V, generator=g, device="cuda"), -1)
    return p.to(dtype), q.to(dtype)


@pytest.mark.parametrize("V,dtype", [(32000, torch.bfloat16), (128256, torch.bfloat16), (8200, torch.float32),
                                     (24, torch.float32)])
def test_draft_sample_parity(L, V, dtype):
    R = 48
    q, _ = _softmax_rows(R, V, 3 + V, dtype)
    req = torch.arange(R, dtype=torch.int32, device="cuda") * 7 + 1
    rnd = torch.full((R,), 5, dtype=torch.int32, device="cuda")
    pos = torch.arange(R, dtype=torch.int32, device="cuda") % 8
    x, z = L.spec_draft_sample(q, req, rnd, pos, seed=0xD7A1)
    Q = synth.to_numpy_rows(q)
    xs, zs = x.cpu().numpy(), z.cpu().numpy().view(np.uint64)
    for r in range(R):
        xo, zo, inv = oracle.draft_sample(Q[r], int(req[r]), 5, int(pos[r]), 0xD7A1)
        assert not inv
        assert xs[r] == xo and zs[r] == zo, f"row {r}"


def test_draft_sample_row_index_and_law(L):
    """Rows picked from a pool by index; many draws from one row follow the row."""
    V, R = 64, 4096
    q, _ = _softmax_rows(3, V, 11, torch.float32, sharp=1.0)
    row = torch.full((R,), 2, dtype=torch.int32, device="cuda")
    req = torch.arange(R, dtype=torch.int32, device="cuda")
    zero = torch.zeros(R, dtype=torch.int32, device="cuda")
    x, _ = L.spec_draft_sample(q, req, zero, zero, seed=9, row=row)
    cnt = torch.bincount(x.long(), minlength=V).cpu().numpy()
    expect = q[2].double().cpu().numpy() / q[2].double().sum().item() * R
    from scipy import stats
    m = expect > 5
    assert (((cnt - expect) ** 2 / expect)[m]).sum() < stats.chi2.ppf(1 - 1e-3, m.sum() - 1)
    Q = synth.to_numpy_rows(q)
    for r in range(0, R, 257):
        assert int(x[r]) == oracle.draft_sample(Q[2], r, 0, 0, 9)[0]


def _random_tree(rng, n, max_w, q_rows_np, V):
    """A tree with up to n nodes: each new node picks a parent among the existing ones
    with fewer than max_w children; its token is drawn from the parent's draft row."""
    parent = np.full(n, -1, np.int32)
    token = np.zeros(n, np.int32)
    kids = np.zeros(n, np.int32)
    for c in range(1, n):
        if rng.random() < 0.1:       # an unused node
            continue
        cands = [u for u in range(c) if (u == 0 or parent[u] >= 0) and kids[u] < max_w]
        u = int(rng.choice(cands))
        parent[c] = u
        kids[u] += 1
        row = q_rows_np[u].astype(np.float64)
        token[c] = rng.choice(V, p=row / row.sum())
    return parent, token


def _run_tree_parity(L, B, n, V, dtype, max_w, seed, eps=0.7):
    p, q = _pair(B * n, V, seed, dtype, eps)
    p = p.view(B, n, V).contiguous()
    q = q.view(B, n, V).contiguous()
    P, Q = synth.to_numpy_rows(p), synth.to_numpy_rows(q)
    Qf = q.float().cpu().numpy()
    rng = np.random.default_rng(seed)
    par = np.zeros((B, n), np.int32)
    tok = np.zeros((B, n), np.int32)
    for b in range(B):
        par[b], tok[b] = _random_tree(rng, n, max_w, Qf[b], V)
    req = torch.arange(B, dtype=torch.int32, device="cuda") + 1000
    rnd = torch.full((B,), 17, dtype=torch.int32, device="cuda")
    t_g, path_g, na_g, z_g = L.spec_verify_tree(p, q, torch.as_tensor(par, device="cuda"),
                                                torch.as_tensor(tok, device="cuda"), req, rnd, seed=0x7EE)
    t_g, path_g, na_g = t_g.cpu().numpy(), path_g.cpu().numpy(), na_g.cpu().numpy()
    z_g = z_g.cpu().numpy().view(np.uint64)
    stats_ = dict(accepted=0, rejected=0)
    for b in range(B):
        na, toks, path, o = oracle.verify_tree(P[b], Q[b], par[b], tok[b], 1000 + b, 17, seed=0x7EE)
        assert na_g[b] == na, f"request {b}: n_accept {na_g[b]} != {na}"
        assert (t_g[b] == toks).all(), f"request {b}: tokens"
        assert (path_g[b] == path).all(), f"request {b}: path"
        assert z_g[b] == o.Z, f"request {b}: Z"
        stats_["accepted"] += na
        stats_["rejected"] += o.n_rejected
    return stats_


@pytest.mark.parametrize("V,dtype,max_w", [(32000, torch.bfloat16, 3), (8200, torch.float32, 4),
                                           (128256, torch.bfloat16, 2)])
def test_tree_parity(L, V, dtype, max_w):
    s = _run_tree_parity(L, B=24, n=16, V=V, dtype=dtype, max_w=max_w, seed=V + max_w)
    assert s["accepted"] > 10 and s["rejected"] > 10     # both branches exercised


def test_tree_parity_wide_low_acceptance(L):
    """Many rejected children per node (low acceptance): long residual chains."""
    s = _run_tree_parity(L, B=16, n=24, V=4096, dtype=torch.bfloat16, max_w=8, seed=5, eps=2.5)
    assert s["rejected"] > 40


def test_chain_tree_equals_spec_verify(L):
    """A chain tree (one child per node) through spec_verify_tree == spec_verify."""
    B, k, V = 32, 6, 32000
    p, q = _pair(B * (k + 1), V, 77, torch.bfloat16)
    p = p.view(B, k + 1, V).contiguous()
    q = q.view(B, k + 1, V).contiguous()
    q[:, k] = 0
    req = torch.arange(B, dtype=torch.int32, device="cuda")
    rnd = torch.full((B,), 3, dtype=torch.int32, device="cuda")
    pos = torch.arange(k, dtype=torch.int32, device="cuda").repeat(B)
    rows = (torch.arange(B, device="cuda")[:, None] * (k + 1) + torch.arange(k, device="cuda")).view(-1).int()
    draft, _ = L.spec_draft_sample(q, req.repeat_interleave(k), rnd.repeat_interleave(k), pos, seed=1, row=rows)
    draft = draft.view(B, k)
    tok_l, na_l, z_l = L.spec_verify(p, q[:, :k].contiguous(), draft, req, rnd, seed=0xC4A1)
    parent = torch.arange(-1, k, dtype=torch.int32, device="cuda").repeat(B, 1).contiguous()
    token = torch.cat([torch.zeros(B, 1, dtype=torch.int32, device="cuda"), draft], 1).contiguous()
    t_t, path_t, na_t, z_t = L.spec_verify_tree(p, q, parent, token, req, rnd, seed=0xC4A1)
    assert (na_t == na_l).all()
    assert (t_t == tok_l).all()
    assert (z_t == z_l).all()


def test_malformed_trees(L):
    B, n, V = 3, 4, 64
    p, q = _pair(B * n, V, 1, torch.float32)
    p, q = p.view(B, n, V).contiguous(), q.view(B, n, V).contiguous()
    parent = torch.tensor([[-1, 0, 3, 0], [-1, 0, 0, 1], [-1, 0, 1, 2]], dtype=torch.int32, device="cuda")
    token = torch.tensor([[0, 1, 2, 3], [0, 1, 2, V], [0, 5, 6, 7]], dtype=torch.int32, device="cuda")
    req = torch.arange(B, dtype=torch.int32, device="cuda")
    _, _, na, _ = L.spec_verify_tree(p, q, parent, token, req, req, seed=2)
    na = na.cpu().numpy()
    assert na[0] == -1 and na[1] == -1 and na[2] >= 0
