"""GPU parity of spec_verify (the C-ABI call) against the CPU oracle, element by
element on the same seeded inputs: accepted count r, every emitted token, and the
Q4.60 residual mass Z are compared BIT-EXACTLY (the integer design leaves no
boundary-ambiguous samples; DESIGN.md s.4)."""
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


def oracle_verify(P, slabs, req, rnd, seed, trace=0):
    B = len(slabs)
    k = P["q"].shape[1]
    tok = np.zeros((B, k + 1), np.int32)
    na = np.zeros(B, np.int32)
    z = np.zeros(B, np.uint64)
    for b in range(B):
        s = slabs[b]
        t, o = oracle.verify_request(P["p"][s], P["q"][s], P["draft"][s], req[b], rnd[b], seed,
                                     trace)
        tok[b], na[b], z[b] = t, o.r, o.Z
    return tok, na, z


def gpu_verify(L, pool, slabs, req, rnd, seed, trace=0):
    dev = pool.p.device
    tok, na, z = L.spec_verify(
        pool.p, pool.q, pool.draft,
        torch.as_tensor(req.astype(np.int64), device=dev).to(torch.int32),
        torch.as_tensor(rnd.astype(np.int64), device=dev).to(torch.int32), seed,
        slab=torch.as_tensor(slabs, dtype=torch.int32, device=dev), trace=trace)
    torch.cuda.synchronize()
    return tok.cpu().numpy(), na.cpu().numpy(), z.cpu().numpy().view(np.uint64)


def check_parity(L, pool, B, seed, rng):
    P = pool.numpy()
    slabs = rng.integers(0, pool.S, size=B).astype(np.int32)
    req = rng.integers(0, 2**24, size=B).astype(np.uint32)
    rnd = rng.integers(0, 5000, size=B).astype(np.uint32)
    g = gpu_verify(L, pool, slabs, req, rnd, seed)
    o = oracle_verify(P, slabs, req, rnd, seed)
    assert (g[1] == o[1]).all(), "accepted counts differ"
    assert (g[2] == o[2]).all(), "residual mass Z differs"
    assert (g[0] == o[0]).all(), "emitted tokens differ"
    return o


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("V", [16, 1000, 8200, 16392, 32000, 128256, 524288])
@pytest.mark.parametrize("k", [1, 4, 8])
def test_spec_verify_parity_grid(L, dtype, V, k):
    pool = synth.make_pool("f2", V=V, k=k, dtype=dtype, n_buckets=4, variants=2, seed=V + k,
                           device="cuda")
    rng = np.random.default_rng(V * 31 + k)
    o = check_parity(L, pool, B=48, seed=1234 + k, rng=rng)
    assert len(np.unique(o[1])) >= 2  # both rejection and acceptance paths exercised


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_spec_verify_parity_k6_mixture(L, dtype):
    pool = synth.make_pool("f1", V=4096, k=6, dtype=dtype, n_buckets=8, variants=2, seed=3,
                           device="cuda")
    check_parity(L, pool, B=96, seed=77, rng=np.random.default_rng(0))


def test_spec_verify_config4_launch(L):
    """Full-size launch configuration of the bench: V=128256, k=8, bf16, B=512."""
    pool = synth.make_pool("f2", V=128256, k=8, dtype="bf16", n_buckets=16, variants=2, seed=4,
                           device="cuda")
    check_parity(L, pool, B=512, seed=0x5D0004, rng=np.random.default_rng(4))


def _pool_from(p, q, draft, dtype):
    tdt = synth.torch_dtype(dtype)
    return synth.Pool(p=torch.as_tensor(p).to(tdt).cuda(), q=torch.as_tensor(q).to(tdt).cuda(),
                      draft=torch.as_tensor(draft, dtype=torch.int32).cuda(), family="custom",
                      n_buckets=1, variants=1)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_special_cases(L, dtype):
    V, k = 16384 + 64, 4  # two bf16 chunks (ragged), three fp32 chunks
    rng = np.random.default_rng(2)
    base = rng.random((k + 1, V)).astype(np.float32)
    base /= base.sum(1, keepdims=True)
    ps, qs, ds = [], [], []
    # 0: p == q -> always accept, bonus from p_k
    ps.append(base.copy()); qs.append(base[:k].copy()); ds.append([1, 2, 3, 4])
    # 1: disjoint supports -> reject at 0, y ~ p_0
    p = np.zeros((k + 1, V), np.float32); q = np.zeros((k, V), np.float32)
    p[:, V // 2:] = 2.0 / V; q[:, :V // 2] = 2.0 / V
    ps.append(p); qs.append(q); ds.append([5, 6, 7, 8])
    # 2: p_r <= q_r everywhere with rejection at 0 -> zero residual, fallback to p_r (AMB-20)
    q2 = base[:k].copy(); p2 = base.copy(); p2[0] = 0.5 * q2[0]
    x2 = int(np.argmax(q2[0])); p2[0, x2] = 0.0
    ps.append(p2); qs.append(q2); ds.append([x2, 1, 2, 3])
    # 3: one-hot residual
    p3 = np.zeros((k + 1, V), np.float32); q3 = np.zeros((k, V), np.float32)
    p3[0, V - 3] = 1.0; q3[0, 11] = 1.0; p3[1:, 0] = 1.0; q3[1:, 0] = 1.0
    ps.append(p3); qs.append(q3); ds.append([11, 0, 0, 0])
    pool = _pool_from(np.stack(ps), np.stack(qs), np.array(ds), dtype)
    P = pool.numpy()
    B = 64
    slabs = np.repeat(np.arange(4, dtype=np.int32), B // 4)
    req = np.arange(B, dtype=np.uint32)
    rnd = np.full(B, 3, np.uint32)
    g = gpu_verify(L, pool, slabs, req, rnd, 9)
    o = oracle_verify(P, slabs, req, rnd, 9)
    for a, b in zip(g, o):
        assert (a == b).all()
    tok, na, z = g
    assert (na[slabs == 0] == k).all()
    assert (na[slabs == 1] == 0).all() and (tok[slabs == 1, 0] >= V // 2).all()
    assert (na[slabs == 2] == 0).all() and (z[slabs == 2] > 0).all()
    assert (tok[slabs == 3, 0] == V - 3).all()


def test_trace_and_seed_change_the_draws(L):
    pool = synth.make_pool("f2", V=1024, k=4, dtype="bf16", n_buckets=4, variants=2, seed=5,
                           device="cuda")
    P = pool.numpy()
    B = 64
    slabs = np.zeros(B, np.int32)
    req = np.arange(B, dtype=np.uint32)
    rnd = np.zeros(B, np.uint32)
    a = gpu_verify(L, pool, slabs, req, rnd, 1, trace=0)
    b = gpu_verify(L, pool, slabs, req, rnd, 1, trace=7)
    ob = oracle_verify(P, slabs, req, rnd, 1, trace=7)
    assert (b[0] == ob[0]).all() and (b[1] == ob[1]).all()
    assert (a[0] != b[0]).any()


def test_workspace_left_zeroed_for_reuse(L):
    pool = synth.make_pool("f2", V=32000, k=4, dtype="bf16", n_buckets=2, variants=2, seed=6,
                           device="cuda")
    B = 32
    ws = torch.zeros(L.spec_verify_workspace_bytes(B, 32000), dtype=torch.uint8, device="cuda")
    req = torch.arange(B, dtype=torch.int32, device="cuda")
    rnd = torch.zeros(B, dtype=torch.int32, device="cuda")
    slab = torch.zeros(B, dtype=torch.int32, device="cuda")
    outs = [L.spec_verify(pool.p, pool.q, pool.draft, req, rnd, 3, slab=slab, workspace=ws)
            for _ in range(3)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[2], outs[0][2])
