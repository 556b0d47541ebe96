"""Pins for SURVEY 8(f) f4 in the oracle: drafting-side sampling and token-tree
verification by multi-step speculative sampling (SpecInfer, cited at P:322; each step is
the rejection rule of P:59-64).  DESIGN.md AMB-34 / AMB-35 state the exact integer forms.

What fixes them from outside the oracle:
* the draft sampler's output law is the row itself (chi-square on V = 16), and on tiny
  rows its choice equals a brute-force inverse CDF in Python integers (Fractions for the
  2^60 quantisation, the oracle's Philox only for the uniform -- pinned by known answers);
* multi-step speculative sampling preserves the target distribution (SpecInfer's
  theorem): the first emitted token of a tree whose root has w i.i.d. children drafted
  from q is distributed as p_root -- chi-square for w = 1..4 -- and in a two-level tree,
  given the accepted first token a, the next emitted token follows p_a;
* a chain (one child per node) is exactly the linear verification (orc_verify_request,
  itself pinned in test_oracle_verify.py);
* special cases: p = q accepts the first child; disjoint supports reject every child and
  emit from p.
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

import oracle


def _rows(V, n, seed, dtype=np.float32, alpha=0.6):
    rng = np.random.default_rng(seed)
    x = rng.dirichlet(np.full(V, alpha), size=n).astype(np.float32)
    if dtype == np.uint16:   # bf16 bit patterns (round to nearest even)
        b = x.view(np.uint32)
        b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
        return b
    return x


def _as_float(rows):
    if rows.dtype == np.uint16:
        return (rows.astype(np.uint32) << 16).view(np.float32)
    return rows


# ---------------------------------------------------------------- draft sampling
def test_draft_sample_law_is_the_row():
    V, n = 16, 60_000
    q = _rows(V, 1, 3)[0]
    obs = np.zeros(V)
    for i in range(n):
        x, Z, inv = oracle.draft_sample(q, i, 0, 0, seed=5)
        assert not inv
        obs[x] += 1
    expect = q.astype(np.float64) / q.sum() * n
    m = expect > 5
    chi2 = (((obs - expect) ** 2 / expect)[m]).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, m.sum() - 1)


@pytest.mark.parametrize("dtype", [np.float32, np.uint16])
def test_draft_sample_brute_force_inverse_cdf(dtype):
    """Tiny rows: the index equals the inverse CDF computed here in exact Python integers."""
    V = 7
    q = _rows(V, 40, 9, dtype)
    seed = 0x1234_5678_9ABC
    for r in range(40):
        for pos in range(3):
            x, Z, _ = oracle.draft_sample(q[r], 100 + r, 7, pos, seed)
            R = [int(Fraction(float(v)) * 2 ** 60) for v in _as_float(q[r])]   # floor: values >= 0
            assert Z == sum(R)
            u = oracle.philox4x32_10([100 + r, 7, (2 << 16) | pos, 0], [seed & 0xFFFFFFFF, seed >> 32])
            U = (int(u[0]) << 32) | int(u[1])
            t = U * Z >> 64
            c, want = 0, None
            for v, Rv in enumerate(R):
                c += Rv
                if c > t:
                    want = v
                    break
            assert x == want


def test_draft_sample_one_hot_and_empty():
    q = np.zeros(32, np.float32)
    q[11] = 1.0
    for i in range(20):
        assert oracle.draft_sample(q, i, 0, 0, 1)[0] == 11
    x, Z, inv = oracle.draft_sample(np.zeros(32, np.float32), 0, 0, 0, 1)
    assert inv and Z == 0 and x == 0


# ---------------------------------------------------------------- tree verification
def _star(p_root, q_root, p_leaf, children):
    """Root with len(children) leaf children (tokens `children`); leaves' rows p_leaf."""
    w = len(children)
    V = p_root.shape[0]
    P = np.stack([p_root] + [p_leaf] * w)
    Q = np.stack([q_root] + [np.zeros(V, p_root.dtype)] * w)
    parent = np.array([-1] + [0] * w, np.int32)
    token = np.array([0] + list(children), np.int32)
    return P, Q, parent, token


@pytest.mark.parametrize("w", [1, 2, 3, 4])
def test_first_token_of_a_tree_is_distributed_as_the_target(w):
    """SpecInfer's theorem: with w children drawn i.i.d. from q, the emitted token after
    the root (the accepted child or the final residual draw) ~ p_root."""
    V, n = 16, 40_000
    p, q = _rows(V, 2, 17 + w)
    p_leaf = _rows(V, 1, 99)[0]
    rng = np.random.default_rng(w)
    qn = q.astype(np.float64) / q.sum()
    obs = np.zeros(V)
    for i in range(n):
        kids = rng.choice(V, size=w, p=qn)
        P, Q, par, tok = _star(p, q, p_leaf, kids)
        na, toks, path, o = oracle.verify_tree(P, Q, par, tok, i, 3, seed=77)
        obs[toks[0]] += 1
        assert o.fallback == 0
    expect = p.astype(np.float64) / p.sum() * n
    m = expect > 5
    chi2 = (((obs - expect) ** 2 / expect)[m]).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, m.sum() - 1)


def test_two_level_tree_second_token_law():
    """Root with 2 children, each with 2 children.  Given that the root's child with token
    a was accepted, the next emitted token follows p_a (the theorem applied at that node,
    whose children were drawn from q_a): chi-square per first token a, pooled."""
    V, n = 6, 60_000
    rows = _rows(V, 2, 5, alpha=1.0)
    p0, q0 = rows[0], rows[1]
    pa = _rows(V, V, 6, alpha=1.0)          # target row after the first token a
    qa = _rows(V, V, 7, alpha=1.0)          # draft row after a
    p_leaf = _rows(V, 1, 8)[0]
    rng = np.random.default_rng(0)
    obs = np.zeros((V, V))
    first = np.zeros(V)
    for i in range(n):
        a = rng.choice(V, size=2, p=q0 / q0.sum())
        b0 = rng.choice(V, size=2, p=qa[a[0]] / qa[a[0]].sum())
        b1 = rng.choice(V, size=2, p=qa[a[1]] / qa[a[1]].sum())
        parent = np.array([-1, 0, 0, 1, 1, 2, 2], np.int32)
        token = np.array([0, a[0], a[1], b0[0], b0[1], b1[0], b1[1]], np.int32)
        P = np.stack([p0, pa[a[0]], pa[a[1]]] + [p_leaf] * 4)
        Q = np.stack([q0, qa[a[0]], qa[a[1]]] + [np.zeros(V, np.float32)] * 4)
        na, toks, path, o = oracle.verify_tree(P, Q, parent, token, i, 0, seed=123)
        first[toks[0]] += 1
        if na >= 1:
            obs[toks[0], toks[1]] += 1
    # the first emitted token ~ p_root whether accepted or drawn
    e1 = p0 / p0.sum() * n
    assert (((first - e1) ** 2 / e1).sum()) < stats.chi2.ppf(1 - 1e-3, V - 1)
    chi2, dof = 0.0, 0
    for a in range(V):
        tot = obs[a].sum()
        if tot < 200:
            continue
        e = pa[a] / pa[a].sum() * tot
        m = e > 5
        chi2 += (((obs[a] - e) ** 2 / e)[m]).sum()
        dof += m.sum() - 1
    assert dof > 10
    assert chi2 < stats.chi2.ppf(1 - 1e-3, dof)


@pytest.mark.parametrize("dtype", [np.float32, np.uint16])
def test_chain_tree_is_the_linear_verification(dtype):
    V, k = 40, 5
    for trial in range(60):
        p = _rows(V, k + 1, 1000 + trial, dtype)
        q = _rows(V, k, 2000 + trial, dtype)
        rng = np.random.default_rng(trial)
        qf = _as_float(q).astype(np.float64)
        draft = np.array([rng.choice(V, p=qf[j] / qf[j].sum()) for j in range(k)], np.int32)
        tok_l, out_l = oracle.verify_request(p, q, draft, 50 + trial, 9, seed=31)
        P = p
        Q = np.concatenate([q, np.zeros((1, V), q.dtype)])
        parent = np.arange(-1, k, dtype=np.int32)
        token = np.concatenate([[0], draft]).astype(np.int32)
        na, toks, path, o = oracle.verify_tree(P, Q, parent, token, 50 + trial, 9, seed=31)
        assert na == out_l.r
        assert (toks == tok_l).all()
        assert o.Z == out_l.Z and o.fallback == out_l.fallback
        assert list(path[:na]) == list(range(1, na + 1))


def test_p_equals_q_accepts_the_first_child():
    V = 32
    p = _rows(V, 1, 4)[0]
    for i in range(200):
        P, Q, par, tok = _star(p, p, p, [i % V, (i + 1) % V, (i + 2) % V])
        na, toks, path, o = oracle.verify_tree(P, Q, par, tok, i, 0, seed=8)
        assert na == 1 and path[0] == 1 and toks[0] == i % V


def test_disjoint_supports_reject_every_child_and_emit_from_p():
    V = 32
    p = np.zeros(V, np.float32)
    q = np.zeros(V, np.float32)
    p[:16] = 1 / 16
    q[16:] = 1 / 16
    for i in range(200):
        kids = [16 + (i + j) % 16 for j in range(3)]
        P, Q, par, tok = _star(p, q, p, kids)
        na, toks, path, o = oracle.verify_tree(P, Q, par, tok, i, 0, seed=8)
        assert na == 0 and o.n_rejected == 3 and toks[0] < 16 and toks[1] == -1


def test_malformed_tree_is_rejected():
    V = 8
    P = _rows(V, 3, 1)
    par = np.array([-1, 2, 0], np.int32)          # parent after child
    assert oracle.verify_tree(P, P, par, np.array([0, 1, 2], np.int32), 0, 0, 1)[0] == -1
    par = np.array([-1, 0, 0], np.int32)
    assert oracle.verify_tree(P, P, par, np.array([0, 1, V], np.int32), 0, 0, 1)[0] == -1
