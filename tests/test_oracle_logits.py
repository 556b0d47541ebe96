"""Pins of the logits-input verification oracle (DESIGN.md AMB-30):
p = softmax(target logits), q = softmax(draft logits), then P:59-64 / P:200.  Nothing
here compares the oracle with itself: the references are math.exp, the fp64 softmax,
the speculative-sampling identity (first emitted token ~ p), the accepted-count law and
exact special cases."""
import math

import numpy as np
import pytest

import oracle

CHI2_15_P001 = 37.70   # chi-square critical values at p = 1e-3
CHI2_4_P001 = 18.47
CHI2_7_P001 = 24.32


def chi2(counts, probs):
    n = counts.sum()
    e = n * probs
    m = e > 0
    return float((((counts - e) ** 2)[m] / e[m]).sum())


def softmax64(z):
    z = np.asarray(z, np.float64)
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def test_exp_hat_against_math_exp():
    d = np.linspace(-28.0, 0.0, 40001).astype(np.float32)
    worst = 0.0
    for x in d[::7]:
        ref = math.exp(float(x))
        worst = max(worst, abs(oracle.exp_hat(float(x)) - ref) / ref)
    assert worst < 2.5e-7, worst           # ~2 fp32 ulp
    assert oracle.exp_hat(0.0) == 1.0
    assert oracle.exp_hat(-28.5) == 0.0 and oracle.exp_hat(-1e30) == 0.0


def _rows(rng, k, V, scale=2.0, eps=0.8):
    zp = (scale * rng.standard_normal((k + 1, V))).astype(np.float32)
    zq = (zp[:k] + eps * rng.standard_normal((k, V))).astype(np.float32)
    return zp, zq


def _drafts(rng, zq, n):
    q = softmax64(zq)
    k, V = q.shape
    return np.stack([rng.choice(V, size=n, p=q[j]) for j in range(k)], axis=1).astype(np.int32)


def test_first_emitted_token_follows_target_softmax():
    """Speculative-sampling identity (leviathan2023fast, relied on at P:59-64): the first
    emitted token is distributed as p_0 = softmax(zp_0), whatever q is."""
    rng = np.random.default_rng(5)
    k, V, n = 4, 16, 200_000
    zp, zq = _rows(rng, k, V)
    d = _drafts(rng, zq, n)
    tok, r = oracle.verify_logits_many(zp, zq, d, np.arange(n), np.zeros(n), seed=91)
    counts = np.bincount(tok[:, 0], minlength=V)
    assert chi2(counts, softmax64(zp[0])) < CHI2_15_P001


def test_accepted_count_law_and_expected_tokens():
    """Identical rows at every position: P(r=j) = b^j (1-b), P(r=k) = b^k with
    b = sum_v min(p_v, q_v) (fp64 softmax); E[tokens] = (1-b^(k+1))/(1-b)."""
    rng = np.random.default_rng(6)
    k, V, n = 4, 32, 200_000
    zp1, zq1 = _rows(rng, 1, V)
    zp = np.repeat(zp1[:1], k + 1, 0)
    zq = np.repeat(zq1[:1], k, 0)
    b = float(np.minimum(softmax64(zp[0]), softmax64(zq[0])).sum())
    d = _drafts(rng, zq, n)
    _, r = oracle.verify_logits_many(zp, zq, d, np.arange(n), np.zeros(n), seed=92)
    probs = np.array([b ** j * (1 - b) for j in range(k)] + [b ** k])
    assert chi2(np.bincount(r, minlength=k + 1), probs) < CHI2_4_P001
    emitted = (r + 1).mean()
    want = (1 - b ** (k + 1)) / (1 - b)
    sd = (r + 1).std() / math.sqrt(n)
    assert abs(emitted - want) < 5 * sd


def test_equal_logits_accept_everything_and_bonus_follows_last_row():
    """zq = zp: p^ = q^ exactly (same integers), so every draft is accepted (u < 1) and
    the bonus token follows softmax(zp_k)."""
    rng = np.random.default_rng(7)
    k, V, n = 3, 16, 100_000
    zp = (2.0 * rng.standard_normal((k + 1, V))).astype(np.float32)
    zq = zp[:k].copy()
    d = _drafts(rng, zq, n)
    tok, r = oracle.verify_logits_many(zp, zq, d, np.arange(n), np.zeros(n), seed=93)
    assert (r == k).all()
    assert chi2(np.bincount(tok[:, k], minlength=V), softmax64(zp[k])) < CHI2_15_P001


def test_disjoint_supports_reject_first_and_residual_is_target():
    """q^ on a half A of the vocabulary, p^ on the complement (logits -100 elsewhere:
    e^-100 < 2^-40, so E = 0): every draft has p^ = 0, r = 0, and y ~ p^ = uniform on
    the complement."""
    rng = np.random.default_rng(8)
    k, V, n = 2, 16, 40_000
    A = rng.permutation(V)[: V // 2]
    inA = np.zeros(V, bool)
    inA[A] = True
    zq = np.where(inA, 0.0, -100.0).astype(np.float32)[None].repeat(k, 0)
    zp = np.where(inA, -100.0, 0.0).astype(np.float32)[None].repeat(k + 1, 0)
    d = rng.choice(A, size=(n, k)).astype(np.int32)
    tok, r = oracle.verify_logits_many(zp, zq, d, np.arange(n), np.zeros(n), seed=94)
    assert (r == 0).all()
    y = tok[:, 0]
    assert (~inA[y]).all()
    probs = np.where(inA, 0.0, 1.0 / (V - V // 2))
    assert chi2(np.bincount(y, minlength=V), probs) < CHI2_7_P001  # 8 cells, 7 dof


def test_bf16_logits_and_slab_batch_agree_with_single_requests():
    """The batch entry point is the single-request definition applied slot by slot, and
    bf16 logits (stored as bit patterns) are read exactly."""
    rng = np.random.default_rng(9)
    S, k, V, B = 3, 4, 300, 10
    zp32 = (2 * rng.standard_normal((S, k + 1, V))).astype(np.float32)
    zq32 = (zp32[:, :k] + rng.standard_normal((S, k, V))).astype(np.float32)
    to_bf16 = lambda x: (x.view(np.uint32) >> 16).astype(np.uint16)  # noqa: E731  (truncation: any bf16 is fine)
    zp, zq = to_bf16(zp32), to_bf16(zq32)
    drafts = rng.integers(0, V, (S, k)).astype(np.int32)
    slab = rng.integers(0, S, B).astype(np.int32)
    req = np.arange(100, 100 + B)
    rnd = rng.integers(0, 50, B)
    tok, r, _ = oracle.verify_logits_batch(zp, zq, drafts, slab, req, rnd, seed=95)
    for b in range(B):
        t1, o = oracle.verify_logits_request(zp[slab[b]], zq[slab[b]], drafts[slab[b]], req[b], rnd[b], seed=95)
        assert (t1 == tok[b]).all() and o.r == r[b]


@pytest.mark.parametrize("dtype", [np.float32, np.uint16])
def test_quantised_softmax_within_1e6_of_fp64_softmax_at_large_V(dtype):
    """AMB-30 against the exact softmax of the STORED logits, at V = 128,256 (configs[3]):
    every probability >= 1e-5 within 1e-6 relative, total variation < 1e-6, and the
    residual mass Z / (Sp Sq) of a row pair within 1e-6 relative of the fp64
    sum_v max(0, p - q) (north_star's tolerance on residual probabilities)."""
    V = 128256
    rng = np.random.default_rng(7 if dtype == np.float32 else 8)
    for trial in range(3):
        ranks = rng.permutation(V) + 1
        zp = (-1.1 * np.log(ranks) + rng.normal(0, 1.5, V)).astype(np.float32)
        zq = (zp + rng.normal(0, 0.8, V)).astype(np.float32)
        if dtype == np.uint16:   # bf16 bit patterns (round to nearest even)
            to_bf = lambda x: ((x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
            zp_s, zq_s = to_bf(zp), to_bf(zq)
            zp_f = (zp_s.astype(np.uint32) << 16).view(np.float32)
            zq_f = (zq_s.astype(np.uint32) << 16).view(np.float32)
        else:
            zp_s, zq_s, zp_f, zq_f = zp, zq, zp, zq
        ref = []
        for zs, zf in ((zp_s, zp_f), (zq_s, zq_f)):
            E, S, m = oracle.logits_row(zs)
            assert m == zf.max()
            ph = E.astype(np.float64) / float(S)
            x = zf.astype(np.float64)
            p = np.exp(x - x.max())
            p /= p.sum()
            big = p >= 1e-5
            assert (np.abs(ph[big] - p[big]) / p[big]).max() < 1e-6
            assert np.abs(ph - p).sum() < 1e-6
            ref.append((E, S, p))
        (Ep, Sp, p), (Eq, Sq, q) = ref
        # the integer residual of spec_verify_logits: max(0, Ep Sq - Eq Sp) / (Sp Sq)
        Ep_o = [int(e) for e in Ep]
        Eq_o = [int(e) for e in Eq]
        Z = sum(max(0, a * Sq - b * Sp) for a, b in zip(Ep_o, Eq_o))
        exact = np.maximum(p - q, 0).sum()
        assert abs(Z / (Sp * Sq) - exact) / exact < 1e-6
