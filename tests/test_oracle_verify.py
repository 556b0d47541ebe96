"""Pins for the oracle's verification step and its RNG.

Every expected value here comes from outside the oracle: published known-answer
vectors, textbook closed forms of speculative sampling (Leviathan et al. / Chen et
al., cited at P:11), exact special cases, and chi-square tests against the target
distribution.  No value is produced by the oracle's own formulas.
"""
import numpy as np
import pytest
import torch
from scipy import stats

import oracle
import synth
from conftest import golden


# ---------------------------------------------------------------- Philox (PIN-R1)
def test_philox_known_answers():
    n = 0
    for line in open(golden("philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        out = oracle.philox4x32_10(w[0:4], w[4:6])
        assert list(out) == w[6:10], line
        n += 1
    assert n == 3


# ---------------------------------------------------------------- helpers
def f1(V, k, beta, seed, dtype=torch.float32):
    g = torch.Generator()
    g.manual_seed(seed)
    p, q, d = synth.f1_rows(V, k, [beta] * (k + 1), g, dtype=dtype)
    return synth.to_numpy_rows(p), synth.to_numpy_rows(q), d.numpy().astype(np.int32)


def trials(p, q, draft, n, seed=7):
    d = np.tile(draft, (n, 1))
    ids = np.arange(n, dtype=np.uint32)
    rounds = np.zeros(n, np.uint32)
    return oracle.verify_many(p, q, d, ids, rounds, seed)


# ---------------------------------------------------------------- closed forms (PIN-C1/C2)
@pytest.mark.parametrize("beta,k,expect", [(0.5, 4, 1.9375), (0.7, 8, None), (0.1, 4, None),
                                           (0.9, 4, None)])
def test_expected_tokens_per_step_closed_form(beta, k, expect):
    """E[tokens per step] = (1 - b^(k+1)) / (1 - b) for per-position acceptance b
    (leviathan2023fast, cited P:11); the mixture rows make b exact."""
    closed = (1 - beta ** (k + 1)) / (1 - beta)
    if expect is not None:
        assert closed == pytest.approx(expect)
    p, q, d = f1(16, k, beta, seed=11)
    n = 200_000
    _, r = trials(p, q, d, n)
    emitted = r + 1
    sigma = emitted.std() / np.sqrt(n)
    assert abs(emitted.mean() - closed) < 5 * sigma + 1e-6


@pytest.mark.parametrize("beta,k", [(0.5, 4), (0.3, 6)])
def test_accepted_count_law_chi_square(beta, k):
    """P(r = j) = b^j (1 - b) for j < k and P(r = k) = b^k (the first rejection of
    independent Bernoulli(b) acceptances)."""
    p, q, d = f1(16, k, beta, seed=3)
    n = 200_000
    _, r = trials(p, q, d, n, seed=99)
    expect = np.array([beta ** j * (1 - beta) for j in range(k)] + [beta ** k]) * n
    obs = np.bincount(r, minlength=k + 1)
    chi2 = ((obs - expect) ** 2 / expect).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, k)


# ---------------------------------------------------------------- PIN-D
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_first_token_distributed_as_target(dtype):
    """The token emitted at position 0 (accepted draft or resample) is distributed
    exactly as p_0 when x_0 ~ q_0 (speculative sampling identity: min(p,q) +
    max(0,p-q) = p).  Brute-force chi-square on V = 16."""
    V, k, n = 16, 3, 400_000
    rng = np.random.default_rng(5)
    g = torch.Generator()
    g.manual_seed(5)
    p = torch.softmax(torch.randn(k + 1, V, generator=g) * 1.5, -1).to(dtype)
    q = torch.softmax(torch.randn(k, V, generator=g) * 1.5, -1).to(dtype)
    pn, qn = synth.to_numpy_rows(p), synth.to_numpy_rows(q)
    qf = q.float().numpy().astype(np.float64)
    drafts = np.stack([rng.choice(V, size=n, p=qf[j] / qf[j].sum()) for j in range(k)], 1)
    tok, r = oracle.verify_many(pn, qn, drafts, np.arange(n), np.zeros(n), seed=123)
    p0 = p.float().numpy().astype(np.float64)[0]
    # The stored rows are not exactly normalised; the emitted law is then
    # min(p,q) + max(0, p-q) * (1 - sum min) / sum max(0,p-q) -- with stored values.
    q0 = qf[0] / qf[0].sum()
    acc = np.minimum(p0, q0)
    res = np.maximum(p0 - q0, 0)
    law = acc + res * (1 - acc.sum()) / res.sum()
    obs = np.bincount(tok[:, 0], minlength=V)
    expect = law * n
    chi2 = ((obs - expect) ** 2 / expect).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, V - 1)
    # and the law is p_0 up to the storage rounding
    assert np.abs(law - p0 / p0.sum()).max() < 2e-2


# ---------------------------------------------------------------- PIN-S special cases
def test_p_equals_q_accepts_everything_bonus_from_p_k():
    V, k = 32, 4
    g = torch.Generator()
    g.manual_seed(1)
    rows = torch.softmax(torch.randn(k + 1, V, generator=g), -1)
    p = rows.numpy().astype(np.float32)
    q = p[:k].copy()
    draft = np.array([3, 9, 0, 31], np.int32)
    n = 100_000
    tok, r = trials(p, q, draft, n)
    assert (r == k).all()
    assert (tok[:, :k] == draft).all()
    obs = np.bincount(tok[:, k], minlength=V)
    law = p[k].astype(np.float64) / p[k].astype(np.float64).sum()
    chi2 = ((obs - law * n) ** 2 / (law * n)).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, V - 1)


def test_disjoint_supports_reject_first_and_sample_p():
    V, k = 16, 4
    p = np.zeros((k + 1, V), np.float32)
    q = np.zeros((k, V), np.float32)
    p[:, 8:] = 1 / 8
    q[:, :8] = 1 / 8
    draft = np.array([0, 1, 2, 3], np.int32)
    n = 80_000
    tok, r = trials(p, q, draft, n)
    assert (r == 0).all()
    assert (tok[:, 1:] == -1).all()
    obs = np.bincount(tok[:, 0], minlength=V)
    assert obs[:8].sum() == 0
    chi2 = ((obs[8:] - n / 8) ** 2 / (n / 8)).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, 7)


def test_one_hot_residual_is_deterministic():
    V, k = 64, 2
    p = np.zeros((k + 1, V), np.float32)
    q = np.zeros((k, V), np.float32)
    p[0, 41] = 1.0
    q[0, 7] = 1.0
    p[1:, 5] = 1.0
    q[1, 5] = 1.0
    tok, r = trials(p, q, np.array([7, 5], np.int32), 1000)
    assert (r == 0).all() and (tok[:, 0] == 41).all()


@pytest.mark.parametrize("beta", [0.25, 0.5, 0.875])
def test_mixture_residual_is_exactly_rho(beta):
    """F1 rows: p = b q + (1-b) rho with disjoint supports: the residual max(0,p-q)
    is (1-b) rho, so every resampled token lies in supp(rho), uniformly, and the
    residual mass Z * 2^-60 equals 1 - b."""
    V, k = 16, 4
    p, q, d = f1(V, k, beta, seed=21)
    n = 100_000
    tok, r = trials(p, q, d, n, seed=5)
    rej = r < k
    ys = tok[np.arange(n), r][rej]
    rho_support = np.nonzero(q[0] == 0)[0]
    assert np.isin(ys[r[rej] == 0], rho_support).all()
    for j in range(k):
        supp = np.nonzero(q[j] == 0)[0]
        yj = tok[np.arange(n), r][r == j]
        assert np.isin(yj, supp).all()
    _, o = oracle.verify_request(p, q, d, req_id=0, round_idx=0, seed=1)
    if o.r < k:
        assert o.Z * 2.0 ** -60 == pytest.approx(1 - beta, rel=1e-6)


# ---------------------------------------------------------------- exactness (PIN-X)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_residual_mass_within_1e6_of_exact(dtype):
    """Q4.60 mass of fl32(p - q) agrees with the exact real residual within 1e-6
    relative (north_star tolerance), on realistic heavy-tailed rows."""
    pool = synth.make_pool("f2", V=4096, k=4, dtype=dtype, n_buckets=4, variants=2, seed=9)
    P = pool.numpy()
    worst = 0.0
    for s in range(pool.S):
        for rid in range(16):
            _, o = oracle.verify_request(P["p"][s], P["q"][s], P["draft"][s], rid, 0, seed=3)
            assert o.invalid == 0
            worst = max(worst, o.z_rel_err)
    assert worst < 1e-6


def test_boundary_ambiguity_of_a_float_cdf_design():
    """PIN-X, second half: how many samples a floating-point CDF would
    leave within 1e-6 Z of a CDF boundary.  The sampled point t is uniform on [0, Z)
    given the rows, so the chance that it lies within eps Z of either edge of the
    emitted token's interval is 2 eps per token with mass, i.e. about 2 eps n_mass in
    total.  Measured on realistic rows (V = 4,096) it matches that law -- far above the
    north_star's 1e-5 at full vocabularies -- which is why the kernel's CDF is an exact
    integer one (identical tokens, zero ambiguous samples; AMB-27)."""
    pool = synth.make_pool("f2", V=4096, k=4, dtype="bf16", n_buckets=4, variants=2, seed=21)
    P = pool.numpy()
    eps, near, n, n_mass = 1e-5, 0, 0, []
    for s in range(pool.S):
        for rid in range(400):
            _, o = oracle.verify_request(P["p"][s], P["q"][s], P["draft"][s], rid, 7, seed=5)
            near += o.margin_rel < eps
            n += 1
        pr = P["p"][s].view(np.uint16).astype(np.uint32) << 16
        p32 = pr.view(np.float32)
        n_mass.append(float((p32[0] > 0).sum()))
    frac = near / n
    predicted = 2 * eps * float(np.mean(n_mass))   # upper-bound scale: every token with mass
    assert 0 < frac < 2 * predicted, (frac, predicted)


def test_sampling_uses_the_64bit_uniform_against_integer_cdf():
    """With two tokens of residual mass a and b, the emitted token is the first
    whose cumulative mass exceeds t = floor(U Z / 2^64): frequency a/(a+b)."""
    V, k = 8, 1
    p = np.zeros((2, V), np.float32)
    q = np.zeros((1, V), np.float32)
    q[0, 0] = 1.0
    p[0, 3] = 0.25
    p[0, 6] = 0.75
    p[1, 0] = 1.0
    n = 100_000
    tok, r = trials(p, q, np.array([0], np.int32), n)
    assert (r == 0).all()
    f = (tok[:, 0] == 3).mean()
    assert abs(f - 0.25) < 5 * np.sqrt(0.25 * 0.75 / n)
    assert set(np.unique(tok[:, 0])) == {3, 6}
