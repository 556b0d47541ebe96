"""SURVEY 8(f) f3 (Fig. 7 analogue): the accuracy of the execution-time
estimate T~ (Eq. 6) against the service a request actually receives in the
token-level simulation -- pinned against closed forms, not against the oracle itself.

Clairvoyant case ("information about both the request length and the acceptance
rate"): F1 mixture rows with per-position acceptance beta = 0.5 exactly (PIN-S: p(x) /
q(x) = beta on the draft support), so the accepted count per round is the truncated
geometric law of PIN-C2 and the measured acceptance rate A (AMB-4: accepted drafts /
proposed drafts) has expectation alpha* = beta (1 - beta^k) / (k (1 - beta)).  Every request
is made perceptible at arrival with A = alpha* and L_pred = L_true.  Eq. 6's denominator
k A + 1 is then exactly the expected tokens per round (1 - beta^(k+1)) / (1 - beta)
(leviathan2023fast, cited at P:11; 1.9375 at beta = 0.5, k = 4), so by the renewal
theorem the realised service E_i = rounds x c_round satisfies E[E_i] / T~_i -> 1 as
L grows (overshoot O(1) rounds).  A dropped "+1", a T_SSM / T_LLM swap (AMB-9) or a
per-round cost that is not the service increment would each move the ratio by far more
than the tolerance.
"""
import numpy as np

import oracle
import synth

MS = 1000


def _run(n, L, k, beta_pool, B, seed):
    pool = synth.make_pool("f1", V=16, k=k, dtype="f32", n_buckets=1, variants=32, seed=seed)
    tr = synth.make_trace(n, seed, arrival="zero", length="uniform", len_min=L, len_max=L)
    tab = synth.slab_table(tr, 1, 32, R=16, seed=seed)
    P = pool.numpy()
    P["slab_tab"], P["R"] = tab, 16
    cfg = oracle.SchedConfig(k=k, t_ssm_us=1 * MS, t_llm_us=10 * MS, seed=seed, s1_up_us=56 * MS)
    sim = oracle.Sim(cfg, tr.arrival_us, np.full(n, L), np.full(n, L))
    alpha_star = beta_pool * (1 - beta_pool ** k) / (k * (1 - beta_pool))
    for i in range(n):
        sim.make_perceptible(i, alpha_star)
    sel, _ = sim.select(B)
    while not sim.state()["done"].all():
        sim.step(P, sel)
    return sim.state(), alpha_star


def test_eq6_unbiased_against_the_token_level_simulation():
    k, L, n = 4, 1500, 96
    st, a = _run(n, L, k, 0.5, 16, 0xF3)
    assert abs(k * a + 1 - 1.9375) < 1e-12                       # (1 - b^5) / (1 - b), b = 1/2
    T = st["T_total_us"].astype(np.float64)
    assert (T == np.floor(L * (k * 1 * MS + 10 * MS) / 1.9375)).all()   # Eq. 6 hand value
    E = st["E_us"].astype(np.float64)
    ratio = E / T
    # renewal theorem: E[rounds] = L / mu + O(1); per-request sd ~ sqrt(L var / mu^3) / (L / mu)
    assert abs(ratio.mean() - 1.0) < 0.01, ratio.mean()
    mape = np.abs(E - T).mean() / T.mean()
    assert mape < 0.05, mape
    # every round charged exactly one round of service
    assert (st["E_us"] == st["rounds"] * (k * 1 * MS + 10 * MS)).all()


def test_estimate_error_grows_when_the_rate_is_wrong():
    """The same runs with A perturbed by +-20 %: the mean ratio moves by the predicted
    factor (k A + 1) / (k A' + 1) -- the estimator's sensitivity, a closed form."""
    k, L, n = 4, 800, 48
    st, a = _run(n, L, k, 0.5, 16, 0xF4)
    T = st["T_total_us"].astype(np.float64)
    E = st["E_us"].astype(np.float64)
    for f in (0.8, 1.2):
        T_wrong = np.floor(L * (k * 1 * MS + 10 * MS) / (k * a * f + 1))
        want = (k * a * f + 1) / (k * a + 1)
        assert abs((E / T_wrong).mean() - want) < 0.02
