"""The oracle's pins must reject plausible misreadings of the paper (mutation check).

Each mutant is the oracle source with ONE rule changed, compiled to a scratch library and
loaded (LAPSSD_ORACLE_LIB) by a subprocess that runs the semi-clairvoyant and
switching-cost pin files; at least one pin must fail for every mutant:

  sjf_reversed      perceptible requests served longest-estimate first (P:202 says SJF)
  perc_last         non-perceptible requests ahead of perceptible ones ("always
                    prioritize scheduling perception requests")
  place_bottom      a stabilised request placed in the bottom queue ("moved to the
                    corresponding queue", AMB-14)
  sjf_on_total      SJF keyed on the total estimate instead of the remaining one (AMB-12)
  fig1_times_A      the Fig. 1 estimate L t_tok * A instead of L t_tok / A
  switch_always     switch-in cost charged to requests that ran in the previous step
  switch_in_E       switching time added to attained service E_i (AMB-24)
  no_semi           every request scheduled as non-perceptible with no estimate (the
                    round-1 advisor's mutation: nonperc = 1, secondary = 0)
  tree_no_renorm    f4 tree: the residual D_i not renormalised before q is subtracted
  tree_stage_p      f4 tree: later children tested against p instead of the residual
  tree_draw_p       f4 tree: after every child is rejected, the token drawn from p_u
  draft_same_u      f4 draft sampler: one uniform for every position (the counter drops pos)
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "lapssd_oracle.c")

MUTANTS = {
    "sjf_reversed": ("f.secondary = sat32(estimate(s, L_rem, s->A[i]));",
                     "f.secondary = 0xFFFFFFFFull - sat32(estimate(s, L_rem, s->A[i]));"),
    "perc_last": ("f.nonperc = !s->perceptible[i];", "f.nonperc = s->perceptible[i];"),
    "place_bottom": ("s->level[i] = (uint8_t)level_of(s->S_up, s->cfg.K, s->T_total[i]);",
                     "s->level[i] = (uint8_t)(s->cfg.K - 1);"),
    "sjf_on_total": ("int64_t L_rem = (int64_t)s->L_pred[i] - s->acc_tok[i];   /* AMB-12 */",
                     "int64_t L_rem = (int64_t)s->L_pred[i];"),
    "fig1_times_A": ("double T = num / A;", "double T = num * A;"),
    "switch_always": ("if (s->in_batch[i]) return 0;", "if (0) return 0;"),
    "switch_in_E": ("s->switch_us[i] += c;", "s->switch_us[i] += c; s->E[i] += c;"),
    "no_semi": [("f.nonperc = !s->perceptible[i];", "f.nonperc = 1;"),
                ("f.secondary = sat32(estimate(s, L_rem, s->A[i]));", "f.secondary = 0;")],
    "tree_no_renorm": ("u128 a = (u128)D << 60, b = (u128)c->Zs[s] * Q;", "u128 a = (u128)D << 60, b = (u128)Q << 60;"),
    "tree_stage_p": ("accept = tree_accept(u24, qx, tree_mass(&c, x), Zs[i]);",
                     "accept = (double)u24 * (double)qx < (double)load_prob(p_rows, dtype, off + x) * 16777216.0;"),
    "tree_draw_p": ("if (stage > 0 && !fallback) {", "if (0) {"),
    "draft_same_u": ("draw(seed, req_id, round_idx, 2u << 8, pos, trace, u4);",
                     "draw(seed, req_id, round_idx, 2u << 8, 0, trace, u4);"),
}

PIN_FILES = ["tests/test_oracle_semiclairvoyant.py", "tests/test_oracle_switch.py"]
F4_FILES = ["tests/test_oracle_f4.py"]


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pins_reject_mutant(name, tmp_path):
    edits = MUTANTS[name]
    edits = edits if isinstance(edits, list) else [edits]
    src = open(SRC).read()
    for old, new in edits:
        assert src.count(old) == 1, f"mutation site of {name} not found exactly once"
        src = src.replace(old, new)
    mut = tmp_path / "lapssd_oracle.c"
    mut.write_text(src)
    so = tmp_path / "libmut.so"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "oracle"), "-o", str(so), str(mut), "-lm"])
    env = dict(os.environ, LAPSSD_ORACLE_LIB=str(so))
    files = F4_FILES if name.startswith(("tree_", "draft_")) else PIN_FILES
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *files],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant {name} passed every pin:\n{r.stdout[-2000:]}"
    assert "failed" in r.stdout, r.stdout[-2000:]


def test_unmutated_oracle_passes_the_same_pins():
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *PIN_FILES],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]
