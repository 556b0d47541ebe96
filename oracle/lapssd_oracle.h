/*
 * lapssd_oracle.h -- CPU ORACLE for the LAPS-SD batched speculative-decoding step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA product path (paper_2505_17074_b200/csrc,
 * include/lapssd.h); both are written independently from PAPER.md (arXiv 2505.17074)
 * and the readings listed in DESIGN.md section 3.
 *
 * Citations: P:NN = PAPER.md line NN.  AMB-n = DESIGN.md reading n.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"):
 *   orc_philox4x32_10 ...... Random123 known-answer vectors (tests/golden/philox_kat.txt)
 *   orc_verify_request ..... closed form E[tokens/step] (Leviathan et al., cited P:11),
 *                            accepted-count law, chi-square "first token ~ p" on V=16,
 *                            special cases p=q / disjoint / one-hot / mixture family
 *   orc_thresholds ......... P:169 formula hand values
 *   orc_eq6 ................ P:196-200 hand values
 *   orc_sim_* .............. Fig. 1 clairvoyant run (R3,R1,R2 / 450 ms) and FCFS /
 *                            LP-SJF (583 / 683 ms) through the token-level simulation,
 *                            perceptible-first + SJF on T~_rem, placement,
 *                            switching-cost hand values,
 *                            Fig. 1 token-level expectations (renewal DP),
 *                            stability deadline (P:194 + 1/t bound), degeneracies,
 *                            invariants
 *   orc_jobs_schedule ...... Fig. 1 printed averages 583 / 683 ms,
 *                            brute-force optimum (orc_brute_force)
 *   orc_brute_force ........ exhaustive enumeration (definition of the optimum)
 */
#ifndef LAPSSD_ORACLE_H
#define LAPSSD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- counter-based RNG: Philox4x32-10 (Salmon et al., SC'11) ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- (1) verification by rejection sampling, P:57-64, P:200 ---- */
enum { ORC_F32 = 0, ORC_BF16 = 1 };

typedef struct {
    int32_t  r;            /* first rejected position, or k if all accepted        */
    int32_t  y;            /* token emitted at position r                          */
    int32_t  fallback;     /* 1: residual mass was 0, sampled from p_r (AMB-20)     */
    int32_t  invalid;      /* 1: no mass at all (contract violation)                */
    uint64_t Z;            /* Q4.60 total residual mass                            */
    uint64_t t;            /* sampled target in [0, Z)                             */
    double   z_real;       /* exact residual mass sum(max(0,p-q)) in long double   */
    double   z_rel_err;    /* |Z*2^-60 - z_real| / z_real                          */
    double   margin_rel;   /* distance of t to nearest CDF boundary / Z            */
} orc_verify_out;

/* p_rows: (k+1) rows of V values; q_rows: k rows of V values; both in `dtype`
 * (bf16 stored as uint16 bit patterns).  draft: k token ids.
 * tokens: k+1 outputs (draft[0..r-1], y, then -1).  Returns r. */
int32_t orc_verify_request(const void *p_rows, const void *q_rows, int32_t dtype,
                           int64_t V, int32_t k, const int32_t *draft,
                           uint32_t req_id, uint32_t round_idx, uint64_t seed,
                           uint32_t trace, int32_t *tokens, orc_verify_out *out);

/* Many independent trials over the same rows (statistical pins). */
void orc_verify_many(const void *p_rows, const void *q_rows, int32_t dtype, int64_t V,
                     int32_t k, int32_t n_trials, const int32_t *drafts,
                     const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                     int32_t *tokens_out, int32_t *r_out);

/* ---- (1b) verification from logits ---- */
typedef struct {
    int32_t  r, y, fallback, pad;
    uint64_t Z_lo, Z_hi;   /* integer residual mass (times Sp Sq when r < k)        */
    uint64_t Sp, Sq;       /* integer softmax masses of the rows at position r      */
} orc_logits_out;

/* e^d on [-28, 0] by a fixed fp32 operation sequence (0 below -28). */
float orc_exp_hat(float d);

/* The quantised softmax of one row: E[v] = floor(exphat(fl32(z[v] - m)) 2^40) into E_out
 * (nullable), returns S = sum E, m_out = the row max. */
uint64_t orc_logits_row(const void *z_row, int32_t dtype, int64_t V, float *m_out, uint64_t *E_out);

/* zp_rows: (k+1) rows of V logits; zq_rows: k rows; dtype as above.  Returns r. */
int32_t orc_verify_logits_request(const void *zp_rows, const void *zq_rows, int32_t dtype,
                                  int64_t V, int32_t k, const int32_t *draft,
                                  uint32_t req_id, uint32_t round_idx, uint64_t seed,
                                  uint32_t trace, int32_t *tokens, orc_logits_out *out);
void orc_verify_logits_many(const void *zp_rows, const void *zq_rows, int32_t dtype, int64_t V,
                            int32_t k, int32_t n_trials, const int32_t *drafts,
                            const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                            int32_t *tokens_out, int32_t *r_out);
void orc_verify_logits_batch(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                             int32_t B, const int32_t *slab, const int32_t *drafts,
                             const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                             int32_t *tokens_out, int32_t *r_out, uint64_t *z_out);

/* ---- (1c) SURVEY 8(f) f4: the steps on either side of verification (AMB-34, AMB-35) ---- */
/* Drafting-side sampling ("the draft model autoregressively generates the
 * subsequent L tokens"): one token from the stored row q (V values, `dtype`) by the exact
 * integer inverse CDF R_v = floor(q[v] 2^60), Z = sum R, U = Philox(req, round,
 * (2 << 16) | pos, trace) lanes 0-1, t = floor(U Z / 2^64), x = min{v : sum_{w<=v} R_w > t}.
 * Returns x (0 if Z = 0, *invalid set); *Z_out = Z. */
int32_t orc_draft_sample(const void *q_row, int32_t dtype, int64_t V, uint32_t req_id,
                         uint32_t round_idx, uint32_t pos, uint64_t seed, uint32_t trace,
                         uint64_t *Z_out, int32_t *invalid);

/* Token-tree verification by multi-step speculative sampling (SpecInfer, cited at P:322;
 * P:59-64 per step).  Node 0 is the root; parent[c] < c for every used node c >= 1
 * (parent[c] < 0: unused); token[c] the draft token of node c; children of u are the used
 * nodes with parent u, in index order.  p_rows / q_rows hold n_nodes rows of V: p_u the
 * target distribution after the prefix ending at u, q_u the draft distribution its
 * children were drawn from.  At node u (depth d) with children c_1..c_w:
 *   stage 0: accept c_1 iff u24 q_u(x) < p_u(x) 2^24 (fp64, exact), u24 from Philox
 *            (req, round, d / 4, trace) lane d % 4 -- the linear verification's rule;
 *   rejecting c_i gives the residual D_i: D_1 = floor(max(0, fl32(p_u - q_u)) 2^60),
 *            D_{i+1} = floor(max(0, D_i 2^60 - Z_i floor(q_u 2^60)) / 2^b(Z_i)), Z_i = sum D_i,
 *            b(Z) the bit length of Z (the normalised residual, scaled; exact integers);
 *   stage i >= 1: accept c_{i+1} iff u24 q_u(x) Z_i < D_i(x) 2^24 (exact integers), u24
 *            from Philox(req, round, (3 << 16) | (u << 8) | ((i-1) / 4), trace) lane (i-1) % 4;
 *   accepted child: emit its token, continue at it; all rejected: emit y ~ D_w; a leaf:
 *   emit the bonus y ~ floor(p_u 2^60); Z_i = 0 after a rejection: y ~ floor(p_u 2^60)
 *   (*fallback, AMB-20).  y by the inverse CDF with U = Philox(req, round, 1 << 8, trace).
 * A chain (one child per node) is exactly orc_verify_request.  tokens[n_nodes]: accepted
 * tokens, y, then -1; path[n_nodes]: accepted nodes then -1.  Returns the accepted count,
 * -1 for a malformed tree (parent >= child, a token outside [0, V)). */
typedef struct {
    int32_t  n_accept, y, final_node, n_rejected, fallback, invalid;
    uint64_t Z;            /* mass of the final draw's row                          */
} orc_tree_out;
int32_t orc_verify_tree(const void *p_rows, const void *q_rows, int32_t dtype, int64_t V,
                        int32_t n_nodes, const int32_t *parent, const int32_t *token,
                        uint32_t req_id, uint32_t round_idx, uint64_t seed, uint32_t trace,
                        int32_t *tokens, int32_t *path, orc_tree_out *out);

/* ---- scheduler pieces, P:161-202 ---- */
enum { ORC_POL_LAPSSD = 0, ORC_POL_FCFS = 1, ORC_POL_LPSJF = 2, ORC_POL_LAS = 3 };
enum { ORC_PLACE_BY_ESTIMATE = 0, ORC_PLACE_STAY = 1 };
enum { ORC_PIN_ON_SELECT = 0, ORC_PIN_ON_STABLE = 1 };
enum { ORC_COST_EQ6 = 0, ORC_COST_FIG1 = 1 };

typedef struct {
    int32_t  policy;
    int32_t  K;            /* number of priority queues, 1..16                      */
    int64_t  s1_up_us;     /* S_1^up                                                */
    double   M;            /* threshold ratio, > 1                                  */
    int32_t  gamma;        /* stability window (rounds), >= 2                       */
    double   delta;        /* stability threshold, >= 0                             */
    int32_t  k;            /* drafts per round (paper's n)                          */
    int64_t  t_ssm_us;     /* T_SSM per drafted token                               */
    int64_t  t_llm_us;     /* T_LLM per verification pass                           */
    int32_t  placement;    /* ORC_PLACE_*                                           */
    int32_t  pin_rule;     /* ORC_PIN_*                                             */
    uint64_t seed;
    int32_t  cost_model;   /* ORC_COST_EQ6: round = k T_SSM + T_LLM, T~ = Eq. 6;
                              ORC_COST_FIG1: round = k t_tok, T~ = L t_tok / A */
    int64_t  t_tok_us;     /* Fig. 1 verification time per candidate token          */
    int64_t  switch_c0_us; /* switch-in cost c0 + c1 (prompt + tokens) (AMB-24)      */
    int64_t  switch_c1_us;
} orc_config;

/* S_up[j] = floor(s1_up * M^j), j = 0..K-2, iterative fp64 multiply. */
int32_t  orc_thresholds(int32_t K, int64_t s1_up_us, double M, int64_t *S_up_out);
/* Eq. (6): floor(L (k T_SSM + T_LLM) / (k A + 1)) in microseconds. */
uint64_t orc_eq6(int64_t L, double A, int32_t k, int64_t t_ssm_us, int64_t t_llm_us);
/* Fig. 1 model: floor(L t_tok / A) microseconds (UINT64_MAX if A = 0). */
uint64_t orc_fig1_est(int64_t L, double A, int64_t t_tok_us);

/* ---- the resident-request simulation (a3-a8) ---- */
typedef struct orc_sim orc_sim;

/* prompt: prompt lengths (switching cost, AMB-24), nullable = 0. */
orc_sim *orc_sim_create(const orc_config *cfg, int32_t n_local, const int64_t *arrival_us,
                        const int32_t *L_true, const int32_t *L_pred, const int32_t *prompt,
                        int32_t rank, int32_t world);
void     orc_sim_destroy(orc_sim *s);
/* Monte-Carlo traces: Philox counter word c3 (AMB-21). */
void     orc_sim_set_trace(orc_sim *s, uint32_t trace);
/* TEST HOOK (Fig. 1(c) clairvoyant case): request i becomes perceptible with rate A
 * through the update's own Stabilized event (estimate, placement, pin rule). */
int32_t  orc_sim_make_perceptible(orc_sim *s, int32_t i, double A);

/* Single-rank select: advance clock, admit, build keys, take top-B.  Returns count;
 * sel_out[B] holds local indices in key order, -1 padded. */
int32_t  orc_sim_select(orc_sim *s, int32_t B, int32_t *sel_out);
/* Multi-rank select, phase 1: advance clock, admit, build keys, write this rank's
 * C smallest eligible keys (ascending, UINT64_MAX padded), each one's switch-in cost
 * if it is selected (switch_out, nullable) and its next arrival. */
void     orc_sim_candidates(orc_sim *s, int32_t C, uint64_t *keys_out, int64_t *switch_out,
                            int64_t *next_arrival_out);
/* Multi-rank select, phase 2: given the gathered candidates of all ranks
 * (world*C keys, their switch-in costs (nullable), world next arrivals), take the
 * global top-B, keep own ids, advance the clock by the global batch's step. */
int32_t  orc_sim_merge(orc_sim *s, const uint64_t *all_keys, const int64_t *all_switch, int32_t C,
                       const int64_t *all_next_arrival, int32_t B, int32_t *sel_out,
                       int32_t *global_count_out);

/* State update after verification (a3): sel[B] local indices (-1 = empty slot),
 * n_accept[B] = r per slot. */
void     orc_sim_update(orc_sim *s, const int32_t *sel, const int32_t *n_accept, int32_t B);

/* One full step over pooled rows: verify every selected request on its slab,
 * update, select the next batch.  slab_tab[n_local*R] maps (request, round) to a
 * slab: idx = round < R ? round : R/2 + (round - R/2) % (R/2).
 * tokens_out[B*(k+1)] and n_accept_out[B] may be NULL. */
int32_t  orc_sim_step(orc_sim *s, const void *p_pool, const void *q_pool,
                      const int32_t *draft_pool, int32_t dtype, int64_t V,
                      const int32_t *slab_tab, int32_t R, int32_t B, int32_t *sel_inout,
                      int32_t *tokens_out, int32_t *n_accept_out, uint64_t *z_out);

typedef struct {
    int64_t now_us;
    int32_t cursor, prev_count;
    int32_t *acc_tok, *acc_draft, *rounds;
    int64_t *E_us, *T_total_us, *C_us, *x_us;
    uint8_t *admitted, *done, *perceptible, *pinned, *level, *running;
    double  *A;
    uint64_t *key;
    int32_t *ring;         /* n_local * gamma */
    int64_t *switch_us;    /* switching time charged on each request's entries (AMB-24) */
    uint8_t *in_batch;     /* in the batch that ran last */
    int64_t step_cost_us;  /* duration of the step that ran last */
    int64_t switch_total_us;
} orc_state_view;
void     orc_sim_view(orc_sim *s, orc_state_view *v);
/* keys exactly as the last select built them (ineligible ones included) */

/* ---- job-level scheduling with known service times (Fig. 1; Eqs. 2-5) ---- */
/* policy: 0 = SJF by est (LAPS-SD, every request perceptible at arrival), 1 = FCFS,
 * 2 = LP-SJF (by L_pred).  Non-preemptive single server.  Returns sum of (C_i - r_i). */
int64_t  orc_jobs_schedule(int32_t policy, int32_t n, const int64_t *arrival_us,
                           const int64_t *service_us, const int64_t *L_pred,
                           const int64_t *est_us, int32_t *order_out, int64_t *C_out);
/* Exhaustive search over all n! orders (n <= 8), simultaneous arrivals at 0.
 * Returns the minimum sum of completion times; best_order_out gets the
 * lexicographically smallest optimal order; all_sums_out (nullable) gets the
 * sum for every permutation in lexicographic order. */
int64_t  orc_brute_force(int32_t n, const int64_t *service_us, int32_t *best_order_out,
                         int64_t *all_sums_out);

#ifdef __cplusplus
}
#endif
#endif
