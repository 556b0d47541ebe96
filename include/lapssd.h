/*
 * lapssd.h -- C-ABI of liblapssd.so: the B200 (sm_100a) hot path of LAPS-SD
 * (arXiv 2505.17074), the per-iteration batched speculative-decoding step over
 * every resident request:
 *
 *   (a1-a2) spec_verify  -- verify k drafts per request by rejection sampling
 *                           (Eq. 1; bonus token P:200)
 *   (a3)    laps_update  -- the LAPS-SD per-request state update
 *                           (P:170-178 lifecycle, P:194 stability, Eq. 6)
 *   (a4-a7) laps_select  -- admission, priority keys, top-B batch, clock
 *                           (P:129-133 inter-queue, P:135-142 / P:202 intra-queue)
 *   laps_step            -- (a1..a7) fused: verify + update + select
 *   (a8)    laps_candidates / laps_merge / laps_step_dist -- request sharding over
 *                           G GPUs with one all-gather of candidate keys per step
 *
 * The scheduling problem the calls follow: requests i arrive at r_i,
 * their execution time is unknown in advance, the system chooses when each runs
 * (x_i) and whether it is preempted at round boundaries; the objective is the mean
 * of C_i - r_i.  "P:NN" is PAPER.md line NN; "AMB-n" is a reading in DESIGN.md s.3.
 *
 * Conventions for every call:
 *  - Pointers marked [device] are CUDA device pointers; [host] are host pointers.
 *    All device buffers are CALLER-OWNED (PyTorch tensors).  The library never
 *    allocates device memory and never frees caller memory.
 *  - Every call is asynchronous on the given stream, enqueues only kernels (no
 *    host synchronisation, no allocation) and may be captured in a CUDA graph,
 *    except lapssd_create (H2D copies of the request arrays), lapssd_read_state
 *    (D2H copies, synchronises the stream) and lapssd_check (synchronises).
 *  - Argument validation is synchronous: a bad argument returns LAPSSD_EINVAL and
 *    enqueues nothing.  A failed launch returns LAPSSD_ECUDA.  The text of the
 *    last error of the calling thread is returned by lapssd_last_error().
 *  - Contract violations detected on the device (e.g. a selected request that is
 *    already complete, a row with no probability mass) set a sticky device flag
 *    that lapssd_check() reports as LAPSSD_ESTATE.
 *  - A handle is bound to one stream at a time and is not thread-safe.
 *  - Times are integer microseconds (int64).  Probabilities are float32 or bf16
 *    in [0, 1]; each stored row of p is expected to sum to about 1 (a verified row pair
 *    whose residual mass exceeds 2 sets device flag 256, see lapssd_check; full
 *    validation: lapssd_set_row_check).
 */
#ifndef LAPSSD_H
#define LAPSSD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *lapssd_stream;   /* == cudaStream_t */

typedef enum {
    LAPSSD_OK = 0,
    LAPSSD_EINVAL = -1,   /* invalid argument, nothing enqueued                      */
    LAPSSD_ECUDA = -2,    /* CUDA launch / copy failure                              */
    LAPSSD_ENCCL = -3,    /* NCCL unavailable or failed                              */
    LAPSSD_ESTATE = -4,   /* device-detected contract violation (sticky flag)        */
    LAPSSD_ENOMEM = -5    /* caller-provided workspace too small                     */
} lapssd_status;

typedef enum { LAPSSD_F32 = 0, LAPSSD_BF16 = 1 } lapssd_dtype;

typedef enum {
    LAPSSD_POL_LAPSSD = 0,  /* Alg. 1                                       */
    LAPSSD_POL_FCFS = 1,    /* first-come-first-serve, non-preemptive            */
    LAPSSD_POL_LPSJF = 2,   /* SJF on predicted output length, non-preemptive   */
    LAPSSD_POL_LAS = 3      /* least attained service on the same K queues      */
} lapssd_policy;

/* Scheduler parameters.  Validation (EINVAL):
 * 1 <= K <= 16, s1_up_us > 0, M > 1, 2 <= gamma <= 32, delta >= 0, 1 <= k <= 16,
 * t_ssm_us >= 0, t_llm_us >= 0, cost_model in {0, 1}, t_tok_us >= 0, switch_c0_us >= 0,
 * switch_c1_us >= 0.  delta == 0 disables stabilisation.
 *
 * Cost model (DESIGN.md AMB-3, AMB-31): LAPSSD_COST_EQ6 -- one round is k*T_SSM + T_LLM of
 * service and T~(L, A) = floor(L (k T_SSM + T_LLM) / (k A + 1)) (Eq. 6);
 * LAPSSD_COST_FIG1 -- the Fig. 1 model: a round verifies k candidates at t_tok
 * each (k*t_tok of service) and T~(L, A) = floor(L t_tok / A) (A = 0: unbounded).
 *
 * Switching cost (DESIGN.md AMB-24): a request that enters the
 * batch without having been in the batch that ran last pays c0 + c1 (prompt + generated
 * tokens) of SYSTEM time: the step lasts one round plus the switch-ins of its batch
 * (the clock and C_i advance by it), while attained service E_i is not charged. */
typedef struct {
    int32_t policy;        /* lapssd_policy                                            */
    int32_t K;             /* number of priority queues Q_1..Q_K                       */
    int64_t s1_up_us;      /* S_1^up; S_j^up = floor(s1_up * M^(j-1)) (AMB-11)  */
    double M;              /* threshold ratio                                          */
    int32_t gamma;         /* stability window in rounds (AMB-7)                */
    double delta;          /* stability threshold on max-min of the window (AMB-6)     */
    int32_t k;             /* drafts per round, the paper's n                  */
    int64_t t_ssm_us;      /* T_SSM per drafted token (Eq. 6, AMB-9)                   */
    int64_t t_llm_us;      /* T_LLM per verification pass (Eq. 6)                      */
    int32_t placement;     /* 0 = queue of T~_total on stabilisation, 1 = stay (AMB-14) */
    int32_t pin_rule;      /* 0 = pin perceptible requests when selected, 1 = when
                              stable (AMB-15)                                          */
    uint64_t seed;         /* Philox key for every draw of the method (AMB-21)         */
    int32_t cost_model;    /* LAPSSD_COST_EQ6 (default) or LAPSSD_COST_FIG1            */
    int64_t t_tok_us;      /* FIG1: verification time per candidate token              */
    int64_t switch_c0_us;  /* switch-in cost c0 + c1 (prompt + tokens), default 0      */
    int64_t switch_c1_us;
} lapssd_config;

enum { LAPSSD_COST_EQ6 = 0, LAPSSD_COST_FIG1 = 1 };

/* The resident requests of this rank.  [host] arrays of n entries, copied at
 * create.  Local request l has global id l*world + rank; arrival_us must be
 * non-decreasing in l (ids encode arrival order, AMB-19).  L_true >= 1 is the
 * output length that ends the request, L_pred >= 1 the predicted length L_i
 * used by Eq. 6 and LP-SJF.  prompt >= 0 is the prompt length the switching
 * cost charges (nullable: all 0).  Global ids must be < 2^24 - 1 (the all-ones key
 * stays unused). */
typedef struct {
    const int64_t *arrival_us;
    const int32_t *L_true;
    const int32_t *L_pred;
    int32_t n;
    int32_t rank, world;
    const int32_t *prompt;
} lapssd_requests;

/* Where a step's probability rows live.  Two layouts:
 *  - slab_tab == NULL: batch layout.  Slot b (0 <= b < B) reads
 *      p[b, 0..k, 0..V), q[b, 0..k-1, 0..V), draft[b, 0..k-1].
 *  - slab_tab != NULL: pooled layout.  p/q/draft are pools of n_slabs slabs of the
 *      same shapes; the request in slot b, local index i, in its round t reads slab
 *      slab_tab[i*R + (t < R ? t : R/2 + (t - R/2) % (R/2))].
 * p: [device] (k+1) x V per slab, q: [device] k x V per slab, row-major, dtype
 * elements; draft: [device] int32 k per slab, drafts x_j sampled from q_j.  p, q and
 * draft may also be pinned host memory (cudaHostAlloc / registered, unified addressing):
 * the kernels then read in place, over PCIe, only the bytes the step needs.
 * With the batch layout the acceptance tests always use the rows of the call itself.
 * V*sizeof(dtype) must be a multiple of 16 and p, q 16-byte aligned. */
typedef struct {
    const void *p;
    const void *q;
    const int32_t *draft;
    int32_t dtype;         /* lapssd_dtype                                             */
    int32_t k;
    int64_t V;
    const int32_t *slab_tab;  /* [device] n_local x R, or NULL                         */
    int32_t R;
    int64_t n_slabs;
} lapssd_rows;

typedef struct lapssd_handle lapssd_handle;

/* ---------------------------------------------------------------------------
 * spec_verify -- stateless batched verification (AMB-1,2,20,21,27)
 *
 * For every slot b < B (rows as in lapssd_rows with slab_tab == NULL, or slab
 * index slab[b] into pools when slab != NULL):
 *   for j = 0..k-1: u24_j = Philox4x32-10(key = seed, ctr = (req_id[b], round_idx[b],
 *     j/4, trace))[j%4] >> 8; accept x_j iff u24_j * q_j(x_j) < p_j(x_j) * 2^24 (fp64,
 *     exact); r = first rejected position, or k.
 *   R_v = floor(max(0, fl32(p_r[v] - q_r[v])) * 2^60) if r < k, else floor(p_k[v]*2^60);
 *   if r < k and sum R = 0 the row p_r is used (AMB-20).  Z = sum_v R_v (exact uint64).
 *   U = 64-bit Philox draw (ctr = (req_id, round, 1<<8, trace)), t = floor(U*Z/2^64),
 *   y = min{ v : sum_{w<=v} R_w > t }.
 * Outputs [device]: tokens[B, k+1] = (x_0..x_{r-1}, y, -1...), n_accept[B] = r,
 * z_fixed[B] = Z (nullable).  req_id, round_idx: [device] uint32 [B].
 * workspace: [device] >= spec_verify_workspace_bytes(B, V), ZERO-FILLED once by the
 * caller before first use; every call leaves it zero-filled again, so the same
 * workspace can be reused without re-zeroing (one call at a time per workspace).
 * Errors: EINVAL (k, V, dtype, alignment, B < 0), ENOMEM (workspace), ECUDA. */
size_t spec_verify_workspace_bytes(int32_t B, int64_t V);
lapssd_status spec_verify(const void *p, const void *q, int32_t dtype, int64_t V, int32_t k,
                          const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                          const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                          int32_t *tokens, int32_t *n_accept, uint64_t *z_fixed,
                          void *workspace, size_t workspace_bytes, lapssd_stream stream);

/* ---------------------------------------------------------------------------
 * spec_verify_logits -- stateless batched verification from LOGITS (
 * P:57-64 Eq. 1 and P:200 with p = softmax of the target head's logits and q = softmax
 * of the draft head's; DESIGN.md AMB-30).
 *
 * zp: [device] pool of (k+1) x V target logits per slab, zq: k x V draft logits per
 * slab, dtype elements (bf16 or fp32), row-major, V*sizeof(dtype) a multiple of 16,
 * 16-byte aligned, V <= 2^23; draft: [device] int32 k per slab; slab: [device] int32
 * [B] slab of slot b (NULL: slot b reads slab b); req_id, round_idx: [device] [B].
 * For every row j of slot b the softmax is quantised exactly:
 *   m = max_v z[v];  E[v] = floor(exphat(fl32(z[v] - m)) * 2^40);  S = sum_v E[v];
 *   exphat(d) = 0 for d < -28, else 2^n * P7(r), n = rint(fl32(d * log2e)),
 *   r = fma(-n, ln2_lo, fma(-n, ln2_hi, d)), P7 = degree-7 Taylor in Horner form with
 *   fma (constants as fp32 hex literals in AMB-30): every operation IEEE fp32 RN.
 * a1: accept x_j iff u24_j * Eq_j(x_j) * Sp_j < 2^24 * Ep_j(x_j) * Sq_j (128-bit
 *   integers; u24_j as in spec_verify); r = first rejection or k.
 * a2: R_v = max(0, Ep_r[v] * Sq_r - Eq_r[v] * Sp_r) if r < k (the residual
 *   max(0, p^ - q^) times Sp Sq), else Ep_k[v]; if r < k and sum R = 0, R_v = Ep_r[v]
 *   (AMB-20).  Z = sum_v R_v (< 2^120), U as in spec_verify,
 *   t = U * (Z >> 64) + floor(U * (Z mod 2^64) / 2^64), y = min{v : sum_{w<=v} R_w > t}.
 * Outputs [device]: tokens[B, k+1] (x_0..x_{r-1}, y, -1...), n_accept[B] = r,
 * z[B, 2] = (Z mod 2^64, Z >> 64) (nullable).
 * Only the rows the tests consult are normalised (pair j only if x_0..x_{j-1} were all
 * accepted, p_k only if all k were): one launch over a persistent grid with a work queue
 * (the results do not depend on it; LAPSSD_LOGITS_EAGER=1 normalises every row instead).
 * workspace: [device] >= spec_verify_logits_workspace_bytes(B, k, V, dtype) bytes, any
 * content (one call at a time per workspace).
 * Errors: EINVAL (k, V, dtype, alignment, B < 0, NULL), ENOMEM (workspace), ECUDA. */
size_t spec_verify_logits_workspace_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype);
lapssd_status spec_verify_logits(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                                 const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                                 const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                                 int32_t *tokens, int32_t *n_accept, uint64_t *z, void *workspace,
                                 size_t workspace_bytes, lapssd_stream stream);

/* ---------------------------------------------------------------------------
 * spec_draft_sample -- drafting-side sampling ("the draft model
 * autoregressively generates the subsequent L tokens"; DESIGN.md AMB-34).  For each of
 * R rows (row r = q + (row ? row[r] : r) * V elements, dtype bf16 / fp32, 16-byte aligned,
 * V*sizeof(dtype) a multiple of 16, V <= 524288):
 *   R_v = floor(q[v] 2^60) (exact), Z = sum_v R_v (uint64), U = Philox4x32-10(key = seed,
 *   ctr = (req_id[r], round_idx[r], (2 << 16) | pos[r], trace)) lanes 0-1 as a 64-bit word,
 *   t = floor(U Z / 2^64), draft_out[r] = min{v : sum_{w<=v} R_w > t}  (0 if Z = 0).
 * pos[r] < 65536 is the draft position (one call per autoregressive step with pos = j,
 * or all positions at once).  Outputs [device]: draft_out[R], z_out[R] (nullable).
 * HBM: one read of each row.  Errors: EINVAL (dtype, V, alignment, R < 0, NULL), ECUDA. */
lapssd_status spec_draft_sample(const void *q, int32_t dtype, int64_t V, const int32_t *row,
                                const uint32_t *req_id, const uint32_t *round_idx, const uint32_t *pos,
                                int32_t R, uint64_t seed, uint32_t trace, int32_t *draft_out,
                                uint64_t *z_out, lapssd_stream stream);

/* ---------------------------------------------------------------------------
 * spec_verify_tree -- token-tree verification by multi-step speculative sampling
 * (SpecInfer, cited at P:322; each step the rule of P:59-64; DESIGN.md
 * AMB-35).  Request b owns a tree of n_nodes (1..64) nodes: node 0 is the root, node
 * c >= 1 is used iff parent[b, c] >= 0, with parent[b, c] < c and token[b, c] in [0, V)
 * its draft token; the children of a node are its used children in index order.
 * p, q: [device] [B, n_nodes, V] rows: p[b, u] the target distribution after the prefix
 * ending at node u, q[b, u] the draft distribution u's children were drawn from.
 * At node u (depth d) with children c_1..c_w:
 *   c_1 is accepted iff u24 q_u(x) < p_u(x) 2^24 (fp64, exact), u24 = Philox(req, round,
 *     d / 4, trace)[d % 4] >> 8 -- exactly spec_verify's test at position d;
 *   rejecting c_i leaves the residual D_i: D_1 = floor(max(0, fl32(p_u - q_u)) 2^60),
 *     D_{i+1} = floor(max(0, D_i 2^60 - Z_i floor(q_u 2^60)) / 2^b(Z_i)), Z_i = sum_v D_i,
 *     b(Z) the bit length of Z (the residual of the normalised D_i, scaled, in exact
 *     128-bit integers: every entry stays below 2^60);
 *   c_{i+1} (i >= 1) is accepted iff u24 q_u(x) Z_i < D_i(x) 2^24 (exact integers),
 *     u24 = Philox(req, round, (3 << 16) | (u << 8) | ((i-1) / 4), trace)[(i-1) % 4] >> 8;
 *   the first accepted child's token is emitted and its subtree continues; if every child
 *   is rejected the token is drawn from D_w, at a leaf the bonus token from floor(p_u 2^60),
 *   and if some Z_i = 0 from floor(p_u 2^60) (AMB-20); draws: U = Philox(req, round,
 *   1 << 8, trace), t = floor(U Z / 2^64), y = min{v : sum_{w<=v} mass_w > t}.
 * A chain (one child per node) gives exactly spec_verify's result.
 * Outputs [device]: tokens[B, n_nodes] (accepted tokens, the drawn token, then -1),
 * path[B, n_nodes] (accepted node indices then -1, nullable), n_accept[B] (-1: malformed
 * tree, nothing else written), z_out[B] (mass of the final draw's row, nullable).
 * HBM per request: the gathered scalars, one pass over (p_u, q_u) per rejected child,
 * one over p_u at a leaf.  Errors: EINVAL (dtype, V, n_nodes, alignment, B < 0, NULL),
 * ECUDA. */
lapssd_status spec_verify_tree(const void *p, const void *q, int32_t dtype, int64_t V, int32_t n_nodes,
                               const int32_t *parent, const int32_t *token, const uint32_t *req_id,
                               const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                               int32_t *tokens, int32_t *path, int32_t *n_accept, uint64_t *z_out,
                               lapssd_stream stream);

/* ---------------------------------------------------------------------------
 * Handle: resident-request state (SoA, ~64 B/request + gamma*4 B ring) in a
 * caller-owned device workspace.  lapssd_create copies the request arrays (H2D on
 * `stream`), zero-initialises state, computes the thresholds of P:169, and sets
 * now = 0.  The first batch comes from laps_select.  max_batch bounds B of every
 * later call; V bounds the rows' vocabulary.
 * Errors: EINVAL (config, n, ids >= 2^24 - 1, max_batch < 1), ENOMEM, ECUDA. */
size_t lapssd_workspace_bytes(const lapssd_config *cfg, int32_t n_local, int32_t max_batch,
                              int64_t V, int32_t world);
lapssd_status lapssd_create(const lapssd_config *cfg, const lapssd_requests *req,
                            int32_t max_batch, int64_t V, void *workspace,
                            size_t workspace_bytes, lapssd_stream stream, lapssd_handle **out);
lapssd_status lapssd_destroy(lapssd_handle *h);

/* laps_update -- (a3) state update of the B verified slots:
 * tokens += min(r+1, L_true - tokens) (AMB-18); accepted drafts += r; rounds += 1;
 * E_i += one round's service (cost model above); ring of cumulative accepted
 * drafts; if the request is non-perceptible and the cumulative acceptance rates
 * a_s/(k s) of the last gamma rounds span < delta: A_i = their mean,
 * perceptible, T~_i = the estimate at L_pred (Eq. 6 or Fig. 1 model), placement
 * (AMB-14); otherwise demotion to the queue of E_i; completion when
 * tokens >= L_true with C_i = now + the step's duration (round + switch-ins).
 * sel: [device] int32 [B] local indices (-1 = empty slot); n_accept: [device] [B].
 * Errors: EINVAL, ECUDA; updating a complete request sets the ESTATE flag. */
lapssd_status laps_update(lapssd_handle *h, const int32_t *sel, const int32_t *n_accept,
                          int32_t B, lapssd_stream stream);

/* laps_select -- (a4-a7): if the previous batch was non-empty, now += its step's
 * duration (one round + the switch-ins it paid, AMB-17, AMB-24); admit every request
 * with arrival <= now; build every resident request's 64-bit priority key
 * (smaller = sooner; AMB-15/16/19):
 *   [63] ineligible | [62] not pinned | [61:58] queue level | [57] non-perceptible |
 *   [56] not running (non-perceptible) | [55:24] T~_rem us saturated (perceptible) or
 *   policy secondary | [23:0] global id
 * and write the B smallest eligible keys' local indices in ascending key order to
 * sel_out [device int32 B] (-1 padded), their count to count_out [device int32,
 * nullable].  Selected requests get x_i = now on first selection and are pinned per
 * pin_rule; those not in the previous batch pay their switch-in cost (AMB-24).  If
 * nothing is eligible, now jumps to the next arrival.
 * Errors: EINVAL (B > max_batch), ECUDA. */
lapssd_status laps_select(lapssd_handle *h, int32_t B, int32_t *sel_out, int32_t *count_out,
                          lapssd_stream stream);

/* laps_step -- one fused step: spec_verify on the current batch sel_inout[B]
 * (from the previous laps_select/laps_step), laps_update of every verified request,
 * then laps_select into sel_inout -- with the results of that exact sequence.
 * Execution (DESIGN.md s.6): the state update depends on r only (known from a1 before
 * any row streams), so the verify kernel's finisher warps run it at kernel start and
 * publish each request's new key; with pooled rows a select kernel on a library-owned
 * side stream (forked from / joined back into `stream` with events, highest launch
 * priority) presorts the other requests, merges the published keys while the rows
 * stream, and commits the next batch once every verify CTA has snapshotted the current
 * one.  Everything is ordered on `stream` when the call's work completes, and the call
 * may be captured in a CUDA graph.  By default the verify kernel starts after all prior
 * work on `stream` (plain stream order).  After lapssd_set_step_overlap(h, 1) a pooled-
 * rows laps_step's verify launch is a programmatic dependent of what precedes it on the
 * stream (the previous laps_step's select): it may start -- and read rows, drafts and
 * the slab table -- before that work completes.  The caller then guarantees that no
 * work it enqueues between consecutive laps_step calls on the stream writes anything the
 * step reads (e.g. a static slab pool); rows produced by a kernel on the same stream need
 * the default.  rows: pooled or batch layout (lapssd_rows).  tokens_out [device,
 * B x (k+1)], n_accept_out [device, B] are nullable.  count_out as in laps_select.
 * Device-side waits carry watchdogs; an expiry sets LAPSSD_ESTATE flags (see
 * lapssd_check) and the step's results are invalid.  Errors: EINVAL, ECUDA. */
lapssd_status laps_step(lapssd_handle *h, const lapssd_rows *rows, int32_t B, int32_t *sel_inout,
                        int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out,
                        lapssd_stream stream);

/* laps_step_logits -- the LAPS-SD step from LOGITS (SURVEY 8(f) f1 inside the step;
 * P:57-64, P:200 with the quantised softmax of spec_verify_logits, DESIGN.md AMB-30):
 * for the batch in sel_inout (as left by laps_select / the previous step), slot b verifies
 * request i = sel_inout[b] exactly as spec_verify_logits would with req_id = the global
 * id (i * world + rank), round_idx = the request's round count, slab = rows->slab_tab[i,
 * slab_round_index(round)] (pooled layout; without a slab table slot b reads slab b),
 * then runs laps_update with the resulting r and laps_select for the next batch.  rows:
 * logits in rows->p ((k+1) x V target logits per slab) and rows->q (k x V draft logits),
 * rows->draft, dtype bf16 / fp32, V <= 2^23.  Outputs [device, nullable: internal
 * buffers]: tokens_out [B, k+1], n_accept_out [B] (-1 and -1 tokens for empty slots),
 * count_out as laps_select.  workspace: [device] >= laps_step_logits_workspace_bytes(B,
 * k, V, dtype) bytes, any content.  One C-ABI call, five launches on the caller's stream
 * (slot counters, the lazy verify, the empty-slot mask, the update, the select); not
 * overlapped like laps_step.  Errors: EINVAL (handle, B, rows, k mismatch, NULL),
 * ENOMEM (workspace), ECUDA. */
size_t laps_step_logits_workspace_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype);
lapssd_status laps_step_logits(lapssd_handle *h, const lapssd_rows *rows, int32_t B, int32_t *sel_inout,
                               int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out, void *workspace,
                               size_t workspace_bytes, lapssd_stream stream);
/* Opt in (enable = 1) or out (0, the default) of overlapping consecutive laps_step /
 * laps_step_dist verify launches (programmatic dependent launch; contract above).
 * Errors: EINVAL (NULL handle). */
lapssd_status lapssd_set_step_overlap(lapssd_handle *h, int32_t enable);
/* Row validation (default off): with enable = 1 the verify kernel of laps_step /
 * laps_step_dist also checks every streamed row pair's residual mass and sets device flag
 * 256 (lapssd_check) for rows that are not probabilities (a vector of 8 entries or a lane
 * of 32 with mass >= 2, five lanes of a 1,024-entry segment with >= 0.25 each, or a segment
 * >= 4): such masses never wrap silently into the integer sums.  Costs ~4 % of the step
 * (measured).  Independently of it, a row pair whose total residual mass exceeds 2 always
 * sets flag 256.  Errors: EINVAL (NULL handle). */
lapssd_status lapssd_set_row_check(lapssd_handle *h, int32_t enable);

/* ---------------------------------------------------------------------------
 * Multi-GPU (a8): requests are sharded by global id mod world; every rank keeps the
 * same global clock.  laps_candidates does laps_select's clock/admission/keys and
 * writes this rank's candidate block of 2C+1 words into cand_out [device u64]:
 * [0, C) its C smallest eligible keys (ascending, UINT64_MAX padded), [C, 2C) each
 * key's switch-in cost in us if it is selected (0 for padding; AMB-24), [2C] this
 * rank's next arrival time (as u64, UINT64_MAX if none).  After an all-gather of the
 * world*(2C+1) words, laps_merge takes the global top-B keys, keeps the ids with
 * id % world == rank as this rank's batch (sel_out, key order) and advances the clock by
 * the GLOBAL batch (one round plus the selected keys' switch-in costs).
 * laps_step_dist = verify + update + candidates + ncclAllGather (on `nccl_comm`, a
 * ncclComm_t created by the caller) + merge, with the results of that sequence; with
 * pooled rows the candidates / all-gather / merge run on the side stream beside the
 * verify kernel as in laps_step.  NCCL is resolved at run time with
 * dlopen("libnccl.so.2"); if unavailable the call returns ENCCL.  tokens_out [device,
 * B_global x (k+1)] and n_accept_out [device, B_global] (nullable) receive this rank's
 * slots' results as in laps_step (slots [count, B_global) of this rank: r = -1). */
lapssd_status laps_candidates(lapssd_handle *h, int32_t C, uint64_t *cand_out,
                              lapssd_stream stream);
lapssd_status laps_merge(lapssd_handle *h, const uint64_t *all_cand, int32_t C, int32_t B,
                         int32_t *sel_out, int32_t *count_out, lapssd_stream stream);
lapssd_status laps_step_dist(lapssd_handle *h, void *nccl_comm, const lapssd_rows *rows,
                             int32_t B_global, int32_t C, int32_t *sel_inout, int32_t *count_out,
                             int32_t *tokens_out, int32_t *n_accept_out,
                             uint64_t *cand_scratch /* [device] (world+1)*(2C+1) words */,
                             lapssd_stream stream);
/* laps_step_candidates -- laps_step_dist without the collective: verify + update of this
 * rank's slots of sel_inout, then this rank's candidate block (2C+1 words, layout as
 * laps_candidates) into cand_out [device], ordered on `stream`.  The caller exchanges the
 * world blocks with a collective of its choice (NCCL, gloo, MPI: world*(2C+1) words in
 * rank order) and calls laps_merge(h, all, C, B_global, sel_inout, ...); the two calls
 * together have the results of laps_step_dist.  Errors: EINVAL, ECUDA. */
lapssd_status laps_step_candidates(lapssd_handle *h, const lapssd_rows *rows, int32_t B_global, int32_t C,
                                   int32_t *sel_inout, int32_t *tokens_out, int32_t *n_accept_out,
                                   uint64_t *cand_out, lapssd_stream stream);
/* laps_step_peer -- the multi-GPU step with the exchange FUSED into the select kernel
 * over peer memory (NVLink / NVSwitch; no collective launch): the verify kernel as in
 * laps_step, and beside it the side select builds this rank's candidate block (C keys,
 * their switch-in costs, its next arrival), stores it into slot `rank` of EVERY rank's
 * exchange buffer through peer pointers and publishes it with a system-scope release of
 * the step's tag, waits (acquire, with a watchdog: flags 16 | 512) for all world blocks in
 * its own buffer, ranks the keys among the world sorted lists and commits this rank's
 * prefix of the global top-B -- the results of laps_step_dist.  Setup, once per handle:
 * every rank allocates a ZERO-FILLED device buffer of lapssd_peer_buffer_bytes(world, C)
 * bytes, the buffers are mapped into every process (CUDA IPC; the binding uses torch's),
 * and lapssd_set_peers(h, peer_bufs, C, stream) passes the world device pointers valid in
 * this process (peer_bufs[rank] = its own buffer; [host] array).  The first batch comes
 * from laps_candidates + an all-gather + laps_merge.  C as below; rows pooled; B_global
 * <= 4096.  tokens_out / n_accept_out as laps_step_dist.  All ranks call laps_step_peer
 * in lockstep.  Errors: EINVAL, ECUDA. */
size_t lapssd_peer_buffer_bytes(int32_t world, int32_t C);
lapssd_status lapssd_set_peers(lapssd_handle *h, void *const *peer_bufs, int32_t C, lapssd_stream stream);
lapssd_status laps_step_peer(lapssd_handle *h, const lapssd_rows *rows, int32_t B_global, int32_t *sel_inout,
                             int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out,
                             lapssd_stream stream);
/* C must be the same on every rank and world*C <= 16384: the caller passes
 * C = min(B_global, max over ranks of n_local).  sel_inout has B_global slots.
 * NCCL plumbing without torch internals: rank 0 calls lapssd_nccl_unique_id, the
 * 128 bytes are broadcast over torch.distributed, every rank calls
 * lapssd_nccl_comm_init. */
lapssd_status lapssd_nccl_unique_id(uint8_t id_out[128]);
lapssd_status lapssd_nccl_comm_init(void **comm_out, int32_t nranks, const uint8_t id[128],
                                    int32_t rank);
lapssd_status lapssd_nccl_comm_destroy(void *comm);

/* ---------------------------------------------------------------------------
 * State snapshot for parity and replay: D2H copies into caller-allocated [host]
 * arrays (any pointer may be NULL to skip), then synchronises the stream. */
typedef struct {
    int64_t now_us;
    int32_t cursor, prev_count;
    int32_t *acc_tok, *acc_draft, *rounds;        /* n each            */
    int64_t *E_us, *T_total_us, *C_us, *x_us;     /* n each            */
    uint8_t *admitted, *done, *perceptible, *pinned, *level, *running; /* n each */
    double *A;                                    /* n                 */
    uint64_t *key;                                /* n: last select's keys */
    int32_t *ring;                                /* n * gamma         */
    int64_t *switch_us;                           /* n: switching time charged on its entries */
    int64_t step_cost_us;     /* out: duration of the step selected last (round + switch-ins) */
    int64_t switch_total_us;  /* out: system time spent switching so far (AMB-24)           */
} lapssd_state_view;
lapssd_status lapssd_read_state(lapssd_handle *h, lapssd_state_view *host_out,
                                lapssd_stream stream);

/* Synchronises the handle's last stream; returns LAPSSD_ESTATE if the device flag
 * is set (and the flag bits in *flags_out, nullable), else LAPSSD_OK.  Bits: 1 update
 * of a completed request, 2 a row with no probability mass, 4 a slot naming a bad
 * request / slab, 8 a descriptor that does not match the batch, 16 a device-side
 * watchdog expired (results invalid) with 32 / 64 / 128 naming the wait (verify
 * finisher / select merge / verify snapshot; 512 with 16: the wait for the peers' candidate
 * blocks, laps_step_peer), 256 a row pair whose residual mass exceeds 2
 * (rows that are not probabilities: the integer sums are invalid, never silently wrapped);
 * lapssd_last_error() then reports the step and slot of the first expiry. */
lapssd_status lapssd_check(lapssd_handle *h, uint32_t *flags_out);

/* Per-kernel timing of laps_step for the next max_steps calls: the library records
 * CUDA events (host objects, created here) immediately before the verify kernel,
 * between verify and select, and after select, on the call's stream.
 * lapssd_profile_read synchronises and returns the summed verify / select times (ms)
 * and the number of steps recorded; it also ends the profiling window.
 * max_steps <= 0 disables profiling. */
lapssd_status lapssd_profile(lapssd_handle *h, int32_t max_steps);
lapssd_status lapssd_profile_read(lapssd_handle *h, double *verify_ms, double *select_ms,
                                  double *presort_ms, int32_t *steps);
/* presort_ms: summed time from the step's start to the end of the side-stream presort
 * (it overlaps the verify kernel; if it exceeds verify_ms the select waits for it). */

/* ---------------------------------------------------------------------------
 * Monte-Carlo replicas (SURVEY §8(d) configs[4]; §8(a) a6 "per-trace top-1").
 * T independent traces, each a simulation of its own requests with its own clock and
 * ONE request served at a time (batch 1).  One laps_mc_step advances every trace
 * by one round: verify the request it runs (a1-a2, Philox c3 = the trace index t), its
 * state update (a3), the trace clock (+ c_round after a round, next arrival when idle,
 * P:84-93), admission, keys and the trace's top-1, x_i / pinning.
 * Per trace the result is exactly that of a single-trace handle (and the oracle) with
 * B = 1 and trace index t; traces share only the slab pool.
 *
 * trace_offsets [host, n_traces+1]: trace t owns requests [off[t], off[t+1]) of the
 *   concatenated arrays; off[0] = 0; arrival_us sorted within each trace; local
 *   request ids (their index within the trace, < 2^24 - 1) are the Philox c0 and the
 *   key id.  Requests of one trace may not exceed 2^24 - 2; the total is < 2^31.
 * rows: pooled layout only; slab_tab is indexed by the GLOBAL request index
 *   (off[t] + local), n_total x R.
 * laps_mc_select: the first selection of every trace (no verification).
 * laps_mc_step: tokens_out [device, T*(k+1)] and n_accept_out [device, T] (nullable:
 *   internal buffers) receive trace t's emitted tokens and r in slot t (r = -1, tokens
 *   untouched for an idle trace); active_out [device int32, nullable] = the number of
 *   traces that selected a request for the next step (0: every trace has finished).
 * lapssd_mc_read: D2H snapshot; the view's arrays hold n_total entries (its now_us /
 *   cursor / prev_count fields are unused), now_us / cursor / sel [host, T] per trace
 *   (sel = local index of the request the trace runs next, or -1).  Synchronises.
 * Errors: EINVAL (config, offsets, ids, unsorted arrivals, rows), ENOMEM, ECUDA;
 *   lapssd_mc_check reports device contract violations as LAPSSD_ESTATE. */
typedef struct lapssd_mc lapssd_mc;
size_t lapssd_mc_workspace_bytes(const lapssd_config *cfg, int32_t n_traces, int64_t n_total, int64_t V);
lapssd_status lapssd_mc_create(const lapssd_config *cfg, int32_t n_traces, const int64_t *trace_offsets,
                               const int64_t *arrival_us, const int32_t *L_true, const int32_t *L_pred,
                               const int32_t *prompt /* [host] nullable: all 0 */, int64_t V, void *workspace, size_t workspace_bytes, lapssd_stream stream,
                               lapssd_mc **out);
lapssd_status lapssd_mc_destroy(lapssd_mc *h);
lapssd_status laps_mc_select(lapssd_mc *h, const lapssd_rows *rows, lapssd_stream stream);
lapssd_status laps_mc_step(lapssd_mc *h, const lapssd_rows *rows, int32_t *tokens_out,
                           int32_t *n_accept_out, int32_t *active_out, lapssd_stream stream);
lapssd_status lapssd_mc_read(lapssd_mc *h, lapssd_state_view *view, int64_t *now_us, int32_t *cursor,
                             int32_t *sel, lapssd_stream stream);
lapssd_status lapssd_mc_check(lapssd_mc *h, uint32_t *flags_out);

/* Thread-local text of the last error ("" if none). */
const char *lapssd_last_error(void);

/* Number of kernel launches the library enqueued since load (evidence counter). */
uint64_t lapssd_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LAPSSD_H */
