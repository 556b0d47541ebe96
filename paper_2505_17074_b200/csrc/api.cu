// api.cu -- the C-ABI of liblapssd.so (include/lapssd.h): validation, workspace
// carving, kernel orchestration, state snapshot, errors, and the NCCL all-gather of
// the multi-GPU step (resolved at run time with dlopen).
#include <cstdlib>
#include <dlfcn.h>

#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lapssd_internal.cuh"

using namespace lapssd;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

lapssd_status fail(lapssd_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
lapssd_status fail(lapssd_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

lapssd_status cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return LAPSSD_OK;
    return fail(LAPSSD_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int32_t n_chunks_of(int64_t V, int32_t dtype) {
    const int64_t te = tile_elems(dtype == LAPSSD_BF16 ? 2 : 4);
    return (int32_t)((V + te - 1) / te);
}
// buffers sized at create hold either dtype: the fp32 chunking has the most chunks
int32_t n_chunks_max(int64_t V) { return n_chunks_of(V, LAPSSD_F32); }

bool rows_ok(int32_t dtype, int64_t V, int32_t k, const void *p, const void *q) {
    if (dtype != LAPSSD_F32 && dtype != LAPSSD_BF16) return false;
    const int64_t esz = dtype == LAPSSD_BF16 ? 2 : 4;
    if (V < 1 || (V * esz) % 16 != 0 || V > (int64_t)kMaxSegs * kSegElems) return false;
    if (k < 1 || k > 16) return false;
    if (((uintptr_t)p | (uintptr_t)q) & 15) return false;
    return true;
}

// Carves a workspace in a fixed order; used both to size and to place.
struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(size_t count) {
        off = align256(off);
        T *ptr = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return ptr;
    }
};

}  // namespace

namespace lapssd {
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
void prepare_all() {
    static std::once_flag once;
    std::call_once(once, [] {
        verify_prepare();
        verify_logits_prepare();
        sched_prepare();
    });
}
}  // namespace lapssd

struct lapssd_handle {
    State st;
    Sched sc;
    int32_t max_batch;
    int64_t V;
    int32_t n_chunks;
    uint64_t *part;
    uint32_t *work;          // verify work-claim counter + retire counter (left zero)
    int32_t *tokens;       // internal outputs when the caller passes NULL
    int32_t *n_accept;
    SlotDesc *desc;        // a1 results for the current batch (valid if desc_valid)
    bool desc_valid = false;
    // laps_step's side-stream select of step t+1 may follow the select of step t directly
    // (it needs the batch that select committed, not the previous verify's completion):
    // true after an incremental laps_step on chain_stream; any other call resets it
    bool side_chained = false;
    bool chain_captured = false;   // the chained step was recorded into a graph
    // lapssd_set_step_overlap: consecutive verify launches may overlap (programmatic
    // dependent launch).  Off by default: the verify kernel then follows all prior work on
    // the caller's stream (a rows-producing kernel of the caller, say).
    bool overlap = false;
    bool check_rows = false;   // lapssd_set_row_check
    cudaStream_t chain_stream = nullptr;
    lapssd_rows last_rows{};  // rows of the previous laps_step (epoch changes with them)
    uint32_t rows_epoch = 1;
    PreSelect *pre = nullptr;    // presort output (side stream)
    SelRec *fin = nullptr;       // finisher records, one per slot (fused select)
    uint32_t *snap = nullptr;    // verify CTAs that have read sel/desc (incremental select)
    uint64_t *fin_key = nullptr; // per-slot published keys (~key, 0 = none) of fin[] (incremental select)
    WaitList wl{};               // the side select's persistent waiting list (wl.valid: host-tracked)
    uint64_t **peer_ptrs = nullptr;  // [device] laps_step_peer: every rank's exchange buffer (kMaxPeers)
    int32_t peer_C = 0;          // 0: no peers set
    cudaStream_t side = nullptr; // side stream for the presort, fork/join events
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t last_stream;
    // profiling window (lapssd_profile): 4 events per recorded step
    std::vector<cudaEvent_t> prof_events;
    int32_t prof_max = 0, prof_used = 0;
    ~lapssd_handle() {
        for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
    }
};

static void carve_state(Carver &cv, State &st, int64_t n, int32_t gamma) {
    const size_t nn = (size_t)(n > 0 ? n : 1);
    st.g = cv.take<Globals>(1);
    st.arrival = cv.take<int64_t>(nn);
    st.L_true = cv.take<int32_t>(nn);
    st.L_pred = cv.take<int32_t>(nn);
    st.prompt = cv.take<int32_t>(nn);
    st.switch_us = cv.take<int64_t>(nn);
    st.acc_tok = cv.take<int32_t>(nn);
    st.acc_draft = cv.take<int32_t>(nn);
    st.rounds = cv.take<int32_t>(nn);
    st.ring = cv.take<int32_t>(nn * (size_t)gamma);
    st.E = cv.take<int64_t>(nn);
    st.T_total = cv.take<int64_t>(nn);
    st.A = cv.take<double>(nn);
    st.flags = cv.take<uint32_t>(nn);
    st.key = cv.take<uint64_t>(nn);
    st.last_sel = cv.take<int32_t>(nn);   // last_sel, C, x, next_tag: all-ones at create (contiguous)
    st.C = cv.take<int64_t>(nn);
    st.x = cv.take<int64_t>(nn);
    st.next_tag = cv.take<uint64_t>(nn);
    st.next_sr = cv.take<int2>(nn);
}

static void carve_handle(Carver &cv, lapssd_handle *h, int32_t n, int32_t gamma, int32_t max_batch,
                         int32_t n_chunks, int32_t k) {
    carve_state(cv, h->st, n, gamma);
    h->part = cv.take<uint64_t>(2 * (size_t)max_batch * n_chunks * kPartWords);  // two parity sets
    h->work = cv.take<uint32_t>(4);
    h->tokens = cv.take<int32_t>((size_t)max_batch * (k + 1));
    h->n_accept = cv.take<int32_t>((size_t)max_batch);
    h->desc = cv.take<SlotDesc>((size_t)max_batch);
    int bp = 1;
    while (bp < max_batch) bp <<= 1;
    h->pre = reinterpret_cast<PreSelect *>(cv.take<uint64_t>(preselect_words(bp)));
    h->fin = cv.take<SelRec>((size_t)max_batch);
    h->snap = cv.take<uint32_t>(1);
    h->fin_key = cv.take<uint64_t>((size_t)max_batch);
    const size_t nn = (size_t)(n > 0 ? n : 1);
    h->wl.keys[0] = cv.take<uint64_t>(nn);
    h->wl.keys[1] = cv.take<uint64_t>(nn);
    h->wl.fresh_i = cv.take<int32_t>((size_t)max_batch);
    h->wl.fresh_key = cv.take<uint64_t>((size_t)max_batch);
    h->wl.meta = cv.take<int32_t>(4);
    h->wl.valid = 0;
    h->peer_ptrs = cv.take<uint64_t *>(64);
}

static lapssd_status check_config(const lapssd_config *c) {
    if (!c) return fail(LAPSSD_EINVAL, "config is NULL");
    if (c->policy < 0 || c->policy > 3) return fail(LAPSSD_EINVAL, "policy %d", c->policy);
    if (c->K < 1 || c->K > 16) return fail(LAPSSD_EINVAL, "K=%d outside 1..16", c->K);
    if (c->s1_up_us <= 0) return fail(LAPSSD_EINVAL, "s1_up_us must be > 0");
    if (!(c->M > 1.0)) return fail(LAPSSD_EINVAL, "M must be > 1");
    if (c->gamma < 2 || c->gamma > 32) return fail(LAPSSD_EINVAL, "gamma must be in 2..32");
    if (!(c->delta >= 0.0)) return fail(LAPSSD_EINVAL, "delta must be >= 0");
    if (c->k < 1 || c->k > 16) return fail(LAPSSD_EINVAL, "k=%d outside 1..16", c->k);
    if (c->t_ssm_us < 0 || c->t_llm_us < 0) return fail(LAPSSD_EINVAL, "negative round cost");
    if (c->placement < 0 || c->placement > 1 || c->pin_rule < 0 || c->pin_rule > 1)
        return fail(LAPSSD_EINVAL, "placement / pin_rule");
    if (c->cost_model != LAPSSD_COST_EQ6 && c->cost_model != LAPSSD_COST_FIG1)
        return fail(LAPSSD_EINVAL, "cost_model %d", c->cost_model);
    if (c->t_tok_us < 0) return fail(LAPSSD_EINVAL, "negative t_tok_us");
    if (c->switch_c0_us < 0 || c->switch_c1_us < 0) return fail(LAPSSD_EINVAL, "negative switching cost");
    return LAPSSD_OK;
}

static void fill_sched(Sched &sc, const lapssd_config *cfg, int32_t n, int32_t rank, int32_t world) {
    sc = Sched{};
    sc.policy = cfg->policy; sc.K = cfg->K; sc.gamma = cfg->gamma; sc.k = cfg->k;
    sc.placement = cfg->placement; sc.pin_rule = cfg->pin_rule;
    sc.n = n; sc.rank = rank; sc.world = world;
    sc.delta = cfg->delta;
    sc.t_ssm_us = cfg->t_ssm_us; sc.t_llm_us = cfg->t_llm_us; sc.t_tok_us = cfg->t_tok_us;
    sc.cost_model = cfg->cost_model;
    // one round's service: k T_SSM + T_LLM (Eq. 6's numerator), or in the
    // Fig. 1 model the k candidates verified at t_tok each (AMB-3)
    sc.c_round_us = cfg->cost_model == LAPSSD_COST_FIG1 ? (int64_t)cfg->k * cfg->t_tok_us
                                                        : (int64_t)cfg->k * cfg->t_ssm_us + cfg->t_llm_us;
    sc.sw_c0_us = cfg->switch_c0_us; sc.sw_c1_us = cfg->switch_c1_us;   // AMB-24
    sc.sw_on = cfg->switch_c0_us > 0 || cfg->switch_c1_us > 0;
    sc.seed = cfg->seed;
    // S_j^up = M^(j-1) S_1^up; zero-based S_up[j] = floor(s1_up * M^j), M^j by
    // iterative fp64 multiplication (AMB-11).
    double m = 1.0;
    for (int j = 0; j < 16; ++j) {
        if (j < cfg->K - 1) {
            const double v = (double)cfg->s1_up_us * m;
            sc.S_up[j] = v >= 9.2e18 ? INT64_MAX : (int64_t)std::floor(v);
            m = m * cfg->M;
        } else {
            sc.S_up[j] = INT64_MAX;
        }
    }
}

// Zero-fill a state workspace, all-ones for last_sel / C / x / next_tag, copy the request
// arrays (prompt nullable: zeros).
static cudaError_t init_state(void *workspace, size_t bytes, const State &st, int64_t n, const int64_t *arrival,
                              const int32_t *L_true, const int32_t *L_pred, const int32_t *prompt, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(workspace, 0, bytes, s);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(st.last_sel, 0xFF,
                            (size_t)((char *)(st.next_tag + (n > 0 ? n : 1)) - (char *)st.last_sel), s);
    if (e == cudaSuccess && n > 0 && prompt)
        e = cudaMemcpyAsync((void *)st.prompt, prompt, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && n > 0) {
        e = cudaMemcpyAsync((void *)st.arrival, arrival, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((void *)st.L_true, L_true, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((void *)st.L_pred, L_pred, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
    }
    return e;
}

extern "C" {

const char *lapssd_last_error(void) { return g_last_error.c_str(); }

uint64_t lapssd_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------- spec_verify
size_t spec_verify_workspace_bytes(int32_t B, int64_t V) {
    if (B < 0 || V < 1) return 0;
    Carver cv{nullptr};
    cv.take<uint64_t>((size_t)(B > 0 ? B : 1) * n_chunks_max(V) * kPartWords);
    cv.take<uint32_t>(2);
    cv.take<SlotDesc>((size_t)(B > 0 ? B : 1));
    return align256(cv.off);
}

static RowsDev rows_dev(const void *p, const void *q, const int32_t *draft, const int32_t *slab_tab,
                        int64_t V, int32_t k, int32_t R, int32_t dtype) {
    RowsDev rw{};
    rw.p = p; rw.q = q; rw.draft = draft; rw.slab_tab = slab_tab;
    rw.V = V; rw.k = k; rw.R = R; rw.dtype = dtype; rw.valid = 1;
    return rw;
}

lapssd_status spec_verify(const void *p, const void *q, int32_t dtype, int64_t V, int32_t k,
                          const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                          const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                          int32_t *tokens, int32_t *n_accept, uint64_t *z_fixed, void *workspace,
                          size_t workspace_bytes, lapssd_stream stream) {
    g_last_error.clear();
    if (B < 0) return fail(LAPSSD_EINVAL, "B < 0");
    if (!rows_ok(dtype, V, k, p, q)) return fail(LAPSSD_EINVAL, "rows: dtype/V/k/alignment");
    if (B == 0) return LAPSSD_OK;
    if (!p || !q || !draft || !req_id || !round_idx || !tokens || !n_accept || !workspace)
        return fail(LAPSSD_EINVAL, "NULL pointer argument");
    if (workspace_bytes < spec_verify_workspace_bytes(B, V))
        return fail(LAPSSD_ENOMEM, "workspace %zu < %zu bytes", workspace_bytes,
                    spec_verify_workspace_bytes(B, V));
    prepare_all();
    VerifyArgs a{};
    a.rows = rows_dev(p, q, draft, nullptr, V, k, 0, dtype);
    a.n_chunks = n_chunks_of(V, dtype);
    a.cpb = verify_cpb(V);
    a.seed = seed; a.trace = trace;
    a.tokens = tokens; a.n_accept = n_accept; a.z = z_fixed;
    Carver cv{(char *)workspace};
    a.part = cv.take<uint64_t>((size_t)B * a.n_chunks * kPartWords);
    a.work = cv.take<uint32_t>(2);
    SlotDesc *desc = cv.take<SlotDesc>((size_t)B);
    a.desc = desc;
    a.sel = nullptr;
    a.err = nullptr;
    a.fuse_update = 0;
    cudaStream_t s = (cudaStream_t)stream;
    lapssd_status st = cuda_status(launch_accept(a.rows, nullptr, nullptr, nullptr, slab, req_id, round_idx,
                                                 seed, trace, B, desc, s), "spec_verify accept");
    if (st != LAPSSD_OK) return st;
    // one launch per sub-batch that fits the kernel's per-CTA snapshot (all of B at usual sizes)
    const int32_t bmax = verify_max_batch(a.n_chunks, 0);
    for (int32_t b0 = 0; b0 < B && st == LAPSSD_OK; b0 += bmax) {
        VerifyArgs ab = a;
        const int32_t nb = B - b0 < bmax ? B - b0 : bmax;
        ab.desc = desc + b0;
        ab.tokens = tokens + (int64_t)b0 * (k + 1);
        ab.n_accept = n_accept + b0;
        ab.z = z_fixed ? z_fixed + b0 : nullptr;
        ab.part = a.part + (int64_t)b0 * a.n_chunks * kPartWords;
        st = cuda_status(launch_verify(ab, nb, s), "spec_verify launch");
    }
    return st;
}

// ---------------------------------------------------------------- f1: verify from logits
size_t spec_verify_logits_workspace_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype) {
    if (B < 0 || k < 1 || k > 16 || V < 1 || (dtype != LAPSSD_BF16 && dtype != LAPSSD_F32)) return 0;
    const int32_t Bn = B > 0 ? B : 1;
    const size_t rows = (size_t)Bn * (size_t)(2 * k + 1);
    Carver cv{nullptr};
    cv.take<float>(rows);
    cv.take<uint64_t>(rows);
    cv.take<char>(logits_lazy_bytes(Bn, k, V, dtype));
    return align256(cv.off);
}

lapssd_status spec_verify_logits(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                                 const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                                 const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                                 int32_t *tokens, int32_t *n_accept, uint64_t *z, void *workspace,
                                 size_t workspace_bytes, lapssd_stream stream) {
    g_last_error.clear();
    if (B < 0) return fail(LAPSSD_EINVAL, "B < 0");
    if (!rows_ok(dtype, V, k, zp, zq)) return fail(LAPSSD_EINVAL, "rows: dtype/V/k/alignment");
    if (V > (int64_t)1 << 23) return fail(LAPSSD_EINVAL, "V > 2^23 (integer softmax mass would overflow)");
    if (B == 0) return LAPSSD_OK;
    if (!zp || !zq || !draft || !req_id || !round_idx || !tokens || !n_accept || !workspace)
        return fail(LAPSSD_EINVAL, "NULL pointer argument");
    if (workspace_bytes < spec_verify_logits_workspace_bytes(B, k, V, dtype))
        return fail(LAPSSD_ENOMEM, "workspace %zu < %zu bytes", workspace_bytes,
                    spec_verify_logits_workspace_bytes(B, k, V, dtype));
    prepare_all();
    Carver cv{(char *)workspace};
    const size_t rows = (size_t)B * (size_t)(2 * k + 1);
    float *m_ws = cv.take<float>(rows);
    uint64_t *S_ws = cv.take<uint64_t>(rows);
    char *lazy_ws = cv.take<char>(logits_lazy_bytes(B, k, V, dtype));
    return cuda_status(launch_verify_logits(zp, zq, dtype, V, k, draft, slab, req_id, round_idx, B, seed, trace,
                                            tokens, n_accept, z, m_ws, S_ws, lazy_ws, (cudaStream_t)stream),
                       "spec_verify_logits");
}

// ---------------------------------------------------------------- f4: draft sampling, tree verification
lapssd_status spec_draft_sample(const void *q, int32_t dtype, int64_t V, const int32_t *row, const uint32_t *req_id,
                                const uint32_t *round_idx, const uint32_t *pos, int32_t R, uint64_t seed,
                                uint32_t trace, int32_t *draft_out, uint64_t *z_out, lapssd_stream stream) {
    g_last_error.clear();
    if (R < 0) return fail(LAPSSD_EINVAL, "R < 0");
    if (!rows_ok(dtype, V, 1, q, q)) return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    if (R == 0) return LAPSSD_OK;
    if (!q || !req_id || !round_idx || !pos || !draft_out) return fail(LAPSSD_EINVAL, "NULL pointer argument");
    prepare_all();
    return cuda_status(launch_draft_sample(q, dtype, V, row, req_id, round_idx, pos, R, seed, trace, draft_out,
                                           z_out, (cudaStream_t)stream),
                       "spec_draft_sample");
}

lapssd_status spec_verify_tree(const void *p, const void *q, int32_t dtype, int64_t V, int32_t n_nodes,
                               const int32_t *parent, const int32_t *token, const uint32_t *req_id,
                               const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                               int32_t *tokens, int32_t *path, int32_t *n_accept, uint64_t *z_out,
                               lapssd_stream stream) {
    g_last_error.clear();
    if (B < 0) return fail(LAPSSD_EINVAL, "B < 0");
    if (n_nodes < 1 || n_nodes > 64) return fail(LAPSSD_EINVAL, "n_nodes=%d outside 1..64", n_nodes);
    if (!rows_ok(dtype, V, 1, p, q)) return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    if (B == 0) return LAPSSD_OK;
    if (!p || !q || !parent || !token || !req_id || !round_idx || !tokens || !n_accept)
        return fail(LAPSSD_EINVAL, "NULL pointer argument");
    prepare_all();
    return cuda_status(launch_verify_tree(p, q, dtype, V, n_nodes, parent, token, req_id, round_idx, B, seed, trace,
                                          tokens, path, n_accept, z_out, (cudaStream_t)stream),
                       "spec_verify_tree");
}

// ---------------------------------------------------------------- handle
size_t lapssd_workspace_bytes(const lapssd_config *cfg, int32_t n_local, int32_t max_batch, int64_t V,
                              int32_t world) {
    (void)world;
    if (!cfg || n_local < 0 || max_batch < 1 || V < 1) return 0;
    lapssd_handle tmp{};
    Carver cv{nullptr};
    carve_handle(cv, &tmp, n_local, cfg->gamma > 0 ? cfg->gamma : 1, max_batch, n_chunks_max(V),
                 cfg->k > 0 ? cfg->k : 1);
    return align256(cv.off);
}

lapssd_status lapssd_create(const lapssd_config *cfg, const lapssd_requests *req, int32_t max_batch,
                            int64_t V, void *workspace, size_t workspace_bytes, lapssd_stream stream,
                            lapssd_handle **out) {
    g_last_error.clear();
    if (!out) return fail(LAPSSD_EINVAL, "out is NULL");
    *out = nullptr;
    lapssd_status st = check_config(cfg);
    if (st != LAPSSD_OK) return st;
    if (!req || req->n < 0 || req->world < 1 || req->rank < 0 || req->rank >= req->world)
        return fail(LAPSSD_EINVAL, "requests: n / rank / world");
    if (req->n > 0 && (!req->arrival_us || !req->L_true || !req->L_pred))
        return fail(LAPSSD_EINVAL, "requests: NULL arrays");
    if ((int64_t)req->n * req->world + req->rank > (1 << 24) - 1)
        return fail(LAPSSD_EINVAL, "global ids must be < 2^24 - 1");   // key ~0 stays unused
    if (req->n > sort_capacity())
        return fail(LAPSSD_EINVAL, "n_local=%d exceeds the single-CTA select capacity %d", req->n,
                    sort_capacity());
    if (max_batch < 1) return fail(LAPSSD_EINVAL, "max_batch < 1");
    if (V < 1 || V > (int64_t)kMaxSegs * kSegElems) return fail(LAPSSD_EINVAL, "V out of range");
    for (int32_t i = 0; i < req->n; ++i) {
        if (req->L_true[i] < 1 || req->L_pred[i] < 1) return fail(LAPSSD_EINVAL, "L < 1 at %d", i);
        if (req->prompt && req->prompt[i] < 0) return fail(LAPSSD_EINVAL, "prompt < 0 at %d", i);
        if (i > 0 && req->arrival_us[i] < req->arrival_us[i - 1])
            return fail(LAPSSD_EINVAL, "arrivals not sorted at %d", i);
    }
    const size_t need = lapssd_workspace_bytes(cfg, req->n, max_batch, V, req->world);
    if (!workspace || workspace_bytes < need)
        return fail(LAPSSD_ENOMEM, "workspace %zu < %zu bytes", workspace_bytes, need);

    prepare_all();
    if (!verify_fits(max_batch, n_chunks_max(V), 0) || !verify_fits(max_batch, n_chunks_max(V), 1))
        return fail(LAPSSD_EINVAL, "max_batch=%d exceeds the verify kernel's per-CTA capacity (%d at this V)",
                    max_batch, verify_max_batch(n_chunks_max(V), 1));
    lapssd_handle *h = new lapssd_handle{};
    Carver cv{(char *)workspace};
    carve_handle(cv, h, req->n, cfg->gamma, max_batch, n_chunks_max(V), cfg->k);
    h->max_batch = max_batch;
    h->V = V;
    h->n_chunks = n_chunks_max(V);
    fill_sched(h->sc, cfg, req->n, req->rank, req->world);
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    cudaError_t e = init_state(workspace, need, h->st, req->n, req->arrival_us, req->L_true, req->L_pred,
                               req->prompt, s);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host arrays may be freed on return
    if (e != cudaSuccess) {
        delete h;
        return cuda_status(e, "lapssd_create");
    }
    *out = h;
    return LAPSSD_OK;
}

lapssd_status lapssd_destroy(lapssd_handle *h) {
    delete h;
    return LAPSSD_OK;
}

// ---------------------------------------------------------------- a3 / a4-a7
lapssd_status laps_update(lapssd_handle *h, const int32_t *sel, const int32_t *n_accept, int32_t B,
                          lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || B < 0 || B > h->max_batch) return fail(LAPSSD_EINVAL, "handle / B");
    if (B > 0 && (!sel || !n_accept)) return fail(LAPSSD_EINVAL, "NULL sel / n_accept");
    h->last_stream = (cudaStream_t)stream;
    h->desc_valid = false;
    return cuda_status(launch_update(h->st, h->sc, sel, n_accept, B, (cudaStream_t)stream), "laps_update");
}

lapssd_status laps_select(lapssd_handle *h, int32_t B, int32_t *sel_out, int32_t *count_out,
                          lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || B < 1 || B > h->max_batch) return fail(LAPSSD_EINVAL, "handle / B");
    if (!sel_out) return fail(LAPSSD_EINVAL, "sel_out is NULL");
    h->last_stream = (cudaStream_t)stream;
    h->desc_valid = false;
    const RowsDev none{};
    return cuda_status(launch_select(h->st, h->sc, none, h->desc, B, sel_out, count_out, (cudaStream_t)stream),
                       "laps_select");
}

// ---------------------------------------------------------------- f1 in the LAPS-SD step
size_t laps_step_logits_workspace_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype) {
    if (!spec_verify_logits_workspace_bytes(B, k, V, dtype)) return 0;
    const int32_t Bn = B > 0 ? B : 1;
    const size_t rows = (size_t)Bn * (size_t)(2 * k + 1);
    Carver cv{nullptr};   // the same carving as laps_step_logits
    cv.take<float>(rows);
    cv.take<uint64_t>(rows);
    cv.take<char>(logits_lazy_bytes(Bn, k, V, dtype));
    cv.take<uint32_t>((size_t)Bn);
    cv.take<uint32_t>((size_t)Bn);
    cv.take<int32_t>((size_t)Bn);
    return align256(cv.off);
}

lapssd_status laps_step_logits(lapssd_handle *h, const lapssd_rows *rows, int32_t B, int32_t *sel_inout,
                               int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out, void *workspace,
                               size_t workspace_bytes, lapssd_stream stream) {
    g_last_error.clear();
    if (!h || B < 1 || B > h->max_batch) return fail(LAPSSD_EINVAL, "handle / B");
    if (!rows || !rows->p || !rows->q || !rows->draft) return fail(LAPSSD_EINVAL, "rows: NULL pointer");
    if (rows->k != h->sc.k) return fail(LAPSSD_EINVAL, "rows.k=%d != config k=%d", rows->k, h->sc.k);
    if (!rows_ok(rows->dtype, rows->V, rows->k, rows->p, rows->q)) return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    if (rows->V > (int64_t)1 << 23) return fail(LAPSSD_EINVAL, "V > 2^23 (integer softmax mass would overflow)");
    if (rows->slab_tab && rows->R < 1) return fail(LAPSSD_EINVAL, "rows.R < 1");
    if (!sel_inout || !workspace) return fail(LAPSSD_EINVAL, "NULL sel / workspace");
    const int32_t k = rows->k;
    if (workspace_bytes < laps_step_logits_workspace_bytes(B, k, rows->V, rows->dtype))
        return fail(LAPSSD_ENOMEM, "workspace %zu < %zu bytes", workspace_bytes,
                    laps_step_logits_workspace_bytes(B, k, rows->V, rows->dtype));
    prepare_all();
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    h->side_chained = false;
    h->wl.valid = 0;
    h->desc_valid = false;
    int32_t *tok = tokens_out ? tokens_out : h->tokens;
    int32_t *na = n_accept_out ? n_accept_out : h->n_accept;
    Carver cv{(char *)workspace};
    const size_t nrow = (size_t)B * (size_t)(2 * k + 1);
    float *m_ws = cv.take<float>(nrow);
    uint64_t *S_ws = cv.take<uint64_t>(nrow);
    char *lazy_ws = cv.take<char>(logits_lazy_bytes(B, k, rows->V, rows->dtype));
    uint32_t *req = cv.take<uint32_t>((size_t)B);
    uint32_t *rnd = cv.take<uint32_t>((size_t)B);
    int32_t *slab = cv.take<int32_t>((size_t)B);
    lapssd_status st = cuda_status(launch_logits_slots(sel_inout, h->st.rounds, rows->slab_tab, rows->R, h->sc.world,
                                                       h->sc.rank, B, req, rnd, slab, s), "laps_step_logits slots");
    if (st != LAPSSD_OK) return st;
    st = cuda_status(launch_verify_logits(rows->p, rows->q, rows->dtype, rows->V, k, rows->draft, slab, req, rnd, B,
                                          h->sc.seed, 0, tok, na, nullptr, m_ws, S_ws, lazy_ws, s),
                     "laps_step_logits verify");
    if (st != LAPSSD_OK) return st;
    st = cuda_status(launch_logits_mask(sel_inout, k, B, tok, na, s), "laps_step_logits mask");
    if (st != LAPSSD_OK) return st;
    st = cuda_status(launch_update(h->st, h->sc, sel_inout, na, B, s), "laps_step_logits update");
    if (st != LAPSSD_OK) return st;
    const RowsDev none{};
    return cuda_status(launch_select(h->st, h->sc, none, h->desc, B, sel_inout, count_out, s),
                       "laps_step_logits select");
}

static lapssd_status fill_step_verify(lapssd_handle *h, const lapssd_rows *rows, int32_t B, int32_t *sel,
                                      int32_t *tokens_out, int32_t *n_accept_out, VerifyArgs &a) {
    if (!rows) return fail(LAPSSD_EINVAL, "rows is NULL");
    if (rows->k != h->sc.k) return fail(LAPSSD_EINVAL, "rows.k=%d != config k=%d", rows->k, h->sc.k);
    if (!rows_ok(rows->dtype, rows->V, rows->k, rows->p, rows->q) || rows->V > h->V)
        return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    if (!rows->p || !rows->q || !rows->draft) return fail(LAPSSD_EINVAL, "rows: NULL pointer");
    if (rows->slab_tab && rows->R < 1) return fail(LAPSSD_EINVAL, "rows.R < 1");
    if (!sel) return fail(LAPSSD_EINVAL, "sel is NULL");
    if (memcmp(&h->last_rows, rows, sizeof *rows) != 0) {
        h->last_rows = *rows;
        h->rows_epoch++;            // cached next-round acceptance tests are for other rows
    }
    a = VerifyArgs{};
    a.rows = rows_dev(rows->p, rows->q, rows->draft, rows->slab_tab, rows->V, rows->k, rows->R, rows->dtype);
    a.rows.epoch = h->rows_epoch;
    a.n_chunks = n_chunks_of(rows->V, rows->dtype);
    a.cpb = verify_cpb(rows->V);
    a.desc = h->desc;
    a.sel = sel;
    a.seed = h->sc.seed; a.trace = 0;
    a.tokens = tokens_out ? tokens_out : h->tokens;
    a.n_accept = n_accept_out ? n_accept_out : h->n_accept;
    a.z = nullptr;
    a.part = h->part; a.work = h->work;
    a.fuse_update = 1;
    a.check_rows = h->check_rows;
    a.st = h->st; a.sc = h->sc;
    a.err = &h->st.g->err;
    (void)B;
    return LAPSSD_OK;
}

// Verification of the current batch: the descriptors come from the previous select
// (fused a1); if that select had no rows (or the state changed since), run a1 first.
// Profiling event record: an external event node when the stream is being captured.
static void prof_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else
        cudaEventRecord(e, s);
}

static lapssd_status step_verify(lapssd_handle *h, const VerifyArgs &a, int32_t *sel, int32_t B,
                                 cudaStream_t s) {
    if (!h->desc_valid || a.rows.slab_tab == nullptr) {   // batch layout: this call's rows
        lapssd_status st = cuda_status(launch_accept(a.rows, sel, &h->st, &h->sc, nullptr, nullptr, nullptr,
                                                     h->sc.seed, 0, B, h->desc, s), "accept");
        if (st != LAPSSD_OK) return st;
    }
    h->desc_valid = false;
    return cuda_status(launch_verify(a, B, s), "verify");
}

lapssd_status laps_step(lapssd_handle *h, const lapssd_rows *rows, int32_t B, int32_t *sel_inout,
                        int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out,
                        lapssd_stream stream) {
    g_last_error.clear();
    if (!h || B < 1 || B > h->max_batch) return fail(LAPSSD_EINVAL, "handle / B");
    VerifyArgs a;
    lapssd_status st = fill_step_verify(h, rows, B, sel_inout, tokens_out, n_accept_out, a);
    if (st != LAPSSD_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    cudaEvent_t *ev = nullptr;
    if (h->prof_used < h->prof_max) ev = &h->prof_events[4 * (size_t)h->prof_used++];
    if (ev) prof_record(ev[0], s);
    int bp = 1;
    while (bp < B) bp <<= 1;
    // pooled rows: incremental select on the side stream (presort, then merge the batch
    // slots as the verify finishers publish them); batch layout: presort + final select
    const bool incremental = rows->slab_tab != nullptr && bp <= 4096;
    // a1 for the current batch, before the fork (both streams read it): always with the
    // batch layout, whose rows are this call's (the previous select could not know them)
    if (!h->desc_valid || rows->slab_tab == nullptr) {
        st = cuda_status(launch_accept(a.rows, sel_inout, &h->st, &h->sc, nullptr, nullptr, nullptr, h->sc.seed, 0,
                                       B, h->desc, s), "accept");
        if (st != LAPSSD_OK) return st;
    }
    // fork: the next selection's side-stream work runs beside the verify kernel (the
    // verify kernel is launched first so it takes its SMs without waiting).  After an
    // incremental step on the same stream the side stream is chained instead: its select
    // already follows the previous select, which committed everything this one reads, so
    // it need not also wait for the previous verify grid to drain -- its presort then
    // runs while that grid's last CTAs sample.  Under capture the side stream must join
    // the capture through a fork.
    cudaStreamCaptureStatus cap_s = cudaStreamCaptureStatusNone, cap_side = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap_s);
    cudaStreamIsCapturing(h->side, &cap_side);
    static const bool no_chain = getenv("LAPSSD_NO_SIDE_CHAIN") != nullptr;  // A/B switch
    const bool capturing = cap_s == cudaStreamCaptureStatusActive;
    const bool fork = no_chain || !incremental || !h->side_chained || h->chain_stream != s || cap_s != cap_side ||
                      capturing != h->chain_captured || !h->desc_valid;
    h->side_chained = false;
    cudaError_t ce = cudaSuccess;
    if (fork) {
        ce = cudaEventRecord(h->ev_fork, s);
        if (ce != cudaSuccess) return cuda_status(ce, "laps_step fork");
    }
    h->desc_valid = false;
    if (incremental) {
        a.fin = h->fin;
        a.fin_key = h->fin_key;
        a.snap = h->snap;
        a.part1 = h->part + (size_t)h->max_batch * h->n_chunks * kPartWords;
        a.work1 = h->work + 2;
        a.vstep = &h->st.g->vstep;
    }
    static const bool no_pdl = getenv("LAPSSD_NO_PDL") != nullptr;  // A/B switch for measurements
    st = cuda_status(launch_verify_grid(a, B, 1, incremental && h->overlap && !no_pdl, s), "laps_step verify");
    if (st != LAPSSD_OK) return st;
    if (ev) prof_record(ev[1], s);
    if (fork) {
        ce = cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        if (ce != cudaSuccess) return cuda_status(ce, "laps_step fork wait");
    }
    if (incremental) {
        static const bool no_wl = getenv("LAPSSD_NO_WAITLIST") != nullptr;   // A/B switch
        const WaitList *wl = no_wl ? nullptr : &h->wl;
        st = cuda_status(launch_select_side(h->st, h->sc, a.rows, sel_inout, h->desc, B, h->pre, h->fin, h->fin_key,
                                            h->snap, (uint32_t)verify_grid(B, a.n_chunks, 1), count_out, h->side,
                                            nullptr, 0, wl),
                         "laps_step select");
        h->wl.valid = wl != nullptr && bp <= 1024;   // the commit leaves the next list
    } else {
        h->wl.valid = 0;
        st = cuda_status(launch_presort(h->st, h->sc, a.rows, sel_inout, B, h->pre, h->side), "laps_step presort");
    }
    if (st != LAPSSD_OK) return st;
    if (ev) prof_record(ev[3], h->side);
    ce = cudaEventRecord(h->ev_join, h->side);
    if (ce != cudaSuccess) return cuda_status(ce, "laps_step join");
    ce = cudaStreamWaitEvent(s, h->ev_join, 0);
    if (ce != cudaSuccess) return cuda_status(ce, "laps_step join wait");
    if (incremental) {
        h->desc_valid = true;
        h->side_chained = true;
        h->chain_stream = s;
        h->chain_captured = capturing;
        if (ev) prof_record(ev[2], s);
        return LAPSSD_OK;
    }
    st = cuda_status(launch_select_final(h->st, h->sc, a.rows, h->desc, B, sel_inout, count_out, h->pre, s),
                     "laps_step select");
    if (st == LAPSSD_OK) h->desc_valid = true;
    if (ev) prof_record(ev[2], s);
    return st;
}

lapssd_status lapssd_set_step_overlap(lapssd_handle *h, int32_t enable) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    h->overlap = enable != 0;
    return LAPSSD_OK;
}

lapssd_status lapssd_set_row_check(lapssd_handle *h, int32_t enable) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    h->check_rows = enable != 0;
    return LAPSSD_OK;
}

lapssd_status lapssd_profile(lapssd_handle *h, int32_t max_steps) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    for (cudaEvent_t e : h->prof_events) cudaEventDestroy(e);
    h->prof_events.clear();
    h->prof_used = 0;
    h->prof_max = max_steps > 0 ? max_steps : 0;
    h->prof_events.resize(4 * (size_t)h->prof_max);
    for (auto &e : h->prof_events) {
        const cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) { h->prof_max = 0; return cuda_status(err, "cudaEventCreate"); }
    }
    return LAPSSD_OK;
}

lapssd_status lapssd_profile_read(lapssd_handle *h, double *verify_ms, double *select_ms, double *presort_ms,
                                  int32_t *steps) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    double v = 0.0, sl = 0.0, pr = 0.0;
    for (int32_t i = 0; i < h->prof_used; ++i) {
        cudaEvent_t *ev = &h->prof_events[4 * (size_t)i];
        float a = 0.f, b = 0.f, c = 0.f;
        cudaError_t e = cudaEventSynchronize(ev[2]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&a, ev[0], ev[1]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&b, ev[1], ev[2]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&c, ev[0], ev[3]);
        if (e != cudaSuccess) return cuda_status(e, "lapssd_profile_read");
        v += a;
        sl += b;
        pr += c;
    }
    if (verify_ms) *verify_ms = v;
    if (select_ms) *select_ms = sl;
    if (presort_ms) *presort_ms = pr;
    if (steps) *steps = h->prof_used;
    h->prof_max = h->prof_used;   // close the window
    return LAPSSD_OK;
}

// ---------------------------------------------------------------- a8
lapssd_status laps_candidates(lapssd_handle *h, int32_t C, uint64_t *cand_out, lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || C < 1 || !cand_out) return fail(LAPSSD_EINVAL, "handle / C / cand_out");
    h->last_stream = (cudaStream_t)stream;
    h->desc_valid = false;
    return cuda_status(launch_candidates(h->st, h->sc, C, cand_out, (cudaStream_t)stream),
                       "laps_candidates");
}

lapssd_status laps_merge(lapssd_handle *h, const uint64_t *all_cand, int32_t C, int32_t B, int32_t *sel_out,
                         int32_t *count_out, lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || C < 1 || !all_cand || !sel_out || B < 1 || B > h->max_batch)
        return fail(LAPSSD_EINVAL, "handle / C / B / pointers");
    if ((int64_t)h->sc.world * C > sort_capacity())
        return fail(LAPSSD_EINVAL, "world*C=%lld exceeds %d", (long long)h->sc.world * C, sort_capacity());
    h->last_stream = (cudaStream_t)stream;
    h->desc_valid = false;
    const RowsDev none{};
    return cuda_status(launch_merge(h->st, h->sc, none, h->desc, all_cand, C, B, sel_out, count_out,
                                    (cudaStream_t)stream),
                       "laps_merge");
}

}  // extern "C"

// NCCL entry points resolved at run time (the process's already-loaded libnccl --
// torch's -- is preferred, so one NCCL serves both).
namespace {
typedef int (*nccl_allgather_t)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_get_id_t)(void *);
struct NcclId { char internal[128]; };
typedef int (*nccl_init_rank_t)(void **, int, NcclId, int);
typedef int (*nccl_destroy_t)(void *);
typedef const char *(*nccl_errstr_t)(int);

void *nccl_lib() {
    static void *h = nullptr;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    return h;
}
template <typename F>
F nccl_sym(const char *name) {
    void *l = nccl_lib();
    return l ? reinterpret_cast<F>(dlsym(l, name)) : nullptr;
}
lapssd_status nccl_status(int rc, const char *what) {
    if (rc == 0) return LAPSSD_OK;
    auto es = nccl_sym<nccl_errstr_t>("ncclGetErrorString");
    return fail(LAPSSD_ENCCL, "%s: %s", what, es ? es(rc) : "nccl error");
}
constexpr int kNcclUint64 = 5;
}  // namespace

extern "C" {

lapssd_status lapssd_nccl_unique_id(uint8_t id_out[128]) {
    auto f = nccl_sym<nccl_get_id_t>("ncclGetUniqueId");
    if (!f) return fail(LAPSSD_ENCCL, "libnccl.so.2 not loadable");
    NcclId id;
    const int rc = f(&id);
    if (rc == 0) memcpy(id_out, id.internal, 128);
    return nccl_status(rc, "ncclGetUniqueId");
}

lapssd_status lapssd_nccl_comm_init(void **comm_out, int32_t nranks, const uint8_t id[128], int32_t rank) {
    auto f = nccl_sym<nccl_init_rank_t>("ncclCommInitRank");
    if (!f) return fail(LAPSSD_ENCCL, "libnccl.so.2 not loadable");
    NcclId nid;
    memcpy(nid.internal, id, 128);
    return nccl_status(f(comm_out, nranks, nid, rank), "ncclCommInitRank");
}

lapssd_status lapssd_nccl_comm_destroy(void *comm) {
    auto f = nccl_sym<nccl_destroy_t>("ncclCommDestroy");
    if (!f) return fail(LAPSSD_ENCCL, "libnccl.so.2 not loadable");
    return nccl_status(f(comm), "ncclCommDestroy");
}

// The multi-GPU step.  allgather == nullptr (laps_step_candidates): stop once this rank's
// candidate block is in cand_scratch[0, 2C+1) and joined into `stream`; the caller
// exchanges the blocks with any collective and calls laps_merge.
static lapssd_status step_dist(lapssd_handle *h, void *nccl_comm, nccl_allgather_t allgather, const lapssd_rows *rows,
                               int32_t B_global, int32_t C, int32_t *sel_inout, int32_t *count_out,
                               int32_t *tokens_out, int32_t *n_accept_out, uint64_t *cand_scratch, cudaStream_t s,
                               const char *who) {
    VerifyArgs a;
    lapssd_status st = fill_step_verify(h, rows, B_global, sel_inout, tokens_out, n_accept_out, a);
    if (st != LAPSSD_OK) return st;
    a.count_dev = &h->st.g->count;   // this rank's slots are [0, count) of the B_global
    h->last_stream = s;
    uint64_t *local = cand_scratch;                 // this rank's block: 2C+1 words
    uint64_t *all = cand_scratch + (2 * (size_t)C + 1);
    int bp = 1;
    while (bp < B_global) bp <<= 1;
    static const bool serial = getenv("LAPSSD_DIST_SERIAL") != nullptr;  // A/B switch
    const bool overlapped = !serial && rows->slab_tab != nullptr && bp <= 4096 && C <= B_global;
    if (!overlapped) {   // verify, then candidates -> all-gather -> merge on the stream
        st = step_verify(h, a, sel_inout, B_global, s);
        if (st != LAPSSD_OK) return st;
        st = cuda_status(launch_candidates(h->st, h->sc, C, local, s), who);
        if (st != LAPSSD_OK || !allgather) return st;
        st = nccl_status(allgather(local, all, 2 * (size_t)C + 1, kNcclUint64, nccl_comm, s), "ncclAllGather");
        if (st != LAPSSD_OK) return st;
        st = cuda_status(launch_merge(h->st, h->sc, a.rows, h->desc, all, C, B_global, sel_inout, count_out, s),
                         who);
        if (st == LAPSSD_OK) h->desc_valid = true;
        return st;
    }
    // Overlapped as laps_step: the verify kernel (finishers run a3 and publish records)
    // on the stream; on the side stream the select kernel builds this rank's candidates
    // from the presort + the published records, the all-gather and the global merge +
    // commit follow, all while the rows stream.  The merge kernel ends with the fenced
    // trigger the next (programmatic) verify launch needs.
    if (!h->desc_valid) {
        st = cuda_status(launch_accept(a.rows, sel_inout, &h->st, &h->sc, nullptr, nullptr, nullptr, h->sc.seed, 0,
                                       B_global, h->desc, s), "accept");
        if (st != LAPSSD_OK) return st;
    }
    cudaError_t ce = cudaEventRecord(h->ev_fork, s);
    if (ce != cudaSuccess) return cuda_status(ce, "step fork");
    h->desc_valid = false;
    a.fin = h->fin;
    a.fin_key = h->fin_key;
    a.snap = h->snap;
    a.part1 = h->part + (size_t)h->max_batch * h->n_chunks * kPartWords;
    a.work1 = h->work + 2;
    a.vstep = &h->st.g->vstep;
    static const bool no_pdl = getenv("LAPSSD_NO_PDL") != nullptr;
    // the split form's merge runs on the caller's stream after a collective of the
    // caller's choosing: the next verify then follows it in plain stream order
    st = cuda_status(launch_verify_grid(a, B_global, 1, allgather && h->overlap && !no_pdl, s), who);
    if (st != LAPSSD_OK) return st;
    ce = cudaStreamWaitEvent(h->side, h->ev_fork, 0);
    if (ce != cudaSuccess) return cuda_status(ce, "step fork wait");
    st = cuda_status(launch_select_side(h->st, h->sc, a.rows, sel_inout, h->desc, B_global, h->pre, h->fin,
                                        h->fin_key, h->snap, (uint32_t)verify_grid(B_global, a.n_chunks, 1),
                                        nullptr, h->side, local, C),
                     who);
    if (st != LAPSSD_OK) return st;
    if (allgather) {
        st = nccl_status(allgather(local, all, 2 * (size_t)C + 1, kNcclUint64, nccl_comm, h->side), "ncclAllGather");
        if (st != LAPSSD_OK) return st;
        st = cuda_status(launch_merge(h->st, h->sc, a.rows, h->desc, all, C, B_global, sel_inout, count_out, h->side),
                         who);
        if (st != LAPSSD_OK) return st;
    }
    ce = cudaEventRecord(h->ev_join, h->side);
    if (ce != cudaSuccess) return cuda_status(ce, "step join");
    ce = cudaStreamWaitEvent(s, h->ev_join, 0);
    if (ce != cudaSuccess) return cuda_status(ce, "step join wait");
    h->desc_valid = allgather != nullptr;   // laps_merge (no rows) leaves the next a1 to the next call
    return LAPSSD_OK;
}

lapssd_status laps_step_dist(lapssd_handle *h, void *nccl_comm, const lapssd_rows *rows, int32_t B_global,
                             int32_t C, int32_t *sel_inout, int32_t *count_out, int32_t *tokens_out,
                             int32_t *n_accept_out, uint64_t *cand_scratch, lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || !nccl_comm || !cand_scratch || B_global < 1 || B_global > h->max_batch || C < 1)
        return fail(LAPSSD_EINVAL, "handle / comm / scratch / B_global / C");
    if ((int64_t)h->sc.world * C > sort_capacity())
        return fail(LAPSSD_EINVAL, "world*C exceeds %d", sort_capacity());
    auto allgather = nccl_sym<nccl_allgather_t>("ncclAllGather");
    if (!allgather) return fail(LAPSSD_ENCCL, "ncclAllGather not found");
    return step_dist(h, nccl_comm, allgather, rows, B_global, C, sel_inout, count_out, tokens_out, n_accept_out,
                     cand_scratch, (cudaStream_t)stream, "laps_step_dist");
}

size_t lapssd_peer_buffer_bytes(int32_t world, int32_t C) {
    if (world < 1 || world > 64 || C < 1) return 0;
    return (size_t)2 * world * (2 * (size_t)C + 2) * sizeof(uint64_t);
}

lapssd_status lapssd_set_peers(lapssd_handle *h, void *const *peer_bufs, int32_t C, lapssd_stream stream) {
    g_last_error.clear();
    if (!h || !peer_bufs || C < 1) return fail(LAPSSD_EINVAL, "handle / peer_bufs / C");
    if (h->sc.world > 64) return fail(LAPSSD_EINVAL, "world > 64");
    if ((int64_t)h->sc.world * C > sort_capacity()) return fail(LAPSSD_EINVAL, "world*C exceeds %d", sort_capacity());
    for (int32_t g = 0; g < h->sc.world; ++g)
        if (!peer_bufs[g] || ((uintptr_t)peer_bufs[g] & 7)) return fail(LAPSSD_EINVAL, "peer buffer %d", g);
    h->peer_C = C;
    return cuda_status(cudaMemcpyAsync(h->peer_ptrs, peer_bufs, sizeof(void *) * h->sc.world, cudaMemcpyHostToDevice,
                                       (cudaStream_t)stream),
                       "lapssd_set_peers");
}

lapssd_status laps_step_peer(lapssd_handle *h, const lapssd_rows *rows, int32_t B_global, int32_t *sel_inout,
                             int32_t *count_out, int32_t *tokens_out, int32_t *n_accept_out, lapssd_stream stream) {
    g_last_error.clear();
    if (!h || B_global < 1 || B_global > h->max_batch) return fail(LAPSSD_EINVAL, "handle / B_global");
    if (!h->peer_C) return fail(LAPSSD_EINVAL, "no peers set (lapssd_set_peers)");
    int bp = 1;
    while (bp < B_global) bp <<= 1;
    if (!rows || !rows->slab_tab || bp > 4096 || h->peer_C > B_global)
        return fail(LAPSSD_EINVAL, "laps_step_peer needs pooled rows, B_global <= 4096 and C <= B_global");
    VerifyArgs a;
    lapssd_status st = fill_step_verify(h, rows, B_global, sel_inout, tokens_out, n_accept_out, a);
    if (st != LAPSSD_OK) return st;
    a.count_dev = &h->st.g->count;   // this rank's slots are [0, count) of the B_global
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    if (!h->desc_valid) {
        st = cuda_status(launch_accept(a.rows, sel_inout, &h->st, &h->sc, nullptr, nullptr, nullptr, h->sc.seed, 0,
                                       B_global, h->desc, s), "accept");
        if (st != LAPSSD_OK) return st;
    }
    // as laps_step: after a peer step on the same stream the side stream is chained (its
    // select follows the previous select, which committed everything this one reads)
    cudaStreamCaptureStatus cap_s = cudaStreamCaptureStatusNone, cap_side = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap_s);
    cudaStreamIsCapturing(h->side, &cap_side);
    static const bool no_chain = getenv("LAPSSD_NO_SIDE_CHAIN") != nullptr;
    const bool capturing = cap_s == cudaStreamCaptureStatusActive;
    const bool fork = no_chain || !h->side_chained || h->chain_stream != s || cap_s != cap_side ||
                      capturing != h->chain_captured || !h->desc_valid;
    h->side_chained = false;
    cudaError_t ce = cudaSuccess;
    if (fork) {
        ce = cudaEventRecord(h->ev_fork, s);
        if (ce != cudaSuccess) return cuda_status(ce, "laps_step_peer fork");
    }
    h->desc_valid = false;
    a.fin = h->fin;
    a.fin_key = h->fin_key;
    a.snap = h->snap;
    a.part1 = h->part + (size_t)h->max_batch * h->n_chunks * kPartWords;
    a.work1 = h->work + 2;
    a.vstep = &h->st.g->vstep;
    static const bool no_pdl = getenv("LAPSSD_NO_PDL") != nullptr;
    st = cuda_status(launch_verify_grid(a, B_global, 1, h->overlap && !no_pdl, s), "laps_step_peer verify");
    if (st != LAPSSD_OK) return st;
    if (fork) {
        ce = cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        if (ce != cudaSuccess) return cuda_status(ce, "laps_step_peer fork wait");
    }
    static const bool no_wl = getenv("LAPSSD_NO_WAITLIST") != nullptr;
    const WaitList *wl = no_wl ? nullptr : &h->wl;
    const PeerArgs pa{h->peer_ptrs, h->peer_C};
    st = cuda_status(launch_select_side(h->st, h->sc, a.rows, sel_inout, h->desc, B_global, h->pre, h->fin,
                                        h->fin_key, h->snap, (uint32_t)verify_grid(B_global, a.n_chunks, 1), count_out,
                                        h->side, nullptr, 0, wl, &pa),
                     "laps_step_peer select");
    if (st != LAPSSD_OK) return st;
    h->wl.valid = wl != nullptr && bp <= 1024;
    ce = cudaEventRecord(h->ev_join, h->side);
    if (ce != cudaSuccess) return cuda_status(ce, "laps_step_peer join");
    ce = cudaStreamWaitEvent(s, h->ev_join, 0);
    if (ce != cudaSuccess) return cuda_status(ce, "laps_step_peer join wait");
    h->desc_valid = true;
    h->side_chained = true;
    h->chain_stream = s;
    h->chain_captured = capturing;
    return LAPSSD_OK;
}

lapssd_status laps_step_candidates(lapssd_handle *h, const lapssd_rows *rows, int32_t B_global, int32_t C,
                                   int32_t *sel_inout, int32_t *tokens_out, int32_t *n_accept_out,
                                   uint64_t *cand_out, lapssd_stream stream) {
    g_last_error.clear();
    if (h) { h->side_chained = false; h->wl.valid = 0; }
    if (!h || !cand_out || B_global < 1 || B_global > h->max_batch || C < 1)
        return fail(LAPSSD_EINVAL, "handle / cand_out / B_global / C");
    if ((int64_t)h->sc.world * C > sort_capacity())
        return fail(LAPSSD_EINVAL, "world*C exceeds %d", sort_capacity());
    return step_dist(h, nullptr, nullptr, rows, B_global, C, sel_inout, nullptr, tokens_out, n_accept_out,
                     cand_out, (cudaStream_t)stream, "laps_step_candidates");
}

// ---------------------------------------------------------------- snapshot / check
lapssd_status lapssd_read_state(lapssd_handle *h, lapssd_state_view *v, lapssd_stream stream) {
    g_last_error.clear();
    if (h) h->side_chained = false;   // (reads only: the waiting list stays valid)
    if (!h || !v) return fail(LAPSSD_EINVAL, "handle / view");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)h->sc.n;
    Globals g{};
    std::vector<uint32_t> flags(n);
    cudaError_t e = cudaMemcpyAsync(&g, h->st.g, sizeof g, cudaMemcpyDeviceToHost, s);
#define CP(dst, src, cnt)                                                                          \
    if (e == cudaSuccess && (dst)) e = cudaMemcpyAsync((dst), (src), sizeof(*(dst)) * (cnt), cudaMemcpyDeviceToHost, s);
    CP(v->acc_tok, h->st.acc_tok, n)
    CP(v->acc_draft, h->st.acc_draft, n)
    CP(v->rounds, h->st.rounds, n)
    CP(v->E_us, h->st.E, n)
    CP(v->T_total_us, h->st.T_total, n)
    CP(v->C_us, h->st.C, n)
    CP(v->x_us, h->st.x, n)
    CP(v->A, h->st.A, n)
    CP(v->key, h->st.key, n)
    CP(v->ring, h->st.ring, n * h->sc.gamma)
    CP(v->switch_us, h->st.switch_us, n)
#undef CP
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(flags.data(), h->st.flags, 4 * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "lapssd_read_state");
    v->now_us = g.now_us;
    v->cursor = g.cursor;
    v->prev_count = g.prev_count;
    v->step_cost_us = h->sc.c_round_us + g.step_sw;
    v->switch_total_us = g.switch_total;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t f = flags[i];
        if (v->admitted) v->admitted[i] = (int32_t)i < g.cursor;
        if (v->done) v->done[i] = (f & F_DONE) != 0;
        if (v->perceptible) v->perceptible[i] = (f & F_PERC) != 0;
        if (v->pinned) v->pinned[i] = (f & F_PINNED) != 0;
        if (v->running) v->running[i] = (f & F_RUNNING) != 0;
        if (v->level) v->level[i] = (uint8_t)((f & F_LEVEL_MASK) >> F_LEVEL_SHIFT);
    }
    return LAPSSD_OK;
}

lapssd_status lapssd_check(lapssd_handle *h, uint32_t *flags_out) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    Globals g{};
    cudaError_t e = cudaStreamSynchronize(h->last_stream);
    if (e == cudaSuccess) e = cudaMemcpy(&g, h->st.g, sizeof g, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "lapssd_check");
    if (flags_out) *flags_out = g.err;
    if (g.err) return fail(LAPSSD_ESTATE, "device contract violation flags 0x%x (first watchdog: step %u slot %u)",
                           g.err, g.err_where >> 16, g.err_where & 0xFFFFu);
    return LAPSSD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- Monte-Carlo replicas

struct lapssd_mc {
    State st;
    Sched sc;
    McDev mc{};
    SlotDesc *desc = nullptr;   // [T] a1 of each trace's selected request
    int32_t *sel = nullptr, *n_accept = nullptr, *tokens = nullptr, *active = nullptr;
    uint64_t *part = nullptr;   // verify scratch: two sets (consecutive sub-launches overlap)
    uint32_t *work = nullptr;   // [4]: two (claim, retired) counter pairs
    uint32_t *par = nullptr;    // [2] = {0, 1}: the set a sub-launch uses (its "step parity")
    size_t part_set = 0;        // words per set
    int32_t T = 0, bmax = 0;
    int64_t n = 0, V = 0;
    cudaStream_t last_stream = nullptr;
};

static void carve_mc(Carver &cv, lapssd_mc *h, int32_t T, int64_t n, int32_t gamma, int32_t k, int64_t V) {
    carve_state(cv, h->st, n, gamma);
    const size_t tt = (size_t)(T > 0 ? T : 1);
    h->mc.g = cv.take<Globals>(tt);
    h->mc.off = cv.take<int64_t>(tt + 1);
    h->mc.last = cv.take<int32_t>(tt);
    h->desc = cv.take<SlotDesc>(tt);
    h->sel = cv.take<int32_t>(tt);
    h->n_accept = cv.take<int32_t>(tt);
    h->tokens = cv.take<int32_t>(tt * (size_t)(k + 1));
    h->active = cv.take<int32_t>(1);
    const int32_t nc = n_chunks_max(V);
    const int32_t bmax = verify_max_batch(nc, 0);
    const int32_t nb = T < bmax ? (T > 0 ? T : 1) : bmax;
    h->part_set = (size_t)nb * nc * kPartWords;
    h->part = cv.take<uint64_t>(2 * h->part_set);
    h->work = cv.take<uint32_t>(4);
    h->par = cv.take<uint32_t>(2);
}

extern "C" {

size_t lapssd_mc_workspace_bytes(const lapssd_config *cfg, int32_t n_traces, int64_t n_total, int64_t V) {
    if (!cfg || n_traces < 1 || n_total < 0 || V < 1) return 0;
    prepare_all();   // the verify sub-launch size depends on the SM count
    lapssd_mc tmp{};
    Carver cv{nullptr};
    carve_mc(cv, &tmp, n_traces, n_total, cfg->gamma > 0 ? cfg->gamma : 1, cfg->k > 0 ? cfg->k : 1, V);
    return align256(cv.off);
}

lapssd_status lapssd_mc_create(const lapssd_config *cfg, int32_t n_traces, const int64_t *trace_offsets,
                               const int64_t *arrival_us, const int32_t *L_true, const int32_t *L_pred,
                               const int32_t *prompt, int64_t V,
                               void *workspace, size_t workspace_bytes, lapssd_stream stream, lapssd_mc **out) {
    g_last_error.clear();
    if (!out) return fail(LAPSSD_EINVAL, "out is NULL");
    *out = nullptr;
    lapssd_status st = check_config(cfg);
    if (st != LAPSSD_OK) return st;
    if (n_traces < 1 || !trace_offsets) return fail(LAPSSD_EINVAL, "n_traces / trace_offsets");
    if (trace_offsets[0] != 0) return fail(LAPSSD_EINVAL, "trace_offsets[0] must be 0");
    const int64_t n = trace_offsets[n_traces];
    if (n > ((int64_t)1 << 31) - 1) return fail(LAPSSD_EINVAL, "more than 2^31-1 requests");
    if (n > 0 && (!arrival_us || !L_true || !L_pred)) return fail(LAPSSD_EINVAL, "requests: NULL arrays");
    if (V < 1 || V > (int64_t)kMaxSegs * kSegElems) return fail(LAPSSD_EINVAL, "V out of range");
    for (int32_t t = 0; t < n_traces; ++t) {
        const int64_t a = trace_offsets[t], b = trace_offsets[t + 1];
        if (b < a) return fail(LAPSSD_EINVAL, "trace_offsets not non-decreasing at %d", t);
        if (b - a > (1 << 24) - 2) return fail(LAPSSD_EINVAL, "trace %d: local ids must be < 2^24 - 1", t);
        for (int64_t i = a; i < b; ++i) {
            if (L_true[i] < 1 || L_pred[i] < 1) return fail(LAPSSD_EINVAL, "L < 1 at %lld", (long long)i);
            if (prompt && prompt[i] < 0) return fail(LAPSSD_EINVAL, "prompt < 0 at %lld", (long long)i);
            if (i > a && arrival_us[i] < arrival_us[i - 1])
                return fail(LAPSSD_EINVAL, "trace %d: arrivals not sorted at %lld", t, (long long)i);
        }
    }
    const size_t need = lapssd_mc_workspace_bytes(cfg, n_traces, n, V);
    if (!workspace || workspace_bytes < need)
        return fail(LAPSSD_ENOMEM, "workspace %zu < %zu bytes", workspace_bytes, need);
    prepare_all();
    lapssd_mc *h = new lapssd_mc{};
    Carver cv{(char *)workspace};
    carve_mc(cv, h, n_traces, n, cfg->gamma, cfg->k, V);
    h->T = n_traces;
    h->n = n;
    h->V = V;
    h->bmax = verify_max_batch(n_chunks_max(V), 0);
    h->mc.T = n_traces;
    fill_sched(h->sc, cfg, 0, 0, 1);   // every trace is its own id space (world 1, local ids)
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    cudaError_t e = init_state(workspace, need, h->st, n, arrival_us, L_true, L_pred, prompt, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync((void *)h->mc.off, trace_offsets, sizeof(int64_t) * (n_traces + 1),
                            cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->sel, 0xFF, sizeof(int32_t) * n_traces, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->mc.last, 0xFF, sizeof(int32_t) * n_traces, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->par + 1, 0x01, 1, s);   // par = {0, 1}
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        delete h;
        return cuda_status(e, "lapssd_mc_create");
    }
    *out = h;
    return LAPSSD_OK;
}

lapssd_status lapssd_mc_destroy(lapssd_mc *h) {
    delete h;
    return LAPSSD_OK;
}

lapssd_status laps_mc_select(lapssd_mc *h, const lapssd_rows *rows, lapssd_stream stream) {
    g_last_error.clear();
    if (!h || !rows || !rows->slab_tab || rows->k != h->sc.k || rows->R < 1)
        return fail(LAPSSD_EINVAL, "handle / rows (pooled layout with slab_tab required)");
    if (!rows_ok(rows->dtype, rows->V, rows->k, rows->p, rows->q) || rows->V > h->V)
        return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    const RowsDev rw = rows_dev(rows->p, rows->q, rows->draft, rows->slab_tab, rows->V, rows->k, rows->R, rows->dtype);
    return cuda_status(launch_mc_step(h->st, h->sc, h->mc, rw, nullptr, h->desc, h->sel, nullptr, s),
                       "laps_mc_select");
}

lapssd_status laps_mc_step(lapssd_mc *h, const lapssd_rows *rows, int32_t *tokens_out, int32_t *n_accept_out,
                           int32_t *active_out, lapssd_stream stream) {
    g_last_error.clear();
    if (!h || !rows || !rows->slab_tab || rows->k != h->sc.k || rows->R < 1)
        return fail(LAPSSD_EINVAL, "handle / rows (pooled layout with slab_tab required)");
    if (!rows_ok(rows->dtype, rows->V, rows->k, rows->p, rows->q) || rows->V > h->V)
        return fail(LAPSSD_EINVAL, "rows: dtype/V/alignment");
    cudaStream_t s = (cudaStream_t)stream;
    h->last_stream = s;
    const RowsDev rw = rows_dev(rows->p, rows->q, rows->draft, rows->slab_tab, rows->V, rows->k, rows->R, rows->dtype);
    int32_t *tok = tokens_out ? tokens_out : h->tokens;
    int32_t *na = n_accept_out ? n_accept_out : h->n_accept;
    // a2: one verified request per trace (slot t), in sub-launches the kernel's per-CTA
    // snapshot holds
    VerifyArgs a{};
    a.rows = rw;
    a.n_chunks = n_chunks_of(rows->V, rows->dtype);
    a.cpb = verify_cpb(rows->V);
    a.seed = h->sc.seed;
    a.part = h->part;
    a.work = h->work;
    a.fuse_update = 0;
    a.err = &h->st.g->err;
    a.part1 = h->part + h->part_set;
    a.work1 = h->work + 2;
    if (active_out) {   // before the verify launches: the select follows the last one directly
        const cudaError_t e = cudaMemsetAsync(active_out, 0, sizeof(int32_t), s);
        if (e != cudaSuccess) return cuda_status(e, "laps_mc_step");
    }
    lapssd_status st = LAPSSD_OK;
    static const bool no_pdl = getenv("LAPSSD_NO_PDL") != nullptr;
    int j = 0;
    for (int32_t b0 = 0; b0 < h->T && st == LAPSSD_OK; b0 += h->bmax, ++j) {
        VerifyArgs ab = a;
        const int32_t nb = h->T - b0 < h->bmax ? h->T - b0 : h->bmax;
        ab.desc = h->desc + b0;
        ab.tokens = tok + (int64_t)b0 * (rows->k + 1);
        ab.n_accept = na + b0;
        ab.vstep = h->par + (j & 1);   // alternate scratch sets
        // the second sub-launch overlaps the first's tail (programmatic dependent launch:
        // its CTAs take SMs as the first's retire; it reads nothing the first writes).  A
        // third one would share the first's set, so only j == 1 overlaps.
        st = cuda_status(launch_verify_grid(ab, nb, 0, j == 1 && !no_pdl, s), "laps_mc_step verify");
    }
    if (st != LAPSSD_OK) return st;
    // a3 + a4-a7 + a1, one warp per trace
    return cuda_status(launch_mc_step(h->st, h->sc, h->mc, rw, na, h->desc, h->sel, active_out, s),
                       "laps_mc_step update/select");
}

lapssd_status lapssd_mc_read(lapssd_mc *h, lapssd_state_view *v, int64_t *now_us, int32_t *cursor, int32_t *sel,
                             lapssd_stream stream) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)h->n, T = (size_t)h->T;
    std::vector<Globals> g(T);
    std::vector<uint32_t> flags(n);
    std::vector<int64_t> off(T + 1);
    cudaError_t e = cudaMemcpyAsync(g.data(), h->mc.g, sizeof(Globals) * T, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(off.data(), h->mc.off, sizeof(int64_t) * (T + 1), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && sel) e = cudaMemcpyAsync(sel, h->sel, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, s);
#define CP(dst, src, cnt)                                                                          \
    if (e == cudaSuccess && v && (dst)) e = cudaMemcpyAsync((dst), (src), sizeof(*(dst)) * (cnt), cudaMemcpyDeviceToHost, s);
    CP(v->acc_tok, h->st.acc_tok, n)
    CP(v->acc_draft, h->st.acc_draft, n)
    CP(v->rounds, h->st.rounds, n)
    CP(v->E_us, h->st.E, n)
    CP(v->T_total_us, h->st.T_total, n)
    CP(v->C_us, h->st.C, n)
    CP(v->x_us, h->st.x, n)
    CP(v->A, h->st.A, n)
    CP(v->key, h->st.key, n)
    CP(v->ring, h->st.ring, n * h->sc.gamma)
    CP(v->switch_us, h->st.switch_us, n)
#undef CP
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(flags.data(), h->st.flags, 4 * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "lapssd_mc_read");
    if (v) {   // per-trace scalars have no place in the view: the totals over the traces
        v->step_cost_us = 0;
        v->switch_total_us = 0;
        for (size_t t = 0; t < T; ++t) v->switch_total_us += g[t].switch_total;
    }
    for (size_t t = 0; t < T; ++t) {
        if (now_us) now_us[t] = g[t].now_us;
        if (cursor) cursor[t] = g[t].cursor;
        if (!v) continue;
        for (int64_t i = off[t]; i < off[t + 1]; ++i) {
            const uint32_t f = flags[i];
            if (v->admitted) v->admitted[i] = (int32_t)(i - off[t]) < g[t].cursor;
            if (v->done) v->done[i] = (f & F_DONE) != 0;
            if (v->perceptible) v->perceptible[i] = (f & F_PERC) != 0;
            if (v->pinned) v->pinned[i] = (f & F_PINNED) != 0;
            if (v->running) v->running[i] = (f & F_RUNNING) != 0;
            if (v->level) v->level[i] = (uint8_t)((f & F_LEVEL_MASK) >> F_LEVEL_SHIFT);
        }
    }
    return LAPSSD_OK;
}

lapssd_status lapssd_mc_check(lapssd_mc *h, uint32_t *flags_out) {
    g_last_error.clear();
    if (!h) return fail(LAPSSD_EINVAL, "handle is NULL");
    Globals g{};
    cudaError_t e = cudaStreamSynchronize(h->last_stream);
    if (e == cudaSuccess) e = cudaMemcpy(&g, h->st.g, sizeof g, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "lapssd_mc_check");
    if (flags_out) *flags_out = g.err;
    if (g.err) return fail(LAPSSD_ESTATE, "device contract violation flags 0x%x (first watchdog: step %u slot %u)",
                           g.err, g.err_where >> 16, g.err_where & 0xFFFFu);
    return LAPSSD_OK;
}

}  // extern "C"
