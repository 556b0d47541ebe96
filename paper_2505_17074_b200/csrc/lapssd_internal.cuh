// lapssd_internal.cuh -- device-side layout and helpers of liblapssd.so (sm_100a).
//
// Product code.  Written from PAPER.md (arXiv 2505.17074) and include/lapssd.h; it
// shares nothing with oracle/.  "P:NN" = PAPER.md line NN, "AMB-n" = DESIGN.md s.3.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lapssd.h"

namespace lapssd {

// ---------------------------------------------------------------- verify tiling
// A work item is chunk c of one row pair: kTileBytes of p_r (and of q_r) -- 16384 bf16
// or 8192 fp32 entries -- split into segments of 1024 entries, each reduced to one
// published u64.  32 KB per row per item: the longest contiguous bulk copy per SM that
// still leaves three ring stages in shared memory (tools/rows_bench.cu: 16 KB items
// stream at 5.7 TB/s, 32 KB items at 6.4 TB/s on the same access pattern).
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSegElems = 1024;                 // entries per published segment sum
constexpr int kTileBytes = 32768;               // bytes of one row per work item
constexpr int kMaxSegs = 512;                   // segments per row: V <= 524288
constexpr int kPartWords = 16;                  // published words per chunk (16 bf16 / 8 fp32 segments)
__host__ __device__ constexpr int tile_elems(int esz) { return kTileBytes / esz; }

// ---------------------------------------------------------------- state flags
enum : uint32_t {
    F_DONE = 1u, F_PERC = 2u, F_PINNED = 4u, F_RUNNING = 8u,
    F_LEVEL_SHIFT = 8u, F_LEVEL_MASK = 0xF00u,
};
enum : uint32_t {
    E_UPDATE_DONE = 1u,    // update on a completed request
    E_NO_MASS = 2u,        // a row with no probability mass at all
    E_BAD_SLOT = 4u,       // slot refers to an out-of-range request
    E_TIMEOUT = 16u,       // a device-side wait exceeded its watchdog (results invalid)
    E_TO_FIN = 32u,        // ... the verify finisher's wait for a slot's segment sums
    E_TO_MERGE = 64u,      // ... the side select's wait for the verified slots' records
    E_TO_SNAP = 128u,      // ... the side select's wait for the verify CTAs' snapshots
    E_MASS = 256u,         // a row pair with residual mass > 2 (not probability rows): sums invalid
    E_TO_PEER = 512u,      // ... (with E_TIMEOUT) the side select's wait for the peers' candidate blocks
};

// Watchdog for device-side spin waits: true once `t0` is more than 2 s in the past.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool waited_too_long(unsigned long long t0) { return gtimer() - t0 > 2000000000ull; }

struct Globals {
    int64_t now_us;
    int32_t cursor;        // requests [0, cursor) are admitted (arrivals sorted)
    int32_t prev_count;    // size of the batch that ran last (global for G > 1)
    int32_t count;         // size of the batch just selected (this rank)
    uint32_t err;          // sticky contract-violation flags
    uint32_t vstep;        // incremental steps committed: parity of the verify buffers
    uint32_t err_where;    // first watchdog expiry: (vstep & 0xFFFF) << 16 | slot
    uint32_t sel_seq;      // selections committed (a request in the batch that ran last has last_sel == sel_seq)
    int64_t step_sw;       // switch-in time of the batch selected last: its step lasts c_round + step_sw (AMB-24)
    int64_t switch_total;  // system time spent switching (AMB-24)
};

// Scheduler constants, passed by value to every kernel.
struct Sched {
    int32_t policy, K, gamma, k;
    int32_t placement, pin_rule;
    int32_t n, rank, world;
    int32_t cost_model;    // LAPSSD_COST_EQ6 / LAPSSD_COST_FIG1
    int32_t sw_on;         // switching cost configured (c0 or c1 > 0)
    double delta;
    int64_t t_ssm_us, t_llm_us, t_tok_us, c_round_us;
    int64_t sw_c0_us, sw_c1_us;
    int64_t S_up[16];
    uint64_t seed;
};

// Resident-request SoA in the caller's workspace.
struct State {
    const int64_t *arrival;
    const int32_t *L_true, *L_pred, *prompt;
    int32_t *last_sel;     // sel_seq of the request's last selection (-1: never)
    int64_t *switch_us;    // switching time charged on the request's entries
    int32_t *acc_tok, *acc_draft, *rounds, *ring;
    int64_t *E, *T_total, *C, *x;
    double *A;
    uint32_t *flags;
    uint64_t *key;
    Globals *g;
    // a1 of the request's NEXT round, computed by the verify finisher off the critical
    // path: valid iff next_tag == (rows_epoch << 32 | rounds[i]).
    uint64_t *next_tag;
    int2 *next_sr;         // (slab, r)
};

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al., SC'11.  Counter (c0..c3) = (request id, round, (tag<<8)|block,
// trace), key = (seed lo, seed hi) (AMB-21).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

// ---------------------------------------------------------------- Eq. (6)
// floor( (L * (k T_SSM + T_LLM)) / (k A + 1) ), fp64 round-to-nearest ops in this
// order (AMB-10).  Explicit _rn intrinsics: never contracted into an FMA.
__device__ __forceinline__ uint64_t eq6_us(int64_t L, double A, const Sched &s) {
    const double num = __dmul_rn((double)L, (double)s.c_round_us);
    const double den = __dadd_rn(__dmul_rn((double)s.k, A), 1.0);
    const double T = __ddiv_rn(num, den);
    if (!(T > 0.0)) return 0;
    if (T >= 1.8e19) return ~0ull;
    return (uint64_t)T;
}

// The Fig. 1 model: L tokens at acceptance rate A need L / A candidates, each
// verified in t_tok: floor((L * t_tok) / A) in fp64, in this order (AMB-31).  A = 0 has
// no finite estimate (saturates) unless nothing is left to generate.
__device__ __forceinline__ uint64_t fig1_us(int64_t L, double A, const Sched &s) {
    const double num = __dmul_rn((double)L, (double)s.t_tok_us);
    const double T = __ddiv_rn(num, A);
    if (!(T > 0.0)) return (L > 0 && s.t_tok_us > 0) ? ~0ull : 0;
    if (T >= 1.8e19) return ~0ull;
    return (uint64_t)T;
}

// T~ of L tokens at rate A under the configured cost model (P:139, P:198 / P:25-26).
__device__ __forceinline__ uint64_t estimate_us(int64_t L, double A, const Sched &s) {
    return s.cost_model == LAPSSD_COST_FIG1 ? fig1_us(L, A, s) : eq6_us(L, A, s);
}

// Switching cost of local request i entering the batch now (AMB-24): 0 if
// it was in the batch that ran last (its last selection is the latest, seq), else
// c0 + c1 (prompt + generated tokens).
__device__ __forceinline__ int64_t switch_in_cost(const State &st, const Sched &s, int32_t i, uint32_t seq) {
    if (!s.sw_on || st.last_sel[i] == (int32_t)seq) return 0;
    return s.sw_c0_us + s.sw_c1_us * ((int64_t)st.prompt[i] + st.acc_tok[i]);
}
// Charge a committed selection (selection number seq + 1) to request i.
__device__ __forceinline__ void charge_switch(const State &st, const Sched &s, int32_t i, uint32_t seq, int64_t c) {
    if (!s.sw_on) return;
    st.last_sel[i] = (int32_t)(seq + 1);
    if (c) st.switch_us[i] += c;
}

// Queue index of attained service / estimate x (AMB-11).
__device__ __forceinline__ int32_t level_of(int64_t x, const Sched &s) {
    int32_t lev = 0;
    while (lev < s.K - 1 && x >= s.S_up[lev]) ++lev;
    return lev;
}

__device__ __forceinline__ uint64_t sat32(uint64_t v) { return v > 0xFFFFFFFFull ? 0xFFFFFFFFull : v; }

// The 64-bit priority key (include/lapssd.h, laps_select).  Smaller = sooner.
// All state fields are passed in (loaded together by the caller: one memory round trip).
#ifdef LAPSSD_SIDE_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
uint64_t build_key(const Sched &s, int32_t i, int32_t cursor, uint32_t fl,
                                              int32_t L_pred, int32_t acc_tok, double A) {
    const uint64_t id = (uint64_t)(i * s.world + s.rank) & 0xFFFFFFull;
    const uint64_t inelig = (i >= cursor || (fl & F_DONE)) ? 1 : 0;
    const uint64_t pinned = (fl & F_PINNED) ? 1 : 0;
    const uint64_t perc = (fl & F_PERC) ? 1 : 0;
    const uint64_t running = (fl & F_RUNNING) ? 1 : 0;
    const uint64_t level = (fl & F_LEVEL_MASK) >> F_LEVEL_SHIFT;
    uint64_t unpinned = 0, lev = 0, nonperc = 0, notrun = 0, sec = 0;
    switch (s.policy) {
    case LAPSSD_POL_FCFS:                           // P:26, non-preemptive
        unpinned = !pinned;
        break;
    case LAPSSD_POL_LPSJF:                          // P:276, SJF on L_pred
        unpinned = !pinned;
        sec = sat32((uint64_t)L_pred);
        break;
    case LAPSSD_POL_LAS:
        unpinned = 1; lev = level; nonperc = 1; notrun = !running;
        break;
    default:                                        // LAPS-SD
        unpinned = !pinned; lev = level; nonperc = !perc;
        if (perc) {
            int64_t L_rem = (int64_t)L_pred - acc_tok;                  // AMB-12
            if (L_rem < 0) L_rem = 0;
            sec = sat32(estimate_us(L_rem, A, s));
        } else {
            notrun = !running;
        }
    }
    return (inelig << 63) | (unpinned << 62) | ((lev & 15) << 58) | (nonperc << 57) |
           (notrun << 56) | (sec << 24) | id;
}

// a3: the state update of local request i after a round with r accepted drafts.
// P:170 (E_i), P:175 (demotion), P:176 + P:194 (stability, A_i), P:139 + P:198
// (T~_i), P:148 (placement, AMB-14), P:177 (completion).  One thread per request.
// Returns the fields the request's new priority key needs.
struct UpdOut {    // the fields a priority key needs, after the update
    uint32_t fl;
    int32_t tok;
    double A;
};
// t_end: the end of the step that ran (now + c_round + its switch-ins): C_i if it completes.
__device__ __forceinline__ UpdOut update_one(const State &st, const Sched &s, int32_t i, int32_t r,
                                             int64_t t_end) {
    uint32_t fl = st.flags[i];
    double A_new = st.A[i];
    if (fl & F_DONE) { atomicOr(&st.g->err, E_UPDATE_DONE); return UpdOut{fl, st.acc_tok[i], A_new}; }
    const int32_t Lt = st.L_true[i];
    int32_t tok = st.acc_tok[i];
    const int32_t emitted = r + 1;                  // r drafts + 1 resampled / bonus
    const int32_t rem = Lt - tok;
    tok += emitted < rem ? emitted : rem;           // clipped at L (AMB-18)
    const int32_t acc = st.acc_draft[i] + r;        // AMB-4
    const int32_t t = st.rounds[i] + 1;
    const int64_t E = st.E[i] + s.c_round_us;
    int32_t *ring = st.ring + (int64_t)i * s.gamma;
    ring[t % s.gamma] = acc;
    int32_t level = (int32_t)((fl & F_LEVEL_MASK) >> F_LEVEL_SHIFT);
    bool demoted = false;
    if (s.policy == LAPSSD_POL_LAPSSD && !(fl & F_PERC)) {
        bool stable = false;
        double mean = 0.0;
        if (t >= s.gamma) {
            double mx = -1.0, mn = 2.0, sum = 0.0;
            for (int32_t sr = t - s.gamma + 1; sr <= t; ++sr) {          // oldest first
                const double rate = __ddiv_rn((double)ring[sr % s.gamma],
                                              (double)((int64_t)s.k * sr));
                mx = rate > mx ? rate : mx;
                mn = rate < mn ? rate : mn;
                sum = __dadd_rn(sum, rate);
            }
            if (__dsub_rn(mx, mn) < s.delta) { stable = true; mean = __ddiv_rn(sum, (double)s.gamma); }
        }
        if (stable) {
            fl |= F_PERC;
            st.A[i] = mean;
            A_new = mean;
            const uint64_t T = estimate_us(st.L_pred[i], mean, s);
            const int64_t Ts = T > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)T;
            st.T_total[i] = Ts;
            if (s.placement == 0) level = level_of(Ts, s);
            if (s.pin_rule == 1) fl |= F_PINNED;
        } else {
            const int32_t lev = level_of(E, s);
            if (lev > level) { level = lev; demoted = true; }
        }
    } else if (s.policy == LAPSSD_POL_LAS) {
        const int32_t lev = level_of(E, s);
        if (lev > level) { level = lev; demoted = true; }
    }
    if (tok >= Lt) {
        fl |= F_DONE;
        st.C[i] = t_end;
    }
    fl = (fl & ~(F_LEVEL_MASK | F_RUNNING)) | ((uint32_t)level << F_LEVEL_SHIFT);
    if (!(fl & F_DONE) && !demoted) fl |= F_RUNNING;
    st.acc_tok[i] = tok;
    st.acc_draft[i] = acc;
    st.rounds[i] = t;
    st.E[i] = E;
    st.flags[i] = fl;
    return UpdOut{fl, tok, A_new};
}

// Inputs of update_one for request i, loaded by the whole warp in one round trip
// (scalars broadcast, ring slot l in lane l).  gamma <= 32.
struct UpdIn {
    uint32_t fl;
    int32_t Lt, Lp, tok, acc, t;
    int64_t E;
    double A;
    int32_t ring;  // this lane's ring slot
};
__device__ __forceinline__ UpdIn load_update_inputs(const State &st, const Sched &s, int32_t i, int lane) {
    UpdIn u;   // L1-bypassing loads: the verify kernel reads state an overlapping grid wrote
    u.fl = __ldcg(st.flags + i);
    u.Lt = st.L_true[i];
    u.Lp = st.L_pred[i];
    u.tok = __ldcg(st.acc_tok + i);
    u.acc = __ldcg(st.acc_draft + i);
    u.t = __ldcg(st.rounds + i);
    u.E = __ldcg(st.E + i);
    u.A = __ldcg(st.A + i);
    u.ring = lane < s.gamma ? __ldcg(st.ring + (int64_t)i * s.gamma + lane) : 0;
    return u;
}

// update_one with preloaded inputs, executed by a full warp (uniform control flow,
// lane 0 stores).  Same arithmetic, same order as update_one.
__device__ __forceinline__ UpdOut update_warp(const State &st, const Sched &s, int32_t i, int32_t r, int64_t t_end,
                                              const UpdIn &u, int lane) {
    uint32_t fl = u.fl;
    UpdOut out{fl, u.tok, u.A};
    if (fl & F_DONE) {
        if (lane == 0) atomicOr(&st.g->err, E_UPDATE_DONE);
        return out;
    }
    int32_t tok = u.tok;
    const int32_t emitted = r + 1;                  // r drafts + 1 resampled / bonus
    const int32_t rem = u.Lt - tok;
    tok += emitted < rem ? emitted : rem;           // clipped at L (AMB-18)
    const int32_t acc = u.acc + r;                  // AMB-4
    const int32_t t = u.t + 1;
    const int64_t E = u.E + s.c_round_us;
    const int slot_new = t % s.gamma;
    const int32_t ring_lane = lane == slot_new ? acc : u.ring;   // ring after this round
    int32_t level = (int32_t)((fl & F_LEVEL_MASK) >> F_LEVEL_SHIFT);
    bool demoted = false;
    if (s.policy == LAPSSD_POL_LAPSSD && !(fl & F_PERC)) {
        bool stable = false;
        double mean = 0.0;
        if (t >= s.gamma) {
            double mx = -1.0, mn = 2.0, sum = 0.0;
            for (int32_t sr = t - s.gamma + 1; sr <= t; ++sr) {          // oldest first
                const int32_t a_s = __shfl_sync(0xFFFFFFFFu, ring_lane, sr % s.gamma);
                const double rate = __ddiv_rn((double)a_s, (double)((int64_t)s.k * sr));
                mx = rate > mx ? rate : mx;
                mn = rate < mn ? rate : mn;
                sum = __dadd_rn(sum, rate);
            }
            if (__dsub_rn(mx, mn) < s.delta) { stable = true; mean = __ddiv_rn(sum, (double)s.gamma); }
        }
        if (stable) {
            fl |= F_PERC;
            out.A = mean;
            const uint64_t T = estimate_us(u.Lp, mean, s);
            const int64_t Ts = T > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)T;
            if (lane == 0) { st.A[i] = mean; st.T_total[i] = Ts; }
            if (s.placement == 0) level = level_of(Ts, s);
            if (s.pin_rule == 1) fl |= F_PINNED;
        } else {
            const int32_t lev = level_of(E, s);
            if (lev > level) { level = lev; demoted = true; }
        }
    } else if (s.policy == LAPSSD_POL_LAS) {
        const int32_t lev = level_of(E, s);
        if (lev > level) { level = lev; demoted = true; }
    }
    if (tok >= u.Lt) {
        fl |= F_DONE;
        if (lane == 0) st.C[i] = t_end;
    }
    fl = (fl & ~(F_LEVEL_MASK | F_RUNNING)) | ((uint32_t)level << F_LEVEL_SHIFT);
    if (!(fl & F_DONE) && !demoted) fl |= F_RUNNING;
    if (lane == slot_new) st.ring[(int64_t)i * s.gamma + slot_new] = acc;
    if (lane == 0) {
        st.acc_tok[i] = tok;
        st.acc_draft[i] = acc;
        st.rounds[i] = t;
        st.E[i] = E;
        st.flags[i] = fl;
    }
    out.fl = fl;
    out.tok = tok;
    return out;
}

__host__ __device__ __forceinline__ int32_t slab_round_index(int32_t t, int32_t R) {
    const int32_t h = R / 2;
    if (t < R) return t;
    if (h == 0) return R - 1;
    return h + (t - h) % h;
}

// ---------------------------------------------------------------- rows + slot descriptors
// Where the probability rows live (device copy of lapssd_rows).
struct RowsDev {
    const void *p;
    const void *q;
    const int32_t *draft;
    const int32_t *slab_tab;    // nullable: batch layout (slot b reads slab b)
    int64_t V;
    int32_t k, R, dtype, valid;
    uint32_t epoch;        // host counter: changes whenever the rows descriptor changes
};

// Per-slot result of the acceptance test (a1), produced by accept_kernel or by the
// tail of select / merge, consumed by verify_kernel.  r < 0 marks an empty slot.
struct __align__(16) SlotDesc {
    int32_t i;        // local request index (-1 for stateless calls)
    int32_t slab;     // slab whose rows this slot reads
    uint32_t req;     // global request id (Philox c0)
    uint32_t round;   // round index (Philox c1)
    int32_t r;        // first rejected position, k if all accepted, -1 empty
    uint32_t trace;   // Philox c3 of the slot's draws (trace index: Monte-Carlo replicas)
    int32_t pad[2];
};

// a1 for one slot: x_j = draft[slab][j]; accept iff u24_j * q_j(x_j) < p_j(x_j) * 2^24
// (fp64, exact), u24_j = Philox(req, round, j/4, trace)[j%4] >> 8 (AMB-21).
// Returns the first rejected position, or k.  The k gathers are independent loads.
template <typename LoadF>
__device__ __forceinline__ int32_t accept_test(const RowsDev &rw, int64_t slab, uint32_t req,
                                               uint32_t rnd, uint32_t trace, uint64_t seed,
                                               LoadF load1) {
    const int k = rw.k;
    const int64_t V = rw.V;
    const int esz = rw.dtype == LAPSSD_BF16 ? 2 : 4;
    const char *pb = (const char *)rw.p + slab * (int64_t)(k + 1) * V * esz;
    const char *qb = (const char *)rw.q + slab * (int64_t)k * V * esz;
    const int32_t *db = rw.draft + slab * k;
    // positions in blocks of 8: within a block the 8 draft loads, then the 16 gathers,
    // are independent (two dependent memory round trips per block)
    for (int j0 = 0; j0 < k; j0 += 8) {
        int32_t x[8];
        float pj[8], qj[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) x[l] = (j0 + l < k) ? db[j0 + l] : 0;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            if (j0 + l < k) {
                pj[l] = load1(pb, (int64_t)(j0 + l) * V + x[l]);
                qj[l] = load1(qb, (int64_t)(j0 + l) * V + x[l]);
            } else {
                pj[l] = 1.0f; qj[l] = 0.0f;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint4 u = philox4x32_10(make_uint4(req, rnd, (uint32_t)(j0 / 4 + h), trace),
                                          (uint32_t)seed, (uint32_t)(seed >> 32));
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const int j = j0 + h * 4 + l;
                if (j < k) {
                    const uint32_t u24 = w[l] >> 8;
                    if (!(__dmul_rn((double)u24, (double)qj[h * 4 + l]) <
                          __dmul_rn((double)pj[h * 4 + l], 16777216.0)))
                        return j;
                }
            }
        }
    }
    return k;
}

__device__ __forceinline__ float load_prob_bf16(const void *base, int64_t idx) {
    return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(base)[idx] << 16);
}
__device__ __forceinline__ float load_prob_f32(const void *base, int64_t idx) {
    return reinterpret_cast<const float *>(base)[idx];
}

// Fill desc for slot b of a handle batch (local request i, or -1): the cached a1 of
// request i's current round if the finisher computed it for these rows, else a1 now.
#ifdef LAPSSD_SIDE_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
SlotDesc make_desc(const RowsDev &rw, const State &st, const Sched &sc,
                                              int32_t b, int32_t i) {
    SlotDesc d;
    d.i = i; d.slab = 0; d.req = 0; d.round = 0; d.r = -1;
    d.trace = 0; d.pad[0] = d.pad[1] = 0;
    if (i < 0) return d;
    const int32_t rnd = st.rounds[i];
    const uint64_t tag = st.next_tag[i];
    const int2 sr = st.next_sr[i];
    d.req = (uint32_t)(i * sc.world + sc.rank);
    d.round = (uint32_t)rnd;
    if (rw.slab_tab && tag == (((uint64_t)rw.epoch << 32) | (uint32_t)rnd)) {
        d.slab = sr.x;
        d.r = sr.y;
        return d;
    }
    int64_t slab = b;
    if (rw.slab_tab) slab = rw.slab_tab[(int64_t)i * rw.R + slab_round_index(rnd, rw.R)];
    d.slab = (int32_t)slab;
    d.r = rw.dtype == LAPSSD_BF16 ? accept_test(rw, slab, d.req, d.round, 0, sc.seed, load_prob_bf16)
                                  : accept_test(rw, slab, d.req, d.round, 0, sc.seed, load_prob_f32);
    if (rw.slab_tab) {  // memoise: a waiting request's round (hence its a1) does not change
        st.next_sr[i] = make_int2(d.slab, d.r);
        st.next_tag[i] = ((uint64_t)rw.epoch << 32) | (uint32_t)rnd;
    }
    return d;
}

// ---------------------------------------------------------------- verify launch
struct SelRec;
struct PreSelect;
struct VerifyArgs {
    RowsDev rows;
    int32_t n_chunks;
    int32_t cpb;                // vocabulary chunks per CTA
    const SlotDesc *desc;       // [B]
    const int32_t *sel;         // handle mode: must match desc[b].i (nullable: stateless)
    uint64_t seed;
    uint32_t trace;
    int32_t *tokens;
    int32_t *n_accept;
    uint64_t *z;
    uint64_t *part;             // [B][n_chunks][kPartWords] segment residual sums
    uint32_t *work;             // [2] item-claim counter, retired CTAs (zero between launches)
    // second (part, work) set and the step counter that picks one: consecutive laps_step
    // launches overlap (programmatic dependent launch), so step t+1 streams into the
    // other set while step t's finishers still read theirs (nullable: one set)
    uint64_t *part1;
    uint32_t *work1;
    const uint32_t *vstep;
    int32_t fuse_update;
    // nullable: the number of leading slots that hold work ([0, *count_dev) of the B
    // slots; the multi-GPU batch keeps this rank's slots first and pads with -1), so the
    // producers never cycle empty items through the ring
    const int32_t *count_dev;
    State st;                   // handle mode only
    Sched sc;
    uint32_t *err;              // sticky device flags (nullable in stateless mode)
    // incremental select (laps_step with pooled rows): each finisher writes its slot's
    // record (new key, next descriptor) and publishes the slot to the side-stream merger
    SelRec *fin;                // [B] one record per slot
    uint64_t *fin_key;          // [B] ~key, release-stored once fin[b] is written (0 = not yet); null: no records
    // +1 per CTA (release) once it has read all it needs of desc[] / sel[]; the side
    // select overwrites those only after every CTA has signalled (nullable)
    uint32_t *snap;
    int32_t check_rows;         // validate the rows' masses in the consumers (E_MASS)
};

enum : uint32_t { E_STALE_DESC = 8u };

// host-side launchers (verify.cu / sched.cu)
cudaError_t launch_accept(const RowsDev &rw, const int32_t *sel, const State *st, const Sched *sc,
                          const int32_t *slab, const uint32_t *req_id, const uint32_t *round_idx,
                          uint64_t seed, uint32_t trace, int32_t B, SlotDesc *desc, cudaStream_t s);
cudaError_t launch_verify(const VerifyArgs &a, int32_t B, cudaStream_t s);
cudaError_t launch_update(const State &st, const Sched &sc, const int32_t *sel,
                          const int32_t *n_accept, int32_t B, cudaStream_t s);
cudaError_t launch_select(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc,
                          int32_t B, int32_t *sel_out, int32_t *count_out, cudaStream_t s);
cudaError_t launch_candidates(const State &st, const Sched &sc, int32_t C, uint64_t *cand_out,
                              cudaStream_t s);
cudaError_t launch_merge(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc,
                         const uint64_t *all_cand, int32_t C, int32_t B, int32_t *sel_out,
                         int32_t *count_out, cudaStream_t s);
// Output of presort_kernel: the clock / admission of the coming select and the sorted
// top-B keys of the requests outside the current batch.
// A selectable request as the fused final select needs it: its key at this select,
// the acceptance-test descriptor of its next round (used if it is selected), its state
// flags at select time and whether it has never been served (x_i < 0).
struct __align__(16) SelRec {
    uint64_t key;
    uint32_t flags;
    int32_t x_unset;
    SlotDesc desc;
};
struct PreSelect {
    int64_t now_us;
    int32_t cursor;
    uint32_t ready;     // set (release) by the presort, cleared by the final select
    uint64_t cand[1];   // [next_pow2(max_batch)] sorted keys, then SelRec rec[...]
};
__host__ __device__ inline int even_up(int x) { return (x + 1) & ~1; }  // keeps SelRec 16-byte aligned
__host__ __device__ inline size_t preselect_words(int bp) {  // uint64 words incl. records
    return 2 + (size_t)even_up(bp) + (size_t)bp * (sizeof(SelRec) / 8);
}
__device__ __forceinline__ SelRec *pre_recs(PreSelect *p, int bp) {
    return reinterpret_cast<SelRec *>(p->cand + even_up(bp));
}
__device__ __forceinline__ const SelRec *pre_recs(const PreSelect *p, int bp) {
    return reinterpret_cast<const SelRec *>(p->cand + even_up(bp));
}
cudaError_t launch_verify_logits(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                                 const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                                 const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                                 int32_t *tokens, int32_t *n_accept, uint64_t *z, float *m_ws, uint64_t *S_ws,
                                 char *lazy_ws, cudaStream_t s);
size_t logits_lazy_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype);   // the lazy form's workspace
cudaError_t launch_logits_slots(const int32_t *sel, const int32_t *rounds, const int32_t *slab_tab, int32_t R,
                                int32_t world, int32_t rank, int32_t B, uint32_t *req, uint32_t *rnd, int32_t *slab,
                                cudaStream_t s);
cudaError_t launch_logits_mask(const int32_t *sel, int32_t k, int32_t B, int32_t *tokens, int32_t *n_accept,
                               cudaStream_t s);
void verify_logits_prepare();
// f4 (draft_tree.cu)
cudaError_t launch_draft_sample(const void *q, int32_t dtype, int64_t V, const int32_t *row_idx,
                                const uint32_t *req, const uint32_t *rnd, const uint32_t *pos, int32_t R,
                                uint64_t seed, uint32_t trace, int32_t *out, uint64_t *z_out, cudaStream_t s);
cudaError_t launch_verify_tree(const void *p, const void *q, int32_t dtype, int64_t V, int32_t n_nodes,
                               const int32_t *parent, const int32_t *token, const uint32_t *req,
                               const uint32_t *rnd, int32_t B, uint64_t seed, uint32_t trace, int32_t *tokens,
                               int32_t *path, int32_t *n_accept, uint64_t *z_out, cudaStream_t s);
cudaError_t launch_presort(const State &st, const Sched &sc, const RowsDev &rw, const int32_t *sel, int32_t B,
                           PreSelect *out, cudaStream_t s);
cudaError_t launch_select_final(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc, int32_t B,
                                int32_t *sel, int32_t *count_out, const PreSelect *pre, cudaStream_t s);
cudaError_t launch_verify_grid(const VerifyArgs &a, int32_t B, int32_t reserve_sms, bool pdl, cudaStream_t s);
int verify_grid(int32_t B, int32_t n_chunks, int32_t reserve_sms);       // CTAs of that launch
bool verify_fits(int32_t B, int32_t n_chunks, int32_t reserve_sms);      // per-CTA snapshot capacity
int verify_max_batch(int32_t n_chunks, int32_t reserve_sms);
// The persistent waiting list of laps_step's side select: the sorted keys of every
// eligible request outside the current batch.  A waiting request's state -- hence its key
// -- does not change, so a step merges the few keys that changed (the verified batch,
// admissions) instead of sorting all N (select_side_kernel).
constexpr int kAdmCap = 1024;   // admissions merged per step (more: the list is rebuilt)
struct WaitList {
    uint64_t *keys[2];     // [n] double buffer, sorted ascending; keys[meta[1]] is current
    int32_t *fresh_i;      // [max_batch] the last commit's verified, not reselected requests
    uint64_t *fresh_key;   // [max_batch] their waiting keys (st.key rewritten at the next select)
    int32_t *meta;         // [4] length, current buffer, fresh count, pad (nullptr: no list)
    int32_t valid;         // the list describes the state (else the side select rebuilds it)
};
// laps_step_peer: every rank's exchange buffer as mapped in this process (device array of
// world pointers; bufs[rank] is this rank's own), C candidates per rank.
struct PeerArgs {
    uint64_t *const *bufs;   // nullptr: no peer exchange
    int32_t C;
};
cudaError_t launch_select_side(const State &st, const Sched &sc, const RowsDev &rw, int32_t *sel, SlotDesc *desc,
                               int32_t B, PreSelect *pre, const SelRec *fin, uint64_t *fin_key, uint32_t *snap,
                               uint32_t snap_target, int32_t *count_out, cudaStream_t s,
                               uint64_t *cand_out = nullptr, int32_t C = 0, const WaitList *wl = nullptr,
                               const PeerArgs *peer = nullptr);
// Monte-Carlo replicas (mc.cu): T traces over one concatenated request SoA.
struct McDev {
    const int64_t *off;         // [T+1] request offsets of the traces
    Globals *g;                 // [T] per-trace clock, cursor, counts
    int32_t *last;              // [T] request verified in the previous step (-1: none)
    int32_t T;
};
cudaError_t launch_mc_step(const State &st, const Sched &sc, const McDev &mc, const RowsDev &rw,
                           const int32_t *n_accept, SlotDesc *desc, int32_t *sel_out, int32_t *active,
                           cudaStream_t s);
int sort_capacity();            // largest key count one select CTA can sort
void prepare_all();             // kernel attributes, once per process (api.cu)
void verify_prepare();
void sched_prepare();
int verify_cpb(int64_t V);      // chunks per CTA chosen for V (env LAPSSD_CPB overrides)
void count_launch(int n = 1);

}  // namespace lapssd
