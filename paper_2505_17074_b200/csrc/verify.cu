// verify.cu -- batched speculative verification by rejection sampling on sm_100a
// (Eq. 1, bonus token P:200; AMB-1, 2, 20, 21, 27).
//
// a1 (accept_kernel, or memoised by the select / the previous step's update): one
//    thread per slot gathers p_j(x_j), q_j(x_j) for the k drafts (independent loads)
//    and applies the exact fp64 test u24*q < p*2^24 with Philox uniforms -> r, in a
//    32-byte SlotDesc.
// a2 (+a3) (verify_kernel): persistent, TMA-fed, one CTA per SM; streams the ONE row
//    pair the algorithm needs -- (p_r, q_r), or p_k on full acceptance -- in 32 KB
//    chunks, reducing the exact Q4.60 residual mass R_v = floor(max(0, fl32(p-q)) * 2^60)
//    to one uint64 per 1024-entry segment (integer sums: exact, order-independent);
//    the finisher of each slot totals Z, draws t = floor(U Z / 2^64), finds the segment
//    holding t, rescans it with warp scans and emits y.  The state update of the slot's
//    request runs first, at kernel start, since it depends on r only.
// HBM bytes per slot: 2 V s (r < k) or V s (r = k), plus k gathered scalars.
#include <cstdlib>

#include "select_core.cuh"

namespace lapssd {

__device__ __forceinline__ uint4 ld_stream(const void *ptr) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr));
    return r;
}

// Q4.60 residual mass of one entry: fl32 subtraction (round to nearest), exact
// power-of-two scaling, truncating conversion.  cvt.rzi.u64.f32 clamps to the
// destination range, so d <= 0 (and NaN) gives 0.
__device__ __forceinline__ uint64_t q460(float p, float q) {
    return __float2ull_rz(__fmul_rn(__fsub_rn(p, q), 0x1p60f));
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <bool BF16> struct Elt;
template <> struct Elt<true> {
    static constexpr int kVec = 8;  // bf16 per 16-byte vector
    static constexpr int kEsz = 2;
    __device__ static uint64_t mass(uint4 p, uint4 q) {
        uint64_t s = 0;
        s += q460(bf_lo(p.x), bf_lo(q.x)); s += q460(bf_hi(p.x), bf_hi(q.x));
        s += q460(bf_lo(p.y), bf_lo(q.y)); s += q460(bf_hi(p.y), bf_hi(q.y));
        s += q460(bf_lo(p.z), bf_lo(q.z)); s += q460(bf_hi(p.z), bf_hi(q.z));
        s += q460(bf_lo(p.w), bf_lo(q.w)); s += q460(bf_hi(p.w), bf_hi(q.w));
        return s;
    }
    __device__ static float elem(uint4 v, int e) {
        const uint32_t w = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
        return (e & 1) ? bf_hi(w) : bf_lo(w);
    }
};
template <> struct Elt<false> {
    static constexpr int kVec = 4;  // fp32 per 16-byte vector
    static constexpr int kEsz = 4;
    __device__ static uint64_t mass(uint4 p, uint4 q) {
        uint64_t s = 0;
        s += q460(__uint_as_float(p.x), __uint_as_float(q.x));
        s += q460(__uint_as_float(p.y), __uint_as_float(q.y));
        s += q460(__uint_as_float(p.z), __uint_as_float(q.z));
        s += q460(__uint_as_float(p.w), __uint_as_float(q.w));
        return s;
    }
    __device__ static float elem(uint4 v, int e) {
        const uint32_t w = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
        return __uint_as_float(w);
    }
};

template <bool BF16>
struct Seg {
    static constexpr int kVec = Elt<BF16>::kVec;
    static constexpr int J = kSegElems / kVec / 32;  // vectors per lane per warp segment
    // This lane's J vectors of the warp segment starting at element `base`.
    __device__ static void load(const char *row, int64_t base, int64_t V, int lane, uint4 (&v)[J]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t e = base + (int64_t)(j * 32 + lane) * kVec;
            v[j] = e < V ? ld_stream(row + e * Elt<BF16>::kEsz) : make_uint4(0, 0, 0, 0);
        }
    }
};

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Residual mass of this lane's share of one warp segment, in groups of 4 vectors per
// row (8 x 16-byte loads in flight per thread for bf16 and fp32 alike).
template <bool BF16>
__device__ __forceinline__ uint64_t lane_mass(const char *prow, const char *qrow, bool use_q,
                                              int64_t base, int64_t V, int lane) {
    using S = Seg<BF16>;
    constexpr int G = 4;
    constexpr int kEsz = Elt<BF16>::kEsz;
    uint64_t s = 0;
#pragma unroll
    for (int g = 0; g < S::J; g += G) {
        uint4 pv[G], qv[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int64_t e = base + (int64_t)((g + j) * 32 + lane) * S::kVec;
            pv[j] = e < V ? ld_stream(prow + e * kEsz) : make_uint4(0, 0, 0, 0);
            qv[j] = (use_q && e < V) ? ld_stream(qrow + e * kEsz) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < G; ++j) s += Elt<BF16>::mass(pv[j], qv[j]);
    }
    return s;
}

// ---------------------------------------------------------------- a1: accept kernel
__global__ void accept_kernel(const RowsDev rw, const int32_t *sel, const State st, const Sched sc,
                              int32_t has_state, const int32_t *slab, const uint32_t *req_id,
                              const uint32_t *round_idx, uint64_t seed, uint32_t trace, int32_t B,
                              SlotDesc *desc) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    if (has_state) {
        desc[b] = make_desc(rw, st, sc, b, sel[b]);
        return;
    }
    SlotDesc d;
    d.i = -1;
    d.slab = slab ? slab[b] : b;
    d.req = req_id[b];
    d.round = round_idx[b];
    d.trace = trace; d.pad[0] = d.pad[1] = 0;
    d.r = rw.dtype == LAPSSD_BF16
              ? accept_test(rw, d.slab, d.req, d.round, trace, seed, load_prob_bf16)
              : accept_test(rw, d.slab, d.req, d.round, trace, seed, load_prob_f32);
    desc[b] = d;
}

cudaError_t launch_accept(const RowsDev &rw, const int32_t *sel, const State *st, const Sched *sc,
                          const int32_t *slab, const uint32_t *req_id, const uint32_t *round_idx,
                          uint64_t seed, uint32_t trace, int32_t B, SlotDesc *desc, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    State st0{};
    Sched sc0{};
    accept_kernel<<<(B + 127) / 128, 128, 0, s>>>(rw, sel, st ? *st : st0, sc ? *sc : sc0, st != nullptr,
                                                  slab, req_id, round_idx, seed, trace, B, desc);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a2: verify kernel
// Persistent, warp-specialised, TMA-fed; one CTA per SM.  CTA = 1 producer warp + 16
// consumer warps + 2 finisher warps.  Work item n = (slot b = n / n_chunks, chunk
// c = n % n_chunks), claimed dynamically (first n = blockIdx.x, then tickets).
//  snapshot: (slab, r) of every slot and the descriptors of the finishers' slots are
//            copied to shared memory first; then the side select may commit the next
//            batch over desc[] / sel[].
//  producer: issues cp.async.bulk of chunk c of p_r (and q_r when r < k) into a ring
//            of shared-memory stages, completion tracked by mbarrier tx-count.
//  consumers: warp w reduces segment w of the stage to one uint64 and publishes it
//            with bit 63 as a ready flag (relaxed store); it then frees the stage.  No
//            block-wide barrier, no fence and no atomic on the streaming path.
//  finishers: slot b belongs to finisher b mod (2 grid).  First the state updates of
//            their slots (+ next-round a1, select record, release-stored tag), then,
//            per slot, wait for all n_chunks*16 ready words, total, sample, emit.
#ifdef LAPSSD_TRACE
#ifndef LAPSSD_TRACE_A
#define LAPSSD_TRACE_A 0
#endif
#ifndef LAPSSD_TRACE_B
#define LAPSSD_TRACE_B 74
#endif
// Diagnostic build only (tools/): fire-and-forget timestamps per (event, item) of two CTAs.
__device__ unsigned long long g_trace[2][16][1024];
__device__ __forceinline__ void trace(int ev, int x) {
    const int slot = blockIdx.x == LAPSSD_TRACE_A ? 0 : blockIdx.x == LAPSSD_TRACE_B ? 1 : -1;
    if (slot < 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[slot][ev][x & 1023] = t;
}
__device__ unsigned long long g_cta_t[10][160];   // start, end, producer last issue, consumer last, finisher last ready, bytes, f-y, f-upd, f-done
__device__ unsigned long long g_fs_trace[8];     // fused final select phases
__device__ unsigned long long g_vstart[64];      // verify CTA 0 start per launch
__device__ unsigned int g_vcount;
extern "C" int lapssd_vstart_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_vstart, sizeof g_vstart);
    unsigned z = 0; cudaMemcpyToSymbol(g_vcount, &z, 4);
    return 0;
}
extern "C" int lapssd_fs_trace_read(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_fs_trace, sizeof g_fs_trace); }
__device__ __forceinline__ void cta_time(int which) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 160) {
        if (which == 0) {
            atomicMin(&g_cta_t[0][blockIdx.x], t);
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_cta_t[9][blockIdx.x] = smid;
        } else {
            atomicMax(&g_cta_t[which][blockIdx.x], t);
        }
    }
}
__device__ __forceinline__ void cta_bytes(unsigned n) {
    if (blockIdx.x < 160) atomicAdd(&g_cta_t[5][blockIdx.x], (unsigned long long)n);
}
extern "C" int lapssd_cta_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_cta_t, sizeof(g_cta_t));
    static unsigned long long init[10][160];
    for (int i = 0; i < 160; ++i) { init[0][i] = ~0ull; for (int j = 1; j < 10; ++j) init[j][i] = 0; }
    cudaMemcpyToSymbol(g_cta_t, init, sizeof(init));
    return 0;
}
#define CTA_TIME(w) cta_time(w)
#define CTA_BYTES(n) cta_bytes(n)
__device__ unsigned long long g_slot_t[3][4096];   // per slot: update start, published, sampled
extern "C" int lapssd_slot_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_slot_t, sizeof g_slot_t);
    static unsigned long long zero[3 * 4096];
    cudaMemcpyToSymbol(g_slot_t, zero, sizeof zero);
    return 0;
}
#define SLOT_TIME(w, b) do { if ((b) < 4096) g_slot_t[w][b] = gtimer(); } while (0)
__device__ unsigned long long g_vstep_t[64][2];   // per committed step: first CTA start, last CTA end
__device__ unsigned long long g_vstep_sm[64][3];  // per committed step: SMs the verify CTAs ran on
extern "C" int lapssd_vstep_sm_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_vstep_sm, sizeof g_vstep_sm);
    static unsigned long long zero[64][3];
    cudaMemcpyToSymbol(g_vstep_sm, zero, sizeof zero);
    return 0;
}
extern "C" int lapssd_vstep_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_vstep_t, sizeof g_vstep_t);
    static unsigned long long init[64][2];
    for (int i = 0; i < 64; ++i) { init[i][0] = ~0ull; init[i][1] = 0; }
    cudaMemcpyToSymbol(g_vstep_t, init, sizeof init);
    return 0;
}
#define VSTEP_TIME(w, v) do { if ((w) == 0) atomicMin(&g_vstep_t[(v) & 63][0], gtimer()); \
                              else atomicMax(&g_vstep_t[(v) & 63][1], gtimer()); } while (0)
extern "C" int lapssd_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
    cudaMemset(nullptr, 0, 0);
    static unsigned long long zero[2 * 16 * 1024];
    cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
    return 0;
}
#define TRACE(ev, x) trace(ev, x)
#else
#define TRACE(ev, x)
#define CTA_TIME(w)
#define CTA_BYTES(n)
#define SLOT_TIME(w, b)
#define VSTEP_TIME(w, v)
#endif
constexpr int kConsumerWarps = 16;                         // all consume every item (one segment each)
constexpr int kGroups = 2;                                 // finisher warps per CTA
constexpr int kVerifyThreads = (1 + kConsumerWarps + kGroups) * 32;  // producer, consumers, finishers
constexpr int kMaxSlots = 4096;                            // slots per launch (4-byte snapshot each)
constexpr int kFinCap = 64;                                // slots per finisher warp
constexpr int kStageBudget = 192 * 1024;                   // shared memory for the ring
#ifndef LAPSSD_POLL_NS
#define LAPSSD_POLL_NS 1024
#endif
#ifndef LAPSSD_POLL_NEAR
#define LAPSSD_POLL_NEAR 2
#endif
#ifndef LAPSSD_POLL_NEAR_NS
#define LAPSSD_POLL_NEAR_NS 128
#endif
constexpr int kPollNearNs = LAPSSD_POLL_NEAR_NS;  // back-off when <= LAPSSD_POLL_NEAR chunks are pending
constexpr int kPollNs = LAPSSD_POLL_NS;  // finisher back-off between polls (measured: 32 ns of polling traffic costs ~2 us/step)

template <bool BF16>
struct VerifyCfg {
    static constexpr int kEsz = BF16 ? 2 : 4;
    static constexpr int kTileElems = tile_elems(kEsz);               // 16384 / 8192 entries per item
    static constexpr int kSegs = kTileElems / kSegElems;              // 16 / 8 segments per chunk
    static constexpr int kCPL = kPartWords / kSegs;                   // chunks per finisher lane: 1 / 2
    static constexpr int kStages = kStageBudget / (2 * kTileBytes);   // 3
    static_assert(kSegs * kCPL == kPartWords && kSegs <= kConsumerWarps, "tiling");
    static_assert(kMaxSegs / kSegs <= 32 * kCPL, "a finisher lane holds at most kCPL chunks");
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// The rows are read once per step, so their bulk copies carry an L2 evict-first policy:
// the 245 MB streamed per step then does not flush the scheduler state, slab table and
// drafts out of L2, whose dependent loads (the update, the next round's a1, the select)
// would otherwise queue behind the stream in HBM.
#ifndef LAPSSD_TMA_EVICT_FIRST
#define LAPSSD_TMA_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
#if LAPSSD_TMA_EVICT_FIRST
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first_policy())
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
#endif
}
// Published segment sums carry bit 63 as a ready flag (a segment's Q4.60 mass is < 2^61),
// so each word is self-describing: no fence or counter orders it against other words.
constexpr uint64_t kReady = 1ull << 63;
__device__ __forceinline__ void st_relaxed(uint64_t *addr, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_relaxed2(const uint64_t *addr) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(addr) : "memory");
    return v;
}
// The N published segment sums of chunk c (one lane per chunk), into w[off..off+N):
// issued together.
template <int N>
__device__ __forceinline__ void load_chunk_words(const uint64_t *part, int c, uint64_t *w) {
#pragma unroll
    for (int h = 0; h < N / 2; ++h) {
        const ulonglong2 v = ld_relaxed2(part + (int64_t)c * kPartWords + 2 * h);
        w[2 * h] = v.x;
        w[2 * h + 1] = v.y;
    }
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *addr) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(addr) : "memory");
    return v;
}

// Next-round a1 of local request i (pooled rows only), one position per lane.  The
// next round is d.round + 1, so the whole chain (slab table -> draft -> gathers) can be
// issued at the start of the finish and overlap the sampling.
struct NextA1 {
    int64_t slab;
    int32_t x;
    float pj, qj;
    bool live;
};
// The chain in three stages (slab table -> draft -> gathers) so that the stages of
// several slots can be issued together: one memory round trip per stage, not per slot.
__device__ __forceinline__ NextA1 next_a1_stage1(const VerifyArgs &a, int32_t i, uint32_t round_next) {
    const RowsDev &rw = a.rows;
    NextA1 n;
    n.live = a.fuse_update && rw.slab_tab != nullptr && i >= 0;
    n.slab = 0;
    n.x = 0;
    n.pj = 1.0f;
    n.qj = 0.0f;
    if (n.live) n.slab = rw.slab_tab[(int64_t)i * rw.R + slab_round_index((int32_t)round_next, rw.R)];
    return n;
}
__device__ __forceinline__ void next_a1_stage2(const VerifyArgs &a, NextA1 &n) {
    const int lane = threadIdx.x & 31;
    if (n.live && lane < a.rows.k) n.x = a.rows.draft[n.slab * a.rows.k + lane];
}
template <bool BF16>
__device__ __forceinline__ void next_a1_stage3(const VerifyArgs &a, NextA1 &n) {
    const int lane = threadIdx.x & 31;
    const RowsDev &rw = a.rows;
    const int k = rw.k;
    if (!n.live || lane >= k) return;
    const int64_t V = rw.V;
    const char *pb = (const char *)rw.p + n.slab * (int64_t)(k + 1) * V * Elt<BF16>::kEsz;
    const char *qb = (const char *)rw.q + n.slab * (int64_t)k * V * Elt<BF16>::kEsz;
    n.pj = BF16 ? load_prob_bf16(pb, (int64_t)lane * V + n.x) : load_prob_f32(pb, (int64_t)lane * V + n.x);
    n.qj = BF16 ? load_prob_bf16(qb, (int64_t)lane * V + n.x) : load_prob_f32(qb, (int64_t)lane * V + n.x);
}
__device__ __forceinline__ int next_a1_store(const VerifyArgs &a, int32_t i, uint32_t req, uint32_t round_next,
                                             const NextA1 &n) {
    const int lane = threadIdx.x & 31;
    if (!n.live) return -1;
    const int k = a.rows.k;
    bool reject = false;
    if (lane < k) {
        const uint4 u = philox4x32_10(make_uint4(req, round_next, (uint32_t)(lane >> 2), 0u), (uint32_t)a.sc.seed,
                                      (uint32_t)(a.sc.seed >> 32));
        const uint32_t w = (lane & 3) == 0 ? u.x : (lane & 3) == 1 ? u.y : (lane & 3) == 2 ? u.z : u.w;
        reject = !(__dmul_rn((double)(w >> 8), (double)n.qj) < __dmul_rn((double)n.pj, 16777216.0));
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, reject);
    const int r = m ? __ffs(m) - 1 : k;
    if (lane == 0) {
        a.st.next_sr[i] = make_int2((int32_t)n.slab, r);
        a.st.next_tag[i] = ((uint64_t)a.rows.epoch << 32) | round_next;
    }
    return r;
}

// Warp-level state update of slot b's request (a3) plus what the next select needs from
// it, run at the START of the verify kernel.  The scheduler state depends on r (fixed by
// a1 before any row streams) and never on the sampled token y, so the update, the new
// priority key and the next round's acceptance test need not wait for the residual
// stream; the record is published to the side-stream select at
// once, which then merges the whole verified batch while the rows are still streaming.
template <bool BF16>
__device__ __forceinline__ void update_slot_warp(const VerifyArgs &a, int b, const SlotDesc &d, const UpdIn &upd,
                                                 int64_t now, const NextA1 &nxt) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) SLOT_TIME(0, b);
    const UpdOut uo = update_warp(a.st, a.sc, d.i, d.r, now, upd, lane);
    if (lane == 0) TRACE(13, b);
    const int r_next = next_a1_store(a, d.i, d.req, d.round + 1, nxt);  // harmless if it completed
    if (a.fin_key && lane == 0) {
        // the request's record for the select: new key and next-round descriptor
        SelRec rec;
        rec.key = build_key(a.sc, d.i, INT32_MAX, uo.fl, upd.Lp, uo.tok, uo.A);
        rec.flags = uo.fl;
        rec.x_unset = 0;
        rec.desc.i = d.i;
        rec.desc.slab = (int32_t)nxt.slab;
        rec.desc.req = d.req;
        rec.desc.round = d.round + 1;
        rec.desc.r = r_next;
        rec.desc.trace = d.trace; rec.desc.pad[0] = rec.desc.pad[1] = 0;
        a.fin[b] = rec;
        a.st.key[d.i] = rec.key;
        // publish the key (release: orders the record before it; nothing waits on it
        // here).  Stored inverted so 0 means "not yet": no key is all ones (ids < 2^24-1)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.fin_key + b), "l"(~rec.key) : "memory");
        SLOT_TIME(1, b);
    }
    __syncwarp();
}

// Warp-level residual draw of slot b once all its (chunk, segment) sums are published:
// total Z, draw t, locate (chunk, segment), rescan that segment in vocabulary order,
// emit.  P:64, AMB-20.  w[h * kSegs + s] = sum of segment s of chunk lane + 32 h.
template <bool BF16>
__device__ __forceinline__ void sample_slot_warp(const VerifyArgs &a, uint64_t *part_set, int b, const SlotDesc &d,
                                                 uint64_t *fb, uint64_t (&w)[kPartWords]) {
    using E = Elt<BF16>;
    using S = Seg<BF16>;
    using TC = VerifyCfg<BF16>;
    constexpr int kSegs = TC::kSegs;
    const int lane = threadIdx.x & 31;
    const int k = a.rows.k, r = d.r, nc = a.n_chunks;
    const int64_t V = a.rows.V;
    const bool use_q = r < k;
    const char *prow = (const char *)a.rows.p + ((int64_t)d.slab * (k + 1) + r) * V * E::kEsz;
    const char *qrow = (const char *)a.rows.q + ((int64_t)d.slab * k + (use_q ? r : 0)) * V * E::kEsz;
    uint64_t *part = part_set + (int64_t)b * nc * kPartWords;
    // chunk sums: cs0 for chunk lane, cs1 for chunk lane + 32 (fp32 tiling only)
    uint64_t cs0 = 0, cs1 = 0;
    uint64_t za = 0;   // Z / 16, which cannot wrap: the row mass check (E_MASS)
#pragma unroll
    for (int x = 0; x < kPartWords; ++x) {
        w[x] &= ~kReady;
        if (x < kSegs) cs0 += w[x]; else cs1 += w[x];
        za += w[x] >> 4;
    }
    uint64_t Z = warp_sum_u64(cs0 + cs1);
    if ((warp_sum_u64(za) >> 57) != 0 && lane == 0 && a.err) atomicOr(a.err, E_MASS);   // mass > 2
    if (lane == 0) TRACE(9, b);
    bool fallback = false;
    if (Z == 0 && use_q) {  // no residual mass while rejecting: the row p_r itself
        fallback = true;
        for (int g = 0; g < nc * kSegs; ++g) {
            const uint64_t m = warp_sum_u64(lane_mass<BF16>(prow, qrow, false, (int64_t)g * kSegElems, V, lane));
            if (lane == 0) fb[g] = m;
        }
        __syncwarp();
        cs0 = cs1 = 0;
        if (lane < nc)
            for (int x = 0; x < kSegs; ++x) cs0 += fb[lane * kSegs + x];
        if (lane + 32 < nc)
            for (int x = 0; x < kSegs; ++x) cs1 += fb[(lane + 32) * kSegs + x];
        Z = warp_sum_u64(cs0 + cs1);
    }
    int y = -1;
    if (Z == 0) {
        if (a.err && lane == 0) atomicOr(a.err, E_NO_MASS);
        y = use_q ? a.rows.draft[(int64_t)d.slab * k + r] : 0;
    } else {
        const uint4 u = philox4x32_10(make_uint4(d.req, d.round, 1u << 8, d.trace), (uint32_t)a.seed,
                                      (uint32_t)(a.seed >> 32));
        const uint64_t U = ((uint64_t)u.x << 32) | u.y;
        uint64_t t = __umul64hi(U, Z);  // floor(U Z / 2^64) in [0, Z)
        int cstar;
        {
            const uint64_t incl = warp_incl_scan_u64(cs0, lane);
            const uint64_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            if (t < tot) {
                const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
                t -= __shfl_sync(0xFFFFFFFFu, incl - cs0, src);
                cstar = src;
            } else {
                t -= tot;
                const uint64_t incl1 = warp_incl_scan_u64(cs1, lane);
                const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl1 > t)) - 1;
                t -= __shfl_sync(0xFFFFFFFFu, incl1 - cs1, src);
                cstar = 32 + src;
            }
        }
        uint64_t ssum = 0;
#pragma unroll
        for (int x = 0; x < kSegs; ++x) {  // the segment sums of chunk cstar, to lanes 0..kSegs-1
            const uint64_t v = __shfl_sync(0xFFFFFFFFu, cstar < 32 ? w[x] : w[(kSegs + x) % kPartWords], cstar & 31);
            if (lane == x) ssum = v;
        }
        if (fallback) ssum = lane < kSegs ? fb[cstar * kSegs + lane] : 0;
        const uint64_t sincl = warp_incl_scan_u64(ssum, lane);
        const int sstar = __ffs(__ballot_sync(0xFFFFFFFFu, lane < kSegs && sincl > t)) - 1;
        t -= __shfl_sync(0xFFFFFFFFu, sincl - ssum, sstar);
        const int64_t base = (int64_t)cstar * TC::kTileElems + (int64_t)sstar * kSegElems;
        if (lane == 0) TRACE(10, b);
        const bool q_in = use_q && !fallback;
        uint4 pv[S::J], qv[S::J];
        S::load(prow, base, V, lane, pv);
        if (q_in) {
            S::load(qrow, base, V, lane, qv);
        } else {
#pragma unroll
            for (int j = 0; j < S::J; ++j) qv[j] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < S::J; ++j) {
            const uint64_t m = E::mass(pv[j], qv[j]);
            const uint64_t incl = warp_incl_scan_u64(m, lane);
            const uint64_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            if (y < 0) {
                if (t < tot) {
                    const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
                    int yy = -1;
                    if (lane == src) {
                        uint64_t tt = t - (incl - m);
                        int e = 0;
                        for (; e < S::kVec; ++e) {
                            const uint64_t me = q460(E::elem(pv[j], e), E::elem(qv[j], e));
                            if (tt < me) break;
                            tt -= me;
                        }
                        yy = (int)(base + (int64_t)(j * 32 + lane) * S::kVec + e);
                    }
                    y = __shfl_sync(0xFFFFFFFFu, yy, src);
                } else {
                    t -= tot;
                }
            }
        }
    }
    if (lane == 0) TRACE(11, b);
    if (a.tokens) {
        int32_t *tok = a.tokens + (int64_t)b * (k + 1);
        const int32_t *dr = a.rows.draft + (int64_t)d.slab * k;
        if (lane <= k) tok[lane] = lane < r ? dr[lane] : lane == r ? y : -1;
    }
    for (int x = lane; x < nc * kPartWords; x += 32)  // unpublish for the next launch / replay
        st_relaxed(part + x, 0ull);
    if (lane == 0) {
        if (a.n_accept) a.n_accept[b] = r;
        if (a.z) a.z[b] = Z;
    }
    __syncwarp();
}

// Slot b is finished (sampled) by finisher f = b mod (kGroups * grid): group f / grid of
// CTA f % grid, so consecutive slots -- which complete together at the end of the
// stream -- are finished by different warps of different CTAs.
__host__ __device__ __forceinline__ int fin_slots(int B, int grid, int f0) {
    return f0 < B ? (B - 1 - f0) / (kGroups * grid) + 1 : 0;
}

// Loads of values another kernel wrote (the batch, the step counter, the clock, the
// scheduler state) bypass L1 (ld.global.cg): with programmatic dependent launch this
// grid starts before the previous one has completed, so nothing may be served from a
// line an earlier grid left in this SM's L1.
__device__ __forceinline__ SlotDesc ld_desc_cg(const SlotDesc *p) {
    const int4 *q = reinterpret_cast<const int4 *>(p);
    const int4 lo = __ldcg(q), hi = __ldcg(q + 1);
    SlotDesc d;
    d.i = lo.x; d.slab = lo.y; d.req = (uint32_t)lo.z; d.round = (uint32_t)lo.w;
    d.r = hi.x; d.trace = (uint32_t)hi.y; d.pad[0] = hi.z; d.pad[1] = hi.w;
    return d;
}

// (slab << 5) | (r + 1) of slot b, 0 = nothing to do: the descriptor checked against
// sel[] (a stale descriptor or a bad slab index is a contract violation, flagged).
__device__ __forceinline__ uint32_t slot_word(const VerifyArgs &a, int b) {
    const int4 *dp = reinterpret_cast<const int4 *>(a.desc + b);
    const int4 dh = __ldcg(dp);  // i, slab, req, round
    int r = __ldcg(dp + 1).x;
    const int si = a.sel ? __ldcg(a.sel + b) : dh.x;
    if (r >= 0 && si != dh.x) {
        if (a.err) atomicOr(a.err, E_STALE_DESC);
        r = -1;
    }
    if (r >= 0 && (uint32_t)dh.y >= (1u << 27)) {
        if (a.err) atomicOr(a.err, E_BAD_SLOT);
        r = -1;
    }
    return r < 0 ? 0u : ((uint32_t)dh.y << 5) | (uint32_t)(r + 1);
}

// L2 prefetch (no shared memory, no completion) of item n's bytes: chunk c of p_r and, if
// r < k, of q_r, for the slot word `it`.
template <bool BF16>
__device__ __forceinline__ void prefetch_item(const VerifyArgs &a, int n, uint32_t it) {
    using E = Elt<BF16>;
    using TC = VerifyCfg<BF16>;
    if (it == 0) return;
    const int kk = a.rows.k, nc = a.n_chunks;
    const int64_t V = a.rows.V;
    const int r = (int)(it & 31u) - 1;
    const int64_t slab = it >> 5;
    const int c = n % nc;
    const int64_t e0 = (int64_t)c * TC::kTileElems;
    const int64_t ne = V - e0 < TC::kTileElems ? V - e0 : TC::kTileElems;
    const uint32_t bytes = (uint32_t)(ne * E::kEsz);
    const char *pr = (const char *)a.rows.p + ((slab * (kk + 1) + r) * V + e0) * E::kEsz;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr), "r"(bytes) : "memory");
    if (r < kk) {
        const char *qr = (const char *)a.rows.q + ((slab * kk + r) * V + e0) * E::kEsz;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(qr), "r"(bytes) : "memory");
    }
}

// Producer: item n (slot n / nc, chunk n % nc) into ring stage st -- chunk c of p_r and,
// when r < k, of q_r, as bulk copies completing on full[st]; nothing for an empty slot.
template <bool BF16>
__device__ __forceinline__ void issue_item(const VerifyArgs &a, uint8_t *s_tiles, uint64_t *full_st, int st, int n,
                                           uint32_t it) {
    using E = Elt<BF16>;
    using TC = VerifyCfg<BF16>;
    if (it == 0) {
        mbar_arrive(full_st);
        return;
    }
    const int kk = a.rows.k, nc = a.n_chunks;
    const int64_t V = a.rows.V;
    const int r = (int)(it & 31u) - 1;
    const int64_t slab = it >> 5;
    const int c = n % nc;
    const int64_t e0 = (int64_t)c * TC::kTileElems;
    const int64_t ne = V - e0 < TC::kTileElems ? V - e0 : TC::kTileElems;
    const uint32_t bytes = (uint32_t)(ne * E::kEsz);
    const char *pr = (const char *)a.rows.p + ((slab * (kk + 1) + r) * V + e0) * E::kEsz;
    uint8_t *dst = s_tiles + (size_t)st * 2 * kTileBytes;
    const bool use_q = r < kk;
    mbar_arrive_tx(full_st, use_q ? 2 * bytes : bytes);
    CTA_BYTES(use_q ? 2 * bytes : bytes);
    tma_load_1d(dst, pr, bytes, full_st);
    if (use_q) {
        const char *qr = (const char *)a.rows.q + ((slab * kk + r) * V + e0) * E::kEsz;
        tma_load_1d(dst + kTileBytes, qr, bytes, full_st);
    }
}

// CHECK: the consumers also validate the rows' masses (E_MASS; lapssd_set_row_check).
template <bool BF16, bool CHECK>
__global__ void __launch_bounds__(kVerifyThreads, 1) verify_kernel(const __grid_constant__ VerifyArgs a,
                                                                    int32_t B) {
    using E = Elt<BF16>;
    using S = Seg<BF16>;
    using TC = VerifyCfg<BF16>;
    constexpr int kStages = VerifyCfg<BF16>::kStages;
    extern __shared__ __align__(128) uint8_t s_tiles[];  // kStages x (p chunk, q chunk)
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ uint32_t s_slot[kMaxSlots];             // per slot: (slab << 5) | (r + 1), 0 = nothing to do
    __shared__ int s_stage[kStages];                   // item in each ring stage (-1: no more items)
    __shared__ SlotDesc s_fin[kGroups][kFinCap];       // the slots each finisher owns
    __shared__ uint64_t s_fb[kGroups][kMaxSegs];       // Z = 0 fallback sums
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nc = a.n_chunks;
    int B_work = B;
    if (a.count_dev) {
        const int c = __ldcg(a.count_dev);
        B_work = c < 0 ? 0 : c < B ? c : B;
    }
    const int n_items = B_work * nc;
    const int grid = (int)gridDim.x;
    // warp 0 producer; warps 1..16 consumers (gw = segment); warps 17, 18 finishers (grp)
    const int gw = warp >= 1 && warp <= kConsumerWarps ? warp - 1 : -1;
    const int grp = warp > kConsumerWarps ? warp - 1 - kConsumerWarps : 0;
    const bool finisher = warp > kConsumerWarps;
    if (tid == 0) CTA_TIME(0);
#ifdef LAPSSD_TRACE
    if (tid == 0 && blockIdx.x == 0) { unsigned c = atomicAdd(&g_vcount, 1u); if (c < 64) g_vstart[c] = gtimer(); }
#endif
    // the next step's launch may start on SMs as ours retire (programmatic dependent
    // launch): it uses the other (part, work) set, and its finishers wait for this grid
    // before touching outputs.  The set is picked by the committed-step parity.
    const uint32_t vstep = a.vstep ? __ldcg(a.vstep) : 0u;
    const int par = (int)(vstep & 1u);
    if (tid == 0) VSTEP_TIME(0, vstep);
#ifdef LAPSSD_TRACE
    if (tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        atomicOr(&g_vstep_sm[vstep & 63][smid >> 6], 1ull << (smid & 63));
    }
#endif
    uint64_t *const part = par ? a.part1 : a.part;
    uint32_t *const work = par ? a.work1 : a.work;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ---- the producer issues this CTA's first kStages items (static: blockIdx.x + s grid)
    // straight from desc[] before the snapshot, so the first bytes are in flight while the
    // snapshot loads run.  desc[] cannot change before this CTA signals `snap` below.
    int k_pre = 0;
    if (tid == 0) {
        for (; k_pre < kStages; ++k_pre) {
            const int n = (int)blockIdx.x + k_pre * grid;
            if (n >= n_items) break;
            s_stage[k_pre] = n;
            issue_item<BF16>(a, s_tiles, &full[k_pre], k_pre, n, slot_word(a, n / nc));
        }
    }
    // ---- snapshot of everything this CTA reads of desc[] / sel[]: the (slab, r) of every
    // slot (items are claimed dynamically, so any slot may come up) and the descriptors
    // of the finishers' slots.  Once every CTA has signalled, the side-stream select may
    // overwrite desc[] / sel[] with the next batch.
    if (!finisher) {
        for (int b = tid; b < B; b += (1 + kConsumerWarps) * 32) s_slot[b] = slot_word(a, b);
    } else {
        const int f0 = grp * grid + (int)blockIdx.x;
        const int nf = fin_slots(B, grid, f0);
        for (int j = lane; j < nf; j += 32) {
            const int b = f0 + j * kGroups * grid;
            SlotDesc d = ld_desc_cg(a.desc + b);
            const int si = a.sel ? __ldcg(a.sel + b) : d.i;
            if (d.r >= 0 && (si != d.i || (uint32_t)d.slab >= (1u << 27))) d.r = -1;
            s_fin[grp][j] = d;
        }
    }
    __syncthreads();
    if (tid == 0 && a.snap) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.snap) : "memory");
    // dependents may launch once every CTA has taken its snapshot of desc[] / sel[]: the
    // next verify (laps_step) and the Monte-Carlo select, which rewrites desc[]
    if (tid == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        // Items are claimed dynamically (first item n = blockIdx.x, then grid + ticket), so
        // SMs that stream faster take more of them; one claim is kept in flight ahead.
        if (lane == 0) {
            // after the static items, claims: kStages grid + ticket, one claim kept in flight
            uint32_t nxt = k_pre == kStages ? (uint32_t)(kStages * grid) + atomicAdd(work, 1u) : (uint32_t)n_items;
            for (int k = k_pre;; ++k) {
                const int st = k % kStages;
                TRACE(1, k & 1023);
                if (k >= kStages) mbar_wait(&empty[st], ((k / kStages) - 1) & 1);
                TRACE(2, k & 1023);
                const int cur = nxt < (uint32_t)n_items ? (int)nxt : n_items;
                if (cur >= n_items) {  // no more items: tell the consumers
                    s_stage[st] = -1;
                    mbar_arrive(&full[st]);
                    break;
                }
                nxt = (uint32_t)(kStages * grid) + atomicAdd(work, 1u);
                s_stage[st] = cur;
                issue_item<BF16>(a, s_tiles, &full[st], st, cur, s_slot[cur / nc]);
                TRACE(8, k & 1023);
                CTA_TIME(2);
            }
            // retire: the last CTA to stop claiming leaves the counters zero for the next launch
            if (atomicAdd(work + 1, 1u) == (uint32_t)grid - 1) {
                work[0] = 0;
                work[1] = 0;
            }
#ifndef LAPSSD_NO_NEXT_PREFETCH
#ifndef LAPSSD_NEXT_PREFETCH_ITEMS
#define LAPSSD_NEXT_PREFETCH_ITEMS 3
#endif
            // The stream of this step is over for this CTA.  If the side select has already
            // committed the NEXT step's batch (laps_step: the step counter advanced), warm L2
            // with the first items the next launch's CTA of the same index will issue, so HBM
            // stays busy across the kernel boundary (the next grid's ramp reads from L2).
            if (a.fin_key && a.vstep) {
                uint32_t v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.vstep) : "memory");
                if (v == vstep + 1) {
                    int nb = B;
                    if (a.count_dev) {
                        const int cc = __ldcg(a.count_dev);
                        nb = cc < 0 ? 0 : cc < B ? cc : B;
                    }
                    for (int s2 = 0; s2 < LAPSSD_NEXT_PREFETCH_ITEMS; ++s2) {
                        const int n2 = (int)blockIdx.x + s2 * grid;
                        if (n2 >= nb * nc) break;
                        prefetch_item<BF16>(a, n2, slot_word(a, n2 / nc));
                    }
                }
            }
#endif
        }
        __syncwarp();
    } else if (finisher) {
        // ------------------------------------------------------------ finisher grp
        const int f0 = grp * grid + (int)blockIdx.x;
        const int nf = fin_slots(B, grid, f0);
        if (a.fuse_update) {
            // the state updates first, two slots at a time: each stage of both slots' loads
            // (state + slab table, drafts, gathers) is one round trip
            // the end of the step being verified: C_i of a request it completes
            const int64_t now = __ldcg(&a.st.g->now_us) + a.sc.c_round_us + __ldcg(&a.st.g->step_sw);
            for (int j = 0; j < nf; j += 2) {
                const SlotDesc d0 = s_fin[grp][j];
                const bool has1 = j + 1 < nf;
                const SlotDesc d1 = s_fin[grp][has1 ? j + 1 : j];
                const bool l0 = d0.r >= 0, l1 = has1 && d1.r >= 0;
                UpdIn u0{}, u1{};
                if (l0) u0 = load_update_inputs(a.st, a.sc, d0.i, lane);
                if (l1) u1 = load_update_inputs(a.st, a.sc, d1.i, lane);
                NextA1 x0 = next_a1_stage1(a, l0 ? d0.i : -1, d0.round + 1);
                NextA1 x1 = next_a1_stage1(a, l1 ? d1.i : -1, d1.round + 1);
                next_a1_stage2(a, x0);
                next_a1_stage2(a, x1);
                next_a1_stage3<BF16>(a, x0);
                next_a1_stage3<BF16>(a, x1);
                if (l0) update_slot_warp<BF16>(a, f0 + j * kGroups * grid, d0, u0, now, x0);
                if (l1) update_slot_warp<BF16>(a, f0 + (j + 1) * kGroups * grid, d1, u1, now, x1);
            }
        }
#if defined(LAPSSD_DIAG) && (LAPSSD_DIAG & 2)
        if (nf >= 0) return;  // diagnostic build: no sampling
#endif
        // outputs (tokens, n_accept, z) and the part words of the previous step's slots are
        // only touched once the previous launch has completed
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int j = 0; j < nf; ++j) {
            const SlotDesc d = s_fin[grp][j];
            const int b = f0 + j * kGroups * grid;
            if (d.r < 0) {  // empty slot: nothing verified
                if (lane == 0 && a.n_accept) a.n_accept[b] = -1;
                continue;
            }
            if (lane == 0) TRACE(5, b);
            const uint64_t *pw = part + (int64_t)b * nc * kPartWords;
            uint64_t w[kPartWords];
            const unsigned long long t_start = gtimer();
            for (;;) {  // every (chunk, segment) sum of slot b published?
#pragma unroll
                for (int x = 0; x < kPartWords; ++x) w[x] = kReady;
#pragma unroll
                for (int h = 0; h < TC::kCPL; ++h)
                    if (lane + 32 * h < nc) load_chunk_words<TC::kSegs>(pw, lane + 32 * h, w + h * TC::kSegs);
                uint64_t all = kReady;
#pragma unroll
                for (int x = 0; x < kPartWords; ++x) all &= w[x];
                const unsigned pending = __ballot_sync(0xFFFFFFFFu, (all & kReady) == 0);
                if (pending == 0) break;
                if (waited_too_long(t_start)) {
                    if (lane == 0 && a.err) {
                        if (!(atomicOr(a.err, E_TIMEOUT | E_TO_FIN) & E_TIMEOUT) && a.st.g)
                            a.st.g->err_where = ((vstep & 0xFFFFu) << 16) | ((uint32_t)b & 0xFFFFu);
                    }
                    break;
                }
                // long back-off while many chunks are outstanding, short once a few are left
                __nanosleep(__popc(pending) <= LAPSSD_POLL_NEAR ? kPollNearNs : kPollNs);
            }
            if (lane == 0) TRACE(6, b);
            if (lane == 0) CTA_TIME(4);
#if defined(LAPSSD_DIAG) && (LAPSSD_DIAG & 4)
            for (int x = lane; x < nc * kPartWords; x += 32)  // diagnostic build: poll, no draw
                st_relaxed(part + (int64_t)b * nc * kPartWords + x, 0ull);
#else
            sample_slot_warp<BF16>(a, part, b, d, s_fb[grp], w);
#endif
            if (lane == 0) TRACE(7, b);
            if (lane == 0) CTA_TIME(8);
            if (lane == 0) SLOT_TIME(2, b);
        }
        if (lane == 0) CTA_TIME(1);
    } else {
        // ------------------------------------------------------------ consumers: every item, segment gw
        // (one stage ring consumed in order by all consumer warps: a stage is refilled only
        // after all of them released it, so no warp can run a phase ahead)
        const int64_t V = a.rows.V;
        for (int k = 0;; ++k) {
            const int st = k % TC::kStages;
            mbar_wait(&full[st], (k / TC::kStages) & 1);
            if (gw == 0 && lane == 0) TRACE(3, k & 1023);
            const int n = s_stage[st];
            if (n < 0) break;
            const uint32_t it = s_slot[n / nc];
            if (it == 0 || gw >= TC::kSegs) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            } else {
                const int b = n / nc, c = n % nc;
                const int r = (int)(it & 31u) - 1;
                const uint4 qmask = r < a.rows.k ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0, 0, 0, 0);
                const uint4 *tp = reinterpret_cast<const uint4 *>(s_tiles + (size_t)st * 2 * kTileBytes);
                const uint4 *tq = tp + kTileBytes / 16;
                {
                    const int seg = gw;
                    const int64_t e_base = (int64_t)c * TC::kTileElems + (int64_t)seg * kSegElems;
                    uint4 pv[S::J], qv[S::J];
#pragma unroll
                    for (int j = 0; j < S::J; ++j) {  // branch-free: load, then mask the tail / absent q
                        const int v = seg * (kSegElems / S::kVec) + j * 32 + lane;
                        pv[j] = tp[v];
                        qv[j] = tq[v];
                    }
                    // the stage is in registers: release it to the producer before the
                    // arithmetic, so the refill's latency overlaps this item's math
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st]);
                    uint64_t m = 0, hi = 0;
#if defined(LAPSSD_DIAG) && (LAPSSD_DIAG & 1)
                    if (pv[0].x == 0x7FFFFFFFu && qv[0].y == 1u) m = 1;  // diagnostic build: no residual math
#else
#pragma unroll
                    for (int j = 0; j < S::J; ++j) {
                        const bool in = e_base + (int64_t)(j * 32 + lane) * S::kVec < V;
                        const uint4 z = make_uint4(0, 0, 0, 0);
                        const uint4 pm = in ? pv[j] : z;  // beyond V the stage holds stale bytes
                        const uint4 qm = in ? make_uint4(qv[j].x & qmask.x, qv[j].y & qmask.y, qv[j].z & qmask.z,
                                                         qv[j].w & qmask.w)
                                            : z;
                        const uint64_t x = E::mass(pm, qm);
                        m += x;
                        hi |= x;
                    }
#endif
                    // (CHECK) Rows of probabilities (entries in [0, 1], row mass ~1) give vector masses
                    // < 2^61, lane sums < 2^61 and segment sums < 2^62; an invalid row is flagged
                    // (E_MASS), never wrapped silently into the sums or the ready bit: a lane
                    // sum cannot wrap unless some vector mass >= 2^61, and the butterfly cannot
                    // unless >= 5 lanes hold >= 2^58 (then the segment's mass exceeds 1.25).
                    hi |= m;
                    bool bad = false;
                    if (CHECK) {
                        const unsigned heavy = __ballot_sync(0xFFFFFFFFu, (m >> 58) != 0);
                        bad = __any_sync(0xFFFFFFFFu, (hi >> 61) != 0) || __popc(heavy) >= 5;
                    }
                    m = warp_sum_u64(m);
                    if (CHECK) {
                        bad |= (m >> 62) != 0;
                        if (bad && lane == 0 && a.err) atomicOr(a.err, E_MASS);
                    }
                    if (lane == 0) st_relaxed(&part[((int64_t)b * nc + c) * kPartWords + seg], m | kReady);
                }
            }
            if (gw == 0 && lane == 0) TRACE(4, k & 1023);
            if (lane == 0) CTA_TIME(3);
        }
    }
    if (tid == 0) CTA_TIME(1);
    if (lane == 0) VSTEP_TIME(1, vstep);
}

int verify_cpb(int64_t V) {
    (void)V;
    return 1;
}


static int g_verify_grid = 0;  // SM count, set once by verify_prepare

template <bool BF16>
static void verify_prepare_t() {
    const size_t smem = (size_t)VerifyCfg<BF16>::kStages * 2 * kTileBytes;
    cudaFuncSetAttribute(verify_kernel<BF16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(verify_kernel<BF16, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(verify_kernel<BF16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(verify_kernel<BF16, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// Once per process, before any launch (see sched_prepare).
void verify_prepare() {
    verify_prepare_t<true>();
    verify_prepare_t<false>();
    cudaFuncSetAttribute(accept_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_verify_grid = sms;
}

int verify_grid(int32_t B, int32_t n_chunks, int32_t reserve_sms) {
    const int sms = g_verify_grid > 0 ? g_verify_grid : 148;
    const int64_t n_items = (int64_t)B * n_chunks;
    const int avail = sms - reserve_sms > 1 ? sms - reserve_sms : 1;  // SMs left for a concurrent kernel
    return n_items < avail ? (int)n_items : avail;
}

bool verify_fits(int32_t B, int32_t n_chunks, int32_t reserve_sms) {
    if (B <= 0) return true;
    const int g = verify_grid(B, n_chunks, reserve_sms);
    return B <= kMaxSlots && fin_slots(B, g, 0) <= kFinCap;
}

int verify_max_batch(int32_t n_chunks, int32_t reserve_sms) {
    int lo = 1, hi = 1 << 20;
    while (lo < hi) {  // largest B that fits (monotone in B)
        const int mid = lo + (hi - lo + 1) / 2;
        if (verify_fits(mid, n_chunks, reserve_sms)) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <bool BF16>
static cudaError_t launch_verify_t(const VerifyArgs &a, int32_t B, int32_t reserve_sms, bool pdl, cudaStream_t s) {
    const size_t smem = (size_t)VerifyCfg<BF16>::kStages * 2 * kTileBytes;
    // Finishers wait on other CTAs' chunks, so all CTAs must be resident together: each
    // CTA needs an SM's shared memory (one CTA per SM) and the grid is at most the SM
    // count minus the SMs left to the side-stream select.  No cooperative attribute: a
    // cooperative launch is serialised against other streams' kernels, which would
    // forbid exactly the overlap with the side kernel.  Device waits have a watchdog.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)verify_grid(B, a.n_chunks, reserve_sms));
    cfg.blockDim = dim3(kVerifyThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return a.check_rows ? cudaLaunchKernelEx(&cfg, verify_kernel<BF16, true>, a, B)
                        : cudaLaunchKernelEx(&cfg, verify_kernel<BF16, false>, a, B);
}

cudaError_t launch_verify_grid(const VerifyArgs &a, int32_t B, int32_t reserve_sms, bool pdl, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    if (!verify_fits(B, a.n_chunks, reserve_sms)) return cudaErrorInvalidValue;  // callers split / validate
    count_launch();
    return a.rows.dtype == LAPSSD_BF16 ? launch_verify_t<true>(a, B, reserve_sms, pdl, s)
                                       : launch_verify_t<false>(a, B, reserve_sms, pdl, s);
}

cudaError_t launch_verify(const VerifyArgs &a, int32_t B, cudaStream_t s) {
    return launch_verify_grid(a, B, 0, false, s);
}

}  // namespace lapssd
