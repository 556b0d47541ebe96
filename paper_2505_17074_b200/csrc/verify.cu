// verify.cu -- batched speculative verification by rejection sampling on sm_100a
// (Eq. 1, bonus token P:200; AMB-1, 2, 20, 21, 27).
//
// a1 (accept_kernel, or fused into the tail of select/merge): one thread per slot
//    gathers p_j(x_j), q_j(x_j) for the k drafts (independent loads) and applies the
//    exact fp64 test u24*q < p*2^24 with Philox uniforms -> r, in a 32-byte SlotDesc.
// a2 (verify_kernel): grid (ceil(n_chunks / cpb), B), 256 threads.  Every thread
//    reads the slot's descriptor with one broadcast load and immediately streams the
//    ONE row pair the algorithm needs -- (p_r, q_r), or p_k on full acceptance -- over
//    its cpb vocabulary chunks of 8192 entries with 128-bit L1::no_allocate loads,
//    reducing the exact Q4.60 residual mass R_v = floor(max(0, fl32(p-q)) * 2^60)
//    to one uint64 per (chunk, warp) (integer sums: exact, order-independent).  The
//    last CTA of the slot (threadfence + atomic ticket) totals Z, draws
//    t = floor(U Z / 2^64), finds the (chunk, warp) segment holding t from the stored
//    sums, rescans that one 1024-entry segment (L2-hot) with a warp inclusive scan,
//    emits y, and -- in laps_step -- runs the state update of that request (a3).
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
    d.pad[0] = d.pad[1] = d.pad[2] = 0;
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
// Persistent, warp-specialised, TMA-fed; one CTA per SM.  CTA = 8 consumer warps +
// 1 producer warp + 1 finisher warp.  Work item n = (slot b = n / n_chunks, chunk
// c = n % n_chunks); a CTA takes items blockIdx.x, blockIdx.x + gridDim.x, ...
//  producer: loads the descriptors of its next 32 items (one per lane), then issues
//            cp.async.bulk of chunk c of p_r (and q_r when r < k) into a ring of
//            shared-memory stages, completion tracked by mbarrier tx-count.
//  consumers: each warp reduces its 1024-entry segment of the stage to one uint64 and
//            publishes it with bit 63 as a ready flag (relaxed store); it then frees the
//            stage (empty barrier counts 8 warp arrivals).  No block-wide barrier, no
//            fence and no atomic on the streaming path.
//  finisher: for every slot whose designated chunk (b % n_chunks) this CTA consumed, polls until all
//            n_chunks*8 warp sums carry the flag, then totals, samples, emits, runs
//            the state update, and computes that request's next-round acceptance test
//            (cached for the next select).  Off the streaming path.
#ifdef LAPSSD_TRACE
// Diagnostic build only (tools/): fire-and-forget timestamps per (event, item) of two CTAs.
__device__ unsigned long long g_trace[2][16][1024];
__device__ __forceinline__ void trace(int ev, int x) {
    const int slot = blockIdx.x == 0 ? 0 : blockIdx.x == 74 ? 1 : -1;
    if (slot < 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[slot][ev][x & 1023] = t;
}
__device__ unsigned long long g_cta_t[2][160];   // first / last instruction per CTA
__device__ unsigned long long g_fs_trace[8];     // fused final select phases
extern "C" int lapssd_fs_trace_read(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_fs_trace, sizeof g_fs_trace); }
__device__ __forceinline__ void cta_time(int which) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 160) {
        if (which == 0) atomicMin(&g_cta_t[0][blockIdx.x], t); else atomicMax(&g_cta_t[1][blockIdx.x], t);
    }
}
extern "C" int lapssd_cta_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_cta_t, sizeof(g_cta_t));
    static unsigned long long init[2][160];
    for (int i = 0; i < 160; ++i) { init[0][i] = ~0ull; init[1][i] = 0; }
    cudaMemcpyToSymbol(g_cta_t, init, sizeof(init));
    return 0;
}
#define CTA_TIME(w) cta_time(w)
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
#endif
constexpr int kConsumerWarps = kWarps;                     // 8 per group
constexpr int kGroups = 2;                                 // consumer groups take alternate items
constexpr int kVerifyThreads = (1 + kGroups * (kConsumerWarps + 1)) * 32;  // producer + groups
constexpr int kFinQ = 64;                                  // finish-queue ring
constexpr int kStageBudget = 192 * 1024;                   // shared memory for the ring

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
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Published warp sums carry bit 63 as a ready flag (a segment's Q4.60 mass is < 2^61),
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
// The 8 published warp sums of chunk c (one lane per chunk): issued together.
__device__ __forceinline__ void load_chunk_words(const uint64_t *part, int c, uint64_t (&w)[kWarps]) {
#pragma unroll
    for (int h = 0; h < kWarps / 2; ++h) {
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
    float pj, qj;
    bool live;
};
template <bool BF16>
__device__ __forceinline__ NextA1 next_a1_load(const VerifyArgs &a, int32_t i, uint32_t round_next) {
    const int lane = threadIdx.x & 31;
    const RowsDev &rw = a.rows;
    NextA1 n;
    n.live = a.fuse_update && rw.slab_tab != nullptr && i >= 0;
    n.slab = 0;
    n.pj = 1.0f;
    n.qj = 0.0f;
    if (!n.live) return n;
    n.slab = rw.slab_tab[(int64_t)i * rw.R + slab_round_index((int32_t)round_next, rw.R)];
    const int k = rw.k;
    if (lane < k) {
        const int64_t V = rw.V;
        const int32_t x = rw.draft[n.slab * k + lane];
        const char *pb = (const char *)rw.p + n.slab * (int64_t)(k + 1) * V * Elt<BF16>::kEsz;
        const char *qb = (const char *)rw.q + n.slab * (int64_t)k * V * Elt<BF16>::kEsz;
        n.pj = BF16 ? load_prob_bf16(pb, (int64_t)lane * V + x) : load_prob_f32(pb, (int64_t)lane * V + x);
        n.qj = BF16 ? load_prob_bf16(qb, (int64_t)lane * V + x) : load_prob_f32(qb, (int64_t)lane * V + x);
    }
    return n;
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

// Warp-level finish of slot b: total Z, draw t, locate (chunk, warp segment), rescan
// that segment (L2-hot) in vocabulary order, emit, update.  P:64, AMB-20.
template <bool BF16>
__device__ __forceinline__ void finish_slot_warp(const VerifyArgs &a, int b, const SlotDesc &d, uint64_t (*fb)[kWarps],
                                                 uint64_t (&w0)[kWarps], uint64_t (&w1)[kWarps], const UpdIn &upd,
                                                 int64_t now, const NextA1 &nxt) {
    using E = Elt<BF16>;
    using S = Seg<BF16>;
    const int lane = threadIdx.x & 31;
    const int k = a.rows.k, r = d.r, nc = a.n_chunks;
    const int64_t V = a.rows.V;
    const bool use_q = r < k;
    const char *prow = (const char *)a.rows.p + ((int64_t)d.slab * (k + 1) + r) * V * E::kEsz;
    const char *qrow = (const char *)a.rows.q + ((int64_t)d.slab * k + (use_q ? r : 0)) * V * E::kEsz;
    const uint64_t *part = a.part + (int64_t)b * nc * kPartWords;
    // chunk sums from the words of the final poll: lane holds chunks lane and lane + 32
    uint64_t cs0 = 0, cs1 = 0;
#pragma unroll
    for (int x = 0; x < kWarps; ++x) {
        w0[x] &= ~kReady;
        w1[x] &= ~kReady;
        cs0 += w0[x];
        cs1 += w1[x];
    }
    uint64_t Z = warp_sum_u64(cs0 + cs1);
    if (lane == 0) TRACE(9, b);
    bool fallback = false;
    if (Z == 0 && use_q) {  // no residual mass while rejecting: the row p_r itself
        fallback = true;
        for (int c = 0; c < nc; ++c)
            for (int w = 0; w < kWarps; ++w) {
                const uint64_t m = warp_sum_u64(
                    lane_mass<BF16>(prow, qrow, false, (int64_t)c * kTile + (int64_t)w * kSegElems, V, lane));
                if (lane == 0) fb[c][w] = m;
            }
        __syncwarp();
        cs0 = cs1 = 0;
        if (lane < nc)
            for (int w = 0; w < kWarps; ++w) cs0 += fb[lane][w];
        if (lane + 32 < nc)
            for (int w = 0; w < kWarps; ++w) cs1 += fb[lane + 32][w];
        Z = warp_sum_u64(cs0 + cs1);
    }
    int y = -1;
    if (Z == 0) {
        if (a.err && lane == 0) atomicOr(a.err, E_NO_MASS);
        y = use_q ? a.rows.draft[(int64_t)d.slab * k + r] : 0;
    } else {
        const uint4 u = philox4x32_10(make_uint4(d.req, d.round, 1u << 8, a.trace), (uint32_t)a.seed,
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
        uint64_t wsum = 0;
#pragma unroll
        for (int x = 0; x < kWarps; ++x) {  // the 8 warp sums of chunk cstar, to lanes 0..7
            const uint64_t v = __shfl_sync(0xFFFFFFFFu, cstar < 32 ? w0[x] : w1[x], cstar & 31);
            if (lane == x) wsum = v;
        }
        if (fallback) wsum = lane < kWarps ? fb[cstar][lane] : 0;
        const uint64_t wincl = warp_incl_scan_u64(wsum, lane);
        const int wstar = __ffs(__ballot_sync(0xFFFFFFFFu, lane < kWarps && wincl > t)) - 1;
        t -= __shfl_sync(0xFFFFFFFFu, wincl - wsum, wstar);
        const int64_t base = (int64_t)cstar * kTile + (int64_t)wstar * kSegElems;
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
        st_relaxed(const_cast<uint64_t *>(part) + x, 0ull);
    if (lane == 0) {
        if (a.n_accept) a.n_accept[b] = r;
        if (a.z) a.z[b] = Z;
    }
    if (lane == 0) TRACE(12, b);
    if (a.fuse_update) {
        const UpdOut uo = update_warp(a.st, a.sc, d.i, r, now, upd, lane);
        if (lane == 0) TRACE(13, b);
        const int r_next = next_a1_store(a, d.i, d.req, d.round + 1, nxt);  // harmless if it completed
        if (a.fuse_select && lane == 0) {
            // the request's record for the fused final select: new key and next descriptor
            SelRec rec;
            rec.key = build_key(a.sc, d.i, INT32_MAX, uo.fl, upd.Lp, uo.tok, uo.A);
            rec.flags = uo.fl;
            rec.x_unset = 0;
            rec.desc.i = d.i;
            rec.desc.slab = (int32_t)nxt.slab;
            rec.desc.req = d.req;
            rec.desc.round = d.round + 1;
            rec.desc.r = r_next;
            rec.desc.pad[0] = rec.desc.pad[1] = rec.desc.pad[2] = 0;
            a.fin[b] = rec;
            a.st.key[d.i] = rec.key;
            __threadfence();
            if (a.pubq) {  // publish: the side-stream merger may take this slot now
                const uint32_t slot = atomicAdd(a.pubq, 1u);
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.pubq + 1 + slot), "r"((uint32_t)b + 1u)
                             : "memory");
            }
        }
    }
    __syncwarp();
}

template <bool BF16>
struct VerifyCfg {
    static constexpr int kTileBytes = kTile * Elt<BF16>::kEsz;        // one row chunk
    static constexpr int kStages = kStageBudget / (2 * kTileBytes);   // 6 (bf16) / 3 (fp32)
};

template <bool BF16>
__global__ void __launch_bounds__(kVerifyThreads, 1) verify_kernel(const __grid_constant__ VerifyArgs a,
                                                                    int32_t B) {
    using E = Elt<BF16>;
    using S = Seg<BF16>;
    constexpr int kTileBytes = VerifyCfg<BF16>::kTileBytes;
    constexpr int kStages = VerifyCfg<BF16>::kStages;
    extern __shared__ __align__(128) uint8_t s_tiles[];  // kStages x (p chunk, q chunk)
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ SlotDesc s_desc[kStages];
    __shared__ int s_chunk[kStages];
    __shared__ volatile int s_q[kGroups][kFinQ];
    __shared__ int4 s_qd[kGroups][kFinQ];      // (i, slab, req, round) of the queued slot
    __shared__ int s_qr[kGroups][kFinQ];       // its r
    __shared__ volatile int s_qhead[kGroups], s_qtail[kGroups];
    __shared__ uint64_t s_fb[kGroups][kMaxChunks][kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nc = a.n_chunks;
    const int n_items = B * nc;
    if (tid == 0) CTA_TIME(0);
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int g = 0; g < kGroups; ++g) { s_qhead[g] = 0; s_qtail[g] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        const int kk = a.rows.k;
        const int64_t V = a.rows.V;
        int k = 0;
        for (int base = blockIdx.x; base < n_items; base += 32 * gridDim.x) {
            // lane l prefetches the descriptor of item base + l * gridDim.x
            const int my_n = base + lane * (int)gridDim.x;
            SlotDesc md;
            md.r = -1;
            md.i = md.slab = 0;
            md.req = md.round = 0;
            if (my_n < n_items) {
                const int b = my_n / nc;
                md = a.desc[b];
                if (md.r >= 0 && a.sel) {
                    const int si = a.sel[b];
                    if (si != md.i) {
                        if (a.err) atomicOr(a.err, E_STALE_DESC);
                        md.r = -1;
                    }
                }
            }
            for (int j = 0; j < 32; ++j, ++k) {
                const int n = base + j * (int)gridDim.x;
                if (n >= n_items) break;
                const int r = __shfl_sync(0xFFFFFFFFu, md.r, j);
                const int slab = __shfl_sync(0xFFFFFFFFu, md.slab, j);
                const int di = __shfl_sync(0xFFFFFFFFu, md.i, j);
                const uint32_t req = __shfl_sync(0xFFFFFFFFu, md.req, j);
                const uint32_t rnd = __shfl_sync(0xFFFFFFFFu, md.round, j);
                if (lane == 0) {
                    const int st = k % kStages;
                    TRACE(1, k);
                    if (k >= kStages) mbar_wait(&empty[st], ((k / kStages) - 1) & 1);
                    TRACE(2, k);
                    const int c = n % nc;
                    SlotDesc d;
                    d.i = di; d.slab = slab; d.req = req; d.round = rnd; d.r = r;
                    d.pad[0] = d.pad[1] = d.pad[2] = 0;
                    s_desc[st] = d;
                    s_chunk[st] = c;
                    if (r < 0) {
                        mbar_arrive(&full[st]);
                    } else {
                        const bool use_q = r < kk;
                        const int64_t e0 = (int64_t)c * kTile;
                        const int64_t ne = V - e0 < kTile ? V - e0 : kTile;
                        const uint32_t bytes = (uint32_t)(ne * E::kEsz);
                        uint8_t *dst = s_tiles + (size_t)st * 2 * kTileBytes;
                        const char *prow = (const char *)a.rows.p + ((int64_t)slab * (kk + 1) + r) * V * E::kEsz;
                        mbar_arrive_tx(&full[st], use_q ? 2 * bytes : bytes);
                        tma_load_1d(dst, prow + e0 * E::kEsz, bytes, &full[st]);
                        if (use_q) {
                            const char *qrow = (const char *)a.rows.q + ((int64_t)slab * kk + r) * V * E::kEsz;
                            tma_load_1d(dst + kTileBytes, qrow + e0 * E::kEsz, bytes, &full[st]);
                        }
                    }
                    TRACE(8, k);
                }
                __syncwarp();
            }
        }
    } else {
    const int grp = (warp - 1) / (kConsumerWarps + 1);
    const int gw = (warp - 1) % (kConsumerWarps + 1);  // 0..7 consumer, 8 finisher
    if (gw == kConsumerWarps) {
        // ------------------------------------------------------------ finisher of group grp
        int head = 0;
        for (;;) {
            while (head == s_qtail[grp]) __nanosleep(32);
            const int b = s_q[grp][head % kFinQ];
            SlotDesc d;
            d.i = s_qd[grp][head % kFinQ].x;
            d.slab = s_qd[grp][head % kFinQ].y;
            d.req = (uint32_t)s_qd[grp][head % kFinQ].z;
            d.round = (uint32_t)s_qd[grp][head % kFinQ].w;
            d.r = s_qr[grp][head % kFinQ];
            ++head;
            __syncwarp();
            if (lane == 0) s_qhead[grp] = head;
            if (b < 0) break;
            if (lane == 0) TRACE(5, b);
            // independent work first, overlapping the wait for the other CTAs' chunks:
            // the state update's inputs and the next round's acceptance-test chain
            UpdIn upd{};
            int64_t now = 0;
            if (a.fuse_update) {
                upd = load_update_inputs(a.st, a.sc, d.i, lane);
                now = a.st.g->now_us;
            }
            const NextA1 nxt = next_a1_load<BF16>(a, d.i, d.round + 1);
            const uint64_t *pw = a.part + (int64_t)b * nc * kPartWords;
            uint64_t w0[kWarps], w1[kWarps];
            const unsigned long long t_start = gtimer();
            for (;;) {  // every (chunk, warp) sum of slot b published?
#pragma unroll
                for (int x = 0; x < kWarps; ++x) w0[x] = w1[x] = kReady;
                if (lane < nc) load_chunk_words(pw, lane, w0);
                if (lane + 32 < nc) load_chunk_words(pw, lane + 32, w1);
                bool ready = true;
#pragma unroll
                for (int x = 0; x < kWarps; ++x) ready &= ((w0[x] & w1[x]) & kReady) != 0;
                if (__all_sync(0xFFFFFFFFu, ready)) break;
                if (waited_too_long(t_start)) {
                    if (lane == 0 && a.err) atomicOr(a.err, E_TIMEOUT);
                    break;
                }
                __nanosleep(32);
            }
            if (lane == 0) TRACE(6, b);
            finish_slot_warp<BF16>(a, b, d, s_fb[grp], w0, w1, upd, now, nxt);
            if (lane == 0) TRACE(7, b);
        }
        if (lane == 0) CTA_TIME(1);
    } else {
    // ---------------------------------------------------------------- consumers of group grp
    int k = grp;
    const int warp_seg = gw;  // this warp's 1024-entry segment of every chunk
    for (int n = blockIdx.x + grp * (int)gridDim.x; n < n_items; n += kGroups * (int)gridDim.x, k += kGroups) {
        const int st = k % kStages;
        mbar_wait(&full[st], (k / kStages) & 1);
        if (warp_seg == 0 && lane == 0) TRACE(3, k);
        const SlotDesc d = s_desc[st];
        const int c = s_chunk[st];
        const int b = n / nc;
        if (d.r >= 0) {
            const uint4 qmask = d.r < a.rows.k ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0, 0, 0, 0);
            const uint4 *tp = reinterpret_cast<const uint4 *>(s_tiles + (size_t)st * 2 * kTileBytes);
            const uint4 *tq = tp + kTileBytes / 16;
            const int64_t e_base = (int64_t)c * kTile + (int64_t)warp_seg * kSegElems;
            const int64_t V = a.rows.V;
            uint4 pv[S::J], qv[S::J];
#pragma unroll
            for (int j = 0; j < S::J; ++j) {  // branch-free: load, then mask the tail / absent q
                const int v = warp_seg * (kSegElems / S::kVec) + j * 32 + lane;
                pv[j] = tp[v];
                qv[j] = tq[v];
            }
            uint64_t m = 0;
#pragma unroll
            for (int j = 0; j < S::J; ++j) {
                const bool in = e_base + (int64_t)(j * 32 + lane) * S::kVec < V;
                const uint4 z = make_uint4(0, 0, 0, 0);
                const uint4 pm = in ? pv[j] : z;  // beyond V the stage holds stale bytes
                const uint4 qm = in ? make_uint4(qv[j].x & qmask.x, qv[j].y & qmask.y, qv[j].z & qmask.z,
                                                 qv[j].w & qmask.w)
                                    : z;
                m += E::mass(pm, qm);
            }
            m = warp_sum_u64(m);
            if (lane == 0) st_relaxed(&a.part[((int64_t)b * nc + c) * kPartWords + warp_seg], m | kReady);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (warp_seg == 0 && lane == 0) TRACE(4, k);
        // slot b is finished by the CTA that consumed its chunk b % nc: spreads the
        // finishing over all CTAs whatever gcd(gridDim, nc) is
        if (d.r >= 0 && c == b % nc && warp_seg == 0 && lane == 0) {
            while (s_qtail[grp] - s_qhead[grp] >= kFinQ) __nanosleep(32);
            s_q[grp][s_qtail[grp] % kFinQ] = b;
            s_qd[grp][s_qtail[grp] % kFinQ] = make_int4(d.i, d.slab, (int)d.req, (int)d.round);
            s_qr[grp][s_qtail[grp] % kFinQ] = d.r;
            __threadfence_block();
            s_qtail[grp] = s_qtail[grp] + 1;
        }
    }
    if (warp_seg == 0 && lane == 0) {
        while (s_qtail[grp] - s_qhead[grp] >= kFinQ) __nanosleep(32);
        s_q[grp][s_qtail[grp] % kFinQ] = -1;
        __threadfence_block();
        s_qtail[grp] = s_qtail[grp] + 1;
    }
    }  // consumers
    }  // consumer groups / finishers
    if (tid == 0) CTA_TIME(1);
    // ------------------------------------------------------------ fused final select
    if (a.fuse_select && !a.pubq) {
        __shared__ int s_last;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            s_last = atomicAdd(a.done_ctas, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
#ifdef LAPSSD_TRACE
            unsigned long long *trp = g_fs_trace;
#else
            unsigned long long *trp = nullptr;
#endif
            fused_final_select(a.st, a.sc, B, const_cast<int32_t *>(a.sel), const_cast<SlotDesc *>(a.desc), a.fin,
                               a.pre, a.count_out, reinterpret_cast<uint64_t *>(s_tiles), trp);
            if (tid == 0) *a.done_ctas = 0;
        }
    }
}

int verify_cpb(int64_t V) {
    (void)V;
    return 1;
}

static int g_verify_grid = 0;

template <bool BF16>
static void verify_prepare_t() {
    const size_t smem = (size_t)VerifyCfg<BF16>::kStages * 2 * VerifyCfg<BF16>::kTileBytes;
    cudaFuncSetAttribute(verify_kernel<BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(verify_kernel<BF16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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

template <bool BF16>
static cudaError_t launch_verify_t(const VerifyArgs &a, int32_t B, int32_t reserve_sms, cudaStream_t s) {
    const size_t smem = (size_t)VerifyCfg<BF16>::kStages * 2 * VerifyCfg<BF16>::kTileBytes;
    const int grid = g_verify_grid > 0 ? g_verify_grid : 148;
    const int n_items = B * a.n_chunks;
    const int avail = grid - reserve_sms > 1 ? grid - reserve_sms : 1;  // SMs left for a concurrent kernel
    const int g = n_items < avail ? n_items : avail;
    // Finishers wait on other CTAs' chunks, so all CTAs must be resident together: each
    // CTA needs an SM's shared memory (one CTA per SM) and the grid is at most the SM
    // count minus the SMs left to the side-stream select.  No cooperative attribute: a
    // cooperative launch is serialised against other streams' kernels, which would
    // forbid exactly the overlap with the side kernel.  Device waits have a watchdog.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(kVerifyThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, verify_kernel<BF16>, a, B);
}

cudaError_t launch_verify_grid(const VerifyArgs &a, int32_t B, int32_t reserve_sms, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    count_launch();
    return a.rows.dtype == LAPSSD_BF16 ? launch_verify_t<true>(a, B, reserve_sms, s)
                                       : launch_verify_t<false>(a, B, reserve_sms, s);
}

cudaError_t launch_verify(const VerifyArgs &a, int32_t B, cudaStream_t s) { return launch_verify_grid(a, B, 0, s); }

}  // namespace lapssd
