// verify.cu -- K_verify: batched speculative verification by rejection sampling on
// sm_100a (Eq. 1, bonus token P:200; AMB-1, 2, 20, 21, 27).
//
// One CTA = one (slot b, vocabulary chunk c) tile.  Grid (n_chunks, B).
//  1. Every CTA re-derives the first rejected position r_b from <= k gathered
//     scalars p_j(x_j), q_j(x_j) and Philox uniforms (warp 0, one lane per j).
//  2. It streams chunk c of the ONE row pair the algorithm needs -- (p_r, q_r), or
//     p_k on full acceptance -- with 128-bit L1::no_allocate loads, and reduces the
//     exact Q4.60 residual mass R_v = floor(max(0, fl32(p - q)) * 2^60) to one
//     uint64 per warp and per chunk (integer sums: order-independent, exact).
//  3. The last CTA to finish slot b (threadfence + atomic ticket) totals Z, draws
//     t = floor(U Z / 2^64), locates the chunk and warp segment holding t from the
//     stored partial sums, rescans that one 1024-element segment (L2-hot) with a
//     warp inclusive scan, emits y, and -- in laps_step -- runs the LAPS-SD state
//     update of that request (fused a3).
// HBM bytes per slot: 2 V s (r < k) or V s (r = k), plus k gathered scalars.
#include <cuda_bf16.h>

#include "lapssd_internal.cuh"

namespace lapssd {

__device__ __forceinline__ uint4 ld_stream(const void *ptr) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr));
    return r;
}

// Q4.60 residual mass of one entry.  fl32 subtraction (round to nearest), exact
// power-of-two scaling, truncating conversion; cvt.rzi.u64.f32 clamps to the
// destination range, so d <= 0 (and NaN) gives 0.
__device__ __forceinline__ uint64_t q460(float p, float q) {
    return __float2ull_rz(__fmul_rn(__fsub_rn(p, q), 0x1p60f));
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <bool BF16> struct Elt;
template <> struct Elt<true> {
    static constexpr int kVec = 8;  // bf16 per 16-byte vector
    __device__ static float load1(const void *base, int64_t idx) {
        const uint16_t b = reinterpret_cast<const uint16_t *>(base)[idx];
        return __uint_as_float((uint32_t)b << 16);
    }
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
    __device__ static float load1(const void *base, int64_t idx) {
        return reinterpret_cast<const float *>(base)[idx];
    }
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
    static constexpr int J = kSegElems / kVec / 32;  // vectors per lane per segment
    static constexpr int kEsz = BF16 ? 2 : 4;

    // Load this lane's J vectors of the warp segment starting at element `base`.
    __device__ static void load(const char *row, int64_t base, int64_t V, int lane, uint4 (&v)[J]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t e = base + (int64_t)(j * 32 + lane) * kVec;
            v[j] = e < V ? ld_stream(row + e * kEsz) : make_uint4(0, 0, 0, 0);
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

// Residual mass of one lane's share of a warp segment.
template <bool BF16>
__device__ __forceinline__ uint64_t lane_mass(const char *prow, const char *qrow, bool use_q,
                                              int64_t base, int64_t V, int lane) {
    using S = Seg<BF16>;
    uint4 pv[S::J], qv[S::J];
    S::load(prow, base, V, lane, pv);
    if (use_q) {
        S::load(qrow, base, V, lane, qv);
    } else {
#pragma unroll
        for (int j = 0; j < S::J; ++j) qv[j] = make_uint4(0, 0, 0, 0);
    }
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < S::J; ++j) s += Elt<BF16>::mass(pv[j], qv[j]);
    return s;
}

template <bool BF16>
__global__ void __launch_bounds__(kThreads, 2) verify_kernel(const VerifyArgs a) {
    using E = Elt<BF16>;
    using S = Seg<BF16>;
    constexpr int kEsz = S::kEsz;
    const int c = blockIdx.x;
    const int b = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = a.k;
    const int64_t V = a.V;

    __shared__ int s_r, s_i, s_last, s_invalid;
    __shared__ int64_t s_slab;
    __shared__ uint32_t s_req, s_round;
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_cs[kMaxChunks];
    __shared__ uint64_t s_fb_ws[kMaxChunks][kWarps];
    __shared__ uint64_t s_Z, s_tl;
    __shared__ int s_cstar, s_wstar, s_y, s_fallback;

    // ---- 1. which request / round / slab, and r (warp 0)
    if (warp == 0) {
        int i = 0;
        uint32_t req = 0, rnd = 0;
        int64_t slab = b;
        if (a.sel) {
            i = a.sel[b];
            if (i >= 0) {
                rnd = (uint32_t)a.st.rounds[i];
                req = (uint32_t)(i * a.sc.world + a.sc.rank);
                if (a.slab_tab)
                    slab = a.slab_tab[(int64_t)i * a.R + slab_round_index((int32_t)rnd, a.R)];
            }
        } else {
            req = a.req_id[b];
            rnd = a.round_idx[b];
            if (a.slab) slab = a.slab[b];
        }
        bool reject = false;
        if (i >= 0 && lane < k) {
            const int32_t x = a.draft[slab * k + lane];
            const char *pb = (const char *)a.p + slab * (int64_t)(k + 1) * V * kEsz;
            const char *qb = (const char *)a.q + slab * (int64_t)k * V * kEsz;
            const float pj = E::load1(pb, (int64_t)lane * V + x);
            const float qj = E::load1(qb, (int64_t)lane * V + x);
            const uint4 u = philox4x32_10(make_uint4(req, rnd, (uint32_t)(lane >> 2), a.trace),
                                          (uint32_t)a.seed, (uint32_t)(a.seed >> 32));
            const uint32_t w = (lane & 3) == 0 ? u.x : (lane & 3) == 1 ? u.y : (lane & 3) == 2 ? u.z : u.w;
            const uint32_t u24 = w >> 8;
            // accept iff u24 * q < p * 2^24 (exact in fp64): u < p/q with u = u24 / 2^24
            reject = !(__dmul_rn((double)u24, (double)qj) < __dmul_rn((double)pj, 16777216.0));
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, reject);
        if (lane == 0) {
            s_r = i < 0 ? -1 : (m ? __ffs(m) - 1 : k);
            s_i = i;
            s_slab = slab;
            s_req = req;
            s_round = rnd;
        }
    }
    __syncthreads();
    const int r = s_r;
    if (r < 0) return;  // empty slot
    const int64_t slab = s_slab;
    const bool use_q = r < k;
    const char *prow = (const char *)a.p + (slab * (int64_t)(k + 1) + r) * V * kEsz;
    const char *qrow = (const char *)a.q + (slab * (int64_t)k + (use_q ? r : 0)) * V * kEsz;

    // ---- 2. stream chunk c, per-warp and per-chunk exact residual mass
    const int64_t seg_base = (int64_t)c * kTile + (int64_t)warp * kSegElems;
    const uint64_t ws = warp_sum_u64(lane_mass<BF16>(prow, qrow, use_q, seg_base, V, lane));
    if (lane == 0) s_warp[warp] = ws;
    __syncthreads();
    const int nc = a.n_chunks;
    uint64_t *part = a.part + (int64_t)b * nc * kPartWords;
    if (tid == 0) {
        uint64_t cs = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            cs += s_warp[w];
            part[(int64_t)c * kPartWords + 1 + w] = s_warp[w];
        }
        part[(int64_t)c * kPartWords] = cs;
        __threadfence();
        const unsigned ticket = atomicAdd(&a.counter[b], 1u);
        s_last = ticket == (unsigned)(nc - 1);
    }
    __syncthreads();
    if (!s_last) return;

    // ---- 3. last CTA of slot b: total, sample, emit, update
    __threadfence();
    for (int c2 = tid; c2 < nc; c2 += kThreads) s_cs[c2] = __ldcg(&part[(int64_t)c2 * kPartWords]);
    __syncthreads();
    if (tid == 0) {
        uint64_t Z = 0;
        for (int c2 = 0; c2 < nc; ++c2) Z += s_cs[c2];
        s_Z = Z;
        s_fallback = (Z == 0 && use_q) ? 1 : 0;
    }
    __syncthreads();
    const bool fallback = s_fallback != 0;
    if (fallback) {
        // AMB-20: no residual mass while rejecting -> sample from p_r itself.
        for (int c2 = 0; c2 < nc; ++c2) {
            const uint64_t w2 = warp_sum_u64(
                lane_mass<BF16>(prow, qrow, false, (int64_t)c2 * kTile + (int64_t)warp * kSegElems, V, lane));
            if (lane == 0) s_fb_ws[c2][warp] = w2;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t Z = 0;
            for (int c2 = 0; c2 < nc; ++c2) {
                uint64_t cs = 0;
                for (int w = 0; w < kWarps; ++w) cs += s_fb_ws[c2][w];
                s_cs[c2] = cs;
                Z += cs;
            }
            s_Z = Z;
        }
        __syncthreads();
    }
    const uint64_t Z = s_Z;
    const bool q_in_mass = use_q && !fallback;
    if (tid == 0) {
        s_invalid = Z == 0;
        if (Z != 0) {
            const uint4 u = philox4x32_10(make_uint4(s_req, s_round, 1u << 8, a.trace),
                                          (uint32_t)a.seed, (uint32_t)(a.seed >> 32));
            const uint64_t U = ((uint64_t)u.x << 32) | u.y;
            uint64_t t = __umul64hi(U, Z);  // floor(U Z / 2^64) in [0, Z)
            int cs = nc - 1;
            for (int c2 = 0; c2 < nc; ++c2) {
                if (t < s_cs[c2]) { cs = c2; break; }
                t -= s_cs[c2];
            }
            int wsel = kWarps - 1;
            for (int w = 0; w < kWarps; ++w) {
                const uint64_t m = fallback ? s_fb_ws[cs][w] : __ldcg(&part[(int64_t)cs * kPartWords + 1 + w]);
                if (t < m) { wsel = w; break; }
                t -= m;
            }
            s_cstar = cs;
            s_wstar = wsel;
            s_tl = t;
        }
    }
    __syncthreads();
    if (s_invalid) {
        if (tid == 0) {
            atomicOr(&a.st.g->err, E_NO_MASS);
            s_y = use_q ? a.draft[slab * k + r] : 0;
        }
    } else if (warp == 0) {
        // rescan the one warp segment that holds t, in element order
        const int64_t base = (int64_t)s_cstar * kTile + (int64_t)s_wstar * kSegElems;
        uint4 pv[S::J], qv[S::J];
        S::load(prow, base, V, lane, pv);
        if (q_in_mass) {
            S::load(qrow, base, V, lane, qv);
        } else {
#pragma unroll
            for (int j = 0; j < S::J; ++j) qv[j] = make_uint4(0, 0, 0, 0);
        }
        uint64_t tl = s_tl;
        int y = -1;
#pragma unroll
        for (int j = 0; j < S::J; ++j) {
            const uint64_t m = E::mass(pv[j], qv[j]);
            const uint64_t incl = warp_incl_scan_u64(m, lane);
            const uint64_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            if (y < 0) {
                if (tl < tot) {
                    const unsigned hit = __ballot_sync(0xFFFFFFFFu, incl > tl);
                    const int src = __ffs(hit) - 1;
                    int yy = -1;
                    if (lane == src) {
                        uint64_t tt = tl - (incl - m);
                        for (int e = 0; e < S::kVec; ++e) {
                            const uint64_t me = q460(E::elem(pv[j], e), E::elem(qv[j], e));
                            if (tt < me) { yy = e; break; }
                            tt -= me;
                        }
                        yy = (int)(base + (int64_t)(j * 32 + lane) * S::kVec + yy);
                    }
                    y = __shfl_sync(0xFFFFFFFFu, yy, src);
                } else {
                    tl -= tot;
                }
            }
        }
        if (lane == 0) s_y = y;
    }
    __syncthreads();
    if (tid == 0) {
        const int y = s_y;
        if (a.tokens) {
            int32_t *tok = a.tokens + (int64_t)b * (k + 1);
            for (int j = 0; j < r; ++j) tok[j] = a.draft[slab * k + j];
            tok[r] = y;
            for (int j = r + 1; j <= k; ++j) tok[j] = -1;
        }
        if (a.n_accept) a.n_accept[b] = r;
        if (a.z) a.z[b] = Z;
        a.counter[b] = 0;  // leave the ticket zeroed for the next launch / graph replay
        if (a.fuse_update && a.sel) update_one(a.st, a.sc, s_i, r, a.st.g->now_us);
    }
}

cudaError_t launch_verify(const VerifyArgs &a, int32_t dtype, int32_t B, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    const dim3 grid((unsigned)a.n_chunks, (unsigned)B);
    if (dtype == LAPSSD_BF16)
        verify_kernel<true><<<grid, kThreads, 0, s>>>(a);
    else
        verify_kernel<false><<<grid, kThreads, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lapssd
