// verify_logits.cu -- verification from LOGITS on sm_100a (Eq. 1
// and P:200 with p = softmax of the target head's logits, q = softmax of the draft
// head's; DESIGN.md AMB-30).
//
// The softmax is quantised so that every decision is an exact integer comparison and
// the result is a pure function of the inputs (bit-identical to the oracle):
//   m_j = max_v z_j[v];  E_j[v] = floor(exphat(fl32(z_j[v] - m_j)) * 2^40);
//   S_j = sum_v E_j[v];  p^_j(v) = E_j[v] / S_j,
// with exphat a FIXED sequence of IEEE fp32 operations (rint, fma, exact 2^n scaling).
// a1: accept x_j iff u24 * Eq * Sp < 2^24 * Ep * Sq (128-bit integers).
// a2: R_v = max(0, Ep_v Sq - Eq_v Sp) (r < k) or Ep_v (r = k); t = floor(U Z / 2^64);
//     y = min{v : sum_{w<=v} R_w > t} (128-bit integers).
//
// norm_kernel: one CTA per (slot, row) of the 2k+1 rows: max, then the integer mass
//   (a second read of the row), ~14 issue slots per entry for the exp (packed fp32x2).
// sample_kernel: one CTA per slot: the k acceptance tests (one lane each), then the
//   residual row pair in 1,024-entry tiles (warp-coalesced 16-byte loads, one tile sum
//   per warp pass), the tile holding t found by warp 0, which rescans that tile.
#include "lapssd_internal.cuh"

namespace lapssd {

typedef unsigned __int128 u128;

// E = floor(exphat(fl32(z - m)) * 2^40) for the exphat of DESIGN.md AMB-30 (the oracle
// writes out the same operation sequence; nothing is shared).  rint(x) for |x| < 2^22
// is (x + 1.5 2^23) - 1.5 2^23 in RN-even, and n sits in the low bits of that sum; the
// final P 2^n 2^40 is one exact multiply by a constructed power of two, then a
// truncating conversion.
// Two entries at once with the packed fp32x2 pipe (FFMA2/FADD2/FMUL2: each half is the
// IEEE RN operation of the definition).  d is clamped to [-28.5, 0]: below -28 the
// definition gives 0, and so does the polynomial there (e^-28 2^40 < 0.77), while the
// clamp keeps 2^n normal.
__device__ __forceinline__ void e40x2(float za, float zb, float ma, float mb, uint64_t &ea, uint64_t &eb) {
    const float2 d0 = __fadd2_rn(make_float2(za, zb), make_float2(-ma, -mb));
    const float2 d = make_float2(fmaxf(fminf(d0.x, 0.0f), -28.5f), fmaxf(fminf(d0.y, 0.0f), -28.5f));
    const float2 x = __fmul2_rn(d, make_float2(0x1.715476p+0f, 0x1.715476p+0f));
    const float2 big = __fadd2_rn(x, make_float2(0x1.8p23f, 0x1.8p23f));
    const float2 nf = __fadd2_rn(big, make_float2(-0x1.8p23f, -0x1.8p23f));
    float2 r = __ffma2_rn(nf, make_float2(-0x1.62e4p-1f, -0x1.62e4p-1f), d);
    r = __ffma2_rn(nf, make_float2(-0x1.7f7d1cp-20f, -0x1.7f7d1cp-20f), r);
    float2 p = make_float2(0x1.a01a02p-13f, 0x1.a01a02p-13f);
    p = __ffma2_rn(p, r, make_float2(0x1.6c16c2p-10f, 0x1.6c16c2p-10f));
    p = __ffma2_rn(p, r, make_float2(0x1.111112p-7f, 0x1.111112p-7f));
    p = __ffma2_rn(p, r, make_float2(0x1.555556p-5f, 0x1.555556p-5f));
    p = __ffma2_rn(p, r, make_float2(0x1.555556p-3f, 0x1.555556p-3f));
    p = __ffma2_rn(p, r, make_float2(0x1p-1f, 0x1p-1f));
    p = __ffma2_rn(p, r, make_float2(1.0f, 1.0f));
    p = __ffma2_rn(p, r, make_float2(1.0f, 1.0f));
    const int na = __float_as_int(big.x) - 0x4B400000, nb = __float_as_int(big.y) - 0x4B400000;
    const float2 sc = make_float2(__int_as_float((167 + na) << 23), __int_as_float((167 + nb) << 23));
    const float2 f = __fmul2_rn(p, sc);   // P 2^(n+40), exact
    ea = __float2ull_rz(f.x);
    eb = __float2ull_rz(f.y);
}

__device__ __forceinline__ uint64_t e40(float z, float m) {
    uint64_t a, b;
    e40x2(z, z, m, m, a, b);
    return a;
}

template <bool BF16> struct LElt;
template <> struct LElt<true> {
    static constexpr int kVec = 8, kEsz = 2;
    __device__ static float get(const uint4 &v, int e) {
        const uint32_t w = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
        return __uint_as_float((e & 1) ? (w & 0xFFFF0000u) : (w << 16));
    }
};
template <> struct LElt<false> {
    static constexpr int kVec = 4, kEsz = 4;
    __device__ static float get(const uint4 &v, int e) {
        return __uint_as_float(e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w);
    }
};

__device__ __forceinline__ u128 shfl_xor_u128(u128 v, int o) {
    const uint64_t lo = __shfl_xor_sync(0xFFFFFFFFu, (uint64_t)v, o);
    const uint64_t hi = __shfl_xor_sync(0xFFFFFFFFu, (uint64_t)(v >> 64), o);
    return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ u128 shfl_up_u128(u128 v, int o) {
    const uint64_t lo = __shfl_up_sync(0xFFFFFFFFu, (uint64_t)v, o);
    const uint64_t hi = __shfl_up_sync(0xFFFFFFFFu, (uint64_t)(v >> 64), o);
    return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
    const uint64_t lo = __shfl_sync(0xFFFFFFFFu, (uint64_t)v, src);
    const uint64_t hi = __shfl_sync(0xFFFFFFFFu, (uint64_t)(v >> 64), src);
    return ((u128)hi << 64) | lo;
}

#ifndef LAPSSD_SAMPLE_THREADS
#define LAPSSD_SAMPLE_THREADS 512
#endif
#ifndef LAPSSD_SAMPLE_MINB
#define LAPSSD_SAMPLE_MINB 2
#endif
constexpr int kLogitThreads = LAPSSD_SAMPLE_THREADS;   // sample kernel: one slot per CTA

// ---------------------------------------------------------------- row normalisers
// Block (slot b, row ri): ri <= k is target row ri, else draft row ri - k - 1.  Two passes
// over the row: the max, then the integer masses (measured: ~4 CTAs per SM keep both the
// HBM stream and the exp arithmetic busy; a one-CTA-per-SM persistent form whose second
// pass hits L2, and a 4-8 CTA cluster holding the row in shared memory, were slower).
constexpr int kNormThreads = 512;

template <bool BF16>
__global__ void __launch_bounds__(kNormThreads) logits_norm_kernel(const char *zp, const char *zq,
                                                                   const int32_t *slab, int64_t V, int32_t k,
                                                                   float *m_out, uint64_t *S_out) {
    using E = LElt<BF16>;
    const int rows = 2 * k + 1;
    const int b = blockIdx.x / rows, ri = blockIdx.x % rows;
    const int64_t s = slab ? slab[b] : b;
    const char *row = ri <= k ? zp + ((s * (k + 1) + ri) * V) * E::kEsz
                              : zq + ((s * k + (ri - k - 1)) * V) * E::kEsz;
    const uint4 *v4 = reinterpret_cast<const uint4 *>(row);
    const int64_t nv = V / E::kVec;
    __shared__ float s_m[kNormThreads / 32];
    __shared__ uint64_t s_S[kNormThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float m = -INFINITY;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const uint4 v = v4[i];
#pragma unroll
        for (int e = 0; e < E::kVec; ++e) m = fmaxf(m, E::get(v, e));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (lane == 0) s_m[warp] = m;
    __syncthreads();
    m = s_m[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s_m[w]);
    uint64_t S = 0;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const uint4 v = v4[i];
#pragma unroll
        for (int e = 0; e < E::kVec; e += 2) {
            uint64_t a, c;
            e40x2(E::get(v, e), E::get(v, e + 1), m, m, a, c);
            S += a + c;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xFFFFFFFFu, S, o);
    if (lane == 0) s_S[warp] = S;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_S[w];
        m_out[(int64_t)b * rows + ri] = m;
        S_out[(int64_t)b * rows + ri] = t;
    }
}

// ---------------------------------------------------------------- accept + residual draw
constexpr int kTileVecs = 4;   // vectors per lane per tile: 1,024 bf16 / 512 fp32 entries

template <bool BF16>
__device__ __forceinline__ u128 entry_mass(float zp, float zq, float mp, float mq, uint64_t Sp, uint64_t Sq,
                                           bool use_q) {
    uint64_t ep, eq;
    e40x2(zp, zq, mp, mq, ep, eq);
    if (!use_q) return (u128)ep;
    const u128 x = (u128)ep * Sq, y = (u128)eq * Sp;
    return x > y ? x - y : 0;
}

template <bool BF16>
__global__ void __launch_bounds__(kLogitThreads, LAPSSD_SAMPLE_MINB) logits_sample_kernel(
    const char *zp, const char *zq, const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
    const uint32_t *round_idx, int64_t V, int32_t k, uint64_t seed, uint32_t trace, const float *m_in,
    const uint64_t *S_in, int32_t *tokens, int32_t *n_accept, uint64_t *z_out, uint32_t *err) {
    using E = LElt<BF16>;
    constexpr int kTile = 32 * kTileVecs * E::kVec;
    extern __shared__ __align__(16) uint8_t s_raw[];
    u128 *tile_sum = reinterpret_cast<u128 *>(s_raw);
    __shared__ int s_r;
    const int b = blockIdx.x;
    const int rows = 2 * k + 1;
    const int64_t s = slab ? slab[b] : b;
    const uint32_t req = req_id[b], rnd = round_idx[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const float *m = m_in + (int64_t)b * rows;
    const uint64_t *S = S_in + (int64_t)b * rows;
    const int32_t *dr = draft + s * k;
    // ---- a1: position j on lane j of warp 0 (k <= 16), first rejection by ballot
    if (warp == 0) {
        bool reject = false;
        if (lane < k) {
            const int x = dr[lane];
            const char *prow = zp + ((s * (k + 1) + lane) * V) * E::kEsz;
            const char *qrow = zq + ((s * k + lane) * V) * E::kEsz;
            const float zpx = BF16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(prow)[x] << 16)
                                   : reinterpret_cast<const float *>(prow)[x];
            const float zqx = BF16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(qrow)[x] << 16)
                                   : reinterpret_cast<const float *>(qrow)[x];
            const uint64_t Ep = e40(zpx, m[lane]), Eq = e40(zqx, m[k + 1 + lane]);
            const uint4 u = philox4x32_10(make_uint4(req, rnd, (uint32_t)(lane >> 2), trace), (uint32_t)seed,
                                          (uint32_t)(seed >> 32));
            const uint32_t w = (lane & 3) == 0 ? u.x : (lane & 3) == 1 ? u.y : (lane & 3) == 2 ? u.z : u.w;
            const uint32_t u24 = w >> 8;
            reject = !((u128)u24 * Eq * S[lane] < (((u128)Ep * S[k + 1 + lane]) << 24));
        }
        const unsigned msk = __ballot_sync(0xFFFFFFFFu, reject);
        if (lane == 0) s_r = msk ? __ffs(msk) - 1 : k;
    }
    __syncthreads();
    const int r = s_r;
    bool use_q = r < k;
    const float mp = m[r];
    const uint64_t Sp = S[r];
    const float mq = use_q ? m[k + 1 + r] : 0.0f;
    const uint64_t Sq = use_q ? S[k + 1 + r] : 0;
    const uint4 *pv = reinterpret_cast<const uint4 *>(zp + ((s * (k + 1) + r) * V) * E::kEsz);
    const uint4 *qv = reinterpret_cast<const uint4 *>(zq + ((s * k + (use_q ? r : 0)) * V) * E::kEsz);
    const int64_t nv = V / E::kVec;
    const int n_tiles = (int)((V + kTile - 1) / kTile);
    // ---- a2: tile sums of the residual mass, one warp per tile (coalesced)
    for (int pass = 0; pass < 2; ++pass) {
        for (int tile = warp; tile < n_tiles; tile += nwarps) {
            u128 acc = 0;
#pragma unroll
            for (int j = 0; j < kTileVecs; ++j) {
                const int64_t vi = (int64_t)tile * (32 * kTileVecs) + j * 32 + lane;
                if (vi < nv) {
                    const uint4 a = pv[vi];
                    const uint4 c = use_q ? qv[vi] : make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int e = 0; e < E::kVec; ++e)
                        acc += entry_mass<BF16>(E::get(a, e), E::get(c, e), mp, mq, Sp, Sq, use_q);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += shfl_xor_u128(acc, o);
            if (lane == 0) tile_sum[tile] = acc;
        }
        __syncthreads();
        // total; no residual mass while rejecting: the row p_r itself (AMB-20)
        __shared__ int s_again;
        if (threadIdx.x == 0) {
            u128 Z = 0;
            for (int t = 0; t < n_tiles; ++t) Z += tile_sum[t];
            s_again = (Z == 0 && use_q) ? 1 : 0;
        }
        __syncthreads();
        if (!s_again) break;
        use_q = false;
        __syncthreads();
    }
    if (warp != 0) return;
    // ---- warp 0: Z, t, the tile holding t, rescan it
    u128 Z = 0;
    for (int t0 = 0; t0 < n_tiles; t0 += 32) Z += t0 + lane < n_tiles ? tile_sum[t0 + lane] : (u128)0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Z += shfl_xor_u128(Z, o);
    int y = -1;
    if (Z == 0) {
        if (lane == 0 && err) atomicOr(err, E_NO_MASS);
        y = r < k ? dr[r] : 0;
    } else {
        const uint4 u = philox4x32_10(make_uint4(req, rnd, 1u << 8, trace), (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint64_t U = ((uint64_t)u.x << 32) | u.y;
        const uint64_t Zhi = (uint64_t)(Z >> 64), Zlo = (uint64_t)Z;
        u128 t = (u128)U * Zhi + (u128)__umul64hi(U, Zlo);
        int tile = -1;
        for (int t0 = 0; t0 < n_tiles && tile < 0; t0 += 32) {
            const u128 v = t0 + lane < n_tiles ? tile_sum[t0 + lane] : (u128)0;
            u128 incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u128 n = shfl_up_u128(incl, o);
                if (lane >= o) incl += n;
            }
            const u128 tot = shfl_u128(incl, 31);
            if (t < tot) {
                const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
                t -= shfl_u128(incl - v, src);
                tile = t0 + src;
            } else {
                t -= tot;
            }
        }
        // rescan the tile: vector j*32 + lane of the tile, in vocabulary order (j, lane, e)
        for (int j = 0; j < kTileVecs && y < 0; ++j) {
            const int64_t vi = (int64_t)tile * (32 * kTileVecs) + j * 32 + lane;
            u128 me[E::kVec];
            u128 msum = 0;
            if (vi < nv) {
                const uint4 a = pv[vi];
                const uint4 c = use_q ? qv[vi] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int e = 0; e < E::kVec; ++e) {
                    me[e] = entry_mass<BF16>(E::get(a, e), E::get(c, e), mp, mq, Sp, Sq, use_q);
                    msum += me[e];
                }
            } else {
#pragma unroll
                for (int e = 0; e < E::kVec; ++e) me[e] = 0;
            }
            u128 incl = msum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u128 n = shfl_up_u128(incl, o);
                if (lane >= o) incl += n;
            }
            const u128 tot = shfl_u128(incl, 31);
            if (t < tot) {
                const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
                int yy = -1;
                if (lane == src) {
                    u128 tt = t - (incl - msum);
                    int e = 0;
                    for (; e < E::kVec - 1; ++e) {
                        if (tt < me[e]) break;
                        tt -= me[e];
                    }
                    yy = (int)(vi * E::kVec + e);
                }
                y = __shfl_sync(0xFFFFFFFFu, yy, src);
            } else {
                t -= tot;
            }
        }
        if (y < 0) y = (int)V - 1;   // unreachable for t < Z
    }
    int32_t *tok = tokens + (int64_t)b * (k + 1);
    if (lane <= k) tok[lane] = lane < r ? dr[lane] : lane == r ? y : -1;
    if (lane == 0) {
        n_accept[b] = r;
        if (z_out) {
            z_out[2 * (int64_t)b] = (uint64_t)Z;
            z_out[2 * (int64_t)b + 1] = (uint64_t)(Z >> 64);
        }
    }
}

size_t logits_tile_smem(int64_t V, int32_t dtype) {
    const int tile = 32 * kTileVecs * (dtype == LAPSSD_BF16 ? 8 : 4);
    return (size_t)((V + tile - 1) / tile) * sizeof(u128);
}

cudaError_t launch_verify_logits(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                                 const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                                 const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                                 int32_t *tokens, int32_t *n_accept, uint64_t *z, float *m_ws, uint64_t *S_ws,
                                 cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    const unsigned rows = (unsigned)(2 * k + 1);
    const size_t smem = logits_tile_smem(V, dtype);
    if (dtype == LAPSSD_BF16) {
        logits_norm_kernel<true><<<(unsigned)B * rows, kNormThreads, 0, s>>>(
            (const char *)zp, (const char *)zq, slab, V, k, m_ws, S_ws);
        count_launch();
        logits_sample_kernel<true><<<(unsigned)B, kLogitThreads, smem, s>>>(
            (const char *)zp, (const char *)zq, draft, slab, req_id, round_idx, V, k, seed, trace, m_ws, S_ws, tokens,
            n_accept, z, nullptr);
    } else {
        logits_norm_kernel<false><<<(unsigned)B * rows, kNormThreads, 0, s>>>(
            (const char *)zp, (const char *)zq, slab, V, k, m_ws, S_ws);
        count_launch();
        logits_sample_kernel<false><<<(unsigned)B, kLogitThreads, smem, s>>>(
            (const char *)zp, (const char *)zq, draft, slab, req_id, round_idx, V, k, seed, trace, m_ws, S_ws, tokens,
            n_accept, z, nullptr);
    }
    count_launch();
    return cudaGetLastError();
}

void verify_logits_prepare() {
    cudaFuncSetAttribute(logits_sample_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(logits_sample_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
}

}  // namespace lapssd
