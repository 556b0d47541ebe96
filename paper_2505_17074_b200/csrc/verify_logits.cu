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
// logits_lazy_kernel (the default): one launch over a persistent grid that normalises only
//   the rows the acceptance tests consult (position j's pair only if x_0..x_{j-1} were
//   accepted), from a work queue (see "lazy form" below); the residual pass sums
//   Sq * sum_{P+} Ep - Sp * sum_{P+} Eq with two uint64 sums per lane (P+ decided by an
//   fp32 screen, the exact 128-bit comparison only where the screen cannot decide).
// norm_kernel + sample_kernel (LAPSSD_LOGITS_EAGER=1, the A/B form): one CTA per (slot,
//   row) of all 2k+1 rows (max, then the integer mass), then one CTA per slot for the k
//   acceptance tests and the residual row pair in 1,024-entry tiles.
#include "lapssd_internal.cuh"

#include <cuda_bf16.h>

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
// f40x2 returns P 2^(n+40) (exact in fp32, before the truncation); e40x2 truncates it.
__device__ __forceinline__ float2 f40x2(float za, float zb, float ma, float mb) {
    const float2 d0 = __fadd2_rn(make_float2(za, zb), make_float2(-ma, -mb));
#ifdef LAPSSD_E40_UPPER_CLAMP
    const float2 d = make_float2(fmaxf(fminf(d0.x, 0.0f), -28.5f), fmaxf(fminf(d0.y, 0.0f), -28.5f));
#else   // z <= m (m is the row max), so fl32(z - m) <= 0: only the lower clamp can act
    const float2 d = make_float2(fmaxf(d0.x, -28.5f), fmaxf(d0.y, -28.5f));
#endif
    // x = fl32(d log2e) as two SCALAR multiplies: ptxas contracts a packed mul.rn.f32x2
    // followed by add.rn.f32x2 into one FFMA2 (one rounding; even with --fmad=false), which
    // would round d log2e + 1.5 2^23 once and take rint of the exact product, not of x
#ifdef LAPSSD_E40_PACKED_MUL   // diagnostic build only: reproduces the contraction
    const float2 x = __fmul2_rn(d, make_float2(0x1.715476p+0f, 0x1.715476p+0f));
#else
    const float2 x = make_float2(__fmul_rn(d.x, 0x1.715476p+0f), __fmul_rn(d.y, 0x1.715476p+0f));
#endif
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
    return __fmul2_rn(p, sc);   // P 2^(n+40), exact
}

__device__ __forceinline__ void e40x2(float za, float zb, float ma, float mb, uint64_t &ea, uint64_t &eb) {
    const float2 f = f40x2(za, zb, ma, mb);
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

#ifndef LAPSSD_NORM_ILP
#define LAPSSD_NORM_ILP 4
#endif
constexpr int kNormIlp = LAPSSD_NORM_ILP;

// Max of the 8 / 4 logits of one vector: bf16 pairs by packed HMNMX2 on the raw words
// (max is exact in any format), fp32 by FMNMX.
template <bool BF16> struct VecMax;
template <> struct VecMax<true> {
    __nv_bfloat162 m = __nv_bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));   // -inf
    __device__ void add(const uint4 &v) {
        m = __hmax2(m, __hmax2(__hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&v.x),
                                       *reinterpret_cast<const __nv_bfloat162 *>(&v.y)),
                               __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&v.z),
                                       *reinterpret_cast<const __nv_bfloat162 *>(&v.w))));
    }
    __device__ float get() const { return fmaxf(__bfloat162float(m.x), __bfloat162float(m.y)); }
};
template <> struct VecMax<false> {
    float m = -INFINITY;
    __device__ void add(const uint4 &v) {
        m = fmaxf(m, fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)),
                           fmaxf(__uint_as_float(v.z), __uint_as_float(v.w))));
    }
    __device__ float get() const { return m; }
};

// Block-wide max of the logits in vectors [lo, hi) of a row (every thread gets it); U
// independent 16-byte loads in flight per thread.
template <bool BF16, int U>
__device__ __forceinline__ float range_max_u(const uint4 *v4, int64_t lo, int64_t hi) {
    __shared__ float s_m[32];
    const int64_t bd = blockDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    VecMax<BF16> acc;
    int64_t i = lo + threadIdx.x;
    for (; i + (U - 1) * bd < hi; i += U * bd) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = v4[i + u * bd];
#pragma unroll
        for (int u = 0; u < U; ++u) acc.add(v[u]);
    }
    for (; i < hi; i += bd) acc.add(v4[i]);
    float m = acc.get();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (lane == 0) s_m[warp] = m;
    __syncthreads();
    m = s_m[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s_m[w]);
    __syncthreads();   // s_m may be reused by the next call
    return m;
}
template <bool BF16>
__device__ __forceinline__ float range_max(const uint4 *v4, int64_t lo, int64_t hi) {
    return range_max_u<BF16, kNormIlp>(v4, lo, hi);
}

// Block-wide integer mass sum E[v] over vectors [lo, hi) for the row max m (thread 0
// gets the total).  U independent 16-byte loads in flight per thread.
template <bool BF16, int U>
__device__ __forceinline__ uint64_t range_sum_u(const uint4 *v4, int64_t lo, int64_t hi, float m) {
    using E = LElt<BF16>;
    __shared__ uint64_t s_S[32];
    const int64_t bd = blockDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t S = 0;
    int64_t i = lo + threadIdx.x;
    for (; i + (U - 1) * bd < hi; i += U * bd) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = v4[i + u * bd];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < E::kVec; e += 2) {
                uint64_t a, c;
                e40x2(E::get(v[u], e), E::get(v[u], e + 1), m, m, a, c);
                S += a + c;
            }
    }
    for (; i < hi; i += bd) {
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
    uint64_t t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_S[w];
    __syncthreads();
    return t;
}
template <bool BF16>
__device__ __forceinline__ uint64_t range_sum(const uint4 *v4, int64_t lo, int64_t hi, float m) {
    return range_sum_u<BF16, kNormIlp>(v4, lo, hi, m);
}

template <bool BF16>
__device__ __forceinline__ const uint4 *row_ptr(const char *zp, const char *zq, int64_t s, int64_t V, int32_t k,
                                                int ri) {
    using E = LElt<BF16>;
    return reinterpret_cast<const uint4 *>(ri <= k ? zp + ((s * (k + 1) + ri) * V) * E::kEsz
                                                   : zq + ((s * k + (ri - k - 1)) * V) * E::kEsz);
}

// Row ri of slot b (target row ri for ri <= k, else draft row ri - k - 1): the max, then
// the integer mass; thread 0 stores (m, S) to m_out[b*rows + ri], S_out[b*rows + ri].
template <bool BF16>
__device__ __forceinline__ void norm_row(const char *zp, const char *zq, const int32_t *slab, int64_t V, int32_t k,
                                         int b, int ri, float *m_out, uint64_t *S_out) {
    using E = LElt<BF16>;
    const int rows = 2 * k + 1;
    const int64_t s = slab ? slab[b] : b;
    const uint4 *v4 = row_ptr<BF16>(zp, zq, s, V, k, ri);
    const int64_t nv = V / E::kVec;
    const float m = range_max<BF16>(v4, 0, nv);
    const uint64_t S = range_sum<BF16>(v4, 0, nv, m);
    if (threadIdx.x == 0) {
        m_out[(int64_t)b * rows + ri] = m;
        S_out[(int64_t)b * rows + ri] = S;
    }
}

template <bool BF16>
__global__ void __launch_bounds__(kNormThreads) logits_norm_kernel(const char *zp, const char *zq,
                                                                   const int32_t *slab, int64_t V, int32_t k,
                                                                   float *m_out, uint64_t *S_out) {
    const int rows = 2 * k + 1;
    norm_row<BF16>(zp, zq, slab, V, k, blockIdx.x / rows, blockIdx.x % rows, m_out, S_out);
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

// a1 at position j: reject iff NOT u24_j * Eq_j(x_j) * Sp_j < 2^24 * Ep_j(x_j) * Sq_j.
template <bool BF16>
__device__ __forceinline__ bool rejects(const char *zp, const char *zq, const int32_t *dr, int64_t s, int j,
                                        uint32_t req, uint32_t rnd, int64_t V, int32_t k, uint64_t seed,
                                        uint32_t trace, const float *m, const uint64_t *S) {
    using E = LElt<BF16>;
    const int x = dr[j];
    const char *prow = zp + ((s * (k + 1) + j) * V) * E::kEsz;
    const char *qrow = zq + ((s * k + j) * V) * E::kEsz;
    const float zpx = BF16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(prow)[x] << 16)
                           : reinterpret_cast<const float *>(prow)[x];
    const float zqx = BF16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(qrow)[x] << 16)
                           : reinterpret_cast<const float *>(qrow)[x];
    const unsigned long long *Su = reinterpret_cast<const unsigned long long *>(S);
    const uint64_t Ep = e40(zpx, __ldcg(m + j)), Eq = e40(zqx, __ldcg(m + k + 1 + j));
    const uint4 u = philox4x32_10(make_uint4(req, rnd, (uint32_t)(j >> 2), trace), (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
    const uint32_t w = (j & 3) == 0 ? u.x : (j & 3) == 1 ? u.y : (j & 3) == 2 ? u.z : u.w;
    const uint32_t u24 = w >> 8;
    return !((u128)u24 * Eq * __ldcg(Su + j) < (((u128)Ep * __ldcg(Su + k + 1 + j)) << 24));
}

// a2 inputs for slot b with r known: the residual row pair (r < k) or the bonus row p_k.
struct Resid {
    const uint4 *pv, *qv;
    float mp, mq;
    uint64_t Sp, Sq;
    bool use_q;
    float invSp, invSq;       // the split-sum pass's float screen (tile_pass_split)
};

template <bool BF16>
__device__ __forceinline__ Resid resid_of(const char *zp, const char *zq, int64_t s, int r, int64_t V, int32_t k,
                                          const float *m, const uint64_t *S) {
    // (L2 reads: in the lazy kernel other CTAs wrote these rows' (m, S) during this launch)
    const unsigned long long *Su = reinterpret_cast<const unsigned long long *>(S);
    Resid q;
    q.use_q = r < k;
    q.mp = __ldcg(m + r);
    q.Sp = __ldcg(Su + r);
    q.mq = q.use_q ? __ldcg(m + k + 1 + r) : 0.0f;
    q.Sq = q.use_q ? __ldcg(Su + k + 1 + r) : 0;
    q.pv = row_ptr<BF16>(zp, zq, s, V, k, r);
    q.qv = row_ptr<BF16>(zp, zq, s, V, k, k + 1 + (q.use_q ? r : 0));
    // 1/S to within 2^-23 relative (two RN roundings)
    q.invSp = __frcp_rn(__ull2float_rn(q.Sp));
    q.invSq = q.use_q ? __frcp_rn(__ull2float_rn(q.Sq)) : 0.0f;
    return q;
}

// Residual mass of tiles [t_lo, t_hi) for r < k without a 128-bit product per entry:
// R_v > 0 iff Ep_v Sq > Eq_v Sp, and over the set P+ where it holds
//   sum R = Sq * sum_{P+} Ep - Sp * sum_{P+} Eq   (exact; both sums < 2^58),
// so each lane keeps two uint64 sums and the tile's 128-bit mass is formed once.
// Membership is screened in fp32: Ep = trunc(fp) is exact as a float (an integer below
// 2^41 with <= 24 significant bits), A = fl(Ep invSp) and B = fl(Eq invSq) are within
// 2^-23 relative of Ep/Sp and Eq/Sq (invS = 1/S to within 2^-23), so x = fl(A - B) is
// within (A+B) 2^-22 of Ep/Sp - Eq/Sq: x > m = (A+B) 2^-20 proves R_v > 0 and x < -m
// proves R_v = 0 (Ep = 0 gives R_v = 0, Eq = 0 < Ep gives R_v > 0).  The entries the
// screen cannot decide (|p^/q^ - 1| below ~2^-19, or exact ties) are decided afterwards by
// the exact 128-bit comparison, out of the unrolled loop.
template <bool BF16>
__device__ __forceinline__ int split_screen(float fp, float fq, const Resid &q) {   // 1 take, 0 skip, 2 exact
    const float tp = truncf(fp), tq = truncf(fq);
    const float2 ab = __fmul2_rn(make_float2(tp, tq), make_float2(q.invSp, q.invSq));
    const float x = __fsub_rn(ab.x, ab.y);
    const float m = __fmul_rn(__fadd_rn(ab.x, ab.y), 0x1p-20f);
    if (tp == 0.0f) return 0;
    if (tq == 0.0f || x > m) return 1;
    if (x < -m) return 0;
    return 2;
}

template <bool BF16>
__device__ __forceinline__ void tile_pass_split(const Resid &q, int64_t nv, int t_lo, int t_hi, u128 *out) {
    using E = LElt<BF16>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int tile = t_lo + warp; tile < t_hi; tile += nwarps) {
        uint64_t sP = 0, sQ = 0;
#pragma unroll
        for (int j = 0; j < kTileVecs; ++j) {
            const int64_t vi = (int64_t)tile * (32 * kTileVecs) + j * 32 + lane;
            if (vi < nv) {
                const uint4 a = q.pv[vi];
                const uint4 c = q.qv[vi];
                uint32_t unc = 0;
#pragma unroll
                for (int e = 0; e < E::kVec; ++e) {
                    const float2 f = f40x2(E::get(a, e), E::get(c, e), q.mp, q.mq);
                    const int d = split_screen<BF16>(f.x, f.y, q);
                    if (d == 1) {
                        sP += __float2ull_rz(f.x);
                        sQ += __float2ull_rz(f.y);
                    }
                    unc |= (uint32_t)(d >> 1) << e;
                }
                while (unc) {   // rare: the exact comparison
                    const int e = __ffs(unc) - 1;
                    unc &= unc - 1;
                    const float2 f = f40x2(E::get(a, e), E::get(c, e), q.mp, q.mq);
                    const uint64_t ep = __float2ull_rz(f.x), eq = __float2ull_rz(f.y);
                    if ((u128)ep * q.Sq > (u128)eq * q.Sp) {
                        sP += ep;
                        sQ += eq;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sP += __shfl_xor_sync(0xFFFFFFFFu, sP, o);
            sQ += __shfl_xor_sync(0xFFFFFFFFu, sQ, o);
        }
        if (lane == 0) out[tile] = (u128)sP * q.Sq - (u128)sQ * q.Sp;
    }
}

// R_v = Ep_r[v] (the bonus row, or AMB-20's fallback): two entries of p per exp call.
template <bool BF16>
__device__ __forceinline__ void tile_pass_p(const Resid &q, int64_t nv, int t_lo, int t_hi, u128 *out) {
    using E = LElt<BF16>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int tile = t_lo + warp; tile < t_hi; tile += nwarps) {
        uint64_t sP = 0;
#pragma unroll
        for (int j = 0; j < kTileVecs; ++j) {
            const int64_t vi = (int64_t)tile * (32 * kTileVecs) + j * 32 + lane;
            if (vi < nv) {
                const uint4 a = q.pv[vi];
#pragma unroll
                for (int e = 0; e < E::kVec; e += 2) {
                    uint64_t x, y;
                    e40x2(E::get(a, e), E::get(a, e + 1), q.mp, q.mp, x, y);
                    sP += x + y;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sP += __shfl_xor_sync(0xFFFFFFFFu, sP, o);
        if (lane == 0) out[tile] = (u128)sP;
    }
}

template <bool BF16>
__device__ __forceinline__ void tile_pass_fast(const Resid &q, int64_t nv, int t_lo, int t_hi, u128 *out) {
    if (q.use_q) tile_pass_split<BF16>(q, nv, t_lo, t_hi, out);
    else tile_pass_p<BF16>(q, nv, t_lo, t_hi, out);
}

// Z = sum of the tile sums; with no residual mass while rejecting, the row p_r itself
// (AMB-20): the tiles are recomputed with use_q = false.  Block-wide; returns use_q.
template <bool BF16>
__device__ __forceinline__ void amb20_fallback(Resid &q, int64_t nv, int n_tiles, u128 *tile_sum) {
    __shared__ int s_again;
    if (threadIdx.x == 0) {
        u128 Z = 0;
        for (int t = 0; t < n_tiles; ++t) Z += tile_sum[t];
        s_again = (Z == 0 && q.use_q) ? 1 : 0;
    }
    __syncthreads();
    if (s_again) {
        q.use_q = false;
        tile_pass_p<BF16>(q, nv, 0, n_tiles, tile_sum);
    }
    __syncthreads();
}

// Warp 0: Z, t = floor(U Z / 2^64), the tile holding t (prefix over tile_sum in shared
// memory), a rescan of that tile in vocabulary order, then the outputs of slot b.
template <bool BF16>
__device__ __forceinline__ void draw_token(const Resid &q, int64_t nv, int n_tiles, const u128 *tile_sum,
                                           const int32_t *dr, int b, int r, uint32_t req, uint32_t rnd, int32_t k,
                                           int64_t V, uint64_t seed, uint32_t trace, int32_t *tokens,
                                           int32_t *n_accept, uint64_t *z_out, uint32_t *err) {
    using E = LElt<BF16>;
    const int lane = threadIdx.x & 31;
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
                const uint4 a = q.pv[vi];
                const uint4 c = q.use_q ? q.qv[vi] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int e = 0; e < E::kVec; ++e) {
                    me[e] = entry_mass<BF16>(E::get(a, e), E::get(c, e), q.mp, q.mq, q.Sp, q.Sq, q.use_q);
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
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *m = m_in + (int64_t)b * rows;
    const uint64_t *S = S_in + (int64_t)b * rows;
    const int32_t *dr = draft + s * k;
    // ---- a1: position j on lane j of warp 0 (k <= 16), first rejection by ballot
    if (warp == 0) {
        const bool reject = lane < k && rejects<BF16>(zp, zq, dr, s, lane, req, rnd, V, k, seed, trace, m, S);
        const unsigned msk = __ballot_sync(0xFFFFFFFFu, reject);
        if (lane == 0) s_r = msk ? __ffs(msk) - 1 : k;
    }
    __syncthreads();
    const int r = s_r;
    Resid q = resid_of<BF16>(zp, zq, s, r, V, k, m, S);
    const int64_t nv = V / E::kVec;
    const int n_tiles = (int)((V + kTile - 1) / kTile);
    tile_pass_fast<BF16>(q, nv, 0, n_tiles, tile_sum);
    __syncthreads();
    amb20_fallback<BF16>(q, nv, n_tiles, tile_sum);
    if (warp == 0)
        draw_token<BF16>(q, nv, n_tiles, tile_sum, dr, b, r, req, rnd, k, V, seed, trace, tokens, n_accept, z_out,
                         err);
}

// ---------------------------------------------------------------- lazy form (one launch)
// Only the rows the method consults are normalised: position j's pair (p_j, q_j) is needed
// only if x_0..x_{j-1} were all accepted, and p_k only if all k were (the
// acceptance tests run in order and stop at the first rejection).  A persistent grid
// claims units, in this order:
//  1. filler: the 2B rows of position 0 (claimed one unit AHEAD, so the claim's latency
//     hides under the current unit);
//  2. published units, FIFO: the pair j+1 (or p_k) published when test j accepts, and the
//     residual parts published when a test rejects (or p_k completes): np parts of tp
//     tiles, each writing its tiles' masses, the last to finish draws the token;
//     speculatively, while CTAs wait for work, test j's acceptance also publishes the
//     pair j+2: a slot's chain of tests is a latency chain (one row pass per position),
//     idle CTAs run it a position ahead, and if test j+1 accepts, test j+2 runs at once.
// A row unit is one whole row, its two passes (max, then mass) back to back on one CTA so
// the second pass hits L2.  Each row is claimed once (a per-row flag); test j runs when
// both rows of position j are done and test j-1 accepted (a per-position counter; the
// party that completes it runs the test, cascading while the next rows are done).
struct LazyArgs {
    const char *zp, *zq;
    const int32_t *draft, *slab;
    const uint32_t *req_id, *round_idx;
    int64_t V;
    int32_t k, B;
    uint64_t seed;
    uint32_t trace;
    float *m;                 // [B rows]
    uint64_t *S;              // [B rows]
    uint32_t *units;          // [ucap] published unit code + 1 (0 = not yet)
    uint32_t *cnt;            // [B (k+1)] position j: rows done + test j-1 accepted
    uint32_t *rowflag;        // [B rows] row claimed
    uint32_t *rpart;          // [B]: residual parts finished
    int32_t *rpos;            // [B]: r + 1 of the slot, 0 while unknown (written before its parts are published)
    uint32_t *ctr;            // [0] filler claims, [1] units published, [2] slots done, [3] tickets
    u128 *tsum;               // [B n_tiles] residual tile masses
    uint32_t ucap;
    int32_t np, tp;           // residual parts per slot, tiles per part
    int32_t *tokens, *n_accept;
    uint64_t *z_out;
    uint32_t *err;
};

#ifndef LAPSSD_LAZY_THREADS
#define LAPSSD_LAZY_THREADS 512
#endif
#ifndef LAPSSD_LAZY_MINB
#define LAPSSD_LAZY_MINB 2
#endif
#ifndef LAPSSD_LAZY_PF      // bytes per L2 bulk prefetch of a row unit's row (0: none)
#define LAPSSD_LAZY_PF 32768
#endif
#ifndef LAPSSD_LAZY_TILES_PER_PART
#define LAPSSD_LAZY_TILES_PER_PART 64
#endif
#ifndef LAPSSD_LAZY_SPEC_IDLE   // speculation d positions ahead only with > (d-1) x this many CTAs waiting
#define LAPSSD_LAZY_SPEC_IDLE 16
#endif
#ifndef LAPSSD_LAZY_SPEC    // speculative rows while CTAs wait: up to this many positions ahead (0: off)
#define LAPSSD_LAZY_SPEC 2
#endif
#ifndef LAPSSD_LAZY_ILP     // loads in flight per thread in the lazy kernel's row passes
#define LAPSSD_LAZY_ILP 2      // (measured: 1 / 2 / 3 / 4 / 6 / 8 -> 0.477 / 0.461 / 0.465 / 0.469 / 0.463 / 0.467 ms)
#endif
constexpr int kLazyThreads = LAPSSD_LAZY_THREADS;
constexpr int kLazyIlp = LAPSSD_LAZY_ILP;

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr uint32_t kExit = 0xFFFFFFFFu;

// Thread 0: the next unit code (row units < B rows, residual parts above), or kExit.  After
// the filler, one ticket per claim (an atomicAdd, no CAS retries: contended CAS claims
// serialised to ~1 per us), then a wait for that entry; a row taken already (claimed
// speculatively) or of a slot already resolved is skipped.
__device__ __forceinline__ uint32_t lazy_claim(const LazyArgs &a, uint32_t first, uint32_t rows) {
    const uint32_t k = (uint32_t)a.k, row_units = (uint32_t)a.B * rows;
    if (ld_acquire_u32(a.ctr) < first) {   // the position-0 filler
        const uint32_t f = atomicAdd(a.ctr, 1u);
        if (f < first) return (f >> 1) * rows + ((f & 1) ? k + 1 : 0);
    }
    for (;;) {
        const uint32_t idx = atomicAdd(a.ctr + 3, 1u);
        uint32_t c = kExit;
        for (;;) {
            if (idx < a.ucap) {
                const uint32_t u = ld_acquire_u32(a.units + idx);
                if (u) { c = u - 1; break; }
            }
            if (ld_acquire_u32(a.ctr + 2) >= (uint32_t)a.B) return kExit;
            __nanosleep(128);
        }
        if (c >= row_units) return c;
        if (__ldcg(a.rpos + c / rows) == 0 && atomicCAS(a.rowflag + c, 0u, 1u) == 0u) return c;
    }
}

// Thread 0: publish n unit codes c0, c0 + step, ...
__device__ __forceinline__ void lazy_publish(const LazyArgs &a, uint32_t c0, uint32_t step, uint32_t n) {
    const uint32_t at = atomicAdd(a.ctr + 1, n);
    for (uint32_t i = 0; i < n; ++i) st_release_u32(a.units + at + i, c0 + i * step + 1);
}

#ifdef LAPSSD_LAZY_TRACE   // diagnostic build only: per-unit (code, smid, claim, start, end)
__device__ unsigned long long g_lazy_tr[16384][4];
__device__ unsigned int g_lazy_n;
extern "C" int lapssd_lazy_trace_read(unsigned long long *out, unsigned *n) {
    cudaMemcpyFromSymbol(n, g_lazy_n, sizeof(unsigned));
    cudaMemcpyFromSymbol(out, g_lazy_tr, sizeof g_lazy_tr);
    unsigned z = 0;
    cudaMemcpyToSymbol(g_lazy_n, &z, sizeof z);
    return 0;
}
#endif

// Thread 0: the rows of position j (the pair, or p_k for j = k) not claimed yet.
__device__ __forceinline__ void publish_position(const LazyArgs &a, int b, int j) {
    const int k = a.k, rows = 2 * k + 1;
    const uint32_t c0 = (uint32_t)(b * rows + j);
    if (__ldcg(a.rowflag + c0) == 0u) lazy_publish(a, c0, 0, 1);
    if (j < k && __ldcg(a.rowflag + c0 + k + 1) == 0u) lazy_publish(a, c0 + k + 1, 0, 1);
}

// Thread 0: test j of slot b is due (rows of position j done, test j-1 accepted).  Runs the
// chain of tests while the next position's rows are already done: acceptance makes
// position j+1 needed and j+2 speculative, rejection at j (or reaching p_k) publishes the
// slot's residual parts.
template <bool BF16>
__device__ __forceinline__ void run_tests(const LazyArgs &a, int b, int j, int64_t s) {
    const int k = a.k, rows = 2 * k + 1;
    for (;;) {
        __threadfence();
        int rr = -1;
        if (j == k) {
            rr = k;   // p_k: every draft accepted
        } else if (rejects<BF16>(a.zp, a.zq, a.draft + s * k, s, j, a.req_id[b], a.round_idx[b], a.V, k, a.seed,
                                 a.trace, a.m + (int64_t)b * rows, a.S + (int64_t)b * rows)) {
            rr = j;
        }
        if (rr >= 0) {
            a.rpos[b] = rr + 1;
            lazy_publish(a, (uint32_t)a.B * rows + (uint32_t)b * a.np, 1, (uint32_t)a.np);
            return;
        }
        publish_position(a, b, j + 1);
#if LAPSSD_LAZY_SPEC
        // a position ahead as well, but only while CTAs wait for work (tickets ahead of
        // the published entries): idle SMs shorten the chain, busy ones are not diverted
        if (j + 2 <= k) {   // position j+1+d while more than (d-1) LAPSSD_LAZY_SPEC_IDLE CTAs wait
            const int32_t waiting = (int32_t)(ld_acquire_u32(a.ctr + 3) - ld_acquire_u32(a.ctr + 1));
            for (int d = 1; d <= LAPSSD_LAZY_SPEC && j + 1 + d <= k; ++d)
                if (waiting > (d - 1) * LAPSSD_LAZY_SPEC_IDLE) publish_position(a, b, j + 1 + d);
        }
#endif
        __threadfence();
        const uint32_t c = atomicAdd(a.cnt + (int64_t)b * (k + 1) + j + 1, 1u) + 1;
        if (c != (j + 1 == k ? 2u : 3u)) return;   // the rows of j+1 are not all done yet
        ++j;
    }
}

// Thread 0 of a CTA that completed row ri of slot b: store (m, S), count the row at its
// position, and run the test if it is due.
template <bool BF16>
__device__ __forceinline__ void row_done(const LazyArgs &a, int b, int ri, int64_t s, float m, uint64_t S) {
    const int k = a.k, rows = 2 * k + 1;
    const int64_t rowi = (int64_t)b * rows + ri;
    a.m[rowi] = m;
    a.S[rowi] = S;
    const int j = ri <= k ? ri : ri - k - 1;
    __threadfence();
    const uint32_t c = atomicAdd(a.cnt + (int64_t)b * (k + 1) + j, 1u) + 1;
    if (c == (j == 0 || j == k ? 2u : 3u)) run_tests<BF16>(a, b, j, s);
}

// The CTA loop.  The next position-0 filler unit is claimed AHEAD (thread 0's atomic is in
// flight while the unit streams), so after a row unit the other threads start the next
// unit at once while thread 0 finishes the pair logic; only once the filler is exhausted
// does a CTA claim (and wait) at the end of a unit.
template <bool BF16>
__global__ void __launch_bounds__(kLazyThreads, LAPSSD_LAZY_MINB) logits_lazy_kernel(const LazyArgs a) {
    using E = LElt<BF16>;
    constexpr int kTile = 32 * kTileVecs * E::kVec;
    extern __shared__ __align__(16) uint8_t s_raw[];
    u128 *tile_sum = reinterpret_cast<u128 *>(s_raw);
    __shared__ uint32_t s_code, s_next;
    __shared__ int s_last;
    const int k = a.k, rows = 2 * k + 1;
    const int64_t nv = a.V / E::kVec;
    const int n_tiles = (int)((a.V + kTile - 1) / kTile);
    const uint32_t row_units = (uint32_t)a.B * rows, first = 2u * (uint32_t)a.B;
    constexpr uint32_t kNone = 0xFFFFFFFEu;
    bool filler_left = true;   // thread 0's view
#ifdef LAPSSD_LAZY_TRACE
    unsigned long long tr_claim = 0, tr_got = 0;
    if (threadIdx.x == 0) tr_claim = gtimer();
#endif
    if (threadIdx.x == 0) s_code = lazy_claim(a, first, (uint32_t)rows);
    __syncthreads();
    uint32_t code = s_code;
    for (;;) {
        if (code == kExit) return;
#ifdef LAPSSD_LAZY_TRACE
        const uint32_t cur = code;
        if (threadIdx.x == 0) tr_got = gtimer();
#endif
        uint32_t nf = first;   // thread 0: the filler unit claimed ahead (first = none)
        if (threadIdx.x == 0 && filler_left) nf = atomicAdd(a.ctr, 1u);
        int r = -1;
        if (code < row_units) {   // ---- a row unit
            const int b = (int)(code / rows), ri = (int)(code % rows);
            const int64_t s = a.slab ? a.slab[b] : b;
            const uint4 *v4 = row_ptr<BF16>(a.zp, a.zq, s, a.V, k, ri);
#if LAPSSD_LAZY_PF > 0   // the whole row requested into L2 up front (the max pass then reads L2)
            if ((threadIdx.x >> 5) == (int)(blockDim.x >> 5) - 1) {
                const int64_t bytes = a.V * E::kEsz;
                for (int64_t o = (int64_t)(threadIdx.x & 31) * LAPSSD_LAZY_PF; o < bytes; o += 32 * LAPSSD_LAZY_PF) {
                    const uint32_t n = (uint32_t)(bytes - o < LAPSSD_LAZY_PF ? bytes - o : LAPSSD_LAZY_PF);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char *)v4 + o), "r"(n)
                                 : "memory");
                }
            }
#endif
            const float m = range_max_u<BF16, kLazyIlp>(v4, 0, nv);
            const uint64_t S = range_sum_u<BF16, kLazyIlp>(v4, 0, nv, m);
            if (threadIdx.x == 0) {
                filler_left = nf < first;
                s_next = filler_left ? (nf >> 1) * rows + ((nf & 1) ? k + 1 : 0) : kNone;
            }
            __syncthreads();
            const uint32_t next = s_next;
            if (threadIdx.x == 0) row_done<BF16>(a, b, ri, s, m, S);
            if (next != kNone) {
                code = next;
#ifdef LAPSSD_LAZY_TRACE
                goto trace;
#endif
                continue;
            }
        } else {                  // ---- a residual part
            const uint32_t pc = code - row_units;
            const int b = (int)(pc / a.np), part = (int)(pc % a.np);
            r = __ldcg(a.rpos + b) - 1;
            const int64_t s = a.slab ? a.slab[b] : b;
            const float *mb = a.m + (int64_t)b * rows;
            const uint64_t *Sb = a.S + (int64_t)b * rows;
            Resid q = resid_of<BF16>(a.zp, a.zq, s, r, a.V, k, mb, Sb);
            u128 *ts = a.tsum + (int64_t)b * n_tiles;
            const int t_lo = part * a.tp, t_hi = min(n_tiles, t_lo + a.tp);
            tile_pass_fast<BF16>(q, nv, t_lo, t_hi, ts);
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const bool last = atomicAdd(a.rpart + b, 1u) == (uint32_t)a.np - 1;
                if (last) __threadfence();
                s_last = last;
                filler_left = nf < first;
                s_next = filler_left ? (nf >> 1) * rows + ((nf & 1) ? k + 1 : 0) : kNone;
            }
            __syncthreads();
            if (s_last) {   // every part is in: Z, the draw, the outputs of slot b
                for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
                    const unsigned long long *w = reinterpret_cast<const unsigned long long *>(ts + t);
                    tile_sum[t] = ((u128)__ldcg(w + 1) << 64) | __ldcg(w);
                }
                __syncthreads();
                amb20_fallback<BF16>(q, nv, n_tiles, tile_sum);
                if (threadIdx.x < 32)
                    draw_token<BF16>(q, nv, n_tiles, tile_sum, a.draft + s * k, b, r, a.req_id[b], a.round_idx[b],
                                     k, a.V, a.seed, a.trace, a.tokens, a.n_accept, a.z_out, a.err);
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.ctr + 2) : "memory");
                }
            }
            const uint32_t next = s_next;
            if (next != kNone) {
                __syncthreads();   // s_next / s_last are rewritten by the next unit
                code = next;
#ifdef LAPSSD_LAZY_TRACE
                goto trace;
#endif
                continue;
            }
        }
        // no filler left: claim (and wait for) a published unit
        if (threadIdx.x == 0) s_code = lazy_claim(a, first, (uint32_t)rows);
        __syncthreads();
        code = s_code;
#ifdef LAPSSD_LAZY_TRACE
    trace:
        if (threadIdx.x == 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            const unsigned i = atomicAdd(&g_lazy_n, 1u);
            if (i < 16384) {
                g_lazy_tr[i][0] = ((unsigned long long)smid << 32) | (cur & 0x7FFFFFFFu) | ((unsigned long long)(r >= 0) << 31);
                g_lazy_tr[i][1] = tr_claim;
                g_lazy_tr[i][2] = tr_got;
                g_lazy_tr[i][3] = gtimer();
            }
            tr_claim = gtimer();
        }
#endif
    }
}

size_t logits_tile_smem(int64_t V, int32_t dtype) {
    const int tile = 32 * kTileVecs * (dtype == LAPSSD_BF16 ? 8 : 4);
    return (size_t)((V + tile - 1) / tile) * sizeof(u128);
}

static int lazy_parts(int64_t V, int32_t dtype, int *tp) {
    const int n_tiles = (int)(logits_tile_smem(V, dtype) / sizeof(u128));
    *tp = LAPSSD_LAZY_TILES_PER_PART;
    return (n_tiles + *tp - 1) / *tp;
}

static size_t lazy_words(int32_t B, int32_t k, int np) {
    // position p is published by test p-1 (needed) and at most by tests p-2 .. p-1-SPEC
    // (ahead), so a row is published at most 1 + LAPSSD_LAZY_SPEC times
    const size_t rows = 2 * (size_t)k + 1, ucap = (size_t)B * ((1 + LAPSSD_LAZY_SPEC) * rows + np) + 4096;
    return ucap + (size_t)B * ((k + 1) + rows + 2) + 8;
}

// Workspace of the lazy form after (m, S): the queue and counters (zeroed per call), then
// the residual tile masses.
size_t logits_lazy_bytes(int32_t B, int32_t k, int64_t V, int32_t dtype) {
    int tp;
    const int np = lazy_parts(V, dtype, &tp);
    return 512 + lazy_words(B, k, np) * sizeof(uint32_t) + (size_t)B * logits_tile_smem(V, dtype);
}

template <bool BF16>
static cudaError_t launch_lazy(const void *zp, const void *zq, int64_t V, int32_t k, const int32_t *draft,
                               const int32_t *slab, const uint32_t *req_id, const uint32_t *round_idx, int32_t B,
                               uint64_t seed, uint32_t trace, int32_t *tokens, int32_t *n_accept, uint64_t *z,
                               float *m_ws, uint64_t *S_ws, char *lazy_ws, size_t smem, cudaStream_t s) {
    static int grid_per_sm = -1, sms = 0;
    static size_t grid_smem = 0;
    if (grid_per_sm < 0 || grid_smem != smem) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&grid_per_sm, logits_lazy_kernel<BF16>, kLazyThreads, smem);
        grid_smem = smem;
        if (grid_per_sm < 1) grid_per_sm = 1;
    }
    const int rows = 2 * k + 1;
    LazyArgs a{};
    a.zp = (const char *)zp; a.zq = (const char *)zq;
    a.draft = draft; a.slab = slab; a.req_id = req_id; a.round_idx = round_idx;
    a.V = V; a.k = k; a.B = B; a.seed = seed; a.trace = trace;
    a.m = m_ws; a.S = S_ws;
    a.np = lazy_parts(V, BF16 ? LAPSSD_BF16 : LAPSSD_F32, &a.tp);
    uint32_t *q = (uint32_t *)(((size_t)lazy_ws + 255) & ~(size_t)255);
    const size_t words = lazy_words(B, k, a.np);
    a.ucap = (uint32_t)((size_t)B * ((1 + LAPSSD_LAZY_SPEC) * rows + a.np) + 4096);
    a.units = q;
    a.cnt = q + a.ucap;
    a.rowflag = a.cnt + (size_t)B * (k + 1);
    a.rpart = a.rowflag + (size_t)B * rows;
    a.rpos = (int32_t *)(a.rpart + B);
    a.ctr = (uint32_t *)(a.rpos + B);
    a.tsum = (u128 *)(((size_t)(q + words) + 255) & ~(size_t)255);
    a.tokens = tokens; a.n_accept = n_accept; a.z_out = z; a.err = nullptr;
    cudaError_t ce = cudaMemsetAsync(q, 0, words * sizeof(uint32_t), s);
    if (ce != cudaSuccess) return ce;
    const int64_t want = (int64_t)B * rows;
    const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)grid_per_sm * sms);
    logits_lazy_kernel<BF16><<<grid, kLazyThreads, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_verify_logits(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                                 const int32_t *draft, const int32_t *slab, const uint32_t *req_id,
                                 const uint32_t *round_idx, int32_t B, uint64_t seed, uint32_t trace,
                                 int32_t *tokens, int32_t *n_accept, uint64_t *z, float *m_ws, uint64_t *S_ws,
                                 char *lazy_ws, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    const unsigned rows = (unsigned)(2 * k + 1);
    const size_t smem = logits_tile_smem(V, dtype);
    const bool eager = getenv("LAPSSD_LOGITS_EAGER") != nullptr;   // A/B: every row, two launches
    if (!eager) {
        return dtype == LAPSSD_BF16
                   ? launch_lazy<true>(zp, zq, V, k, draft, slab, req_id, round_idx, B, seed, trace, tokens, n_accept,
                                       z, m_ws, S_ws, lazy_ws, smem, s)
                   : launch_lazy<false>(zp, zq, V, k, draft, slab, req_id, round_idx, B, seed, trace, tokens, n_accept,
                                        z, m_ws, S_ws, lazy_ws, smem, s);
    }
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

// ---------------------------------------------------------------- laps_step_logits
// The Philox counters and slabs of the handle's batch, on the device: slot b verifies
// request i = sel[b] at its current round (req = global id i * world + rank, as laps_step),
// with the round's slab from the slab table (or slab b: the batch layout).  Empty slots
// (sel < 0) verify slab 0 as a dummy and are masked afterwards.
__global__ void logits_slots_kernel(const int32_t *sel, const int32_t *rounds, const int32_t *slab_tab, int32_t R,
                                    int32_t world, int32_t rank, int32_t B, uint32_t *req, uint32_t *rnd,
                                    int32_t *slab) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int32_t i = sel[b];
    if (i < 0) {
        req[b] = 0; rnd[b] = 0; slab[b] = 0;
        return;
    }
    const int32_t t = rounds[i];
    req[b] = (uint32_t)(i * world + rank);
    rnd[b] = (uint32_t)t;
    slab[b] = slab_tab ? slab_tab[(int64_t)i * R + slab_round_index(t, R)] : b;
}

__global__ void logits_mask_kernel(const int32_t *sel, int32_t k, int32_t B, int32_t *tokens, int32_t *n_accept) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || sel[b] >= 0) return;
    n_accept[b] = -1;
    for (int j = 0; j <= k; ++j) tokens[(int64_t)b * (k + 1) + j] = -1;
}

cudaError_t launch_logits_slots(const int32_t *sel, const int32_t *rounds, const int32_t *slab_tab, int32_t R,
                                int32_t world, int32_t rank, int32_t B, uint32_t *req, uint32_t *rnd, int32_t *slab,
                                cudaStream_t s) {
    logits_slots_kernel<<<(B + 255) / 256, 256, 0, s>>>(sel, rounds, slab_tab, R, world, rank, B, req, rnd, slab);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_logits_mask(const int32_t *sel, int32_t k, int32_t B, int32_t *tokens, int32_t *n_accept,
                               cudaStream_t s) {
    logits_mask_kernel<<<(B + 255) / 256, 256, 0, s>>>(sel, k, B, tokens, n_accept);
    count_launch();
    return cudaGetLastError();
}

void verify_logits_prepare() {
    cudaFuncSetAttribute(logits_sample_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(logits_sample_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(logits_lazy_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(logits_lazy_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
}

}  // namespace lapssd
