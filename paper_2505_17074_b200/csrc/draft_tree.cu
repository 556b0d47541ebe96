// draft_tree.cu -- SURVEY 8(f) f4 on sm_100a: the steps on either side of verification.
//
// spec_draft_sample ("the draft model autoregressively generates the subsequent L
//   tokens"; DESIGN.md AMB-34): one token per stored row by the exact integer inverse
//   CDF -- R_v = floor(q[v] 2^60), Z = sum R (exact uint64), U a 64-bit Philox uniform
//   (counter word (2 << 16) | pos), t = floor(U Z / 2^64), x = min{v : sum_{w<=v} R_w > t}.
// spec_verify_tree (SpecInfer's multi-step speculative sampling, cited at P:322; each
//   step the rule of P:59-64; AMB-35): per request a token tree; at a node the children
//   are tested in index order, the first with the linear verification's exact rule, the
//   later ones against the residual of the normalised D_i, D_{i+1} = floor(max(0, D_i 2^60 -
//   Z_i floor(q 2^60)) / 2^b(Z_i)) (exact 128-bit integers; b = bit length), by an exact
//   128-bit comparison; the first accepted child is emitted and
//   its subtree continues; if all are rejected the token comes from the last residual, at
//   a leaf the bonus token from p.  A chain is exactly spec_verify.
//
// Both are streaming row passes: one CTA per row (draft) or per tree (verify), 16 warps,
// each warp reducing 1,024-entry segments (16-byte loads, no L1 allocation) to one uint64
// in shared memory; the total is exact and order-independent; the draw finds the segment
// holding t by a warp scan and rescans that one segment.
#include "lapssd_internal.cuh"

namespace lapssd {
namespace {

typedef unsigned __int128 u128;

constexpr int kRowThreads = 512;        // draft sampling: one row per CTA, 4 CTAs per SM
#ifndef LAPSSD_TREE_THREADS
#define LAPSSD_TREE_THREADS 512
#endif
constexpr int kTreeThreads = LAPSSD_TREE_THREADS;   // tree verification: one CTA per SM
#ifndef LAPSSD_TREES_PER_CTA
#define LAPSSD_TREES_PER_CTA 1
#endif
constexpr int kTreesPerCta = LAPSSD_TREES_PER_CTA;  // trees per CTA (measured: 2 / 4 / 8 per CTA slower: 0.44 / 0.52 / 1.0 ms)
constexpr int kTreeMax = 64;            // nodes per tree

__device__ __forceinline__ uint4 ld_nc(const void *ptr) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr));
    return r;
}

// floor(max(0, fl32(p - q)) 2^60): fp32 RN difference, exact power-of-two scale, truncating
// conversion (cvt.rzi clamps negatives and NaN to 0).
__device__ __forceinline__ uint64_t mass460(float p, float q) {
    return __float2ull_rz(__fmul_rn(__fsub_rn(p, q), 0x1p60f));
}

template <bool BF16> struct RowElt;
template <> struct RowElt<true> {
    static constexpr int kVec = 8, kEsz = 2;
    __device__ static float get(const uint4 &v, int e) {
        const uint32_t w = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
        return __uint_as_float((e & 1) ? (w & 0xFFFF0000u) : (w << 16));
    }
};
template <> struct RowElt<false> {
    static constexpr int kVec = 4, kEsz = 4;
    __device__ static float get(const uint4 &v, int e) {
        return __uint_as_float(e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w);
    }
};

__device__ __forceinline__ uint64_t wsum(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ uint64_t wscan(uint64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Stage mass of one entry (AMB-35): D_1 = mass460(p, q); D_{s+1} = floor(max(0, D_s 2^60 -
// Z_s floor(q 2^60)) / 2^b(Z_s)).  stage 0: the row p alone (bonus / fallback / draft).
struct StageMass {
    int stage;
    const uint64_t *Zs;      // shared: Z_1..Z_{stage-1}
    const int *zb;           // shared: their bit lengths
    __device__ __forceinline__ uint64_t operator()(float p, float q) const {
        if (stage == 0) return mass460(p, 0.0f);
        uint64_t D = mass460(p, q);
        if (stage == 1) return D;
        const uint64_t Q = mass460(q, 0.0f);
        for (int s = 1; s < stage; ++s) {
            const u128 a = (u128)D << 60, b = (u128)Zs[s] * Q;
            D = a > b ? (uint64_t)((a - b) >> zb[s]) : 0;
        }
        return D;
    }
};

// The same stage mass with the stage a compile-time constant S (1..4) and Z_s / b(Z_s) in
// registers: the chain unrolls without branches or shared-memory loads per entry.
template <int S>
struct StageMassT {
    uint64_t z[S];
    int zb[S];
    __device__ __forceinline__ StageMassT(const uint64_t *Zs, const int *b) {
#pragma unroll
        for (int s = 1; s < S; ++s) { z[s] = Zs[s]; zb[s] = b[s]; }
    }
    __device__ __forceinline__ uint64_t operator()(float p, float q) const {
        uint64_t D = mass460(p, q);
        if (S == 1) return D;
        const uint64_t Q = mass460(q, 0.0f);
#pragma unroll
        for (int s = 1; s < S; ++s) {
            const u128 a = (u128)D << 60, b = (u128)z[s] * Q;
            D = a > b ? (uint64_t)((a - b) >> zb[s]) : 0;
        }
        return D;
    }
};

// The threads that work on one row: the whole CTA (draft sampling) or one group of warps
// of it (tree verification runs several trees per CTA); sync() is a named barrier.
struct Grp {
    int tid, nt, bar;
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory");
    }
};

// One pass over a row pair: seg[s] = the masses of segment s, returns Z (group-wide).
template <bool BF16, class MassF>
__device__ uint64_t row_pass(const char *prow, const char *qrow, int64_t V, const MassF &mass, uint64_t *seg,
                             uint64_t *s_tot, const Grp &gr) {
    using E = RowElt<BF16>;
    constexpr int J = kSegElems / E::kVec / 32;   // vectors per lane per segment
    const int lane = gr.tid & 31, warp = gr.tid >> 5;
    const int nseg = (int)((V + kSegElems - 1) / kSegElems);
    uint64_t mine = 0;
    const int nwarps = gr.nt >> 5;
    for (int s = warp; s < nseg; s += nwarps) {
        const int64_t base = (int64_t)s * kSegElems;
        uint4 pv[J], qv[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t e = base + (int64_t)(j * 32 + lane) * E::kVec;
            const bool in = e < V;
            pv[j] = in ? ld_nc(prow + e * E::kEsz) : make_uint4(0, 0, 0, 0);
            qv[j] = (in && qrow) ? ld_nc(qrow + e * E::kEsz) : make_uint4(0, 0, 0, 0);
        }
        uint64_t m = 0;
#pragma unroll
        for (int j = 0; j < J; ++j)
#pragma unroll
            for (int e = 0; e < E::kVec; ++e) m += mass(E::get(pv[j], e), E::get(qv[j], e));
        m = wsum(m);
        if (lane == 0) seg[s] = m;
        mine += m;
    }
    if (gr.tid == 0) *s_tot = 0;
    gr.sync();
    if (lane == 0 && mine) atomicAdd((unsigned long long *)s_tot, (unsigned long long)mine);
    gr.sync();
    const uint64_t Z = *s_tot;
    gr.sync();
    return Z;
}

// row_pass / row_search for a runtime stage: compile-time chains for stages 0..4.
template <bool BF16>
__device__ uint64_t stage_pass(const char *prow, const char *qrow, int64_t V, int stage, const uint64_t *Zs,
                               const int *zb, uint64_t *seg, uint64_t *s_tot, const Grp &gr);
template <bool BF16>
__device__ int stage_search(const char *prow, const char *qrow, int64_t V, int stage, const uint64_t *Zs,
                            const int *zb, const uint64_t *seg, uint64_t t);

// Warp 0: y = min{v : sum_{w<=v} mass_w > t} for t < Z, from the segment sums and one rescan.
template <bool BF16, class MassF>
__device__ int row_search(const char *prow, const char *qrow, int64_t V, const MassF &mass, const uint64_t *seg,
                          uint64_t t) {
    using E = RowElt<BF16>;
    constexpr int J = kSegElems / E::kVec / 32;
    const int lane = threadIdx.x & 31;   // one warp
    const int nseg = (int)((V + kSegElems - 1) / kSegElems);
    int sstar = nseg - 1;
    for (int s0 = 0; s0 < nseg; s0 += 32) {
        const uint64_t v = s0 + lane < nseg ? seg[s0 + lane] : 0;
        const uint64_t incl = wscan(v, lane);
        const uint64_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (t < tot) {
            const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
            t -= __shfl_sync(0xFFFFFFFFu, incl - v, src);
            sstar = s0 + src;
            break;
        }
        t -= tot;
    }
    const int64_t base = (int64_t)sstar * kSegElems;
    for (int j = 0; j < J; ++j) {   // vocabulary order: vector j*32 + lane, entries in order
        const int64_t e0 = base + (int64_t)(j * 32 + lane) * E::kVec;
        uint64_t me[E::kVec], msum = 0;
        uint4 pv = make_uint4(0, 0, 0, 0), qv = make_uint4(0, 0, 0, 0);
        if (e0 < V) {
            pv = ld_nc(prow + e0 * E::kEsz);
            if (qrow) qv = ld_nc(qrow + e0 * E::kEsz);
        }
#pragma unroll
        for (int e = 0; e < E::kVec; ++e) {
            me[e] = e0 < V ? mass(E::get(pv, e), E::get(qv, e)) : 0;
            msum += me[e];
        }
        const uint64_t incl = wscan(msum, lane);
        const uint64_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (t < tot) {
            const int src = __ffs(__ballot_sync(0xFFFFFFFFu, incl > t)) - 1;
            int yy = 0;
            if (lane == src) {
                uint64_t tt = t - (incl - msum);
                int e = 0;
                for (; e < E::kVec - 1; ++e) {
                    if (tt < me[e]) break;
                    tt -= me[e];
                }
                yy = (int)(e0 + e);
            }
            return __shfl_sync(0xFFFFFFFFu, yy, src);
        }
        t -= tot;
    }
    return (int)(V - 1);   // unreachable for t < Z
}

template <bool BF16>
__device__ uint64_t stage_pass(const char *prow, const char *qrow, int64_t V, int stage, const uint64_t *Zs,
                               const int *zb, uint64_t *seg, uint64_t *s_tot, const Grp &gr) {
    switch (stage) {
    case 0: return row_pass<BF16>(prow, nullptr, V, StageMass{0, nullptr, nullptr}, seg, s_tot, gr);
    case 1: return row_pass<BF16>(prow, qrow, V, StageMassT<1>(Zs, zb), seg, s_tot, gr);
    case 2: return row_pass<BF16>(prow, qrow, V, StageMassT<2>(Zs, zb), seg, s_tot, gr);
    case 3: return row_pass<BF16>(prow, qrow, V, StageMassT<3>(Zs, zb), seg, s_tot, gr);
    case 4: return row_pass<BF16>(prow, qrow, V, StageMassT<4>(Zs, zb), seg, s_tot, gr);
    default: return row_pass<BF16>(prow, qrow, V, StageMass{stage, Zs, zb}, seg, s_tot, gr);
    }
}
template <bool BF16>
__device__ int stage_search(const char *prow, const char *qrow, int64_t V, int stage, const uint64_t *Zs,
                            const int *zb, const uint64_t *seg, uint64_t t) {
    switch (stage) {
    case 0: return row_search<BF16>(prow, nullptr, V, StageMass{0, nullptr, nullptr}, seg, t);
    case 1: return row_search<BF16>(prow, qrow, V, StageMassT<1>(Zs, zb), seg, t);
    case 2: return row_search<BF16>(prow, qrow, V, StageMassT<2>(Zs, zb), seg, t);
    case 3: return row_search<BF16>(prow, qrow, V, StageMassT<3>(Zs, zb), seg, t);
    case 4: return row_search<BF16>(prow, qrow, V, StageMassT<4>(Zs, zb), seg, t);
    default: return row_search<BF16>(prow, qrow, V, StageMass{stage, Zs, zb}, seg, t);
    }
}

__device__ __forceinline__ uint64_t philox_u64(uint32_t req, uint32_t rnd, uint32_t c2, uint32_t trace,
                                               uint64_t seed) {
    const uint4 u = philox4x32_10(make_uint4(req, rnd, c2, trace), (uint32_t)seed, (uint32_t)(seed >> 32));
    return ((uint64_t)u.x << 32) | u.y;
}

// ---------------------------------------------------------------- draft sampling
template <bool BF16>
__global__ void __launch_bounds__(kRowThreads) draft_sample_kernel(const char *q, const int32_t *row_idx, int64_t V,
                                                                   const uint32_t *req, const uint32_t *rnd,
                                                                   const uint32_t *pos, uint64_t seed, uint32_t trace,
                                                                   int32_t *out, uint64_t *z_out) {
    __shared__ uint64_t seg[kMaxSegs];
    __shared__ uint64_t s_tot;
    const int r = blockIdx.x;
    const int64_t row = row_idx ? row_idx[r] : r;
    const char *qrow = q + row * V * RowElt<BF16>::kEsz;
    const StageMass m{0, nullptr, nullptr};
    const Grp gr{(int)threadIdx.x, (int)blockDim.x, 0};
    const uint64_t Z = row_pass<BF16>(qrow, nullptr, V, m, seg, &s_tot, gr);   // (draft: stage 0 = the row)
    if (threadIdx.x >= 32) return;
    int x = 0;
    if (Z) {
        const uint64_t U = philox_u64(req[r], rnd[r], (2u << 16) | pos[r], trace, seed);
        x = row_search<BF16>(qrow, nullptr, V, m, seg, __umul64hi(U, Z));
    }
    if (threadIdx.x == 0) {
        out[r] = x;
        if (z_out) z_out[r] = Z;
    }
}

// ---------------------------------------------------------------- tree verification
// u24 q(x) Z < D(x) 2^24 exactly, q(x) = m 2^e2 the stored float.
__device__ __forceinline__ bool tree_accept(uint32_t u24, float qx, uint64_t Dx, uint64_t Z) {
    if (Dx == 0) return false;
    if (!(qx > 0.0f)) return true;
    const uint32_t bits = __float_as_uint(qx);
    const int ex = (int)((bits >> 23) & 0xFF);
    uint64_t m = bits & 0x7FFFFFu;
    int e2 = -149;
    if (ex) { m |= 0x800000u; e2 = ex - 150; }
    const int sh = 24 - e2;                               // compare u24 m Z < D 2^sh
    const int dbits = 64 - __clzll((long long)Dx);
    if (dbits + sh > 127) return true;                    // D 2^sh >= 2^127 > u24 m Z
    return (u128)u24 * m * Z < ((u128)Dx << sh);
}

// kTreesPerCta trees per CTA, one group of kTreeThreads / kTreesPerCta threads each (named
// barrier 1 + group): while one tree waits on a gather, a barrier or its loads, the others
// issue.
template <bool BF16>
__global__ void __launch_bounds__(kTreeThreads, 1) tree_verify_kernel(const char *p, const char *q, int64_t V,
                                                                  int32_t n_nodes, const int32_t *parent,
                                                                  const int32_t *token, const uint32_t *req_id,
                                                                  const uint32_t *round_idx, uint64_t seed,
                                                                  uint32_t trace, int32_t *tokens, int32_t *path,
                                                                  int32_t *n_accept, uint64_t *z_out, int32_t B) {
    using E = RowElt<BF16>;
    constexpr int GT = kTreeThreads / kTreesPerCta;
    __shared__ uint64_t seg_all[kTreesPerCta][kMaxSegs];
    __shared__ uint64_t s_tot_all[kTreesPerCta];
    __shared__ uint64_t s_Zs_all[kTreesPerCta][kTreeMax + 1];
    __shared__ int s_zb_all[kTreesPerCta][kTreeMax + 1];
    __shared__ int s_par_all[kTreesPerCta][kTreeMax], s_tok_all[kTreesPerCta][kTreeMax];
    __shared__ int s_dep_all[kTreesPerCta][kTreeMax], s_ch_all[kTreesPerCta][kTreeMax];
    __shared__ int s_ok_all[kTreesPerCta], s_w_all[kTreesPerCta], s_acc_all[kTreesPerCta];
    const int g = (int)threadIdx.x / GT;
    const Grp gr{(int)threadIdx.x % GT, GT, 1 + g};
    const int tid = gr.tid;
    const int b = blockIdx.x * kTreesPerCta + g, n = n_nodes;
    if (b >= B) return;
    uint64_t *seg = seg_all[g];
    uint64_t *s_Zs = s_Zs_all[g];
    int *s_zb = s_zb_all[g], *s_par = s_par_all[g], *s_tok = s_tok_all[g], *s_dep = s_dep_all[g], *s_ch = s_ch_all[g];
    int &s_ok = s_ok_all[g], &s_w = s_w_all[g], &s_acc = s_acc_all[g];
    uint64_t *s_tot = &s_tot_all[g];
    const uint32_t req = req_id[b], rnd = round_idx[b];
    const int32_t *par_g = parent + (int64_t)b * n;
    const int32_t *tok_g = token + (int64_t)b * n;
    const char *pb = p + (int64_t)b * n * V * E::kEsz;
    const char *qb = q + (int64_t)b * n * V * E::kEsz;
    int32_t *tok_o = tokens + (int64_t)b * n;
    int32_t *path_o = path ? path + (int64_t)b * n : nullptr;
    for (int c = tid; c < n; c += GT) {
        s_par[c] = par_g[c];
        s_tok[c] = tok_g[c];
        tok_o[c] = -1;
        if (path_o) path_o[c] = -1;
    }
    gr.sync();
    if (tid == 0) {   // structure: parent before child, tokens in range
        int ok = 1;
        s_dep[0] = 0;
        for (int c = 1; c < n && ok; ++c) {
            const int pc = s_par[c];
            if (pc < 0) { s_dep[c] = -1; continue; }
            if (pc >= c || s_dep[pc] < 0 || s_tok[c] < 0 || s_tok[c] >= V) ok = 0;
            else s_dep[c] = s_dep[pc] + 1;
        }
        s_ok = ok;
    }
    gr.sync();
    if (!s_ok) {
        if (tid == 0) { n_accept[b] = -1; if (z_out) z_out[b] = 0; }
        return;
    }
    int u = 0, nacc = 0;
    for (;;) {
        if (tid == 0) {
            int w = 0;
            for (int c = u + 1; c < n; ++c)
                if (s_par[c] == u) s_ch[w++] = c;
            s_w = w;
        }
        gr.sync();
        const int w = s_w;
        const char *prow = pb + (int64_t)u * V * E::kEsz;
        const char *qrow = qb + (int64_t)u * V * E::kEsz;
        int next = -1, stage = 0;
        bool fallback = false;
        for (int i = 0; i < w; ++i) {
            if (tid == 0) {
                const int x = s_tok[s_ch[i]];
                const float px = E::get(ld_nc(prow + ((int64_t)x - (x % E::kVec)) * E::kEsz), x % E::kVec);
                const float qx = E::get(ld_nc(qrow + ((int64_t)x - (x % E::kVec)) * E::kEsz), x % E::kVec);
                bool acc;
                if (i == 0) {   // the linear verification's rule at depth d
                    const int d = s_dep[u];
                    const uint4 r4 = philox4x32_10(make_uint4(req, rnd, (uint32_t)(d >> 2), trace), (uint32_t)seed,
                                                   (uint32_t)(seed >> 32));
                    const uint32_t wv = (d & 3) == 0 ? r4.x : (d & 3) == 1 ? r4.y : (d & 3) == 2 ? r4.z : r4.w;
                    acc = __dmul_rn((double)(wv >> 8), (double)qx) < __dmul_rn((double)px, 16777216.0);
                } else {        // against the normalised residual D_i
                    const uint32_t c2 = (3u << 16) | ((uint32_t)u << 8) | (uint32_t)((i - 1) >> 2);
                    const uint4 r4 = philox4x32_10(make_uint4(req, rnd, c2, trace), (uint32_t)seed,
                                                   (uint32_t)(seed >> 32));
                    const int l = (i - 1) & 3;
                    const uint32_t wv = l == 0 ? r4.x : l == 1 ? r4.y : l == 2 ? r4.z : r4.w;
                    const StageMass m{i, s_Zs, s_zb};
                    acc = tree_accept(wv >> 8, qx, m(px, qx), s_Zs[i]);
                }
                s_acc = acc;
            }
            gr.sync();
            if (s_acc) { next = s_ch[i]; break; }
            // D_{i+1} and its total (the segment sums stay for a final draw from it)
            const uint64_t Z = stage_pass<BF16>(prow, qrow, V, i + 1, s_Zs, s_zb, seg, s_tot, gr);
            stage = i + 1;
            if (tid == 0) {
                s_Zs[stage] = Z;
                s_zb[stage] = 64 - __clzll((long long)Z);
            }
            gr.sync();
            if (Z == 0) { fallback = true; break; }   // AMB-20: no residual mass
        }
        if (next >= 0) {
            if (tid == 0) {
                tok_o[nacc] = s_tok[next];
                if (path_o) path_o[nacc] = next;
            }
            ++nacc;
            u = next;
            gr.sync();
            continue;
        }
        // the emitted token: from D_stage (every child rejected), else from the row p_u
        // (a leaf's bonus token or the AMB-20 fallback)
        uint64_t Z;
        int st_draw = stage;
        if (stage > 0 && !fallback) {
            Z = s_Zs[stage];
        } else {
            st_draw = 0;
            Z = stage_pass<BF16>(prow, nullptr, V, 0, s_Zs, s_zb, seg, s_tot, gr);
        }
        if (tid < 32) {
            int y = 0;
            if (Z) {
                const uint64_t U = philox_u64(req, rnd, 1u << 8, trace, seed);
                y = stage_search<BF16>(prow, qrow, V, st_draw, s_Zs, s_zb, seg, __umul64hi(U, Z));
            }
            if (tid == 0) {
                tok_o[nacc] = y;
                n_accept[b] = nacc;
                if (z_out) z_out[b] = Z;
            }
        }
        return;
    }
}

}  // namespace

cudaError_t launch_draft_sample(const void *q, int32_t dtype, int64_t V, const int32_t *row_idx,
                                const uint32_t *req, const uint32_t *rnd, const uint32_t *pos, int32_t R,
                                uint64_t seed, uint32_t trace, int32_t *out, uint64_t *z_out, cudaStream_t s) {
    if (R <= 0) return cudaSuccess;
    if (dtype == LAPSSD_BF16)
        draft_sample_kernel<true><<<R, kRowThreads, 0, s>>>((const char *)q, row_idx, V, req, rnd, pos, seed, trace,
                                                            out, z_out);
    else
        draft_sample_kernel<false><<<R, kRowThreads, 0, s>>>((const char *)q, row_idx, V, req, rnd, pos, seed, trace,
                                                             out, z_out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_verify_tree(const void *p, const void *q, int32_t dtype, int64_t V, int32_t n_nodes,
                               const int32_t *parent, const int32_t *token, const uint32_t *req,
                               const uint32_t *rnd, int32_t B, uint64_t seed, uint32_t trace, int32_t *tokens,
                               int32_t *path, int32_t *n_accept, uint64_t *z_out, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    if (dtype == LAPSSD_BF16)
        tree_verify_kernel<true><<<(B + kTreesPerCta - 1) / kTreesPerCta, kTreeThreads, 0, s>>>(
            (const char *)p, (const char *)q, V, n_nodes, parent, token, req, rnd, seed, trace, tokens, path,
            n_accept, z_out, B);
    else
        tree_verify_kernel<false><<<(B + kTreesPerCta - 1) / kTreesPerCta, kTreeThreads, 0, s>>>(
            (const char *)p, (const char *)q, V, n_nodes, parent, token, req, rnd, seed, trace, tokens, path,
            n_accept, z_out, B);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lapssd
