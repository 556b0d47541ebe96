// select_core.cuh -- block-level selection primitives shared by the select kernels
// (sched.cu) and the fused final select at the end of the verify kernel (verify.cu):
// warp-register bitonic sort + merge-path block sort, radix top-B selection, admission,
// key building and commits.  PAPER.md P:129-142; DESIGN.md s.6.
#pragma once

#include "lapssd_internal.cuh"

namespace lapssd {

constexpr int kSelThreads = 1024;
constexpr int kSideThreads = 1024;     // side-stream select (measured: 512 is slower)
constexpr int kSortCap = 16384;          // keys per CTA (bitonic in place above kMergeCap)
constexpr int kMergeCap = 8192;          // keys sorted by warp-sort + merge-path (2 buffers)
constexpr int kFastTopCap = 4096;        // top-B by full sort up to this many keys (else radix select)

// ---------------------------------------------------------------- block sort
__device__ inline void bitonic_sort(uint64_t *s, int n) {  // n power of two, ascending, in place
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = s[i], y = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) { s[i] = y; s[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

// Sort one 64-key run held as (lo = element lane, hi = element lane + 32).
__device__ __forceinline__ void warp_sort64(uint64_t &lo, uint64_t &hi, int lane) {
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                const bool asc = true;  // k == 64: (e & 64) == 0 for every element
                const uint64_t a = lo < hi ? lo : hi, b = lo < hi ? hi : lo;
                lo = asc ? a : b;
                hi = asc ? b : a;
            } else {
                const bool lower = (lane & j) == 0;
                {
                    const uint64_t p = __shfl_xor_sync(0xFFFFFFFFu, lo, j);
                    const bool asc = ((lane & k) == 0);
                    lo = (lower == asc) ? (lo < p ? lo : p) : (lo > p ? lo : p);
                }
                {
                    const uint64_t p = __shfl_xor_sync(0xFFFFFFFFu, hi, j);
                    const bool asc = (((lane + 32) & k) == 0);
                    hi = (lower == asc) ? (hi < p ? hi : p) : (hi > p ? hi : p);
                }
            }
        }
    }
}

// Register-resident bitonic sort of n keys held in s (n = E * T, T = n / E threads
// take part; the block's other threads only join the barriers).  Thread t holds the
// elements e(m) = (t/32)*32E + 32m + lane, m < E, so a partner at distance j < 32 is a
// warp shuffle, 32 <= j < 32E is a swap inside the thread, and only j >= 32E goes
// through shared memory.  Ascending; result back in s.
template <int E>
__device__ void bitonic_reg(uint64_t *s, int n) {
    const int T = n / E;
    const int t = threadIdx.x;
    const bool on = t < T;
    const int lane = t & 31;
    const int ebase = (t >> 5) * 32 * E + lane;   // element of v[m] is ebase + 32 m
    uint64_t v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = on ? s[ebase + 32 * m] : ~0ull;
    for (int k = 2; k <= n; k <<= 1) {
        int j = k >> 1;
        if (j >= 32 * E) {  // cross-warp distances: in shared memory
            if (on) {
#pragma unroll
                for (int m = 0; m < E; ++m) s[ebase + 32 * m] = v[m];
            }
            __syncthreads();
            for (; j >= 32 * E; j >>= 1) {
                if (on) {
#pragma unroll
                    for (int m = 0; m < E; ++m) {
                        const int e = ebase + 32 * m;
                        const uint64_t b = s[e ^ j];
                        const bool lower = (e & j) == 0, asc = (e & k) == 0;
                        v[m] = (lower == asc) ? (v[m] < b ? v[m] : b) : (v[m] > b ? v[m] : b);
                    }
                }
                __syncthreads();
                if (on) {
#pragma unroll
                    for (int m = 0; m < E; ++m) s[ebase + 32 * m] = v[m];
                }
                __syncthreads();
            }
        }
        // inside the thread: distances 32*dm for dm = E/2 .. 1 (compile-time register indices)
#pragma unroll
        for (int dm = E / 2; dm >= 1; dm >>= 1) {
            if (32 * dm <= j) {
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    if ((m & dm) == 0) {
                        const bool asc = ((ebase + 32 * m) & k) == 0;
                        const uint64_t a = v[m], b = v[m | dm];
                        const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
                        v[m] = asc ? lo : hi;
                        v[m | dm] = asc ? hi : lo;
                    }
                }
            }
        }
        if (j >= 32) j = 16;
        for (; j > 0; j >>= 1) {  // inside the warp
            const bool lower = (lane & j) == 0;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const uint64_t p = __shfl_xor_sync(0xFFFFFFFFu, v[m], j);
                const bool asc = ((ebase + 32 * m) & k) == 0;
                v[m] = (lower == asc) ? (v[m] < p ? v[m] : p) : (v[m] > p ? v[m] : p);
            }
        }
    }
    __syncthreads();
    if (on) {
#pragma unroll
        for (int m = 0; m < E; ++m) s[ebase + 32 * m] = v[m];
    }
    __syncthreads();
}

// Block sort front end: picks E so that n / E threads fit in the block.
__device__ inline void block_sort_reg(uint64_t *s, int n) {
    int T = 1;
    while (T * 2 <= (int)blockDim.x) T <<= 1;
    if (n < 64) {
        bitonic_sort(s, n);
        return;
    }
    const int E = n / T > 0 ? n / T : 1;
    if (n / E < 32) { bitonic_sort(s, n); return; }
    switch (E) {
    case 1: bitonic_reg<1>(s, n); break;
    case 2: bitonic_reg<2>(s, n); break;
    case 4: bitonic_reg<4>(s, n); break;
    case 8: bitonic_reg<8>(s, n); break;
    default: bitonic_sort(s, n); break;
    }
}

// Sorts n (power of two) keys; returns the buffer holding the result (a or b).
#ifdef LAPSSD_SIDE_NOINLINE
__device__ __noinline__
#else
__device__ inline
#endif
uint64_t *block_sort(uint64_t *a, uint64_t *b, int n) {
    if (n < 64 || n > kMergeCap || b == nullptr) {
        bitonic_sort(a, n);
        return a;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int run = warp; run < n / 64; run += nwarps) {
        uint64_t lo = a[run * 64 + lane], hi = a[run * 64 + 32 + lane];
        warp_sort64(lo, hi, lane);
        a[run * 64 + lane] = lo;
        a[run * 64 + 32 + lane] = hi;
    }
    __syncthreads();
    uint64_t *src = a, *dst = b;
    const int T = blockDim.x;
    int per = 1;  // outputs per thread: a power of two, so no thread's range crosses a pair
    while (per * 2 * T <= n) per *= 2;
    for (int w = 64; w < n; w <<= 1) {
        for (int o0 = threadIdx.x * per; o0 < n; o0 += T * per) {
            const int pair = o0 / (2 * w);
            const int d0 = o0 - pair * 2 * w;
            const uint64_t *A = src + pair * 2 * w;
            const uint64_t *Bv = A + w;
            int lo = d0 - w > 0 ? d0 - w : 0, hi = d0 < w ? d0 : w;
            while (lo < hi) {  // number of A elements among the first d0 outputs
                const int mid = (lo + hi) >> 1;
                if (A[mid] <= Bv[d0 - 1 - mid]) lo = mid + 1; else hi = mid;
            }
            int i = lo, j = d0 - lo;
            for (int e = 0; e < per; ++e) {
                const bool takeA = j >= w || (i < w && A[i] <= Bv[j]);
                dst[o0 + e] = takeA ? A[i++] : Bv[j++];
            }
        }
        __syncthreads();
        uint64_t *t = src; src = dst; dst = t;
    }
    return src;
}

// The B smallest of n keys, sorted ascending, into out[0..bp) (bp = next_pow2(B) with
// UINT64_MAX padding); tmp is bp words of scratch.  MSB-first radix select finds the
// B-th smallest key T with eight 256-bin histogram passes (keys are unique: the id is
// in the low bits), then the keys <= T are compacted and only they are sorted.
#ifdef LAPSSD_SIDE_NOINLINE
__device__ __noinline__
#else
__device__ inline
#endif
uint64_t *select_topB(const uint64_t *keys, int n, int B, uint64_t *out, uint64_t *tmp, int bp) {
    __shared__ int hist[256];
    __shared__ uint64_t s_prefix, s_mask;
    __shared__ int s_remaining, s_done;
    __shared__ int s_scan[64];
    const int want = B < n ? B : n;
    if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_remaining = want; s_done = 0; }
    __syncthreads();
    for (int shift = 56; shift >= 0 && want > 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        if (s_done) break;
        const uint64_t prefix = s_prefix, mask = s_mask;
        // keys share their high bytes (flags, level, a zero estimate field), so most land
        // in one bin: aggregate equal bins across the warp first (one atomic per bin per
        // warp instead of one per key)
        const int n32 = (n + 31) & ~31;
        for (int i = threadIdx.x; i < n32; i += blockDim.x) {
            int bin = 256;  // no bin: out of range or outside the prefix
            if (i < n) {
                const uint64_t key = keys[i];
                if ((key & mask) == prefix) bin = (int)((key >> shift) & 255);
            }
            const unsigned peers = __match_any_sync(__activemask(), bin);
            if (bin < 256 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int loc[8], sum = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { loc[e] = hist[lane * 8 + e]; sum += loc[e]; }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            const int rem = s_remaining;
            const unsigned hit = __ballot_sync(0xFFFFFFFFu, incl >= rem);
            const int src = __ffs(hit) - 1;
            if (lane == src) {
                int acc = incl - sum;
                int dgt = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (acc + loc[e] >= rem) { dgt = lane * 8 + e; break; }
                    acc += loc[e];
                }
                const int cnt = hist[dgt];
                s_prefix = prefix | ((uint64_t)dgt << shift);
                s_mask = mask | (255ull << shift);
                s_remaining = rem - acc;
                if (rem - acc == cnt) s_done = 1;  // every key of this bin is needed
            }
        }
        __syncthreads();
    }
    // threshold: all keys matching the final prefix pattern up to its mask, i.e. key <= T
    const uint64_t T = want > 0 ? (s_prefix | ~s_mask) : 0;
    // compact keys <= T (exactly `want` of them) in index order, then sort
    const int per = (n + (int)blockDim.x - 1) / (int)blockDim.x;
    const int lo = (int)threadIdx.x * per;
    int mine = 0;
    // keys are unique except UINT64_MAX padding: take keys < T, plus T itself unless it
    // is the padding value (then the tail is filled with padding below)
    const bool t_real = T != ~0ull;
    for (int i = lo; i < lo + per && i < n; ++i) mine += want > 0 && (keys[i] < T || (t_real && keys[i] == T));
    int total = 0;
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        int x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += v;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int w = lane < (int)(blockDim.x >> 5) ? s_scan[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += v;
            }
            s_scan[32 + lane] = w;
        }
        __syncthreads();
        int pos = (warp > 0 ? s_scan[32 + warp - 1] : 0) + x - mine;
        total = s_scan[32 + (int)(blockDim.x >> 5) - 1];
        for (int i = lo; i < lo + per && i < n; ++i)
            if (want > 0 && (keys[i] < T || (t_real && keys[i] == T)) && pos < bp) out[pos++] = keys[i];
    }
    for (int i = total + (int)threadIdx.x; i < bp; i += blockDim.x) out[i] = ~0ull;
    __syncthreads();
    return block_sort(out, bp >= 64 && bp <= kMergeCap ? tmp : nullptr, bp);
}

__device__ __forceinline__ int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

// Same contract as select_topB.  When the caller has npow2 more words of scratch and
// npow2 <= kMergeCap, a full block sort (warp-register runs + merge-path, ~log2(n/64)
// barriers) is much shorter than eight radix passes of barriers; keys[0..npow2) must be
// padded with UINT64_MAX and is clobbered.  topB_smem_words sizes the caller's buffer.  The result is the first bp words of the
// sorted buffer, with the entries from B on reset to UINT64_MAX (select_topB's padding).
__device__ inline const uint64_t *select_topB_fast(uint64_t *keys, int n, int B, uint64_t *out, uint64_t *tmp,
                                                   int bp, uint64_t *scratch) {
    const int np = next_pow2(n > 0 ? n : 1);
    if (scratch == nullptr || np < bp || np < 64 || np > kFastTopCap) return select_topB(keys, n, B, out, tmp, bp);
    uint64_t *s = block_sort(keys, scratch, np);
    for (int b = B + (int)threadIdx.x; b < bp; b += blockDim.x) s[b] = ~0ull;
    __syncthreads();
    return s;
}

// Shared-memory words for keys[np] + out[bp] + tmp[bp] (+ scratch[np] on the fast path).
__host__ __device__ inline size_t topB_smem_words(int np, int bp) {
    return (size_t)np + 2 * (size_t)bp + (np >= bp && np >= 64 && np <= kFastTopCap ? (size_t)np : 0);
}

__host__ __device__ inline size_t sort_smem_bytes(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return (size_t)p * sizeof(uint64_t) * (p >= 64 && p <= kMergeCap ? 2 : 1);
}

// Block-wide exclusive scan of one int per thread.
__device__ inline int block_excl_scan(int v, int *s_tmp, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += n;
    }
    if (lane == 31) s_tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (int)(blockDim.x >> 5) ? s_tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= o) w += n;
        }
        s_tmp[32 + lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int before = warp > 0 ? s_tmp[32 + warp - 1] : 0;
    *total = s_tmp[32 + (int)(blockDim.x >> 5) - 1];
    __syncthreads();
    return before + x - v;
}

// a7 (first half) + a4: advance the clock by the step that ran (its round plus the
// switch-ins it paid), admit arrivals.
// Arrivals are sorted, so the admitted set is the prefix [0, cursor).
__device__ inline void advance_and_admit(const State &st, const Sched &sc, int64_t *s_now, int *s_cursor) {
    if (threadIdx.x == 0) {
        int64_t now = st.g->now_us;
        if (st.g->prev_count > 0) now += sc.c_round_us + st.g->step_sw;   // AMB-17, AMB-24
        *s_now = now;
        *s_cursor = st.g->cursor;
    }
    __syncthreads();
    const int64_t now = *s_now;
    int cursor = *s_cursor;
    for (;;) {
        const int idx = cursor + (int)threadIdx.x;
        const bool adm = idx < sc.n && st.arrival[idx] <= now;
        const int cnt = __syncthreads_count(adm);
        cursor += cnt;
        if (cnt < (int)blockDim.x) break;
    }
    if (threadIdx.x == 0) *s_cursor = cursor;
    __syncthreads();
}

// Build every key into global and shared memory (padded to npow2 with UINT64_MAX)
// and clear the running flags (they describe the round that just ran).
__device__ inline void build_keys(const State &st, const Sched &sc, int cursor, uint64_t *s_keys, int npow2) {
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < sc.n) {
            const uint32_t fl = st.flags[i];
            const int32_t lp = st.L_pred[i], tok = st.acc_tok[i];
            const double A = st.A[i];
            key = build_key(sc, i, cursor, fl, lp, tok, A);
            st.key[i] = key;
            if (fl & F_RUNNING) st.flags[i] = fl & ~F_RUNNING;
        }
        s_keys[i] = key;
    }
    __syncthreads();
}

// Commit one selected request: first-service time and pinning (AMB-15, AMB-25), and its
// switch-in cost for selection number seq + 1 (AMB-24), which it returns.
__device__ __forceinline__ int64_t commit_one(const State &st, const Sched &sc, int32_t i, int64_t now,
                                              uint32_t seq) {
    if (st.x[i] < 0) st.x[i] = now;                                // x_i
    const uint32_t fl = st.flags[i];
    bool pin = false;
    if (sc.policy == LAPSSD_POL_FCFS || sc.policy == LAPSSD_POL_LPSJF) pin = true;
    else if (sc.policy == LAPSSD_POL_LAPSSD && sc.pin_rule == 0 && (fl & F_PERC)) pin = true;
    if (pin && !(fl & F_PINNED)) st.flags[i] = fl | F_PINNED;
    const int64_t c = switch_in_cost(st, sc, i, seq);
    charge_switch(st, sc, i, seq, c);
    return c;
}

// Block-wide sum of the committed switch-in costs and the commit's globals: the step of
// the batch just selected lasts c_round + sw (nothing when the batch is empty), the
// selection counter advances.  Every thread passes its partial sum; thread 0 writes.
__device__ inline void commit_switch(const State &st, const Sched &sc, int64_t part, int global_count,
                                     unsigned long long *s_sum) {
    if (sc.sw_on) {
        if (threadIdx.x == 0) *s_sum = 0;
        __syncthreads();
        if (part) atomicAdd(s_sum, (unsigned long long)part);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t sw = sc.sw_on && global_count > 0 ? (int64_t)*s_sum : 0;
        st.g->step_sw = sw;
        st.g->switch_total += sw;
        st.g->sel_seq = st.g->sel_seq + 1;
    }
}



}  // namespace lapssd
