// sched.cu -- LAPS-SD scheduler kernels on sm_100a: state update (a3), admission +
// priority keys + top-B selection + clock (a4-a7), and the multi-GPU candidate /
// merge halves of the global top-B (a8).  PAPER.md P:84-93.
//
// Selection runs in ONE CTA of 1024 threads: every resident request's 64-bit key is
// built from the SoA state, the keys are sorted in shared memory -- each warp sorts
// 64-key runs in registers with a shuffle bitonic network (no barriers), then
// merge-path rounds double the run length (one barrier per round) -- and the first B
// eligible keys become the batch.  The tail of the same kernel runs the acceptance
// test (a1) of every newly selected slot, so the next verify launch starts streaming
// after a single descriptor load.
#include "lapssd_internal.cuh"

namespace lapssd {

constexpr int kSelThreads = 1024;
constexpr int kSortCap = 16384;          // keys per CTA (bitonic in place above kMergeCap)
constexpr int kMergeCap = 8192;          // keys sorted by warp-sort + merge-path (2 buffers)

int sort_capacity() { return kSortCap; }

// ---------------------------------------------------------------- a3 standalone
__global__ void update_kernel(const State st, const Sched sc, const int32_t *sel,
                              const int32_t *n_accept, int32_t B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int32_t i = sel[b];
    if (i < 0) return;
    if (i >= sc.n) { atomicOr(&st.g->err, E_BAD_SLOT); return; }
    update_one(st, sc, i, n_accept[b], st.g->now_us);
}

cudaError_t launch_update(const State &st, const Sched &sc, const int32_t *sel,
                          const int32_t *n_accept, int32_t B, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    update_kernel<<<(B + 255) / 256, 256, 0, s>>>(st, sc, sel, n_accept, B);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- block sort
__device__ void bitonic_sort(uint64_t *s, int n) {  // n power of two, ascending, in place
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

// Sorts n (power of two) keys; returns the buffer holding the result (a or b).
__device__ uint64_t *block_sort(uint64_t *a, uint64_t *b, int n) {
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
    const int per = n >= T ? n / T : 1;
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
__device__ uint64_t *select_topB(const uint64_t *keys, int n, int B, uint64_t *out, uint64_t *tmp, int bp) {
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
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t key = keys[i];
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
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

__host__ __device__ inline size_t sort_smem_bytes(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return (size_t)p * sizeof(uint64_t) * (p >= 64 && p <= kMergeCap ? 2 : 1);
}

// Block-wide exclusive scan of one int per thread.
__device__ int block_excl_scan(int v, int *s_tmp, int *total) {
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

// a7 (first half) + a4: advance the clock by the round that ran, admit arrivals.
// Arrivals are sorted, so the admitted set is the prefix [0, cursor).
__device__ void advance_and_admit(const State &st, const Sched &sc, int64_t *s_now, int *s_cursor) {
    if (threadIdx.x == 0) {
        int64_t now = st.g->now_us;
        if (st.g->prev_count > 0) now += sc.c_round_us;         // AMB-17
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
__device__ void build_keys(const State &st, const Sched &sc, int cursor, uint64_t *s_keys, int npow2) {
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

// Commit one selected request: first-service time and pinning (AMB-15, AMB-25).
__device__ __forceinline__ void commit_one(const State &st, const Sched &sc, int32_t i, int64_t now) {
    if (st.x[i] < 0) st.x[i] = now;                                // x_i
    const uint32_t fl = st.flags[i];
    bool pin = false;
    if (sc.policy == LAPSSD_POL_FCFS || sc.policy == LAPSSD_POL_LPSJF) pin = true;
    else if (sc.policy == LAPSSD_POL_LAPSSD && sc.pin_rule == 0 && (fl & F_PERC)) pin = true;
    if (pin && !(fl & F_PINNED)) st.flags[i] = fl | F_PINNED;
}

// ---------------------------------------------------------------- a4-a7 select
__global__ void __launch_bounds__(kSelThreads) select_kernel(const State st, const Sched sc, const RowsDev rw,
                                                              SlotDesc *desc, int32_t B, int32_t *sel_out,
                                                              int32_t *count_out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor, s_count;
    advance_and_admit(st, sc, &s_now, &s_cursor);
    const int64_t now = s_now;
    const int cursor = s_cursor;
    const int npow2 = next_pow2(sc.n > 0 ? sc.n : 1);
    build_keys(st, sc, cursor, s_buf, npow2);
    const int bp = next_pow2(B);
    const uint64_t *keys = select_topB(s_buf, sc.n, B, s_buf + npow2, s_buf + npow2 + bp, bp);
    // eligible keys (bit 63 clear) form a prefix of the sorted array
    const int lim = B < bp ? B : bp;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int valid = 0;
    for (int b = threadIdx.x; b < lim; b += blockDim.x) valid += (keys[b] >> 63) == 0;
    if (valid) atomicAdd(&s_count, valid);
    __syncthreads();
    const int cnt = s_count;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t i = -1;
        if (b < cnt) {
            const uint32_t id = (uint32_t)(keys[b] & 0xFFFFFFull);
            i = (int32_t)(id / (uint32_t)sc.world);
            commit_one(st, sc, i, now);
        }
        sel_out[b] = i;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, i);    // a1 for the next verify
    }
    if (threadIdx.x == 0) {
        int64_t nnow = now;
        if (cnt == 0 && cursor < sc.n) {                             // idle: jump
            const int64_t nxt = st.arrival[cursor];
            if (nxt > nnow) nnow = nxt;
        }
        st.g->now_us = nnow;
        st.g->cursor = cursor;
        st.g->prev_count = cnt;
        st.g->count = cnt;
        if (count_out) *count_out = cnt;
    }
}

static void set_smem_attr(const void *fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // same L1/shared split as the verify kernel: no carveout reconfiguration between launches
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// ---------------------------------------------------------------- split select
// Keys of requests outside the current batch do not depend on this step's
// verification, so presort_kernel computes them -- clock advance, admission, keys,
// top-B, sorted -- on a side stream while the verify kernel streams.  After the join,
// select_final_kernel rebuilds only the B updated keys, sorts them and merges the two
// sorted lists: the top-B of the union is the top-B of all keys.
__global__ void __launch_bounds__(kSelThreads) presort_kernel(const State st, const Sched sc, const int32_t *sel,
                                                               int32_t B, PreSelect *out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor;
    __shared__ uint32_t s_member[kSortCap / 32];
    const int n = sc.n;
    for (int w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) s_member[w] = 0;
    advance_and_admit(st, sc, &s_now, &s_cursor);   // ends with a barrier
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        const int i = sel[b];
        if (i >= 0) atomicOr(&s_member[i >> 5], 1u << (i & 31));
    }
    __syncthreads();
    const int npow2 = next_pow2(n > 0 ? n : 1);
    const int cursor = s_cursor;
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < n && !((s_member[i >> 5] >> (i & 31)) & 1u)) {
            const uint32_t fl = st.flags[i];
            const int32_t lp = st.L_pred[i], tok = st.acc_tok[i];
            const double A = st.A[i];
            key = build_key(sc, i, cursor, fl, lp, tok, A);
            st.key[i] = key;
            if (key >> 63) key = ~0ull;   // ineligible: never selected
        }
        s_buf[i] = key;
    }
    __syncthreads();
    const int bp = next_pow2(B);
    const uint64_t *top = select_topB(s_buf, n, B, s_buf + npow2, s_buf + npow2 + bp, bp);
    for (int b = threadIdx.x; b < bp; b += blockDim.x) out->cand[b] = top[b];
    if (threadIdx.x == 0) {
        out->now_us = s_now;
        out->cursor = s_cursor;
    }
}

__global__ void __launch_bounds__(kSelThreads) select_final_kernel(const State st, const Sched sc, const RowsDev rw,
                                                                    SlotDesc *desc, int32_t B, int32_t *sel,
                                                                    int32_t *count_out, const PreSelect *pre) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int s_count;
    const int bp = next_pow2(B);
    const int64_t now = pre->now_us;
    const int cursor = pre->cursor;
    // keys of the verified batch, after their update
    for (int b = threadIdx.x; b < bp; b += blockDim.x) {
        uint64_t key = ~0ull;
        const int i = b < B ? sel[b] : -1;
        if (i >= 0) {
            const uint32_t fl = st.flags[i];
            const int32_t lp = st.L_pred[i], tok = st.acc_tok[i];
            const double A = st.A[i];
            key = build_key(sc, i, cursor, fl, lp, tok, A);
            st.key[i] = key;
            if (fl & F_RUNNING) st.flags[i] = fl & ~F_RUNNING;
        }
        s_buf[b] = key;
    }
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const uint64_t *bk = block_sort(s_buf, bp >= 64 && bp <= kMergeCap ? s_buf + bp : nullptr, bp);
    // merge path: first B outputs of merge(batch keys, presorted candidates)
    uint64_t *merged = (bk == s_buf) ? s_buf + bp : s_buf;
    const uint64_t *cand = pre->cand;
    for (int o = threadIdx.x; o < B; o += blockDim.x) {
        int lo = o - bp > 0 ? o - bp : 0, hi = o < bp ? o : bp;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (bk[mid] <= cand[o - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        const int i = lo, j = o - lo;
        const bool takeA = j >= bp || (i < bp && bk[i] <= cand[j]);
        merged[o] = takeA ? bk[i] : cand[j];
    }
    __syncthreads();
    int valid = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) valid += (merged[b] >> 63) == 0;
    if (valid) atomicAdd(&s_count, valid);
    __syncthreads();
    const int cnt = s_count;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t i = -1;
        if (b < cnt) {
            const uint32_t id = (uint32_t)(merged[b] & 0xFFFFFFull);
            i = (int32_t)(id / (uint32_t)sc.world);
            commit_one(st, sc, i, now);
        }
        sel[b] = i;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, i);
    }
    if (threadIdx.x == 0) {
        int64_t nnow = now;
        if (cnt == 0 && cursor < sc.n) {
            const int64_t nxt = st.arrival[cursor];
            if (nxt > nnow) nnow = nxt;
        }
        st.g->now_us = nnow;
        st.g->cursor = cursor;
        st.g->prev_count = cnt;
        st.g->count = cnt;
        if (count_out) *count_out = cnt;
    }
}

cudaError_t launch_presort(const State &st, const Sched &sc, const int32_t *sel, int32_t B, PreSelect *out,
                           cudaStream_t s) {
    static bool attr = false;
    if (!attr) { set_smem_attr((const void *)presort_kernel); attr = true; }
    int np = 1, bp = 1;
    while (np < (sc.n > 0 ? sc.n : 1)) np <<= 1;
    while (bp < B) bp <<= 1;
    presort_kernel<<<1, kSelThreads, (size_t)(np + 2 * bp) * sizeof(uint64_t), s>>>(st, sc, sel, B, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_final(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc, int32_t B,
                                int32_t *sel, int32_t *count_out, const PreSelect *pre, cudaStream_t s) {
    static bool attr = false;
    if (!attr) { set_smem_attr((const void *)select_final_kernel); attr = true; }
    int bp = 1;
    while (bp < B) bp <<= 1;
    select_final_kernel<<<1, kSelThreads, (size_t)(2 * bp) * sizeof(uint64_t), s>>>(st, sc, rw, desc, B, sel,
                                                                                     count_out, pre);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc, int32_t B,
                          int32_t *sel_out, int32_t *count_out, cudaStream_t s) {
    static bool attr = false;
    if (!attr) { set_smem_attr((const void *)select_kernel); attr = true; }
    int np = 1, bp = 1;
    while (np < (sc.n > 0 ? sc.n : 1)) np <<= 1;
    while (bp < B) bp <<= 1;
    select_kernel<<<1, kSelThreads, (size_t)(np + 2 * bp) * sizeof(uint64_t), s>>>(st, sc, rw, desc, B,
                                                                                    sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 candidates
// cand_out[0..C) = this rank's C smallest eligible keys (UINT64_MAX padded),
// cand_out[C] = its next arrival time (UINT64_MAX if none).
__global__ void __launch_bounds__(kSelThreads) candidates_kernel(const State st, const Sched sc, int32_t C,
                                                                  uint64_t *cand_out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor;
    advance_and_admit(st, sc, &s_now, &s_cursor);
    const int npow2 = next_pow2(sc.n > 0 ? sc.n : 1);
    build_keys(st, sc, s_cursor, s_buf, npow2);
    const bool two = npow2 >= 64 && npow2 <= kMergeCap;
    const uint64_t *keys = block_sort(s_buf, two ? s_buf + npow2 : nullptr, npow2);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const uint64_t key = c < npow2 ? keys[c] : ~0ull;
        cand_out[c] = (key >> 63) ? ~0ull : key;
    }
    if (threadIdx.x == 0) {
        cand_out[C] = s_cursor < sc.n ? (uint64_t)st.arrival[s_cursor] : ~0ull;
        st.g->now_us = s_now;
        st.g->cursor = s_cursor;
    }
}

cudaError_t launch_candidates(const State &st, const Sched &sc, int32_t C, uint64_t *cand_out,
                              cudaStream_t s) {
    static bool attr = false;
    if (!attr) { set_smem_attr((const void *)candidates_kernel); attr = true; }
    candidates_kernel<<<1, kSelThreads, sort_smem_bytes(sc.n > 0 ? sc.n : 1), s>>>(st, sc, C, cand_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 merge
// all_cand: world blocks of (C keys, 1 next-arrival word).  Global top-B by key;
// this rank keeps the ids with id % world == rank, in key order.
__global__ void __launch_bounds__(kSelThreads) merge_kernel(const State st, const Sched sc, const RowsDev rw,
                                                             SlotDesc *desc, const uint64_t *all_cand,
                                                             int32_t C, int32_t B, int32_t *sel_out,
                                                             int32_t *count_out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int s_tmp[64];
    __shared__ int s_gcount;
    __shared__ unsigned long long s_next;
    const int total = sc.world * C;
    const int npow2 = next_pow2(total > 0 ? total : 1);
    if (threadIdx.x == 0) { s_gcount = 0; s_next = ~0ull; }
    __syncthreads();
    for (int x = threadIdx.x; x < npow2; x += blockDim.x) {
        uint64_t key = ~0ull;
        if (x < total) key = all_cand[(int64_t)(x / C) * (C + 1) + (x % C)];
        s_buf[x] = key;
    }
    for (int g = threadIdx.x; g < sc.world; g += blockDim.x)
        atomicMin(&s_next, (unsigned long long)all_cand[(int64_t)g * (C + 1) + C]);
    __syncthreads();
    const bool two = npow2 >= 64 && npow2 <= kMergeCap;
    const uint64_t *keys = block_sort(s_buf, two ? s_buf + npow2 : nullptr, npow2);
    // global batch: first B valid keys; own = id % world == rank
    const int lim = B < npow2 ? B : npow2;
    const int per = (lim + (int)blockDim.x - 1) / (int)blockDim.x;
    const int lo = (int)threadIdx.x * per;
    int own = 0, valid = 0;
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = keys[x];
        if (key >> 63) continue;
        ++valid;
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        own += (int)(id % (uint32_t)sc.world) == sc.rank;
    }
    if (valid) atomicAdd(&s_gcount, valid);
    int n_own = 0;
    int pos = block_excl_scan(own, s_tmp, &n_own);
    const int64_t now = st.g->now_us;
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = keys[x];
        if (key >> 63) continue;
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        if ((int)(id % (uint32_t)sc.world) == sc.rank) {
            const int32_t i = (int32_t)(id / (uint32_t)sc.world);
            sel_out[pos] = i;
            commit_one(st, sc, i, now);
            if (rw.valid) desc[pos] = make_desc(rw, st, sc, pos, i);
            ++pos;
        }
    }
    for (int b = n_own + (int)threadIdx.x; b < B; b += blockDim.x) {
        sel_out[b] = -1;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, -1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int g = s_gcount;
        int64_t nnow = now;
        if (g == 0 && s_next != ~0ull && (int64_t)s_next > nnow) nnow = (int64_t)s_next;
        st.g->now_us = nnow;
        st.g->prev_count = g;
        st.g->count = n_own;
        if (count_out) *count_out = n_own;
    }
}

cudaError_t launch_merge(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc,
                         const uint64_t *all_cand, int32_t C, int32_t B, int32_t *sel_out,
                         int32_t *count_out, cudaStream_t s) {
    static bool attr = false;
    if (!attr) { set_smem_attr((const void *)merge_kernel); attr = true; }
    const int total = sc.world * C;
    merge_kernel<<<1, kSelThreads, sort_smem_bytes(total > 0 ? total : 1), s>>>(st, sc, rw, desc, all_cand, C,
                                                                                B, sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lapssd
