// sched.cu -- LAPS-SD scheduler kernels on sm_100a: state update (a3), admission +
// priority keys + top-B selection + clock (a4-a7), and the multi-GPU candidate /
// merge halves of the global top-B (a8).  PAPER.md P:84-93.
//
// Selection runs in ONE CTA of 1024 threads: every resident request's 64-bit key is
// built in registers from the SoA state, the keys are bitonic-sorted in shared memory
// (<= 16384 keys = 128 KiB), and the first B eligible ones become the batch.  With N
// in the low thousands per GPU this is a few microseconds, independent of V.
#include "lapssd_internal.cuh"

namespace lapssd {

constexpr int kSelThreads = 1024;
constexpr int kSortCap = 16384;

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

// ---------------------------------------------------------------- block helpers
__device__ void bitonic_sort(uint64_t *s, int n) {  // n power of two, ascending
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

__device__ __forceinline__ int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

// Block-wide exclusive scan of one int per thread (kSelThreads threads).
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

// Build every key, store them (global + shared, padded to npow2 with UINT64_MAX),
// clear the running flags (they describe the round that just ran).
__device__ void build_keys(const State &st, const Sched &sc, int cursor, uint64_t *s_keys, int npow2) {
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < sc.n) {
            const uint32_t fl = st.flags[i];
            key = build_key(st, sc, i, cursor, fl);
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
__global__ void __launch_bounds__(kSelThreads) select_kernel(const State st, const Sched sc, int32_t B,
                                                              int32_t *sel_out, int32_t *count_out) {
    extern __shared__ uint64_t s_keys[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor, s_count;
    advance_and_admit(st, sc, &s_now, &s_cursor);
    const int64_t now = s_now;
    const int cursor = s_cursor;
    const int npow2 = next_pow2(sc.n > 0 ? sc.n : 1);
    build_keys(st, sc, cursor, s_keys, npow2);
    bitonic_sort(s_keys, npow2);
    // eligible keys (bit 63 clear) form a prefix of the sorted array
    const int lim = B < npow2 ? B : npow2;
    int valid = 0;
    for (int b = threadIdx.x; b < lim; b += blockDim.x) valid += (s_keys[b] >> 63) == 0;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    if (valid) atomicAdd(&s_count, valid);
    __syncthreads();
    const int cnt = s_count;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t i = -1;
        if (b < cnt) {
            const uint32_t id = (uint32_t)(s_keys[b] & 0xFFFFFFull);
            i = (int32_t)(id / (uint32_t)sc.world);
            commit_one(st, sc, i, now);
        }
        sel_out[b] = i;
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

cudaError_t launch_select(const State &st, const Sched &sc, int32_t B, int32_t *sel_out,
                          int32_t *count_out, cudaStream_t s) {
    int npow2 = 1;
    while (npow2 < (sc.n > 0 ? sc.n : 1)) npow2 <<= 1;
    const size_t smem = (size_t)npow2 * sizeof(uint64_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSortCap * (int)sizeof(uint64_t));
        attr = true;
    }
    select_kernel<<<1, kSelThreads, smem, s>>>(st, sc, B, sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 candidates
// cand_out[0..C) = this rank's C smallest eligible keys (UINT64_MAX padded),
// cand_out[C] = its next arrival time (UINT64_MAX if none).
__global__ void __launch_bounds__(kSelThreads) candidates_kernel(const State st, const Sched sc, int32_t C,
                                                                  uint64_t *cand_out) {
    extern __shared__ uint64_t s_keys[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor;
    advance_and_admit(st, sc, &s_now, &s_cursor);
    const int npow2 = next_pow2(sc.n > 0 ? sc.n : 1);
    build_keys(st, sc, s_cursor, s_keys, npow2);
    bitonic_sort(s_keys, npow2);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const uint64_t key = c < npow2 ? s_keys[c] : ~0ull;
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
    int npow2 = 1;
    while (npow2 < (sc.n > 0 ? sc.n : 1)) npow2 <<= 1;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(candidates_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSortCap * (int)sizeof(uint64_t));
        attr = true;
    }
    candidates_kernel<<<1, kSelThreads, (size_t)npow2 * sizeof(uint64_t), s>>>(st, sc, C, cand_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 merge
// all_cand: world blocks of (C keys, 1 next-arrival word).  Global top-B by key;
// this rank keeps the ids with id % world == rank, in key order.
__global__ void __launch_bounds__(kSelThreads) merge_kernel(const State st, const Sched sc,
                                                             const uint64_t *all_cand, int32_t C, int32_t B,
                                                             int32_t *sel_out, int32_t *count_out) {
    extern __shared__ uint64_t s_keys[];
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
        s_keys[x] = key;
    }
    for (int g = threadIdx.x; g < sc.world; g += blockDim.x)
        atomicMin(&s_next, (unsigned long long)all_cand[(int64_t)g * (C + 1) + C]);
    __syncthreads();
    bitonic_sort(s_keys, npow2);
    // global batch: first B valid keys; own = id % world == rank
    const int lim = B < npow2 ? B : npow2;
    const int per = (lim + (int)blockDim.x - 1) / (int)blockDim.x;
    const int lo = (int)threadIdx.x * per;
    int own = 0, valid = 0;
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = s_keys[x];
        if (key >> 63) continue;
        ++valid;
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        own += (int)(id % (uint32_t)sc.world) == sc.rank;
    }
    if (valid) atomicAdd(&s_gcount, valid);
    int n_own = 0;
    const int pos0 = block_excl_scan(own, s_tmp, &n_own);
    int pos = pos0;
    const int64_t now = st.g->now_us;
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = s_keys[x];
        if (key >> 63) continue;
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        if ((int)(id % (uint32_t)sc.world) == sc.rank) {
            const int32_t i = (int32_t)(id / (uint32_t)sc.world);
            sel_out[pos++] = i;
            commit_one(st, sc, i, now);
        }
    }
    for (int b = n_own + (int)threadIdx.x; b < B; b += blockDim.x) sel_out[b] = -1;
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

cudaError_t launch_merge(const State &st, const Sched &sc, const uint64_t *all_cand, int32_t C,
                         int32_t B, int32_t *sel_out, int32_t *count_out, cudaStream_t s) {
    int npow2 = 1;
    const int total = sc.world * C;
    while (npow2 < (total > 0 ? total : 1)) npow2 <<= 1;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSortCap * (int)sizeof(uint64_t));
        attr = true;
    }
    merge_kernel<<<1, kSelThreads, (size_t)npow2 * sizeof(uint64_t), s>>>(st, sc, all_cand, C, B,
                                                                           sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lapssd
