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
#include <cstdlib>

#include "select_core.cuh"

namespace lapssd {

#ifdef LAPSSD_TRACE
__device__ unsigned long long g_side_iter[128][2];
__device__ unsigned int g_side_n;
extern "C" int lapssd_side_trace_read(unsigned long long *out, unsigned *n) {
    cudaMemcpyFromSymbol(out, g_side_iter, sizeof g_side_iter);
    cudaMemcpyFromSymbol(n, g_side_n, sizeof(unsigned));
    unsigned z = 0;
    cudaMemcpyToSymbol(g_side_n, &z, sizeof z);
    return 0;
}
#ifdef LAPSSD_TRACE_SIDE   // per-iteration side-kernel events (perturbs the side kernel)
#define ITRACE(m) do { if (threadIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); \
    unsigned i = g_side_n++; if (i < 128) { g_side_iter[i][0] = t; g_side_iter[i][1] = (unsigned long long)(m); } } } while (0)
#else
#define ITRACE(m)
#endif
#define SSTEP(k) do { if (threadIdx.x == 0) g_sstep_t[vstep0 & 63][k] = gtimer(); } while (0)
__device__ unsigned long long g_siter[64][8][3];   // per step, first 8 merge passes: time, collected, merged
extern "C" int lapssd_siter_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_siter, sizeof g_siter);
    static unsigned long long zero[64][8][3];
    cudaMemcpyToSymbol(g_siter, zero, sizeof zero);
    return 0;
}
#define SITER(it, a, b) do { if (threadIdx.x == 0 && (it) < 8) { g_siter[vstep0 & 63][it][0] = gtimer(); \
    g_siter[vstep0 & 63][it][1] = (a); g_siter[vstep0 & 63][it][2] = (b); } } while (0)
__device__ unsigned long long g_sel_trace[16];
__device__ unsigned long long g_dbg_rec[16][4];
extern "C" int lapssd_dbg_rec_read(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_dbg_rec, sizeof g_dbg_rec); }
__device__ unsigned long long g_sstep_t[64][10];   // per committed step: side start, presort, merged, snap, end
extern "C" int lapssd_sstep_trace_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_sstep_t, sizeof g_sstep_t);
    static unsigned long long zero[64][10];
    cudaMemcpyToSymbol(g_sstep_t, zero, sizeof zero);
    return 0;
}
__device__ unsigned long long g_send[64];
__device__ unsigned int g_scount;
extern "C" int lapssd_send_read(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_send, sizeof g_send);
    unsigned z = 0; cudaMemcpyToSymbol(g_scount, &z, 4);
    return 0;
}
#define STRACE(i) do { if (threadIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_sel_trace[i] = t; } } while (0)
extern "C" int lapssd_sel_trace_read(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_sel_trace, sizeof g_sel_trace); }
#else
#define STRACE(i)
#define ITRACE(m)
#define SSTEP(k)
#define SITER(it, a, b)
#endif



int sort_capacity() { return kSortCap; }

static void set_smem_attr(const void *fn);
__global__ void select_kernel(const State, const Sched, const RowsDev, SlotDesc *, int32_t, int32_t *, int32_t *);

// ---------------------------------------------------------------- a3 standalone
__global__ void update_kernel(const State st, const Sched sc, const int32_t *sel,
                              const int32_t *n_accept, int32_t B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int32_t i = sel[b];
    if (i < 0) return;
    if (i >= sc.n) { atomicOr(&st.g->err, E_BAD_SLOT); return; }
    update_one(st, sc, i, n_accept[b], st.g->now_us + sc.c_round_us + st.g->step_sw);
}

cudaError_t launch_update(const State &st, const Sched &sc, const int32_t *sel,
                          const int32_t *n_accept, int32_t B, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    update_kernel<<<(B + 255) / 256, 256, 0, s>>>(st, sc, sel, n_accept, B);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a4-a7 select
__global__ void __launch_bounds__(kSelThreads) select_kernel(const State st, const Sched sc, const RowsDev rw,
                                                              SlotDesc *desc, int32_t B, int32_t *sel_out,
                                                              int32_t *count_out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int64_t s_now;
    __shared__ int s_cursor, s_count;
    __shared__ unsigned long long s_sw;
    advance_and_admit(st, sc, &s_now, &s_cursor);
    const int64_t now = s_now;
    const int cursor = s_cursor;
    const uint32_t seq = st.g->sel_seq;
    const int npow2 = next_pow2(sc.n > 0 ? sc.n : 1);
    build_keys(st, sc, cursor, s_buf, npow2);
    const int bp = next_pow2(B);
    const uint64_t *keys = select_topB_fast(s_buf, sc.n, B, s_buf + npow2, s_buf + npow2 + bp, bp, s_buf + npow2 + 2 * bp);
    // eligible keys (bit 63 clear) form a prefix of the sorted array
    const int lim = B < bp ? B : bp;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int valid = 0;
    for (int b = threadIdx.x; b < lim; b += blockDim.x) valid += (keys[b] >> 63) == 0;
    if (valid) atomicAdd(&s_count, valid);
    __syncthreads();
    const int cnt = s_count;
    int64_t sw = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t i = -1;
        if (b < cnt) {
            const uint32_t id = (uint32_t)(keys[b] & 0xFFFFFFull);
            i = (int32_t)(id / (uint32_t)sc.world);
            sw += commit_one(st, sc, i, now, seq);
        }
        sel_out[b] = i;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, i);    // a1 for the next verify
    }
    commit_switch(st, sc, sw, cnt, &s_sw);
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
__global__ void __launch_bounds__(kSelThreads) presort_kernel(const State st, const Sched sc, const RowsDev rw,
                                                               const int32_t *sel, int32_t B, PreSelect *out) {
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
    const uint64_t *top = select_topB_fast(s_buf, n, B, s_buf + npow2, s_buf + npow2 + bp, bp, s_buf + npow2 + 2 * bp);
    // records for the fused final select: flags, first-service marker, and the
    // acceptance-test descriptor of the candidate's current round (cached or computed)
    SelRec *rec = pre_recs(out, bp);
    for (int b = threadIdx.x; b < bp; b += blockDim.x) {
        const uint64_t key = top[b];
        out->cand[b] = key;
        SelRec r;
        r.key = key;
        r.flags = 0;
        r.x_unset = 0;
        r.desc.i = -1; r.desc.slab = 0; r.desc.req = 0; r.desc.round = 0; r.desc.r = -1;
        r.desc.trace = 0; r.desc.pad[0] = r.desc.pad[1] = 0;
        if (key != ~0ull) {
            const int32_t i = (int32_t)((uint32_t)(key & 0xFFFFFFull) / (uint32_t)sc.world);
            r.flags = st.flags[i];
            r.x_unset = st.x[i] < 0;
            if (rw.valid) r.desc = make_desc(rw, st, sc, 0, i);
        }
        rec[b] = r;
    }
    if (threadIdx.x == 0) {
        out->now_us = s_now;
        out->cursor = s_cursor;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&out->ready), "r"(1u) : "memory");
    }
}

__global__ void __launch_bounds__(kSelThreads) select_final_kernel(const State st, const Sched sc, const RowsDev rw,
                                                                    SlotDesc *desc, int32_t B, int32_t *sel,
                                                                    int32_t *count_out, const PreSelect *pre) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int s_count;
    __shared__ unsigned long long s_sw;
    STRACE(0);
    const int bp = next_pow2(B);
    const int64_t now = pre->now_us;
    const int cursor = pre->cursor;
    const uint32_t seq = st.g->sel_seq;
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
    uint64_t *cand = s_buf + 2 * bp;  // presorted candidates, staged in shared memory
    for (int b = threadIdx.x; b < bp; b += blockDim.x) cand[b] = pre->cand[b];
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    STRACE(1);
    const uint64_t *bk = block_sort(s_buf, bp >= 64 && bp <= kMergeCap ? s_buf + bp : nullptr, bp);
    STRACE(2);
    // merge path: first B outputs of merge(batch keys, presorted candidates)
    uint64_t *merged = (bk == s_buf) ? s_buf + bp : s_buf;
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
    STRACE(3);
    int valid = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) valid += (merged[b] >> 63) == 0;
    if (valid) atomicAdd(&s_count, valid);
    __syncthreads();
    const int cnt = s_count;
    STRACE(4);
    int64_t sw = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t i = -1;
        if (b < cnt) {
            const uint32_t id = (uint32_t)(merged[b] & 0xFFFFFFull);
            i = (int32_t)(id / (uint32_t)sc.world);
            sw += commit_one(st, sc, i, now, seq);
        }
        sel[b] = i;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, i);
    }
    commit_switch(st, sc, sw, cnt, &s_sw);
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
        const_cast<PreSelect *>(pre)->ready = 0;
    }
    __syncthreads();
    STRACE(5);
}

// Shared-memory words of the side select before the waiting-list regions: the larger of
// the phase-1 buffers (top-B, or the full sort that rebuilds the waiting list) and the
// phase-2 / commit buffers (4 lists of bp keys, slot / candidate maps, records).
__host__ __device__ inline size_t side_r0_words(int n, int bp) {
    int np = 1;
    while (np < (n > 0 ? n : 1)) np <<= 1;
    const size_t a = topB_smem_words(np, bp);
    const size_t a2 = (np >= 64 && np <= kMergeCap) ? 2 * (size_t)np : (size_t)np;
    const size_t b = 4 * (size_t)bp + (2 * (size_t)((n + 7) & ~7) * sizeof(int16_t) + 64 +
                                       (bp <= 1024 ? 2 * (size_t)bp * sizeof(SelRec) : 0) + 7) / 8;
    size_t r = a > a2 ? a : a2;
    r = r > b ? r : b;
    return (r + 1) & ~(size_t)1;
}
// admissions [kAdmCap], Kw [bp], S [bp + kAdmCap], rank histogram [bp + kAdmCap + 1] ints
__host__ __device__ inline size_t side_wl_words(int bp) {
    return 2 * (size_t)kAdmCap + 2 * (size_t)bp + ((size_t)bp + kAdmCap + 2) / 2;
}

// ---------------------------------------------------------------- incremental select
// One CTA on the side stream, concurrent with the verify kernel (which leaves it one
// SM).  Phase 1 = the presort above.  Phase 2: the verify finishers publish each
// batch slot as soon as its record (new key, flags, next descriptor) is written; this
// CTA repeatedly takes the newly published slots, sorts their keys and merges them into
// its sorted running list, keeping only the first B (an element ranked >= B can never
// re-enter the top B).  When every verified slot has arrived the list IS the next
// batch, and the commit (x_i, pinning, running flags, descriptors, clock) follows.
__global__ void __launch_bounds__(kSideThreads) select_side_kernel(const State st, const Sched sc, const RowsDev rw,
                                                                   int32_t *sel, SlotDesc *desc, int32_t B,
                                                                   PreSelect *pre, const SelRec *fin, uint64_t *fin_key,
                                                                   uint32_t *snap, uint32_t snap_target,
                                                                   int32_t *count_out, uint64_t *cand_out,
                                                                   int32_t C, const WaitList wl, const PeerArgs peer) {
    extern __shared__ uint64_t s_buf[];
    STRACE(8);
#ifdef LAPSSD_TRACE
    const uint32_t vstep0 = st.g->vstep;
    if (threadIdx.x == 0) {
        g_sstep_t[vstep0 & 63][0] = gtimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_sstep_t[vstep0 & 63][5] = smid;
    }
#endif
    __shared__ int64_t s_now;
    __shared__ int s_cursor, s_expected, s_merged, s_m, s_count;
    __shared__ uint32_t s_member[kSortCap / 32];
    __shared__ uint32_t s_pend[4096 / 32];    // expected slots not yet merged (B <= 4096 here)
    __shared__ int s_snap_ok;
    __shared__ unsigned long long s_sw_side;
    __shared__ int s_cursor0, s_na, s_wlen, s_rebuild, s_par, s_xw, s_xa, s_nkw;
    const int n = sc.n;
    const int T = blockDim.x;
    const int bp = next_pow2(B);
    const int npow2 = next_pow2(n > 0 ? n : 1);
    // the persistent waiting list (WaitList): its regions follow the phase-1/2 buffers
    const bool use_wl = wl.meta != nullptr;
    uint64_t *s_adm = s_buf + side_r0_words(n, bp);      // [kAdmCap] this step's admissions, sorted
    // (with no list these regions are not allocated and not touched)
    uint64_t *s_kw = s_adm + kAdmCap;                     // [bp] verified, not reselected: waiting keys
    uint64_t *s_S = s_kw + bp;                            // [bp + kAdmCap] merge(A suffix, Kw)
    int *s_hist = reinterpret_cast<int *>(s_S + bp + kAdmCap);   // [bp + kAdmCap + 1] rank histogram
    // peer exchange (laps_step_peer): the G candidate lists, after the waiting-list regions
    uint64_t *s_lists = s_buf + side_r0_words(n, bp) + (use_wl ? side_wl_words(bp) : 0);
    if (threadIdx.x == 0) s_cursor0 = st.g->cursor;
    // ---------------- phase 1: presort of every request outside the batch
    for (int w = threadIdx.x; w < (n + 31) / 32; w += T) s_member[w] = 0;
    for (int w = threadIdx.x; w < 4096 / 32; w += T) s_pend[w] = 0;
    if (threadIdx.x == 0) { s_expected = 0; s_merged = 0; s_m = 0; s_count = 0; s_snap_ok = snap == nullptr; }
    advance_and_admit(st, sc, &s_now, &s_cursor);   // ends with a barrier
    SSTEP(6);
    int expected = 0;
    for (int b = threadIdx.x; b < B; b += T) {
        const int i = sel[b];
        if (i >= 0) atomicOr(&s_member[i >> 5], 1u << (i & 31));
        const SlotDesc d = desc[b];
        if (d.r >= 0 && i >= 0 && d.i == i) {   // the slots the verify kernel updates and publishes
            ++expected;
            atomicOr(&s_pend[b >> 5], 1u << (b & 31));
        }
    }
    if (expected) atomicAdd(&s_expected, expected);
    __syncthreads();
    SSTEP(7);
    const int cursor = s_cursor;
    const uint64_t *top;
    // rebuild the waiting list from every request's state: no valid list, or a burst of
    // admissions larger than the admission buffer
    if (threadIdx.x == 0) {
        s_na = cursor - s_cursor0;
        s_rebuild = !use_wl || !wl.valid || s_na > kAdmCap;
        s_wlen = use_wl ? wl.meta[0] : 0;
        s_par = use_wl ? (wl.meta[1] & 1) : 0;
    }
    __syncthreads();
    if (s_rebuild) {
        // ---- every key of the requests outside the batch (the old presort)
        for (int i = threadIdx.x; i < npow2; i += T) {
            uint64_t key = ~0ull;
            if (i < n && !((s_member[i >> 5] >> (i & 31)) & 1u)) {
                const uint32_t fl = st.flags[i];
                const int32_t lp = st.L_pred[i], tok = st.acc_tok[i];
                const double A = st.A[i];
                const int32_t rnd = st.rounds[i];
                const uint64_t tag = st.next_tag[i];
                key = build_key(sc, i, cursor, fl, lp, tok, A);
                st.key[i] = key;
                if (key >> 63) key = ~0ull;   // ineligible: never selected
                // a1 of a waiting request's current round, memoised once (make_desc stores it):
                // the records below then never wait on row gathers under the verify stream
                else if (rw.valid && rw.slab_tab && tag != (((uint64_t)rw.epoch << 32) | (uint32_t)rnd))
                    (void)make_desc(rw, st, sc, 0, i);
            }
            s_buf[i] = key;
        }
        __syncthreads();
        SSTEP(8);
        if (use_wl) {
            // the whole list sorted: the waiting list (eligible keys form a prefix), written
            // to the current buffer; no admissions pending (they are in it)
            const uint64_t *srt = block_sort(s_buf, npow2 >= 64 && npow2 <= kMergeCap ? s_buf + npow2 : nullptr,
                                             npow2);
            int m = 0;
            for (int i = threadIdx.x; i < n; i += T) m += srt[i] != ~0ull;
            __shared__ int s_m_el;
            if (threadIdx.x == 0) s_m_el = 0;
            __syncthreads();
            if (m) atomicAdd(&s_m_el, m);
            __syncthreads();
            uint64_t *wl_cur = wl.keys[s_par];
            for (int i = threadIdx.x; i < s_m_el; i += T) wl_cur[i] = srt[i];
            if (threadIdx.x == 0) { s_wlen = s_m_el; s_na = 0; }
            // candidates: the first bp (padding beyond the list)
            uint64_t *cand = s_buf + (srt == s_buf ? npow2 : 0);
            if (npow2 < bp || npow2 > kMergeCap) cand = s_S;   // no second buffer: the S region
            __syncthreads();
            for (int b = threadIdx.x; b < bp; b += T) cand[b] = b < s_m_el ? srt[b] : ~0ull;
            __syncthreads();
            top = cand;
        } else {
            top = select_topB_fast(s_buf, n, B, s_buf + npow2, s_buf + npow2 + bp, bp, s_buf + npow2 + 2 * bp);
        }
    } else {
        // ---- persistent list: the keys that changed since the last commit are the
        // verified batch's (published in phase 2), the last commit's verified-but-not-
        // reselected requests (their key drops the running bit now: rewritten) and the
        // admissions; every other waiting key is unchanged (a waiting request's
        // state does not change)
        const int nf = wl.meta[2];
        for (int f = threadIdx.x; f < nf; f += T) st.key[wl.fresh_i[f]] = wl.fresh_key[f];
        const int na = s_na;
        const int nap = next_pow2(na > 0 ? na : 1);
        uint64_t *tmp = s_S;             // sort scratch (free until the commit)
        for (int x = threadIdx.x; x < nap; x += T) {
            uint64_t key = ~0ull;
            if (x < na) {
                const int i = s_cursor0 + x;
                key = build_key(sc, i, cursor, st.flags[i], st.L_pred[i], st.acc_tok[i], st.A[i]);
                st.key[i] = key;
                if (key >> 63) key = ~0ull;
            }
            s_adm[x] = key;
        }
        __syncthreads();
        if (na > 1) {
            const uint64_t *srt = block_sort(s_adm, nap >= 64 && nap <= kMergeCap ? tmp : nullptr, nap);
            if (srt != s_adm) {
                for (int x = threadIdx.x; x < nap; x += T) s_adm[x] = srt[x];
                __syncthreads();
            }
        }
        // candidates: the first bp of merge(waiting list, admissions)
        const uint64_t *W = wl.keys[s_par];
        const int wlen = s_wlen;
        uint64_t *cand = s_buf;
        uint64_t *wtop = s_buf + bp;
        for (int b = threadIdx.x; b < bp; b += T) wtop[b] = b < wlen ? __ldcg(W + b) : ~0ull;
        __syncthreads();
        for (int o = threadIdx.x; o < bp; o += T) {   // merge path over (wtop[bp], s_adm[na])
            int lo = o - na > 0 ? o - na : 0, hi = o < bp ? o : bp;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (wtop[mid] <= s_adm[o - 1 - mid]) lo = mid + 1; else hi = mid;
            }
            const int i = lo, j = o - lo;
            const bool takeA = j >= na || (i < bp && wtop[i] <= s_adm[j]);
            cand[o] = takeA ? wtop[i] : s_adm[j];
        }
        __syncthreads();
        top = cand;
    }
    SSTEP(9);
    SelRec *crec = pre_recs(pre, bp);
    for (int b = threadIdx.x; b < bp; b += T) {
        const uint64_t key = top[b];
        pre->cand[b] = key;
        SelRec r;
        r.key = key;
        r.flags = 0;
        r.x_unset = 0;
        r.desc.i = -1; r.desc.slab = 0; r.desc.req = 0; r.desc.round = 0; r.desc.r = -1;
        r.desc.trace = 0; r.desc.pad[0] = r.desc.pad[1] = 0;
        if (key != ~0ull) {
            const int32_t i = (int32_t)((uint32_t)(key & 0xFFFFFFull) / (uint32_t)sc.world);
            r.flags = st.flags[i];
            r.x_unset = st.x[i] < 0;
            if (rw.valid && rw.slab_tab) r.desc = make_desc(rw, st, sc, 0, i);
        }
        crec[b] = r;
    }
    __syncthreads();
    ITRACE(200000);
    SSTEP(1);
    // ---------------- phase 2: fold in the verified batch as it is published
    uint64_t *L = s_buf;                      // [bp] running top-B, sorted
    uint64_t *L2 = s_buf + bp;                // [bp]
    uint64_t *nk = s_buf + 2 * bp;            // [bp] newly published keys
    uint64_t *ntmp = s_buf + 3 * bp;          // [bp]
    int16_t *slot_of = reinterpret_cast<int16_t *>(s_buf + 4 * bp);   // [n]: batch slot, or -1
    int16_t *cand_of = slot_of + ((n + 7) & ~7);                       // [n]: candidate index, or -1
    // record copies in shared memory (bp <= 1024), so the commit needs no dependent loads
    SelRec *brec = reinterpret_cast<SelRec *>(cand_of + ((n + 7) & ~7));
    SelRec *srec = brec + bp;
    const bool rec_smem = bp <= 1024;
    constexpr int kTopReg = 4096 / kSideThreads;   // bp <= 4096 on this path
    uint64_t topv[kTopReg];   // L <- top (they may overlap: read all, barrier, write)
#pragma unroll
    for (int u = 0; u < kTopReg; ++u) {
        const int b = threadIdx.x + u * T;
        topv[u] = b < bp ? top[b] : ~0ull;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kTopReg; ++u) {
        const int b = threadIdx.x + u * T;
        if (b < bp) L[b] = topv[u];
    }
    if (rec_smem)
        for (int b = threadIdx.x; b < bp; b += T) srec[b] = crec[b];
    for (int i = threadIdx.x; i < n; i += T) { slot_of[i] = -1; cand_of[i] = -1; }
    __syncthreads();
    for (int b = threadIdx.x; b < bp; b += T) {
        const uint64_t key = L[b];
        if (key != ~0ull) cand_of[(uint32_t)(key & 0xFFFFFFull) / (uint32_t)sc.world] = (int16_t)b;
        if (b < B && sel[b] >= 0) slot_of[sel[b]] = (int16_t)b;
    }
    __syncthreads();
    const int need = s_expected;
    const unsigned long long t_start = gtimer();
    int iter = 0;
    for (;; ++iter) {
        __syncthreads();               // everyone has finished with s_m / s_merged
        if (s_merged >= need) break;
        if (waited_too_long(t_start)) {  // watchdog: never hang the GPU
            if (threadIdx.x == 0) atomicOr(&st.g->err, E_TIMEOUT | E_TO_MERGE);
            break;
        }
        // collect the slots published since the last pass: their keys (stored as ~key,
        // 0 = not yet; release-stored after the record) -- one round trip per pass
        for (int b = threadIdx.x; b < B; b += T) {
            if (!((s_pend[b >> 5] >> (b & 31)) & 1u)) continue;
            uint64_t v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(fin_key + b) : "memory");
            if (v == 0) continue;
            nk[atomicAdd(&s_m, 1)] = ~v;
            fin_key[b] = 0;   // consumed (the next step's verify starts after this kernel)
            atomicAnd(&s_pend[b >> 5], ~(1u << (b & 31)));
        }
        if (threadIdx.x == 0 && !s_snap_ok) {   // verify CTAs' snapshot, polled alongside
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(snap) : "memory");
            if (v >= snap_target) s_snap_ok = 1;
        }
        __syncthreads();
        const int m = s_m;
        SITER(iter, m, s_merged);
        if (m == 0 || (m < 32 && s_merged + m < need)) {   // merge in batches of >= 32, or the last ones
            __nanosleep(100);
            continue;
        }
        ITRACE(m);
        const int mp = next_pow2(m);
        for (int x = m + (int)threadIdx.x; x < mp; x += T) nk[x] = ~0ull;
        __syncthreads();
        ITRACE(300000 + m);
        const uint64_t *snk = block_sort(nk, mp >= 64 && mp <= kMergeCap ? ntmp : nullptr, mp);
        ITRACE(400000 + m);
        for (int o = threadIdx.x; o < bp; o += T) {   // first bp outputs of merge(L, snk)
            int lo = o - mp > 0 ? o - mp : 0, hi = o < bp ? o : bp;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (L[mid] <= snk[o - 1 - mid]) lo = mid + 1; else hi = mid;
            }
            const int i = lo, j = o - lo;
            const bool takeA = j >= mp || (i < bp && L[i] <= snk[j]);
            L2[o] = takeA ? L[i] : snk[j];
        }
        __syncthreads();
        for (int o = threadIdx.x; o < bp; o += T) L[o] = L2[o];
        __syncthreads();
        if (threadIdx.x == 0) { s_merged += m; s_m = 0; }
    }
    SSTEP(2);
    // every verify CTA has read what it needs of sel[] / desc[] (usually long ago): only
    // now may the commit overwrite them
    if (snap && threadIdx.x == 0) {
        const unsigned long long t0 = gtimer();
        while (!s_snap_ok) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(snap) : "memory");
            if (v >= snap_target) break;
            if (waited_too_long(t0)) { atomicOr(&st.g->err, E_TIMEOUT | E_TO_SNAP); break; }
            __nanosleep(64);
        }
        *snap = 0;
    }
    // the verified slots' records (their keys were merged above): one parallel round trip
    if (rec_smem)
        for (int b = threadIdx.x; b < B; b += T) brec[b] = fin[b];
    __syncthreads();
#ifdef LAPSSD_TRACE
    for (int b = threadIdx.x; b < B && b < 16; b += T) {
        g_dbg_rec[b][0] = brec[b].key;
        g_dbg_rec[b][1] = ((uint64_t)(uint32_t)brec[b].desc.i << 32) | (uint32_t)brec[b].desc.r;
        g_dbg_rec[b][2] = (uint64_t)(uint32_t)sel[b];
        g_dbg_rec[b][3] = L[b];
    }
#endif
    if (cand_out) {
        // multi-GPU (a8): this rank's C best keys (+ its next arrival) for the all-gather;
        // merge_kernel commits the global batch.  The verified batch's running flags are
        // cleared here, as candidates_kernel does after building its keys.
        const uint32_t seq = st.g->sel_seq;
        for (int c = threadIdx.x; c < C; c += T) {
            const uint64_t key = c < bp ? L[c] : ~0ull;
            const bool ok = (key >> 63) == 0;
            cand_out[c] = ok ? key : ~0ull;
            cand_out[C + c] = ok ? (uint64_t)switch_in_cost(st, sc, (int32_t)((uint32_t)(key & 0xFFFFFFull) /
                                                                              (uint32_t)sc.world), seq)
                                 : 0ull;
        }
        for (int b = threadIdx.x; b < B; b += T) {
            const int i = sel[b];
            if (i < 0) continue;
            st.flags[i] = (rec_smem ? brec[b].flags : fin[b].flags) & ~F_RUNNING;
        }
        if (threadIdx.x == 0) {
            cand_out[2 * C] = s_cursor < n ? (uint64_t)st.arrival[s_cursor] : ~0ull;
            st.g->now_us = s_now;
            st.g->cursor = s_cursor;
        }
        return;
    }
    ITRACE(100000);
    SSTEP(3);
    // ---------------- commit
    __shared__ int s_gcount;
    __shared__ unsigned long long s_gsw, s_gnext;
    if (peer.bufs) {
        // multi-GPU (a8) fused over peer memory (laps_step_peer): this rank's candidate
        // block -- its C best keys, their switch-in costs, its next arrival -- is stored
        // into slot `rank` of every rank's exchange buffer over NVLink (UVA peer pointers),
        // published by a system-scope release of the step's tag; then this CTA waits for
        // all G tags in its own buffer, ranks every key among the G sorted lists (its
        // index plus a binary search in each other list: the global top-B is a prefix of
        // each list) and commits THIS rank's prefix -- the same result as all-gather +
        // merge_kernel, in one kernel and without a collective launch.
        const int G = sc.world, Cp = peer.C, W2 = 2 * Cp + 2;
        const uint64_t tag = (uint64_t)st.g->vstep + 1;
        const int par = (int)(tag & 1);
        const uint32_t seq0 = st.g->sel_seq;
        for (int g = 0; g < G; ++g) {
            uint64_t *dst = peer.bufs[g] + ((size_t)par * G + sc.rank) * W2;
            for (int c = threadIdx.x; c < Cp; c += T) {
                const uint64_t key = c < bp ? L[c] : ~0ull;
                const bool ok = (key >> 63) == 0;
                dst[c] = ok ? key : ~0ull;
                dst[Cp + c] = ok ? (uint64_t)switch_in_cost(st, sc, (int32_t)((uint32_t)(key & 0xFFFFFFull) /
                                                                             (uint32_t)sc.world), seq0)
                                 : 0ull;
            }
            if (threadIdx.x == 0) dst[2 * Cp] = s_cursor < n ? (uint64_t)st.arrival[s_cursor] : ~0ull;
        }
        // the CTA barrier orders every thread's block stores before the release stores of
        // the tags (PTX release is cumulative over what happens-before it, barrier included)
        __syncthreads();
        if (threadIdx.x < G) {
            uint64_t *tg = peer.bufs[threadIdx.x] + ((size_t)par * G + sc.rank) * W2 + 2 * Cp + 1;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(tg), "l"(tag) : "memory");
        }
        if (threadIdx.x < G) {   // wait for every rank's block of this step (own buffer)
            const uint64_t *tg = peer.bufs[sc.rank] + ((size_t)par * G + threadIdx.x) * W2 + 2 * Cp + 1;
            const unsigned long long t0 = gtimer();
            for (;;) {
                uint64_t v;
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(tg) : "memory");
                if (v == tag) break;
                if (waited_too_long(t0)) { atomicOr(&st.g->err, E_TIMEOUT | E_TO_PEER); break; }
                __nanosleep(64);
            }
        }
        if (threadIdx.x == 0) { s_count = 0; s_gcount = 0; s_gsw = 0; s_gnext = ~0ull; }
        __syncthreads();
        const uint64_t *own = peer.bufs[sc.rank] + (size_t)par * G * W2;
        for (int x = threadIdx.x; x < G * Cp; x += T) s_lists[x] = __ldcg(own + (size_t)(x / Cp) * W2 + (x % Cp));
        for (int g = threadIdx.x; g < G; g += T)
            atomicMin(&s_gnext, (unsigned long long)__ldcg(own + (size_t)g * W2 + 2 * Cp));
        __syncthreads();
        int mine = 0, gsel = 0;
        unsigned long long gsw = 0;
        for (int x = threadIdx.x; x < G * Cp; x += T) {
            const int g = x / Cp, c = x % Cp;
            const uint64_t key = s_lists[x];
            if (key >> 63) continue;                       // padding (ineligible)
            int rk = c;
            for (int h = 0; h < G && rk < B; ++h) {
                if (h == g) continue;
                const uint64_t *Lh = s_lists + (size_t)h * Cp;
                int lo = 0, hi = Cp;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (Lh[mid] < key) lo = mid + 1; else hi = mid;
                }
                rk += lo;
            }
            if (rk >= B) continue;
            ++gsel;
            gsw += __ldcg(own + (size_t)g * W2 + Cp + c);
            mine += g == sc.rank;
        }
        if (mine) atomicAdd(&s_count, mine);
        if (gsel) atomicAdd(&s_gcount, gsel);
        if (gsw) atomicAdd(&s_gsw, gsw);
        __syncthreads();
    } else {
        int valid = 0;
        for (int b = threadIdx.x; b < B; b += T) valid += (L[b] >> 63) == 0;
        if (valid) atomicAdd(&s_count, valid);
        __syncthreads();
        if (threadIdx.x == 0) { s_gcount = s_count; s_gsw = 0; s_gnext = s_cursor < n ? (uint64_t)st.arrival[s_cursor] : ~0ull; }
        __syncthreads();
    }
    const int cnt = s_count;                 // this rank's selected: the first cnt of L
    const int gcount = s_gcount;             // the global batch
    ITRACE(100001);
    const int64_t now = s_now;
    const uint32_t seq = st.g->sel_seq;
    int64_t sw = 0;
    uint8_t *mark = reinterpret_cast<uint8_t *>(L2);     // [bp] 1 reselected, 2 +pin
    int32_t *old_i = reinterpret_cast<int32_t *>(nk);    // [bp] the verified batch
    for (int b = threadIdx.x; b < bp; b += T) { mark[b] = 0; old_i[b] = b < B ? sel[b] : -1; }
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += T) {
        SlotDesc d;
        d.i = -1; d.slab = 0; d.req = 0; d.round = 0; d.r = -1;
        d.trace = 0; d.pad[0] = d.pad[1] = 0;
        if (b < cnt) {
            const int i = (int)((uint32_t)(L[b] & 0xFFFFFFull) / (uint32_t)sc.world);
            const int sl = slot_of[i];
            const SelRec &rec = sl >= 0 ? (rec_smem ? brec[sl] : fin[sl])
                                        : (rec_smem ? srec[cand_of[i]] : crec[cand_of[i]]);
            d = rec.desc;
            if (!rw.slab_tab) d = make_desc(rw, st, sc, b, i);   // batch layout: slab = slot
            bool pin = false;
            if (sc.policy == LAPSSD_POL_FCFS || sc.policy == LAPSSD_POL_LPSJF) pin = true;
            else if (sc.policy == LAPSSD_POL_LAPSSD && sc.pin_rule == 0 && (rec.flags & F_PERC)) pin = true;
            if (sl >= 0) {
                mark[sl] = pin ? 2 : 1;
            } else {
                if (pin && !(rec.flags & F_PINNED)) st.flags[i] = rec.flags | F_PINNED;
                if (rec.x_unset) st.x[i] = now;      // x_i
            }
            const int64_t c = sl >= 0 ? 0 : switch_in_cost(st, sc, i, seq);   // the verified batch ran last
            charge_switch(st, sc, i, seq, c);
            sw += c;
        }
        sel[b] = d.i;
        desc[b] = d;
    }
    // the step lasts one round plus the switch-ins of the GLOBAL batch (AMB-24)
    commit_switch(st, sc, peer.bufs ? (threadIdx.x == 0 ? (int64_t)s_gsw : 0) : sw, gcount, &s_sw_side);
    __syncthreads();
    ITRACE(100002);
    for (int b = threadIdx.x; b < B; b += T) {   // the verified batch: running flags cleared
        const int i = old_i[b];
        if (i < 0) continue;
        uint32_t fl = (rec_smem ? brec[b].flags : fin[b].flags) & ~F_RUNNING;
        if (mark[b] == 2) fl |= F_PINNED;
        st.flags[i] = fl;
    }
    if (threadIdx.x == 0) {
        int64_t nnow = now;
        if (gcount == 0 && s_gnext != ~0ull && (int64_t)s_gnext > nnow) nnow = (int64_t)s_gnext;   // idle: jump
        st.g->now_us = nnow;
        st.g->cursor = s_cursor;
        st.g->prev_count = gcount;
        st.g->count = cnt;
        if (count_out) *count_out = cnt;
        st.g->vstep = st.g->vstep + 1;   // the next verify launch streams into the other set
    }
    // The next verify launch carries the programmatic-serialization attribute (it overlaps
    // the current one), and under stream capture that attribute makes every incoming
    // kernel->kernel edge programmatic -- including the one from this kernel.  So this
    // kernel triggers its dependents explicitly, and only once the commit (batch,
    // descriptors, clock, step counter, snapshot counter reset) is performed at GPU scope;
    // the verify kernel reads these with L2 (.cg) loads.
    __threadfence();
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    ITRACE(100003);
    STRACE(9);
    if (use_wl) {
        // ---- the next waiting list, off the critical path (only the next side select reads
        // it): W' = merge(W[x_W:], A[x_A:], Kw) where x_W / x_A are the selected prefixes
        // of the list and of the admissions (the top-B of a union of sorted lists takes a
        // prefix of each) and Kw the verified requests that were not reselected, with the
        // running bit dropped (AMB-16: it describes the round that just ran)
        if (threadIdx.x == 0) { s_xw = 0; s_xa = 0; s_nkw = 0; }
        __syncthreads();
        int xw = 0, xa = 0;
        for (int b = threadIdx.x; b < cnt; b += T) {
            const int i = (int)((uint32_t)(L[b] & 0xFFFFFFull) / (uint32_t)sc.world);
            if (slot_of[i] >= 0) continue;
            if (i >= s_cursor0 && i < s_cursor0 + s_na) ++xa; else ++xw;
        }
        if (xw) atomicAdd(&s_xw, xw);
        if (xa) atomicAdd(&s_xa, xa);
        const bool notrun_bit = sc.policy == LAPSSD_POL_LAS || sc.policy == LAPSSD_POL_LAPSSD;
        for (int b = threadIdx.x; b < B; b += T) {
            const int i = old_i[b];
            if (i < 0 || mark[b]) continue;
            const SelRec &rec = rec_smem ? brec[b] : fin[b];
            if (rec.key >> 63) continue;                            // completed
            const uint64_t key = rec.key | ((notrun_bit && (sc.policy == LAPSSD_POL_LAS || !(rec.flags & F_PERC)))
                                                ? (1ull << 56) : 0ull);
            s_kw[atomicAdd(&s_nkw, 1)] = key;
        }
        __syncthreads();
        const int nkw = s_nkw;
        for (int x = nkw + (int)threadIdx.x; x < bp; x += T) s_kw[x] = ~0ull;
        __syncthreads();
        const uint64_t *kw = block_sort(s_kw, bp >= 64 && bp <= kMergeCap ? ntmp : nullptr, bp);
        for (int f = threadIdx.x; f < nkw; f += T) {
            wl.fresh_key[f] = kw[f];
            wl.fresh_i[f] = (int32_t)((uint32_t)(kw[f] & 0xFFFFFFull) / (uint32_t)sc.world);
        }
        // S = merge(A[x_A:na), Kw[0:nkw))
        const int xa0 = s_xa, na = s_na, nA = na - xa0, nS = nA + nkw;
        const uint64_t *Aw = s_adm + xa0;
        for (int o = threadIdx.x; o < nS; o += T) {
            int lo = o - nkw > 0 ? o - nkw : 0, hi = o < nA ? o : nA;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (Aw[mid] <= kw[o - 1 - mid]) lo = mid + 1; else hi = mid;
            }
            const int i = lo, j = o - lo;
            const bool takeA = j >= nkw || (i < nA && Aw[i] <= kw[j]);
            s_S[o] = takeA ? Aw[i] : kw[j];
        }
        __syncthreads();
        // W' = merge(W[x_W:wlen), S) by ranks: W[j] goes to (j - x_W) + r_j with r_j = #{S < W[j]}
        // (a binary search in shared memory; coalesced loads and stores), and S[c] to
        // c + #{j : r_j <= c} (a histogram of the r_j and its prefix sum)
        const uint64_t *W = wl.keys[s_par];
        uint64_t *Wn = wl.keys[s_par ^ 1];
        const int x0 = s_xw, wlen = s_wlen, m = wlen - x0;
        for (int c = threadIdx.x; c <= nS; c += T) s_hist[c] = 0;
        __syncthreads();
        for (int j = x0 + (int)threadIdx.x; j < wlen; j += T) {
            const uint64_t w = __ldcg(W + j);
            int lo = 0, hi = nS;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (s_S[mid] < w) lo = mid + 1; else hi = mid;
            }
            Wn[(j - x0) + lo] = w;
            if (nS) atomicAdd(&s_hist[lo], 1);
        }
        __syncthreads();
        if (nS) {
            // inclusive prefix sum of s_hist[0..nS) (<= bp + kAdmCap entries), warp 0
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                int carry = 0;
                for (int c0 = 0; c0 < nS; c0 += 32) {
                    int v = c0 + lane < nS ? s_hist[c0 + lane] : 0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                        if (lane >= o) v += u;
                    }
                    if (c0 + lane < nS) s_hist[c0 + lane] = v + carry;
                    carry += __shfl_sync(0xFFFFFFFFu, v, 31);
                }
            }
            __syncthreads();
            for (int c = threadIdx.x; c < nS; c += T) Wn[c + s_hist[c]] = s_S[c];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            wl.meta[0] = m + nS;
            wl.meta[1] = s_par ^ 1;
            wl.meta[2] = nkw;
        }
    }
#ifdef LAPSSD_TRACE
    if (threadIdx.x == 0) g_sstep_t[vstep0 & 63][4] = gtimer();
    if (threadIdx.x == 0) { unsigned c = atomicAdd(&g_scount, 1u); if (c < 64) g_send[c] = gtimer(); }
#endif
}

cudaError_t launch_select_side(const State &st, const Sched &sc, const RowsDev &rw, int32_t *sel, SlotDesc *desc,
                               int32_t B, PreSelect *pre, const SelRec *fin, uint64_t *fin_key, uint32_t *snap,
                               uint32_t snap_target, int32_t *count_out, cudaStream_t s, uint64_t *cand_out,
                               int32_t C, const WaitList *wl, const PeerArgs *peer) {
    int bp = 1;
    while (bp < B) bp <<= 1;
    WaitList w{};
    if (wl && wl->meta && !cand_out && bp <= 1024) w = *wl;   // else: the per-step presort
    PeerArgs pa{};
    if (peer) pa = *peer;
    const size_t smem = (side_r0_words(sc.n, bp) + (w.meta ? side_wl_words(bp) : 0) +
                         (pa.bufs ? (size_t)sc.world * pa.C : 0)) * sizeof(uint64_t);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;   // shared memory of one CTA (sched_prepare)
    // highest launch priority: when an SM frees up, the block scheduler places this one
    // CTA before the waiting CTAs of the next (programmatically launched) verify grid
    static int prio = [] {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        return hi;
    }();
    static const bool no_prio = getenv("LAPSSD_SIDE_NO_PRIORITY") != nullptr;  // A/B switch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kSideThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    cfg.attrs = attr;
    cfg.numAttrs = no_prio ? 0 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, select_side_kernel, st, sc, rw, sel, desc, B, pre, fin, fin_key,
                                             snap, snap_target, count_out, cand_out, C, w, pa);
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_presort(const State &st, const Sched &sc, const RowsDev &rw, const int32_t *sel, int32_t B,
                           PreSelect *out, cudaStream_t s) {
    int np = 1, bp = 1;
    while (np < (sc.n > 0 ? sc.n : 1)) np <<= 1;
    while (bp < B) bp <<= 1;
    presort_kernel<<<1, kSelThreads, topB_smem_words(np, bp) * sizeof(uint64_t), s>>>(st, sc, rw, sel, B, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_final(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc, int32_t B,
                                int32_t *sel, int32_t *count_out, const PreSelect *pre, cudaStream_t s) {
    int bp = 1;
    while (bp < B) bp <<= 1;
    select_final_kernel<<<1, kSelThreads, (size_t)(3 * bp) * sizeof(uint64_t), s>>>(st, sc, rw, desc, B, sel,
                                                                                     count_out, pre);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc, int32_t B,
                          int32_t *sel_out, int32_t *count_out, cudaStream_t s) {
    int np = 1, bp = 1;
    while (np < (sc.n > 0 ? sc.n : 1)) np <<= 1;
    while (bp < B) bp <<= 1;
    select_kernel<<<1, kSelThreads, topB_smem_words(np, bp) * sizeof(uint64_t), s>>>(st, sc, rw, desc, B,
                                                                                    sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 candidates
// cand_out[0..C) = this rank's C smallest eligible keys (UINT64_MAX padded),
// cand_out[C..2C) = their switch-in costs if selected (AMB-24), cand_out[2C] = its next
// arrival time (UINT64_MAX if none).
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
    const uint32_t seq = st.g->sel_seq;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const uint64_t key = c < npow2 ? keys[c] : ~0ull;
        const bool ok = (key >> 63) == 0;
        cand_out[c] = ok ? key : ~0ull;
        cand_out[C + c] = ok ? (uint64_t)switch_in_cost(st, sc, (int32_t)((uint32_t)(key & 0xFFFFFFull) /
                                                                          (uint32_t)sc.world), seq)
                             : 0ull;
    }
    if (threadIdx.x == 0) {
        cand_out[2 * C] = s_cursor < sc.n ? (uint64_t)st.arrival[s_cursor] : ~0ull;
        st.g->now_us = s_now;
        st.g->cursor = s_cursor;
    }
}

cudaError_t launch_candidates(const State &st, const Sched &sc, int32_t C, uint64_t *cand_out,
                              cudaStream_t s) {
    candidates_kernel<<<1, kSelThreads, sort_smem_bytes(sc.n > 0 ? sc.n : 1), s>>>(st, sc, C, cand_out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a8 merge
// all_cand: world blocks of (C keys, C switch-in costs, 1 next-arrival word).  Global
// top-B by key; this rank keeps the ids with id % world == rank, in key order; the step
// lasts one round plus the switch-ins of the whole global batch (AMB-24).
__global__ void __launch_bounds__(kSelThreads) merge_kernel(const State st, const Sched sc, const RowsDev rw,
                                                             SlotDesc *desc, const uint64_t *all_cand,
                                                             int32_t C, int32_t B, int32_t *sel_out,
                                                             int32_t *count_out) {
    extern __shared__ uint64_t s_buf[];
    __shared__ int s_tmp[64];
    __shared__ int s_gcount;
    __shared__ unsigned long long s_next, s_sw;
    // Every rank's candidate list is sorted (candidates_kernel), so the global order is a
    // G-way merge: each key's global rank = its index in its own list + the number of
    // smaller keys in every other list (keys are unique: the global id is in the low
    // bits).  Each thread ranks a run of kRun consecutive keys of one list: one binary
    // search per other list for the first key, then a forward scan (the counts are
    // monotone along the run).  Keys ranked < B land at their rank in top[].
    const int G = sc.world;
    const int total = G * C;
    const int lim = B < total ? B : total;
    const int64_t blk = 2 * (int64_t)C + 1;   // words per rank
    uint64_t *lists = s_buf;            // [G*C]
    uint64_t *top = s_buf + total;      // [lim] the global top-B, ascending
    uint64_t *top_sw = top + lim;       // [lim] their switch-in costs
    if (threadIdx.x == 0) { s_gcount = 0; s_next = ~0ull; }
    __syncthreads();
    for (int x = threadIdx.x; x < total; x += blockDim.x)
        lists[x] = all_cand[(int64_t)(x / C) * blk + (x % C)];
    for (int x = threadIdx.x; x < lim; x += blockDim.x) { top[x] = ~0ull; top_sw[x] = 0; }
    for (int g = threadIdx.x; g < G; g += blockDim.x)
        atomicMin(&s_next, (unsigned long long)all_cand[(int64_t)g * blk + 2 * C]);
    __syncthreads();
    constexpr int kRun = 8;
    const int runs_per_list = (C + kRun - 1) / kRun;
    for (int u = threadIdx.x; u < G * runs_per_list; u += blockDim.x) {
        const int g = u / runs_per_list, c0 = (u % runs_per_list) * kRun;
        if (c0 >= lim) continue;                       // rank >= own index >= B
        const uint64_t *Lg = lists + (int64_t)g * C;
        if (Lg[c0] == ~0ull) continue;                 // padding (ineligible) from here on
        int rk[kRun];
#pragma unroll
        for (int e = 0; e < kRun; ++e) rk[e] = c0 + e;
        for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            const uint64_t *Lh = lists + (int64_t)h * C;
            int lo = 0, hi = C;                          // lower_bound of the run's first key
            const uint64_t x0 = Lg[c0];
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (Lh[mid] < x0) lo = mid + 1; else hi = mid;
            }
#pragma unroll
            for (int e = 0; e < kRun; ++e) {
                if (c0 + e >= C) break;
                const uint64_t x = Lg[c0 + e];
                while (lo < C && Lh[lo] < x) ++lo;
                rk[e] += lo;
            }
        }
#pragma unroll
        for (int e = 0; e < kRun; ++e) {
            if (c0 + e >= C) break;
            const uint64_t x = Lg[c0 + e];
            if (x != ~0ull && rk[e] < lim) {
                top[rk[e]] = x;
                top_sw[rk[e]] = all_cand[(int64_t)g * blk + C + c0 + e];
            }
        }
    }
    __syncthreads();
    const uint64_t *keys = top;
    // global batch: first B valid keys; own = id % world == rank
    const int per = (lim + (int)blockDim.x - 1) / (int)blockDim.x;
    const int lo = (int)threadIdx.x * per;
    int own = 0, valid = 0;
    int64_t sw = 0;   // switch-ins of the GLOBAL batch
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = keys[x];
        if (key >> 63) continue;
        ++valid;
        sw += (int64_t)top_sw[x];
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        own += (int)(id % (uint32_t)sc.world) == sc.rank;
    }
    if (valid) atomicAdd(&s_gcount, valid);
    int n_own = 0;
    int pos = block_excl_scan(own, s_tmp, &n_own);
    const int64_t now = st.g->now_us;
    const uint32_t seq = st.g->sel_seq;
    for (int x = lo; x < lo + per && x < lim; ++x) {
        const uint64_t key = keys[x];
        if (key >> 63) continue;
        const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
        if ((int)(id % (uint32_t)sc.world) == sc.rank) {
            const int32_t i = (int32_t)(id / (uint32_t)sc.world);
            sel_out[pos] = i;
            (void)commit_one(st, sc, i, now, seq);   // its cost is the candidate's, summed above
            if (rw.valid) desc[pos] = make_desc(rw, st, sc, pos, i);
            ++pos;
        }
    }
    for (int b = n_own + (int)threadIdx.x; b < B; b += blockDim.x) {
        sel_out[b] = -1;
        if (rw.valid) desc[b] = make_desc(rw, st, sc, b, -1);
    }
    __syncthreads();
    commit_switch(st, sc, sw, s_gcount, &s_sw);
    if (threadIdx.x == 0) {
        const int g = s_gcount;
        int64_t nnow = now;
        if (g == 0 && s_next != ~0ull && (int64_t)s_next > nnow) nnow = (int64_t)s_next;
        st.g->now_us = nnow;
        st.g->prev_count = g;
        st.g->count = n_own;
        if (count_out) *count_out = n_own;
        st.g->vstep = st.g->vstep + 1;   // overlapped laps_step_dist: the next verify's buffer set
    }
    // the next verify launch may be a programmatic dependent (see select_side_kernel)
    __threadfence();
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

cudaError_t launch_merge(const State &st, const Sched &sc, const RowsDev &rw, SlotDesc *desc,
                         const uint64_t *all_cand, int32_t C, int32_t B, int32_t *sel_out,
                         int32_t *count_out, cudaStream_t s) {
    const int total = sc.world * C;
    const size_t smem = ((size_t)total + 2 * (size_t)(B < total ? B : total)) * sizeof(uint64_t);
    merge_kernel<<<1, kSelThreads, smem > 0 ? smem : 8, s>>>(st, sc, rw, desc, all_cand, C,
                                                                                B, sel_out, count_out);
    count_launch();
    return cudaGetLastError();
}

// Kernel attributes are set once, at handle creation: cudaFuncSetAttribute may wait for
// the device to go idle, which must never happen while a verify and a side kernel that
// wait on each other are in flight.
void sched_prepare() {
    set_smem_attr((const void *)select_kernel);
    set_smem_attr((const void *)candidates_kernel);
    set_smem_attr((const void *)merge_kernel);
    set_smem_attr((const void *)presort_kernel);
    set_smem_attr((const void *)select_final_kernel);
    set_smem_attr((const void *)select_side_kernel);
    cudaFuncSetAttribute((const void *)select_side_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    (void)cudaGetLastError();   // an attribute error must not surface as a later launch error
}

}  // namespace lapssd
