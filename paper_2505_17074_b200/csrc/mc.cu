// mc.cu -- the Monte-Carlo replica engine (SURVEY §8(d) configs[4], §8(a) a6 segmented):
// T independent traces, each a batch-1 simulation of its own requests with its own
// clock (one request served at a time), advanced together one round per step.
//
// One step = the verify kernel over T slots (slot t = the request trace t runs, rows of
// its slab, Philox c3 = t) and mc_step_kernel: one warp per trace runs
//   (a3) the state update of the request just verified,
//   (a7) the trace clock (+c_round after a round, AMB-17; jump to the next arrival when
//        idle),
//   (a4) admission of the trace's arrivals up to its clock,
//   (a5, a6) every request's priority key and the trace's top-1 (warp min: P:129-133),
//        with x_i and pinning on selection (AMB-15, AMB-25),
//   (a1) the acceptance test of the selected request's round for the next verify.
// The per-trace result is exactly the single-trace handle's (and the oracle's) with
// B = 1; traces share nothing but the slab pool.
#include <cstdlib>

#include "select_core.cuh"

namespace lapssd {

#ifndef LAPSSD_MC_MINB   // resident 256-thread CTAs per SM the register budget is sized for
#define LAPSSD_MC_MINB 4
#endif
__global__ void __launch_bounds__(256, LAPSSD_MC_MINB) mc_step_kernel(const State st, const Sched sc, const McDev mc,
                                                      const RowsDev rw, const int32_t *n_accept, SlotDesc *desc,
                                                      int32_t *sel_out, int32_t *active) {
    const int lane = threadIdx.x & 31;
    const int t = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
    if (t >= mc.T) return;
    const int64_t off = mc.off[t];
    const int n = (int)(mc.off[t + 1] - off);
    Globals *g = mc.g + t;
    // (a3) the round this trace just verified
    if (n_accept && lane == 0) {
        // r of the round that ran is the descriptor's (a1 before the rows streamed; the
        // verify kernel only copies it to n_accept), so this kernel reads nothing the
        // verify kernel writes and may overlap its tail
        const SlotDesc d = desc[t];
        const int r = d.r;
        if (d.i >= 0 && r >= 0) update_one(st, sc, d.i, r, g->now_us + sc.c_round_us + g->step_sw);
    }
    __syncwarp();
    // (a7 + a4) clock and admission over the trace's sorted arrivals
    int64_t now = g->now_us;
    if (g->prev_count > 0) now += sc.c_round_us + g->step_sw;   // AMB-17, AMB-24
    int cursor = g->cursor;
    const int cursor0 = cursor;
    for (;;) {
        const int j = cursor + lane;
        const bool adm = j < n && st.arrival[off + j] <= now;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, adm);
        cursor += __popc(m);
        if (m != 0xFFFFFFFFu) break;
    }
    // (a5 + a6) keys (local ids: the trace is its own id space) and the top-1.  Batch 1
    // changes few keys per step: the request just verified (its update), the one that
    // ran before it (its running flag is cleared) and the new admissions; every other
    // key is unchanged (flags, level, estimate and pin move only for the running
    // request).  So after the first select only those are recomputed, then the warp
    // takes the minimum of the trace's stored keys (4 KB for 512 requests).
    auto rekey = [&](int64_t i) {
        const uint32_t fl = st.flags[i];
        const uint64_t key = build_key(sc, (int32_t)(i - off), cursor, fl, st.L_pred[i], st.acc_tok[i], st.A[i]);
        st.key[i] = key;
        if (fl & F_RUNNING) st.flags[i] = fl & ~F_RUNNING;   // they describe the round that ran
        return key;
    };
    uint64_t best = ~0ull;
    if (!n_accept) {                                         // first select: every key
        for (int j = lane; j < n; j += 32) {
            const uint64_t key = rekey(off + j);
            best = key < best ? key : best;
        }
    } else {
        const int32_t ran = desc[t].i, before = mc.last[t];
        if (lane == 0 && ran >= 0) rekey(ran);
        if (lane == 1 && before >= 0 && before != ran) rekey(before);
        for (int j = cursor0 + lane; j < cursor; j += 32) rekey(off + j);   // admitted now
        __syncwarp();
        if (lane == 0) mc.last[t] = ran;
        constexpr int U = 4;                                 // independent loads in flight
        for (int j0 = 0; j0 < n; j0 += 32 * U) {
            uint64_t kv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * 32 + lane;
                kv[u] = j < n ? st.key[off + j] : ~0ull;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) best = kv[u] < best ? kv[u] : best;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        best = v < best ? v : best;
    }
    const bool have = (best >> 63) == 0;
    const int jsel = have ? (int)(best & 0xFFFFFFull) : -1;
    if (lane == 0) {
        SlotDesc d;
        d.i = -1; d.slab = 0; d.req = 0; d.round = 0; d.r = -1;
        d.trace = (uint32_t)t; d.pad[0] = d.pad[1] = 0;
        int64_t nnow = now;
        const uint32_t seq = g->sel_seq;
        int64_t sw = 0;
        if (have) {
            const int64_t i = off + jsel;
            sw = commit_one(st, sc, (int32_t)i, now, seq);   // switch-in unless it just ran (AMB-24)
            // (a1) for the next verify: x_j ~ q_j of the slab of this round, Philox c3 = t
            const int32_t rnd = st.rounds[i];
            const int64_t slab = rw.slab_tab[i * rw.R + slab_round_index(rnd, rw.R)];
            d.i = (int32_t)i;
            d.slab = (int32_t)slab;
            d.req = (uint32_t)jsel;
            d.round = (uint32_t)rnd;
            d.r = rw.dtype == LAPSSD_BF16 ? accept_test(rw, slab, d.req, d.round, (uint32_t)t, sc.seed, load_prob_bf16)
                                          : accept_test(rw, slab, d.req, d.round, (uint32_t)t, sc.seed, load_prob_f32);
            if (active) atomicAdd(active, 1);
        } else if (cursor < n) {                                 // idle: jump to the next arrival
            const int64_t nxt = st.arrival[off + cursor];
            if (nxt > nnow) nnow = nxt;
        }
        desc[t] = d;
        if (sel_out) sel_out[t] = jsel;
        g->now_us = nnow;
        g->cursor = cursor;
        g->prev_count = have ? 1 : 0;
        g->count = have ? 1 : 0;
        g->step_sw = sw;
        g->switch_total += sw;
        g->sel_seq = seq + 1;
    }
    // this grid is a programmatic dependent of the last verify sub-launch: it completes
    // only after that grid has (so whatever follows it on the stream -- the next step's
    // verify, a read of n_accept -- is ordered after the verify's writes)
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

cudaError_t launch_mc_step(const State &st, const Sched &sc, const McDev &mc, const RowsDev &rw,
                           const int32_t *n_accept, SlotDesc *desc, int32_t *sel_out, int32_t *active,
                           cudaStream_t s) {
    if (mc.T <= 0) return cudaSuccess;
    const int warps_per_block = 8;
    const int blocks = (mc.T + warps_per_block - 1) / warps_per_block;
    // a programmatic dependent of the last verify sub-launch: its warps start on SMs as
    // that grid's CTAs retire (the verify CTAs trigger after snapshotting desc[])
    static const bool no_pdl = getenv("LAPSSD_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(32 * warps_per_block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (no_pdl || !n_accept) ? 0 : 1;   // only right after laps_mc_step's verify
    const cudaError_t e = cudaLaunchKernelEx(&cfg, mc_step_kernel, st, sc, mc, rw, n_accept, desc, sel_out, active);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace lapssd
