// kernels_fused.cuh — one pass per round: apply(t-1) fused with quantize(t).
//
// In the step pipeline both halves read the round's gradient g_t: the apply of
// round t-1 needs it for the local update loc_{t+1} = W_t - eta_l * g_t
// (engine.py:385-392) and quantize(t) folds it into the residual
// (codec.py:181-193). One kernel reads g_t once:
//
//   reads  g_t 4 | r 8 | W 4 | codes(t-1) N/4  (APPLY_Q)  or  gsum(t-1) 4 (APPLY_F)
//   writes r' 8 | codes(t) 1/4 | W 4 | loc 4
//   = 32 + (N+1)/4 B/elem (APPLY_Q) vs 36.5 + N/4 for K1 + K2 separately.
//
// With the fused P2P exchange the kernel both waits for the peers' codes of round t-1
// and for the release of the slot round t writes into, and its last CTA publishes
// ready(t) and freed(t-1). (A TMA-ring variant of this kernel was measured ~3 %
// slower at ResNet-50 size and removed.)
#pragma once
#include "kernels.cuh"

namespace cdsgd {

enum { APPLY_Q = 0, APPLY_F = 1, APPLY_L = 2 };  // L: loc = W - eta_l*g only (W already final)

struct FusedArgs {
    // quantize(t)
    const float* g;
    const void* r_in;  // double* (exact) or float* (fp32-residual fast mode): the kernel's TR
    void* r_out;
    uint32_t* words;   // local packed output when not exchanging
    double alpha;
    uint64_t tag;
    // apply(t-1)
    void* W;  // float* or double* (the kernel's TW)
    float* loc;
    const uint32_t* gathered;  // APPLY_Q: codes of all ranks, rank stride `stride`
    int64_t stride;
    const float* gsum;         // APPLY_F
    float scale;               // APPLY_F: (float)(eta_g / N)
    double inv_n;
    float eta_l;
    // APPLY_Q decode: exact = every partial sum j*alpha (|j| <= N) representable, so the
    // SWAR count + table is bitwise the ascending fp64 sum; otherwise (e.g. alpha = 0.3 at
    // N >= 3) the tile takes the per-element path with the sequential sum of
    // engine.py:250-255 (inv_n_or_zero = 1/N for power-of-two N, else 0: divide).
    int exact;
    double eta_g_d, inv_n_or_zero, eta_l_d;
    int nranks;
    uint64_t skip_below;
    double* gnorm;
    uint64_t* err;
    P2PArgs xq;  // exchange of round t's codes (wait: slot freed; publish: ready)
    P2PArgs xa;  // exchange of round t-1's codes (wait: ready; publish: freed)
    unsigned int* sched;  // [2] dynamic tile scheduler {next tile, CTAs done}; nullptr = static ranges
    double* gclear[2];    // grad-norm ring slots to zero (see pdl_enter), nullable
};


// The pointers a task's loads and stores need (and the p2p-wait test), held in registers from
// BEFORE the grid-dependency wait: read from the kernel parameters after it, they were
// dependent constant-bank loads on every warp's path to its first load (the p2p test alone:
// 258 -> 57 cycles per warp once precomputed, ResNet-20-sized layouts).
struct HotPtrs {
    const float* g;
    const void* r_in;
    void* r_out;
    void* W;
    float* loc;
    const uint32_t* gathered;
    const uint64_t* err;
    double* sink;
    int p2p_wait;  // the launch waits on peer flags (p2p_wait2's test, known before the wait)
    __device__ __forceinline__ explicit HotPtrs(const FusedArgs& a)
        : g(a.g), r_in(a.r_in), r_out(a.r_out), W(a.W), loc(a.loc), gathered(a.gathered), err(a.err), sink(g_sink),
          p2p_wait(p2p_has_wait(a.xq) || p2p_has_wait(a.xa) ? 1 : 0) {}
    // opaque from here on: the compiler can no longer re-read them from the parameter bank
    __device__ __forceinline__ void pin_here() {
        asm volatile("" : "+l"(g), "+l"(r_in), "+l"(r_out), "+l"(W), "+l"(loc), "+l"(gathered), "+l"(err), "+l"(sink),
                     "+r"(p2p_wait));
    }
};

// Development probe (-DCDSGD_PROBE_TIMING builds only, loaded through CDSGD_LIB): per-warp
// clock64 stamps of the launch's phases, read back by cdsgd_diag_probe (scripts/small_probe.py).
#ifdef CDSGD_PROBE_TIMING
constexpr int PROBE_WARPS = 8192, PROBE_PTS = 16;
__device__ unsigned long long g_probe[PROBE_WARPS * PROBE_PTS];
// stamps go to shared memory (no global address to rematerialise from the constant bank at
// every stamp, which inflated the phases it measured) and are copied out at the kernel's end
__shared__ unsigned long long s_probe[8 * PROBE_PTS];
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// a real instruction consuming v: the warp waits for v's load here (scoreboard), so the next
// stamp measures arrival
__device__ __forceinline__ void probe_touch(uint32_t v) {
    __shared__ volatile uint32_t s_sink;
    if (v == 0x7fc0beefu) s_sink = v;  // a branch on v: cannot be dropped or run ahead of the load
}
#define CDSGD_PROBE(i)                                                                          \
    do {                                                                                        \
        if ((threadIdx.x & 31) == 0)                                                            \
            s_probe[(threadIdx.x >> 5) * PROBE_PTS + (i)] = (i) == 0 || (i) == 7 ? globaltimer_ns() : clock64(); \
    } while (0)
__device__ __forceinline__ void probe_flush() {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if ((threadIdx.x & 31) == 0 && w < PROBE_WARPS && (threadIdx.x >> 5) < 8)
        for (int i = 0; i < PROBE_PTS; ++i) g_probe[w * PROBE_PTS + i] = s_probe[(threadIdx.x >> 5) * PROBE_PTS + i];
}
#else
#define CDSGD_PROBE(i) do {} while (0)
#endif


// Round gating from the device error word and the peers' poison flags: an error of an
// EARLIER round (smaller tag) stops the quantize and the apply below skip_below (sticky
// abort); an error found by this launch never suppresses its own scan (the reported index
// stays the first non-finite element, codec.py:182-185). Read lazily — after a warp's first
// loads are in flight — so the error word costs no round trip of its own on launch-bound
// layouts (an error of this launch is >= tag and >= skip_below, so reading it late is the
// same test).
struct RoundFlags {
    bool have = false, issued = false, peer_failed = false, q_off = false, a_off = false;
    uint64_t e0v = ~0ull;
    // Issue the error word's load (once per warp). Every warp of the launch reads the same
    // word, and an SM's responses come back roughly in issue order: issued AFTER a task's
    // data loads it arrived ~1,000 cycles after them on ResNet-20-sized layouts; issued
    // before them it is back by the time they are. A weak load suffices: the words the
    // previous rounds' kernels wrote are visible after the grid-dependency wait, and this
    // launch's own error records never change the test (see above).
    __device__ __forceinline__ void issue(const uint64_t* err) {
        if (issued) return;
        if (err != nullptr) asm volatile("ld.global.u64 %0, [%1];" : "=l"(e0v) : "l"(err) : "memory");
        issued = true;
    }
    __device__ __forceinline__ void resolve(const FusedArgs& a, const uint64_t* err) {
        if (have) return;
        issue(err);
        q_off = e0v < a.tag || peer_failed;
        a_off = e0v < a.skip_below || peer_failed;
        have = true;
    }
};

// One task of the vector path: CH chunks of 128 elements (from chunk c0) of the tile at
// element e0 / word w0, all loads issued before any use. A key's last tile (ne < TILE_ELEMS
// elements) uses masked accesses; padding quantizes to code 00 (the
// reference's zero padding of the last word, codec.py:131-143) and is never stored.
// WHOLE: a whole tile (ne == TILE_ELEMS), every access unmasked — the compiler drops the
// masked-access branches and their registers (CDSGD_FULL_SPEC=0 disables the split).
#ifndef CDSGD_FULL_SPEC
#define CDSGD_FULL_SPEC 1
#endif
// A task's loaded operands (registers)
template <int NR, int APPLY, int CH, typename TW, typename TR>
struct TaskRegs {
    float4 gv[CH], sv[CH];
    WV<TW> wv[CH];
    WV<TR> rv[CH];
    uint32_t cw[APPLY == APPLY_Q ? NR : 1];
};
// Issue every load of a task (error word first on small layouts, see RoundFlags::issue).
template <int NR, int APPLY, int CH, typename TW, bool WHOLE, typename TR>
__device__ __forceinline__ void fused_vec_load(const FusedArgs& a, const HotPtrs& h, int lane, int64_t e0, int64_t w0,
                                               int ne, int nw, int c0, RoundFlags& fl,
                                               TaskRegs<NR, APPLY, CH, TW, TR>& L) {
    if constexpr (CH == 1) fl.issue(h.err);
    if constexpr (APPLY == APPLY_Q) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
            L.cw[r] = lane < nw ? ld_word(h.gathered + r * a.stride + w0 + lane) : 0u;
    }
    CDSGD_PROBE(15);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int64_t e = e0 + 128 * (c0 + c) + 4 * lane;
        const int nv = WHOLE ? 4 : nvalid4(ne, 128 * (c0 + c) + 4 * lane);
        L.gv[c] = ld_stream_m(h.g + e, nv);
        ldw4(static_cast<const TR*>(h.r_in) + e, nv, L.rv[c]);
        ldw4(static_cast<const TW*>(h.W) + e, nv, L.wv[c]);
        if constexpr (APPLY == APPLY_F) L.sv[c] = ld_stream_m(a.gsum + e, nv);
    }
}

template <int NR, int APPLY, int CH, typename TW, bool WHOLE, typename TR>
__device__ __forceinline__ uint32_t fused_vec_task(const FusedArgs& a, const HotPtrs& h, const float* s_upd, const double* s_upd64,
                                                   int lane, int64_t e0, int64_t w0, int ne, int nw, int c0,
                                                   RoundFlags& fl, uint32_t ahi, uint32_t alo,
                                                   uint64_t& bad_idx, uint64_t& bad_sym, double& gsq, int& isq,
                                                   TaskRegs<NR, APPLY, CH, TW, TR>& L, bool loaded) {
    uint32_t myword = 0;
    TW* const W = static_cast<TW*>(h.W);
    TR* const r_out = static_cast<TR*>(h.r_out);
    if (CH != 1 || !loaded) fused_vec_load<NR, APPLY, CH, TW, WHOLE, TR>(a, h, lane, e0, w0, ne, nw, c0, fl, L);
    float4(&gv)[CH] = L.gv;
    float4(&sv)[CH] = L.sv;
    WV<TW>(&wv)[CH] = L.wv;
    WV<TR>(&rv)[CH] = L.rv;
    uint32_t(&cw)[APPLY == APPLY_Q ? NR : 1] = L.cw;
#ifdef CDSGD_PROBE_TIMING
    CDSGD_PROBE(12);
    probe_touch(__float_as_uint(gv[0].x));
    CDSGD_PROBE(8);
    probe_touch(static_cast<uint32_t>(__double_as_longlong(static_cast<double>(rv[0].v[0]))));
    probe_touch(static_cast<uint32_t>(__double_as_longlong(static_cast<double>(wv[0].v[0]))));
    if constexpr (APPLY == APPLY_Q) probe_touch(cw[0]);
    CDSGD_PROBE(9);
#endif
    if constexpr (CH == 1) fl.resolve(a, h.err);  // small layouts: the error word's read overlaps the loads above
    const bool a_off = fl.a_off, q_off = fl.q_off;
#ifdef CDSGD_PROBE_TIMING
    probe_touch(q_off ? 1u : 0u);
    CDSGD_PROBE(10);
#endif
    // Small layouts (CH == 1) compute unconditionally and send an aborted round's stores to a
    // sink: with `if (!a_off)` around the apply, ptxas sank the W load into that branch, i.e.
    // behind the error word's round trip (two dependent trips per task instead of one).
    constexpr bool SINK = CH == 1;
    const int a_on = a_off ? 0 : 1;
    // many ranks (N > 5): each lane sums the counts of ITS word over the ranks once (the words
    // of a chunk are read by 4 lanes each), then a chunk shuffles 5 counters instead of N words.
    // Fewer ranks shuffle the words: at N = 2 / 4 the 5 shuffles measured slower in the engine
    // (F 200 vs 186 us at N = 2) although the standalone kernel gained.
    Counts wc{0u, 0u, 0u, 0u, 0u};
    if constexpr (APPLY == APPLY_Q && NR > 5) {
#pragma unroll
        for (int r = 0; r < NR; ++r) count_add(wc, cw[r]);
    }
    uint32_t v[CH];
    bool bad = false;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int64_t e = e0 + 128 * (c0 + c) + 4 * lane;
        const int nv = WHOLE ? 4 : nvalid4(ne, 128 * (c0 + c) + 4 * lane);
        float g4[4] = {gv[c].x, gv[c].y, gv[c].z, gv[c].w};
        WV<TW>& w4 = wv[c];
        const TR(&r4)[4] = rv[c].v;
        if (SINK || !a_off) {
            float l4[4];
            if constexpr (APPLY == APPLY_Q) {
                Counts cnt{0u, 0u, 0u, 0u, 0u};
                if constexpr (NR > 5) {
                    cnt = shfl_counts(wc, 8 * (c0 + c) + (lane >> 2));
                } else {
#pragma unroll
                    for (int r = 0; r < NR; ++r) count_add(cnt, __shfl_sync(FULL, cw[r], 8 * (c0 + c) + (lane >> 2)));
                }
                int cq[4];
                lane_counts(cnt, lane, cq);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    w4.v[q] = w_sub_tab(w4.v[q], s_upd, s_upd64, cq[q] + NR);
                    l4[q] = loc_of(w4.v[q], g4[q], a.eta_l, a.eta_l_d);
                    isq += a_on * cq[q] * cq[q];
                }
                const int jb = 4 * (lane & 3);
                const uint32_t vm = nv >= 4 ? 0xffu : (1u << (2 * nv)) - 1u;  // padding codes are not checked
                if (!a_off && ((cnt.rsv >> (2 * jb)) & vm) != 0u) {
                    const int q = __ffs((cnt.rsv >> (2 * jb)) & vm & 0x55u) / 2;
                    bad_sym = static_cast<uint64_t>(e + q) < bad_sym ? static_cast<uint64_t>(e + q) : bad_sym;
                }
            } else if constexpr (APPLY == APPLY_F) {
                const float s4[4] = {sv[c].x, sv[c].y, sv[c].z, sv[c].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    w4.v[q] = w_sub_full(w4.v[q], s4[q], a.scale, a.eta_g_d, a.inv_n_or_zero, a.nranks);
                    l4[q] = loc_of(w4.v[q], g4[q], a.eta_l, a.eta_l_d);
                    if (a.gnorm != nullptr && !a_off) {
                        const double m = s4[q] * a.inv_n;
                        gsq = __fma_rn(m, m, gsq);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) l4[q] = loc_of(w4.v[q], g4[q], a.eta_l, a.eta_l_d);
            }
            TW* const wdst = SINK && a_off ? sink_of<TW>(h.sink, lane) : W + e;
            float* const ldst = SINK && a_off ? sink_of<float>(h.sink, lane) : h.loc + e;
            if constexpr (APPLY != APPLY_L) stw4(wdst, w4, nv);
            st_stream_m(ldst, l4[0], l4[1], l4[2], l4[3], nv);
        }
        if (SINK || !q_off) {
            TR o[4];
            uint32_t code = 0;
            bool b = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) code |= quant1_lean(r4[q], g4[q], a.alpha, ahi, alo, o[q], b) << (2 * q);
            bad |= b && !q_off;
            TR* const rdst = SINK && q_off ? sink_of<TR>(h.sink, lane) : r_out + e;
            st_stream_m(rdst, o[0], o[1], o[2], o[3], nv);
            v[c] = q_off ? 0u : code << (8 * (lane & 3));
        } else {
            v[c] = 0;
        }
    }
    CDSGD_PROBE(11);
    if (__any_sync(FULL, bad)) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const float g4[4] = {gv[c].x, gv[c].y, gv[c].z, gv[c].w};
            const TR(&r4)[4] = rv[c].v;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (nonfinite(r4[q] + static_cast<TR>(g4[q]))) {
                    const uint64_t idx =
                        a.tag | static_cast<uint64_t>(e0 + 128 * (c0 + c) + 4 * lane + q);
                    bad_idx = idx < bad_idx ? idx : bad_idx;
                }
        }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] |= __shfl_xor_sync(FULL, v[c], 1);
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] |= __shfl_xor_sync(FULL, v[c], 2);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint32_t w = __shfl_sync(FULL, v[c], 4 * (lane & 7));
        if ((lane >> 3) == c0 + c) myword = w;
    }
    return myword;
}

// Data moved with 128/256-bit coalesced loads straight into registers (all loads of a
// tile issued first), two 256-thread CTAs per SM, dynamic tile scheduling.
// CH = chunks of 128 elements per task: 4 (a whole tile) for large layouts, 1 for small
// ones (ResNet-20-sized), where 4x more warps in flight beat the per-tile latency chain.
// fp64 weights add 8 B per element to each task's loads in flight (g 16 + r 32 + W 32 bytes per
// lane per chunk): CDSGD_F64_MINB / CDSGD_F64_CH select CTAs per SM and chunks per task for TW=double.
#ifndef CDSGD_F64_MINB
#define CDSGD_F64_MINB 2
#endif
#ifndef CDSGD_F64_CH
#define CDSGD_F64_CH 4
#endif

template <int NR, int APPLY, int CH = CHUNKS, typename TW = float, typename TR = double>
__global__ void __launch_bounds__(256, sizeof(TW) == 8 ? CDSGD_F64_MINB : 2) k_fused_ldg(FusedArgs a, KeyTab kt, DecodeTab tab) {
    constexpr int SPL = CHUNKS / CH;  // tasks per tile
    CDSGD_PROBE(0);
    CDSGD_PROBE(1);
    __shared__ float s_upd[2 * MAX_RANKS + 1];
    __shared__ double s_upd64[2 * MAX_RANKS + 1];
    TW* const W = static_cast<TW*>(a.W);
    // Everything that reads only constant inputs (decode table, key table, schedule) runs
    // BEFORE griddepcontrol.wait, overlapping the previous kernel's tail: on launch-bound
    // layouts the key seek (two dependent key-table loads) was part of every round's latency.
    const int lane = threadIdx.x & 31;
    const uint32_t ahi = static_cast<uint32_t>(__double2hiint(a.alpha));
    const uint32_t alo = static_cast<uint32_t>(__double2loint(a.alpha));
    const int64_t ntasks = kt.ntiles * SPL;
    int64_t tb, te;
    warp_range(ntasks, tb, te);
    uint64_t bad_idx = NO_ERR, bad_sym = NO_ERR;
    double gsq = 0.0;
    int isq = 0;
    // Dynamic schedule: warps claim CLAIM consecutive tasks at a time from a global ticket,
    // so the kernel ends when the work does, not when the slowest static range does.
    // small layouts (fewer than ~4 tasks per warp): claim single tasks for parallelism
    const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
    const unsigned CLAIM = ntasks < 4 * nwarps ? 1u : 2u;
    const int64_t tail_from = ntasks - nwarps;
    // one wave of tasks (small layouts): each warp takes its own, no ticket and no end-of-launch
    // ticket reset (a fence + atomic per CTA on one counter)
    bool dyn = a.sched != nullptr && ntasks > nwarps * static_cast<int64_t>(CLAIM);
    if constexpr (CH == 1) {  // held in a register across the wait (not re-derived from a.sched after it)
        int d = dyn ? 1 : 0;
        asm volatile("" : "+r"(d));
        dyn = d != 0;
    }
    int64_t cbase = 0, cend = 0;
    // first claim static (warp w: tasks [w*CLAIM, (w+1)*CLAIM)), later claims from the ticket
    // offset by nwarps*CLAIM: no burst of one atomic per warp on a single counter at launch
    // (it serialised ~2,400 warps for several us on ResNet-20-sized layouts)
    const int64_t first_dyn = nwarps * CLAIM;
    if (dyn) {
        cbase = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * CLAIM;
        cend = cbase + (int64_t)CLAIM < ntasks ? cbase + (int64_t)CLAIM : ntasks;
        tb = cbase;
        te = cbase < ntasks ? ntasks : cbase;  // loop bound; real bound checked per claim
    }
    if (APPLY == APPLY_Q && threadIdx.x < 2 * NR + 1) {
        s_upd[threadIdx.x] = tab.upd[threadIdx.x];
        s_upd64[threadIdx.x] = tab.upd64[threadIdx.x];
    }
    TileCursor cc;
    if (tb < te) {
        if (kt.tiles != nullptr) cc.from_table(kt, tb / SPL);
        else cc.seek_warp(kt, tb / SPL, lane);
    }
    // A task's placement (tile element/word offsets, sizes, vector-path alignment) depends only
    // on the key table and the buffer addresses: the first task's is computed here, before the
    // wait, so that after it a warp goes straight to its loads (on one-wave layouts the ~100
    // instructions of this setup, times 4 warps per scheduler, delayed the last loads by
    // several hundred cycles).
    struct TaskDesc {
        int64_t e0, w0;
        int ne, nw, c0;
        bool fast;
    };
    auto describe = [&](int64_t task) {
        TaskDesc d;
        const int64_t ti = task / SPL;
        d.c0 = static_cast<int>(task % SPL) * CH;  // first chunk of this task
        if (kt.tiles != nullptr) {
            if (ti != cc.t0) cc.from_table(kt, ti);
        } else {
            if (ti < cc.t0) cc.seek_warp(kt, ti, lane);
            cc.advance_warp(kt, ti, lane);
        }
        const int64_t j = ti - cc.t0;
        d.e0 = cc.e0 + j * TILE_ELEMS;
        d.w0 = cc.w0 + j * TILE_WORDS;
        const int64_t ne64 = cc.e1 - d.e0;
        d.ne = ne64 < TILE_ELEMS ? static_cast<int>(ne64) : TILE_ELEMS;
        const int64_t nw64 = cc.w1 - d.w0;
        d.nw = nw64 < TILE_WORDS ? static_cast<int>(nw64) : TILE_WORDS;
        const int64_t e0 = d.e0;
        d.fast = aligned_to(a.g + e0, 16) && aligned_to(static_cast<const TR*>(a.r_in) + e0, 4 * sizeof(TR)) &&
                 aligned_to(static_cast<TR*>(a.r_out) + e0, 4 * sizeof(TR)) && aligned_to(W + e0, 4 * sizeof(TW)) &&
                 aligned_to(a.loc + e0, 16) && (APPLY != APPLY_F || aligned_to(a.gsum + e0, 16)) &&
                 (APPLY != APPLY_Q || a.exact);
        return d;
    };
    TaskDesc td{};
    if (CH == 1 && tb < te) td = describe(tb);  // (large layouts: in the loop, fewer live registers)
    HotPtrs hot(a);
    if constexpr (CH == 1) hot.pin_here();
    if (APPLY == APPLY_Q) __syncthreads();  // s_upd, before the wait (off the critical path)
    CDSGD_PROBE(2);
    pdl_enter(a.gclear[0], a.gclear[1]);  // from here on: memory the preceding kernels write
    CDSGD_PROBE(3);
    RoundFlags fl;
    // Small layouts, first task: its loads go out right after the wait — everything they need
    // was computed before it (on a one-wave grid the loop setup between the wait and the loads,
    // times four warps per scheduler, was several hundred cycles of every round). Not with a
    // peer-flag wait (N > 1, P2P): the codes are only complete after it.
    TaskRegs<NR, APPLY, CH, TW, TR> L;
    bool pre = false;
    if constexpr (CH == 1) {
        pre = tb < te && td.fast && !hot.p2p_wait;
        if (pre) {
            if (CDSGD_FULL_SPEC && td.ne == TILE_ELEMS)
                fused_vec_load<NR, APPLY, CH, TW, true, TR>(a, hot, lane, td.e0, td.w0, td.ne, td.nw, td.c0, fl, L);
            else
                fused_vec_load<NR, APPLY, CH, TW, false, TR>(a, hot, lane, td.e0, td.w0, td.ne, td.nw, td.c0, fl, L);
        }
    }
    // (no barrier when there is nothing to wait for; small layouts test the flag computed pre-wait)
    fl.peer_failed = (CH != 1 || hot.p2p_wait) && p2p_wait2(a.xq, a.xa);
    CDSGD_PROBE(13);
    if constexpr (CH != 1) {  // bandwidth-bound launches: read the error word up front (fewer live registers)
        fl.resolve(a, a.err);
        __syncthreads();
    }
    if (tb < te) {
        for (int64_t task = tb; task < te; ++task) {
            if (dyn) {
                if (task >= cend) {  // claim the next batch (single tasks in the last ~one per warp)
                    const unsigned cl = task < tail_from ? CLAIM : 1u;
                    unsigned t0 = 0;
                    if (lane == 0) t0 = atomicAdd(a.sched, cl);
                    const int64_t nb = first_dyn + static_cast<int64_t>(__shfl_sync(FULL, t0, 0));
                    if (nb >= ntasks) break;
                    task = nb;
                    cend = nb + (int64_t)cl < ntasks ? nb + (int64_t)cl : ntasks;
                }
            }
            if (CH != 1 || task != tb) td = describe(task);
            const int64_t e0 = td.e0, w0 = td.w0;
            const int ne = td.ne, nw = td.nw, c0 = td.c0;
            const bool fast = td.fast;
            if (!fast && c0 != 0) continue;  // misaligned tiles: one task does the whole tile
            uint32_t myword = 0;
            CDSGD_PROBE(14);
            if (fast) {
                const bool loaded = pre && task == tb;
                if (CDSGD_FULL_SPEC && ne == TILE_ELEMS)
                    myword = fused_vec_task<NR, APPLY, CH, TW, true, TR>(a, hot, s_upd, s_upd64, lane, e0, w0, ne, nw, c0, fl,
                                                                     ahi, alo, bad_idx, bad_sym, gsq, isq, L, loaded);
                else
                    myword = fused_vec_task<NR, APPLY, CH, TW, false, TR>(a, hot, s_upd, s_upd64, lane, e0, w0, ne, nw, c0, fl,
                                                                      ahi, alo, bad_idx, bad_sym, gsq, isq, L, loaded);
            } else {
                fl.resolve(a, a.err);
                const bool a_off = fl.a_off, q_off = fl.q_off;
                uint32_t cw[APPLY == APPLY_Q ? NR : 1];
                if constexpr (APPLY == APPLY_Q) {
#pragma unroll
                    for (int r = 0; r < NR; ++r) cw[r] = lane < nw ? a.gathered[r * a.stride + w0 + lane] : 0u;
                }
#pragma unroll 2
                for (int s = 0; s < TILE_ELEMS / 32; ++s) {
                    const int el = 32 * s + lane;
                    int cn = 0;
                    bool rsv = false;
                    uint32_t cds[APPLY == APPLY_Q ? NR : 1];
                    if constexpr (APPLY == APPLY_Q) {
#pragma unroll
                        for (int r = 0; r < NR; ++r) {
                            const uint32_t cd = (__shfl_sync(FULL, cw[r], 2 * s + (lane >> 4)) >> (2 * (lane & 15))) & 3u;
                            cds[r] = cd;
                            rsv |= cd == 3u;
                            cn += (cd == 1u) - (cd == 2u);
                        }
                    }
                    bool p = false, m = false;
                    if (el < ne) {
                        const int64_t e = e0 + el;
                        const float gval = a.g[e];
                        if (!a_off) {
                            TW wn;
                            if constexpr (APPLY == APPLY_Q) {
                                if (a.exact) {
                                    wn = w_sub_tab(W[e], s_upd, s_upd64, cn + NR);
                                    isq += cn * cn;
                                } else {  // sequential ascending-rank fp64 sum, as K2's generic path
                                    bool r2 = false;
                                    const double mean = apply_mean_general(cds, NR, a.alpha, a.inv_n_or_zero, r2);
                                    wn = w_sub_mean(W[e], a.eta_g_d, mean);
                                    if (a.gnorm != nullptr) gsq = __fma_rn(mean, mean, gsq);
                                }
                                if (rsv) bad_sym = static_cast<uint64_t>(e) < bad_sym ? static_cast<uint64_t>(e) : bad_sym;
                            } else if constexpr (APPLY == APPLY_F) {
                                const float sv1 = a.gsum[e];
                                wn = w_sub_full(W[e], sv1, a.scale, a.eta_g_d, a.inv_n_or_zero, a.nranks);
                                if (a.gnorm != nullptr) { const double mm = sv1 * a.inv_n; gsq = __fma_rn(mm, mm, gsq); }
                            } else {
                                wn = W[e];
                            }
                            if constexpr (APPLY != APPLY_L) W[e] = wn;
                            a.loc[e] = loc_of(wn, gval, a.eta_l, a.eta_l_d);
                        }
                        if (!q_off) {
                            TR o;
                            bool b;
                            const uint32_t code = quant1(static_cast<const TR*>(a.r_in)[e], gval, a.alpha, o, b);
                            static_cast<TR*>(a.r_out)[e] = o;
                            p = code == 1u;
                            m = code == 2u;
                            if (b) {
                                const uint64_t idx = a.tag | static_cast<uint64_t>(e);
                                bad_idx = idx < bad_idx ? idx : bad_idx;
                            }
                        }
                    }
                    const uint32_t pm = __ballot_sync(FULL, p);
                    const uint32_t mm = __ballot_sync(FULL, m);
                    if (lane == 2 * s) myword = interleave_codes(pm, mm);
                    if (lane == 2 * s + 1) myword = interleave_codes(pm >> 16, mm >> 16);
                }
            }
            CDSGD_PROBE(4);
            const bool mine_word = !fast || ((lane >> 3) >= c0 && (lane >> 3) < c0 + CH);
            if (lane < nw && !fl.q_off && mine_word) {
                if (a.xq.nranks > 0) {
                    for (int r = 0; r < a.xq.nranks; ++r)
                        if (a.xq.dst[r] != nullptr) a.xq.dst[r][w0 + lane] = myword;
                } else {
                    a.words[w0 + lane] = myword;
                }
            }
        }
    }
    CDSGD_PROBE(5);
    if (a.gnorm != nullptr) block_atomic_add_counts(isq, gsq, tab.sq_scale, a.gnorm);
    CDSGD_PROBE(6);
    if (a.err != nullptr) {
        bad_idx = warp_min_u64(bad_idx);
        bad_sym = warp_min_u64(bad_sym);
        if (lane == 0 && bad_idx != NO_ERR)
            atomicMin(reinterpret_cast<unsigned long long*>(a.err), static_cast<unsigned long long>(bad_idx));
        if (lane == 0 && bad_sym != NO_ERR)
            atomicMin(reinterpret_cast<unsigned long long*>(a.err + 1), static_cast<unsigned long long>(bad_sym));
    }
    if (dyn) {  // the last CTA out resets the ticket for the next launch on this stream
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
                a.sched[0] = 0u;
                a.sched[1] = 0u;
                __threadfence();
            }
        }
    }
    p2p_publish2(a.xq, a.xa, a.xq.counter != nullptr ? a.xq.counter : a.xa.counter);
    CDSGD_PROBE(7);
#ifdef CDSGD_PROBE_TIMING
    probe_flush();
#endif
}
}  // namespace cdsgd
