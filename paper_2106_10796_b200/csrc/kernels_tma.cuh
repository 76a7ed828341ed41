// kernels_tma.cuh — TMA-staged (cp.async.bulk + mbarrier) variants of K1 and K3.
//
// Each warp owns a contiguous range of tiles (as in kernels.cuh) and an S-slot
// ring in shared memory. Lane 0 arms slot s's mbarrier with the tile's byte
// count and issues 1-D bulk copies (TMA engine, no registers held) for the tile
// S-1 positions ahead; the warp then waits on the current slot's barrier and
// computes from shared memory. Loads of S-1 tiles per warp are therefore always
// in flight (~12 KB/warp for K1 at S=3) independent of register pressure —
// latency-hiding by the async copy engine instead of by occupancy. Results are
// stored straight from registers with 128/256-bit coalesced st.global.
//
// fp64 tiles are read from smem as two 16-byte halves per lane in a swizzled
// order (lanes 4..7 of each quarter-warp read their upper half first), which
// makes every 128-bit LDS phase cover all 32 banks exactly once.
//
// Tiles that are partial (last tile of a key) or not 16/32-byte aligned are not
// staged; the warp processes them with the coalesced global-memory paths.
#pragma once
#include "kernels.cuh"

namespace cdsgd {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2; selp.b32 %0, 1, 0, P1; }"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

// 4 consecutive elements [4*lane, 4*lane+4) of a 128-element chunk in smem.
__device__ __forceinline__ void lds4(const float* chunk, int lane, float (&v)[4]) {
    const float4 t = reinterpret_cast<const float4*>(chunk)[lane];
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
#ifndef CDSGD_LDS_SWIZZLE
#define CDSGD_LDS_SWIZZLE 0
#endif
__device__ __forceinline__ void lds4(const double* chunk, int lane, double (&v)[4]) {
    const double2* p = reinterpret_cast<const double2*>(chunk) + 2 * lane;
#if CDSGD_LDS_SWIZZLE
    const int sw = (lane >> 2) & 1;  // conflict-free 128-bit phases, at the cost of 8 selects
    const double2 a = p[sw];
    const double2 b = p[sw ^ 1];
    v[0] = sw ? b.x : a.x; v[1] = sw ? b.y : a.y;
    v[2] = sw ? a.x : b.x; v[3] = sw ? a.y : b.y;
#else
    const double2 a = p[0];  // 2-way bank conflict per 128-bit phase, no selects
    const double2 b = p[1];
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
#endif
}

}  // namespace tma

// CTA = WARPS warps, one CTA per SM (the smem ring, not occupancy, hides latency).

// ================================================================ K1 (TMA)
template <typename G, typename TR>
__device__ __noinline__ uint64_t rescan_nonfinite(const G* sg, const TR* sr, int lane, int64_t e0, uint64_t tag,
                                                  uint64_t bad_idx) {
    for (int c = 0; c < CHUNKS; ++c)
        for (int q = 0; q < 4; ++q) {
            const int el = 128 * c + 4 * lane + q;
            if (nonfinite(sr[el] + static_cast<TR>(sg[el]))) {
                const uint64_t idx = tag | static_cast<uint64_t>(e0 + el);
                bad_idx = idx < bad_idx ? idx : bad_idx;
            }
        }
    return bad_idx;
}

template <typename G, int WARPS, int S, typename TR = double>
struct QuantSmem {
    static constexpr int GB = TILE_ELEMS * sizeof(G);
    static constexpr int RB = TILE_ELEMS * sizeof(TR);
    static constexpr int SLOT = GB + RB;
    static constexpr int WARP = S * SLOT;
    static constexpr int BYTES = WARPS * WARP + WARPS * S * 8;
};

template <typename G, int WARPS, int S, typename TR = double>
__global__ void __launch_bounds__(WARPS * 32, 1)
    k_quantize_tma(const G* __restrict__ g, const TR* r_in, TR* r_out, uint32_t* __restrict__ words,
                   KeyTab kt, double alpha, uint64_t* err, uint64_t tag, P2PArgs x) {
    using SM = QuantSmem<G, WARPS, S, TR>;
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter(nullptr, nullptr);
    const bool peer_failed = p2p_wait(x);  // fused exchange: peers have released the slot we are about to fill
    // sticky abort: only errors of EARLIER rounds (smaller tag) stop the kernel, so one CTA's
    // finding never suppresses another CTA's scan of this round (first index stays exact)
    const bool aborted = peer_failed || (err != nullptr && *reinterpret_cast<volatile uint64_t*>(err) < tag);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned char* ring = smem + warp * SM::WARP;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * SM::WARP) + warp * S;
    int64_t tb, te;
    warp_range(kt.ntiles, tb, te);
    if (aborted) te = tb;  // sticky abort: no work, but still take part in the exchange protocol
    uint64_t bad_idx = NO_ERR;
    if (tb < te) {
    if (lane == 0) {
        for (int s = 0; s < S; ++s) tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    TileCursor pc, cc;
    pc.seek(kt, tb);
    cc = pc;
    uint32_t staged = 0, phase = 0;
    auto issue = [&](int64_t ti, int slot) {
        pc.advance_to(kt, ti);
        const int64_t e0 = pc.e0 + (ti - pc.t0) * TILE_ELEMS;
        const bool full = pc.e1 - e0 >= TILE_ELEMS;
        const bool ok = full && aligned_to(g + e0, 16) && aligned_to(r_in + e0, 16) &&
                        aligned_to(r_out + e0, 4 * sizeof(TR));
        if (ok) {
            if (lane == 0) {
                unsigned char* sl = ring + slot * SM::SLOT;
                tma::arrive_expect_tx(&bars[slot], SM::SLOT);
                tma::bulk_g2s(sl, g + e0, SM::GB, &bars[slot]);
                tma::bulk_g2s(sl + SM::GB, r_in + e0, SM::RB, &bars[slot]);
            }
            staged |= 1u << slot;
        } else {
            staged &= ~(1u << slot);
        }
    };
    for (int i = 0; i < S - 1 && tb + i < te; ++i) issue(tb + i, i);
    int slot = 0;
    for (int64_t ti = tb; ti < te; ++ti) {
        if (ti + S - 1 < te) {
            __syncwarp();  // every lane is done reading the slot being refilled (WAR; no proxy fence needed)
            issue(ti + S - 1, slot == 0 ? S - 1 : slot - 1);
        }
        cc.advance_to(kt, ti);
        const int64_t j = ti - cc.t0;
        const int64_t e0 = cc.e0 + j * TILE_ELEMS;
        const int64_t w0 = cc.w0 + j * TILE_WORDS;
        const int64_t ne64 = cc.e1 - e0;
        const int ne = ne64 < TILE_ELEMS ? static_cast<int>(ne64) : TILE_ELEMS;
        const int64_t nw64 = cc.w1 - w0;
        const int nw = nw64 < TILE_WORDS ? static_cast<int>(nw64) : TILE_WORDS;
        uint32_t myword = 0;
        if (staged & (1u << slot)) {
            tma::wait(&bars[slot], (phase >> slot) & 1u);
            phase ^= 1u << slot;
            const G* sg = reinterpret_cast<const G*>(ring + slot * SM::SLOT);
            const TR* sr = reinterpret_cast<const TR*>(ring + slot * SM::SLOT + SM::GB);
            // phase A: every smem read of the tile first (one dependency level)
            G gv[CHUNKS][4];
            TR rv[CHUNKS][4];
#pragma unroll
            for (int c = 0; c < CHUNKS; ++c) {
                tma::lds4(sg + 128 * c, lane, gv[c]);
                tma::lds4(sr + 128 * c, lane, rv[c]);
            }
            // phase B: fp64 threshold + residual, 256-bit stores
            uint32_t v[CHUNKS];
            bool bad = false;
            const uint32_t ahi = static_cast<uint32_t>(__double2hiint(alpha));
            const uint32_t alo = static_cast<uint32_t>(__double2loint(alpha));
#pragma unroll
            for (int c = 0; c < CHUNKS; ++c) {
                TR o[4];
                uint32_t code = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) code |= quant1_lean(rv[c][q], gv[c][q], alpha, ahi, alo, o[q], bad) << (2 * q);
                st_stream(r_out + e0 + 128 * c + 4 * lane, o[0], o[1], o[2], o[3]);
                v[c] = code << (8 * (lane & 3));
            }
            if (__any_sync(FULL, bad))  // rare: locate the first non-finite accumulator of the tile
                bad_idx = rescan_nonfinite(sg, sr, lane, e0, tag, bad_idx);
            // phase C: pack 4 lanes x 8 bits per word, the 4 chunks' shuffle chains interleaved
#pragma unroll
            for (int c = 0; c < CHUNKS; ++c) v[c] |= __shfl_xor_sync(FULL, v[c], 1);
#pragma unroll
            for (int c = 0; c < CHUNKS; ++c) v[c] |= __shfl_xor_sync(FULL, v[c], 2);
#pragma unroll
            for (int c = 0; c < CHUNKS; ++c) {
                const uint32_t w = __shfl_sync(FULL, v[c], 4 * (lane & 7));
                if ((lane >> 3) == c) myword = w;
            }
        } else {
#pragma unroll 4
            for (int s = 0; s < TILE_ELEMS / 32; ++s) {
                const int el = 32 * s + lane;
                bool p = false, m = false;
                if (el < ne) {
                    TR o;
                    bool b;
                    const uint32_t code = quant1(r_in[e0 + el], g[e0 + el], alpha, o, b);
                    r_out[e0 + el] = o;
                    p = code == 1u;
                    m = code == 2u;
                    if (b) {
                        const uint64_t idx = tag | static_cast<uint64_t>(e0 + el);
                        bad_idx = idx < bad_idx ? idx : bad_idx;
                    }
                }
                const uint32_t pm = __ballot_sync(FULL, p);
                const uint32_t mm = __ballot_sync(FULL, m);
                if (lane == 2 * s) myword = interleave_codes(pm, mm);
                if (lane == 2 * s + 1) myword = interleave_codes(pm >> 16, mm >> 16);
            }
        }
        if (lane < nw) {
            if (x.nranks > 0) {
                // fused all-gather: the word goes straight into every rank's slot (NVLink stores)
                for (int r = 0; r < x.nranks; ++r) x.dst[r][w0 + lane] = myword;
            } else {
                words[w0 + lane] = myword;
            }
        }
        slot = slot + 1 == S ? 0 : slot + 1;
    }
    }  // tb < te
    if (err != nullptr) {
        bad_idx = warp_min_u64(bad_idx);
        if (lane == 0 && bad_idx != NO_ERR)
            atomicMin(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(bad_idx));
    }
    p2p_publish(x);
}

// ================================================================ K3 (TMA)
template <int WARPS, int S, typename TW = float>
struct ApplyFSmem {
    static constexpr int WB = TILE_ELEMS * static_cast<int>(sizeof(TW));
    static constexpr int SLOT = WB + 2 * TILE_ELEMS * 4;  // W | gsum | g_next
    static constexpr int WARP = S * SLOT;
    static constexpr int BYTES = WARPS * WARP + WARPS * S * 8;
};

template <int WARPS, int S, typename TW = float>
__global__ void __launch_bounds__(WARPS * 32, 1) k_apply_full_tma(ApplyFArgs a) {
    using SM = ApplyFSmem<WARPS, S, TW>;
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_enter(a.gclear[0], a.gclear[1]);
    if (a.err != nullptr && *reinterpret_cast<volatile const uint64_t*>(a.err) < a.skip_below) return;
    TW* const W = static_cast<TW*>(a.W);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned char* ring = smem + warp * SM::WARP;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * SM::WARP) + warp * S;
    const bool do_loc = a.loc != nullptr;
    const int64_t ntiles = (a.n + TILE_ELEMS - 1) / TILE_ELEMS;
    int64_t tb, te;
    warp_range(ntiles, tb, te);
    double gsq = 0.0;
    if (tb < te) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) tma::mbar_init(&bars[s], 1);
            tma::fence_mbar_init();
        }
        __syncwarp();
        uint32_t staged = 0, phase = 0;
        auto issue = [&](int64_t ti, int slot) {
            const int64_t e0 = ti * TILE_ELEMS;
            const bool ok = e0 + TILE_ELEMS <= a.n && aligned_to(W + e0, 4 * sizeof(TW)) && aligned_to(a.gsum + e0, 16) &&
                            (!do_loc || (aligned_to(a.gnext + e0, 16) && aligned_to(a.loc + e0, 16)));
            if (ok) {
                if (lane == 0) {
                    unsigned char* sl = ring + slot * SM::SLOT;
                    tma::arrive_expect_tx(&bars[slot], SM::WB + TILE_ELEMS * 4 * (do_loc ? 2 : 1));
                    tma::bulk_g2s(sl, W + e0, SM::WB, &bars[slot]);
                    tma::bulk_g2s(sl + SM::WB, a.gsum + e0, TILE_ELEMS * 4, &bars[slot]);
                    if (do_loc) tma::bulk_g2s(sl + SM::WB + TILE_ELEMS * 4, a.gnext + e0, TILE_ELEMS * 4, &bars[slot]);
                }
                staged |= 1u << slot;
            } else {
                staged &= ~(1u << slot);
            }
        };
        for (int i = 0; i < S - 1 && tb + i < te; ++i) issue(tb + i, i);
        int slot = 0;
        for (int64_t ti = tb; ti < te; ++ti) {
            if (ti + S - 1 < te) {
                __syncwarp();  // every lane is done reading the slot being refilled (WAR; no proxy fence needed)
                issue(ti + S - 1, slot == 0 ? S - 1 : slot - 1);
            }
            const int64_t e0 = ti * TILE_ELEMS;
            if (staged & (1u << slot)) {
                tma::wait(&bars[slot], (phase >> slot) & 1u);
                phase ^= 1u << slot;
                const TW* sw = reinterpret_cast<const TW*>(ring + slot * SM::SLOT);
                const float* sl = reinterpret_cast<const float*>(ring + slot * SM::SLOT + SM::WB);
#pragma unroll
                for (int c = 0; c < CHUNKS; ++c) {
                    const int64_t e = e0 + 128 * c + 4 * lane;
                    TW w4[4];
                    float s4[4], g4[4];
                    tma::lds4(sw + 128 * c, lane, w4);
                    tma::lds4(sl + 128 * c, lane, s4);
                    if (do_loc) tma::lds4(sl + TILE_ELEMS + 128 * c, lane, g4);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        w4[q] = w_sub_full(w4[q], s4[q], a.scale, a.eta_g_d, a.inv_n_or_zero, a.nranks);
                        if (do_loc) g4[q] = loc_of(w4[q], g4[q], a.eta_l, a.eta_l_d);
                        if (a.gnorm != nullptr) {
                            const double m = s4[q] * a.inv_n;
                            gsq = __fma_rn(m, m, gsq);
                        }
                    }
                    st_stream(W + e, w4[0], w4[1], w4[2], w4[3]);
                    if (do_loc) st_stream(a.loc + e, g4[0], g4[1], g4[2], g4[3]);
                }
            } else {
                const int64_t e1 = e0 + TILE_ELEMS < a.n ? e0 + TILE_ELEMS : a.n;
                for (int64_t i = e0 + lane; i < e1; i += 32) {
                    const float s = a.gsum[i];
                    const TW wn = w_sub_full(W[i], s, a.scale, a.eta_g_d, a.inv_n_or_zero, a.nranks);
                    W[i] = wn;
                    if (do_loc) a.loc[i] = loc_of(wn, a.gnext[i], a.eta_l, a.eta_l_d);
                    if (a.gnorm != nullptr) {
                        const double m = s * a.inv_n;
                        gsq = __fma_rn(m, m, gsq);
                    }
                }
            }
            slot = slot + 1 == S ? 0 : slot + 1;
        }
    }
    if (a.gnorm != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gsq += __shfl_xor_sync(FULL, gsq, o);
        if (lane == 0 && gsq != 0.0) atomicAdd(a.gnorm, gsq);
    }
}

}  // namespace cdsgd
