// kernels.cuh — sm_100a device code of the CD-SGD hot path.
//
// Data layout in HBM (one rank):
//   g        fp32[n]          this round's gradient (caller-owned)
//   r[2]     fp64[n]          ping-pong error-feedback residual (exact mode)
//   words    u32[W(n)]        2-bit codes, 16 per word, packing restarts per key
//   W, loc   fp32[n]          replicated global weights / local compute weights
//
// Work unit: a "tile" = up to 32 packed words (512 elements) of ONE key. Tiles
// never straddle keys (per-key packing restart, codec.py:147-148 via
// engine.py:397-402), so only the last tile of a key can be partial. Warps claim
// tiles from a global ticket (or own a contiguous range), walk keys
// incrementally and, for full 32B-aligned tiles, move data with 128-bit
// (fp32) and 256-bit (fp64) vector loads/stores: lane l owns elements
// [128c + 4l, 128c + 4l + 4) of chunk c (c = 0..3), so every warp-wide access
// is fully coalesced. Codes are packed with two xor-shuffles (4 lanes -> one
// word) and one index shuffle so lane j stores word j (one 128 B store).
// Partial / misaligned tiles take a coalesced scalar path that packs with
// __ballot_sync (lane l owns element 32s + l) and a Morton bit interleave.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cdsgd {

constexpr unsigned FULL = 0xffffffffu;
constexpr int TILE_WORDS = 32;
constexpr int TILE_ELEMS = 512;
constexpr int CHUNKS = 4;           // 128-element chunks per tile (fast path)
constexpr uint64_t NO_ERR = ~0ull;
constexpr int MAX_RANKS_P2P = 8;  // fused NVLink exchange: one box of <= 8 GPUs

struct KeyTab {
    const int64_t* eoff;  // [nkeys+1] element offsets
    const int64_t* woff;  // [nkeys+1] word offsets
    const int64_t* toff;  // [nkeys+1] tile offsets
    int32_t nkeys;
    int64_t ntiles;
    // Per-tile metadata {e0 lo, e0 hi, w0, ne | nw << 16} (nullptr for very large layouts):
    // one 16-byte load locates a tile, instead of a key search (two dependent rounds of key-table
    // loads) — on launch-bound layouts that search was a visible part of every round's latency.
    const int4* tiles;
};

// ---------------------------------------------------------------- memory helpers
__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
struct d4 { double x, y, z, w; };
__device__ __forceinline__ d4 ld_stream(const double* p) {
    d4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
#ifndef CDSGD_ST_HINT
#define CDSGD_ST_HINT "cs"  // streaming stores (vs L1::no_allocate: -1 us on F and K2 at ResNet-50 size)
#endif
__device__ __forceinline__ void st_stream(double* p, double a, double b, double c, double d) {
    asm volatile("st.global." CDSGD_ST_HINT ".v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b),
                 "d"(c), "d"(d));
}
__device__ __forceinline__ void st_stream(float* p, float a, float b, float c, float d) {
    asm volatile("st.global." CDSGD_ST_HINT ".v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b),
                 "f"(c), "f"(d));
}
__device__ __forceinline__ uint32_t ld_word(const uint32_t* p) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Masked 4-element accesses for the last (partial) chunk of a key: nv = valid elements
// (>= 4: one vector access; 1..3: scalar accesses; missing loads read as 0). Lets the
// vector paths take partial tiles too — a latency-bound per-element fallback on the
// final tile of a launch (ResNet-50's fc bias) measured as a ~14 us straggler.
__device__ __forceinline__ float4 ld_stream_m(const float* p, int nv) {
    if (nv >= 4) return ld_stream(p);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nv > 0) v.x = p[0];
    if (nv > 1) v.y = p[1];
    if (nv > 2) v.z = p[2];
    return v;
}
__device__ __forceinline__ d4 ld_stream_m(const double* p, int nv) {
    if (nv >= 4) return ld_stream(p);
    d4 v{0.0, 0.0, 0.0, 0.0};
    if (nv > 0) v.x = p[0];
    if (nv > 1) v.y = p[1];
    if (nv > 2) v.z = p[2];
    return v;
}
template <typename T>
__device__ __forceinline__ void st_stream_m(T* p, T a, T b, T c, T d, int nv) {
    if (nv >= 4) {
        st_stream(p, a, b, c, d);
        return;
    }
    if (nv > 0) p[0] = a;
    if (nv > 1) p[1] = b;
    if (nv > 2) p[2] = c;
}
// valid elements of the 4 starting at tile offset off, in a tile of ne elements
__device__ __forceinline__ int nvalid4(int ne, int off) {
    const int v = ne - off;
    return v < 0 ? 0 : (v > 4 ? 4 : v);
}

__device__ __forceinline__ bool aligned_to(const void* p, uintptr_t a) {
    return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

// 16 low bits of x spread to the even bit positions of a 32-bit word.
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x &= 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}
// Word of 16 two-bit codes from plus/minus lane masks (bit i = element i).
__device__ __forceinline__ uint32_t interleave_codes(uint32_t plus16, uint32_t minus16) {
    return spread16(plus16) | (spread16(minus16) << 1);
}

__device__ __forceinline__ bool nonfinite(double a) {
    return (static_cast<uint32_t>(__double2hiint(a)) & 0x7ff00000u) == 0x7ff00000u;
}

// ---------------------------------------------------------------- tile walking
// Warp `wid` of `nwarps` owns tiles [t_begin, t_end). The key containing a tile
// is found once by binary search, then advanced incrementally.
struct TileCursor {
    int k;
    int64_t t0, t1;  // tile range of key k
    int64_t e0, e1;  // element range of key k
    int64_t w0, w1;  // word range of key k
    __device__ __forceinline__ void load(const KeyTab& kt, int key) {
        k = key;
        t0 = __ldg(kt.toff + k); t1 = __ldg(kt.toff + k + 1);
        e0 = __ldg(kt.eoff + k); e1 = __ldg(kt.eoff + k + 1);
        w0 = __ldg(kt.woff + k); w1 = __ldg(kt.woff + k + 1);
    }
    __device__ __forceinline__ void seek(const KeyTab& kt, int64_t tile) {
        int lo = 0, hi = kt.nkeys - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (__ldg(kt.toff + mid) <= tile) lo = mid; else hi = mid - 1;
        }
        load(kt, lo);
    }
    // Warp-collective seek (every lane calls it with the same tile): 32 candidate keys per
    // round, so <= 1024 keys take two dependent loads instead of log2(nkeys). On small
    // layouts this search was most of a warp's latency chain before its first tile.
    __device__ __forceinline__ void seek_warp(const KeyTab& kt, int64_t tile, int lane) {
        int lo = 0, hi = kt.nkeys - 1;  // toff[lo] <= tile; the answer is in [lo, hi]
        while (lo < hi) {
            const int step = (hi - lo + 32) / 32;
            const int cand = lo + lane * step < hi ? lo + lane * step : hi;
            const unsigned ok = __ballot_sync(0xffffffffu, __ldg(kt.toff + cand) <= tile);
            const int last = 31 - __clz(ok);  // lane 0 (cand == lo) always qualifies
            const int nlo = lo + last * step < hi ? lo + last * step : hi;
            const int nhi = lo + (last + 1) * step - 1 < hi ? lo + (last + 1) * step - 1 : hi;
            lo = nlo;
            hi = last == 31 ? hi : nhi;
        }
        load(kt, lo);
    }
    // Warp-collective forward move: the next key directly, or a seek for a longer jump
    // (dynamically scheduled warps jump ~2 tiles x #warps between claims: walking key by
    // key cost one dependent load per key — ~800 per claim on a 2,000-key layout).
    __device__ __forceinline__ void advance_warp(const KeyTab& kt, int64_t tile, int lane) {
        if (tile < t1) return;
        if (k + 2 > kt.nkeys || tile < __ldg(kt.toff + k + 2)) load(kt, k + 1);
        else seek_warp(kt, tile, lane);
    }
    __device__ __forceinline__ void advance_to(const KeyTab& kt, int64_t tile) {
        while (tile >= t1) load(kt, k + 1);
    }
    // Cursor over exactly tile `tile` from the per-tile table (kt.tiles != nullptr): t0 = tile,
    // t1 = tile + 1, so the element / word ranges are the tile's own (the key index is unused).
    __device__ __forceinline__ void from_table(const KeyTab& kt, int64_t tile) {
        const int4 d = __ldg(kt.tiles + tile);
        k = -1;
        t0 = tile;
        t1 = tile + 1;
        e0 = (static_cast<int64_t>(static_cast<uint32_t>(d.y)) << 32) | static_cast<uint32_t>(d.x);
        e1 = e0 + (d.w & 0xffff);
        w0 = d.z;
        w1 = w0 + (d.w >> 16);
    }
};

__device__ __forceinline__ void warp_range(int64_t ntiles, int64_t& b, int64_t& e) {
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    // one task per warp or fewer (launch-bound layouts): no 64-bit division in the prologue
    const int64_t per = ntiles <= nw ? 1 : (ntiles + nw - 1) / nw;
    b = wid * per;
    e = b + per < ntiles ? b + per : ntiles;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
    // error indices are the exception: one vote skips the 10-shuffle chain (it sat on every
    // warp's exit path, a visible share of a launch-bound round)
    if (!__any_sync(FULL, v != ~0ull)) return ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// CTA-wide sum of one double per thread into *dst with ONE atomic per CTA (every thread of
// the CTA must call it). Per-warp atomics on one address serialise at L2: ~2,400 of them
// per launch on small layouts, a visible share of a few-microsecond kernel.
__device__ __forceinline__ void block_atomic_add(double v, double* dst) {
    __shared__ double s_part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int warp = threadIdx.x >> 5, nwarp = (blockDim.x + 31) >> 5;
    __syncthreads();  // s_part may still be read by a previous call
    if ((threadIdx.x & 31) == 0) s_part[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = (threadIdx.x < nwarp) ? s_part[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
        if (threadIdx.x == 0 && t != 0.0) atomicAdd(dst, t);
    }
}
// The same for a grad-norm partial given as an integer count sum (the exact decode table:
// sum of cnt^2, times sq_scale = (alpha/N)^2) plus a double part that is zero on that path:
// the integer goes through one redux.sync per warp instead of a dependent chain of ten
// 64-bit shuffles + adds, and the double chain runs only in warps that hold a nonzero part.
// The CTA's value is gsq + isq * sq_scale with the integer summed exactly first.
__device__ __forceinline__ void block_atomic_add_counts(int isq, double gsq, double sq_scale, double* dst) {
    __shared__ double s_dpart[32];
    __shared__ unsigned s_ipart[32];
    const unsigned wi = __reduce_add_sync(FULL, static_cast<unsigned>(isq));
    if (__any_sync(FULL, gsq != 0.0)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gsq += __shfl_xor_sync(FULL, gsq, o);
    }
    const int warp = threadIdx.x >> 5, nwarp = (blockDim.x + 31) >> 5;
    __syncthreads();  // the parts may still be read by a previous call
    if ((threadIdx.x & 31) == 0) {
        s_ipart[warp] = wi;
        s_dpart[warp] = gsq;
    }
    __syncthreads();
    if (warp == 0) {
        double t = (threadIdx.x < nwarp) ? s_dpart[threadIdx.x] : 0.0;
        if (__any_sync(FULL, t != 0.0)) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
        }
        uint64_t ti = 0;  // 64-bit CTA total (per-warp sums are 32-bit)
        for (int w = 0; w < nwarp; ++w) ti += s_ipart[w];
        t += static_cast<double>(ti) * sq_scale;
        if (threadIdx.x == 0 && t != 0.0) atomicAdd(dst, t);
    }
}

// ================================================================ peer exchange (P2P over NVLink)
// Fused exchange protocol (see cdsgd_b200.cu, engine): K1 of round t stores every
// packed word straight into each peer's gathered slot (NVLink stores through
// symmetric-memory mappings) and the last CTA publishes ready[slot][me] = t+1 on
// every peer with a system-scope release; K2 acquires ready[slot][*] >= t+1 before
// reading and finally publishes freed[slot][me] = t+1 so producers may reuse the
// slot. Waits spin on LOCAL memory with a timeout: on expiry the kernel records
// EXCHANGE_TIMEOUT in err[1] and continues, so a lost peer can never hang the GPU.
constexpr uint64_t EXCHANGE_TIMEOUT = 0xFFFFFFFFFFFFFFFEull;
struct P2PArgs {
    uint32_t* dst[MAX_RANKS_P2P];       // per rank r: where my words land in r's slot (nullptr = none)
    uint64_t* publish[MAX_RANKS_P2P];   // per rank r: my flag cell in r's memory
    const uint64_t* wait_flags;         // local flags [nranks] to wait on (nullptr = no wait)
    uint64_t wait_value;
    uint64_t publish_value;
    unsigned int* counter;              // local grid-completion counter (0 between launches)
    uint64_t* err;                      // err[1] receives EXCHANGE_TIMEOUT
    int nranks;                         // 0: exchange disabled
    int sc_fence;                       // A/B knob: fence.sc.sys + relaxed counter instead of acq_rel
};

// Programmatic dependent launch (engine kernels are launched with programmatic stream
// serialization): a kernel may become resident while its stream predecessor drains, so
// every engine kernel calls pdl_wait() before its first memory access (a no-op without
// the attribute), then pdl_trigger() so its own successor's launch overlaps its body.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Grad-norm ring: the kernel accumulating round p zeroes the slots of rounds p+1 and p+2
// (two ahead covers the N=1 fold, which accumulates two rounds); stream order makes this
// race-free and removes a memset (and a PDL break) per round.
__device__ __forceinline__ void pdl_enter(double* clear0, double* clear1) {
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (clear0 != nullptr) *clear0 = 0.0;
        if (clear1 != nullptr) *clear1 = 0.0;
    }
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Release pattern for a batch of flags: ONE system-scope fence, then relaxed strong
// stores. (A st.release.sys per flag costs a fence each: 8 of them in the last CTA of a
// fused launch at N=4 measured ~13 us.)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Failure propagation: a rank whose error word is set (numeric error of any round, peer
// failure, timeout) publishes its flags with POISON set. Waiters treat a poisoned flag as
// arrived (no hang), record PEER_FAILED in their err[1] and skip the apply / quantize, so no
// replica applies stale or garbage codes after a rank failed — the reference aborts every
// worker at the failing round. cdsgd_engine_check reports it (CDSGD_ERR_PEER).
constexpr uint64_t POISON = 1ull << 62;
constexpr uint64_t PEER_FAILED = 0xFFFFFFFFFFFFFFFDull;

// Thread 0: wait until every wait_flags[r] >= wait_value (timeout -> EXCHANGE_TIMEOUT);
// returns true if some flag carries POISON.
__device__ __forceinline__ bool p2p_wait_t0(const P2PArgs& x, long long t0) {
    bool poisoned = false;
    if (x.nranks <= 0 || x.wait_flags == nullptr || x.wait_value == 0) return false;
    for (int r = 0; r < x.nranks; ++r) {
        uint64_t f;
        while ((f = ld_acquire_sys(x.wait_flags + r)) < x.wait_value) {
            __nanosleep(64);
            if (clock64() - t0 > (20ll << 30)) {  // ~10 s at 2 GHz
                if (x.err) atomicExch(reinterpret_cast<unsigned long long*>(x.err + 1), EXCHANGE_TIMEOUT);
                break;
            }
        }
        poisoned |= (f & POISON) != 0;
    }
    if (poisoned && x.err)
        atomicMin(reinterpret_cast<unsigned long long*>(x.err + 1), static_cast<unsigned long long>(PEER_FAILED));
    return poisoned;
}

// Block-wide wait; true (in every thread) if a peer published a poisoned flag.
__device__ __forceinline__ bool p2p_wait(const P2PArgs& x) {
    __shared__ int s_poison;
    if (!(x.nranks > 0 && x.wait_flags != nullptr && x.wait_value != 0)) return false;
    if (threadIdx.x == 0) s_poison = p2p_wait_t0(x, clock64()) ? 1 : 0;
    __syncthreads();
    return s_poison != 0;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_sys(unsigned int* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Thread 0 of each CTA, after a __syncthreads: count the CTA in on the grid-completion
// counter; true for the last CTA. The acq_rel system-scope atomic releases every write
// of the CTA (cumulative through the barrier), remote NVLink stores included, and the
// last CTA's atomic acquires all of them, so its st.release.sys flags publish the whole
// grid's output. (A full fence.sc.sys per CTA measured ~15 us slower per launch at N=4.)
__device__ __forceinline__ bool grid_arrive_last(unsigned int* counter, bool sc_fence) {
    unsigned prev;
    if (sc_fence) {
        __threadfence_system();
        prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) __threadfence_system();
    } else {
        prev = atom_add_acq_rel_sys(counter, 1u);
    }
    if (prev != gridDim.x - 1) return false;
    *counter = 0u;  // ready for the next launch (stream-ordered)
    return true;
}

// Value the last CTA publishes: POISON set if this rank has recorded any error (its own
// numeric error, reserved symbol, timeout or a peer failure) by the end of the launch.
__device__ __forceinline__ uint64_t publish_word(const P2PArgs& x) {
    if (x.err == nullptr) return x.publish_value;
    const volatile uint64_t* e = reinterpret_cast<const volatile uint64_t*>(x.err);
    return (e[0] != NO_ERR || e[1] != NO_ERR) ? (x.publish_value | POISON) : x.publish_value;
}

// Block-wide epilogue: the last CTA to finish publishes publish_value to every peer.
__device__ __forceinline__ void p2p_publish(const P2PArgs& x) {
    if (x.nranks <= 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (grid_arrive_last(x.counter, x.sc_fence != 0)) {
            fence_acq_rel_sys();
            const uint64_t v = publish_word(x);
            for (int r = 0; r < x.nranks; ++r)
                if (x.publish[r] != nullptr) st_relaxed_sys(x.publish[r], v);
        }
    }
}

// One barrier for both waits (each waits only if armed); true if a peer is poisoned.
__device__ __forceinline__ bool p2p_has_wait(const P2PArgs& x) {
    return x.nranks > 0 && x.wait_flags != nullptr && x.wait_value != 0;
}
__device__ __forceinline__ bool p2p_wait2(const P2PArgs& a, const P2PArgs& b) {
    __shared__ int s_poison2;
    // nothing to wait for (N = 1, local codes): no barrier on the launch's critical path
    if (!p2p_has_wait(a) && !p2p_has_wait(b)) return false;
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        const bool pa = p2p_wait_t0(a, t0);
        const bool pb = p2p_wait_t0(b, t0);
        s_poison2 = (pa || pb) ? 1 : 0;
    }
    __syncthreads();
    return s_poison2 != 0;
}

__device__ __forceinline__ void p2p_publish2(const P2PArgs& a, const P2PArgs& b, unsigned int* counter) {
    if (a.nranks <= 0 && b.nranks <= 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (grid_arrive_last(counter, (a.nranks > 0 ? a.sc_fence : b.sc_fence) != 0)) {
            const P2PArgs* xs[2] = {&a, &b};
            fence_acq_rel_sys();
            for (int i = 0; i < 2; ++i) {
                const uint64_t v = publish_word(*xs[i]);
                for (int r = 0; r < xs[i]->nranks; ++r)
                    if (xs[i]->publish[r] != nullptr) st_relaxed_sys(xs[i]->publish[r], v);
            }
        }
    }
}

// ================================================================ K1: quantize
// codec.quantize (codec.py:164-194) per key, fp64 exact:
//   acc = r + (double)g; plus = acc >= a; minus = acc <= -a;
//   r' = acc - (plus ? a : minus ? -a : 0.0); code 01/10/00.
template <typename G>
__device__ __forceinline__ uint32_t quant1(double r, G g, double alpha, double& rn, bool& bad) {
    const double acc = __dadd_rn(r, static_cast<double>(g));
    bad = nonfinite(acc);
    const bool p = acc >= alpha;
    const bool m = acc <= -alpha;
    const double em = p ? alpha : (m ? -alpha : 0.0);
    rn = __dsub_rn(acc, em);
    return p ? 1u : (m ? 2u : 0u);
}

// Lean form of quant1 for the staged fast path (same bits, fewer instructions):
//   nz = |acc| >= alpha  (== plus || minus for non-NaN acc)
//   r' = nz ? acc + s : acc,  s = -copysign(alpha, acc)   (x + (-y) == x - y exactly,
//        so this is acc - alpha on plus, acc - (-alpha) on minus; ties give +0.0 as
//        in the reference; acc = -0.0 passes through unchanged)
//   code = nz ? 1 + signbit(acc) : 0
// Non-finite accumulators only raise `bad` (the caller rescans for the index).
template <typename G>
__device__ __forceinline__ uint32_t quant1_lean(double r, G g, double alpha, uint32_t alpha_hi, uint32_t alpha_lo,
                                                double& rn, bool& bad) {
    const double acc = __dadd_rn(r, static_cast<double>(g));
    const double aa = fabs(acc);
    bad |= !(aa < __longlong_as_double(0x7ff0000000000000ll));
    const bool nz = aa >= alpha;
    const uint32_t ah = static_cast<uint32_t>(__double2hiint(acc));
    const double sg = __hiloint2double(static_cast<int>(alpha_hi | (~ah & 0x80000000u)), static_cast<int>(alpha_lo));
    const double t = __dadd_rn(acc, sg);
    rn = nz ? t : acc;
    return nz ? 1u + (ah >> 31) : 0u;
}

// fp32-residual FAST mode (opt-in; not the reference's arithmetic): the same operations
// restated in fp32 — acc = r + g, plus = acc >= a, minus = acc <= -a, r' = acc - emitted,
// all fp32 with a = (float)alpha — checked bitwise against the fp32 restatement oracle
// (oracle/cdsgd_oracle.py quantize_f32). 12.25 instead of 20.25 B/elem in the quantizer.
template <typename G>
__device__ __forceinline__ uint32_t quant1(float r, G g, double alpha, float& rn, bool& bad) {
    const float af = static_cast<float>(alpha);
    const float acc = __fadd_rn(r, static_cast<float>(g));
    bad = !(fabsf(acc) < __int_as_float(0x7f800000));
    const bool p = acc >= af;
    const bool m = acc <= -af;
    const float em = p ? af : (m ? -af : 0.0f);
    rn = __fsub_rn(acc, em);
    return p ? 1u : (m ? 2u : 0u);
}
template <typename G>
__device__ __forceinline__ uint32_t quant1_lean(float r, G g, double alpha, uint32_t, uint32_t, float& rn, bool& bad) {
    const float af = static_cast<float>(alpha);
    const float acc = __fadd_rn(r, static_cast<float>(g));
    const float aa = fabsf(acc);
    bad |= !(aa < __int_as_float(0x7f800000));
    const bool nz = aa >= af;
    const uint32_t ab = static_cast<uint32_t>(__float_as_int(acc));
    const float sg = __int_as_float(static_cast<int>(static_cast<uint32_t>(__float_as_int(af)) | (~ab & 0x80000000u)));
    const float t = __fadd_rn(acc, sg);
    rn = nz ? t : acc;
    return nz ? 1u + (ab >> 31) : 0u;
}
__device__ __forceinline__ bool nonfinite(float a) { return !(fabsf(a) < __int_as_float(0x7f800000)); }

// ================================================================ decode helpers
// Exact-alpha mode (the usual alpha = 0.5): every partial sum j*alpha, |j| <= N,
// is representable, so the ascending-worker fp64 sum of engine.py:250-253 equals
// cnt*alpha for cnt = #plus - #minus regardless of order. The host precomputes,
// in fp64 exactly as the reference does, tab[cnt + N] = (cnt*alpha)/N and the
// rounded fp32 update eta_g*mean; the kernel only counts codes (SWAR over
// 4-bit fields: even elements at bits 4i, odd at 4i+2 before the shift).
constexpr int MAX_RANKS = 16;
struct DecodeTab {
    double mean[2 * MAX_RANKS + 1];   // (cnt*alpha)/N
    float upd[2 * MAX_RANKS + 1];     // (float)(eta_g * mean)       fp32 weights
    double upd64[2 * MAX_RANKS + 1];  // eta_g * mean (fp64 product)  fp64 weights: the reference's exact update
    double sq_scale;                  // (alpha/N)^2: grad-norm metric from integer sum(cnt^2)
};

// ---------------------------------------------------------------- weight arithmetic
// The global weights W are fp64 (exact mode, default: the reference keeps every weight in
// fp64, numcore.py:95, SPEC "64-bit reals internally") or fp32 (fast mode). In fp64 every
// update is the reference's own operation sequence — W - eta*mean with the product rounded
// once (engine.py:511) — so W is bitwise the reference's on compressed rounds and whenever
// the round mean is exact (N = 1); the compute weights loc = fl32(W - eta_l*g) are the
// reference's fp64 local update (engine.py:268-274) rounded once to fp32. In fp32 W is
// rounded once per round (a random-walk drift).
// Compiler barrier on a value: it must be materialised here (keeps a load from being sunk
// into a later conditional block); no instruction is emitted.
__device__ __forceinline__ void pin(float& x) { asm volatile("" : "+f"(x)); }
__device__ __forceinline__ void pin(double& x) { asm volatile("" : "+d"(x)); }

template <typename TW> struct WV;  // 4 consecutive weights of one lane
template <> struct WV<float> { float v[4]; };
template <> struct WV<double> { double v[4]; };
__device__ __forceinline__ void ldw4(const float* p, int nv, WV<float>& w) {
    const float4 t = ld_stream_m(p, nv);
    w.v[0] = t.x; w.v[1] = t.y; w.v[2] = t.z; w.v[3] = t.w;
}
__device__ __forceinline__ void ldw4(const double* p, int nv, WV<double>& w) {
    const d4 t = ld_stream_m(p, nv);
    w.v[0] = t.x; w.v[1] = t.y; w.v[2] = t.z; w.v[3] = t.w;
}
template <typename TW>
__device__ __forceinline__ void stw4(TW* p, const WV<TW>& w, int nv) {
    st_stream_m(p, w.v[0], w.v[1], w.v[2], w.v[3], nv);
}
// W - eta*mean from the decode table (code count c = #plus - #minus, already offset by N)
__device__ __forceinline__ float w_sub_tab(float w, const float* u32, const double*, int c) {
    return __fsub_rn(w, u32[c]);
}
__device__ __forceinline__ double w_sub_tab(double w, const float*, const double* u64, int c) {
    return __dsub_rn(w, u64[c]);
}
// W - eta*mean for a general fp64 mean (non-exact alpha decode)
__device__ __forceinline__ float w_sub_mean(float w, double eta, double mean) {
    return __fsub_rn(w, __double2float_rn(__dmul_rn(eta, mean)));
}
__device__ __forceinline__ double w_sub_mean(double w, double eta, double mean) {
    return __dsub_rn(w, __dmul_rn(eta, mean));
}
// W - eta*(gsum/N): the full-precision (correction) branch, gsum the fp32 sum over ranks.
// fp32: one fma with (float)(eta/N); fp64: the reference's mean = sum/N, W - eta*mean
__device__ __forceinline__ float w_sub_full(float w, float s, float scale, double, double, int) {
    return __fmaf_rn(-scale, s, w);
}
__device__ __forceinline__ double w_sub_full(double w, float s, float, double eta, double inv_n_or_zero, int nr) {
    const double m = inv_n_or_zero != 0.0 ? __dmul_rn(static_cast<double>(s), inv_n_or_zero)
                                          : __ddiv_rn(static_cast<double>(s), static_cast<double>(nr));
    return __dsub_rn(w, __dmul_rn(eta, m));
}
// compute weights: W' - eta_l*g (engine.py:268-274), stored fp32
__device__ __forceinline__ float loc_of(float w, float g, float eta_l, double) { return __fmaf_rn(-eta_l, g, w); }
__device__ __forceinline__ float loc_of(double w, float g, float, double eta_l) {
    return __double2float_rn(__dsub_rn(w, __dmul_rn(eta_l, static_cast<double>(g))));
}

// Counts over ranks for the 16 codes of one word position: returns packed 4-bit
// plus/minus counters for even (field 4i) and odd (field 4i) elements, and a
// reserved-symbol mask (bit 2i set if code i of some rank is 11).
struct Counts {
    uint32_t pe, po, me, mo, rsv;
};
__device__ __forceinline__ void count_add(Counts& c, uint32_t w);
// The counters of lane `src` (a word's counts summed over ranks, see fused_vec_task)
__device__ __forceinline__ Counts shfl_counts(const Counts& w, int src) {
    return Counts{__shfl_sync(FULL, w.pe, src), __shfl_sync(FULL, w.po, src), __shfl_sync(FULL, w.me, src),
                  __shfl_sync(FULL, w.mo, src), __shfl_sync(FULL, w.rsv, src)};
}
__device__ __forceinline__ void count_add(Counts& c, uint32_t w) {
    c.pe += w & 0x11111111u;
    c.me += (w >> 1) & 0x11111111u;
    c.po += (w >> 2) & 0x11111111u;
    c.mo += (w >> 3) & 0x11111111u;
    c.rsv |= w & (w >> 1) & 0x55555555u;
}
// Signed counts of this lane's 4 code positions 4*(lane&3) .. +3 in one word:
// shift the SWAR counters once, then extract fields with constant shifts.
__device__ __forceinline__ void lane_counts(const Counts& c, int lane, int (&out)[4]) {
    const int sh = 8 * (lane & 3);
    const uint32_t pe = c.pe >> sh, me = c.me >> sh, po = c.po >> sh, mo = c.mo >> sh;
    out[0] = static_cast<int>(pe & 15u) - static_cast<int>(me & 15u);
    out[1] = static_cast<int>(po & 15u) - static_cast<int>(mo & 15u);
    out[2] = static_cast<int>((pe >> 4) & 15u) - static_cast<int>((me >> 4) & 15u);
    out[3] = static_cast<int>((po >> 4) & 15u) - static_cast<int>((mo >> 4) & 15u);
}
__device__ __forceinline__ double decode1(uint32_t code, double alpha) {
    return code == 1u ? alpha : (code == 2u ? -alpha : 0.0);
}

// Scatter of a correction round's gradient to the element owners (P2P exact mode):
// element e, owned by rank o = e / chunk, lands at base[o] + e, where base[o] is owner o's
// receive row for this rank shifted by -o*chunk. Each owner then reduces its shard from
// LOCAL memory (the NVLink transfer is fire-and-forget stores issued while the gradient
// streams through the kernel anyway, instead of latency-bound remote loads).
struct StageDst {
    float* base[MAX_RANKS_P2P];
    int64_t chunk;  // elements per owner, a multiple of 4; 0 = no staging
};
// Owner row of element e given the owner o0 of the tile start and the next boundary bnd.
__device__ __forceinline__ float* stage_at(const StageDst& s, int64_t e, int o0, int64_t bnd) {
    const int o = s.chunk >= TILE_ELEMS ? o0 + (e >= bnd ? 1 : 0) : static_cast<int>(e / s.chunk);
    return s.base[o] + e;
}

// ================================================================ K2: apply_quant
// Fused: decode N gathered payloads, ascending-rank fp64 sum / N (engine.py:249-255),
// W' = W - eta_g*mean (engine.py:511) on fp32 W, loc = W' - eta_l*g_next (Eq. 11,
// engine.py:385-392), optional sum(mean^2) (engine.py:521).
struct ApplyQArgs {
    void* W;  // float* or double* (the kernel's TW)
    const uint32_t* gathered;
    int64_t stride;  // words between ranks
    const float* gnext;
    float* loc;
    double alpha, inv_n_or_zero, eta_g_d, eta_l_d;  // inv_n_or_zero: 1/N if N is pow2 else 0
    float eta_l;
    int nranks;
    int exact;  // exact-alpha table mode
    uint64_t* err;
    uint64_t skip_below;
    double* gnorm;
    P2PArgs x;      // fused exchange: wait for peers' codes, then release the slot
    StageDst gs;    // chunk != 0: also scatter g_next to the element owners (P2P correction round)
    P2PArgs xs;     // staging protocol: wait gfreed, publish gready
    unsigned int* sched;  // [2] dynamic tile scheduler {next tile, CTAs done}; nullptr = static ranges
    // N=1, the round after this one is a correction whose mean is g_next itself: also apply
    // it here after the local update (W - eta_g*g_next), with its grad-norm into gnorm2.
    float fold_scale;   // fp32 weights: (float)eta_g
    int fold;           // 1: fold on
    double* gnorm2;
    double* gclear[2];  // grad-norm ring slots to zero (see pdl_enter), nullable
};

__device__ __forceinline__ double apply_mean_general(const uint32_t* codes, int nr, double alpha,
                                                     double inv_n, bool& rsv) {
    double tot = 0.0;
    for (int r = 0; r < nr; ++r) {
        const uint32_t c = codes[r];
        rsv |= c == 3u;
        const double d = decode1(c, alpha);
        tot = r == 0 ? d : __dadd_rn(tot, d);
    }
    return inv_n != 0.0 ? __dmul_rn(tot, inv_n) : __ddiv_rn(tot, static_cast<double>(nr));
}

// Write-only scratch for the stores of an aborted round on the branch-free small-layout
// paths (32 lanes x 32 bytes; concurrent garbage writes from every warp are harmless).
__device__ __align__(32) double g_sink[32 * 4];
template <typename T>
__device__ __forceinline__ T* sink_of(double* sink, int lane) {
    return reinterpret_cast<T*>(sink + 4 * lane);
}

// K2's operands of one task (registers), see apply_vec_load.
template <int NR, typename TW, int CH>
struct K2Regs {
    uint32_t wv[NR > 0 ? NR : 1];
    WV<TW> wt[CH];
    float4 gt[CH];
};
// K2 pointers held in registers from before the grid-dependency wait on small layouts
// (see HotPtrs in kernels_fused.cuh: parameter reloads after the wait were on every warp's
// path to its loads).
struct K2Hot {
    void* W;
    const uint32_t* gathered;
    const float* gnext;
    float* loc;
    double* sink;
    int p2p_wait;
    __device__ __forceinline__ explicit K2Hot(const ApplyQArgs& a)
        : W(a.W), gathered(a.gathered), gnext(a.gnext), loc(a.loc), sink(g_sink),
          p2p_wait(p2p_has_wait(a.x) || p2p_has_wait(a.xs) ? 1 : 0) {}
    __device__ __forceinline__ void pin_here() {
        asm volatile("" : "+l"(W), "+l"(gathered), "+l"(gnext), "+l"(loc), "+l"(sink), "+r"(p2p_wait));
    }
};

// K2 vector path for one task: CH chunks of 128 elements (from chunk c0) of a tile (exact-alpha
// table, compile-time rank count). Tiles of ne < TILE_ELEMS elements (a key's last) use masked
// accesses; padding codes are ignored.
template <int NR, typename TW, bool WHOLE, int CH>  // WHOLE: whole tile, unmasked accesses (see fused_vec_task)
__device__ __forceinline__ void apply_vec_load(const ApplyQArgs& a, const K2Hot& h, int lane, int64_t e0, int64_t w0,
                                               int ne, int nw, int c0, bool do_loc, K2Regs<NR, TW, CH>& L) {
    constexpr int R = NR > 0 ? NR : 1;
#pragma unroll
    for (int r = 0; r < R; ++r) L.wv[r] = lane < nw ? ld_word(h.gathered + r * a.stride + w0 + lane) : 0u;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int64_t e = e0 + 128 * (c0 + c) + 4 * lane;
        const int nv = WHOLE ? 4 : nvalid4(ne, 128 * (c0 + c) + 4 * lane);
        ldw4(static_cast<const TW*>(h.W) + e, nv, L.wt[c]);
        if (do_loc) L.gt[c] = ld_stream_m(h.gnext + e, nv);
    }
}
template <int NR, typename TW, bool WHOLE, int CH>
__device__ __forceinline__ void apply_vec_tile(const ApplyQArgs& a, const K2Hot& h, const float* s_upd,
                                               const double* s_upd64, int nr, int lane, int64_t e0, int64_t w0, int ne,
                                               int nw, int c0, bool do_loc, int so0, int64_t sbnd, bool a_off,
                                               int& isq, double& gsq2, uint64_t& bad_idx, K2Regs<NR, TW, CH>& L,
                                               bool loaded) {
    constexpr int R = NR > 0 ? NR : 1;
    constexpr bool SINK = CH == 1;  // small layouts: aborted rounds store to the sink (no branch, see fused_vec_task)
    TW* const W = static_cast<TW*>(h.W);
    if (CH != 1 || !loaded) apply_vec_load<NR, TW, WHOLE, CH>(a, h, lane, e0, w0, ne, nw, c0, do_loc, L);
    uint32_t(&wv)[R] = L.wv;
    WV<TW>(&wt)[CH] = L.wt;
    float4(&gt)[CH] = L.gt;
    const int a_on = a_off ? 0 : 1;
    Counts wc{0u, 0u, 0u, 0u, 0u};  // this lane's word, counts summed over the ranks (NR > 5)
    if constexpr (NR > 5) {
#pragma unroll
        for (int r = 0; r < R; ++r) count_add(wc, wv[r]);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int64_t e = e0 + 128 * (c0 + c) + 4 * lane;
        const int nv = WHOLE ? 4 : nvalid4(ne, 128 * (c0 + c) + 4 * lane);
        Counts cnt{0u, 0u, 0u, 0u, 0u};
        if constexpr (NR > 5) {  // (see fused_vec_task)
            cnt = shfl_counts(wc, 8 * (c0 + c) + (lane >> 2));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) count_add(cnt, __shfl_sync(FULL, wv[r], 8 * (c0 + c) + (lane >> 2)));
        }
        const int jb = 4 * (lane & 3);  // first code position of this lane in the word
        WV<TW>& w4 = wt[c];
        float g4[4];
        if (do_loc) { g4[0] = gt[c].x; g4[1] = gt[c].y; g4[2] = gt[c].z; g4[3] = gt[c].w; }
        float l4[4];
        int cq[4];
        lane_counts(cnt, lane, cq);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            w4.v[q] = w_sub_tab(w4.v[q], s_upd, s_upd64, cq[q] + nr);
            if (do_loc) l4[q] = loc_of(w4.v[q], g4[q], a.eta_l, a.eta_l_d);
            isq += a_on * cq[q] * cq[q];
            if (a.fold) {  // N=1 correction round t+1: W_{t+2} = W_{t+1} - eta*g_{t+1} (mean = g itself)
                w4.v[q] = w_sub_full(w4.v[q], g4[q], a.fold_scale, a.eta_g_d, 1.0, 1);
                const double m = static_cast<double>(g4[q]);
                if (!SINK || !a_off) gsq2 = __fma_rn(m, m, gsq2);  // (a two-chain tree measured 2 us slower)
            }
        }
        const uint32_t vm = nv >= 4 ? 0xffu : (1u << (2 * nv)) - 1u;  // padding codes are not checked
        if (!a_off && ((cnt.rsv >> (2 * jb)) & vm) != 0u) {
            const int q = __ffs((cnt.rsv >> (2 * jb)) & vm & 0x55u) / 2;
            const uint64_t idx = static_cast<uint64_t>(e + q);
            bad_idx = idx < bad_idx ? idx : bad_idx;
        }
        if (nv > 0) {
            stw4(SINK && a_off ? sink_of<TW>(h.sink, lane) : W + e, w4, nv);
            if (do_loc)
                st_stream_m(SINK && a_off ? sink_of<float>(h.sink, lane) : h.loc + e, l4[0], l4[1], l4[2], l4[3], nv);
            if (a.gs.chunk != 0 && !a_off) st_stream_m(stage_at(a.gs, e, so0, sbnd), g4[0], g4[1], g4[2], g4[3], nv);
        }
    }
}

// NR > 0: compile-time rank count; NR == 0: runtime (generic).
// 3 CTAs per SM at N=1 (80 registers, a 24-byte spill): 88 -> 82 us at ResNet-50 size, the
// extra warps keep more loads in flight; more ranks spill more, so they keep 2.
// WIDE = 1: one 512-thread CTA per SM (the same 16 warps and register budget as 2 x 256), so
// a grid of (SMs - R) CTAs leaves R whole SMs free — launched beside a correction all-reduce,
// whose NCCL CTAs (104 KB smem, 52K registers each) cannot share an SM with this kernel.
// CH = chunks of 128 elements per task: 4 (a whole tile) for large layouts, 1 for small ones
// (4x the warps in flight; the first task's loads issued straight after the wait, as in
// k_fused_ldg).
#ifndef CDSGD_K2_MINB
#define CDSGD_K2_MINB (NR == 1 && sizeof(TW) == 4 ? 3 : 2)
#endif
template <int NR, int WIDE = 0, typename TW = float, int CH = CHUNKS>
__global__ void __launch_bounds__(WIDE ? 512 : 256, WIDE ? 1 : CDSGD_K2_MINB) k_apply_quant(ApplyQArgs a, KeyTab kt, DecodeTab tab) {
    constexpr int SPL = CHUNKS / CH;  // tasks per tile
    __shared__ double s_mean[2 * MAX_RANKS + 1];
    __shared__ double s_upd64[2 * MAX_RANKS + 1];
    __shared__ float s_upd[2 * MAX_RANKS + 1];
    TW* const W = static_cast<TW*>(a.W);
    const int nr = NR > 0 ? NR : a.nranks;
    if (threadIdx.x < 2 * nr + 1) {
        s_mean[threadIdx.x] = tab.mean[threadIdx.x];
        s_upd[threadIdx.x] = tab.upd[threadIdx.x];
        s_upd64[threadIdx.x] = tab.upd64[threadIdx.x];
    }
    const int64_t ntasks = kt.ntiles * SPL;
    int64_t tb, te;
    warp_range(ntasks, tb, te);
    const int lane = threadIdx.x & 31;
    double gsq = 0.0, gsq2 = 0.0;
    int isq = 0;  // sum of cnt^2 on the table path: gsq += isq * (alpha/N)^2
    uint64_t bad_idx = NO_ERR;
    const bool do_loc = a.loc != nullptr;
    // small layouts (fewer than ~4 tasks per warp): claim single tasks for parallelism
    const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
    const unsigned CLAIM = ntasks < 4 * nwarps ? 1u : 2u;
    const int64_t tail_from = ntasks - nwarps;  // single-task claims from here on
    // one wave of tasks (small layouts): each warp takes its own, no ticket and no end-of-launch
    // ticket reset (a fence + atomic per CTA on one counter)
    bool dyn = a.sched != nullptr && ntasks > nwarps * static_cast<int64_t>(CLAIM);
    int64_t cend = 0;
    const int64_t first_dyn = nwarps * CLAIM;  // first claim static, then tickets (see k_fused_ldg)
    if (dyn) {
        tb = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * CLAIM;
        cend = tb + (int64_t)CLAIM < ntasks ? tb + (int64_t)CLAIM : ntasks;
        te = tb < ntasks ? ntasks : tb;
    }
    // constant inputs (tables, schedule, key seek) before griddepcontrol.wait (see k_fused_ldg)
    TileCursor kc;
    if (tb < te) {
        if (kt.tiles != nullptr) kc.from_table(kt, tb / SPL);
        else kc.seek_warp(kt, tb / SPL, lane);
    }
    struct TaskDesc {
        int64_t e0, w0;
        int ne, nw, c0;
        bool fast;
    };
    auto describe = [&](int64_t task) {
        TaskDesc d;
        const int64_t ti = task / SPL;
        d.c0 = static_cast<int>(task % SPL) * CH;
        if (kt.tiles != nullptr) kc.from_table(kt, ti);
        else kc.advance_warp(kt, ti, lane);
        const int64_t j = ti - kc.t0;
        d.e0 = kc.e0 + j * TILE_ELEMS;
        d.w0 = kc.w0 + j * TILE_WORDS;
        const int64_t ne64 = kc.e1 - d.e0;
        d.ne = ne64 < TILE_ELEMS ? static_cast<int>(ne64) : TILE_ELEMS;
        const int64_t nw64 = kc.w1 - d.w0;
        d.nw = nw64 < TILE_WORDS ? static_cast<int>(nw64) : TILE_WORDS;
        d.fast = NR > 0 && a.exact && aligned_to(W + d.e0, 4 * sizeof(TW)) &&
                 (!do_loc || (aligned_to(a.gnext + d.e0, 16) && aligned_to(a.loc + d.e0, 16)));
        return d;
    };
    TaskDesc td{};
    if (CH == 1 && tb < te) td = describe(tb);
    K2Hot hot(a);
    if constexpr (CH == 1) {
        hot.pin_here();
        int d = dyn ? 1 : 0;
        asm volatile("" : "+r"(d));
        dyn = d != 0;
    }
    if constexpr (CH == 1) __syncthreads();  // s_mean / s_upd, before the wait
    pdl_enter(a.gclear[0], a.gclear[1]);
    K2Regs<NR, TW, CH> L;
    bool pre = false;
    if constexpr (CH == 1) {  // first task's loads right after the wait (not behind a peer-flag wait)
        pre = tb < te && td.fast && !hot.p2p_wait;
        if (pre) {
            if (td.ne == TILE_ELEMS)
                apply_vec_load<NR, TW, true, CH>(a, hot, lane, td.e0, td.w0, td.ne, td.nw, td.c0, do_loc, L);
            else
                apply_vec_load<NR, TW, false, CH>(a, hot, lane, td.e0, td.w0, td.ne, td.nw, td.c0, do_loc, L);
        }
    }
    const bool peer_failed = (CH != 1 || hot.p2p_wait) && p2p_wait2(a.x, a.xs);
    bool skip;
    if constexpr (CH == 1) {  // error word read after the loads went out (weak load, see RoundFlags)
        uint64_t e0v = ~0ull;
        if (a.err != nullptr) asm volatile("ld.global.u64 %0, [%1];" : "=l"(e0v) : "l"(a.err) : "memory");
        skip = peer_failed || e0v < a.skip_below;
    } else {
        skip = peer_failed || (a.err != nullptr && *reinterpret_cast<volatile uint64_t*>(a.err) < a.skip_below);
        __syncthreads();
    }
    if (tb < te && (CH == 1 || !skip)) {
        for (int64_t task = tb; task < te; ++task) {
            if (dyn && task >= cend) {
                const unsigned cl = task < tail_from ? CLAIM : 1u;
                unsigned t0 = 0;
                if (lane == 0) t0 = atomicAdd(a.sched, cl);
                const int64_t nb = first_dyn + static_cast<int64_t>(__shfl_sync(FULL, t0, 0));
                if (nb >= ntasks) break;
                task = nb;
                cend = nb + (int64_t)cl < ntasks ? nb + (int64_t)cl : ntasks;
            }
            if (CH != 1 || task != tb) td = describe(task);
            const int64_t e0 = td.e0, w0 = td.w0;
            const int ne = td.ne, nw = td.nw, c0 = td.c0;
            const bool fast = td.fast;
            if (!fast && c0 != 0) continue;  // misaligned tiles: one task does the whole tile
            int so0 = 0;
            int64_t sbnd = 0;
            if (a.gs.chunk != 0) {
                so0 = static_cast<int>(e0 / a.gs.chunk);
                sbnd = (so0 + 1) * a.gs.chunk;
            }
            const bool a_off = CH == 1 && skip;  // (large layouts: the loop only runs when !skip)
            if (fast) {
                const bool loaded = pre && task == tb;
                if (ne == TILE_ELEMS)
                    apply_vec_tile<NR, TW, true, CH>(a, hot, s_upd, s_upd64, nr, lane, e0, w0, ne, nw, c0, do_loc, so0,
                                                     sbnd, a_off, isq, gsq2, bad_idx, L, loaded);
                else
                    apply_vec_tile<NR, TW, false, CH>(a, hot, s_upd, s_upd64, nr, lane, e0, w0, ne, nw, c0, do_loc, so0,
                                                      sbnd, a_off, isq, gsq2, bad_idx, L, loaded);
            } else if (!a_off) {
                // generic path: lane l owns element 32s + l; word (2s + l/16), code l%16
                uint32_t wv[MAX_RANKS];
                const bool wl = lane < nw;
                for (int r = 0; r < nr; ++r) wv[r] = wl ? a.gathered[r * a.stride + w0 + lane] : 0u;
#pragma unroll 2
                for (int s = 0; s < TILE_ELEMS / 32; ++s) {
                    const int el = 32 * s + lane;
                    uint32_t codes[MAX_RANKS];
                    for (int r = 0; r < nr; ++r)
                        codes[r] = (__shfl_sync(FULL, wv[r], 2 * s + (lane >> 4)) >> (2 * (lane & 15))) & 3u;
                    if (el < ne) {
                        const int64_t e = e0 + el;
                        bool rsv = false;
                        double mean;
                        TW wn;
                        if (a.exact) {
                            int cn = 0;
                            for (int r = 0; r < nr; ++r) {
                                rsv |= codes[r] == 3u;
                                cn += (codes[r] == 1u) - (codes[r] == 2u);
                            }
                            mean = s_mean[cn + nr];
                            wn = w_sub_tab(W[e], s_upd, s_upd64, cn + nr);
                        } else {
                            mean = apply_mean_general(codes, nr, a.alpha, a.inv_n_or_zero, rsv);
                            wn = w_sub_mean(W[e], a.eta_g_d, mean);
                        }
                        if (do_loc) a.loc[e] = loc_of(wn, a.gnext[e], a.eta_l, a.eta_l_d);
                        if (a.fold) {
                            const float gn = a.gnext[e];
                            wn = w_sub_full(wn, gn, a.fold_scale, a.eta_g_d, 1.0, 1);
                            gsq2 = __fma_rn(static_cast<double>(gn), static_cast<double>(gn), gsq2);
                        }
                        W[e] = wn;
                        if (a.gs.chunk != 0) *stage_at(a.gs, e, so0, sbnd) = a.gnext[e];
                        if (a.gnorm != nullptr) gsq = __fma_rn(mean, mean, gsq);
                        if (rsv) bad_idx = static_cast<uint64_t>(e) < bad_idx ? static_cast<uint64_t>(e) : bad_idx;
                    }
                }
            }
        }
    }
    if (a.gnorm != nullptr) block_atomic_add_counts(isq, gsq, tab.sq_scale, a.gnorm);
    if (a.gnorm2 != nullptr) block_atomic_add(gsq2, a.gnorm2);
    if (a.err != nullptr) {
        bad_idx = warp_min_u64(bad_idx);
        if (lane == 0 && bad_idx != NO_ERR)
            atomicMin(reinterpret_cast<unsigned long long*>(a.err + 1), static_cast<unsigned long long>(bad_idx));
    }
    if (dyn) {  // last CTA out resets the ticket (skipped CTAs still count)
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
    p2p_publish2(a.x, a.xs, a.x.counter != nullptr ? a.x.counter : a.xs.counter);
}

// ================================================================ dequantize / aggregate
// codec.dequantize (n = 1) and server_aggregate's quantized branch: fp64 out.
__global__ void __launch_bounds__(256) k_dequant_sum(const uint32_t* __restrict__ words, int nr,
                                                     int64_t stride, KeyTab kt, double alpha,
                                                     double* __restrict__ out, uint64_t* err) {
    int64_t tb, te;
    warp_range(kt.ntiles, tb, te);
    if (tb >= te) return;
    const int lane = threadIdx.x & 31;
    const double inv_n = (nr & (nr - 1)) == 0 ? 1.0 / nr : 0.0;
    TileCursor kc;
    kc.seek(kt, tb);
    uint64_t bad_idx = NO_ERR;
    for (int64_t ti = tb; ti < te; ++ti) {
        kc.advance_to(kt, ti);
        const int64_t j = ti - kc.t0;
        const int64_t e0 = kc.e0 + j * TILE_ELEMS;
        const int64_t w0 = kc.w0 + j * TILE_WORDS;
        const int64_t ne64 = kc.e1 - e0;
        const int ne = ne64 < TILE_ELEMS ? static_cast<int>(ne64) : TILE_ELEMS;
        const int64_t nw64 = kc.w1 - w0;
        const int nw = nw64 < TILE_WORDS ? static_cast<int>(nw64) : TILE_WORDS;
        for (int s = 0; s < TILE_ELEMS / 32; ++s) {
            const int el = 32 * s + lane;
            const int wi = 2 * s + (lane >> 4);
            if (el < ne && wi < nw) {
                double tot = 0.0;
                bool rsv = false;
                for (int r = 0; r < nr; ++r) {
                    const uint32_t c = (words[r * stride + w0 + wi] >> (2 * (lane & 15))) & 3u;
                    rsv |= c == 3u;
                    const double d = decode1(c, alpha);
                    tot = r == 0 ? d : __dadd_rn(tot, d);
                }
                out[e0 + el] = inv_n != 0.0 ? __dmul_rn(tot, inv_n) : __ddiv_rn(tot, static_cast<double>(nr));
                if (rsv) bad_idx = static_cast<uint64_t>(e0 + el) < bad_idx ? static_cast<uint64_t>(e0 + el) : bad_idx;
            }
        }
    }
    if (err != nullptr) {
        bad_idx = warp_min_u64(bad_idx);
        if (lane == 0 && bad_idx != NO_ERR)
            atomicMin(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(bad_idx));
    }
}

template <typename G>
__global__ void k_aggregate_full(const G* __restrict__ grads, int nc, int64_t stride, int64_t n,
                                 double* __restrict__ out) {
    const double inv_n = (nc & (nc - 1)) == 0 ? 1.0 / nc : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double tot = static_cast<double>(grads[i]);
        for (int c = 1; c < nc; ++c) tot = __dadd_rn(tot, static_cast<double>(grads[c * stride + i]));
        out[i] = inv_n != 0.0 ? __dmul_rn(tot, inv_n) : __ddiv_rn(tot, static_cast<double>(nc));
    }
}

// ================================================================ pack / unpack
__global__ void k_pack(const uint8_t* __restrict__ sym, int64_t n, uint32_t* __restrict__ words,
                       uint64_t* err) {
    const int64_t nw = (n + 15) / 16;
    uint64_t bad_idx = NO_ERR;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int j = 0; j < 16; ++j) {
            const int64_t i = 16 * w + j;
            if (i < n) {
                const uint32_t s = sym[i];
                if (s > 2u && static_cast<uint64_t>(i) < bad_idx) bad_idx = static_cast<uint64_t>(i);
                v |= (s & 3u) << (2 * j);
            }
        }
        words[w] = v;
    }
    if (err != nullptr && bad_idx != NO_ERR)
        atomicMin(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(bad_idx));
}

__global__ void k_unpack(const uint32_t* __restrict__ words, int64_t length, uint8_t* __restrict__ sym) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < length; i += (int64_t)gridDim.x * blockDim.x)
        sym[i] = static_cast<uint8_t>((words[i >> 4] >> (2 * (i & 15))) & 3u);
}

// ================================================================ K3: apply_full + elementwise
// Correction round: W' = W - (eta_g/N)*gsum ; loc = W' - eta_l*g_next.
struct ApplyFArgs {
    void* W;  // float* or double*
    const float* gsum;
    const float* gnext;
    float* loc;
    float scale;   // (float)(eta_g / N)   fp32 weights
    float eta_l;
    double inv_n;  // for the grad-norm metric
    double eta_g_d, eta_l_d, inv_n_or_zero;  // fp64 weights: mean = gsum/N, W - eta*mean
    int nranks;
    int64_t n;
    const uint64_t* err;
    uint64_t skip_below;
    double* gnorm;
    double* gclear[2];
};

// engine.global_update / local_update with fp64 math (exact reference arithmetic
// for fp64 operands; one rounding to the output type otherwise).
template <typename T> __device__ __forceinline__ double to_d(T v) { return static_cast<double>(v); }
template <typename T> __device__ __forceinline__ T from_d(double v);
template <> __device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double from_d<double>(double v) { return v; }

template <typename TW, typename TM>
__global__ void k_global_update(TW* __restrict__ w, const TM* __restrict__ mean, int64_t n, double eta) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        w[i] = from_d<TW>(__dsub_rn(to_d(w[i]), __dmul_rn(eta, to_d(mean[i]))));
}

template <typename TB, typename TG, typename TO>
__global__ void k_local_update(const TB* __restrict__ base, const TG* __restrict__ g, TO* __restrict__ out,
                               int64_t n, double eta_l) {
    pdl_enter(nullptr, nullptr);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = from_d<TO>(__dsub_rn(to_d(base[i]), __dmul_rn(eta_l, to_d(g[i]))));
}

}  // namespace cdsgd
