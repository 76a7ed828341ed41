// kernels_corr.cuh — correction rounds over NVLink without NCCL (fused exchange mode).
//
// Reference semantics (engine.py:252, 255, 511): the k-th round pushes full-precision
// gradients, the server sums them in ascending worker id in fp64, divides by N and
// applies W -= eta * mean. Here, with every rank holding a W replica in symmetric
// memory and owning one shard [o*chunk, (o+1)*chunk) of the elements:
//   stage     (round t)   g_t -> my staging slot (pull, default), or each element into its
//             OWNER's receive row [my rank] (push: NVLink stores); fused into K2, which
//             streams g_t anyway, or k_stage; release gready[slot][me] = t+1 everywhere
//   k_reduce  (round t+1) for MY shard: acquire all gready, read the N ranks' values
//             (pull: remote loads; push: local rows), fp64 ascending-rank sum, / N (the
//             reference's arithmetic), W' = W - eta*mean rounded once to fp32, store W'
//             into EVERY rank's W replica (NVLink stores); publish gfreed (stages
//             reusable), the shard's sum(mean^2) and wdone[me] = t+1
//   k_wait_sum            acquire all wdone (W' complete everywhere), grad-norm total
// Per rank this moves 2(N-1)/N * 4n bytes each way over NVLink (a ring all-reduce's
// volume) but nothing through intermediate HBM FIFOs and no NCCL kernels. The sum is
// bitwise the reference's, and W replicas stay identical because each shard's W' is
// computed once and broadcast.
#pragma once
#include "kernels.cuh"

namespace cdsgd {

struct StageArgs {
    const float* g;
    StageDst gs;  // owners' receive rows (kernels.cuh)
    int64_t n;
    P2PArgs x;  // wait: gfreed[slot][*] (previous use released); publish: gready[slot][me]
};

__global__ void __launch_bounds__(256) k_stage(StageArgs a) {
    pdl_enter(nullptr, nullptr);
    p2p_wait(a.x);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const bool vec = aligned_to(a.g, 16);
    int64_t done = 0;
    if (vec) {  // chunk is a multiple of 4: a float4 never straddles two owners
        const int64_t nv = a.n / 4;
        for (int64_t i = tid; i < nv; i += nth) {
            const float4 v = ld_stream(a.g + 4 * i);
            st_stream(a.gs.base[(4 * i) / a.gs.chunk] + 4 * i, v.x, v.y, v.z, v.w);
        }
        done = nv * 4;
    }
    for (int64_t i = done + tid; i < a.n; i += nth) a.gs.base[i / a.gs.chunk][i] = a.g[i];
    p2p_publish(a.x);
}

struct ReduceArgs {
    const float* stage[MAX_RANKS_P2P];  // rank r's staged g, indexed by element (mapped or local row)
    void* Wdst[MAX_RANKS_P2P];          // rank r's W replica (mapped; TW), or gsum (SUM mode, fp32)
    const void* W;                      // my W replica (read; TW)
    int64_t s0, s1;                     // my shard [s0, s1)
    int nranks;
    double eta_g;
    double inv_n;                       // 1/N when N is a power of two, else 0 (divide)
    double* gacc;                       // local accumulator of sum(mean^2) (0 between launches)
    double* gpart_dst[MAX_RANKS_P2P];   // rank r's gpart[me]
    P2PArgs xa;                         // wait: gready[slot][*] >= t+1; publish: gfreed[slot][me]
    P2PArgs xb;                         // publish: wdone[me]
    int ndst;                           // destinations written: Wdst[0, ndst) (0 = all NR)
};

template <typename TW> __device__ __forceinline__ TW round_w(double v);
template <> __device__ __forceinline__ float round_w<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double round_w<double>(double v) { return v; }

template <int NR, typename TW>
__device__ __forceinline__ TW reduce_apply1(const float (&g)[NR], TW w, double eta, double inv_n, double& msq) {
    double tot = static_cast<double>(g[0]);
#pragma unroll
    for (int r = 1; r < NR; ++r) tot = __dadd_rn(tot, static_cast<double>(g[r]));   // engine.py:250-253
    const double mean = inv_n != 0.0 ? __dmul_rn(tot, inv_n) : __ddiv_rn(tot, static_cast<double>(NR));
    msq = __fma_rn(mean, mean, msq);
    return round_w<TW>(__dsub_rn(static_cast<double>(w), __dmul_rn(eta, mean)));  // engine.py:511
}

// SUM mode (p2p exchange's NCCL-free correction all-reduce): the shard's fp64 ascending
// sum rounded once to fp32 is stored into every rank's gsum (Wdst), W is not touched and
// K3 applies it after K2 in stream order — a deterministic all-reduce whose result is
// bitwise equal on all ranks and at least as accurate as a fp32 ring sum.
template <int NR>
__device__ __forceinline__ float sum1(const float (&g)[NR]) {
    double tot = static_cast<double>(g[0]);
#pragma unroll
    for (int r = 1; r < NR; ++r) tot = __dadd_rn(tot, static_cast<double>(g[r]));
    return __double2float_rn(tot);
}

template <int NR, bool SUM = false, typename TW = float>  // TW: W element type (SUM: fp32 gsum)
__global__ void __launch_bounds__(256) k_reduce(ReduceArgs a) {
    pdl_enter(nullptr, nullptr);
    p2p_wait(a.xa);
    const TW* const Wl = static_cast<const TW*>(a.W);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t len = a.s1 - a.s0;
    const int nd = a.ndst > 0 ? a.ndst : NR;
    double msq = 0.0;
    bool vec = SUM || aligned_to(Wl + a.s0, 4 * sizeof(TW));
#pragma unroll
    for (int r = 0; r < NR; ++r)
        vec = vec && aligned_to(a.stage[r] + a.s0, 16) &&
              aligned_to(static_cast<TW*>(a.Wdst[r < nd ? r : 0]) + a.s0, 4 * sizeof(TW));
    // one 4-element group at element e from the loaded stage values and (non-SUM) weights
    auto group = [&](int64_t e, const float4 (&gv)[NR], const WV<TW>& wv) {
        float g0[NR], g1[NR], g2[NR], g3[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) { g0[r] = gv[r].x; g1[r] = gv[r].y; g2[r] = gv[r].z; g3[r] = gv[r].w; }
        WV<TW> o;
        if constexpr (SUM) {
            o.v[0] = sum1<NR>(g0); o.v[1] = sum1<NR>(g1); o.v[2] = sum1<NR>(g2); o.v[3] = sum1<NR>(g3);
        } else {
            o.v[0] = reduce_apply1<NR, TW>(g0, wv.v[0], a.eta_g, a.inv_n, msq);
            o.v[1] = reduce_apply1<NR, TW>(g1, wv.v[1], a.eta_g, a.inv_n, msq);
            o.v[2] = reduce_apply1<NR, TW>(g2, wv.v[2], a.eta_g, a.inv_n, msq);
            o.v[3] = reduce_apply1<NR, TW>(g3, wv.v[3], a.eta_g, a.inv_n, msq);
        }
#pragma unroll
        for (int r = 0; r < NR; ++r)  // NVLink stores (every rank's replica / gsum)
            if (r < nd) stw4(static_cast<TW*>(a.Wdst[r]) + e, o, 4);
    };
    int64_t done = 0;
    if (vec) {
        // U float4 positions per thread per iteration, every (remote) load issued before any use
        constexpr int U = NR <= 4 ? 4 : 2;
        const int64_t nv = len / 4;
        int64_t i = tid;
        for (; i + (U - 1) * nth < nv; i += U * nth) {
            float4 gv[U][NR];
            WV<TW> wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t e = a.s0 + 4 * (i + u * nth);
#pragma unroll
                for (int r = 0; r < NR; ++r) gv[u][r] = ld_stream(a.stage[r] + e);  // pull: NVLink loads
                if constexpr (!SUM) ldw4(Wl + e, 4, wv[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) group(a.s0 + 4 * (i + u * nth), gv[u], wv[u]);
        }
        for (; i < nv; i += nth) {
            const int64_t e = a.s0 + 4 * i;
            float4 gv[NR];
            WV<TW> wv;
#pragma unroll
            for (int r = 0; r < NR; ++r) gv[r] = ld_stream(a.stage[r] + e);
            if constexpr (!SUM) ldw4(Wl + e, 4, wv);
            group(e, gv, wv);
        }
        done = 4 * nv;
    }
    for (int64_t i = done + tid; i < len; i += nth) {
        const int64_t e = a.s0 + i;
        float g[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) g[r] = a.stage[r][e];
        TW o;
        if constexpr (SUM) o = sum1<NR>(g);
        else o = reduce_apply1<NR, TW>(g, Wl[e], a.eta_g, a.inv_n, msq);
#pragma unroll
        for (int r = 0; r < NR; ++r)
            if (r < nd) static_cast<TW*>(a.Wdst[r])[e] = o;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) msq += __shfl_xor_sync(FULL, msq, o);
    if (!SUM && (threadIdx.x & 31) == 0 && msq != 0.0) atomicAdd(a.gacc, msq);
    // last CTA: broadcast the shard's sum(mean^2), then release gfreed and wdone
    __syncthreads();
    if (threadIdx.x == 0) {
        if (grid_arrive_last(a.xa.counter, a.xa.sc_fence != 0)) {
            if (!SUM) {
                const double total = *reinterpret_cast<volatile double*>(a.gacc);
                *reinterpret_cast<volatile double*>(a.gacc) = 0.0;  // ready for the next correction round
                for (int r = 0; r < a.nranks; ++r) *reinterpret_cast<volatile double*>(a.gpart_dst[r]) = total;
            }
            fence_acq_rel_sys();  // orders the gpart stores too
            for (int r = 0; r < a.nranks; ++r) {
                if (a.xa.publish[r] != nullptr) st_relaxed_sys(a.xa.publish[r], a.xa.publish_value);
                if (a.xb.publish[r] != nullptr) st_relaxed_sys(a.xb.publish[r], a.xb.publish_value);
            }
        }
    }
}

// Empty kernel: a stream-ordered marker (CDSGD_AR_FIRST gate before the correction all-reduce).
__global__ void k_noop() {}

// One thread: release publish_value to every rank's flag cell after everything earlier on
// this stream (copy-engine transfers included) has completed.
__global__ void k_flags(P2PArgs x) {
    if (threadIdx.x == 0) {
        fence_acq_rel_sys();
        for (int r = 0; r < x.nranks; ++r)
            if (x.publish[r] != nullptr) st_relaxed_sys(x.publish[r], x.publish_value);
    }
}

// One thread: acquire flags (W' shards of every rank have landed), then optionally
// total the per-shard sum(mean^2) into the round's grad-norm slot.
__global__ void k_wait_sum(P2PArgs x, const double* gpart, int n, double* out, double* clear0, double* clear1) {
    pdl_enter(clear0, clear1);
    p2p_wait(x);
    if (threadIdx.x == 0 && out != nullptr) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += *reinterpret_cast<const volatile double*>(gpart + r);
        *out = s;
    }
}

}  // namespace cdsgd
