// cdsgd_b200.cu — C ABI, launch logic, NCCL exchange and the per-rank step
// engine of the B200-native CD-SGD hot path. Declarations and the reference
// interface each entry point replaces: include/cdsgd_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: a no-op unless a profiler is attached

#include "cdsgd_b200.h"
#include "kernels.cuh"
#include "kernels_tma.cuh"
#include "kernels_fused.cuh"
#include "kernels_corr.cuh"

using namespace cdsgd;

// ------------------------------------------------------------------ errors
namespace {
thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
}  // namespace

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess) return fail(CDSGD_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)
#define NCCL_TRY(expr)                                                                   \
    do {                                                                                 \
        ncclResult_t r_ = (expr);                                                        \
        if (r_ != ncclSuccess) return fail(CDSGD_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
    } while (0)
#define LAUNCH_CHECK()                                                                   \
    do {                                                                                 \
        g_launches.fetch_add(1, std::memory_order_relaxed);                              \
        cudaError_t e_ = cudaGetLastError();                                             \
        if (e_ != cudaSuccess) return fail(CDSGD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------------ device facts
namespace {
struct DeviceInfo {
    int sms = 0;
};
DeviceInfo& dev_info() {
    static thread_local DeviceInfo cache[16];
    int d = 0;
    cudaGetDevice(&d);
    DeviceInfo& di = cache[d & 15];
    if (di.sms == 0) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, d);
        if (di.sms <= 0) di.sms = 148;
    }
    return di;
}
// Resident CTAs of a kernel, cached per (kernel, block size, device): the occupancy query
// is a driver call, and launch-bound layouts (ResNet-20) pay for every host microsecond.
template <typename K>
int resident_blocks(K kernel, int threads) {
    struct Entry { const void* k; int threads, dev, blocks; };
    static thread_local Entry cache[64];
    static thread_local int used = 0;
    int d = 0;
    cudaGetDevice(&d);
    for (int i = 0; i < used; ++i)
        if (cache[i].k == reinterpret_cast<const void*>(kernel) && cache[i].threads == threads && cache[i].dev == d)
            return cache[i].blocks;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int blocks = per_sm * dev_info().sms;
    if (used < 64) cache[used++] = Entry{reinterpret_cast<const void*>(kernel), threads, d, blocks};
    return blocks;
}
constexpr int THREADS = 256;
constexpr int WARPS_PER_BLOCK = THREADS / 32;

template <typename K>
int tile_grid(K kernel, int64_t ntiles) {
    const int64_t want = (ntiles + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    const int64_t cap = resident_blocks(kernel, THREADS);
    return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}
template <typename K>
int flat_grid(K kernel, int64_t work) {
    const int64_t want = (work + THREADS - 1) / THREADS;
    const int64_t cap = resident_blocks(kernel, THREADS);
    return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Engine-path kernels are launched with programmatic stream serialization: the next
// round's grid is scheduled while this one drains and blocks in pdl_enter() until it has
// completed (kernels.cuh). CDSGD_NO_PDL=1 launches them plainly (A/B knob).
bool pdl_on() {
    static const bool v = [] {
        const char* e = getenv("CDSGD_NO_PDL");
        return !(e != nullptr && e[0] == '1');
    }();
    return v;
}
// Set while enqueueing an apply right after a correction all-reduce was issued on the
// exchange stream: a PDL launch would make the apply's CTAs resident (spinning in
// griddepcontrol.wait) while the previous kernel drains, so they hold every SM when the
// all-reduce becomes eligible and NCCL's kernel starts only once the apply retires
// (measured at N=2: ~90 us late per correction). A plain launch lets the high-priority
// exchange stream's CTAs in first.
thread_local bool tl_plain_launch = false;
struct PlainLaunchScope {
    bool prev;
    explicit PlainLaunchScope(bool on) : prev(tl_plain_launch) { tl_plain_launch = on || prev; }
    ~PlainLaunchScope() { tl_plain_launch = prev; }
};
template <typename... P, typename... A>
void launch_pdl(void (*kernel)(P...), int grid, int block, size_t smem, cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_on() && !tl_plain_launch) ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);  // errors: cudaGetLastError
}

// TMA-staged kernels (K1, K3): one CTA per SM, dynamic smem ring.
template <typename K>
bool prepare_tma(K kernel, int smem_bytes) {
    int d = 0;
    cudaGetDevice(&d);
    // cudaFuncSetAttribute is cheap but not free; remember per (kernel, device)
    struct Key { const void* k; int d; };
    static thread_local Key seen[64];
    static thread_local int nseen = 0;
    for (int i = 0; i < nseen; ++i)
        if (seen[i].k == reinterpret_cast<const void*>(kernel) && seen[i].d == d) return true;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
        return false;
    if (nseen < 64) seen[nseen++] = Key{reinterpret_cast<const void*>(kernel), d};
    return true;
}
// SMs the engine leaves free for the exchange while a correction all-reduce is in flight
// (0 = none): the TMA kernels (1 CTA per SM) and the wide K2 are capped at SMs - reserve.
thread_local int tl_reserve_sms = 0;
struct ReserveScope {
    int prev;
    explicit ReserveScope(int r) : prev(tl_reserve_sms) { tl_reserve_sms = r; }
    ~ReserveScope() { tl_reserve_sms = prev; }
};
inline int tma_grid(int64_t ntiles, int warps) {
    const int64_t want = (ntiles + warps - 1) / warps;
    const int64_t cap = std::max(1, dev_info().sms - tl_reserve_sms);
    return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}
// Tuning knobs for development sweeps: CDSGD_TMA_CFG (K1) / CDSGD_TMA_CFG2 (K2, K3) = <warps>x<stages>.
int read_cfg(const char* name, int dflt) {
    const char* e = getenv(name);
    int w = 0, st = 0;
    if (e == nullptr || sscanf(e, "%dx%d", &w, &st) != 2) return dflt;
    return w * 10 + st;
}
int tma_cfg() {
    static const int v = read_cfg("CDSGD_TMA_CFG", 162);
    return v;
}
int tma_cfg2() {  // K3
    static const int v = read_cfg("CDSGD_TMA_CFG2", 84);
    return v;
}
template <int WP, int ST, typename TW = float>
int launch_af_tma(const ApplyFArgs& a, cudaStream_t st) {
    using SM = ApplyFSmem<WP, ST, TW>;
    static_assert(SM::BYTES <= 227 * 1024, "smem");
    if (!prepare_tma(k_apply_full_tma<WP, ST, TW>, SM::BYTES)) return fail(CDSGD_ERR_CUDA, "smem attribute");
    launch_pdl(k_apply_full_tma<WP, ST, TW>, tma_grid((a.n + TILE_ELEMS - 1) / TILE_ELEMS, WP), WP * 32, SM::BYTES,
               st, a);
    return CDSGD_OK;
}
int launch_af_tma_cfg(const ApplyFArgs& a, int wdt, cudaStream_t st) {
    if (wdt == CDSGD_F64) return launch_af_tma<8, 3, double>(a, st);  // 8 KB slots: 3 stages fit
    switch (tma_cfg2()) {
        case 162: return launch_af_tma<16, 2>(a, st);
        case 83: return launch_af_tma<8, 3>(a, st);
        default: return launch_af_tma<8, 4>(a, st);
    }
}
template <typename G, int WARPS, int ST, typename TR = double>
int launch_quant_tma(const G* g, const TR* r_in, TR* r_out, uint32_t* words, KeyTab kt, double alpha,
                     uint64_t* err, uint64_t tag, cudaStream_t st, const P2PArgs& x) {
    using SM = QuantSmem<G, WARPS, ST, TR>;
    static_assert(SM::BYTES <= 227 * 1024, "smem");
    if (!prepare_tma(k_quantize_tma<G, WARPS, ST, TR>, SM::BYTES)) return fail(CDSGD_ERR_CUDA, "smem attribute");
    launch_pdl(k_quantize_tma<G, WARPS, ST, TR>, tma_grid(kt.ntiles, WARPS), WARPS * 32, SM::BYTES, st, g, r_in, r_out,
               words, kt, alpha, err, tag, x);
    return CDSGD_OK;
}
// fp32-residual fast mode: 16 warps x 3 stages of 4 KB slots (g + r, fp32)
int launch_quant_tma_cfg(const float* g, const float* r_in, float* r_out, uint32_t* words, KeyTab kt, double alpha,
                         uint64_t* err, uint64_t tag, cudaStream_t st, const P2PArgs& x) {
    return launch_quant_tma<float, 16, 3, float>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
}
// residual of either type behind void* (the engine's residual_dtype)
int launch_quant_tma_rdt(const float* g, int rdt, const void* r_in, void* r_out, uint32_t* words, KeyTab kt,
                         double alpha, uint64_t* err, uint64_t tag, cudaStream_t st, const P2PArgs& x);
template <typename G>
int launch_quant_tma_cfg(const G* g, const double* r_in, double* r_out, uint32_t* words, KeyTab kt, double alpha,
                         uint64_t* err, uint64_t tag, cudaStream_t st, const P2PArgs& x) {
    if constexpr (sizeof(G) == 8) {
        return launch_quant_tma<G, 8, 3>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
    } else {
    switch (tma_cfg()) {
        case 43: return launch_quant_tma<G, 4, 3>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
        case 46: return launch_quant_tma<G, 4, 6>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
        case 83: return launch_quant_tma<G, 8, 3>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
        case 84: return launch_quant_tma<G, 8, 4>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
        default: return launch_quant_tma<G, 16, 2>(g, r_in, r_out, words, kt, alpha, err, tag, st, x);
    }
    }
}
int launch_quant_tma_rdt(const float* g, int rdt, const void* r_in, void* r_out, uint32_t* words, KeyTab kt,
                         double alpha, uint64_t* err, uint64_t tag, cudaStream_t st, const P2PArgs& x) {
    if (rdt == CDSGD_F32)
        return launch_quant_tma_cfg(g, static_cast<const float*>(r_in), static_cast<float*>(r_out), words, kt, alpha,
                                    err, tag, st, x);
    return launch_quant_tma_cfg(g, static_cast<const double*>(r_in), static_cast<double*>(r_out), words, kt, alpha,
                                err, tag, st, x);
}
}  // namespace

// ------------------------------------------------------------------ layout
constexpr int64_t MAX_TILE_TABLE = int64_t(1) << 17;  // tiles (64M elements): a 2 MB table
struct cdsgd_layout {
    int32_t nkeys = 0;
    int64_t n = 0, nwords = 0, ntiles = 0;
    std::vector<int64_t> eoff, woff, toff;
    int64_t* dev = nullptr;  // [3 * (nkeys+1)]: eoff | woff | toff
    int4* tiles = nullptr;   // [ntiles] per-tile metadata (layouts of <= MAX_TILE_TABLE tiles)
    int device = 0;
    KeyTab tab() const {
        KeyTab k;
        k.eoff = dev;
        k.woff = dev + (nkeys + 1);
        k.toff = dev + 2 * (nkeys + 1);
        k.nkeys = nkeys;
        k.ntiles = ntiles;
        k.tiles = tiles;
        return k;
    }
};

extern "C" int cdsgd_abi_version(void) { return CDSGD_ABI_VERSION; }
extern "C" const char* cdsgd_last_error(void) { return g_err; }
extern "C" uint64_t cdsgd_launch_count(void) { return g_launches.load(); }
#ifdef CDSGD_PROBE_TIMING
// development builds only: the fused kernel's per-warp phase stamps of its last launch
extern "C" int cdsgd_diag_probe(unsigned long long* host, int64_t n) {
    const int64_t cap = static_cast<int64_t>(cdsgd::PROBE_WARPS) * cdsgd::PROBE_PTS;
    if (cudaMemcpyFromSymbol(host, cdsgd::g_probe, sizeof(unsigned long long) * (n < cap ? n : cap)) != cudaSuccess)
        return CDSGD_ERR_CUDA;
    return CDSGD_OK;
}
#endif

extern "C" int cdsgd_layout_create(const int64_t* lengths, int32_t n_keys, cdsgd_layout** out) {
    if (out == nullptr) return fail(CDSGD_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n_keys < 1 || lengths == nullptr) return fail(CDSGD_ERR_ARG, "layout needs at least one key");
    cdsgd_layout* L = new cdsgd_layout();
    L->nkeys = n_keys;
    L->eoff.assign(n_keys + 1, 0);
    L->woff.assign(n_keys + 1, 0);
    L->toff.assign(n_keys + 1, 0);
    for (int32_t k = 0; k < n_keys; ++k) {
        if (lengths[k] < 1) {
            delete L;
            return fail(CDSGD_ERR_ARG, "key %d has non-positive length %lld", k, (long long)lengths[k]);
        }
        const int64_t w = (lengths[k] + 15) / 16;
        L->eoff[k + 1] = L->eoff[k] + lengths[k];
        L->woff[k + 1] = L->woff[k] + w;
        L->toff[k + 1] = L->toff[k] + (w + TILE_WORDS - 1) / TILE_WORDS;
    }
    L->n = L->eoff[n_keys];
    L->nwords = L->woff[n_keys];
    L->ntiles = L->toff[n_keys];
    cudaGetDevice(&L->device);
    std::vector<int64_t> h;
    h.insert(h.end(), L->eoff.begin(), L->eoff.end());
    h.insert(h.end(), L->woff.begin(), L->woff.end());
    h.insert(h.end(), L->toff.begin(), L->toff.end());
    cudaError_t e = cudaMalloc(&L->dev, h.size() * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMemcpy(L->dev, h.data(), h.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
    // per-tile table (16 B per 512 elements, capped at 2 MB; CDSGD_NO_TILE_TABLE=1 disables)
    const char* nt = getenv("CDSGD_NO_TILE_TABLE");
    if (e == cudaSuccess && L->ntiles <= MAX_TILE_TABLE && L->ntiles > 0 && !(nt != nullptr && nt[0] == '1') &&
        L->nwords < (int64_t(1) << 31)) {
        std::vector<int4> t(L->ntiles);
        for (int32_t k = 0; k < n_keys; ++k)
            for (int64_t ti = L->toff[k]; ti < L->toff[k + 1]; ++ti) {
                const int64_t j = ti - L->toff[k];
                const int64_t e0 = L->eoff[k] + j * TILE_ELEMS, w0 = L->woff[k] + j * TILE_WORDS;
                const int64_t ne = std::min<int64_t>(TILE_ELEMS, L->eoff[k + 1] - e0);
                const int64_t nw = std::min<int64_t>(TILE_WORDS, L->woff[k + 1] - w0);
                t[ti] = make_int4(static_cast<int>(static_cast<uint32_t>(e0)), static_cast<int>(e0 >> 32),
                                  static_cast<int>(w0), static_cast<int>(ne | (nw << 16)));
            }
        e = cudaMalloc(&L->tiles, t.size() * sizeof(int4));
        if (e == cudaSuccess) e = cudaMemcpy(L->tiles, t.data(), t.size() * sizeof(int4), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        if (L->dev) cudaFree(L->dev);
        if (L->tiles) cudaFree(L->tiles);
        delete L;
        return fail(CDSGD_ERR_CUDA, "layout upload: %s", cudaGetErrorString(e));
    }
    *out = L;
    return CDSGD_OK;
}

extern "C" int cdsgd_layout_destroy(cdsgd_layout* L) {
    if (L == nullptr) return CDSGD_OK;
    if (L->dev) cudaFree(L->dev);
    if (L->tiles) cudaFree(L->tiles);
    delete L;
    return CDSGD_OK;
}
extern "C" int64_t cdsgd_layout_elems(const cdsgd_layout* L) { return L ? L->n : -1; }
extern "C" int64_t cdsgd_layout_words(const cdsgd_layout* L) { return L ? L->nwords : -1; }
extern "C" int32_t cdsgd_layout_keys(const cdsgd_layout* L) { return L ? L->nkeys : -1; }
extern "C" int cdsgd_layout_offsets(const cdsgd_layout* L, int64_t* eoff, int64_t* woff) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (eoff) memcpy(eoff, L->eoff.data(), L->eoff.size() * sizeof(int64_t));
    if (woff) memcpy(woff, L->woff.data(), L->woff.size() * sizeof(int64_t));
    return CDSGD_OK;
}

// ------------------------------------------------------------------ codec entry points
extern "C" int cdsgd_quantize(const cdsgd_layout* L, const void* grad, int32_t gdt, const double* r_in,
                              double* r_out, uint32_t* words, double alpha, uint64_t* err, uint64_t tag,
                              void* stream) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (!(alpha > 0.0)) return fail(CDSGD_ERR_ARG, "threshold alpha must be > 0");
    if (L->n == 0) return CDSGD_OK;
    if (!grad || !r_in || !r_out || !words) return fail(CDSGD_ERR_ARG, "NULL buffer");
    const KeyTab kt = L->tab();
    int rc;
    const P2PArgs nox{};
    if (gdt == CDSGD_F32)
        rc = launch_quant_tma_cfg(static_cast<const float*>(grad), r_in, r_out, words, kt, alpha, err, tag, S(stream),
                                  nox);
    else if (gdt == CDSGD_F64)
        rc = launch_quant_tma_cfg(static_cast<const double*>(grad), r_in, r_out, words, kt, alpha, err, tag,
                                  S(stream), nox);
    else
        return fail(CDSGD_ERR_ARG, "grad dtype must be CDSGD_F32 or CDSGD_F64");
    if (rc != CDSGD_OK) return rc;
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_quantize_f32r(const cdsgd_layout* L, const float* grad, const float* r_in, float* r_out,
                                   uint32_t* words, double alpha, uint64_t* err, uint64_t tag, void* stream) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (!(alpha > 0.0)) return fail(CDSGD_ERR_ARG, "threshold alpha must be > 0");
    if (L->n == 0) return CDSGD_OK;
    if (!grad || !r_in || !r_out || !words) return fail(CDSGD_ERR_ARG, "NULL buffer");
    const P2PArgs nox{};
    const int rc = launch_quant_tma_cfg(grad, r_in, r_out, words, L->tab(), alpha, err, tag, S(stream), nox);
    if (rc != CDSGD_OK) return rc;
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_dequantize_sum(const cdsgd_layout* L, const uint32_t* words, int32_t np, int64_t stride,
                                    double alpha, double* out, uint64_t* err, void* stream) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (np < 1) return fail(CDSGD_ERR_ARG, "need at least one payload");
    if (!(alpha > 0.0)) return fail(CDSGD_ERR_ARG, "threshold must be > 0");
    if (L->n == 0) return CDSGD_OK;
    const KeyTab kt = L->tab();
    const int grid = tile_grid(k_dequant_sum, kt.ntiles);
    k_dequant_sum<<<grid, THREADS, 0, S(stream)>>>(words, np, stride, kt, alpha, out, err);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_aggregate_full(const void* grads, int32_t dt, int32_t nc, int64_t stride, int64_t n,
                                    double* out, void* stream) {
    if (nc < 1) return fail(CDSGD_ERR_ARG, "need at least one contribution");
    if (n == 0) return CDSGD_OK;
    if (dt == CDSGD_F32) {
        k_aggregate_full<float><<<flat_grid(k_aggregate_full<float>, n), THREADS, 0, S(stream)>>>(
            static_cast<const float*>(grads), nc, stride, n, out);
    } else if (dt == CDSGD_F64) {
        k_aggregate_full<double><<<flat_grid(k_aggregate_full<double>, n), THREADS, 0, S(stream)>>>(
            static_cast<const double*>(grads), nc, stride, n, out);
    } else {
        return fail(CDSGD_ERR_ARG, "bad dtype");
    }
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_pack_symbols(const uint8_t* sym, int64_t n, uint32_t* words, uint64_t* err, void* stream) {
    if (n < 0) return fail(CDSGD_ERR_ARG, "n must be >= 0");
    if (n == 0) return CDSGD_OK;
    k_pack<<<flat_grid(k_pack, (n + 15) / 16), THREADS, 0, S(stream)>>>(sym, n, words, err);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_unpack_symbols(const uint32_t* words, int64_t length, uint8_t* sym, void* stream) {
    if (length < 0) return fail(CDSGD_ERR_ARG, "length must be >= 0");
    if (length == 0) return CDSGD_OK;
    k_unpack<<<flat_grid(k_unpack, length), THREADS, 0, S(stream)>>>(words, length, sym);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_global_update(void* w, int32_t wdt, const void* mean, int32_t mdt, int64_t n, double eta,
                                   void* stream) {
    if (eta < 0) return fail(CDSGD_ERR_ARG, "eta_global must be >= 0");
    if (n == 0) return CDSGD_OK;
#define GU(TW, TM)                                                                               \
    k_global_update<TW, TM><<<flat_grid(k_global_update<TW, TM>, n), THREADS, 0, S(stream)>>>(  \
        static_cast<TW*>(w), static_cast<const TM*>(mean), n, eta)
    if (wdt == CDSGD_F32 && mdt == CDSGD_F32) GU(float, float);
    else if (wdt == CDSGD_F32 && mdt == CDSGD_F64) GU(float, double);
    else if (wdt == CDSGD_F64 && mdt == CDSGD_F32) GU(double, float);
    else if (wdt == CDSGD_F64 && mdt == CDSGD_F64) GU(double, double);
    else return fail(CDSGD_ERR_ARG, "bad dtype");
#undef GU
    LAUNCH_CHECK();
    return CDSGD_OK;
}

extern "C" int cdsgd_local_update(const void* base, int32_t bdt, const void* g, int32_t gdt, void* out,
                                  int32_t odt, int64_t n, double eta_l, void* stream) {
    if (eta_l < 0) return fail(CDSGD_ERR_ARG, "eta_local must be >= 0");
    if (n == 0) return CDSGD_OK;
    if (bdt < 0 || bdt > 1 || gdt < 0 || gdt > 1 || odt < 0 || odt > 1) return fail(CDSGD_ERR_ARG, "bad dtype");
#define LU(TB, TG, TO)                                                                                   \
    launch_pdl(k_local_update<TB, TG, TO>, flat_grid(k_local_update<TB, TG, TO>, n), THREADS, 0, S(stream), \
               static_cast<const TB*>(base), static_cast<const TG*>(g), static_cast<TO*>(out), n, eta_l)
    const int code = bdt * 4 + gdt * 2 + odt;
    switch (code) {
        case 0: LU(float, float, float); break;
        case 1: LU(float, float, double); break;
        case 2: LU(float, double, float); break;
        case 3: LU(float, double, double); break;
        case 4: LU(double, float, float); break;
        case 5: LU(double, float, double); break;
        case 6: LU(double, double, float); break;
        default: LU(double, double, double); break;
    }
#undef LU
    LAUNCH_CHECK();
    return CDSGD_OK;
}

// ------------------------------------------------------------------ fused apply
namespace {
// True if every partial sum j*alpha (|j| <= nr) is exactly representable, i.e. the
// ascending fp64 sum of nr decoded values equals cnt*alpha in any order.
bool alpha_exact(double alpha, int nr) {
    for (int j = 1; j <= nr; ++j) {
        const double v = static_cast<double>(j) * alpha;
        if (static_cast<long double>(v) != static_cast<long double>(j) * static_cast<long double>(alpha)) return false;
        if (!std::isfinite(v)) return false;
    }
    return true;
}
void build_tab(DecodeTab& tab, double alpha, double eta_g, int nr) {
    memset(&tab, 0, sizeof(tab));
    for (int c = -nr; c <= nr; ++c) {
        const double total = static_cast<double>(c) * alpha;          // exact (alpha_exact)
        const double mean = total / static_cast<double>(nr);          // engine.py:255
        tab.mean[c + nr] = mean;
        tab.upd[c + nr] = static_cast<float>(eta_g * mean);           // engine.py:511 (eta*mean), fp32 W
        tab.upd64[c + nr] = eta_g * mean;                             // the reference's own product, fp64 W
    }
    tab.sq_scale = (alpha / nr) * (alpha / nr);
}
inline bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

int small_grid_cap();
int launch_apply_quant(const cdsgd_layout* L, void* W, int wdt, const uint32_t* gathered, int nr, int64_t stride,
                       double alpha, double eta_g, const float* gnext, float* loc, double eta_l, uint64_t* err,
                       uint64_t skip_below, double* gnorm, const DecodeTab* tab_in, int exact_in,
                       cudaStream_t st, const P2PArgs* x = nullptr, const StageDst* gs = nullptr,
                       const P2PArgs* xs = nullptr, unsigned int* sched = nullptr, float fold_scale = 0.f,
                       double* gnorm2 = nullptr, double* const* gclear = nullptr) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (nr < 1 || nr > MAX_RANKS - 1) return fail(CDSGD_ERR_ARG, "nranks must be in [1, %d]", MAX_RANKS - 1);
    if ((gnext == nullptr) != (loc == nullptr)) return fail(CDSGD_ERR_ARG, "g_next and loc_out go together");
    if (L->n == 0) return CDSGD_OK;
    ApplyQArgs a;
    a.W = W;
    a.gathered = gathered;
    a.stride = stride;
    a.gnext = gnext;
    a.loc = loc;
    a.alpha = alpha;
    a.inv_n_or_zero = pow2(nr) ? 1.0 / nr : 0.0;
    a.eta_g_d = eta_g;
    a.eta_l_d = eta_l;
    a.eta_l = static_cast<float>(eta_l);
    a.nranks = nr;
    a.err = err;
    a.skip_below = skip_below;
    a.gnorm = gnorm;
    a.x = x != nullptr ? *x : P2PArgs{};
    a.gs = gs != nullptr ? *gs : StageDst{};
    a.xs = xs != nullptr ? *xs : P2PArgs{};
    a.sched = sched;
    a.fold_scale = fold_scale;
    a.fold = fold_scale != 0.f ? 1 : 0;
    a.gnorm2 = gnorm2;
    a.gclear[0] = gclear != nullptr ? gclear[0] : nullptr;
    a.gclear[1] = gclear != nullptr ? gclear[1] : nullptr;
    DecodeTab tab;
    int exact;
    if (tab_in != nullptr) {
        tab = *tab_in;
        exact = exact_in;
    } else {
        exact = alpha_exact(alpha, nr) ? 1 : 0;
        build_tab(tab, alpha, eta_g, nr);
    }
    a.exact = exact;
    const KeyTab kt = L->tab();
    if (tl_reserve_sms > 0 && nr > 1 && nr <= 8 && a.sched != nullptr) {
        // beside a correction all-reduce: one 512-thread CTA per SM on SMs - reserve (the
        // dynamic tile scheduler balances the work over however many CTAs run)
        const int grid = std::max(1, dev_info().sms - tl_reserve_sms);
#define AQW(R)                                                                                 \
    case R:                                                                                    \
        if (wdt == CDSGD_F64) launch_pdl(k_apply_quant<R, 1, double>, grid, 2 * THREADS, 0, st, a, kt, tab); \
        else launch_pdl(k_apply_quant<R, 1, float>, grid, 2 * THREADS, 0, st, a, kt, tab);         \
        break
        switch (nr) { AQW(2); AQW(3); AQW(4); AQW(5); AQW(6); AQW(7); AQW(8); }
#undef AQW
        LAUNCH_CHECK();
        return CDSGD_OK;
    }
    // one-wave layouts (a 128-element chunk task for every resident warp or fewer): chunk tasks,
    // as the fused kernel (4x the warps in flight). Above that whole tiles: at 2^20 elements
    // (4 chunk tasks per warp) chunk tasks measured 17 vs 11 us.
#define AQ(R, TW)                                                                                       \
    case R:                                                                                             \
        if (kt.ntiles * CHUNKS <= static_cast<int64_t>(resident_blocks(k_apply_quant<R, 0, TW, 1>, THREADS)) * \
                                      WARPS_PER_BLOCK)                                                  \
            launch_pdl(k_apply_quant<R, 0, TW, 1>,                                                      \
                       std::min(tile_grid(k_apply_quant<R, 0, TW, 1>, kt.ntiles * CHUNKS), small_grid_cap()), THREADS, \
                       0, st, a, kt, tab);                                                              \
        else                                                                                            \
            launch_pdl(k_apply_quant<R, 0, TW>, tile_grid(k_apply_quant<R, 0, TW>, kt.ntiles), THREADS, 0, st, a, kt, \
                       tab);                                                                            \
        break
    if (wdt == CDSGD_F64) {
        switch (nr) {
            AQ(1, double); AQ(2, double); AQ(3, double); AQ(4, double); AQ(5, double); AQ(6, double); AQ(7, double);
            AQ(8, double);
            default:
                launch_pdl(k_apply_quant<0, 0, double>, tile_grid(k_apply_quant<0, 0, double>, kt.ntiles), THREADS, 0,
                           st, a, kt, tab);
        }
    } else {
        switch (nr) {
            AQ(1, float); AQ(2, float); AQ(3, float); AQ(4, float); AQ(5, float); AQ(6, float); AQ(7, float);
            AQ(8, float);
            default:
                launch_pdl(k_apply_quant<0, 0, float>, tile_grid(k_apply_quant<0, 0, float>, kt.ntiles), THREADS, 0, st,
                           a, kt, tab);
        }
    }
#undef AQ
    LAUNCH_CHECK();
    return CDSGD_OK;
}

int launch_apply_full(void* W, int wdt, const float* gsum, int nr, int64_t n, double eta_g, const float* gnext,
                      float* loc, double eta_l, const uint64_t* err, uint64_t skip_below, double* gnorm,
                      cudaStream_t st, double* const* gclear = nullptr) {
    if (nr < 1) return fail(CDSGD_ERR_ARG, "nranks must be >= 1");
    if ((gnext == nullptr) != (loc == nullptr)) return fail(CDSGD_ERR_ARG, "g_next and loc_out go together");
    if (n == 0) return CDSGD_OK;
    ApplyFArgs a;
    a.W = W;
    a.gsum = gsum;
    a.gnext = gnext;
    a.loc = loc;
    a.scale = static_cast<float>(eta_g / nr);
    a.eta_l = static_cast<float>(eta_l);
    a.inv_n = 1.0 / nr;
    a.eta_g_d = eta_g;
    a.eta_l_d = eta_l;
    a.inv_n_or_zero = pow2(nr) ? 1.0 / nr : 0.0;
    a.nranks = nr;
    a.n = n;
    a.err = err;
    a.skip_below = skip_below;
    a.gnorm = gnorm;
    a.gclear[0] = gclear != nullptr ? gclear[0] : nullptr;
    a.gclear[1] = gclear != nullptr ? gclear[1] : nullptr;
    const int rc = launch_af_tma_cfg(a, wdt, st);
    if (rc != CDSGD_OK) return rc;
    LAUNCH_CHECK();
    return CDSGD_OK;
}
// Fused apply(t-1) + quantize(t), register-staged (measured faster than a TMA-ring variant).
// Chunk-sized tasks (CH=1) below this many whole tiles per resident warp (CDSGD_CH1_TPW; 0 = never)
int ch1_tiles_per_warp() {
    static const int v = [] {
        const char* e = getenv("CDSGD_CH1_TPW");
        return e != nullptr ? atoi(e) : 2;
    }();
    return v;
}
// Grid cap for chunk-task (small-layout) launches, in CTAs per SM (CDSGD_SMALL_CTAS_PER_SM;
// default: no cap). Fewer CTAs leave slots for the next round's grid to become resident early
// under programmatic dependent launch.
int small_grid_cap() {
    static const int v = [] {
        const char* e = getenv("CDSGD_SMALL_CTAS_PER_SM");
        const int c = e != nullptr ? atoi(e) : 0;
        return c > 0 ? c * dev_info().sms : (1 << 30);
    }();
    return v;
}
// Chunks per task of the fused kernel for several ranks' codes with fp64 weights: whole tiles
// spill at 128 registers (F<4>: 120 B), half tiles do not — F 190 vs 194 us at N=4, 182 vs
// 186 at N=2 (CDSGD_MR_CH=4 restores whole tiles). (K2 with half tiles measured no better.)
bool mr_half_tiles() {
    static const bool v = [] {
        const char* e = getenv("CDSGD_MR_CH");
        return e == nullptr || atoi(e) != 4;
    }();
    return v;
}
template <int NR, int AP, typename TW, typename TR, int CHL>
int launch_fused_ch(const FusedArgs& a, const KeyTab& kt, const DecodeTab& tab, cudaStream_t st) {
    // fewer than 2 whole-tile tasks per resident warp: split tiles into chunk tasks
    const int64_t warps =
        static_cast<int64_t>(resident_blocks(k_fused_ldg<NR, AP, CHL, TW, TR>, THREADS)) * WARPS_PER_BLOCK;
    if (kt.ntiles < ch1_tiles_per_warp() * warps)
        launch_pdl(k_fused_ldg<NR, AP, 1, TW, TR>,
                   std::min(tile_grid(k_fused_ldg<NR, AP, 1, TW, TR>, kt.ntiles * CHUNKS), small_grid_cap()), THREADS,
                   0, st, a, kt, tab);
    else
        launch_pdl(k_fused_ldg<NR, AP, CHL, TW, TR>,
                   tile_grid(k_fused_ldg<NR, AP, CHL, TW, TR>, kt.ntiles * (CHUNKS / CHL)), THREADS, 0, st, a, kt, tab);
    return CDSGD_OK;
}
template <int NR, int AP, typename TW, typename TR>
int launch_fused_cfg(const FusedArgs& a, const KeyTab& kt, const DecodeTab& tab, cudaStream_t st) {
    constexpr int CHL = sizeof(TW) == 8 ? CDSGD_F64_CH : CHUNKS;  // chunks per task on large layouts
    if constexpr (sizeof(TW) == 8 && NR >= 2 && AP == APPLY_Q)
        if (mr_half_tiles()) return launch_fused_ch<NR, AP, TW, TR, 2>(a, kt, tab, st);
    return launch_fused_ch<NR, AP, TW, TR, CHL>(a, kt, tab, st);
}
template <typename TW, typename TR>
int launch_fused_t(int nr, int apply, const FusedArgs& a, const KeyTab& kt, const DecodeTab& tab, cudaStream_t st) {
    if (apply == APPLY_L) return launch_fused_cfg<1, APPLY_L, TW, TR>(a, kt, tab, st);  // W final: loc + quantize only
    if (apply == APPLY_F) return launch_fused_cfg<1, APPLY_F, TW, TR>(a, kt, tab, st);
    switch (nr) {
        case 1: return launch_fused_cfg<1, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 2: return launch_fused_cfg<2, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 3: return launch_fused_cfg<3, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 4: return launch_fused_cfg<4, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 5: return launch_fused_cfg<5, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 6: return launch_fused_cfg<6, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 7: return launch_fused_cfg<7, APPLY_Q, TW, TR>(a, kt, tab, st);
        case 8: return launch_fused_cfg<8, APPLY_Q, TW, TR>(a, kt, tab, st);
        default: return fail(CDSGD_ERR_ARG, "fused step supports 1..8 ranks");
    }
}
// weight / residual precision modes: exact (fp64 W, fp64 r), fp32 W (fp64 r), fast (fp32 W, fp32 r)
bool modes_ok(int wdt, int rdt) { return rdt == CDSGD_F64 ? (wdt == CDSGD_F64 || wdt == CDSGD_F32) : wdt == CDSGD_F32; }
int launch_fused(int nr, int apply, int wdt, int rdt, const FusedArgs& a, const KeyTab& kt, const DecodeTab& tab,
                 cudaStream_t st) {
    if (!modes_ok(wdt, rdt)) return fail(CDSGD_ERR_ARG, "fp32 residuals need fp32 weights (the fast mode)");
    const int rc = rdt == CDSGD_F32   ? launch_fused_t<float, float>(nr, apply, a, kt, tab, st)
                   : wdt == CDSGD_F64 ? launch_fused_t<double, double>(nr, apply, a, kt, tab, st)
                                      : launch_fused_t<float, double>(nr, apply, a, kt, tab, st);
    if (rc != CDSGD_OK) return rc;
    LAUNCH_CHECK();
    return CDSGD_OK;
}
bool wdt_ok(int wdt) { return wdt == CDSGD_F32 || wdt == CDSGD_F64; }
}  // namespace

extern "C" int cdsgd_apply_quant(const cdsgd_layout* L, void* W, int32_t wdt, const uint32_t* gathered, int32_t nr,
                                 int64_t stride, double alpha, double eta_g, const float* gnext, float* loc,
                                 double eta_l, uint64_t* err, uint64_t skip_below, double* gnorm, void* stream) {
    if (!(alpha > 0.0)) return fail(CDSGD_ERR_ARG, "threshold alpha must be > 0");
    if (!wdt_ok(wdt)) return fail(CDSGD_ERR_ARG, "weights dtype must be CDSGD_F32 or CDSGD_F64");
    return launch_apply_quant(L, W, wdt, gathered, nr, stride, alpha, eta_g, gnext, loc, eta_l, err, skip_below,
                              gnorm, nullptr, 0, S(stream));
}

extern "C" int cdsgd_apply_full(void* W, int32_t wdt, const float* gsum, int32_t nr, int64_t n, double eta_g,
                                const float* gnext, float* loc, double eta_l, const uint64_t* err,
                                uint64_t skip_below, double* gnorm, void* stream) {
    if (!wdt_ok(wdt)) return fail(CDSGD_ERR_ARG, "weights dtype must be CDSGD_F32 or CDSGD_F64");
    return launch_apply_full(W, wdt, gsum, nr, n, eta_g, gnext, loc, eta_l, err, skip_below, gnorm, S(stream));
}

extern "C" int cdsgd_fused_round(const cdsgd_layout* L, const float* grad, const void* r_in, void* r_out,
                                 int32_t r_dtype, uint32_t* words, double alpha, uint64_t* err, uint64_t err_tag, void* W,
                                 int32_t wdt, float* loc, const uint32_t* gathered, int32_t nr, int64_t stride, double eta_g,
                                 double eta_l, uint64_t skip_below, double* gnorm, void* stream) {
    if (L == nullptr) return fail(CDSGD_ERR_ARG, "layout is NULL");
    if (!(alpha > 0.0)) return fail(CDSGD_ERR_ARG, "threshold alpha must be > 0");
    if (eta_g < 0 || eta_l < 0) return fail(CDSGD_ERR_ARG, "learning rates must be >= 0");
    if (nr < 1 || nr > MAX_RANKS_P2P) return fail(CDSGD_ERR_ARG, "nranks must be in [1, %d]", MAX_RANKS_P2P);
    if (L->n == 0) return CDSGD_OK;
    if (!grad || !r_in || !r_out || !words || !W || !loc) return fail(CDSGD_ERR_ARG, "NULL buffer");
    if (!wdt_ok(wdt)) return fail(CDSGD_ERR_ARG, "weights dtype must be CDSGD_F32 or CDSGD_F64");
    if (!wdt_ok(r_dtype)) return fail(CDSGD_ERR_ARG, "residual dtype must be CDSGD_F32 or CDSGD_F64");
    FusedArgs a{};
    a.g = grad;
    a.r_in = r_in;
    a.r_out = r_out;
    a.words = words;
    a.alpha = alpha;
    a.tag = err_tag;
    a.W = W;
    a.loc = loc;
    a.gathered = gathered;
    a.stride = stride;
    a.scale = static_cast<float>(eta_g / nr);
    a.inv_n = 1.0 / nr;
    a.eta_l = static_cast<float>(eta_l);
    a.exact = alpha_exact(alpha, nr) ? 1 : 0;
    a.eta_g_d = eta_g;
    a.eta_l_d = eta_l;
    a.nranks = nr;
    a.inv_n_or_zero = pow2(nr) ? 1.0 / nr : 0.0;
    a.skip_below = skip_below;
    a.gnorm = gathered != nullptr ? gnorm : nullptr;
    a.err = err;
    a.sched = nullptr;  // static tile ranges: no scheduler state shared between callers
    DecodeTab tab;
    build_tab(tab, alpha, eta_g, nr);
    return launch_fused(nr, gathered != nullptr ? APPLY_Q : APPLY_L, wdt, r_dtype, a, L->tab(), tab, S(stream));
}

// ------------------------------------------------------------------ NCCL exchange
struct cdsgd_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0;
};

extern "C" int cdsgd_comm_unique_id(void* out) {
    static_assert(sizeof(ncclUniqueId) == CDSGD_UNIQUE_ID_BYTES, "ncclUniqueId size");
    if (out == nullptr) return fail(CDSGD_ERR_ARG, "out is NULL");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return CDSGD_OK;
}

extern "C" int cdsgd_comm_init(const void* uid, int32_t nranks, int32_t rank, cdsgd_comm** out) {
    if (out == nullptr || uid == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CDSGD_ERR_ARG, "bad rank %d of %d", rank, nranks);
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    cdsgd_comm* c = new cdsgd_comm();
    c->nranks = nranks;
    c->rank = rank;
    // The correction all-reduce (4n bytes) runs beside HBM-bound kernels: 64 channels
    // measured 257 vs 276 us standalone at N=4 and +4 % (N=2) / +2 % (N=4) end to end.
    // CDSGD_NCCL_MIN_CTAS overrides (0 = NCCL's default); NCCL_MIN_NCHANNELS still wins.
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    const char* mc = getenv("CDSGD_NCCL_MIN_CTAS");
    const int min_ctas = mc != nullptr ? atoi(mc) : 64;
    if (min_ctas > 0 && getenv("NCCL_MIN_NCHANNELS") == nullptr && getenv("NCCL_MIN_CTAS") == nullptr)
    {
        cfg.minCTAs = min_ctas;
        cfg.maxCTAs = min_ctas;  // the default cap is below 64 (ncclInvalidArgument otherwise)
    }
    // CDSGD_NCCL_ALGO: an NCCL_ALGO value for this communicator only (e.g. "allreduce:nvls" for
    // the fp32 correction all-reduce), set around its creation so the framework's own
    // communicators (fp64 all-reduces, broadcasts) keep every algorithm (development A/B)
    // (CDSGD_NCCL_PROTO likewise for NCCL_PROTO)
    struct ScopedEnv {
        const char* name;
        bool set = false, had = false;
        std::string prev;
        ScopedEnv(const char* n, const char* v) : name(n) {
            if (v == nullptr) return;
            const char* p = getenv(n);
            had = p != nullptr;
            if (had) prev = p;
            setenv(n, v, 1);
            set = true;
        }
        ~ScopedEnv() {
            if (!set) return;
            if (had) setenv(name, prev.c_str(), 1);
            else unsetenv(name);
        }
    };
    ncclResult_t r;
    {
        const ScopedEnv algo("NCCL_ALGO", getenv("CDSGD_NCCL_ALGO"));
        const ScopedEnv proto("NCCL_PROTO", getenv("CDSGD_NCCL_PROTO"));
        r = ncclCommInitRankConfig(&c->nccl, nranks, id, rank, &cfg);
    }
    if (r != ncclSuccess) {
        delete c;
        return fail(CDSGD_ERR_NCCL, "ncclCommInitRankConfig: %s", ncclGetErrorString(r));
    }
    *out = c;
    return CDSGD_OK;
}

extern "C" int cdsgd_comm_destroy(cdsgd_comm* c) {
    if (c == nullptr) return CDSGD_OK;
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
    return CDSGD_OK;
}

extern "C" int cdsgd_allgather_words(cdsgd_comm* c, const uint32_t* send, uint32_t* recv, int64_t words,
                                     void* stream) {
    if (c == nullptr) return fail(CDSGD_ERR_ARG, "comm is NULL");
    NCCL_TRY(ncclAllGather(send, recv, static_cast<size_t>(words), ncclUint32, c->nccl, S(stream)));
    return CDSGD_OK;
}

extern "C" int cdsgd_allreduce_sum_f32(cdsgd_comm* c, const float* send, float* recv, int64_t n, void* stream) {
    if (c == nullptr) return fail(CDSGD_ERR_ARG, "comm is NULL");
    NCCL_TRY(ncclAllReduce(send, recv, static_cast<size_t>(n), ncclFloat, ncclSum, c->nccl, S(stream)));
    return CDSGD_OK;
}

// ------------------------------------------------------------------ step engine
struct cdsgd_engine {
    cdsgd_engine_desc d{};
    const cdsgd_layout* L = nullptr;
    cdsgd_comm* comm = nullptr;
    cudaStream_t xs = nullptr, xs2 = nullptr;  // exchange streams (xs2: copy-engine share)
    // one stream per peer for the copy-engine share's peer copies, so the N-1 transfers of a
    // phase run on several copy engines at once instead of back to back on xs2
    cudaStream_t xsc[MAX_RANKS_P2P] = {nullptr};
    cudaEvent_t evc[MAX_RANKS_P2P] = {nullptr};
    cudaEvent_t evfork = nullptr;
    bool ce_parallel = false;          // CDSGD_CE_PARALLEL=1: one stream per peer copy
    cudaEvent_t evC = nullptr;
    cudaEvent_t evQ[2] = {nullptr, nullptr};
    cudaEvent_t evX[2] = {nullptr, nullptr};
    // Split correction apply (CDSGD_SPLIT_APPLY=1): NCCL's share [0, split_off) of a correction
    // all-reduce ends before the copy engines' all-gather of the rest, so K3 applies that prefix
    // once evN fires and the rest after evX (0 = not split). Parity-green, measured within noise
    // (N=4 441/442 -> 446/442, N=2 250 -> 246 Gelem/s: the two halves' tails and the prefix's
    // HBM traffic beside the all-gather cost what the earlier start gains) -> off by default.
    cudaEvent_t evN[2] = {nullptr, nullptr};
    int64_t split_off[2] = {0, 0};
    bool split_apply = false;
    DecodeTab tab{};
    int exact = 0;
    bool uses_local = false;
    int64_t n_warmup = 0;
    // state
    int64_t t = 0;
    int rcur = 0;
    bool compute_is_loc = false;
    bool pending = false;
    int64_t pend_t = 0;
    bool pend_comp = false;
    const float* pend_grad = nullptr;
    bool failed = false;
    int64_t err_base = 0;
    std::vector<int8_t> rlog;  // residual index at the entry of rounds err_base..t-1
    // fused P2P exchange (symmetric memory): peer buffer bases and protocol state
    bool p2p = false;
    char* peer[MAX_RANKS_P2P] = {nullptr};
    int64_t off_slot[2] = {0, 0}, off_ready = 0, off_freed = 0;
    int64_t last_use[2] = {-1, -1};  // last compressed round that filled slot p
    bool xused[2] = {false, false};  // round parity p used the NCCL stream
    unsigned int* counters = nullptr;  // [4] grid-completion counters (K1/fused, K2, stage, reduce)
    // P2P correction rounds (sharded exact reduce over NVLink, no NCCL)
    int64_t chunk = 0;  // elements per shard owner (P2P exact correction), a multiple of 4
    // P2P exact staging: false = pull (my g_t stays local, owners load it over NVLink),
    // true = push (K2 stores each element into its owner's receive row). Pull measured
    // faster at N=4 (461 vs 442 Gelem/s): the pushes make K2 NVLink-bound. CDSGD_STAGE_PUSH=1.
    bool stage_push = false;
    int64_t off_W = 0, off_stage[2] = {0, 0}, off_gready = 0, off_gfreed = 0, off_wdone = 0, off_gpart = 0;
    int64_t off_gsum[2] = {0, 0};
    // P2P mode: fraction of each correction all-reduce moved by the copy engines
    // (p2p_ce_allreduce on stream xs2) beside NCCL's share (0 = NCCL only)
    double ce_frac = 0.0;
    int64_t last_stage[2] = {-1, -1};  // last correction round that used staging slot s
    int64_t ncorr = 0;                 // P2P correction rounds staged so far (slot = ncorr & 1)
    int pend_slot = 0;                 // staging slot of the pending correction round
    int64_t s0 = 0, s1 = 0;            // this rank's shard of elements
    double* gacc = nullptr;            // shard sum(mean^2) accumulator
    unsigned int* sched = nullptr;     // [4] dynamic tile schedulers: fused kernel [0,1], K2 [2,3]
    bool fuse = false;                 // apply(t-1) + quantize(t) in one kernel (N=1 or P2P)
    bool pcorr = false;                // P2P mode: correction rounds by the exact sharded NVLink reduce
    bool plain_after_ar = false;       // plain (non-PDL) launch of the apply beside a correction all-reduce
    bool fuse_after_ar = false;        // N>1: quantize(t+1) fused with the correction's apply, after the all-reduce
    bool ar_first = true;              // gate the apply behind a marker on the exchange stream (CDSGD_AR_FIRST)
    // Copy-engine share, second half deferred to the next step (CDSGD_CE_DEFER, default on): the
    // shard reduce runs on C right after the apply of the correction step (all SMs but NCCL's,
    // instead of starving beside it), and the all-gather on the copy engines overlaps K1.
    bool ce_defer = true;
    struct CePending {
        bool on = false;
        int64_t p = 0, off = 0, cnt = 0, ck = 0, m0 = 0, m1 = 0;
        int s = 0;
        const float* g = nullptr;
    } ce_pend;
    cudaEvent_t evG = nullptr;
    cudaEvent_t evR = nullptr;         // the deferred copy-engine reduce is done (on C)
    int reserve_sms = 0;               // SMs left free for the all-reduce's CTAs (CDSGD_RESERVE_SMS)
    // NCCL symmetric-window correction all-reduce (CDSGD_NCCL_SYM=1, p2p mode): g_t staged into an
    // ncclMemAlloc'ed, window-registered buffer (by K2, which streams g_t anyway), all-reduced into a
    // registered gsum buffer with NCCL's symmetric-memory kernels. Parity-green but measured slower
    // at N=2 (200 Gelem/s, 232 with NCCL_NVLS_ENABLE=0, vs 252 for the default split): an option.
    bool nccl_sym = false;
    void* sym_stage[2] = {nullptr, nullptr};
    void* sym_gsum[2] = {nullptr, nullptr};
    ncclWindow_t win[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t ar_round = -1;             // correction round whose all-reduce is in flight on the exchange streams
    bool diag_local_codes = false;     // timing diagnostic: store codes only locally
    bool diag_no_wait = false;         // timing diagnostic: skip the code-exchange flag waits
    int sc_fence = 0;                  // CDSGD_SC_FENCE=1: fence.sc.sys publish (A/B knob)
    // profiling: event pairs per kernel class (0 quant, 1 apply_q, 2 apply_f, 3 local, 4 exchange, 5 fused,
    // 6 stage, 7 reduce, 8 wait, 9 fused local-only, 10 copy-engine share of a correction all-reduce)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> prof_marks;  // (class, index of start event)
};

namespace {
// Records a start event on `st` and returns its pool index (or -1 when not profiling).
long prof_start(cdsgd_engine* E, int cls, cudaStream_t st) {
    if (!E->prof) return -1;
    while (E->ev_pool.size() < E->ev_used + 2) {
        cudaEvent_t ev;
        if (cudaEventCreate(&ev) != cudaSuccess) return -1;
        E->ev_pool.push_back(ev);
    }
    const size_t i = E->ev_used;
    E->ev_used += 2;
    cudaEventRecord(E->ev_pool[i], st);
    E->prof_marks.emplace_back(cls, i);
    return static_cast<long>(i);
}
void prof_stop(cdsgd_engine* E, long i, cudaStream_t st) {
    if (i >= 0) cudaEventRecord(E->ev_pool[i + 1], st);
}

// Worker._push_compressed (engine.py:345-355) + should_compress (engine.py:217-223).
int round_compressed(const cdsgd_engine* E, int64_t t, bool* out) {
    const bool in_warm = E->uses_local && t < E->n_warmup;
    if (in_warm) { *out = false; return CDSGD_OK; }
    if (E->d.algo == CDSGD_ALGO_BITSGD) { *out = true; return CDSGD_OK; }
    if (E->d.algo == CDSGD_ALGO_CDSGD) {
        if (E->d.force_compress) { *out = true; return CDSGD_OK; }
        const int64_t count = t - E->n_warmup + 1;
        if (count < 1) return fail(CDSGD_ERR_ARG, "count must be >= 1 (engine.py:221-222)");
        *out = (count % E->d.k) != 0;
        return CDSGD_OK;
    }
    *out = false;
    return CDSGD_OK;
}

int64_t words_of(const cdsgd_engine* E) { return E->L->nwords; }

// Grad-norm ring: round p's slot. With >= 4 slots the kernel accumulating round p zeroes
// the slots of the next two rounds in-kernel (pdl_enter), so no memset breaks the
// programmatic-launch chain; a shorter ring falls back to a memset per round.
double* gnorm_slot(const cdsgd_engine* E, int64_t p) {
    return (E->d.gnorm_sq != nullptr && E->d.gnorm_ring > 0) ? E->d.gnorm_sq + (p % E->d.gnorm_ring) : nullptr;
}
bool gnorm_ahead(const cdsgd_engine* E) { return E->d.gnorm_sq != nullptr && E->d.gnorm_ring >= 4; }
void gnorm_clears(const cdsgd_engine* E, int64_t first, double** clr) {
    clr[0] = gnorm_ahead(E) ? gnorm_slot(E, first) : nullptr;
    clr[1] = gnorm_ahead(E) ? gnorm_slot(E, first + 1) : nullptr;
}

// ---- P2P correction rounds (kernels_corr.cuh)
template <typename T>
T* at(char* base, int64_t off) { return reinterpret_cast<T*>(base + off); }

// Round t is a correction: g_t goes to staging slot ncorr & 1 where every rank can
// read it. prepare_stage fills the destination + protocol and advances the state;
// the copy is then either fused into K2 (which reads g_t anyway) or run by k_stage.
void prepare_stage(cdsgd_engine* E, int64_t t, StageDst* dst, P2PArgs* x) {
    const int nr = E->d.nranks, me = E->d.rank;
    const int s = static_cast<int>(E->ncorr & 1);
    char* local = E->peer[me];
    *dst = StageDst{};
    if (E->stage_push) {
        dst->chunk = E->chunk;
        for (int o = 0; o < nr; ++o)  // owner o's receive row [me], indexed by element
            dst->base[o] = at<float>(E->peer[o], E->off_stage[s]) + (static_cast<int64_t>(me) - o) * E->chunk;
    } else {  // pull: g_t stays in my own stage; owners read it over NVLink
        dst->chunk = std::max<int64_t>(E->L->n, TILE_ELEMS) + 4;
        dst->base[0] = at<float>(local, E->off_stage[s]);
    }
    *x = P2PArgs{};
    x->nranks = nr;
    for (int r = 0; r < nr; ++r) x->publish[r] = at<uint64_t>(E->peer[r], E->off_gready) + s * nr + me;
    x->wait_flags = at<const uint64_t>(local, E->off_gfreed) + s * nr;
    x->wait_value = E->last_stage[s] >= 0 ? static_cast<uint64_t>(E->last_stage[s]) + 1 : 0;
    x->publish_value = static_cast<uint64_t>(t) + 1;
    x->counter = E->counters + 2;
    x->sc_fence = E->sc_fence;
    x->err = E->d.err;
    E->last_stage[s] = t;
    E->pend_slot = s;
    E->ncorr += 1;
}

int p2p_stage(cdsgd_engine* E, int64_t t, const float* g, cudaStream_t C) {
    StageArgs a{};
    a.g = g;
    a.n = E->L->n;
    prepare_stage(E, t, &a.gs, &a.x);
    const long pi = prof_start(E, 6, C);
    launch_pdl(k_stage, flat_grid(k_stage, (a.n + 3) / 4), THREADS, 0, C, a);
    prof_stop(E, pi, C);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

// The reduce runs beside the next round's quantize kernel; one CTA per SM measured best
// (fewer CTAs starve the remote loads: 64 -> 374 us, 32 -> 578 us at N=4).
// CDSGD_REDUCE_CTAS overrides (default: number of SMs).
int reduce_ctas() {
    static const int v = [] {
        const char* e = getenv("CDSGD_REDUCE_CTAS");
        const int x = e != nullptr ? atoi(e) : 0;
        return x > 0 ? x : dev_info().sms;
    }();
    return v;
}
template <int NR, bool SUM = false, typename TW = float>
void launch_reduce_t(const ReduceArgs& a, int64_t len, cudaStream_t C) {
    const int grid = std::min(flat_grid(k_reduce<NR, SUM, TW>, (len + 3) / 4), reduce_ctas());
    launch_pdl(k_reduce<NR, SUM, TW>, grid, THREADS, 0, C, a);
}
template <int NR>
void launch_reduce_w(const ReduceArgs& a, int64_t len, int wdt, cudaStream_t C) {
    if (wdt == CDSGD_F64) launch_reduce_t<NR, false, double>(a, len, C);
    else launch_reduce_t<NR, false, float>(a, len, C);
}

int p2p_ce_reduce_gather(cdsgd_engine* E, int64_t p, const float* g, cudaStream_t R, cudaStream_t X, int s,
                         int64_t ck, int64_t m0, int64_t m1);

// Issue the deferred second half of a correction's copy-engine share: the reduce on C (this
// step's stream, before anything else of the step), the all-gather on xs2; then the correction's
// completion event evX on xs joins NCCL's share (xs) and the copy-engine share (xs2).
int p2p_ce_finish(cdsgd_engine* E, cudaStream_t C) {
    if (!E->ce_pend.on) return CDSGD_OK;
    const auto cp = E->ce_pend;
    E->ce_pend.on = false;
    const int rc = p2p_ce_reduce_gather(E, cp.p, cp.g, C, E->xs2, cp.s, cp.ck, cp.m0, cp.m1);
    if (rc != CDSGD_OK) return rc;
    CUDA_TRY(cudaEventRecord(E->evC, E->xs2));
    CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evC, 0));
    CUDA_TRY(cudaEventRecord(E->evX[cp.p & 1], E->xs));
    return CDSGD_OK;
}

// Flag publication of the copy-engine phases: a 1-thread k_flags kernel (it can wait up to
// ~13 us for an SM beside K2/K1 at N=4), or with CDSGD_FLAG_MEMOPS=1 a stream memory
// operation (cuStreamWriteValue64, whose system-wide fence before the write orders every
// earlier copy of the stream first; no SM). Measured: memops 436-438 vs 441 Gelem/s at N=4,
// 247 vs 250 at N=2 — no gain, so the kernel stays the default.
using StreamWrite64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
StreamWrite64Fn stream_write64() {
    static const StreamWrite64Fn fn = [] {
        const char* e = getenv("CDSGD_FLAG_MEMOPS");
        if (e == nullptr || atoi(e) == 0) return static_cast<StreamWrite64Fn>(nullptr);
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<StreamWrite64Fn>(nullptr);
        return reinterpret_cast<StreamWrite64Fn>(p);
    }();
    return fn;
}
int publish_flags(const P2PArgs& x, cudaStream_t s) {
    if (const StreamWrite64Fn fn = stream_write64()) {
        bool ok = true;
        for (int r = 0; r < x.nranks && ok; ++r)
            if (x.publish[r] != nullptr)
                ok = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(x.publish[r]),
                        static_cast<cuuint64_t>(x.publish_value), 0) == CUDA_SUCCESS;
        if (ok) return CDSGD_OK;
        return fail(CDSGD_ERR_CUDA, "cuStreamWriteValue64 failed (unset CDSGD_FLAG_MEMOPS to use the flag kernel)");
    }
    k_flags<<<1, 32, 0, s>>>(x);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

// Peer copies of one copy-engine phase: copy k (dst[k] <- src[k], bytes[k]) on stream xsc[k],
// forked from and joined back into X, so the transfers to different peers overlap on several
// copy engines (CDSGD_CE_PARALLEL=1; serially on X by default).
int ce_copies(cdsgd_engine* E, cudaStream_t X, int ncopy, void* const* dst, const void* const* src,
              const size_t* bytes) {
    if (!E->ce_parallel || ncopy <= 1) {
        for (int k = 0; k < ncopy; ++k)
            if (bytes[k]) CUDA_TRY(cudaMemcpyAsync(dst[k], src[k], bytes[k], cudaMemcpyDeviceToDevice, X));
        return CDSGD_OK;
    }
    CUDA_TRY(cudaEventRecord(E->evfork, X));
    for (int k = 0; k < ncopy; ++k) {
        CUDA_TRY(cudaStreamWaitEvent(E->xsc[k], E->evfork, 0));
        if (bytes[k]) CUDA_TRY(cudaMemcpyAsync(dst[k], src[k], bytes[k], cudaMemcpyDeviceToDevice, E->xsc[k]));
        CUDA_TRY(cudaEventRecord(E->evc[k], E->xsc[k]));
    }
    for (int k = 0; k < ncopy; ++k) CUDA_TRY(cudaStreamWaitEvent(X, E->evc[k], 0));
    return CDSGD_OK;
}

// Part of a correction round's all-reduce on the COPY ENGINES: elements [off, off + cnt)
// of g_p. Each owner's slice goes to its receive row by cudaMemcpyAsync (no SMs), each
// owner sums its shard from local rows (fp64, ascending rank, rounded once to fp32 — the
// same value on every rank), and the sum shard is copied into every rank's gsum. Flags
// order the phases. Runs beside ncclAllReduce of [0, off) (split_correction).
int p2p_ce_allreduce(cdsgd_engine* E, int64_t p, const float* g, cudaStream_t X, int64_t off, int64_t cnt) {
    const int nr = E->d.nranks, me = E->d.rank;
    const int s = static_cast<int>(E->ncorr & 1);
    char* local = E->peer[me];
    const int64_t ck = (((cnt + nr - 1) / nr) + 3) / 4 * 4;  // shard per owner, <= E->chunk
    const int64_t m0 = std::min<int64_t>(off + cnt, off + ck * me), m1 = std::min<int64_t>(off + cnt, m0 + ck);
    P2PArgs fw{};  // 1. flow control: every owner finished reading its row `me` of slot s
    fw.nranks = nr;
    fw.wait_flags = at<const uint64_t>(local, E->off_gfreed) + s * nr;
    fw.wait_value = E->last_stage[s] >= 0 ? static_cast<uint64_t>(E->last_stage[s]) + 1 : 0;
    fw.err = E->d.err;
    E->last_stage[s] = p;
    E->ncorr += 1;
    if (fw.wait_value != 0) {
        k_wait_sum<<<1, 32, 0, X>>>(fw, nullptr, 0, nullptr, nullptr, nullptr);
        LAUNCH_CHECK();
    }
    {  // 2. reduce-scatter: my slice of owner o's shard -> o's row `me` (my own slice is read in place)
        void* dst[MAX_RANKS_P2P];
        const void* src[MAX_RANKS_P2P];
        size_t bytes[MAX_RANKS_P2P];
        for (int k = 1; k < nr; ++k) {
            const int o = (me + k) % nr;
            const int64_t o0 = std::min<int64_t>(off + cnt, off + ck * o), o1 = std::min<int64_t>(off + cnt, o0 + ck);
            dst[k - 1] = at<float>(E->peer[o], E->off_stage[s]) + static_cast<int64_t>(me) * ck;
            src[k - 1] = g + o0;
            bytes[k - 1] = o1 > o0 ? static_cast<size_t>(o1 - o0) * sizeof(float) : 0;
        }
        const int rc = ce_copies(E, X, nr - 1, dst, src, bytes);
        if (rc != CDSGD_OK) return rc;
    }
    P2PArgs fr{};
    fr.nranks = nr;
    for (int r = 0; r < nr; ++r) fr.publish[r] = at<uint64_t>(E->peer[r], E->off_gready) + s * nr + me;
    fr.publish_value = static_cast<uint64_t>(p) + 1;
    {
        const int rc = publish_flags(fr, X);
        if (rc != CDSGD_OK) return rc;
    }
    if (E->ce_defer) {  // steps 3-5 are issued by the next step (p2p_ce_finish)
        E->ce_pend.on = true;
        E->ce_pend.p = p;
        E->ce_pend.off = off;
        E->ce_pend.cnt = cnt;
        E->ce_pend.ck = ck;
        E->ce_pend.m0 = m0;
        E->ce_pend.m1 = m1;
        E->ce_pend.s = s;
        E->ce_pend.g = g;
        return CDSGD_OK;
    }
    return p2p_ce_reduce_gather(E, p, g, X, X, s, ck, m0, m1);
}

// Steps 3-5 of the copy-engine share: the shard reduce (a kernel) on stream R, the all-gather
// copies, flags and the completion wait on stream X.
int p2p_ce_reduce_gather(cdsgd_engine* E, int64_t p, const float* g, cudaStream_t R, cudaStream_t X, int s,
                         int64_t ck, int64_t m0, int64_t m1) {
    const int nr = E->d.nranks, me = E->d.rank;
    char* local = E->peer[me];
    ReduceArgs a{};  // 3. my shard from the N local rows -> my gsum (fp32 of the fp64 sum)
    for (int r = 0; r < nr; ++r) {
        a.stage[r] = r == me ? g : at<const float>(local, E->off_stage[s]) + static_cast<int64_t>(r) * ck - m0;
        a.xa.publish[r] = at<uint64_t>(E->peer[r], E->off_gfreed) + s * nr + me;
    }
    a.Wdst[0] = at<float>(local, E->off_gsum[p & 1]);
    a.ndst = 1;
    a.s0 = m0;
    a.s1 = m1;
    a.nranks = nr;
    a.xa.nranks = nr;
    a.xa.wait_flags = at<const uint64_t>(local, E->off_gready) + s * nr;
    a.xa.wait_value = static_cast<uint64_t>(p) + 1;
    a.xa.publish_value = static_cast<uint64_t>(p) + 1;
    a.xa.counter = E->counters + 3;
    a.xa.sc_fence = E->sc_fence;
    a.xa.err = E->d.err;
    if (m1 > m0) {
        switch (nr) {
            case 2: launch_reduce_t<2, true>(a, m1 - m0, R); break;
            case 3: launch_reduce_t<3, true>(a, m1 - m0, R); break;
            case 4: launch_reduce_t<4, true>(a, m1 - m0, R); break;
            case 5: launch_reduce_t<5, true>(a, m1 - m0, R); break;
            case 6: launch_reduce_t<6, true>(a, m1 - m0, R); break;
            case 7: launch_reduce_t<7, true>(a, m1 - m0, R); break;
            case 8: launch_reduce_t<8, true>(a, m1 - m0, R); break;
            default: return fail(CDSGD_ERR_ARG, "P2P correction supports 2..8 ranks");
        }
        LAUNCH_CHECK();
    } else {  // empty shard: still take part in the ready / freed protocol
        k_wait_sum<<<1, 32, 0, R>>>(a.xa, nullptr, 0, nullptr, nullptr, nullptr);
        LAUNCH_CHECK();
        k_flags<<<1, 32, 0, R>>>(a.xa);
        LAUNCH_CHECK();
    }
    if (R != X) {  // the all-gather (copy engines) after the reduce, on the exchange stream
        CUDA_TRY(cudaEventRecord(E->evR, R));
        CUDA_TRY(cudaStreamWaitEvent(X, E->evR, 0));
    }
    if (m1 > m0) {  // 4. all-gather of my sum shard, then wdone[me]
        void* dst[MAX_RANKS_P2P];
        const void* src[MAX_RANKS_P2P];
        size_t bytes[MAX_RANKS_P2P];
        for (int k = 1; k < nr; ++k) {
            const int r = (me + k) % nr;
            dst[k - 1] = at<float>(E->peer[r], E->off_gsum[p & 1]) + m0;
            src[k - 1] = at<const float>(local, E->off_gsum[p & 1]) + m0;
            bytes[k - 1] = static_cast<size_t>(m1 - m0) * sizeof(float);
        }
        const int rc = ce_copies(E, X, nr - 1, dst, src, bytes);
        if (rc != CDSGD_OK) return rc;
    }
    P2PArgs fd{};
    fd.nranks = nr;
    for (int r = 0; r < nr; ++r) fd.publish[r] = at<uint64_t>(E->peer[r], E->off_wdone) + me;
    fd.publish_value = static_cast<uint64_t>(p) + 1;
    {
        const int rc = publish_flags(fd, X);
        if (rc != CDSGD_OK) return rc;
    }
    P2PArgs w{};  // 5. every rank's shard has landed in my gsum
    w.nranks = nr;
    w.wait_flags = at<const uint64_t>(local, E->off_wdone);
    w.wait_value = static_cast<uint64_t>(p) + 1;
    w.err = E->d.err;
    k_wait_sum<<<1, 32, 0, X>>>(w, nullptr, 0, nullptr, nullptr, nullptr);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

// Apply correction round p: reduce my shard from every rank's stage, broadcast W',
// then wait until every shard has landed (W == W_{p+1} everywhere).
int p2p_reduce(cdsgd_engine* E, int64_t p, cudaStream_t C) {
    const int nr = E->d.nranks, me = E->d.rank;
    const int s = E->pend_slot;
    char* local = E->peer[me];
    ReduceArgs a{};
    for (int r = 0; r < nr; ++r) {
        a.stage[r] = E->stage_push ? at<const float>(local, E->off_stage[s]) + static_cast<int64_t>(r) * E->chunk - E->s0
                                   : at<const float>(E->peer[r], E->off_stage[s]);
        a.Wdst[r] = E->peer[r] + E->off_W;
        a.gpart_dst[r] = at<double>(E->peer[r], E->off_gpart) + s * nr + me;
        a.xa.publish[r] = at<uint64_t>(E->peer[r], E->off_gfreed) + s * nr + me;
        a.xb.publish[r] = at<uint64_t>(E->peer[r], E->off_wdone) + me;
    }
    a.W = local + E->off_W;
    a.s0 = E->s0;
    a.s1 = E->s1;
    a.nranks = nr;
    a.eta_g = E->d.eta_global;
    a.inv_n = pow2(nr) ? 1.0 / nr : 0.0;
    a.gacc = E->gacc;
    a.xa.nranks = nr;
    a.xa.wait_flags = at<const uint64_t>(local, E->off_gready) + s * nr;
    a.xa.wait_value = static_cast<uint64_t>(p) + 1;
    a.xa.publish_value = static_cast<uint64_t>(p) + 1;
    a.xa.counter = E->counters + 3;
    a.xa.sc_fence = E->sc_fence;
    a.xa.err = E->d.err;
    a.xb.nranks = nr;
    a.xb.publish_value = static_cast<uint64_t>(p) + 1;
    const long pi = prof_start(E, 7, C);
    const int64_t len = E->s1 - E->s0;
    switch (nr) {
        case 2: launch_reduce_w<2>(a, len, E->d.weights_dtype, C); break;
        case 3: launch_reduce_w<3>(a, len, E->d.weights_dtype, C); break;
        case 4: launch_reduce_w<4>(a, len, E->d.weights_dtype, C); break;
        case 5: launch_reduce_w<5>(a, len, E->d.weights_dtype, C); break;
        case 6: launch_reduce_w<6>(a, len, E->d.weights_dtype, C); break;
        case 7: launch_reduce_w<7>(a, len, E->d.weights_dtype, C); break;
        case 8: launch_reduce_w<8>(a, len, E->d.weights_dtype, C); break;
        default: return fail(CDSGD_ERR_ARG, "P2P correction supports 2..8 ranks");
    }
    LAUNCH_CHECK();
    P2PArgs w{};
    w.nranks = nr;
    w.wait_flags = at<const uint64_t>(local, E->off_wdone);
    w.wait_value = static_cast<uint64_t>(p) + 1;
    w.err = E->d.err;
    double* gn = gnorm_slot(E, p);
    double* clr[2];
    gnorm_clears(E, p + 1, clr);
    prof_stop(E, pi, C);
    const long pw = prof_start(E, 8, C);
    launch_pdl(k_wait_sum, 1, 32, 0, C, w, at<const double>(local, E->off_gpart) + s * nr, nr, gn, clr[0], clr[1]);
    prof_stop(E, pw, C);
    LAUNCH_CHECK();
    return CDSGD_OK;
}

// Start the reduce of correction round t on the exchange stream once this rank's
// stage is written (recorded on C), so it overlaps the next round's quantize.
int p2p_reduce_async(cdsgd_engine* E, int64_t t, cudaStream_t C) {
    CUDA_TRY(cudaEventRecord(E->evQ[t & 1], C));
    CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evQ[t & 1], 0));
    const int rc = p2p_reduce(E, t, E->xs);
    if (rc != CDSGD_OK) return rc;
    CUDA_TRY(cudaEventRecord(E->evX[t & 1], E->xs));
    E->xused[t & 1] = true;
    return CDSGD_OK;
}

// NCCL symmetric-window correction all-reduce of round t (CDSGD_NCCL_SYM): stage g_t into the
// registered buffer unless K2 already did, then all-reduce it on the exchange stream after
// everything on C (the staging) — evX[t] marks completion for K3(t).
int sym_allreduce(cdsgd_engine* E, int64_t t, const float* g, bool staged, cudaStream_t C) {
    const int s = static_cast<int>(t & 1);
    const size_t bytes = 4 * static_cast<size_t>(E->L->n);
    if (!staged) CUDA_TRY(cudaMemcpyAsync(E->sym_stage[s], g, bytes, cudaMemcpyDeviceToDevice, C));
    CUDA_TRY(cudaEventRecord(E->evQ[s], C));
    CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evQ[s], 0));
    const long pi = prof_start(E, 4, E->xs);
    NCCL_TRY(ncclAllReduce(E->sym_stage[s], E->d.gsum[s], static_cast<size_t>(E->L->n), ncclFloat, ncclSum,
                           E->comm->nccl, E->xs));
    prof_stop(E, pi, E->xs);
    CUDA_TRY(cudaEventRecord(E->evX[s], E->xs));
    return CDSGD_OK;
}
StageDst sym_stage_dst(const cdsgd_engine* E, int64_t t) {
    StageDst d{};
    d.chunk = std::max<int64_t>(E->L->n, TILE_ELEMS) + 4;  // one "owner": element e lands at base[0] + e
    d.base[0] = static_cast<float*>(E->sym_stage[t & 1]);
    return d;
}

// Finish round p: wait for its exchange, then K2 (codes) or K3 (full) fused with
// the local update from g_next (nullable).
int engine_apply(cdsgd_engine* E, int64_t p, bool comp, const float* gp, const float* gnext, cudaStream_t C,
                 const StageDst* gs = nullptr, const P2PArgs* xs = nullptr, bool fold = false) {
    const int nr = E->d.nranks;
    if (!comp && E->p2p && E->pcorr) {  // P2P correction: exact sharded reduce, then (optionally) the local update
        int rc = CDSGD_OK;
        if (E->xused[p & 1]) CUDA_TRY(cudaStreamWaitEvent(C, E->evX[p & 1], 0));  // reduce already ran on X
        else rc = p2p_reduce(E, p, C);
        if (rc == CDSGD_OK && gnext != nullptr)
            rc = cdsgd_local_update(E->d.weights, E->d.weights_dtype, gnext, CDSGD_F32, E->d.loc, CDSGD_F32, E->L->n,
                                    E->d.eta_local, C);
        return rc;
    }
    const int64_t soff = nr > 1 && E->xused[p & 1] && !comp ? E->split_off[p & 1] : 0;
    if (nr > 1 && E->xused[p & 1]) CUDA_TRY(cudaStreamWaitEvent(C, soff > 0 ? E->evN[p & 1] : E->evX[p & 1], 0));
    const int64_t rel = p - E->err_base + 1;
    const uint64_t skip_below = rel <= 0 ? 0ull : (static_cast<uint64_t>(rel) << CDSGD_INDEX_BITS);
    double* gn = gnorm_slot(E, p);
    if (gn != nullptr && !gnorm_ahead(E)) CUDA_TRY(cudaMemsetAsync(gn, 0, sizeof(double), C));
    double* clr[2];
    gnorm_clears(E, p + (comp && fold ? 2 : 1), clr);
    float* loc = gnext ? E->d.loc : nullptr;
    if (comp) {
        P2PArgs x{};
        if (E->p2p) {
            const int q = static_cast<int>(p & 1);
            char* local = E->peer[E->d.rank];
            x.nranks = nr;
            for (int r = 0; r < nr; ++r)
                x.publish[r] = reinterpret_cast<uint64_t*>(E->peer[r] + E->off_freed) + q * nr + E->d.rank;
            x.wait_flags = reinterpret_cast<const uint64_t*>(local + E->off_ready) + q * nr;
            x.wait_value = static_cast<uint64_t>(p) + 1;
            x.publish_value = static_cast<uint64_t>(p) + 1;
            x.counter = E->counters + 1;
            x.sc_fence = E->sc_fence;
            x.err = E->d.err;
            if (E->diag_no_wait) x.wait_value = 0;
        }
        double* gn2 = fold ? gnorm_slot(E, p + 1) : nullptr;  // grad-norm slot of the folded correction p+1
        if (gn2 != nullptr && !gnorm_ahead(E)) CUDA_TRY(cudaMemsetAsync(gn2, 0, sizeof(double), C));
        const long pi = prof_start(E, 1, C);
        const int rc = launch_apply_quant(E->L, E->d.weights, E->d.weights_dtype, E->d.gathered[p & 1], nr, words_of(E),
                                          E->d.alpha,
                                          E->d.eta_global, gnext, loc, E->d.eta_local, E->d.err, skip_below, gn,
                                          &E->tab, E->exact, C, &x, gs, xs,
                                          E->sched != nullptr ? E->sched + 2 : nullptr,
                                          fold ? static_cast<float>(E->d.eta_global) : 0.f, gn2, clr);
        prof_stop(E, pi, C);
        return rc;
    }
    const float* gsum = nr > 1 ? E->d.gsum[p & 1] : gp;
    const long pi = prof_start(E, 2, C);
    int rc = launch_apply_full(E->d.weights, E->d.weights_dtype, gsum, nr, soff > 0 ? soff : E->L->n, E->d.eta_global,
                               gnext, loc, E->d.eta_local, E->d.err, skip_below, gn, C, clr);
    if (rc == CDSGD_OK && soff > 0) {  // the copy engines' share, once every rank's shard has landed
        CUDA_TRY(cudaStreamWaitEvent(C, E->evX[p & 1], 0));
        const size_t es = E->d.weights_dtype == CDSGD_F64 ? sizeof(double) : sizeof(float);
        rc = launch_apply_full(static_cast<char*>(E->d.weights) + es * soff, E->d.weights_dtype, gsum + soff, nr,
                               E->L->n - soff, E->d.eta_global, gnext != nullptr ? gnext + soff : nullptr,
                               loc != nullptr ? loc + soff : nullptr, E->d.eta_local, E->d.err, skip_below, gn, C);
    }
    prof_stop(E, pi, C);
    return rc;
}
}  // namespace

extern "C" int cdsgd_engine_create(const cdsgd_engine_desc* d, const cdsgd_layout* L, cdsgd_comm* comm,
                                   cdsgd_engine** out) {
    if (out == nullptr || d == nullptr || L == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    *out = nullptr;
    if (d->algo < CDSGD_ALGO_SSGD || d->algo > CDSGD_ALGO_CDSGD) return fail(CDSGD_ERR_ARG, "unknown algo %d", d->algo);
    if (d->nranks < 1 || d->nranks > MAX_RANKS - 1) return fail(CDSGD_ERR_ARG, "workers must be in [1, %d]", MAX_RANKS - 1);
    if (d->rank < 0 || d->rank >= d->nranks) return fail(CDSGD_ERR_ARG, "rank out of range");
    if (d->k < 1) return fail(CDSGD_ERR_ARG, "k must be >= 1");
    if (d->warmup_n < 0) return fail(CDSGD_ERR_ARG, "warmup_n must be >= 0");
    if (!(d->alpha > 0.0)) return fail(CDSGD_ERR_ARG, "alpha must be > 0");
    if (!(d->eta_global > 0.0) || !(d->eta_local > 0.0)) return fail(CDSGD_ERR_ARG, "learning rates must be > 0");
    if (!wdt_ok(d->weights_dtype)) return fail(CDSGD_ERR_ARG, "weights_dtype must be CDSGD_F32 or CDSGD_F64");
    if (!wdt_ok(d->residual_dtype) || !modes_ok(d->weights_dtype, d->residual_dtype))
        return fail(CDSGD_ERR_ARG, "residual_dtype must be CDSGD_F64, or CDSGD_F32 with fp32 weights (fast mode)");
    if (!d->weights || !d->loc || !d->residual[0] || !d->residual[1] || !d->gathered[0] || !d->gathered[1] || !d->err)
        return fail(CDSGD_ERR_ARG, "NULL engine buffer");
    if (d->nranks > 1 && (comm == nullptr || !d->gsum[0] || !d->gsum[1]))
        return fail(CDSGD_ERR_ARG, "nranks > 1 needs a comm and gsum buffers");
    if (comm != nullptr && (comm->nranks != d->nranks || comm->rank != d->rank))
        return fail(CDSGD_ERR_ARG, "comm rank/size mismatch");
    cdsgd_engine* E = new cdsgd_engine();
    E->d = *d;
    E->L = L;
    E->comm = comm;
    E->uses_local = (d->algo == CDSGD_ALGO_LUSGD || d->algo == CDSGD_ALGO_CDSGD) && !d->bypass_local;
    E->n_warmup = (d->algo == CDSGD_ALGO_LUSGD || d->algo == CDSGD_ALGO_CDSGD) ? d->warmup_n : 0;
    E->exact = alpha_exact(d->alpha, d->nranks) ? 1 : 0;
    build_tab(E->tab, d->alpha, d->eta_global, d->nranks);
    E->compute_is_loc = E->uses_local && E->n_warmup == 0;
    {
        const char* nf = getenv("CDSGD_NO_FUSE");
        E->fuse = d->nranks == 1 && !(nf != nullptr && nf[0] == '1');
        // A/B knob: plain launch of the apply beside a correction all-reduce (measured no gain at
        // N=2: 296 vs 301 Gelem/s — the apply's CTAs fill every SM either way)
        // The correction all-reduce's NCCL kernel must get SMs before the apply (K2) grid fills
        // them all: a marker kernel on the exchange stream gates the apply, so NCCL's kernel is
        // eligible first and overlaps K2 (it used to start only when K2 retired). Measured
        // +2.5 % at N=2, +5-7 % at N=4 (436 vs 413 Gelem/s). CDSGD_AR_FIRST=0 disables.
        const char* cd = getenv("CDSGD_CE_DEFER");
        E->ce_defer = !(cd != nullptr && cd[0] == '0');
        const char* af = getenv("CDSGD_AR_FIRST");
        E->ar_first = !(af != nullptr && af[0] == '0');
        const char* fa = getenv("CDSGD_FUSE_AFTER_AR");
        E->fuse_after_ar = fa != nullptr && fa[0] == '1';
        const char* rs = getenv("CDSGD_RESERVE_SMS");
        E->reserve_sms = rs != nullptr ? std::max(0, atoi(rs)) : 0;
        const char* pa = getenv("CDSGD_PLAIN_AFTER_AR");
        E->plain_after_ar = pa != nullptr && pa[0] == '1';
        const char* sa = getenv("CDSGD_SPLIT_APPLY");
        E->split_apply = sa != nullptr && sa[0] == '1';
        const char* ns = getenv("CDSGD_STATIC_SCHED");
        if (!(ns != nullptr && ns[0] == '1')) {
            if (cudaMalloc(&E->sched, 4 * sizeof(unsigned int)) != cudaSuccess ||
                cudaMemset(E->sched, 0, 4 * sizeof(unsigned int)) != cudaSuccess)
                E->sched = nullptr;
        }
    }
    cudaError_t e = cudaSuccess;
    if (d->gnorm_sq != nullptr && d->gnorm_ring > 0)  // slots are zeroed ahead in-kernel from here on
        e = cudaMemset(d->gnorm_sq, 0, static_cast<size_t>(d->gnorm_ring) * sizeof(double));
    if (d->nranks > 1 && e == cudaSuccess) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        e = cudaStreamCreateWithPriority(&E->xs, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&E->xs2, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evC, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evfork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evG, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evR, cudaEventDisableTiming);
        for (int i = 0; i < d->nranks && i < MAX_RANKS_P2P && e == cudaSuccess; ++i) {
            e = cudaStreamCreateWithPriority(&E->xsc[i], cudaStreamNonBlocking, hi);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evc[i], cudaEventDisableTiming);
        }
        // per-peer copy streams: measured no gain at N=4 (414 vs 420 Gelem/s serial; the copy
        // engines' share takes as long either way) -> off by default, CDSGD_CE_PARALLEL=1 enables
        const char* cs = getenv("CDSGD_CE_PARALLEL");
        E->ce_parallel = cs != nullptr && cs[0] == '1';
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&E->evQ[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evX[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&E->evN[i], cudaEventDisableTiming);
        }
    }
    if (e != cudaSuccess) {
        cdsgd_engine_destroy(E);
        return fail(CDSGD_ERR_CUDA, "engine streams/events: %s", cudaGetErrorString(e));
    }
    *out = E;
    return CDSGD_OK;
}

namespace {
int64_t align256(int64_t v) { return (v + 255) & ~int64_t(255); }
// Shard owned by each rank in the P2P exact correction: ceil(n/N) rounded up to 4 elements.
int64_t p2p_chunk(int32_t nranks, int64_t n) { return (((n + nranks - 1) / nranks) + 3) / 4 * 4; }
// Symmetric buffer: codes slot 0 | slot 1 | ready[2][N] | freed[2][N] | W [n] |
// recv 0 [N][chunk] | recv 1 [N][chunk] | gready[2][N] | gfreed[2][N] | wdone[N] | gpart[2][N] |
// gsum 0 [n] | gsum 1 [n] | end
// Alignment of the streamed arrays inside the symmetric buffer (CDSGD_P2P_ALIGN bytes, a power
// of two >= 256; default 256): W, the staging rows and gsum start on this boundary.
int64_t p2p_align() {
    static const int64_t v = [] {
        const char* e = getenv("CDSGD_P2P_ALIGN");
        const long long a = e != nullptr ? atoll(e) : 256;
        return a >= 256 && (a & (a - 1)) == 0 ? static_cast<int64_t>(a) : int64_t(256);
    }();
    return v;
}
void p2p_offsets(int32_t nranks, int64_t n, int64_t words, int64_t* off /* [14] */) {
    const int64_t A = p2p_align();
    auto up = [A](int64_t x) { return (x + A - 1) / A * A; };
    const int64_t flags = align256(2 * nranks * 8);
    const int64_t recv = up(4 * static_cast<int64_t>(nranks) * p2p_chunk(nranks, n));
    off[0] = 0;
    off[1] = align256(static_cast<int64_t>(nranks) * words * 4);
    off[2] = 2 * off[1];
    off[3] = off[2] + flags;
    off[4] = up(off[3] + flags);
    off[5] = off[4] + up(8 * n);        // W replica (sized for fp64 weights)
    off[6] = off[5] + recv;
    off[7] = off[6] + recv;
    off[8] = off[7] + flags;
    off[9] = off[8] + flags;
    off[10] = off[9] + align256(nranks * 8);
    off[11] = up(off[10] + flags);      // gsum 0
    off[12] = off[11] + up(4 * n);      // gsum 1
    off[13] = off[12] + up(4 * n);      // end
}
}  // namespace

extern "C" int64_t cdsgd_p2p_bytes(int32_t nranks, int64_t n, int64_t words) {
    int64_t off[14];
    p2p_offsets(nranks, n, words, off);
    return off[13];
}

extern "C" int64_t cdsgd_p2p_weights_offset(int32_t nranks, int64_t n, int64_t words) {
    int64_t off[14];
    p2p_offsets(nranks, n, words, off);
    return off[4];
}

// Native symmetric buffer: cudaMalloc'd, zero-filled, exported as a CUDA IPC handle that
// the other ranks of the box map with cudaIpcOpenMemHandle (peer access enabled lazily).
static_assert(sizeof(cudaIpcMemHandle_t) == CDSGD_P2P_HANDLE_BYTES, "IPC handle size");
extern "C" int cdsgd_p2p_buffer_alloc(int64_t bytes, void** ptr, void* handle) {
    if (ptr == nullptr || handle == nullptr || bytes <= 0) return fail(CDSGD_ERR_ARG, "bad p2p buffer arguments");
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
    cudaError_t e = cudaMemset(p, 0, static_cast<size_t>(bytes));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaIpcMemHandle_t h{};
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return fail(CDSGD_ERR_CUDA, "p2p buffer: %s", cudaGetErrorString(e));
    }
    std::memcpy(handle, &h, sizeof(h));
    *ptr = p;
    return CDSGD_OK;
}
extern "C" int cdsgd_p2p_buffer_open(const void* handle, void** ptr) {
    if (ptr == nullptr || handle == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return CDSGD_OK;
}
extern "C" int cdsgd_p2p_buffer_close(void* peer_ptr) {
    if (peer_ptr == nullptr) return CDSGD_OK;
    CUDA_TRY(cudaIpcCloseMemHandle(peer_ptr));
    return CDSGD_OK;
}
extern "C" int cdsgd_p2p_buffer_free(void* ptr) {
    if (ptr == nullptr) return CDSGD_OK;
    CUDA_TRY(cudaFree(ptr));
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_attach_p2p(cdsgd_engine* E, void* const* peer_bases, int32_t nranks,
                                       int32_t exact_correction) {
    if (E == nullptr || peer_bases == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    if (nranks != E->d.nranks || nranks < 2) return fail(CDSGD_ERR_ARG, "attach_p2p needs nranks == workers >= 2");
    if (nranks > MAX_RANKS_P2P) return fail(CDSGD_ERR_ARG, "fused exchange supports at most %d ranks", MAX_RANKS_P2P);
    if (E->t != 0) return fail(CDSGD_ERR_STATE, "attach_p2p must precede the first round");
    for (int r = 0; r < nranks; ++r) {
        if (peer_bases[r] == nullptr || (reinterpret_cast<uintptr_t>(peer_bases[r]) & 255) != 0)
            return fail(CDSGD_ERR_ARG, "peer base %d is NULL or not 256-byte aligned", r);
        E->peer[r] = static_cast<char*>(peer_bases[r]);
    }
    int64_t off[14];
    p2p_offsets(nranks, E->L->n, E->L->nwords, off);
    E->off_slot[0] = off[0];
    E->off_slot[1] = off[1];
    E->off_ready = off[2];
    E->off_freed = off[3];
    E->off_W = off[4];
    E->off_stage[0] = off[5];
    E->off_stage[1] = off[6];
    E->off_gready = off[7];
    E->off_gfreed = off[8];
    E->off_wdone = off[9];
    E->off_gpart = off[10];
    E->off_gsum[0] = off[11];
    E->off_gsum[1] = off[12];
    char* local = E->peer[E->d.rank];
    // correction sums land in symmetric memory (the NCCL-free all-reduce stores shards there)
    E->d.gsum[0] = reinterpret_cast<float*>(local + E->off_gsum[0]);
    E->d.gsum[1] = reinterpret_cast<float*>(local + E->off_gsum[1]);
    E->d.gathered[0] = reinterpret_cast<uint32_t*>(local + E->off_slot[0]);
    E->d.gathered[1] = reinterpret_cast<uint32_t*>(local + E->off_slot[1]);
    // the W replica moves into symmetric memory when peers store their W' shards into it (the
    // exact correction); CDSGD_W_SYMMETRIC=1 moves it in every P2P mode (A/B; worker.py follows
    // the same rule for its view of W)
    void* wsym = local + E->off_W;
    const char* wsm = getenv("CDSGD_W_SYMMETRIC");
    const bool w_move = exact_correction != 0 || (wsm != nullptr && wsm[0] == '1');
    if (w_move && wsym != E->d.weights) {
        const size_t wb = E->d.weights_dtype == CDSGD_F64 ? 8 : 4;
        CUDA_TRY(cudaMemcpy(wsym, E->d.weights, wb * E->L->n, cudaMemcpyDeviceToDevice));
        E->d.weights = wsym;
    }
    const int64_t chunk = p2p_chunk(nranks, E->L->n);
    E->chunk = chunk;
    E->s0 = std::min<int64_t>(E->L->n, chunk * E->d.rank);
    E->s1 = std::min<int64_t>(E->L->n, E->s0 + chunk);
    if (E->counters == nullptr) {
        CUDA_TRY(cudaMalloc(&E->counters, 4 * sizeof(unsigned int)));
        CUDA_TRY(cudaMemset(E->counters, 0, 4 * sizeof(unsigned int)));
    }
    if (E->gacc == nullptr) {
        CUDA_TRY(cudaMalloc(&E->gacc, sizeof(double)));
        CUDA_TRY(cudaMemset(E->gacc, 0, sizeof(double)));
    }
    E->p2p = true;
    E->pcorr = exact_correction != 0;
    {
        const char* nr = getenv("CDSGD_DIAG_NO_REMOTE_CODES");  // timing diagnostic only: wrong results
        E->diag_local_codes = nr != nullptr && nr[0] == '1';
        const char* nw = getenv("CDSGD_DIAG_NO_WAIT");  // timing diagnostic only: races, wrong results
        E->diag_no_wait = nw != nullptr && nw[0] == '1';
        // measured best share on B200: 0.3 at N=2 (+4 %), 0.55 at N=4 (+5 %); CDSGD_CE_FRAC overrides
        // below ~8M elements the copy-engine phases' fixed costs (peer copies, flag kernels,
        // waits) outweigh the contention they save (1M elements: 133 -> 101 Gelem/s at N=4)
        const char* cf = getenv("CDSGD_CE_FRAC");
        const double dflt = E->L->n < (int64_t(1) << 23) ? 0.0 : (nranks == 2 ? 0.3 : 0.55);
        E->ce_frac = exact_correction ? 0.0 : (cf == nullptr ? dflt : std::min(1.0, std::max(0.0, atof(cf))));
        const char* sp = getenv("CDSGD_STAGE_PUSH");
        E->stage_push = sp != nullptr && sp[0] == '1';
        const char* sf = getenv("CDSGD_SC_FENCE");
        E->sc_fence = sf != nullptr && sf[0] == '1';
    }
    {
        const char* nf = getenv("CDSGD_NO_FUSE");
        E->fuse = !(nf != nullptr && nf[0] == '1');
    }
    {
        const char* ns = getenv("CDSGD_NCCL_SYM");
        if (ns != nullptr && ns[0] == '1' && !exact_correction && E->comm != nullptr) {
            const size_t bytes = 4 * static_cast<size_t>(E->L->n);
            for (int i = 0; i < 2; ++i) {
                NCCL_TRY(ncclMemAlloc(&E->sym_stage[i], bytes));
                NCCL_TRY(ncclMemAlloc(&E->sym_gsum[i], bytes));
                NCCL_TRY(ncclCommWindowRegister(E->comm->nccl, E->sym_stage[i], bytes, &E->win[2 * i],
                                                NCCL_WIN_COLL_SYMMETRIC));
                NCCL_TRY(ncclCommWindowRegister(E->comm->nccl, E->sym_gsum[i], bytes, &E->win[2 * i + 1],
                                                NCCL_WIN_COLL_SYMMETRIC));
                E->d.gsum[i] = static_cast<float*>(E->sym_gsum[i]);
            }
            E->nccl_sym = true;
            E->ce_frac = 0.0;
        }
    }
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_join(cdsgd_engine* E, void* stream) {
    if (E == nullptr) return fail(CDSGD_ERR_ARG, "NULL engine");
    const int rf = p2p_ce_finish(E, S(stream));  // a deferred copy-engine half is part of "issued"
    if (rf != CDSGD_OK) return rf;
    if (E->xs == nullptr || E->t == 0) return CDSGD_OK;
    for (int64_t u = E->t - 1; u >= 0 && u >= E->t - 2; --u)
        if (E->xused[u & 1]) CUDA_TRY(cudaStreamWaitEvent(S(stream), E->evX[u & 1], 0));
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_profile_begin(cdsgd_engine* E) {
    if (E == nullptr) return fail(CDSGD_ERR_ARG, "NULL engine");
    E->prof = true;
    E->ev_used = 0;
    E->prof_marks.clear();
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_profile_end(cdsgd_engine* E, double* out) {
    if (E == nullptr || out == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    E->prof = false;
    for (int i = 0; i < 22; ++i) out[i] = 0.0;
    for (const auto& m : E->prof_marks) {
        CUDA_TRY(cudaEventSynchronize(E->ev_pool[m.second + 1]));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, E->ev_pool[m.second], E->ev_pool[m.second + 1]));
        out[2 * m.first] += ms;
        out[2 * m.first + 1] += 1.0;
    }
    E->prof_marks.clear();
    E->ev_used = 0;
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_destroy(cdsgd_engine* E) {
    if (E == nullptr) return CDSGD_OK;
    if (E->xs) cudaStreamSynchronize(E->xs);
    if (E->xs2) cudaStreamSynchronize(E->xs2);
    for (cudaEvent_t ev : E->ev_pool) cudaEventDestroy(ev);
    if (E->evC) cudaEventDestroy(E->evC);
    for (int i = 0; i < 2; ++i) {
        if (E->evQ[i]) cudaEventDestroy(E->evQ[i]);
        if (E->evX[i]) cudaEventDestroy(E->evX[i]);
        if (E->evN[i]) cudaEventDestroy(E->evN[i]);
    }
    if (E->xs) cudaStreamDestroy(E->xs);
    if (E->xs2) cudaStreamDestroy(E->xs2);
    for (int i = 0; i < MAX_RANKS_P2P; ++i) {
        if (E->xsc[i]) {
            cudaStreamSynchronize(E->xsc[i]);
            cudaStreamDestroy(E->xsc[i]);
        }
        if (E->evc[i]) cudaEventDestroy(E->evc[i]);
    }
    if (E->evfork) cudaEventDestroy(E->evfork);
    if (E->evG) cudaEventDestroy(E->evG);
    if (E->evR) cudaEventDestroy(E->evR);
    for (int i = 0; i < 4; ++i)
        if (E->win[i] != nullptr && E->comm != nullptr) ncclCommWindowDeregister(E->comm->nccl, E->win[i]);
    for (int i = 0; i < 2; ++i) {
        if (E->sym_stage[i]) ncclMemFree(E->sym_stage[i]);
        if (E->sym_gsum[i]) ncclMemFree(E->sym_gsum[i]);
    }
    if (E->counters) cudaFree(E->counters);
    if (E->gacc) cudaFree(E->gacc);
    if (E->sched) cudaFree(E->sched);
    delete E;
    return CDSGD_OK;
}

extern "C" double cdsgd_engine_ce_fraction(const cdsgd_engine* E) { return E != nullptr && E->p2p ? E->ce_frac : 0.0; }

extern "C" int cdsgd_engine_round_compressed(const cdsgd_engine* E, int64_t t) {
    bool c = false;
    if (E == nullptr || round_compressed(E, t, &c) != CDSGD_OK) return -1;
    return c ? 1 : 0;
}

// NVTX range per engine step, named by the round's kind (host-side phase markers for nsys-style
// timelines: "cdsgd round (compressed)" / "(correction)")
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

extern "C" int cdsgd_engine_step(cdsgd_engine* E, const float* g, void* stream) {
    if (E == nullptr || g == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    bool comp_ = false;
    round_compressed(E, E->t, &comp_);
    const NvtxRange nvtx_(comp_ ? "cdsgd round (compressed)" : "cdsgd round (correction / full)");
    if (E->failed) return fail(CDSGD_ERR_STATE, "engine failed at an earlier round; see cdsgd_engine_check");
    if (E->t - E->err_base >= (int64_t(1) << 23))
        return fail(CDSGD_ERR_STATE, "cdsgd_engine_check must run at least every 2^23 rounds");
    cudaStream_t C = S(stream);
    const int64_t t = E->t;
    bool comp = false;
    int rc = p2p_ce_finish(E, C);  // the previous correction's deferred copy-engine reduce + all-gather
    if (rc != CDSGD_OK) return rc;
    rc = round_compressed(E, t, &comp);
    if (rc != CDSGD_OK) return rc;
    const int nr = E->d.nranks;
    const int64_t nw = words_of(E);
    uint32_t* mine = E->d.gathered[t & 1] + static_cast<int64_t>(E->d.rank) * nw;
    const bool sync_path0 = !E->uses_local || t < E->n_warmup - 1;
    if (E->p2p && E->pcorr && E->pending && !E->pend_comp) {
        // ---- previous round was a P2P correction whose reduce runs on stream X:
        // quantize(t) overlaps it; then loc_{t+1} = W_t - eta_l*g_t once W_t is complete
        E->rlog.push_back(static_cast<int8_t>(E->rcur));
        if (comp) {
            const int p = static_cast<int>(t & 1);
            char* local = E->peer[E->d.rank];
            P2PArgs x{};
            x.nranks = nr;
            for (int r = 0; r < nr; ++r) {
                x.dst[r] = reinterpret_cast<uint32_t*>(E->peer[E->diag_local_codes ? E->d.rank : r] + E->off_slot[p]) +
                           static_cast<int64_t>(E->d.rank) * nw;
                x.publish[r] = reinterpret_cast<uint64_t*>(E->peer[r] + E->off_ready) + p * nr + E->d.rank;
            }
            x.wait_flags = reinterpret_cast<const uint64_t*>(local + E->off_freed) + p * nr;
            x.wait_value = E->last_use[p] >= 0 ? static_cast<uint64_t>(E->last_use[p]) + 1 : 0;
            x.publish_value = static_cast<uint64_t>(t) + 1;
            x.counter = E->counters;
            x.sc_fence = E->sc_fence;
            if (E->diag_no_wait) x.wait_value = 0;
            x.err = E->d.err;
            const uint64_t tag = static_cast<uint64_t>(t - E->err_base) << CDSGD_INDEX_BITS;
            const long pi = prof_start(E, 0, C);
            rc = launch_quant_tma_rdt(g, E->d.residual_dtype, E->d.residual[E->rcur], E->d.residual[E->rcur ^ 1], mine,
                                      E->L->tab(), E->d.alpha, E->d.err, tag, C, x);
            if (rc == CDSGD_OK) {
                g_launches.fetch_add(1, std::memory_order_relaxed);
                const cudaError_t le = cudaGetLastError();
                if (le != cudaSuccess) rc = fail(CDSGD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(le));
            }
            prof_stop(E, pi, C);
            if (rc != CDSGD_OK) return rc;
            E->last_use[p] = t;
            E->rcur ^= 1;
        }
        rc = engine_apply(E, E->pend_t, false, E->pend_grad, g, C);  // wait X, loc = W_t - eta_l*g_t
        if (rc != CDSGD_OK) return rc;
        E->xused[t & 1] = false;
        if (!comp) {  // another correction round: stage g_t and start its reduce on X
            rc = p2p_stage(E, t, g, C);
            if (rc != CDSGD_OK) return rc;
            rc = p2p_reduce_async(E, t, C);
            if (rc != CDSGD_OK) return rc;
        }
        E->pending = true;
        E->pend_t = t;
        E->pend_comp = comp;
        E->pend_grad = g;
        E->compute_is_loc = true;
        E->t = t + 1;
        return CDSGD_OK;
    }
    // N>1, the round after a correction: apply the correction (its all-reduced sum) fused with
    // this round's quantize, AFTER the all-reduce, instead of quantizing beside it and running
    // K3 afterwards (CDSGD_FUSE_AFTER_AR; p2p exchange with the NCCL / copy-engine all-reduce)
    const bool fuse_after_ar = E->fuse_after_ar && E->pending && !E->pend_comp && nr > 1 && E->p2p && !E->pcorr &&
                               E->xused[E->pend_t & 1];
    if (E->fuse && comp && !sync_path0 &&
        (fuse_after_ar || (E->pending ? (E->pend_comp || nr == 1) : nr == 1))) {
        // ---- one kernel: apply(t-1) fused with quantize(t); both read g_t once. With nothing
        // pending (first local round, or N=1 after a folded correction) the apply part is just
        // loc_{t+1} = W_t - eta_l*g_t.
        const bool has_pend = E->pending;
        const int64_t pnd = has_pend ? E->pend_t : t;
        FusedArgs a{};
        a.g = g;
        a.r_in = E->d.residual[E->rcur];
        a.r_out = E->d.residual[E->rcur ^ 1];
        a.words = mine;
        a.alpha = E->d.alpha;
        a.tag = static_cast<uint64_t>(t - E->err_base) << CDSGD_INDEX_BITS;
        a.W = E->d.weights;
        a.loc = E->d.loc;
        a.gathered = E->d.gathered[pnd & 1];
        a.stride = nw;
        // N=1 correction round: the mean is g_{t-1} itself; N>1: the all-reduced sum
        a.gsum = fuse_after_ar ? E->d.gsum[pnd & 1] : E->pend_grad;
        if (fuse_after_ar) CUDA_TRY(cudaStreamWaitEvent(C, E->evX[pnd & 1], 0));
        a.scale = static_cast<float>(E->d.eta_global / nr);
        a.inv_n = 1.0 / nr;
        a.eta_l = static_cast<float>(E->d.eta_local);
        a.exact = E->exact;
        a.eta_g_d = E->d.eta_global;
        a.eta_l_d = E->d.eta_local;
        a.nranks = nr;
        a.inv_n_or_zero = pow2(nr) ? 1.0 / nr : 0.0;
        const int64_t rel = pnd - E->err_base + 1;
        a.skip_below = rel <= 0 ? 0ull : (static_cast<uint64_t>(rel) << CDSGD_INDEX_BITS);
        a.err = E->d.err;
        a.sched = E->sched;
        if (has_pend) {
            a.gnorm = gnorm_slot(E, pnd);
            if (a.gnorm != nullptr && !gnorm_ahead(E)) CUDA_TRY(cudaMemsetAsync(a.gnorm, 0, sizeof(double), C));
            gnorm_clears(E, pnd + 1, a.gclear);
        }
        if (!has_pend) a.skip_below = 0;
        if (E->p2p) {
            const int p = static_cast<int>(t & 1), q = static_cast<int>(pnd & 1);
            char* local = E->peer[E->d.rank];
            a.xq.nranks = a.xa.nranks = nr;
            for (int r = 0; r < nr; ++r) {
                a.xq.dst[r] = reinterpret_cast<uint32_t*>(E->peer[E->diag_local_codes ? E->d.rank : r] + E->off_slot[p]) +
                              static_cast<int64_t>(E->d.rank) * nw;
                a.xq.publish[r] = reinterpret_cast<uint64_t*>(E->peer[r] + E->off_ready) + p * nr + E->d.rank;
                a.xa.publish[r] = reinterpret_cast<uint64_t*>(E->peer[r] + E->off_freed) + q * nr + E->d.rank;
            }
            a.xq.wait_flags = reinterpret_cast<const uint64_t*>(local + E->off_freed) + p * nr;
            a.xq.wait_value = E->last_use[p] >= 0 ? static_cast<uint64_t>(E->last_use[p]) + 1 : 0;
            a.xq.publish_value = static_cast<uint64_t>(t) + 1;
            a.xq.counter = E->counters;
            a.xq.sc_fence = E->sc_fence;
            a.xq.err = E->d.err;
            a.xa.wait_flags = reinterpret_cast<const uint64_t*>(local + E->off_ready) + q * nr;
            a.xa.wait_value = static_cast<uint64_t>(pnd) + 1;
            a.xa.publish_value = static_cast<uint64_t>(pnd) + 1;
            a.xa.counter = E->counters;
            a.xa.sc_fence = E->sc_fence;
            a.xa.err = E->d.err;
            if (E->diag_no_wait) a.xq.wait_value = a.xa.wait_value = 0;
            if (!has_pend || fuse_after_ar) a.xa.nranks = 0;  // no codes to consume (local-only / full apply)
            E->last_use[p] = t;
        }
        E->rlog.push_back(static_cast<int8_t>(E->rcur));
        const long pi = prof_start(E, has_pend ? 5 : 9, C);
        const int ap = !has_pend ? APPLY_L : (E->pend_comp ? APPLY_Q : APPLY_F);
        rc = launch_fused(nr, ap, E->d.weights_dtype, E->d.residual_dtype, a, E->L->tab(), E->tab, C);
        prof_stop(E, pi, C);
        if (rc != CDSGD_OK) return rc;
        E->rcur ^= 1;
        E->xused[t & 1] = false;
        E->pending = true;
        E->pend_t = t;
        E->pend_comp = true;
        E->pend_grad = g;
        E->compute_is_loc = true;
        E->t = t + 1;
        return CDSGD_OK;
    }
    // 1. this round's contribution (K1 on compressed rounds); right after a correction round
    // its all-reduce is still in flight (ReserveScope: leave SMs to its CTAs)
    E->rlog.push_back(static_cast<int8_t>(E->rcur));
    const ReserveScope reserve1(E->ar_round >= 0 && E->ar_round == t - 1 ? E->reserve_sms : 0);
    if (comp) {
        const uint64_t tag = static_cast<uint64_t>(t - E->err_base) << CDSGD_INDEX_BITS;
        const long pi = prof_start(E, 0, C);
        if (E->p2p) {
            // K1 with the all-gather fused in: words go straight into every rank's slot p
            const int p = static_cast<int>(t & 1);
            char* local = E->peer[E->d.rank];
            P2PArgs x{};
            x.nranks = nr;
            for (int r = 0; r < nr; ++r) {
                x.dst[r] = reinterpret_cast<uint32_t*>(E->peer[r] + E->off_slot[p]) + static_cast<int64_t>(E->d.rank) * nw;
                x.publish[r] = reinterpret_cast<uint64_t*>(E->peer[r] + E->off_ready) + p * nr + E->d.rank;
            }
            x.wait_flags = reinterpret_cast<const uint64_t*>(local + E->off_freed) + p * nr;
            x.wait_value = E->last_use[p] >= 0 ? static_cast<uint64_t>(E->last_use[p]) + 1 : 0;
            x.publish_value = static_cast<uint64_t>(t) + 1;
            x.counter = E->counters;
            x.sc_fence = E->sc_fence;
            if (E->diag_no_wait) x.wait_value = 0;
            x.err = E->d.err;
            rc = launch_quant_tma_rdt(g, E->d.residual_dtype, E->d.residual[E->rcur], E->d.residual[E->rcur ^ 1], mine,
                                      E->L->tab(), E->d.alpha, E->d.err, tag, C, x);
            if (rc == CDSGD_OK) {
                g_launches.fetch_add(1, std::memory_order_relaxed);
                const cudaError_t le = cudaGetLastError();
                if (le != cudaSuccess) rc = fail(CDSGD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(le));
            }
            E->last_use[p] = t;
        } else {
            if (E->d.residual_dtype == CDSGD_F32)
                rc = cdsgd_quantize_f32r(E->L, g, static_cast<const float*>(E->d.residual[E->rcur]),
                                         static_cast<float*>(E->d.residual[E->rcur ^ 1]), mine, E->d.alpha, E->d.err,
                                         tag, C);
            else
                rc = cdsgd_quantize(E->L, g, CDSGD_F32, static_cast<const double*>(E->d.residual[E->rcur]),
                                    static_cast<double*>(E->d.residual[E->rcur ^ 1]), mine, E->d.alpha, E->d.err, tag,
                                    C);
        }
        prof_stop(E, pi, C);
        if (rc != CDSGD_OK) return rc;
        E->rcur ^= 1;
    }
    // 2. exchange round t on the engine's stream (codes are already delivered when fused)
    E->split_off[t & 1] = 0;
    E->xused[t & 1] = nr > 1 && (!E->p2p || (!comp && !E->pcorr));
    // the split pays only when the all-reduce overlaps compute: a synchronous round (ssgd,
    // warm-up) waits for it at once, and NCCL alone is faster there (ssgd N=4: 0.57 vs 0.69 ms)
    if (E->xused[t & 1] && !comp && E->p2p && E->ce_frac > 0.0 && !sync_path0) {
        // correction all-reduce split between NCCL (stream X, SMs) and the copy engines
        // (stream X2): the copy engines barely contend with the compute kernels
        const int64_t n = E->L->n;
        int64_t cnt = std::min<int64_t>(n, static_cast<int64_t>(E->ce_frac * n) / 4 * 4);
        int64_t off = n - cnt;
        // split apply: NCCL's share ends on a tile boundary (both K3 halves keep the TMA path)
        const int64_t off_t = off / TILE_ELEMS * TILE_ELEMS;
        const bool split = E->split_apply && off_t > 0 && (n - off_t) % 4 == 0;
        if (split) {
            off = off_t;
            cnt = n - off;
        }
        CUDA_TRY(cudaEventRecord(E->evQ[t & 1], C));
        CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evQ[t & 1], 0));
        CUDA_TRY(cudaStreamWaitEvent(E->xs2, E->evQ[t & 1], 0));
        if (E->ar_first) {  // the apply on C waits for this marker: NCCL's kernel is eligible first
            k_noop<<<1, 32, 0, E->xs>>>();
            LAUNCH_CHECK();
            CUDA_TRY(cudaEventRecord(E->evG, E->xs));
        }
        const long pi = prof_start(E, 4, E->xs);
        if (off > 0)
            NCCL_TRY(ncclAllReduce(g, E->d.gsum[t & 1], static_cast<size_t>(off), ncclFloat, ncclSum, E->comm->nccl,
                                   E->xs));
        prof_stop(E, pi, E->xs);
        if (split) {
            CUDA_TRY(cudaEventRecord(E->evN[t & 1], E->xs));
            E->split_off[t & 1] = off;
        }
        const long pc = prof_start(E, 10, E->xs2);
        rc = p2p_ce_allreduce(E, t, g, E->xs2, off, cnt);
        if (rc != CDSGD_OK) return rc;
        prof_stop(E, pc, E->xs2);
        if (!E->ce_pend.on) {  // (deferred: the next step's p2p_ce_finish records evX)
            CUDA_TRY(cudaEventRecord(E->evC, E->xs2));
            CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evC, 0));
            CUDA_TRY(cudaEventRecord(E->evX[t & 1], E->xs));
        }
    } else if (E->xused[t & 1] && !comp && E->nccl_sym) {
        // deferred until after the apply below, which stages g_t into the registered buffer
    } else if (E->xused[t & 1]) {
        CUDA_TRY(cudaEventRecord(E->evQ[t & 1], C));
        CUDA_TRY(cudaStreamWaitEvent(E->xs, E->evQ[t & 1], 0));
        if (E->ar_first && !comp) {
            k_noop<<<1, 32, 0, E->xs>>>();
            LAUNCH_CHECK();
            CUDA_TRY(cudaEventRecord(E->evG, E->xs));
        }
        const long pi = prof_start(E, 4, E->xs);
        if (comp) {
            NCCL_TRY(ncclAllGather(mine, E->d.gathered[t & 1], static_cast<size_t>(nw), ncclUint32, E->comm->nccl, E->xs));
        } else {
            NCCL_TRY(ncclAllReduce(g, E->d.gsum[t & 1], static_cast<size_t>(E->L->n), ncclFloat, ncclSum,
                                   E->comm->nccl, E->xs));
        }
        prof_stop(E, pi, E->xs);
        CUDA_TRY(cudaEventRecord(E->evX[t & 1], E->xs));
    }
    // 3. apply
    const PlainLaunchScope plain(E->xused[t & 1] && !comp && E->plain_after_ar);
    // the all-reduce of correction round t is in flight from here until K3(t) waits for it:
    // the apply below (K2(t-1)) and the next round's quantize run beside it
    if (E->xused[t & 1] && !comp) E->ar_round = t;
    const ReserveScope reserve3(E->xused[t & 1] && !comp ? E->reserve_sms : 0);
    const bool sync_path = !E->uses_local || t < E->n_warmup - 1;
    const bool sym_ar = E->xused[t & 1] && !comp && E->nccl_sym;
    if (E->ar_first && E->xused[t & 1] && !comp && !E->nccl_sym) CUDA_TRY(cudaStreamWaitEvent(C, E->evG, 0));
    if (sync_path) {
        if (E->pending) return fail(CDSGD_ERR_STATE, "internal: pending round on the synchronous path");
        if (sym_ar) {
            rc = sym_allreduce(E, t, g, false, C);
            if (rc != CDSGD_OK) return rc;
        }
        if (!comp && E->p2p && E->pcorr) {
            rc = p2p_stage(E, t, g, C);
            if (rc != CDSGD_OK) return rc;
        }
        rc = engine_apply(E, t, comp, g, nullptr, C);
        if (rc != CDSGD_OK) return rc;
        E->compute_is_loc = false;
    } else {
        bool staged = false;
        if (E->pending && !comp && E->p2p && E->pcorr && E->pend_comp) {
            // correction round after a compressed one: K2(t-1) also writes g_t to the stage
            StageDst dst{};
            P2PArgs xs{};
            prepare_stage(E, t, &dst, &xs);
            rc = engine_apply(E, E->pend_t, E->pend_comp, E->pend_grad, g, C, &dst, &xs);
            staged = true;
        } else if (E->pending && !comp && nr == 1 && E->pend_comp && E->fuse) {
            // N=1: this correction round's mean is g_t itself -> apply it in the same pass
            rc = engine_apply(E, E->pend_t, true, E->pend_grad, g, C, nullptr, nullptr, /*fold=*/true);
            if (rc != CDSGD_OK) return rc;
            E->pending = false;
            E->compute_is_loc = true;
            E->t = t + 1;
            return CDSGD_OK;
        } else if (E->pending && sym_ar && E->pend_comp) {
            // K2(t-1) streams g_t for the local update anyway: it also stages it for the all-reduce
            const StageDst dst = sym_stage_dst(E, t);
            rc = engine_apply(E, E->pend_t, E->pend_comp, E->pend_grad, g, C, &dst, nullptr);
            if (rc == CDSGD_OK) rc = sym_allreduce(E, t, g, true, C);
            staged = true;
        } else if (E->pending) {
            rc = engine_apply(E, E->pend_t, E->pend_comp, E->pend_grad, g, C);
        } else {
            // first local round: loc_{t+1} = W_t - eta_l * g_t (engine.py:380-382, 385-391)
            const long pi = prof_start(E, 3, C);
            rc = cdsgd_local_update(E->d.weights, E->d.weights_dtype, g, CDSGD_F32, E->d.loc, CDSGD_F32, E->L->n,
                                    E->d.eta_local, stream);
            prof_stop(E, pi, C);
        }
        if (rc != CDSGD_OK) return rc;
        if (sym_ar && !staged) {
            rc = sym_allreduce(E, t, g, false, C);
            if (rc != CDSGD_OK) return rc;
        }
        if (!comp && E->p2p && E->pcorr && !staged) {  // after apply(t-1) finished writing W: peers may target it
            rc = p2p_stage(E, t, g, C);
            if (rc != CDSGD_OK) return rc;
        }
        if (!comp && E->p2p && E->pcorr) {
            rc = p2p_reduce_async(E, t, C);
            if (rc != CDSGD_OK) return rc;
        }
        E->pending = true;
        E->pend_t = t;
        E->pend_comp = comp;
        E->pend_grad = g;
        E->compute_is_loc = true;
    }
    E->t = t + 1;
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_flush(cdsgd_engine* E, void* stream) {
    if (E == nullptr) return fail(CDSGD_ERR_ARG, "NULL engine");
    const int rf = p2p_ce_finish(E, S(stream));
    if (rf != CDSGD_OK) return rf;
    if (!E->pending) return CDSGD_OK;
    const int rc = engine_apply(E, E->pend_t, E->pend_comp, E->pend_grad, nullptr, S(stream));
    if (rc != CDSGD_OK) return rc;
    E->pending = false;
    E->pend_grad = nullptr;
    // The next round computes at the now-current global weights' local step;
    // loc already holds W_{t-1} - eta_l*g_{t-1}, which is what round t reads.
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_get_state(const cdsgd_engine* E, cdsgd_engine_state* out) {
    if (E == nullptr || out == nullptr) return fail(CDSGD_ERR_ARG, "NULL argument");
    out->t = E->t;
    out->residual_index = E->rcur;
    out->compute_is_loc = E->compute_is_loc ? 1 : 0;
    out->pending = E->pending ? 1 : 0;
    out->last_compressed = E->pend_comp ? 1 : 0;
    out->failed = E->failed ? 1 : 0;
    return CDSGD_OK;
}

extern "C" int cdsgd_engine_check(cdsgd_engine* E, void* stream, int64_t* round, int64_t* index) {
    if (E == nullptr) return fail(CDSGD_ERR_ARG, "NULL engine");
    CUDA_TRY(cudaStreamSynchronize(S(stream)));
    if (E->xs) CUDA_TRY(cudaStreamSynchronize(E->xs));
    if (E->comm != nullptr) {
        ncclResult_t ar = ncclSuccess;
        NCCL_TRY(ncclCommGetAsyncError(E->comm->nccl, &ar));
        if (ar != ncclSuccess) return fail(CDSGD_ERR_NCCL, "NCCL async error: %s", ncclGetErrorString(ar));
    }
    uint64_t h[2];
    CUDA_TRY(cudaMemcpy(h, E->d.err, sizeof(h), cudaMemcpyDeviceToHost));
    if (h[0] != NO_ERR) {
        const int64_t rel = static_cast<int64_t>(h[0] >> CDSGD_INDEX_BITS);
        const int64_t idx = static_cast<int64_t>(h[0] & ((uint64_t(1) << CDSGD_INDEX_BITS) - 1));
        const int64_t s = E->err_base + rel;
        if (round) *round = s;
        if (index) *index = idx;
        if (rel >= 0 && rel < static_cast<int64_t>(E->rlog.size())) E->rcur = E->rlog[rel];
        E->failed = true;
        return fail(CDSGD_ERR_NUMERIC, "non-finite accumulated gradient at round %lld, element %lld",
                    (long long)s, (long long)idx);
    }
    if (h[1] == EXCHANGE_TIMEOUT) {
        E->failed = true;
        return fail(CDSGD_ERR_STATE, "fused exchange timed out waiting for a peer (lost rank?)");
    }
    if (h[1] == PEER_FAILED) {
        E->failed = true;
        return fail(CDSGD_ERR_PEER, "a peer rank failed (numeric error); this rank stopped applying rounds");
    }
    if (h[1] != NO_ERR) {
        if (index) *index = static_cast<int64_t>(h[1]);
        E->failed = true;
        return fail(CDSGD_ERR_CORRUPT, "reserved symbol 11 at element %lld", (long long)h[1]);
    }
    E->err_base = E->t;
    E->rlog.clear();
    return CDSGD_OK;
}
