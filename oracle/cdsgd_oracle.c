/*
 * cdsgd_oracle.c — C restatement of the reference CD-SGD round (TEST
 * INFRASTRUCTURE / CPU BASELINE ONLY; never linked into the product).
 *
 * Restates, in the same IEEE fp64 operation order as the reference NumPy code
 * (so results are bit-identical; compiled with -ffp-contract=off, no fast-math):
 *   codec.quantize        pkg/src/cdsgd/codec.py:164-194 (per key, engine.py:397-402)
 *   codec.pack_symbols    codec.py:140-151
 *   codec.dequantize      codec.py:197-206
 *   server_aggregate      engine.py:249-255 (ascending worker id, then / N)
 *   server apply          engine.py:511   (W -= eta * mean)
 *   local_update          engine.py:268-274 (base - eta_l * g)
 * Parallelised with OpenMP across packed words / elements; every output element
 * is computed by exactly one thread with the reference's arithmetic, so the
 * thread count never changes a bit.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NO_ERR INT64_MAX

int cdsgd_ref_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void cdsgd_ref_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* codec.py:181-193 for one element: returns the 2-bit code. */
static inline uint32_t quant1(double r, double g, double alpha, double* rn) {
    const double acc = r + g;
    const int plus = acc >= alpha;
    const int minus = acc <= -alpha;
    const double emitted = (plus ? alpha : 0.0) + (minus ? -alpha : 0.0);
    *rn = acc - emitted;
    return plus ? 1u : (minus ? 2u : 0u);
}

/* Quantize every key of a layout (key lengths `sizes`), fp32 gradient.
 * r_in/r_out may alias. Returns the first flat index with a non-finite
 * accumulator (nothing is meaningful then), or -1. */
int64_t cdsgd_ref_quantize_layout(const double* r_in, const float* g, double* r_out, uint32_t* words,
                                  const int64_t* sizes, int32_t n_keys, double alpha) {
    int64_t bad = NO_ERR;
    int64_t e0 = 0, w0 = 0;
    for (int32_t k = 0; k < n_keys; ++k) {
        const int64_t n = sizes[k], nw = (n + 15) / 16;
        /* codec.py:182-185: the finiteness check precedes any mutation */
        int64_t kb = NO_ERR;
#pragma omp parallel for reduction(min : kb) schedule(static)
        for (int64_t i = 0; i < n; ++i)
            if (!isfinite(r_in[e0 + i] + (double)g[e0 + i]) && i < kb) kb = i;
        if (kb != NO_ERR) { bad = e0 + kb; break; }
#pragma omp parallel for schedule(static)
        for (int64_t w = 0; w < nw; ++w) {
            uint32_t v = 0;
            for (int j = 0; j < 16; ++j) {
                const int64_t i = 16 * w + j;
                if (i < n) v |= quant1(r_in[e0 + i], (double)g[e0 + i], alpha, &r_out[e0 + i]) << (2 * j);
            }
            words[w0 + w] = v;
        }
        e0 += n;
        w0 += nw;
    }
    return bad == NO_ERR ? -1 : bad;
}

/* Decode N payload buffers (rank-major, `stride` words apart), ascending-order
 * fp64 sum, / N (engine.py:249-255). Returns first reserved-symbol flat index or -1. */
int64_t cdsgd_ref_aggregate_quant(const uint32_t* words, int32_t nr, int64_t stride, const int64_t* sizes,
                                  int32_t n_keys, double alpha, double* mean) {
    int64_t bad = NO_ERR;
    int64_t e0 = 0, w0 = 0;
    for (int32_t k = 0; k < n_keys; ++k) {
        const int64_t n = sizes[k];
#pragma omp parallel for reduction(min : bad) schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            double total = 0.0;
            for (int r = 0; r < nr; ++r) {
                const uint32_t c = (words[r * stride + w0 + i / 16] >> (2 * (i % 16))) & 3u;
                if (c == 3u && e0 + i < bad) bad = e0 + i;
                const double d = c == 1u ? alpha : (c == 2u ? -alpha : 0.0);
                total = r == 0 ? d : total + d;
            }
            mean[e0 + i] = total / (double)nr;
        }
        e0 += n;
        w0 += (n + 15) / 16;
    }
    return bad == NO_ERR ? -1 : bad;
}

/* Full-precision branch: ascending sum of fp32 grads (as fp64) / N. */
void cdsgd_ref_aggregate_full(const float* grads, int32_t nr, int64_t stride, int64_t n, double* mean) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double total = (double)grads[i];
        for (int r = 1; r < nr; ++r) total = total + (double)grads[r * stride + i];
        mean[i] = total / (double)nr;
    }
}

/* engine.py:511 / 258-265 */
void cdsgd_ref_global_update(double* w, const double* mean, int64_t n, double eta) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) w[i] = w[i] - eta * mean[i];
}

/* engine.py:268-274 */
void cdsgd_ref_local_update(const double* base, const float* g, double* out, int64_t n, double eta_l) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = base[i] - eta_l * (double)g[i];
}

/* codec.py:140-151 / 154-161 */
int64_t cdsgd_ref_pack(const uint8_t* sym, int64_t n, uint32_t* words) {
    int64_t bad = NO_ERR;
    const int64_t nw = (n + 15) / 16;
#pragma omp parallel for reduction(min : bad) schedule(static)
    for (int64_t w = 0; w < nw; ++w) {
        uint32_t v = 0;
        for (int j = 0; j < 16; ++j) {
            const int64_t i = 16 * w + j;
            if (i < n) {
                if (sym[i] > 2 && i < bad) bad = i;
                v |= (uint32_t)(sym[i] & 3u) << (2 * j);
            }
        }
        words[w] = v;
    }
    return bad == NO_ERR ? -1 : bad;
}

void cdsgd_ref_unpack(const uint32_t* words, int64_t length, uint8_t* sym) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < length; ++i) sym[i] = (uint8_t)((words[i / 16] >> (2 * (i % 16))) & 3u);
}
