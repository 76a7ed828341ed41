/*
 * cdsgd_b200.h — C ABI of the B200-native CD-SGD hot path (libcdsgd_b200.so).
 *
 * The reference (cdsgd 0.1.0, pure Python/NumPy) exposes this path as a Python
 * function API: codec.quantize / dequantize / pack_symbols / unpack_symbols
 * (pkg/src/cdsgd/codec.py:140-206) and engine.should_compress /
 * server_aggregate / global_update / local_update (pkg/src/cdsgd/engine.py:217-274),
 * driven per round by Worker.compute_push / ServerNode._handle_push /
 * Worker.apply_pull (engine.py:357-430, 477-517). Every entry point below cites
 * the reference interface it replaces. A reference-side binding (ctypes) is
 * shown in INTEGRATION.md; paper_2106_10796_b200/_lib.py is exactly that binding.
 *
 * Conventions
 *  - Plain pointers and sizes only. Device pointers are CUDA global memory on
 *    the current device; `stream` is a cudaStream_t (NULL = legacy default).
 *  - Every call is asynchronous on `stream` unless stated; nothing allocates on
 *    the hot path (layouts, comms and engines allocate once at creation).
 *  - Return value: 0 on success, a negative CDSGD_ERR_* code otherwise; the
 *    message is available from cdsgd_last_error() (thread-local).
 *  - Data errors found on the device (non-finite accumulator, reserved code 11)
 *    are reported through a caller-owned device word `err` (initialise to
 *    CDSGD_NO_ERROR = UINT64_MAX) that the kernels atomicMin with
 *    (tag | flat element index); the host reads it at a sync point.
 *  - Arithmetic of the codec is IEEE fp64 with round-to-nearest and no
 *    contraction, so codes and residuals are bit-identical to the reference.
 */
#ifndef CDSGD_B200_H
#define CDSGD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDSGD_ABI_VERSION 2

#define CDSGD_OK 0
#define CDSGD_ERR_ARG -1     /* bad argument: maps to CodecError / LayoutError / ConfigError */
#define CDSGD_ERR_CUDA -2    /* CUDA runtime failure */
#define CDSGD_ERR_NCCL -3    /* NCCL failure */
#define CDSGD_ERR_STATE -4   /* engine used out of order (maps to SchedulingError) */
#define CDSGD_ERR_NUMERIC -5 /* a step hit a non-finite accumulator (CodecNumericError) */
#define CDSGD_ERR_CORRUPT -6 /* reserved symbol 11 in a payload (CorruptPayloadError) */
#define CDSGD_ERR_PEER -7    /* another rank failed (its flags arrived poisoned); nothing was applied after it */

#define CDSGD_NO_ERROR 0xFFFFFFFFFFFFFFFFull
#define CDSGD_INDEX_BITS 40 /* err word = (step_tag << 40) | flat element index */

#define CDSGD_F32 0
#define CDSGD_F64 1

#define CDSGD_ALGO_SSGD 0
#define CDSGD_ALGO_LUSGD 1
#define CDSGD_ALGO_BITSGD 2
#define CDSGD_ALGO_CDSGD 3

typedef struct cdsgd_layout cdsgd_layout;
typedef struct cdsgd_comm cdsgd_comm;
typedef struct cdsgd_engine cdsgd_engine;

/* ------------------------------------------------------------------ status */
int cdsgd_abi_version(void);
const char* cdsgd_last_error(void);
/* Number of this library's kernels launched so far in this process (evidence counter). */
uint64_t cdsgd_launch_count(void);

/* ------------------------------------------------------------------ layout
 * Replaces numcore.Layout (numcore.py:48-84): a contiguous partition of the flat
 * vector into keys. Packing restarts at each key (engine.py:397-402,
 * codec.py:147-148), so word offsets are prefix sums of ceil(len_k/16).
 * Key lengths must be >= 1 (numcore.py:59-60). Allocates device key tables once. */
int cdsgd_layout_create(const int64_t* key_lengths, int32_t n_keys, cdsgd_layout** out);
int cdsgd_layout_destroy(cdsgd_layout* layout);
int64_t cdsgd_layout_elems(const cdsgd_layout* layout);
int64_t cdsgd_layout_words(const cdsgd_layout* layout);
int32_t cdsgd_layout_keys(const cdsgd_layout* layout);
/* Host copies of the (n_keys+1)-entry element / word offset tables. */
int cdsgd_layout_offsets(const cdsgd_layout* layout, int64_t* elem_off, int64_t* word_off);

/* ------------------------------------------------------------------ codec (K1)
 * Replaces codec.quantize (codec.py:164-194), applied to every key of `layout`
 * exactly as Worker.compute_push does (engine.py:397-402):
 *   acc = r_in + (double)g ; +a if acc >= a, -a if acc <= -a, else 0 ;
 *   r_out = acc - emitted ; 2-bit codes packed 16/word LE, zero pad per key.
 * `grad` is fp32 (grad_dtype CDSGD_F32) or fp64 (CDSGD_F64). r_in may equal r_out.
 * Non-finite acc: atomicMin(err, err_tag | flat index); the caller must then keep
 * r_in (no-mutation-on-error, codec.py:181-185). If *err < err_tag at launch (an
 * error recorded by an EARLIER round, whose tag is smaller) the kernel does nothing
 * (sticky abort); an error of the same tag never stops the scan, so the reported
 * index is the first non-finite element. */
int cdsgd_quantize(const cdsgd_layout* layout, const void* grad, int32_t grad_dtype,
                   const double* r_in, double* r_out, uint32_t* words, double alpha,
                   uint64_t* err, uint64_t err_tag, void* stream);

/* FAST MODE (opt-in, not the reference's arithmetic): cdsgd_quantize restated in fp32 —
 * acc = r_in + g, +a if acc >= a, -a if acc <= -a (a = (float)alpha), r_out = acc - emitted,
 * all fp32 — for an fp32 residual: 12.25 instead of 20.25 bytes per element. Bitwise against
 * the fp32 restatement oracle (oracle/cdsgd_oracle.py quantize_f32), not the reference. */
int cdsgd_quantize_f32r(const cdsgd_layout* layout, const float* grad, const float* r_in, float* r_out,
                        uint32_t* words, double alpha, uint64_t* err, uint64_t err_tag, void* stream);

/* Replaces codec.dequantize (codec.py:197-206) when n_payloads == 1 and the
 * quantized branch of engine.server_aggregate (engine.py:249-255) otherwise:
 * out[i] = (sum over payload p ascending of decode_p[i]) / n_payloads, fp64.
 * Payload p's words start at words + p * payload_stride_words. Reserved symbol
 * 11 within a key's length: atomicMin(err, flat index) (pad bits not checked). */
int cdsgd_dequantize_sum(const cdsgd_layout* layout, const uint32_t* words, int32_t n_payloads,
                         int64_t payload_stride_words, double alpha, double* out,
                         uint64_t* err, void* stream);

/* Full-precision branch of engine.server_aggregate (engine.py:252-255):
 * out[i] = (sum over c ascending of (double)grads[c*stride + i]) / n_contrib. */
int cdsgd_aggregate_full(const void* grads, int32_t dtype, int32_t n_contrib, int64_t stride,
                         int64_t n, double* out, void* stream);

/* codec.pack_symbols / unpack_symbols (codec.py:140-161), one key of `n` symbols.
 * pack: symbol > 2 -> atomicMin(err, index). */
int cdsgd_pack_symbols(const uint8_t* symbols, int64_t n, uint32_t* words, uint64_t* err,
                       void* stream);
int cdsgd_unpack_symbols(const uint32_t* words, int64_t length, uint8_t* symbols, void* stream);

/* engine.global_update (engine.py:258-265): w -= eta * mean (fp64 math). */
int cdsgd_global_update(void* weights, int32_t w_dtype, const void* mean, int32_t m_dtype,
                        int64_t n, double eta, void* stream);
/* engine.local_update (engine.py:268-274): out = base - eta_l * grad (fp64 math). */
int cdsgd_local_update(const void* base, int32_t base_dtype, const void* grad, int32_t g_dtype,
                       void* out, int32_t out_dtype, int64_t n, double eta_l, void* stream);

/* ------------------------------------------------------------------ fused apply (K2/K3)
 * K2 — compressed round: ServerNode._handle_push's decode + ascending-worker sum
 * + /N + W -= eta_g*mean (engine.py:249-255, 509-511) on a replicated W of w_dtype
 * (CDSGD_F64: the reference's own fp64 operations; CDSGD_F32: one fp32 rounding per round),
 * fused with the next local update loc = W' - eta_l*g_next (engine.py:385-392,
 * Eq. 11). `gathered` holds nranks payload buffers, rank r at r*rank_stride_words.
 * g_next / loc_out may be NULL (no local update). gnorm_sq (nullable) receives
 * += sum(mean^2) (engine.py:521). Skips all work if *err < skip_below. */
int cdsgd_apply_quant(const cdsgd_layout* layout, void* weights, int32_t w_dtype, const uint32_t* gathered,
                      int32_t nranks, int64_t rank_stride_words, double alpha, double eta_g,
                      const float* g_next, float* loc_out, double eta_l, uint64_t* err,
                      uint64_t skip_below, double* gnorm_sq, void* stream);
/* K3 — correction round (engine.py:252 full branch + 511): W -= eta_g * gsum/nranks,
 * then loc = W' - eta_l*g_next. gsum is the (NCCL) fp32 sum over ranks. */
int cdsgd_apply_full(void* weights, int32_t w_dtype, const float* gsum, int32_t nranks, int64_t n, double eta_g,
                     const float* g_next, float* loc_out, double eta_l, const uint64_t* err,
                     uint64_t skip_below, double* gnorm_sq, void* stream);

/* One round of the step in ONE pass over g_t (the kernel the engine runs on compressed
 * rounds): quantize(t) as cdsgd_quantize (codes to `words`, residual r_in -> r_out, err as
 * there, err_tag = this round's tag) fused with the apply of round t-1 — the decode +
 * ascending-worker sum of `gathered` (nranks payloads, rank stride rank_stride_words),
 * W -= eta_g*mean and loc = W' - eta_l*g_t (engine.py:249-255, 385-392, 509-511) — so g_t
 * is read once for both. gathered == NULL: nothing to apply, only loc = W - eta_l*g_t.
 * The apply part is skipped if *err < skip_below. nranks <= 8. Decode as K2 (exact table
 * when every j*alpha is representable, else the sequential fp64 sum). gnorm_sq: += the
 * round t-1 mean's sum of squares (nullable). */
int cdsgd_fused_round(const cdsgd_layout* layout, const float* grad, const void* r_in, void* r_out,
                      int32_t r_dtype, uint32_t* words, double alpha, uint64_t* err, uint64_t err_tag, void* weights,
                      int32_t w_dtype, float* loc, const uint32_t* gathered, int32_t nranks, int64_t rank_stride_words,
                      double eta_g, double eta_l, uint64_t skip_below, double* gnorm_sq, void* stream);

/* ------------------------------------------------------------------ exchange (NCCL)
 * Replaces the PS message passing of _run_lockstep (engine.py:627-661) /
 * socket transport (protocol.py:214-288): one rank per GPU, NCCL over NVLink. */
#define CDSGD_UNIQUE_ID_BYTES 128
int cdsgd_comm_unique_id(void* out_id /* CDSGD_UNIQUE_ID_BYTES */);
int cdsgd_comm_init(const void* unique_id, int32_t nranks, int32_t rank, cdsgd_comm** out);
int cdsgd_comm_destroy(cdsgd_comm* comm);
/* recv[r*words .. +words) = send of rank r; send may be recv + rank*words (in place). */
int cdsgd_allgather_words(cdsgd_comm* comm, const uint32_t* send, uint32_t* recv, int64_t words,
                          void* stream);
int cdsgd_allreduce_sum_f32(cdsgd_comm* comm, const float* send, float* recv, int64_t n,
                            void* stream);

/* ------------------------------------------------------------------ step engine
 * One CD-SGD worker (Algorithm 1; Worker + the replicated ServerNode) per GPU.
 * engine_step(t) with this round's gradient g_t (computed at the weights from
 * cdsgd_engine_compute_weights):
 *   - quantize g_t with the key-segmented K1 (compressed rounds) into this rank's
 *     slot of gathered[t%2], then exchange round t on the engine's own stream
 *     (ncclAllGather of words, or ncclAllReduce of g_t on correction/warm-up rounds);
 *   - finish round t-1 on `stream`: wait for its exchange, K2/K3 apply fused with
 *     the local update loc_{t+1} = W_t - eta_l * g_t (engine.py:385-392).
 * Round t's exchange therefore overlaps the producer's compute of t+1 — the
 * paper's compute/communication overlap. Warm-up rounds before warmup_n-1 and
 * the non-local algorithms (ssgd/bitsgd) complete synchronously.
 * cdsgd_engine_flush applies the last pending round (W = W_T).
 * At N=1 and with the P2P exchange, apply(t-1) and quantize(t) run as ONE kernel that
 * reads g_t once; at N=1 a correction round is applied inside the preceding apply (its
 * mean is g_t itself). Engine kernels are launched with programmatic stream
 * serialization: each waits (griddepcontrol.wait) for its stream predecessor before
 * touching memory, so caller kernels on `stream` keep plain stream-order semantics.
 * The grad-norm ring is zeroed by create and then kept zero ahead in-kernel.
 * Buffers are caller-owned device memory (sizes in the struct comments). */
typedef struct {
    int32_t algo;      /* CDSGD_ALGO_* (engine.py:76) */
    int32_t nranks;    /* workers N */
    int32_t rank;      /* this worker id */
    int32_t k;         /* k-step period, >= 1 */
    int32_t warmup_n;  /* >= 0 */
    int32_t force_compress; /* engine.py:300, 351-352 */
    int32_t bypass_local;   /* engine.py:301, 310 */
    int32_t gnorm_ring;     /* entries in gnorm_sq (0 = no grad-norm metric) */
    int32_t weights_dtype;  /* CDSGD_F64: exact (the reference's fp64 W, bitwise on compressed rounds);
                               CDSGD_F32: fast (W rounded to fp32 every round) */
    int32_t residual_dtype; /* CDSGD_F64: exact (bitwise the reference's residual and codes);
                               CDSGD_F32: fast mode (fp32 restatement, 12.25 B/elem quantizer; needs fp32 W) */
    double alpha, eta_global, eta_local;
    void* weights;           /* [n] fp64 or fp32 (weights_dtype), replicated global weights W */
    float* loc;              /* [n] fp32, local (compute) weights */
    void* residual[2];       /* [n] fp64 (or fp32: residual_dtype) each, ping-pong error-feedback residual */
    uint32_t* gathered[2];   /* [nranks * words] each */
    float* gsum[2];          /* [n] fp32 each (nranks > 1; may be NULL when nranks == 1) */
    uint64_t* err;           /* [2] device words, init CDSGD_NO_ERROR */
    double* gnorm_sq;        /* [gnorm_ring] device, nullable; zeroed by create, round t valid for ring-2 rounds */
} cdsgd_engine_desc;

typedef struct {
    int64_t t;               /* rounds started */
    int32_t residual_index;  /* which residual[] buffer is current */
    int32_t compute_is_loc;  /* 1: next gradient is computed at loc, 0: at weights */
    int32_t pending;         /* 1 if round t-1 is exchanged but not applied */
    int32_t last_compressed; /* 1 if round t-1 pushed codes */
    int32_t failed;          /* 1 after a numeric error was reported */
} cdsgd_engine_state;

int cdsgd_engine_create(const cdsgd_engine_desc* desc, const cdsgd_layout* layout,
                        cdsgd_comm* comm /* NULL iff nranks == 1 */, cdsgd_engine** out);
int cdsgd_engine_destroy(cdsgd_engine* eng);
int cdsgd_engine_step(cdsgd_engine* eng, const float* grad, void* stream);
int cdsgd_engine_flush(cdsgd_engine* eng, void* stream);
int cdsgd_engine_get_state(const cdsgd_engine* eng, cdsgd_engine_state* out);
/* Synchronises `stream`, reads the error words. Returns CDSGD_OK, or
 * CDSGD_ERR_NUMERIC with *round / *index filled (index is flat; the residual
 * index is restored to the buffer valid before that round), or CDSGD_ERR_CORRUPT. */
int cdsgd_engine_check(cdsgd_engine* eng, void* stream, int64_t* round, int64_t* index);
/* 1 if round `t` (0-based) pushes codes under the engine's schedule (engine.py:345-355). */
int cdsgd_engine_round_compressed(const cdsgd_engine* eng, int64_t t);
/* Fused NVLink exchange (replaces the NCCL all-gather of codes on compressed rounds).
 * Every rank allocates one symmetric buffer of cdsgd_p2p_bytes(nranks, n, words) bytes
 * (zero-filled; cdsgd_p2p_buffer_alloc/_open below, or torch symmetric memory), maps all peers' buffers, and passes
 * the nranks base addresses (index = rank, 256-byte aligned) before round 0. K1 then
 * stores each packed word directly into every rank's slot and publishes a release
 * flag; K2 acquires all ranks' flags (spin on local memory, ~10 s timeout ->
 * CDSGD_ERR_STATE at cdsgd_engine_check) and releases the slot. Correction rounds
 * are all-reduced on the engine's streams (overlapped with compute), split between
 * ncclAllReduce and the copy engines (peer cudaMemcpyAsync reduce-scatter, fp64 shard
 * sums, all-gather; 30 % of the elements at N=2, 55 % at N>=3, from 8M elements, on
 * rounds whose all-reduce overlaps compute) unless
 * exact_correction != 0: then g_t is staged in the symmetric buffer and in the next
 * round every rank reduces its shard of elements from all ranks' stages (fp64,
 * ascending rank — bitwise the reference's sum, engine.py:250-255), applies
 * W -= eta*mean and stores the W' shard into every rank's replica (no NCCL at all).
 * Requires nranks <= 8 (one NVSwitch box). */
int64_t cdsgd_p2p_bytes(int32_t nranks, int64_t n, int64_t words);
/* Byte offset of the W replica inside the symmetric buffer (attach moves W there:
 * peers store their W' shards of correction rounds into it). */
int64_t cdsgd_p2p_weights_offset(int32_t nranks, int64_t n, int64_t words);
int cdsgd_engine_attach_p2p(cdsgd_engine* eng, void* const* peer_bases, int32_t nranks, int32_t exact_correction);
/* A symmetric buffer without torch: cudaMalloc'd and zero-filled on the current device,
 * with its CUDA IPC handle (CDSGD_P2P_HANDLE_BYTES bytes) for the other ranks of the box;
 * _open maps a peer's buffer (peer access enabled on first use), _close unmaps it, _free
 * releases the local one (after every rank has stopped using it). */
#define CDSGD_P2P_HANDLE_BYTES 64
int cdsgd_p2p_buffer_alloc(int64_t bytes, void** ptr, void* handle);
int cdsgd_p2p_buffer_open(const void* handle, void** ptr);
int cdsgd_p2p_buffer_close(void* peer_ptr);
int cdsgd_p2p_buffer_free(void* ptr);
/* Make `stream` wait for every exchange the engine has issued so far. */
int cdsgd_engine_join(cdsgd_engine* eng, void* stream);
/* Per-kernel timing with CUDA events recorded on the launching streams around
 * each K1 / K2 / K3 / local-update launch and each NCCL call, between _begin and
 * _end. _end synchronises and writes 22 doubles, (ms, launches) per class:
 * quantize, apply_quant, apply_full, local_update, exchange (NCCL), fused
 * (apply(t-1) + quantize(t) in one kernel), stage, reduce (P2P correction), wait
 * (P2P correction completion), fused_local (quantize(t) + local update only),
 * exchange_ce (the copy-engine share of a correction all-reduce). */
int cdsgd_engine_profile_begin(cdsgd_engine* eng);
int cdsgd_engine_profile_end(cdsgd_engine* eng, double* out22);
/* Fraction of each correction all-reduce moved by the copy engines (P2P mode; 0 = NCCL
 * only; after cdsgd_engine_attach_p2p). */
double cdsgd_engine_ce_fraction(const cdsgd_engine* eng);

#ifdef __cplusplus
}
#endif
#endif /* CDSGD_B200_H */
