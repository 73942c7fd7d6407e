/*
 * kvq.h -- C ABI of the B200-native KVQuant decode hot path (arXiv 2401.18079).
 *
 * One handle = one layer's compressed KV cache (per-layer codebooks, PAPER.md P:303,
 * P:322).  Keys are stored per channel and pre-RoPE, Values
 * per token, as b-bit codes (b in {2,3,4}) indexing a non-uniform
 * codebook, with a per-vector dense-and-sparse split of about f = 1%
 * fp16 outliers kept compressed along the token axis so an append only
 * touches array tails.  Decode attention runs directly on that cache:
 * codebook dequantization with the affine fold, RoPE applied on the fly
 * to the dequantized pre-RoPE Keys, the sparse outlier terms in the
 * same launch.  See DESIGN.md for the readings of the paper (R1..R22) that
 * fix every detail the paper leaves open, and for the GPU data layout.
 *
 * Conventions for every call:
 *   - No exception crosses the ABI.  Every call returns a kvq_status; on failure the
 *     thread-local kvq_last_error() holds a message.
 *   - Validation runs synchronously before anything is enqueued; a failed call changes
 *     nothing and leaves outputs untouched.
 *   - Problems detected on the device (Key-outlier capacity overflow, asynchronous CUDA
 *     faults) are STICKY: the next call on that cache (or kvq_sync) returns them.
 *   - "device or host" buffers: the library detects host memory (pinned or pageable)
 *     with cudaPointerGetAttributes and stages it through device scratch on the call's
 *     stream (H2D before, D2H after, all stream ordered: a page-locked host output is
 *     valid once the stream reaches the end of the call; pageable host memory makes the
 *     call synchronous).  Device buffers must live on cfg.device (else KVQ_EDEVICE).
 *     With KVQ_FLAG_TRUST_DEVICE_PTRS the check is skipped and pointers are assumed
 *     to be device pointers on cfg.device.
 *   - Borrowed buffers must stay valid until the stream reaches the call.
 *   - Threading: one writer per cache (append / prefill), and at most ONE attend
 *     (kvq_decode_attend / kvq_decode_attend_partial) in flight per cache: every attend
 *     on a cache uses that cache's split-partial scratch and merge tickets, so two
 *     attends on the same cache must be ordered by the caller (same stream, or an
 *     event between streams).  Attends never overlap a writer on another stream.
 *     Distinct caches are independent (each has its own scratch).
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 */
#ifndef KVQ_H_
#define KVQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KVQ_OK = 0,
    KVQ_EINVAL = 1,     /* bad bits/ppm/codebook/thresholds/argument */
    KVQ_ESHAPE = 2,     /* unsupported or inconsistent head shape */
    KVQ_EEMPTY = 3,     /* attend on an empty cache */
    KVQ_ECAPACITY = 4,  /* token capacity exceeded, or (sticky) Key-outlier capacity */
    KVQ_EDEVICE = 5,    /* pointer or stream on the wrong device */
    KVQ_ECUDA = 6       /* CUDA runtime error (sticky when asynchronous) */
} kvq_status;

typedef struct kvq_cache kvq_cache;

#define KVQ_FLAG_TRUST_DEVICE_PTRS 1u
/* Opt-in programmatic dependent launch for the decode order "kvq_append(k, v) then
 * kvq_decode_attend(q)" on one stream: the attend's prologue (query RoPE, per-query
 * tables; it reads only q and the cache's constant parameters) overlaps the append
 * kernel, and its first read of cache contents waits for the append (griddepcontrol).
 * CONTRACT: with this flag the caller guarantees that q is complete in stream order
 * BEFORE kvq_append is enqueued, i.e. no kernel that writes q is enqueued between the
 * append and the attend.  Without the flag the attend waits for all prior work. */
#define KVQ_FLAG_DECODE_PDL 2u

typedef struct {
    int32_t n_q_heads;          /* H_q >= 1 */
    int32_t n_kv_heads;         /* H_kv >= 1, H_q % H_kv == 0; GQA group G = H_q/H_kv.
                                   Attend tilings of this build: G in {1, 2, 4, 8} at 2-4
                                   bits (G = 8: LLaMA-2-70B); 4-bit GQA needs an fp16-exact
                                   Value decode codebook (R23); other (bits, G) are rejected
                                   at create with KVQ_ESHAPE */
    int32_t head_dim;           /* d; this build supports d == 128 */
    int32_t bits;               /* b in {2, 3, 4} */
    int32_t outlier_ppm;        /* f in parts per million, 0 <= ppm < 500000;
                                   per-token Value outliers k = ceil(ppm*D/1e6) (R2) */
    int64_t capacity_tokens;    /* preallocated tokens; the cache never reallocates
                                   (fixes the copy-on-append of P:686-687) */
    int64_t k_outlier_capacity; /* Key-outlier records; 0 = auto (2*k + 64 per token) */
    int64_t pos_base;           /* RoPE position of cached token 0 (sequence shards) */
    double rope_theta;          /* RoPE base, 10000 for LLaMA/Mistral */
    int32_t device;             /* CUDA device ordinal */
    uint32_t flags;             /* KVQ_FLAG_* */
} kvq_config;

typedef struct {
    /* Host pointers, copied at creation.  Codebooks: 2^bits fp32, strictly ascending
     * (encode).  Decode codebooks may differ (Q-Norm; reading R9);
     * NULL means "same as encode". */
    const float *key_cb_enc, *key_cb_dec;
    const float *val_cb_enc, *val_cb_dec;
    /* Per-channel Key thresholds [D] (offline calibrated).  s_c and z_c
     * are derived as fp32((hi-lo)/2), fp32((hi+lo)/2) in fp64 (reading R6). */
    const float *key_lo, *key_hi;
} kvq_params;

/* Create a layer cache.  Validates: bits, ppm, D = H_kv*d <= 8192, d == 128, H_q % H_kv,
 * strictly ascending finite codebooks, finite lo <= hi, k < D, capacity > 0.
 * Allocates every device buffer up front.  Returns KVQ_EINVAL / KVQ_ESHAPE /
 * KVQ_ECUDA (allocation) on failure with *out untouched. */
kvq_status kvq_cache_create(const kvq_config *cfg, const kvq_params *params, kvq_cache **out);

/* Free every device buffer.  NULL is a no-op. */
void kvq_cache_destroy(kvq_cache *cache);

/* Quantize-on-append of one decode token.
 * k_prerope_f16: [D] fp16 pre-RoPE Key;  v_f16: [D] fp16 Value (device or host).
 * Keys: outlier iff x < lo_c or x > hi_c; code = ENC(clamp(x)) (R4, R5, R8).
 * Values: two-sided top-k split with ties to the lower index (R2, R3), (s,z) from
 * the kept range, code = ENC(clamp(v)).  Codes, outliers, (s,z) are appended at the
 * tails.  KVQ_ECAPACITY when the token capacity is full. */
kvq_status kvq_append(kvq_cache *cache, const void *k_prerope_f16, const void *v_f16,
                      void *stream);

/* Block quantization of T prompt tokens (a9; "future work" in the paper).
 * K_f16, V_f16: [T][D] fp16, row major.  Result is identical to T kvq_append calls. */
kvq_status kvq_prefill_quantize(kvq_cache *cache, const void *K_f16, const void *V_f16,
                                int64_t T, void *stream);

/* Single-token decode attention over all cached tokens (a1-a7):
 *   o_g = softmax_n( RoPE(q_g,pos) . RoPE(K^_{n,h(g)}, pos_base+n) / sqrt(d) ) V^_{n,h(g)}
 * q_f16: [H_q][d] fp16 PRE-RoPE queries; o: [H_q][d] fp32.  One fused launch (query
 * prologue + split-T tile loop + split merge).  KVQ_EEMPTY on an empty cache. */
kvq_status kvq_decode_attend(kvq_cache *cache, const void *q_f16, int64_t pos, float *o,
                             void *stream);

/* Same as kvq_decode_attend but returns this cache's un-normalized partial
 *   part: [H_q][d+2] fp32 = (sum_n p_n V^_n [d], m, l)
 * with p_n = 2^(s'_n - m), s'_n the score in log2 units (s_n * log2 e), l = sum p_n.
 * An empty cache yields (0, -inf, 0).  Used for sequence sharding. */
kvq_status kvq_decode_attend_partial(kvq_cache *cache, const void *q_f16, int64_t pos,
                                     float *part, void *stream);

/* Batched decode (the paper's BS = 4 rows): one decode step for B
 * independent sequences, each with its own cache, query q[i] ([H_q][d] fp16, device), position
 * pos[i] and output o[i] ([H_q][d] fp32, device).  When every cache is attended by the same
 * kernel family (the warp-autonomous MHA kernel, or the tensor-core GQA kernel) with the same
 * bits / codebook kind / head shape and B <= 64, the B attends are ONE launch whose CTAs are
 * split over the sequences in proportion to their lengths (one wave for many short contexts
 * instead of B latency-bound launches); otherwise (other shapes) it is B ordinary attends.
 * Same errors per sequence as kvq_decode_attend. */
kvq_status kvq_decode_attend_batch(kvq_cache *const *caches, int32_t B, const void *const *q,
                                   const int64_t *pos, float *const *o, void *stream);

/* Batched partials: as kvq_decode_attend_batch, but writes each cache's un-normalized partial
 * part[i] ([H_q][d+2] fp32, device; see kvq_decode_attend_partial).  Every cache must hold at
 * least one token.  Used for chunk-paged sequences (paper_2401_18079_b200/paged.py: the chunks
 * of many sequences in one launch, then kvq_merge_partials per sequence). */
kvq_status kvq_decode_attend_batch_partial(kvq_cache *const *caches, int32_t B, const void *const *q,
                                           const int64_t *pos, float *const *part, void *stream);

/* Exact log-sum-exp merge of P partials (fixed order 0..P-1), the merge step of the
 * north_star's sequence sharding:
 *   m = max_i m_i;  l = sum_i 2^(m_i - m) l_i;  o = sum_i 2^(m_i - m) o_i / l
 *   parts: [P][H_q][d+2] fp32 (device or host); o: [H_q][d] fp32.
 * device: the CUDA device to run on. */
kvq_status kvq_merge_partials(const float *parts, int32_t P, int32_t H_q, int32_t d,
                              float *o, int32_t device, void *stream);

/* Number of cached tokens (host shadow; no sync). */
int64_t kvq_num_tokens(const kvq_cache *cache);

/* Drop every cached token (capacity kept).  Stream ordered after prior work on
 * `stream`. */
kvq_status kvq_reset(kvq_cache *cache, void *stream);

/* Snapshot / restore (checkpoint / resume; SPEC S:535-536 cache dump / load).  The snapshot is
 * the device state of the cached tokens (code words, outlier buckets and counts, Value (s, z),
 * CSR / CSC records) behind a header with the cache's shape; it restores into any cache created
 * with the same configuration (heads, bits, D, outlier fraction) and enough capacity, which then
 * continues exactly as the original would (appends, attends).  Both calls synchronize the device.
 *   kvq_snapshot_bytes: bytes a snapshot of the current contents needs.
 *   kvq_snapshot: writes it to host memory `host` of `bytes` bytes (KVQ_EINVAL if too small).
 *   kvq_restore: replaces the cache's contents (KVQ_ESHAPE: other configuration; KVQ_ECAPACITY:
 *   more tokens or Key outliers than the cache holds; KVQ_EINVAL: not a snapshot / truncated). */
kvq_status kvq_snapshot_bytes(kvq_cache *cache, int64_t *bytes);
kvq_status kvq_snapshot(kvq_cache *cache, void *host, int64_t bytes);
kvq_status kvq_restore(kvq_cache *cache, const void *host, int64_t bytes);

/* Move an EMPTY cache to another position range: token t of the cache is position
 * pos_base + t from now on (cfg.pos_base at create).  KVQ_EINVAL if the cache holds tokens
 * or pos_base < 0.  Lets a pool reuse fixed-size chunk caches across sequences (paged.py). */
kvq_status kvq_set_pos_base(kvq_cache *cache, int64_t pos_base);

/* Synchronize the cache's device and surface sticky errors. */
kvq_status kvq_sync(kvq_cache *cache);

/* Canonical export of tokens [t0, t1) (synchronizes).  Host buffers, caller owned:
 *   kcodes, vcodes : uint8 [t1-t0][D]        (codes in channel order)
 *   kptr           : int64 [t1-t0+1]         (absolute CSC offsets into the Key
 *                                             outlier array; kptr[0] = start)
 *   kidx, kval     : uint16 [kptr[last]-kptr[0]]  channel, fp16 bits
 *   vidx, vval     : uint16 [t1-t0][k]       channel (ascending), fp16 bits
 *   vs, vz         : float  [t1-t0]
 * Any pointer may be NULL to skip that array (kidx/kval need kptr).  Use
 * kvq_key_outlier_span first to size kidx/kval. */
typedef struct {
    uint8_t *kcodes;
    int64_t *kptr;
    uint16_t *kidx, *kval;
    uint8_t *vcodes;
    uint16_t *vidx, *vval;
    float *vs, *vz;
} kvq_export_buf;

kvq_status kvq_key_outlier_span(kvq_cache *cache, int64_t t0, int64_t t1, int64_t *begin,
                                int64_t *end);
kvq_status kvq_export(kvq_cache *cache, int64_t t0, int64_t t1, kvq_export_buf *buf);

/* Introspection for benchmarks and tests. */
typedef struct {
    int32_t heads_per_cta;      /* query heads per attend CTA (HG) */
    int32_t splits;             /* token splits per head group of the last attend */
    int32_t value_outliers;     /* k per token */
    int32_t words_per_token;    /* packed 32-bit code words per token per K or V */
    int64_t capacity_tokens;
    int64_t k_outlier_capacity;
    int64_t device_bytes;       /* bytes of device memory owned */
    int32_t attend_kernel;      /* kernel of the last attend: 1 = warp-autonomous (MHA, 2-3 bits,
                                   csrc/kvq_attend_wa.cu), 2 = GQA (G = 2, 4, 8, 2-3 bits: att_wgt_kernel, K scores on the tensor cores; KVQ_WGT_OFF=1: the LUT kernel att_wag_kernel),
                                   0 = two-halves (csrc/kvq_attend.cu),
                                   -1 = none yet */
    int32_t bucket_heads;       /* query heads per outlier bucket group */
} kvq_info;
kvq_status kvq_get_info(const kvq_cache *cache, kvq_info *info);

/* Force the number of token splits per head group for attend (0 = auto). */
kvq_status kvq_set_splits(kvq_cache *cache, int32_t splits);

/* Diagnostics: per-phase cycle sums of the attend kernel since the last call
 * (out[0..4]: -, ready wait, K phase, softmax phase, V phase; out[5]: tiles;
 * out[6..8] / out[9..11]: wait / compaction / TMA issue of the two producer warps), summed
 * over CTAs.  Only when the process was started with KVQ_PHASE_TIMERS=1. */
kvq_status kvq_phase_timers(kvq_cache *cache, uint64_t *out /* host [16] */);

/* Online per-channel Key thresholds ("Online for K", tab:calibration
 * P:1036-1064): lo_c / hi_c computed on the GPU from the Keys of a prefill block rather
 * than offline calibration data.  Per channel over the T tokens: n = ceil(ppm T / 1e6)
 * outliers, the ceil(n/2) largest and floor(n/2) smallest excluded (R2, R3); lo_c / hi_c =
 * the smallest / largest kept value (the floor(n/2)-th and (T-1-ceil(n/2))-th order statistics;
 * -0 returned as +0).  K_f16 [T][D] fp16 pre-RoPE Keys (device or host); key_lo, key_hi [D]
 * fp32 (device or host; host outputs make the call synchronous).  The result is meant for
 * kvq_cache_create's kvq_params.key_lo / key_hi.  KVQ_EINVAL when 2 ceil(n/2) >= T. */
kvq_status kvq_key_thresholds_online(const void *K_f16, int64_t T, int32_t D, int32_t outlier_ppm,
                                     float *key_lo, float *key_hi, int32_t device, void *stream);

/* Mixed-precision sensitivity (sec:appendix-mp, eq:opt2 P:1336-1339):
 *   Omega = (A - Q(A))^T F^D (A - Q(A)) = sum_{n,c} F[n][c] (A[n][c] - A^[n][c])^2
 * for the tokens [t0, t0 + T) of `cache`, which the caller has quantized into it (the cache is
 * created at the candidate LOWER precision with that layer's codebooks and thresholds
 * "quantization error computed at the lower precision").  A^ is the dequantized cache entry
 * (outliers exact; else Chat_dec[code] s + z, fp64 from the stored fp32 values, R5 / R6).
 *   K_f16, V_f16 : [T][D] fp16, the same pre-RoPE Keys / Values that were appended (device or host)
 *   FK, FV       : [T][D] fp32 diagonal Fisher weights (>= 0; device or host), NULL = all ones
 *                  (plain squared quantization error, the "quantization error-based" baseline)
 *   omega        : double [2] (device or host; host makes the call synchronous) =
 *                  (Omega over the Keys, Omega over the Values); Omega_i = sum of the two (R26).
 * Accumulated in fp64 with atomics: the summation order is not fixed (results agree to ~1e-15
 * relative).  KVQ_EINVAL when the token range is not cached. */
kvq_status kvq_layer_sensitivity(kvq_cache *cache, const void *K_f16, const void *V_f16, const float *FK,
                                 const float *FV, int64_t t0, int64_t T, double *omega, void *stream);

/* Diagonal Fisher information (F^D = diag(g (.) g), the F^D of eq:opt2): F[i] += g[i]^2 for n elements,
 * fp32 with one rounding per step (fmaf).  F, g: device pointers on `device`. */
kvq_status kvq_fisher_accumulate(float *F, const float *g, int64_t n, int32_t device, void *stream);

/* One-shot mixed-precision assignment: the demote_count layers with
 * the smallest omega (ties to the lower layer index) get bits_low, the rest bits_high.
 * Host only.  omega [L] >= 0, bits_out [L].  KVQ_EINVAL when demote_count is outside [0, L] or
 * an omega is negative / NaN. */
kvq_status kvq_assign_bits(const double *omega, int32_t L, int32_t demote_count, int32_t bits_high,
                           int32_t bits_low, int32_t *bits_out);

/* Offline calibration of one layer on the GPU: everything kvq_params needs,
 * from N calibration tokens (P:316-322 eq:fisher_kmeans, P:340, P:355-358 eq:qnorm):
 *   key_lo, key_hi  per-channel order statistics over the N tokens, exactly as
 *                   kvq_key_thresholds_online (R2, R3)
 *   key_cb, val_cb  2^bits centroids of Fisher-weighted Lloyd k-means on the normalized kept
 *                   values (Keys: lo_c <= x <= hi_c, x' = (x - z_c)/s_c; Values: per token the
 *                   two-sided top-k outliers removed, x' = (v - z_n)/s_n; fp64), initialised at
 *                   the bin centres -1 + (2j+1)/k, ties to the lower centroid, empty clusters
 *                   keep their centroid, stop when the largest move < tol or after max_iter
 *                   updates (readings R27, R28)
 *   *_cb_dec        Q-Norm'd decode codebooks (eq:qnorm; moments of the normalized points and of
 *                   their encode-codebook values) when cfg.qnorm, else copies of the encode ones
 * Codebooks are stored as fp32, or as fp16 values when cfg.fp16_codebooks (R23); an entry that
 * would not exceed its predecessor after rounding is bumped to the next representable value.
 *   K_cal, V_cal : [N][D] fp16 (device or host);  FK, FV : [N][D] fp32 Fisher diagonals (device or
 *   host) or NULL (ones);  outputs: key_lo, key_hi [D], codebooks [2^bits] fp32, iters [2] int32
 *   (Lloyd updates run for the Keys / Values; may be NULL) -- device or host, host makes the
 *   call synchronous.  D % 128 == 0, D <= 8192.  Deterministic for a given input (fixed grid,
 *   fixed reduction order).  KVQ_EINVAL on bad bits / ppm / max_iter / tol or too many outliers
 *   for N tokens. */
typedef struct {
    int32_t bits;            /* 2, 3 or 4 */
    int32_t outlier_ppm;     /* as kvq_config.outlier_ppm */
    int32_t max_iter;        /* >= 1 */
    int32_t qnorm;           /* 1: Q-Norm'd decode codebooks */
    int32_t fp16_codebooks;  /* 1: store fp16 values (R23) */
    int32_t reserved;
    double tol;              /* >= 0; 0 runs max_iter updates */
} kvq_calib_config;
kvq_status kvq_calibrate_layer(const void *K_cal, const void *V_cal, const float *FK, const float *FV, int64_t N,
                               int32_t D, const kvq_calib_config *cfg, float *key_lo, float *key_hi,
                               float *key_cb, float *key_cb_dec, float *val_cb, float *val_cb_dec,
                               int32_t *iters, int32_t device, void *stream);

/* ------------------------------------------------------------------------------------
 * fp16 comparator cache (BASELINE config C3 "4-bit vs 3-bit vs fp16 cache"): the paper's
 * baseline decode is fp16 mat-vec against an fp16 cache of post-RoPE Keys ("Key fp16
 * Matvec", "Value fp16 Matvec", the ~1.4x speedup of P:80).  Same decode step as the
 * quantized cache (pre-RoPE q and its position in, fp32 o out), dense fp16 storage:
 *   append : K_n is rotated by RoPE at position pos_base + n with exact fp64 angles and
 *            rounded once to fp16 (R11, R12); V_n is stored as given.
 *   attend : o_g = softmax_n(RoPE(q_g, pos) . K_n / sqrt(d)) V_n, fp32 softmax and P.V.
 * cfg fields used: n_q_heads, n_kv_heads (G = H_q / H_kv), head_dim (128), capacity_tokens,
 * pos_base, rope_theta, device, flags (KVQ_FLAG_TRUST_DEVICE_PTRS); bits / outlier_ppm /
 * k_outlier_capacity are ignored.  Same error, ownership and threading conventions as the
 * quantized cache (one writer, one attend in flight per cache). */
typedef struct kvq_f16_cache kvq_f16_cache;
kvq_status kvq_f16_cache_create(const kvq_config *cfg, kvq_f16_cache **out);
void kvq_f16_cache_destroy(kvq_f16_cache *cache);
/* T tokens: K_f16, V_f16 [T][D] fp16 pre-RoPE Keys and Values (device or host). */
kvq_status kvq_f16_append(kvq_f16_cache *cache, const void *K_f16, const void *V_f16, int64_t T,
                          void *stream);
/* q_f16 [H_q][d] pre-RoPE; o [H_q][d] fp32.  KVQ_EEMPTY on an empty cache. */
kvq_status kvq_f16_decode_attend(kvq_f16_cache *cache, const void *q_f16, int64_t pos, float *o,
                                 void *stream);
/* Stored post-RoPE Keys and Values of tokens [t0, t1) as fp16 bits [t1-t0][D] (host buffers,
 * either may be NULL; synchronizes). */
kvq_status kvq_f16_export(kvq_f16_cache *cache, int64_t t0, int64_t t1, uint16_t *k_out, uint16_t *v_out);
int64_t kvq_f16_num_tokens(const kvq_f16_cache *cache);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *kvq_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int32_t kvq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_H_ */
