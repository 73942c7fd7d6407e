/*
 * kvq_oracle.c -- KVQuant (arXiv 2401.18079) CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, obviously-correct reference for the decode hot path
 * (quantize-on-append + decode attention over the compressed cache).  It is written
 * from PAPER.md alone and shares no code, header, table or constant with the CUDA
 * product (paper_2401_18079_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Arithmetic: fp64 everywhere, except the storage precisions the cache itself defines
 * (fp16 outlier values, fp32 affine scale/offset, fp32 codebooks) -- DESIGN.md
 * readings R6, R20.  Every function below cites the PAPER.md passage ("P:<line>") it
 * follows; DESIGN.md "Readings" lists where the paper is silent and what we chose.
 *
 * Pin status (tests/test_oracle_*.py):
 *   rope            pinned  (d=2 hand value, matrix form, norm, relative-position law)
 *   enc             pinned  (SPEC worked values, exact-rational brute-force argmin)
 *   outlier select  pinned  (SPEC worked example, brute force over tie patterns)
 *   key/value quant pinned  (round trip on grid, error bound, exact outliers)
 *   attend          pinned  (lossless mode == textbook fp64 attention and torch SDPA;
 *                            hand-computed d=2 score with a non-identity Key affine,
 *                            S:506; dominant-score selection returns the hand-
 *                            dequantized V^_t; uniform scores -> mean of
 *                            hand-dequantized V^ incl. a lower-index tie)
 *   merge           pinned  (any partition == unsplit)
 *   key thresholds  pinned  (online: numpy sort order statistics; brute-force outlier
 *    (online)               counts per channel; the two-sided kept range of S:328-333)
 *   f64_to_f16      pinned  (numpy's IEEE round-to-nearest-even float16 conversion,
 *                            including ties, subnormals and overflow)
 *   f16cache_key    pinned  (== f64_to_f16 of the pinned kvo_rope; position 0 == identity)
 *   attend_dense    pinned  (torch SDPA in fp64 on the RoPE'd query; == the lossless-mode
 *                            kvo_attend when the stored Keys are exact)
 *   attention values on realistic synthetic data: "parity unpinned" beyond the special
 *   cases above (the oracle is the reference) -- see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

int kvo_version(void) { return 1; }

/* ---------------------------------------------------------------- fp16 decode ---- */
/* IEEE binary16 -> double, exact.  K, V, q arrive as fp16. */
double kvo_f16_to_f64(uint16_t h) {
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24); /* subnormal: m * 2^-24 */
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(m | 0x400), e - 25);
    return sign ? -v : v;
}

/* --------------------------------------------------------------------- RoPE ---- */
/* Element-wise RoPE, HF pairing (i, i+d/2), theta_i = base^(-2i/d), i = 0..d/2-1.
 * PAPER.md Appendix "RoPE Equation": out = x (.) cos + rot(x) (.) sin
 * with rot(x) = [-x_{d/2+1..d}, x_{1..d/2}].  Position is an exact integer; angles in
 * fp64 (R11, R12). */
void kvo_rope(const double *x, int d, int64_t pos, double theta_base, double *out) {
    int half = d / 2;
    for (int i = 0; i < half; ++i) {
        double theta = pow(theta_base, -2.0 * (double)i / (double)d);
        double ang = (double)pos * theta;
        double c = cos(ang), s = sin(ang);
        double a = x[i], b = x[i + half];
        out[i] = a * c - b * s;
        out[i + half] = b * c + a * s;
    }
}

/* ------------------------------------------------------- affine (normalization) ---- */
/* Kept range [lo, hi] normalized to [-1, 1]: x' = (x - z)/s with
 * s = (hi-lo)/2, z = (hi+lo)/2, evaluated in fp64 and stored as fp32 (reading R6).
 * hi == lo gives s = 0 (reading R7). */
void kvo_affine_from_range(double lo, double hi, float *s, float *z) {
    *s = (float)((hi - lo) / 2.0);
    *z = (float)((hi + lo) / 2.0);
}

/* ---------------------------------------------------------------- ENC (nuqX) ---- */
/* Nearest-signpost encode against the per-layer codebook:
 * code = #{ j in [0, nlev-1) : 2*(y - z) > s * (c_j + c_{j+1}) }   (reading R8)
 * i.e. the index of the nearest centroid to (y-z)/s, ties to the lower index.  The
 * codebook is strictly ascending.  Plain count over all midpoints, fp64. */
int kvo_enc(double y, float s, float z, const float *cb, int nlev) {
    double lhs = 2.0 * (y - (double)z);
    int code = 0;
    for (int j = 0; j + 1 < nlev; ++j) {
        double mid = (double)cb[j] + (double)cb[j + 1];
        double rhs = (double)s * mid;
        if (lhs > rhs) code++;
    }
    return code;
}

/* ------------------------------------------------------------- Key quantize ---- */
/* Per-channel pre-RoPE Key quantization with offline-calibrated thresholds
 * (P:265-273): for each channel c,
 *   outlier  <=>  x_c < lo_c  or  x_c > hi_c            (reading R4)
 *   code_c   =   ENC(clamp(x_c, lo_c, hi_c); s_c, z_c)    (reading R5)
 * Outliers are recorded with their original fp16 value, ascending channel order
 * (CSC column for this token).  Returns the number of outliers. */
int kvo_quantize_key(const uint16_t *x, int D, const float *lo, const float *hi,
                     const float *cb, int nlev, uint16_t *codes, int32_t *out_idx,
                     uint16_t *out_val) {
    int n = 0;
    for (int c = 0; c < D; ++c) {
        double xv = kvo_f16_to_f64(x[c]);
        double l = (double)lo[c], h = (double)hi[c];
        float s, z;
        kvo_affine_from_range(l, h, &s, &z);
        double y = xv < l ? l : (xv > h ? h : xv);
        codes[c] = (uint16_t)kvo_enc(y, s, z, cb, nlev);
        if (xv < l || xv > h) {
            out_idx[n] = c;
            out_val[n] = x[c];
            n++;
        }
    }
    return n;
}

/* ------------------------------------------------- Value outlier selection ---- */
/* Number of per-token Value outliers: k = ceil(f * D) with f = ppm / 1e6, in integers
 * (reading R2). */
int kvo_outlier_count(int D, int ppm) {
    return (int)(((int64_t)ppm * (int64_t)D + 999999) / 1000000);
}

static _Thread_local const double *g_sort_vals;   /* per-thread qsort context */
static int cmp_desc_val_asc_idx(const void *a, const void *b) {
    int i = *(const int *)a, j = *(const int *)b;
    double x = g_sort_vals[i], y = g_sort_vals[j];
    if (x > y) return -1;
    if (x < y) return 1;
    return (i < j) ? -1 : (i > j);
}
static int cmp_asc_val_asc_idx(const void *a, const void *b) {
    int i = *(const int *)a, j = *(const int *)b;
    double x = g_sort_vals[i], y = g_sort_vals[j];
    if (x < y) return -1;
    if (x > y) return 1;
    return (i < j) ? -1 : (i > j);
}

/* Two-sided per-token outlier split ("upper and lower outlier thresholds";
 * topk P:1028-1031), reading R3: the ceil(k/2) largest values (value desc, index asc),
 * then the floor(k/2) smallest of the remainder (value asc, index asc).  -0 == +0 by
 * construction of fp64 comparison.  Writes a 0/1 mask.  (The qsort comparator reads a
 * thread-local key array, so tokens may be quantized on several threads.) */
void kvo_select_outliers(const uint16_t *v, int D, int k, uint8_t *mask) {
    double *vals = (double *)malloc(sizeof(double) * (size_t)D);
    int *order = (int *)malloc(sizeof(int) * (size_t)D);
    for (int c = 0; c < D; ++c) vals[c] = kvo_f16_to_f64(v[c]);
    memset(mask, 0, (size_t)D);
    int ku = (k + 1) / 2, kl = k / 2;
    g_sort_vals = vals;
    for (int c = 0; c < D; ++c) order[c] = c;
    qsort(order, (size_t)D, sizeof(int), cmp_desc_val_asc_idx);
    for (int r = 0; r < ku; ++r) mask[order[r]] = 1;
    int m = 0;
    for (int c = 0; c < D; ++c)
        if (!mask[c]) order[m++] = c;
    qsort(order, (size_t)m, sizeof(int), cmp_asc_val_asc_idx);
    for (int r = 0; r < kl; ++r) mask[order[r]] = 1;
    free(vals);
    free(order);
}

/* Per-token Value quantization, thresholds and scale computed online (P:265-269,
 * P:367-370): select outliers, lo/hi = min/max of kept values, (s, z) from [lo, hi],
 * code = ENC(clamp(v_c, lo, hi); s, z).  Outliers recorded ascending by channel
 * (CSR row for this token).  identity_affine != 0 is the TEST-ONLY
 * lossless mode of reading R19 (s = 1, z = 0).  Returns k. */
int kvo_quantize_value(const uint16_t *v, int D, int ppm, const float *cb, int nlev,
                       int identity_affine, uint16_t *codes, int32_t *out_idx,
                       uint16_t *out_val, float *s_out, float *z_out) {
    int k = kvo_outlier_count(D, ppm);
    uint8_t *mask = (uint8_t *)malloc((size_t)D);
    kvo_select_outliers(v, D, k, mask);
    double lo = INFINITY, hi = -INFINITY;
    for (int c = 0; c < D; ++c) {
        if (mask[c]) continue;
        double x = kvo_f16_to_f64(v[c]);
        if (x < lo) lo = x;
        if (x > hi) hi = x;
    }
    float s, z;
    if (identity_affine) {
        s = 1.0f;
        z = 0.0f;
    } else {
        kvo_affine_from_range(lo, hi, &s, &z);
    }
    int n = 0;
    for (int c = 0; c < D; ++c) {
        double x = kvo_f16_to_f64(v[c]);
        double y = identity_affine ? x : (x < lo ? lo : (x > hi ? hi : x));
        codes[c] = (uint16_t)kvo_enc(y, s, z, cb, nlev);
        if (mask[c]) {
            out_idx[n] = c;
            out_val[n] = v[c];
            n++;
        }
    }
    *s_out = s;
    *z_out = z;
    free(mask);
    return n;
}

/* ------------------------------------------------------------------- Prefill ---- */
/* Prefill = T successive appends (reading: north_star "quantize-on-append for new and
 * prefill tokens"; P:684-685 block compression is future work in the paper).  Output is
 * the canonical cache: codes [T][D], Key CSC (kptr[T+1], channel, fp16 value), Value
 * CSR with k entries per token (implicit row pointer n*k), Value (s, z) per token.
 * Returns total Key nnz, or -1 if it would exceed kcap. */
int64_t kvo_prefill(int64_t T, int D, const uint16_t *K, const uint16_t *V,
                    const float *key_lo, const float *key_hi, const float *cbK,
                    const float *cbV, int nlev, int ppm, int value_identity_affine,
                    uint16_t *kcodes, int64_t *kptr, int32_t *kidx, uint16_t *kval,
                    int64_t kcap, uint16_t *vcodes, int32_t *vidx, uint16_t *vval,
                    float *vs, float *vz) {
    /* Tokens are independent: each is quantized exactly as kvo_quantize_key /
     * kvo_quantize_value define, possibly on several OpenMP threads; the Key-outlier CSC is
     * then laid out in token order, so the result equals T successive appends. */
    int k = kvo_outlier_count(D, ppm);
    int32_t *cnt = (int32_t *)malloc(sizeof(int32_t) * (size_t)(T > 0 ? T : 1));
    if (!cnt) return -2;
#pragma omp parallel
    {
        int32_t *tidx = (int32_t *)malloc(sizeof(int32_t) * (size_t)D);
        uint16_t *tval = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)D);
#pragma omp for schedule(dynamic, 64)
        for (int64_t n = 0; n < T; ++n) {
            cnt[n] = kvo_quantize_key(K + n * D, D, key_lo, key_hi, cbK, nlev, kcodes + n * D,
                                      tidx, tval);
            kvo_quantize_value(V + n * D, D, ppm, cbV, nlev, value_identity_affine,
                               vcodes + n * D, vidx + n * k, vval + n * k, vs + n, vz + n);
        }
        free(tidx);
        free(tval);
    }
    kptr[0] = 0;
    for (int64_t n = 0; n < T; ++n) kptr[n + 1] = kptr[n] + cnt[n];
    free(cnt);
    if (kptr[T] > kcap) return -1;
    /* the Key outliers of every token at its CSC column (same quantization, rerun) */
#pragma omp parallel
    {
        uint16_t *tcode = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)D);
#pragma omp for schedule(dynamic, 64)
        for (int64_t n = 0; n < T; ++n)
            kvo_quantize_key(K + n * D, D, key_lo, key_hi, cbK, nlev, tcode, kidx + kptr[n],
                             kval + kptr[n]);
        free(tcode);
    }
    return kptr[T];
}

/* ------------------------------------------------------------------ Attend ---- */
/* Decode attention over the compressed cache, plain definition (reading R13):
 *   K^_{n,c} = x  if (n,c) is a Key outlier, else  Chat_K[code]*s_c + z_c
 *   V^_{n,c} = v  if (n,c) is a Value outlier, else Chat_V[code]*s_n + z_n
 *   q~ = RoPE(q_g, pos); k~_n = RoPE(K^_{n,h}, pos_base + n)
 *   s_n = q~ . k~_n / sqrt(d);  m = max s_n;  p_n = exp(s_n - m);  l = sum p_n
 *   partial_g = (sum_n p_n V^_{n,h}, m, l),  o_g = partial / l
 * h = floor(g / G), G = H_q / H_kv.  Chat_* are the DECODE codebooks (Q-Norm'd or equal
 * to the encode ones; reading R9).  Outputs parts [H_q][d+2] in
 * fp64.  OpenMP (when compiled in) parallelizes over query heads only; each head is
 * computed exactly as the serial loop. */
void kvo_attend(int64_t T, int H_q, int H_kv, int d, const uint16_t *kcodes,
                const int64_t *kptr, const int32_t *kidx, const uint16_t *kval,
                const uint16_t *vcodes, int kper, const int32_t *vidx,
                const uint16_t *vval, const float *vs, const float *vz,
                const float *key_lo, const float *key_hi, const float *cbK_dec,
                const float *cbV_dec, const uint16_t *q, int64_t pos, int64_t pos_base,
                double theta_base, double *parts, int nthreads) {
    int D = H_kv * d;
    int G = H_q / H_kv;
    double inv_sqrt_d = 1.0 / sqrt((double)d);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int g = 0; g < H_q; ++g) {
        int h = g / G;
        double *qv = (double *)malloc(sizeof(double) * (size_t)d);
        double *qr = (double *)malloc(sizeof(double) * (size_t)d);
        double *kh = (double *)malloc(sizeof(double) * (size_t)d);
        double *kr = (double *)malloc(sizeof(double) * (size_t)d);
        double *vh = (double *)malloc(sizeof(double) * (size_t)d);
        double *sc = (double *)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));
        double *acc = parts + (size_t)g * (size_t)(d + 2);
        for (int i = 0; i < d; ++i) qv[i] = kvo_f16_to_f64(q[(size_t)g * d + i]);
        kvo_rope(qv, d, pos, theta_base, qr);
        double m = -INFINITY;
        for (int64_t n = 0; n < T; ++n) {
            for (int i = 0; i < d; ++i) {
                int c = h * d + i;
                float s, z;
                kvo_affine_from_range((double)key_lo[c], (double)key_hi[c], &s, &z);
                kh[i] = (double)cbK_dec[kcodes[n * D + c]] * (double)s + (double)z;
            }
            for (int64_t r = kptr[n]; r < kptr[n + 1]; ++r) {
                int c = kidx[r];
                if (c >= h * d && c < (h + 1) * d) kh[c - h * d] = kvo_f16_to_f64(kval[r]);
            }
            kvo_rope(kh, d, pos_base + n, theta_base, kr);
            double dot = 0.0;
            for (int i = 0; i < d; ++i) dot += qr[i] * kr[i];
            sc[n] = dot * inv_sqrt_d;
            if (sc[n] > m) m = sc[n];
        }
        double l = 0.0;
        for (int i = 0; i < d; ++i) acc[i] = 0.0;
        for (int64_t n = 0; n < T; ++n) {
            double p = exp(sc[n] - m);
            l += p;
            for (int i = 0; i < d; ++i) {
                int c = h * d + i;
                vh[i] = (double)cbV_dec[vcodes[n * D + c]] * (double)vs[n] + (double)vz[n];
            }
            for (int r = 0; r < kper; ++r) {
                int c = vidx[n * kper + r];
                if (c >= h * d && c < (h + 1) * d) vh[c - h * d] = kvo_f16_to_f64(vval[n * kper + r]);
            }
            for (int i = 0; i < d; ++i) acc[i] += p * vh[i];
        }
        acc[d] = m;
        acc[d + 1] = l;
        free(qv); free(qr); free(kh); free(kr); free(vh); free(sc);
    }
}

/* -------------------------------------------------------------------- Merge ---- */
/* Exact log-sum-exp merge of partials over disjoint token sets (north_star; textbook):
 *   m = max m_i;  l = sum e^{m_i - m} l_i;  o = sum e^{m_i - m} o_i / l,
 * in fixed order i = 0..P-1.  parts: [P][H][d+2] (o_unnorm, m, l). */
void kvo_merge(int P, int H, int d, const double *parts, double *o) {
    for (int g = 0; g < H; ++g) {
        double m = -INFINITY;
        for (int i = 0; i < P; ++i) {
            double mi = parts[((size_t)i * H + g) * (d + 2) + d];
            if (mi > m) m = mi;
        }
        double l = 0.0;
        double *og = o + (size_t)g * d;
        for (int c = 0; c < d; ++c) og[c] = 0.0;
        for (int i = 0; i < P; ++i) {
            const double *pi = parts + ((size_t)i * H + g) * (d + 2);
            if (pi[d + 1] == 0.0) continue; /* empty shard */
            double w = exp(pi[d] - m);
            l += w * pi[d + 1];
            for (int c = 0; c < d; ++c) og[c] += w * pi[c];
        }
        for (int c = 0; c < d; ++c) og[c] /= l;
    }
}

/* ------------------------------------------- online per-channel Key thresholds ---- */
/* "Online for K" (tab:calibration): the per-channel Key outlier
 * thresholds and scaling factors computed from the Keys being quantized instead of offline
 * calibration data.  Per channel c over the T tokens of a block: n = ceil(f T) outliers
 * (integer ceil from ppm, reading R2), the ceil(n/2) largest and floor(n/2) smallest excluded
 * (two-sided, reading R3), lo_c / hi_c = the smallest / largest kept value -- i.e. the
 * floor(n/2)-th and (T-1-ceil(n/2))-th order statistics.  -0 is returned as +0 (R3). */
static int cmp_f64(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}
int kvo_key_thresholds_online(int64_t T, int D, const uint16_t *K, int ppm, float *lo, float *hi) {
    int64_t n = (int64_t)(((int64_t)ppm * T + 999999) / 1000000);
    int64_t ku = (n + 1) / 2, kl = n / 2;
    if (T < 1 || ku + kl >= T) return -1;
    double *col = (double *)malloc(sizeof(double) * (size_t)T);
    for (int c = 0; c < D; ++c) {
        for (int64_t t = 0; t < T; ++t) col[t] = kvo_f16_to_f64(K[(size_t)t * D + c]);
        qsort(col, (size_t)T, sizeof(double), cmp_f64);
        double l = col[kl], h = col[T - 1 - ku];
        lo[c] = (float)(l == 0.0 ? 0.0 : l);
        hi[c] = (float)(h == 0.0 ? 0.0 : h);
    }
    free(col);
    return 0;
}

/* ------------------------------------------------------ fp16 comparator cache ---- */
/* The paper's baseline decode is fp16 mat-vec against an fp16 cache of post-RoPE Keys
 * ("Key fp16 Matvec", "Value fp16 Matvec"; BASELINE config C3 "fp16 cache").
 * kvo_f64_to_f16: IEEE binary16 round-to-nearest-even of a double, one rounding. */
uint16_t kvo_f64_to_f16(double x) {
    uint16_t sign = signbit(x) ? 0x8000u : 0u;
    double a = fabs(x);
    if (isnan(x)) return 0x7e00u;
    if (a >= 65520.0) return sign | 0x7c00u;           /* rounds to infinity */
    if (a < ldexp(1.0, -14)) {                          /* subnormal: multiples of 2^-24 */
        double q = a * ldexp(1.0, 24);
        double f = floor(q);
        double r = q - f;
        uint32_t m = (uint32_t)f;
        if (r > 0.5 || (r == 0.5 && (m & 1u))) m++;
        return sign | (uint16_t)m;                      /* m == 1024 is the smallest normal */
    }
    int e;
    double fr = frexp(a, &e);                           /* a = fr * 2^e, fr in [0.5, 1) */
    double q = ldexp(fr, 11);                           /* 11 significant bits */
    double f = floor(q);
    double r = q - f;
    uint32_t m = (uint32_t)f;
    if (r > 0.5 || (r == 0.5 && (m & 1u))) m++;
    if (m == 2048) { m = 1024; e++; }
    int be = e - 1 + 15;                                /* biased exponent of 1.xxx * 2^(e-1) */
    if (be >= 31) return sign | 0x7c00u;
    return sign | (uint16_t)(be << 10) | (uint16_t)(m - 1024);
}

/* Stored Key of the fp16 cache: RoPE at position pos (fp64, kvo_rope) of every head of one
 * token, rounded once to fp16.  x, out: [H d] fp16 bits. */
void kvo_f16cache_key(const uint16_t *x, int H, int d, int64_t pos, double theta_base, uint16_t *out) {
    double *xv = (double *)malloc(sizeof(double) * (size_t)d);
    double *xr = (double *)malloc(sizeof(double) * (size_t)d);
    for (int h = 0; h < H; ++h) {
        for (int i = 0; i < d; ++i) xv[i] = kvo_f16_to_f64(x[(size_t)h * d + i]);
        kvo_rope(xv, d, pos, theta_base, xr);
        for (int i = 0; i < d; ++i) out[(size_t)h * d + i] = kvo_f64_to_f16(xr[i]);
    }
    free(xv);
    free(xr);
}

/* Decode attention over a dense cache of post-RoPE Keys (plain definition, reading R13):
 *   q~ = RoPE(q_g, pos); s_n = q~ . K_n / sqrt(d); o_g = sum_n e^{s_n - m} V_n / sum e^{s_n - m}
 * Kpost, V: [T][H_kv d] fp16 bits; q [H_q][d] fp16 bits; o [H_q][d]. */
void kvo_attend_dense(int64_t T, int H_q, int H_kv, int d, const uint16_t *Kpost,
                      const uint16_t *V, const uint16_t *q, int64_t pos, double theta_base,
                      double *o) {
    int G = H_q / H_kv, D = H_kv * d;
    double *qv = (double *)malloc(sizeof(double) * (size_t)d);
    double *qr = (double *)malloc(sizeof(double) * (size_t)d);
    double *s = (double *)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));
    for (int g = 0; g < H_q; ++g) {
        int h = g / G;
        for (int i = 0; i < d; ++i) qv[i] = kvo_f16_to_f64(q[(size_t)g * d + i]);
        kvo_rope(qv, d, pos, theta_base, qr);
        double m = -INFINITY;
        for (int64_t n = 0; n < T; ++n) {
            double acc = 0.0;
            for (int i = 0; i < d; ++i) acc += qr[i] * kvo_f16_to_f64(Kpost[(size_t)n * D + h * d + i]);
            s[n] = acc / sqrt((double)d);
            if (s[n] > m) m = s[n];
        }
        double l = 0.0;
        double *og = o + (size_t)g * d;
        for (int i = 0; i < d; ++i) og[i] = 0.0;
        for (int64_t n = 0; n < T; ++n) {
            double p = exp(s[n] - m);
            l += p;
            for (int i = 0; i < d; ++i) og[i] += p * kvo_f16_to_f64(V[(size_t)n * D + h * d + i]);
        }
        for (int i = 0; i < d; ++i) og[i] /= l;
    }
    free(qv);
    free(qr);
    free(s);
}

/* ------------------------------------------------------------------ Packing ---- */
/* Canonical exchange packing ("packed into 32-bit words"): code j occupies bits
 * [j*b, (j+1)*b) of a little-endian bitstream, bit 0 = LSB of word 0; codes straddle
 * words for b = 3; words = ceil(n*b/32); pad bits zero. */
void kvo_pack(const uint16_t *codes, int64_t n, int bits, uint32_t *words) {
    int64_t nw = (n * bits + 31) / 32;
    for (int64_t w = 0; w < nw; ++w) words[w] = 0;
    for (int64_t j = 0; j < n; ++j) {
        for (int b = 0; b < bits; ++b) {
            int64_t bit = j * bits + b;
            if ((codes[j] >> b) & 1) words[bit / 32] |= (uint32_t)1 << (bit % 32);
        }
    }
}

void kvo_unpack(const uint32_t *words, int64_t n, int bits, uint16_t *codes) {
    for (int64_t j = 0; j < n; ++j) {
        uint16_t c = 0;
        for (int b = 0; b < bits; ++b) {
            int64_t bit = j * bits + b;
            if ((words[bit / 32] >> (bit % 32)) & 1) c |= (uint16_t)(1 << b);
        }
        codes[j] = c;
    }
}
