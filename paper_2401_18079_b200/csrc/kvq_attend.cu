// kvq_attend.cu -- ATT: fused single-token decode attention over the compressed cache.
//
// One launch per attend:
//   grid  = n_head_groups x splits (head group fastest), 256 threads, 1 CTA / SM.
//   Staging: every 32-token tile of the CTA's head group (K code words, V code words,
//          per-token (s,z), CSC pointers, Value and Key outlier records) is moved
//          global -> shared by TMA bulk copies (cp.async.bulk + mbarrier complete_tx)
//          into a STAGES-deep ring, issued STAGES-1 tiles ahead by warp 0, so the compute
//          phases never wait on HBM latency.
//   a1 QP  each CTA rotates its HG query heads with exact fp64 angles (R11, R12) and
//          folds 1/sqrt(d) * log2(e) into q~.
//   LUTs   K: per (query head g, RoPE pair i) a 2^{2b}-entry table of fp16 pairs
//          (A, B) with  A = q~_i K^_i(a) + q~_i' K^_i'(b),  B = q~_i' K^_i(a) - q~_i K^_i'(b)
//          for K^_c(a) = Chat_K[a] s_c + z_c -- the paper's per-channel LUT
//          taken one step further: the query and the per-channel affine are folded in, so
//          one lookup + 2 FMAs per RoPE pair yields  cos(n'th_i) A + sin(n'th_i) B, which
//          is exactly the pair's contribution to q~ . RoPE(K^_n, n').
//          Pairs carrying a heavy Key channel get fp32 tables (precision, DESIGN 9).
//          V: the shared codebook as a pair table, lane-private copies (conflict-free).
//   a2 KS  lane = token of the tile, warp w = RoPE pairs 8w..8w+7 for all heads;
//          fp16 x fp16 -> fp32 FMAs (fma.rn.f32.f16).
//   a3     Key outliers of the tile add (x - K^(code)) * dscore/dK (same launch).
//   a4     exact online softmax in base 2 (running max, rescale on change).
//   a5 PV  lane = CPL channels:  sum_n (p_n s_n) Chat_V[code] + sum_n p_n z_n  (affine fold).
//   a6     Value outliers add p_n (v - V^(code)).
//   a7 MRG the last CTA of each head group merges the split partials (log-sum-exp).
#include "kvq_internal.cuh"

#include <math_constants.h>

namespace kvq {
namespace {

constexpr int ATT_THREADS = 512;
constexpr int ATT_WARPS = 16;
constexpr int KPW = kPairs / ATT_WARPS;   // RoPE pairs per warp in the K phase

// ------------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// acc += lo(x)*lo(y) ; acc2 += hi(x)*hi(y)   (fp16 products, fp32 accumulation)
__device__ __forceinline__ void fma2_f16_f32(uint32_t x, uint32_t y, float &acc, float &acc2) {
    asm("{\n\t.reg .b16 x0, x1, y0, y1;\n\t"
        "mov.b32 {x0, x1}, %2;\n\t"
        "mov.b32 {y0, y1}, %3;\n\t"
        "fma.rn.f32.f16 %0, x0, y0, %0;\n\t"
        "fma.rn.f32.f16 %1, x1, y1, %1;\n\t}"
        : "+f"(acc), "+f"(acc2)
        : "r"(x), "r"(y));
}

// acc_a += w*lo(v) ; acc_b += w*hi(v)   with w a scalar fp16
__device__ __forceinline__ void fma_w_f16x2(uint16_t w, uint32_t v, float &acc_a, float &acc_b) {
    asm("{\n\t.reg .b16 v0, v1;\n\t"
        "mov.b32 {v0, v1}, %3;\n\t"
        "fma.rn.f32.f16 %0, %2, v0, %0;\n\t"
        "fma.rn.f32.f16 %1, %2, v1, %1;\n\t}"
        : "+f"(acc_a), "+f"(acc_b)
        : "h"(w), "r"(v));
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- configuration --
constexpr int cpl_for(int bits, int /*hg*/) {
    // V channels per lane: whole 32-bit words of codes per lane (b=4: 8, b=2/3: 32);
    // one (head, token-group) task per warp needs HG * 128/CPL <= 16 (see caps below)
    return bits == 4 ? 8 : 32;
}

template <int BITS, int HG>
struct Cfg {
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int HMAX = BITS == 4 ? 4 : 8;   // fp32 "heavy" pairs per head
    static constexpr int CPL = cpl_for(BITS, HG);
    static constexpr size_t klut = (size_t)HG * kPairs * NE * 4;
    static constexpr size_t vlut = (size_t)NE * 32 * 4;
    static constexpr size_t hlut = (size_t)HG * HMAX * NE * 8;
    static constexpr size_t cis = (size_t)kPairs * 32 * 8;
    static constexpr size_t small =
        HG * kHeadDim * 4              /* qs */
        + ATT_WARPS * HG * 32 * 4      /* red */
        + HG * 32 * 4 * 2              /* p, kcorr */
        + 4 * 33 * 4                   /* per-token record sub-ranges + prefix */
        + HG * kHeadDim * 4 * 2 + 64 * 4 /* staged s_c, z_c of the group, codebooks */
        + HG * 32 * 2                  /* w16 */
        + HG * kHeadDim * 4            /* osp */
        + 64 * 16 * 3 + 64 * 8         /* anc64, rot64, qcis, anc32 */
        + 64 * 4                       /* theta32 */
        + HG * 4 * 8                   /* per-head scalars */
        + HG * 64 * 4 + HG * 64        /* bound, heavy flags */
        + HG * 16 * 4                  /* heavy pair list + counts */
        + 256;
    static constexpr size_t fixed = klut + vlut + hlut + cis + small;
};

struct Params {
    const __half *q;
    int64_t pos, T;
    int S;               // splits
    int ntiles;
    float *out;
    float *parts;
    unsigned *tickets;
    int write_partial;
    // stage ring layout (bytes), computed on the host
    int stages;
    int krec_cap;        // u32 records per stage buffer (multiple of 4)
    unsigned st_base, st_bytes, so_kw, so_vw, so_vsz, so_kptr, so_vrec, so_krec;
    unsigned long long *timers;   // optional [8] phase cycle sums (diagnostics), may be null
};

template <int BITS, int HG, int G>
__global__ void __launch_bounds__(ATT_THREADS, 1) att_kernel(DevCache c, Params P) {
    using C = Cfg<BITS, HG>;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int HKV = HG / G;
    constexpr int QWC = HKV * 4 * BITS;             // K (and V) words per token in the CTA
    constexpr int CPL = C::CPL;                     // V channels per lane
    constexpr int VWL = CPL * BITS / 32;            // V words per lane per token
    constexpr int HMAX = C::HMAX;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sp = smem_raw;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += C::klut;
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += C::hlut;
    float2 *cis_s = reinterpret_cast<float2 *>(sp); sp += C::cis;
    float *qs = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *red = reinterpret_cast<float *>(sp); sp += ATT_WARPS * HG * 32 * 4;
    float *p_s = reinterpret_cast<float *>(sp); sp += HG * 32 * 4;
    float *kcorr = reinterpret_cast<float *>(sp); sp += HG * 32 * 4;
    int *rk_beg = reinterpret_cast<int *>(sp); sp += 33 * 4;   // K records of this head group
    int *rk_len = reinterpret_cast<int *>(sp); sp += 33 * 4;
    int *rv_beg = reinterpret_cast<int *>(sp); sp += 33 * 4;   // V records of this head group
    int *rv_len = reinterpret_cast<int *>(sp); sp += 33 * 4;
    float *ks_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;   // s_c of the group's channels
    float *kz_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;             // 4 codebooks
    float *osp = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    double2 *anc64 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double2 *rot64 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double2 *qcis = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    float2 *anc32 = reinterpret_cast<float2 *>(sp); sp += 64 * 8;
    float *theta32 = reinterpret_cast<float *>(sp); sp += 64 * 4;
    float *lut_inv = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *alpha_s = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *beta_s = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *m_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *l_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *z_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    uint16_t *w16 = reinterpret_cast<uint16_t *>(sp); sp += HG * 32 * 2;
    float *bound_s = reinterpret_cast<float *>(sp); sp += HG * 64 * 4;
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(sp); sp += HG * 64;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *flag_s = reinterpret_cast<int *>(sp); sp += 16;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + P.st_base - 64);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_hg = c.H_q / HG;
    const int hg = blockIdx.x % n_hg;
    const int split = blockIdx.x / n_hg;
    const int g0 = hg * HG;          // first query head
    const int h0 = g0 / G;           // first KV head
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int D = c.D;
    const int kv = c.kv;
    const float *ks = c.kpar, *kz = c.kpar + D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;   // decode codebooks

    auto stage_ptr = [&](int st) -> unsigned char * { return smem_raw + P.st_base + (size_t)st * P.st_bytes; };

    // ----------------------------------------------------------- TMA producer
    // kp_lo/kp_hi: CSC pointers of the next tile to issue (prefetched one issue ahead)
    uint32_t kp_lo = 0, kp_hi = 0;
    auto kptr_at = [&](int t, uint32_t &lo, uint32_t &hi) {
        const int64_t n0 = (int64_t)t * 32;
        const int64_t n1 = n0 + 32 < P.T ? n0 + 32 : P.T;
        lo = __ldg(c.kptr + n0);
        hi = __ldg(c.kptr + n1);
    };
    auto issue = [&](int t, int st) {   // producer warp only
        if (t >= t_end) return;
        unsigned char *sb = stage_ptr(st);
        uint64_t *bar = bars + st;
        const uint32_t klo = __shfl_sync(0xffffffffu, kp_lo, 0);
        const uint32_t khi = __shfl_sync(0xffffffffu, kp_hi, 0);
        const uint32_t ka = klo & ~3u;
        uint32_t kn = ((khi + 3u) & ~3u) - ka;
        if (kn > (uint32_t)P.krec_cap) kn = (uint32_t)P.krec_cap;
        const unsigned b_kw = 32u * QWC * 4u;
        const unsigned b_vrec = 32u * (unsigned)kv * 4u;
        const unsigned total = 2u * b_kw + 256u + 192u + b_vrec + kn * 4u;
        if (lane == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, total);
        }
        __syncwarp();
        const int64_t n0 = (int64_t)t * 32;
        if (lane == 0)
            bulk_g2s(sb + P.so_kw, c.kcodes + ((int64_t)t * c.QW + h0 * 4 * BITS) * 32, b_kw, bar);
        if (lane == 1) bulk_g2s(sb + P.so_vsz, c.vsz + n0, 256u, bar);
        if (lane == 2) bulk_g2s(sb + P.so_kptr, c.kptr + n0, 192u, bar);
        if (lane == 3 && b_vrec) bulk_g2s(sb + P.so_vrec, c.vout + n0 * kv, b_vrec, bar);
        if (lane == 4 && kn) bulk_g2s(sb + P.so_krec, c.kout + ka, kn * 4u, bar);
        if (lane == 5)
            bulk_g2s(sb + P.so_vw, c.vcodes + ((int64_t)t * c.H_kv + h0) * 32 * 4 * BITS, b_kw, bar);
        // prefetch the CSC range of the tile after this one
        if (lane == 0 && t + 1 < t_end) kptr_at(t + 1, kp_lo, kp_hi);
    };

    if (tid == 0) {
        for (int s = 0; s < P.stages; ++s) mbar_init(bars + s, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == ATT_WARPS - 1) {   // the producer warp (also issues inside the tile loop)
        if (lane == 0 && t_begin < t_end) kptr_at(t_begin, kp_lo, kp_hi);
        for (int s = 0; s < P.stages - 1; ++s) issue(t_begin + s, s);
    }

    // ---------------------------------------------------------------- prologue
    if (tid < 64) {
        const int i = tid;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        theta32[i] = (float)th;
        double s, co;
        sincos((double)P.pos * th, &s, &co);
        qcis[i] = make_double2(co, s);
        const double a0 = (double)(c.pos_base + (int64_t)t_begin * kTileTokens) * th;
        sincos(a0, &s, &co);
        anc64[i] = make_double2(co, s);
        anc32[i] = make_float2((float)co, (float)s);
        sincos(32.0 * th, &s, &co);
        rot64[i] = make_double2(co, s);
    }
    for (int x = tid; x < HG * kHeadDim; x += ATT_THREADS) osp[x] = 0.f;
    for (int x = tid; x < HKV * kHeadDim; x += ATT_THREADS) {
        ks_s[x] = ks[h0 * kHeadDim + x];
        kz_s[x] = kz[h0 * kHeadDim + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
    for (int x = tid; x < HG * 32; x += ATT_THREADS) kcorr[x] = 0.f;
    if (tid < 16) flag_s[tid] = 0;
    __syncthreads();
    // a1: q~ = RoPE(q, pos) * log2(e)/sqrt(d)
    const double qscale = 1.4426950408889634 / sqrt((double)kHeadDim);
    for (int x = tid; x < HG * 64; x += ATT_THREADS) {
        const int g = x >> 6, i = x & 63;
        const __half *qg = P.q + (int64_t)(g0 + g) * kHeadDim;
        const double a = (double)__half2float(qg[i]), b = (double)__half2float(qg[i + 64]);
        const double2 cs = qcis[i];
        qs[g * kHeadDim + i] = (float)((a * cs.x - b * cs.y) * qscale);
        qs[g * kHeadDim + i + 64] = (float)((b * cs.x + a * cs.y) * qscale);
    }
    __syncthreads();
    // K tables: per (head, pair) bound of |A|,|B|.  The few pairs carrying a heavy Key
    // channel (bound > 1/4 of the head max, at most HMAX per head) get fp32 tables and
    // are accumulated in fp32; the rest use fp16 tables scaled by the largest remaining
    // bound.
    for (int x = tid; x < HG * 64; x += ATT_THREADS) {
        const int g = x >> 6, i = x & 63;
        const int kvh = (g0 + g) / G;
        const int ci = kvh * kHeadDim + i, cj = ci + 64;
        const float mx = fmaxf(fabsf(cbK[0] * ks[ci] + kz[ci]), fabsf(cbK[CM] * ks[ci] + kz[ci]));
        const float my = fmaxf(fabsf(cbK[0] * ks[cj] + kz[cj]), fabsf(cbK[CM] * ks[cj] + kz[cj]));
        const float qa = fabsf(qs[g * kHeadDim + i]), qb = fabsf(qs[g * kHeadDim + i + 64]);
        bound_s[x] = fmaxf(qa * mx + qb * my, qb * mx + qa * my);
    }
    __syncthreads();
    for (int g = warp; g < HG; g += ATT_WARPS) {
        const float b0 = bound_s[g * 64 + lane], b1 = bound_s[g * 64 + 32 + lane];
        const float M = warp_max(fmaxf(b0, b1));
        float tau = 0.25f * M;
        unsigned m0 = __ballot_sync(0xffffffffu, b0 > tau), m1 = __ballot_sync(0xffffffffu, b1 > tau);
        while (__popc(m0) + __popc(m1) > HMAX) {
            tau *= 1.25f;
            m0 = __ballot_sync(0xffffffffu, b0 > tau);
            m1 = __ballot_sync(0xffffffffu, b1 > tau);
        }
        const unsigned lt = (1u << lane) - 1u;
        const int n0c = __popc(m0);
        if ((m0 >> lane) & 1u) hv_pair[g * 8 + __popc(m0 & lt)] = lane;
        if ((m1 >> lane) & 1u) hv_pair[g * 8 + n0c + __popc(m1 & lt)] = lane + 32;
        heavy_s[g * 64 + lane] = (m0 >> lane) & 1u;
        heavy_s[g * 64 + 32 + lane] = (m1 >> lane) & 1u;
        const float rest = warp_max(fmaxf(((m0 >> lane) & 1u) ? 0.f : b0, ((m1 >> lane) & 1u) ? 0.f : b1));
        if (lane == 0) {
            hv_n[g] = n0c + __popc(m1);
            int e = 0;     // scale so that |entry| <= 2^14 (fp16 max 65504)
            if (rest > 0.f && isfinite(rest)) e = 14 - ilogbf(rest) - 1;
            e = max(-100, min(100, e));
            alpha_s[g] = ldexpf(1.f, e);      // temp: table scale
            lut_inv[g] = ldexpf(1.f, -e);
        }
    }
    __syncthreads();
    // K table entries
    for (int x = tid; x < HG * 64; x += ATT_THREADS) {
        const int g = x >> 6, i = x & 63;
        const int kvh = (g0 + g) / G;
        const int ci = kvh * kHeadDim + i, cj = ci + 64;
        const float sc = alpha_s[g];
        const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
        const float qa = qa1 * sc, qb = qb1 * sc;
        float X[1 << BITS], Y[1 << BITS];
#pragma unroll
        for (int a = 0; a <= CM; ++a) {
            X[a] = cbK[a] * ks[ci] + kz[ci];
            Y[a] = cbK[a] * ks[cj] + kz[cj];
        }
        uint32_t *dst = klut + (size_t)(g * 64 + i) * NE;
        const bool heavy = heavy_s[x] != 0;
        int hslot = 0;
        if (heavy)
            for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
#pragma unroll 1
        for (int bb = 0; bb <= CM; ++bb) {
            float yb = 0.f;
#pragma unroll
            for (int u = 0; u <= CM; ++u) yb = (u == bb) ? Y[u] : yb;
#pragma unroll
            for (int a = 0; a <= CM; ++a) {
                const int e = a | (bb << BITS);
                if (heavy) {
                    dst[e] = 0u;
                    hlut[(g * HMAX + hslot) * NE + e] = make_float2(qa1 * X[a] + qb1 * yb, qb1 * X[a] - qa1 * yb);
                } else {
                    dst[e] = pack_half2(qa * X[a] + qb * yb, qb * X[a] - qa * yb);
                }
            }
        }
    }
    // V table: lane-private copies (entry e for lane slot l at word e*32 + l)
    for (int x = tid; x < NE * 32; x += ATT_THREADS) {
        const int e = x >> 5;
        vlut[x] = pack_half2(cbV[e & CM], cbV[e >> BITS]);
    }

    // per-lane constants for the K phase: cis(j * theta_i) for this warp's KPW pairs
    float t1c[KPW], t1s[KPW];
#pragma unroll
    for (int k = 0; k < KPW; ++k) {
        const int i = warp * KPW + k;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        float s, co;
        sincosf((float)((double)lane * th), &s, &co);
        t1c[k] = co;
        t1s[k] = s;
    }

    // V-phase task mapping: one (query head, token group) task per warp
    constexpr int LH = kHeadDim / CPL;          // lanes per token per head
    constexpr int TPW = 32 / LH;                // tokens per warp task
    constexpr int NTASK = HG * (32 / TPW);      // tasks per tile
    static_assert(NTASK <= ATT_WARPS, "V tasks must fit the CTA's warps");
    const bool vtask = warp < NTASK;
    const int vh = vtask ? warp / (32 / TPW) : 0;            // local query head
    const int vj = (warp % (32 / TPW)) * TPW + lane / LH;    // token in the tile
    const int vq = lane % LH;                                // channel group in the head
    const int vkv = vh / G;                                  // local kv head
    float acc[CPL];
#pragma unroll
    for (int x = 0; x < CPL; ++x) acc[x] = 0.f;

    // running softmax state (S-phase warps: warp g <-> head g)
    float m_run = -CUDART_INF_F, l_run = 0.f, z_run = 0.f;
    int E_cur = -126;     // dense V accumulator units: 2^E_cur (CTA uniform)

    const int kbit0 = 2 * BITS * KPW * warp;
    const int kq0 = kbit0 >> 5, kshift = kbit0 & 31;
    const int c_lo = h0 * kHeadDim, c_hi = (h0 + HKV) * kHeadDim;
    __syncthreads();

    unsigned long long tm[6] = {0, 0, 0, 0, 0, 0};
    long long tc0 = clock64(), tc1;
    const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
    for (int t = t_begin; t < t_end; ++t) {
        const int it = t - t_begin;
        const int st = it % P.stages;
        mbar_wait(bars + st, (unsigned)((it / P.stages) & 1));
        tc1 = clock64(); tm[1] += tc1 - tc0; tc0 = tc1;
        unsigned char *sb = stage_ptr(st);
        const uint32_t *kw_s = reinterpret_cast<const uint32_t *>(sb + P.so_kw);
        const uint32_t *vw_s = reinterpret_cast<const uint32_t *>(sb + P.so_vw);
        const float2 *vsz_s = reinterpret_cast<const float2 *>(sb + P.so_vsz);
        const uint32_t *kptr_s = reinterpret_cast<const uint32_t *>(sb + P.so_kptr);
        const uint32_t *vrec_s = reinterpret_cast<const uint32_t *>(sb + P.so_vrec);
        const uint32_t *krec_s = reinterpret_cast<const uint32_t *>(sb + P.so_krec);
        const int64_t n0 = (int64_t)t * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        const uint32_t ka = kptr_s[0] & ~3u;
        auto krec = [&](uint32_t r) -> uint32_t {
            const uint32_t off = r - ka;
            if (off < (uint32_t)P.krec_cap) return krec_s[off];
            return __ldcg(c.kout + r);    // beyond the staged window (very dense tiles)
        };

        // ---- per-token record sub-ranges of this head group: records are channel-sorted,
        //      so the first record >= c is popc(ballot(ch < c)) past the token's start
        for (int j = warp; j < 32; j += ATT_WARPS) {
            int kb = 0, kn = 0, vb = 0, vn = 0;
            if (j < ntok) {
                const uint32_t r0 = kptr_s[j], r1 = kptr_s[j + 1];
                int below_lo = 0, below_hi = 0;
                for (uint32_t rb = r0; rb < r1; rb += 32) {
                    const uint32_t r = rb + lane;
                    const int ch = r < r1 ? (int)(krec(r) & 0xffffu) : 0x7fffffff;
                    below_lo += __popc(__ballot_sync(0xffffffffu, ch < c_lo));
                    below_hi += __popc(__ballot_sync(0xffffffffu, ch < c_hi));
                }
                kb = (int)r0 + below_lo;
                kn = below_hi - below_lo;
                below_lo = below_hi = 0;
                for (int rb = 0; rb < kv; rb += 32) {
                    const int r = rb + lane;
                    const int ch = r < kv ? (int)(vrec_s[j * kv + r] & 0xffffu) : 0x7fffffff;
                    below_lo += __popc(__ballot_sync(0xffffffffu, ch < c_lo));
                    below_hi += __popc(__ballot_sync(0xffffffffu, ch < c_hi));
                }
                vb = j * kv + below_lo;
                vn = below_hi - below_lo;
            }
            if (lane == 0) { rk_beg[j] = kb; rk_len[j] = kn; rv_beg[j] = vb; rv_len[j] = vn; }
        }

        // ------------------------------------------------------------ a2: K dense
        {
            float acc_c[HG], acc_s[HG];
#pragma unroll
            for (int g = 0; g < HG; ++g) { acc_c[g] = 0.f; acc_s[g] = 0.f; }
            unsigned long long win[HKV];
#pragma unroll
            for (int h = 0; h < HKV; ++h) {
                unsigned long long w64 = kw_s[(h * 4 * BITS + kq0) * 32 + lane];
                if (kshift + 2 * BITS * KPW > 32)
                    w64 |= (unsigned long long)kw_s[(h * 4 * BITS + kq0 + 1) * 32 + lane] << 32;
                win[h] = w64 >> kshift;
            }
#pragma unroll
            for (int k = 0; k < KPW; ++k) {
                const int i = warp * KPW + k;
                const float2 an = anc32[i];
                const float cc = an.x * t1c[k] - an.y * t1s[k];
                const float ss = an.x * t1s[k] + an.y * t1c[k];
                const uint32_t cs = pack_half2(cc, ss);
                cis_s[i * 32 + lane] = make_float2(cc, ss);
#pragma unroll
                for (int h = 0; h < HKV; ++h) {
                    const int pc = (int)((win[h] >> (2 * BITS * k)) & (NE - 1));
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int g = h * G + gg;
                        const uint32_t ab = klut[(g * 64 + i) * NE + pc];
                        fma2_f16_f32(ab, cs, acc_c[g], acc_s[g]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < HG; ++g) red[(warp * HG + g) * 32 + lane] = acc_c[g] + acc_s[g];
        }
        __syncthreads();
        tc1 = clock64(); tm[2] += tc1 - tc0; tc0 = tc1;

        // --------------------- a3: K outliers + heavy pairs, flat over the CTA's threads
        {
            int kl = rk_len[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, kl, o);
                if (lane >= o) kl += y;
            }
            const int ktot = __shfl_sync(0xffffffffu, kl, 31);
            for (int xb = warp * 32; xb < ktot; xb += ATT_THREADS) {
                const int x = xb + lane;
                int j = 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, kl, j + o - 1);
                    if (v <= x) j += o;
                }
                const int excl = __shfl_sync(0xffffffffu, kl, (j + 31) & 31);
                if (x >= ktot) continue;
                const uint32_t rec = krec((uint32_t)(rk_beg[j] + (x - (j ? excl : 0))));
                const int ch = (int)(rec & 0xffffu);
                const int kvl = (ch >> 7) - h0;
                const int cc = ch & 127, i = cc & 63, up = cc >> 6;
                const int bit = 2 * BITS * i;
                const int wq = kvl * 4 * BITS + (bit >> 5);
                unsigned long long w64 = kw_s[wq * 32 + j];
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + j] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const int code = (pc >> (up * BITS)) & CM;
                const float xval = __half2float(__ushort_as_half((uint16_t)(rec >> 16)));
                const int cl = kvl * kHeadDim + cc;
                const float delta = xval - (cbKs[code] * ks_s[cl] + kz_s[cl]);
                const float2 cs = cis_s[i * 32 + j];
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    const int g = kvl * G + gg;
                    const float qa = qs[g * kHeadDim + i], qb = qs[g * kHeadDim + i + 64];
                    atomicAdd(&kcorr[g * 32 + j], delta * (up ? (qb * cs.x - qa * cs.y) : (qa * cs.x + qb * cs.y)));
                }
            }
            // heavy RoPE pairs in fp32: items (head g, heavy slot, token j)
            for (int x = tid; x < HG * HMAX * 32; x += ATT_THREADS) {
                const int g = x / (HMAX * 32), hs = (x / 32) % HMAX, j = x & 31;
                if (hs >= hv_n[g] || j >= ntok) continue;
                const int i = hv_pair[g * 8 + hs];
                const int bit = 2 * BITS * i;
                const int wq = (g / G) * 4 * BITS + (bit >> 5);
                unsigned long long w64 = kw_s[wq * 32 + j];
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + j] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const float2 ab = hlut[(g * HMAX + hs) * NE + pc];
                const float2 cs = cis_s[i * 32 + j];
                atomicAdd(&kcorr[g * 32 + j], cs.x * ab.x + cs.y * ab.y);
            }
            // TMA producer for tile t + STAGES - 1 (the buffer of tile t-1 is free): the last
            // warp issues here so that no warp's K phase waits on it
            if (warp == ATT_WARPS - 1) issue(t + P.stages - 1, (it + P.stages - 1) % P.stages);
        }
        __syncthreads();
        tc1 = clock64(); tm[0] += tc1 - tc0; tc0 = tc1;

        // ------------------------------------------------------- a4: online softmax
        {
            float smax = lane < ntok ? vsz_s[lane].x : 0.f;
            smax = warp_max(smax);
            int E_new = E_cur;
            if (smax > 0.f) E_new = max(E_cur, ilogbf(smax) + 1);
            for (int g = warp; g < HG; g += ATT_WARPS) {
                const int j = lane;
                const bool valid = j < ntok;
                float s = 0.f;
#pragma unroll
                for (int w = 0; w < ATT_WARPS; ++w) s += red[(w * HG + g) * 32 + j];
                s = valid ? s * lut_inv[g] + kcorr[g * 32 + j] : -CUDART_INF_F;
                kcorr[g * 32 + j] = 0.f;
                const float mt = warp_max(s);
                const float m_new = fmaxf(m_run, mt);
                const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run - m_new);
                const float p = valid ? exp2f(s - m_new) : 0.f;
                const float2 sz = valid ? vsz_s[j] : make_float2(0.f, 0.f);
                l_run = l_run * alpha + warp_sum(p);
                z_run = z_run * alpha + warp_sum(p * sz.y);
                m_run = m_new;
                p_s[g * 32 + j] = p;
                w16[g * 32 + j] = __half_as_ushort(__float2half_rn(p * ldexpf(sz.x, -E_new)));
                if (alpha != 1.f) {
#pragma unroll
                    for (int x = 0; x < kHeadDim / 32; ++x) osp[g * kHeadDim + x * 32 + lane] *= alpha;
                }
                if (lane == 0) beta_s[g] = alpha * ldexpf(1.f, E_cur - E_new);
            }
            E_cur = E_new;
        }
        __syncthreads();
        tc1 = clock64(); tm[3] += tc1 - tc0; tc0 = tc1;

        // -------------------------------------------------------- a5: P.V dense
        if (vtask) {
            const float b = beta_s[vh];
            if (b != 1.f) {
#pragma unroll
                for (int x = 0; x < CPL; ++x) acc[x] *= b;
            }
            const uint16_t w = w16[vh * 32 + vj];
            uint32_t vw[VWL];
            const uint32_t *src = vw_s + (vkv * 32 + vj) * (4 * BITS) + vq * VWL;
#pragma unroll
            for (int x = 0; x < VWL; ++x) vw[x] = src[x];
#pragma unroll
            for (int pp = 0; pp < CPL / 2; ++pp) {
                const int bit = 2 * BITS * pp;
                const int wi = bit >> 5, sh = bit & 31;
                uint32_t pc;
                if (sh + 2 * BITS <= 32) pc = (vw[wi] >> sh) & (NE - 1);
                else pc = (uint32_t)((((unsigned long long)vw[wi + 1] << 32) | vw[wi]) >> sh) & (NE - 1);
                const uint32_t cv = vlut[pc * 32 + lane];
                fma_w_f16x2(w, cv, acc[2 * pp], acc[2 * pp + 1]);
            }
        }

        // ------------------------------- a6: V outliers (flat over relevant records)
        {
            int vl = rv_len[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, vl, o);
                if (lane >= o) vl += y;
            }
            const int vtot = __shfl_sync(0xffffffffu, vl, 31);
            for (int xb = warp * 32; xb < vtot; xb += ATT_THREADS) {
                const int x = xb + lane;
                int j = 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, vl, j + o - 1);
                    if (v <= x) j += o;
                }
                const int excl = __shfl_sync(0xffffffffu, vl, (j + 31) & 31);
                if (x >= vtot) continue;
                const uint32_t rec = vrec_s[rv_beg[j] + (x - (j ? excl : 0))];
                const int ch = (int)(rec & 0xffffu);
                const int kvl = (ch >> 7) - h0;
                const int bit = BITS * (ch & 127);
                const uint32_t *vrow = vw_s + (kvl * 32 + j) * (4 * BITS);
                unsigned long long w64 = vrow[bit >> 5];
                if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)vrow[(bit >> 5) + 1] << 32;
                const int code = (int)((w64 >> (bit & 31)) & CM);
                const float2 sz = vsz_s[j];
                const float xval = __half2float(__ushort_as_half((uint16_t)(rec >> 16)));
                const float delta = xval - (cbVs[code] * sz.x + sz.y);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    const int g = kvl * G + gg;
                    atomicAdd(&osp[g * kHeadDim + (ch & 127)], p_s[g * 32 + j] * delta);
                }
            }
        }

        // advance anchors to the next tile (fp64 complex rotation by 32 theta_i)
        if (tid < 64) {
            const double2 a = anc64[tid], r = rot64[tid];
            const double2 b = make_double2(a.x * r.x - a.y * r.y, a.x * r.y + a.y * r.x);
            anc64[tid] = b;
            anc32[tid] = make_float2((float)b.x, (float)b.y);
        }
        __syncthreads();
        tc1 = clock64(); tm[4] += tc1 - tc0; tc0 = tc1;
    }
    if (P.timers && tid == 0) {
#pragma unroll
        for (int x = 0; x < 5; ++x) atomicAdd(P.timers + x, tm[x]);
        atomicAdd(P.timers + 5, (unsigned long long)(t_end - t_begin));
    }

    // ------------------------------------------------------------ write partial
    for (int g = warp; g < HG; g += ATT_WARPS)
        if (lane == 0) { m_fin[g] = m_run; l_fin[g] = l_run; z_fin[g] = z_run; }
    {
        const float sc = ldexpf(1.f, E_cur);
        float *dst = osp + vh * kHeadDim + vq * CPL;
        if (vtask) {
#pragma unroll
            for (int x = 0; x < CPL; ++x) atomicAdd(&dst[x], acc[x] * sc);
        }
    }
    __syncthreads();
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    for (int x = tid; x < HG * kHeadDim; x += ATT_THREADS) {
        const int g = x >> 7, ch = x & 127;
        part[(g0 + g) * (kHeadDim + 2) + ch] = osp[x] + z_fin[g];
    }
    if (tid < HG) {
        part[(g0 + tid) * (kHeadDim + 2) + kHeadDim] = m_fin[tid];
        part[(g0 + tid) * (kHeadDim + 2) + kHeadDim + 1] = l_fin[tid];
    }
    // ------------------------------------------------------- a7: split merge
    __threadfence();
    __syncthreads();
    int *s_last = flag_s + 1;
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.tickets[hg], 1u);
        *s_last = (prev == (unsigned)(P.S - 1));
    }
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    for (int x = tid; x < HG * (kHeadDim + 2); x += ATT_THREADS) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        const int gq = g0 + g;
        float m = -CUDART_INF_F;
        for (int s = 0; s < P.S; ++s)
            m = fmaxf(m, __ldcg(P.parts + ((int64_t)s * c.H_q + gq) * (kHeadDim + 2) + kHeadDim));
        float l = 0.f, o = 0.f;
        for (int s = 0; s < P.S; ++s) {
            const float *ps = P.parts + ((int64_t)s * c.H_q + gq) * (kHeadDim + 2);
            const float ls = __ldcg(ps + kHeadDim + 1);
            if (ls == 0.f) continue;
            const float wgt = exp2f(__ldcg(ps + kHeadDim) - m);
            l += wgt * ls;
            if (ch < kHeadDim) o += wgt * __ldcg(ps + ch);
        }
        if (P.write_partial) {
            const float v = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
            P.out[gq * (kHeadDim + 2) + ch] = v;
        } else if (ch < kHeadDim) {
            P.out[gq * kHeadDim + ch] = o / l;
        }
    }
    if (tid == 0) P.tickets[hg] = 0;
}

__global__ void merge_kernel(const float *__restrict__ parts, int Pn, int H, int d, float *o) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= H * d) return;
    const int g = x / d, ch = x % d;
    float m = -CUDART_INF_F;
    for (int s = 0; s < Pn; ++s) m = fmaxf(m, parts[((int64_t)s * H + g) * (d + 2) + d]);
    float l = 0.f, acc = 0.f;
    for (int s = 0; s < Pn; ++s) {
        const float *ps = parts + ((int64_t)s * H + g) * (d + 2);
        if (ps[d + 1] == 0.f) continue;
        const float w = exp2f(ps[d] - m);
        l += w * ps[d + 1];
        acc += w * ps[ch];
    }
    o[x] = acc / l;
}

constexpr size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

template <int BITS, int HG>
size_t layout(const DevCache &c, Params &P) {
    using C = Cfg<BITS, HG>;
    const int HKV = HG / c.G;
    const size_t qwc = (size_t)HKV * 4 * BITS;
    size_t off = 0;
    P.so_kw = (unsigned)off; off = align128(off + 32 * qwc * 4);
    P.so_vw = (unsigned)off; off = align128(off + 32 * qwc * 4);
    P.so_vsz = (unsigned)off; off = align128(off + 256);
    P.so_kptr = (unsigned)off; off = align128(off + 192);
    P.so_vrec = (unsigned)off; off = align128(off + (size_t)32 * c.kv * 4);
    P.so_krec = (unsigned)off;
    const size_t limit = 227 * 1024;
    const size_t base = align128(C::fixed + 64);
    P.st_base = (unsigned)base;
    for (int stages = 3; stages >= 2; --stages) {
        for (int krec = 2048; krec >= 256; krec -= 256) {
            const size_t stb = align128(off + (size_t)krec * 4);
            const size_t total = base + stages * stb;
            if (total <= limit) {
                P.stages = stages;
                P.krec_cap = krec;
                P.st_bytes = (unsigned)stb;
                return total;
            }
        }
    }
    return 0;
}

template <int BITS, int HG, int G>
cudaError_t launch_t(const DevCache &c, Params &P, int grid, cudaStream_t s) {
    const size_t smem = layout<BITS, HG>(c, P);
    if (smem == 0) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(att_kernel<BITS, HG, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    att_kernel<BITS, HG, G><<<grid, ATT_THREADS, smem, s>>>(c, P);
    return cudaGetLastError();
}

template <int BITS, int HG>
cudaError_t launch_g(const DevCache &c, Params &P, int grid, cudaStream_t s) {
    switch (c.G) {
        case 1: return launch_t<BITS, HG, 1>(c, P, grid, s);
        case 2: if constexpr (HG >= 2) return launch_t<BITS, HG, 2>(c, P, grid, s); break;
        case 4: if constexpr (HG >= 4) return launch_t<BITS, HG, 4>(c, P, grid, s); break;
        case 8: if constexpr (HG >= 8) return launch_t<BITS, HG, 8>(c, P, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

template <int BITS>
cudaError_t launch_b(const DevCache &c, Params &P, int hg, int grid, cudaStream_t s) {
    switch (hg) {
        case 1: return launch_g<BITS, 1>(c, P, grid, s);
        case 2: if constexpr (BITS <= 3) return launch_g<BITS, 2>(c, P, grid, s); break;
        case 4: if constexpr (BITS <= 3) return launch_g<BITS, 4>(c, P, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

}  // namespace

int attend_heads_per_cta(int bits, int H_q, int G) {
    const int cap = bits == 4 ? 1 : 4;   // V tasks: HG * 128/CPL <= 16 warps
    for (int hg = cap; hg >= 1; hg >>= 1)
        if (H_q % hg == 0 && hg % G == 0) return hg;
    return 0;
}

size_t attend_smem_bytes(int bits, int hg) {
    switch (bits * 100 + hg) {
        case 201: return Cfg<2, 1>::fixed;
        case 202: return Cfg<2, 2>::fixed;
        case 204: return Cfg<2, 4>::fixed;
        case 301: return Cfg<3, 1>::fixed;
        case 302: return Cfg<3, 2>::fixed;
        case 304: return Cfg<3, 4>::fixed;
        case 401: return Cfg<4, 1>::fixed;
    }
    return 0;
}

int attend_auto_splits(const DevCache &c, int64_t T, int hg) {
    const int ntiles = (int)((T + 31) / 32);
    const int n_hg = c.H_q / hg;
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int S = (sms + n_hg - 1) / n_hg;
    if (S > ntiles) S = ntiles;
    if (S < 1) S = 1;
    return S;
}

cudaError_t launch_attend(const DevCache &c, const AttendArgs &a, int *splits_used, cudaStream_t s) {
    const int hg = attend_heads_per_cta(c.bits, c.H_q, c.G);
    if (hg == 0) return cudaErrorInvalidValue;
    const int ntiles = (int)((a.T + 31) / 32);
    int S = a.splits > 0 ? a.splits : attend_auto_splits(c, a.T, hg);
    if (S > ntiles) S = ntiles;
    if (S < 1) S = 1;
    Params P{};
    P.q = a.q; P.pos = a.pos; P.T = a.T; P.S = S; P.ntiles = ntiles;
    P.out = a.out; P.parts = a.parts; P.tickets = a.tickets; P.write_partial = a.write_partial;
    P.timers = a.timers;
    const int grid = (c.H_q / hg) * S;
    if (splits_used) *splits_used = S;
    switch (c.bits) {
        case 2: return launch_b<2>(c, P, hg, grid, s);
        case 3: return launch_b<3>(c, P, hg, grid, s);
        case 4: return launch_b<4>(c, P, hg, grid, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_merge(const float *parts, int Pn, int H, int d, float *o, cudaStream_t s) {
    const int n = H * d;
    merge_kernel<<<(n + 255) / 256, 256, 0, s>>>(parts, Pn, H, d, o);
    return cudaGetLastError();
}

}  // namespace kvq
