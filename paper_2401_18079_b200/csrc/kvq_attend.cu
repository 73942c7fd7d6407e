// kvq_attend.cu -- ATT: fused single-token decode attention over the compressed cache.
//
// One launch per attend:
//   grid  = n_head_groups x splits (head group fastest), 256 threads, 1 CTA / SM.
//   a1 QP  each CTA rotates its HG query heads with exact fp64 angles (R11, R12) and
//          folds 1/sqrt(d) * log2(e) into q~.
//   LUTs   K: per (query head g, RoPE pair i) a 2^{2b}-entry table of fp16 pairs
//          (A, B) with  A = q~_i K^_i(a) + q~_i' K^_i'(b),  B = q~_i' K^_i(a) - q~_i K^_i'(b)
//          for K^_c(a) = Chat_K[a] s_c + z_c -- the paper's per-channel LUT
//          taken one step further: the query and the per-channel affine are folded in, so
//          one lookup + 2 FMAs per RoPE pair yields  cos(n'th_i) A + sin(n'th_i) B, which
//          is exactly the pair's contribution to q~ . RoPE(K^_n, n').
//          V: the shared codebook, lane-private copies (conflict-free).
//   a2 KS  lane = token of a 32-token tile, warp w = RoPE pairs 8w..8w+7 for all heads;
//          fp32 accumulation of fp16 products (fma.rn.f32.f16).
//   a3     Key outliers of the tile add  (x - K^(code)) * dscore/dK  (same launch).
//   a4     exact online softmax in base 2 (running max, rescale on change).
//   a5 PV  lane = 32 channels, V^ = s_n Chat_V[code] + z_n folded as
//          sum_n (p_n s_n) Chat_V[code] + sum_n p_n z_n  (affine fold).
//   a6     Value outliers add p_n (v - V^(code)).
//   a7 MRG the last CTA of each head group merges the split partials (log-sum-exp).
#include "kvq_internal.cuh"

#include <math_constants.h>

namespace kvq {
namespace {

constexpr int ATT_THREADS = 256;
constexpr int ATT_WARPS = 8;

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

struct Params {
    const __half *q;
    int64_t pos, T;
    int S;               // splits
    int ntiles;
    float *out;
    float *parts;
    unsigned *tickets;
    int write_partial;
};

template <int BITS, int HG>
struct Smem {
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int HMAX = BITS == 4 ? 4 : 8;   // fp32 "heavy" pairs per head
    static constexpr size_t klut = (size_t)HG * kPairs * NE * 4;
    static constexpr size_t vlut = (size_t)NE * 32 * 4;
    static constexpr size_t hlut = (size_t)HG * HMAX * NE * 8;
    static constexpr size_t cis = (size_t)kPairs * 32 * 8;
    static constexpr size_t fixed =
        HG * kHeadDim * 4              /* qs */
        + ATT_WARPS * HG * 32 * 4      /* red */
        + HG * 32 * 4 * 2              /* p, kcorr */
        + HG * 32 * 2                  /* w16 */
        + HG * kHeadDim * 4            /* osp */
        + 64 * 16 + 64 * 8 + 64 * 16   /* anc64, anc32, rot64 */
        + 64 * 4                       /* theta32 */
        + 40 * 4 + 32 * 8              /* kptr slice, vsz slice */
        + HG * 4 * 8                   /* per-head scalars */
        + HG * 64 * 4 + HG * 64        /* bound, heavy flags */
        + HG * 16 * 4                  /* heavy pair list + counts */
        + 64;
    static constexpr size_t total = klut + vlut + hlut + cis + fixed + 128;
};

template <int BITS, int HG, int G>
__global__ void __launch_bounds__(ATT_THREADS, 1) att_kernel(DevCache c, Params P) {
    constexpr int NE = 1 << (2 * BITS);
    constexpr int CM = (1 << BITS) - 1;
    constexpr int HKV = HG / G;
    constexpr int NWW = (BITS == 2) ? 1 : 2;      // K words per (lane, kv head, warp)
    constexpr int LPT = 4 * HG;                     // V lanes per token
    constexpr int SLOTS = ATT_THREADS / LPT;        // tokens per V step
    constexpr int VSTEPS = (32 + SLOTS - 1) / SLOTS;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *sp = smem_raw;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += Smem<BITS, HG>::klut;
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += Smem<BITS, HG>::vlut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += Smem<BITS, HG>::hlut;
    float2 *cis_s = reinterpret_cast<float2 *>(sp); sp += Smem<BITS, HG>::cis;
    float *qs = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *red = reinterpret_cast<float *>(sp); sp += ATT_WARPS * HG * 32 * 4;
    float *p_s = reinterpret_cast<float *>(sp); sp += HG * 32 * 4;
    float *kcorr = reinterpret_cast<float *>(sp); sp += HG * 32 * 4;
    float *osp = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    double2 *anc64 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double2 *rot64 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    float2 *anc32 = reinterpret_cast<float2 *>(sp); sp += 64 * 8;
    float *theta32 = reinterpret_cast<float *>(sp); sp += 64 * 4;
    float2 *vsz_s = reinterpret_cast<float2 *>(sp); sp += 32 * 8;
    uint32_t *kptr_s = reinterpret_cast<uint32_t *>(sp); sp += 40 * 4;
    float *lut_inv = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *alpha_s = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *beta_s = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *m_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *l_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *z_fin = reinterpret_cast<float *>(sp); sp += HG * 4;
    uint16_t *w16 = reinterpret_cast<uint16_t *>(sp); sp += HG * 32 * 2;
    int *flag_s = reinterpret_cast<int *>(sp); sp += 16;
    float *bound_s = reinterpret_cast<float *>(sp); sp += HG * 64 * 4;
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(sp); sp += HG * 64;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    constexpr int HMAX = Smem<BITS, HG>::HMAX;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_hg = c.H_q / HG;
    const int hg = blockIdx.x % n_hg;
    const int split = blockIdx.x / n_hg;
    const int g0 = hg * HG;          // first query head
    const int h0 = g0 / G;           // first KV head
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int D = c.D;
    const float *ks = c.kpar, *kz = c.kpar + D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;   // decode codebooks

    // ---------------------------------------------------------------- prologue
    __shared__ double2 qcis[64];
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
    // K LUT: per (head, pair) bound of |A|,|B|.  The few pairs carrying a heavy Key
    // channel (bound > 1/4 of the head max, at most HMAX per head) get fp32 tables and
    // are accumulated exactly in fp32 (a3'); the rest use fp16 tables whose scale is set
    // by the largest remaining bound.
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
    if (warp < HG) {
        const float b0 = bound_s[warp * 64 + lane], b1 = bound_s[warp * 64 + 32 + lane];
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
        if ((m0 >> lane) & 1u) hv_pair[warp * 8 + __popc(m0 & lt)] = lane;
        if ((m1 >> lane) & 1u) hv_pair[warp * 8 + n0c + __popc(m1 & lt)] = lane + 32;
        heavy_s[warp * 64 + lane] = (m0 >> lane) & 1u;
        heavy_s[warp * 64 + 32 + lane] = (m1 >> lane) & 1u;
        const float rest = warp_max(fmaxf(((m0 >> lane) & 1u) ? 0.f : b0, ((m1 >> lane) & 1u) ? 0.f : b1));
        if (lane == 0) {
            hv_n[warp] = n0c + __popc(m1);
            // scale so that |entry| <= 2^14 (fp16 max 65504)
            int e = 0;
            if (rest > 0.f && isfinite(rest)) e = 14 - ilogbf(rest) - 1;
            e = max(-100, min(100, e));
            alpha_s[warp] = ldexpf(1.f, e);      // temp: LUT scale
            lut_inv[warp] = ldexpf(1.f, -e);
        }
    }
    __syncthreads();
    // K LUT entries
    for (int x = tid; x < HG * 64; x += ATT_THREADS) {
        const int g = x >> 6, i = x & 63;
        const int kvh = (g0 + g) / G;
        const int ci = kvh * kHeadDim + i, cj = ci + 64;
        const float sc = alpha_s[g];
        const float qa = qs[g * kHeadDim + i] * sc, qb = qs[g * kHeadDim + i + 64] * sc;
        float X[1 << BITS], Y[1 << BITS];
#pragma unroll
        for (int a = 0; a <= CM; ++a) {
            X[a] = cbK[a] * ks[ci] + kz[ci];
            Y[a] = cbK[a] * ks[cj] + kz[cj];
        }
        uint32_t *dst = klut + (size_t)(g * 64 + i) * NE;
        const bool heavy = heavy_s[x] != 0;
        int hslot = -1;
        if (heavy)
            for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
        const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
        for (int e0 = 0; e0 < NE; ++e0) {
            const int e = (e0 + lane) & (NE - 1);
            const int a = e & CM, bb = e >> BITS;
            float xa = 0.f, yb = 0.f;
#pragma unroll
            for (int u = 0; u <= CM; ++u) { xa = (u == a) ? X[u] : xa; yb = (u == bb) ? Y[u] : yb; }
            if (heavy) {
                dst[e] = 0u;
                hlut[(g * HMAX + hslot) * NE + e] = make_float2(qa1 * xa + qb1 * yb, qb1 * xa - qa1 * yb);
            } else {
                const float A = qa * xa + qb * yb;
                const float B = qb * xa - qa * yb;
                dst[e] = pack_half2(A, B);
            }
        }
    }
    // V LUT: lane-private copies (entry e for lane slot l at word e*32 + l)
    for (int x = tid; x < NE * 32; x += ATT_THREADS) {
        const int e = x >> 5;
        vlut[x] = pack_half2(cbV[e & CM], cbV[e >> BITS]);
    }

    // per-lane constants for the K phase: cis(j * theta_i) for this warp's 8 pairs
    float t1c[8], t1s[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = warp * 8 + k;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        float s, co;
        sincosf((float)((double)lane * th), &s, &co);
        t1c[k] = co;
        t1s[k] = s;
    }

    // V-phase mapping
    const int cg = tid % LPT, slot = tid / LPT;
    const int vh = cg >> 2, qq = cg & 3;             // local query head, quarter
    const int vkvh = (g0 + vh) / G;                  // global kv head for V
    const int vword0 = (vkvh * 4 + qq) * BITS;       // first word of the lane's 32 channels
    float acc[32];
#pragma unroll
    for (int x = 0; x < 32; ++x) acc[x] = 0.f;

    // running softmax state (S-phase warps: warp g <-> head g)
    float m_run = -CUDART_INF_F, l_run = 0.f, z_run = 0.f;
    int E_cur = -126;     // dense V accumulator units: 2^E_cur

    // K-phase word window
    const int kbit0 = 16 * BITS * warp;
    const int kq0 = kbit0 >> 5, kshift = kbit0 & 31;

    uint32_t kw[HKV][NWW], vw[VSTEPS][BITS];
    uint32_t kptr_next = 0;
    float2 vsz_next = make_float2(0.f, 0.f);

    auto load_tile = [&](int t, uint32_t (&kwo)[HKV][NWW], uint32_t (&vwo)[VSTEPS][BITS]) {
        const uint32_t *kb = c.kcodes + (int64_t)t * c.QW * 32;
#pragma unroll
        for (int h = 0; h < HKV; ++h)
#pragma unroll
            for (int x = 0; x < NWW; ++x)
                kwo[h][x] = __ldg(kb + ((h0 + h) * 4 * BITS + kq0 + x) * 32 + lane);
#pragma unroll
        for (int st = 0; st < VSTEPS; ++st) {
            const int j = slot + st * SLOTS;
            const int64_t n = (int64_t)t * 32 + (j < 32 ? j : 0);
            const uint32_t *vb = c.vcodes + n * c.VW + vword0;
#pragma unroll
            for (int x = 0; x < BITS; ++x) vwo[st][x] = (j < 32) ? __ldg(vb + x) : 0u;
        }
        if (tid < 33) {
            int64_t n = (int64_t)t * 32 + tid;
            if (n > P.T) n = P.T;
            kptr_next = __ldg(c.kptr + n);
        }
        if (tid >= 64 && tid < 96) {
            int64_t n = (int64_t)t * 32 + (tid - 64);
            vsz_next = n < P.T ? __ldg(c.vsz + n) : make_float2(0.f, 0.f);
        }
    };

    if (t_begin < t_end) load_tile(t_begin, kw, vw);
    __syncthreads();

    for (int t = t_begin; t < t_end; ++t) {
        const int64_t n0 = (int64_t)t * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        // publish this tile's small arrays, then prefetch the next tile
        if (tid < 33) kptr_s[tid] = kptr_next;
        if (tid >= 64 && tid < 96) vsz_s[tid - 64] = vsz_next;
        uint32_t kwn[HKV][NWW], vwn[VSTEPS][BITS];
        if (t + 1 < t_end) load_tile(t + 1, kwn, vwn);

        // ------------------------------------------------------------ a2: K dense
        {
            float acc_c[HG], acc_s[HG];
#pragma unroll
            for (int g = 0; g < HG; ++g) { acc_c[g] = 0.f; acc_s[g] = 0.f; }
            unsigned long long win[HKV];
#pragma unroll
            for (int h = 0; h < HKV; ++h) {
                unsigned long long w64 = kw[h][0];
                if (NWW == 2) w64 |= (unsigned long long)kw[h][NWW - 1] << 32;
                win[h] = w64 >> kshift;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = warp * 8 + k;
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

        // ----------------------------------------------------- a3: K outliers
        {
            const uint32_t r0 = kptr_s[0], r1 = kptr_s[ntok];
            for (uint32_t r = r0 + tid; r < r1; r += ATT_THREADS) {
                // token of record r: largest j with kptr_s[j] <= r
                int lo = 0, hi = ntok - 1;
                while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (kptr_s[mid] <= r) lo = mid; else hi = mid - 1; }
                const int j = lo;
                const uint32_t rec = __ldg(c.kout + r);
                const int ch = (int)(rec & 0xffffu);
                const int kvh = ch >> 7;
                if (kvh < h0 || kvh >= h0 + HKV) continue;
                const int cc = ch & 127, i = cc & 63, up = cc >> 6;
                const int bit = 2 * BITS * i;
                const uint32_t *kb = c.kcodes + (int64_t)t * c.QW * 32;
                const int wq = kvh * 4 * BITS + (bit >> 5);
                unsigned long long w64 = __ldg(kb + wq * 32 + j);
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)__ldg(kb + (wq + 1) * 32 + j) << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const int code = (pc >> (up * BITS)) & CM;
                const float xval = __half2float(__ushort_as_half((uint16_t)(rec >> 16)));
                const float delta = xval - (cbK[code] * ks[ch] + kz[ch]);
                const float2 cs = cis_s[i * 32 + j];
                const float co = cs.x, si = cs.y;
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    const int g = (kvh - h0) * G + gg;
                    const float qa = qs[g * kHeadDim + i], qb = qs[g * kHeadDim + i + 64];
                    const float d = up ? (qb * co - qa * si) : (qa * co + qb * si);
                    atomicAdd(&kcorr[g * 32 + j], delta * d);
                }
            }
            // a2': heavy RoPE pairs in fp32 (tables hlut; cis of the tile from the K phase)
            for (int x = tid; x < HG * 8 * 32; x += ATT_THREADS) {
                const int g = x >> 8, slot = (x >> 5) & 7, j = x & 31;
                if (slot >= hv_n[g] || j >= ntok) continue;
                const int i = hv_pair[g * 8 + slot];
                const int kvh = (g0 + g) / G;
                const int bit = 2 * BITS * i;
                const uint32_t *kb = c.kcodes + (int64_t)t * c.QW * 32;
                const int wq = kvh * 4 * BITS + (bit >> 5);
                unsigned long long w64 = __ldg(kb + wq * 32 + j);
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)__ldg(kb + (wq + 1) * 32 + j) << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const float2 ab = hlut[(g * HMAX + slot) * NE + pc];
                const float2 cs = cis_s[i * 32 + j];
                atomicAdd(&kcorr[g * 32 + j], cs.x * ab.x + cs.y * ab.y);
            }
        }
        __syncthreads();

        // ------------------------------------------------------- a4: softmax
        {
            // CTA-uniform V scale exponent from the tile's max s_n
            float smax = lane < ntok ? vsz_s[lane].x : 0.f;
            smax = warp_max(smax);
            int E_new = E_cur;
            if (smax > 0.f) E_new = max(E_cur, ilogbf(smax) + 1);
            if (warp < HG) {
                const int g = warp;
                float s = 0.f;
#pragma unroll
                for (int w = 0; w < ATT_WARPS; ++w) s += red[(w * HG + g) * 32 + lane];
                s = s * lut_inv[g] + kcorr[g * 32 + lane];
                kcorr[g * 32 + lane] = 0.f;
                const bool valid = lane < ntok;
                if (!valid) s = -CUDART_INF_F;
                const float mt = warp_max(s);
                const float m_new = fmaxf(m_run, mt);
                const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run - m_new);
                const float p = valid ? exp2f(s - m_new) : 0.f;
                const float2 sz = vsz_s[lane];
                l_run = l_run * alpha + warp_sum(p);
                z_run = z_run * alpha + warp_sum(p * sz.y);
                m_run = m_new;
                p_s[g * 32 + lane] = p;
                const float wv = p * ldexpf(sz.x, -E_new);
                w16[g * 32 + lane] = __half_as_ushort(__float2half_rn(wv));
                if (lane == 0) {
                    alpha_s[g] = alpha;
                    beta_s[g] = alpha * ldexpf(1.f, E_cur - E_new);
                    if (alpha != 1.f || E_new != E_cur) flag_s[0] = 1;
                }
            }
            E_cur = E_new;
        }
        __syncthreads();

        // -------------------------------------------------------- a5: P.V dense
        const bool rescale = flag_s[0] != 0;
        if (rescale) {
            const float b = beta_s[vh];
            if (b != 1.f) {
#pragma unroll
                for (int x = 0; x < 32; ++x) acc[x] *= b;
            }
            for (int x = tid; x < HG * kHeadDim; x += ATT_THREADS) osp[x] *= alpha_s[x >> 7];
        }
#pragma unroll
        for (int st = 0; st < VSTEPS; ++st) {
            const int j = slot + st * SLOTS;
            if (j < 32) {
                const uint16_t w = w16[vh * 32 + j];
#pragma unroll
                for (int pp = 0; pp < 16; ++pp) {
                    const int bit = 2 * BITS * pp;
                    uint32_t pc;
                    if (BITS == 2) {
                        pc = (vw[st][bit >> 5] >> (bit & 31)) & (NE - 1);
                    } else if (BITS == 4) {
                        pc = (vw[st][bit >> 5] >> (bit & 31)) & (NE - 1);
                    } else {  // 3 bits: 96-bit group, pairs straddle word boundaries
                        const int wi = bit >> 5, sh = bit & 31;
                        if (sh + 6 <= 32) pc = (vw[st][wi] >> sh) & 63u;
                        else pc = (uint32_t)((((unsigned long long)vw[st][wi + 1] << 32) | vw[st][wi]) >> sh) & 63u;
                    }
                    const uint32_t cv = vlut[pc * 32 + lane];
                    fma_w_f16x2(w, cv, acc[2 * pp], acc[2 * pp + 1]);
                }
            }
        }
        if (rescale) {
            __syncthreads();
            if (tid == 0) flag_s[0] = 0;
        }

        // ---------------------------------------------------- a6: V outliers
        {
            const int kv = c.kv;
            const int nrec = ntok * kv;
            const uint32_t *vo = c.vout + n0 * kv;
            for (int r = tid; r < nrec; r += ATT_THREADS) {
                const uint32_t rec = __ldg(vo + r);
                const int ch = (int)(rec & 0xffffu);
                const int kvh = ch >> 7;
                if (kvh < h0 || kvh >= h0 + HKV) continue;
                const int j = r / kv;
                const int bit = BITS * ch;
                const uint32_t *vrow = c.vcodes + (n0 + j) * c.VW;
                unsigned long long w64 = __ldg(vrow + (bit >> 5));
                if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)__ldg(vrow + (bit >> 5) + 1) << 32;
                const int code = (int)((w64 >> (bit & 31)) & CM);
                const float2 sz = vsz_s[j];
                const float xval = __half2float(__ushort_as_half((uint16_t)(rec >> 16)));
                const float delta = xval - (cbV[code] * sz.x + sz.y);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    const int g = (kvh - h0) * G + gg;
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
#pragma unroll
        for (int h = 0; h < HKV; ++h)
#pragma unroll
            for (int x = 0; x < NWW; ++x) kw[h][x] = kwn[h][x];
#pragma unroll
        for (int st = 0; st < VSTEPS; ++st)
#pragma unroll
            for (int x = 0; x < BITS; ++x) vw[st][x] = vwn[st][x];
        __syncthreads();
    }

    // ------------------------------------------------------------ write partial
    if (warp < HG && lane == 0) { m_fin[warp] = m_run; l_fin[warp] = l_run; z_fin[warp] = z_run; }
    {
        // dense P.V accumulators are in units of 2^-E_cur; threads whose slot had no
        // token (HG == 1) hold zeros.
        const float sc = ldexpf(1.f, E_cur);
        float *dst = osp + vh * kHeadDim + qq * 32;
#pragma unroll
        for (int x = 0; x < 32; ++x) atomicAdd(&dst[x], acc[x] * sc);
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
    __shared__ int s_last;
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.tickets[hg], 1u);
        s_last = (prev == (unsigned)(P.S - 1));
    }
    __syncthreads();
    if (!s_last) return;
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
            float v = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
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

template <int BITS, int HG, int G>
cudaError_t launch_t(const DevCache &c, const Params &P, int grid, cudaStream_t s) {
    const size_t smem = Smem<BITS, HG>::total;
    cudaError_t e = cudaFuncSetAttribute(att_kernel<BITS, HG, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    att_kernel<BITS, HG, G><<<grid, ATT_THREADS, smem, s>>>(c, P);
    return cudaGetLastError();
}

template <int BITS, int HG>
cudaError_t launch_g(const DevCache &c, const Params &P, int grid, cudaStream_t s) {
    switch (c.G) {
        case 1: return launch_t<BITS, HG, 1>(c, P, grid, s);
        case 2: if constexpr (HG >= 2) return launch_t<BITS, HG, 2>(c, P, grid, s); break;
        case 4: if constexpr (HG >= 4) return launch_t<BITS, HG, 4>(c, P, grid, s); break;
        case 8: if constexpr (HG >= 8) return launch_t<BITS, HG, 8>(c, P, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

template <int BITS>
cudaError_t launch_b(const DevCache &c, const Params &P, int hg, int grid, cudaStream_t s) {
    switch (hg) {
        case 1: return launch_g<BITS, 1>(c, P, grid, s);
        case 2: return launch_g<BITS, 2>(c, P, grid, s);
        case 4: if constexpr (BITS <= 3) return launch_g<BITS, 4>(c, P, grid, s); break;
        case 8: if constexpr (BITS <= 3) return launch_g<BITS, 8>(c, P, grid, s); break;
    }
    return cudaErrorInvalidValue;
}

}  // namespace

int attend_heads_per_cta(int bits, int H_q, int G) {
    const int cap = bits == 4 ? 2 : 8;
    for (int hg = cap; hg >= 1; hg >>= 1)
        if (H_q % hg == 0 && hg % G == 0) return hg;
    return 0;
}

size_t attend_smem_bytes(int bits, int hg) {
    switch (bits * 100 + hg) {
        case 201: return Smem<2, 1>::total;
        case 202: return Smem<2, 2>::total;
        case 204: return Smem<2, 4>::total;
        case 208: return Smem<2, 8>::total;
        case 301: return Smem<3, 1>::total;
        case 302: return Smem<3, 2>::total;
        case 304: return Smem<3, 4>::total;
        case 308: return Smem<3, 8>::total;
        case 401: return Smem<4, 1>::total;
        case 402: return Smem<4, 2>::total;
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
    Params P;
    P.q = a.q; P.pos = a.pos; P.T = a.T; P.S = S; P.ntiles = ntiles;
    P.out = a.out; P.parts = a.parts; P.tickets = a.tickets; P.write_partial = a.write_partial;
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
