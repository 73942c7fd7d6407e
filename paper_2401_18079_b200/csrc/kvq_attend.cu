// kvq_attend.cu -- ATT: fused single-token decode attention over the compressed cache.
//
// One launch per attend.  grid = n_head_groups x splits (head group
// fastest), one CTA per SM, each CTA a contiguous range of 32-token tiles of one group of
// HG query heads.  The CTA's 16 warps form four independent quads; quad q takes the tiles
// q, q+4, q+8, ... of the range, so four tiles are in flight and a quad only ever waits for
// its own four warps (one named barrier per tile):
//   load   at the top of a tile the quad's 128 threads cp.async (16 B each) its next tile --
//          K/V code words, per-token (s,z), outlier items of this head group -- into a
//          shared ring slot; completion arrives on the slot's mbarrier.
//   a2+a3  K: warp w of the quad takes RoPE pairs 16w..16w+15 of every head (lane = token):
//          pair-table lookups (fp16 x fp16 -> fp32), Key-outlier and heavy-pair terms in fp32
//          summed in fixed point with shared integer atomics.  -> quad barrier
//   a4     online softmax in base 2, warp w = head w (4 partial sums per token);
//   a5+a6  P.V on the tensor cores (mma.m16n8k16: A = Value codes through a pair table,
//          B = fp16 weights p s 2^-E, warp w = KV head w for MHA), Value-outlier terms in
//          fixed point folded into the accumulators.
//   a7     the quads' partials are merged, then the last CTA of each head group merges the
//          split partials (log-sum-exp, ticket counter).
//   Tables (built per CTA, a1): q~ = RoPE(q, pos) with exact fp64 angles (R11, R12) times
//   log2(e)/sqrt(d); per (query head g, RoPE pair i) a 2^{2b}-entry table of fp16 pairs
//   (A, B), A = q~_i K^_i(a) + q~_i' K^_i'(b), B = q~_i' K^_i(a) - q~_i K^_i'(b) with
//   K^_c(a) = Chat_K[a] s_c + z_c: the paper's per-channel LUT with the query
//   and the affine folded in, so one lookup + 2 FMAs give cos(n' th_i) A + sin(n' th_i) B,
//   exactly the pair's share of q~ . RoPE(K^_n, n') (RoPE after dequantization, P:379,
//   P:730).  Pairs carrying a heavy Key channel use fp32 tables.  V: the
//   shared codebook as a table of (Chat[a], Chat[b]) fp16 pairs, one copy per lane.
#include "kvq_internal.cuh"

#include <math_constants.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace kvq {
namespace {

constexpr int NQ = 4;                         // quads: independent 4-warp pipelines
constexpr int QWARPS = 4;                     // warps per quad
constexpr int QT = QWARPS * 32;               // threads per quad
constexpr int ATT_THREADS = NQ * QT;          // 16 warps: 4 per SM sub-partition
constexpr int KPW = kPairs / QWARPS;          // RoPE pairs per warp in the K phase (16)
constexpr int NANC = 3;                       // per-quad ring of tile anchors (written 2 ahead)

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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// 16-byte cp.async (LDGSTS, L2 only) and the mbarrier arrival fired by its completion
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
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

// d += A * B on the tensor cores: mma.m16n8k16, fp16 operands, fp32 accumulation
__device__ __forceinline__ void mma_f16_f32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
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
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Score terms summed with shared integer atomics (no native float atomics in shared memory):
// fixed point with 2^-16 resolution in log2-score units, |term| clamped to 2^15.
constexpr float kKfixScale = 65536.f;
__device__ __forceinline__ int kfix_of(float v) {
    return __float2int_rn(fminf(fmaxf(v, -32768.f), 32767.f) * kKfixScale);
}
// 2^k as a float for k in [-126, 127] (clamped); exact, no libm call
__device__ __forceinline__ float pow2i(int k) {
    k = max(-126, min(127, k));
    return __int_as_float((k + 127) << 23);
}
// floor(log2(x)) of a positive normal float (x = 0 or subnormal gives -127)
__device__ __forceinline__ int ilog2f(float x) { return ((__float_as_int(x) >> 23) & 255) - 127; }
// 32-bit shared-window load
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// warp max of floats with one REDUX via an order-preserving integer map
__device__ __forceinline__ float warp_max_redux(float v) {
    unsigned u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    u = __reduce_max_sync(0xffffffffu, u);
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(u);
}

// ---------------------------------------------------------------- configuration --

template <int BITS, int HG>
struct Cfg {
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int HMAX = 4;                   // fp32 "heavy" pairs per head
    static constexpr size_t klut = (size_t)HG * kPairs * NE * 4;
    static constexpr size_t vlut = (size_t)NE * 32 * 4;
    static constexpr size_t hlut = (size_t)HG * HMAX * NE * 8;
    static constexpr size_t t1 = (size_t)kPairs * 32 * 8;       // prologue only (in the ring)
    // per quad: red[2], kfix[2], p, w16, vfix, anchors[NANC], beta/m/l/z
    static constexpr size_t quad =
        2 * QWARPS * HG * 32 * 4 + 2 * HG * 32 * 4 + HG * 32 * 4 + HG * 32 * 2 + HG * kHeadDim * 4
        + NANC * 64 * 8 + HG * 4 * 4 + 64;
    static constexpr size_t small =
        HG * kHeadDim * 4              /* qs */
        + NQ * quad
        + 64 * 16                      /* rot128 */
        + 64 * 5 * 8                   /* cis(2^k theta_i) */
        + HG * 4 * 2                   /* lut scale / inverse */
        + HG * 24 * 4                  /* heavy pair list, counts, flat list */
        + HG * kHeadDim * 4 * 2 + 64 * 4 /* staged s_c, z_c of the group, codebooks */
        + 16 * 4 + 16 * 16             /* flags, slot headers */
        + 512;
    static constexpr size_t fixed = klut + vlut + hlut + small;
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
    // ring layout (bytes), computed on the host
    int spq, scap_k, scap_v;      // ring slots per quad; outlier items a slot holds (mult. of 4)
    unsigned st_base, st_bytes, so_kw, so_vw, so_vsz, so_kit, so_vit;
    unsigned long long *timers;   // optional diagnostics, may be null
};

template <int BITS, int HG, int G>
__global__ void __launch_bounds__(ATT_THREADS, 1) att_kernel(DevCache c, Params P) {
    using C = Cfg<BITS, HG>;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int HKV = HG / G;
    constexpr int QWC = HKV * 4 * BITS;             // K (and V) words per token in the CTA
    constexpr int HMAX = C::HMAX;
    constexpr int KWW = 2 * BITS * KPW / 32;        // K code words of a warp's pairs (per head)

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sp = smem_raw;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += C::klut;
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += C::hlut;
    float *qs = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    unsigned char *quad_base = sp; sp += NQ * C::quad;
    double2 *rot128 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;   // rotation by 128 theta
    float2 *cisp = reinterpret_cast<float2 *>(sp); sp += 64 * 5 * 8;   // cis(2^k theta_i) [i][k]
    float *lut_inv = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *lut_sc = reinterpret_cast<float *>(sp); sp += HG * 4;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_combo = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;   // flat (head, slot) list
    float *ks_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;   // s_c of the group
    float *kz_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;             // 4 codebooks
    int *flag_s = reinterpret_cast<int *>(sp); sp += 16 * 4;
    int *hdr_s = reinterpret_cast<int *>(sp); sp += 16 * 16;               // per ring slot
    // mbarriers just below the ring: full[slot] (the cp.async of a tile have landed)
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + P.st_base - 128);
    uint64_t *full_b = bars;   // [NQ * SPQ]
    // prologue-only scratch in the (not yet used) ring
    float2 *t1tab = reinterpret_cast<float2 *>(smem_raw + P.st_base);
    double2 *qcis = reinterpret_cast<double2 *>(smem_raw + P.st_base + C::t1);
    float *bound_s = reinterpret_cast<float *>(smem_raw + P.st_base + C::t1 + 64 * 16);
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(smem_raw + P.st_base + C::t1 + 64 * 16 + HG * 64 * 4);

    const long long t_kernel0 = clock64();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_hg = c.H_q / HG;
    const int hg = blockIdx.x % n_hg;
    const int split = blockIdx.x / n_hg;
    const int g0 = hg * HG;          // first query head
    const int h0 = g0 / G;           // first KV head
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int ntl = t_end - t_begin;
    const int D = c.D;
    const int kv = c.kv;
    const float *ks = c.kpar, *kz = c.kpar + D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;   // decode codebooks
    const int c_lo = h0 * kHeadDim, c_hi = (h0 + HKV) * kHeadDim;
    const int SPQ = P.spq;     // private ring slots per quad

    // quad scratch
    const int q = warp / QWARPS, w = warp % QWARPS, qtid = tid % QT;
    struct Quad {
        float *red;       // [2][QWARPS][HG][32] partial scores
        int *kfix;        // [2][HG][32] Key-outlier + heavy-pair terms, fixed point
        float *p_s;       // [HG][32]
        uint16_t *w16;    // [HG][32] fp16 weights p s 2^-E
        int *vfix;        // [HG][128] Value-outlier sums of the tile, fixed point
        float2 *anc;      // [NANC][64] tile anchors cis(n0 theta_i)
        float *beta, *m_fin, *l_fin, *z_fin;   // [HG]
    };
    auto quad_at = [&](int qq) -> Quad {
        Quad Q;
        unsigned char *p = quad_base + qq * C::quad;
        Q.red = reinterpret_cast<float *>(p); p += 2 * QWARPS * HG * 32 * 4;
        Q.kfix = reinterpret_cast<int *>(p); p += 2 * HG * 32 * 4;
        Q.p_s = reinterpret_cast<float *>(p); p += HG * 32 * 4;
        Q.vfix = reinterpret_cast<int *>(p); p += HG * kHeadDim * 4;
        Q.anc = reinterpret_cast<float2 *>(p); p += NANC * 64 * 8;
        Q.beta = reinterpret_cast<float *>(p); p += HG * 4;
        Q.m_fin = reinterpret_cast<float *>(p); p += HG * 4;
        Q.l_fin = reinterpret_cast<float *>(p); p += HG * 4;
        Q.z_fin = reinterpret_cast<float *>(p); p += HG * 4;
        Q.w16 = reinterpret_cast<uint16_t *>(p);
        return Q;
    };
    const Quad Q = quad_at(q);
    auto stage_ptr = [&](int st) -> unsigned char * { return smem_raw + P.st_base + (size_t)st * P.st_bytes; };

    if (tid == 0) {
        for (int s = 0; s < NQ * SPQ; ++s) mbar_init(full_b + s, 1);   // the expect_tx arrival
        mbar_fence_init();
    }

    // ---------------------------------------------------------------- prologue
    if (tid < 64) {
        const int i = tid;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        double s, co;
        sincos((double)P.pos * th, &s, &co);
        qcis[i] = make_double2(co, s);
        sincos((double)(NQ * kTileTokens) * th, &s, &co);
        rot128[i] = make_double2(co, s);
    }
    for (int x = tid; x < kPairs * 5; x += ATT_THREADS) {
        const int i = x / 5, k = x % 5;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        double s, co;
        sincos((double)(1 << k) * th, &s, &co);
        cisp[x] = make_float2((float)co, (float)s);
    }
    for (int x = tid; x < kPairs * 32; x += ATT_THREADS) {
        const int i = x >> 5, j = x & 31;
        const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
        double s, co;
        sincos((double)j * th, &s, &co);
        t1tab[x] = make_float2((float)co, (float)s);
    }
    for (int x = tid; x < NQ * HG * kHeadDim; x += ATT_THREADS) quad_at(x / (HG * kHeadDim)).vfix[x % (HG * kHeadDim)] = 0;
    for (int x = tid; x < NQ * 2 * HG * 32; x += ATT_THREADS) quad_at(x / (2 * HG * 32)).kfix[x % (2 * HG * 32)] = 0;
    for (int x = tid; x < HKV * kHeadDim; x += ATT_THREADS) {
        ks_s[x] = ks[c_lo + x];
        kz_s[x] = kz[c_lo + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
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
        const int ci = (g / G) * kHeadDim + i, cj = ci + 64;
        const float mx = fmaxf(fabsf(cbK[0] * ks_s[ci] + kz_s[ci]), fabsf(cbK[CM] * ks_s[ci] + kz_s[ci]));
        const float my = fmaxf(fabsf(cbK[0] * ks_s[cj] + kz_s[cj]), fabsf(cbK[CM] * ks_s[cj] + kz_s[cj]));
        const float qa = fabsf(qs[g * kHeadDim + i]), qb = fabsf(qs[g * kHeadDim + i + 64]);
        bound_s[x] = fmaxf(qa * mx + qb * my, qb * mx + qa * my);
    }
    __syncthreads();
    for (int g = warp; g < HG; g += ATT_THREADS / 32) {
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
            lut_sc[g] = ldexpf(1.f, e);
            lut_inv[g] = ldexpf(1.f, -e);
        }
    }
    __syncthreads();
    if (tid == 0) {   // flat (head, heavy slot) list for the K phase
        int nc = 0;
        for (int g = 0; g < HG; ++g)
            for (int h = 0; h < hv_n[g]; ++h) hv_combo[nc++] = g * 8 + h;
        flag_s[2] = nc;
    }
    // K table entries: one (head, pair, second code) row of 2^b entries per work item
    for (int x = tid; x < HG * 64 * (CM + 1); x += ATT_THREADS) {
        const int bb = x % (CM + 1), gi = x / (CM + 1);
        const int g = gi >> 6, i = gi & 63;
        const int ci = (g / G) * kHeadDim + i, cj = ci + 64;
        const float sc = lut_sc[g];
        const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
        const float qa = qa1 * sc, qb = qb1 * sc;
        const float yb = cbK[bb] * ks_s[cj] + kz_s[cj];
        uint32_t *dst = klut + (size_t)(g * 64 + i) * NE + (bb << BITS);
        const bool heavy = heavy_s[gi] != 0;
        int hslot = 0;
        if (heavy)
            for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
#pragma unroll
        for (int a = 0; a <= CM; ++a) {
            const float xa = cbK[a] * ks_s[ci] + kz_s[ci];
            if (heavy) {
                dst[a] = 0u;
                hlut[(g * HMAX + hslot) * NE + (bb << BITS) + a] =
                    make_float2(qa1 * xa + qb1 * yb, qb1 * xa - qa1 * yb);
            } else {
                dst[a] = pack_half2(qa * xa + qb * yb, qb * xa - qa * yb);
            }
        }
    }
    // V table: lane-private copies (entry e for lane slot l at word e*32 + l)
    for (int x = tid; x < NE * 32; x += ATT_THREADS) {
        const int e = x >> 5;
        vlut[x] = pack_half2(cbV[e & CM], cbV[e >> BITS]);
    }
    // per-lane constants of the K phase: cis(j theta_i) for this warp's KPW pairs
    float t1c[KPW], t1s[KPW];
#pragma unroll
    for (int k = 0; k < KPW; ++k) {
        const float2 v = t1tab[(w * KPW + k) * 32 + lane];
        t1c[k] = v.x;
        t1s[k] = v.y;
    }
    // anchors of each quad's first two tiles; the fp64 running anchor of the next one stays in
    // registers of the quad's warp 0 (pairs lane, lane + 32)
    double2 amaster[2];
    if (w == 0) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int i = lane + 32 * h2;
            const double th = pow(c.theta, -2.0 * (double)i / (double)kHeadDim);
            double s, co;
            for (int a = 0; a < 2; ++a) {
                const double a0 = (double)(c.pos_base + (int64_t)(t_begin + q + NQ * a) * kTileTokens) * th;
                sincos(a0, &s, &co);
                Q.anc[a * 64 + i] = make_float2((float)co, (float)s);
            }
            amaster[h2] = make_double2(co, s);
        }
    }
    __syncthreads();   // tables ready; the ring (t1tab) is free from here on
    const int n_combo = flag_s[2];
    const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
    unsigned long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    // ------------------------------------------------------- tile loads (cp.async)
    // Quad q handles the CTA's tiles it = q + 4i and owns SPQ private ring slots: tile i goes
    // to slot q*SPQ + i % SPQ, loaded with TMA bulk copies issued by the quad's warps,
    // completion counted on the slot's mbarrier (complete_tx).  (16-byte cp.async from 128
    // threads measured ~2000 cycles of issue per tile under the LDS load of the K phase.)  The
    // slot's previous tile (i - SPQ) is free once every warp of the quad is past the quad
    // barrier of tile i - SPQ + 1: tile i + 1 is loaded at the top of tile i when SPQ >= 3,
    // right after the barrier of tile i when SPQ == 2.  Outlier counts are read one load
    // ahead (registers).
    const int nqt = ntl > q ? (ntl - q + NQ - 1) / NQ : 0;   // tiles of this quad
    uint32_t nk_nx = 0, nv_nx = 0;     // counts of the quad's next tile to load
    auto read_counts = [&](int it, uint32_t &nk, uint32_t &nv) {
        nk = nv = 0;
        if (it < ntl) {
            const uint32_t *gc = c.gcnt + ((int64_t)(t_begin + it) * c.NG + hg) * 2;
            nk = __ldg(gc);
            nv = __ldg(gc + 1);
        }
    };
    auto load_tile = [&](int ii, uint32_t nk, uint32_t nv) {   // quad iteration ii
        if (ii >= nqt || lane != 0) return;
        const int si = q * SPQ + ii % SPQ;
        const int ti = t_begin + q + NQ * ii;
        const bool kov = nk > (uint32_t)P.scap_k, vov = nv > (uint32_t)P.scap_v;
        const uint32_t bk = kov ? 0u : ((nk + 3u) & ~3u) * 4u;
        const uint32_t bv = vov ? 0u : ((nv + 3u) & ~3u) * 4u;
        const unsigned b_kw = QWC * 32u * 4u;
        unsigned char *sb = stage_ptr(si);
        uint64_t *bar = full_b + si;
        const int64_t bucket = (int64_t)ti * c.NG + hg;
        // TMA bulk copies, one or two per warp of the quad (an issue holds its warp for
        // ~150 cycles); the expect_tx arrival (warp 0) publishes the header written before it
        if (w == 0) {
            int *hdr = hdr_s + si * 4;
            hdr[0] = kov ? 0 : (int)nk;
            hdr[1] = vov ? 0 : (int)nv;
            hdr[2] = kov;
            hdr[3] = vov;
            mbar_expect_tx(bar, 2u * b_kw + 256u + bk + bv);
            bulk_g2s(sb + P.so_kw, c.kcodes + ((int64_t)ti * c.QW + h0 * 4 * BITS) * 32, b_kw, bar);
        } else if (w == 1) {
            bulk_g2s(sb + P.so_vw, c.vcodes + ((int64_t)ti * c.H_kv + h0) * 32 * 4 * BITS, b_kw, bar);
        } else if (w == 2) {
            bulk_g2s(sb + P.so_vsz, c.vsz + (int64_t)ti * 32, 256u, bar);
            if (bk) bulk_g2s(sb + P.so_kit, c.kit + bucket * c.kcap_g, bk, bar);
        } else {
            if (bv) bulk_g2s(sb + P.so_vit, c.vit + bucket * c.vcap_g, bv, bar);
        }
    };
    if (nqt > 0) {
        uint32_t nk0, nv0;
        read_counts(q, nk0, nv0);
        read_counts(q + NQ, nk_nx, nv_nx);
        load_tile(0, nk0, nv0);
    }
    auto load_next = [&](int i) {   // tile i + 1 of the quad
        const uint32_t nk = nk_nx, nv = nv_nx;
        read_counts(q + NQ * (i + 2), nk_nx, nv_nx);
        load_tile(i + 1, nk, nv);
    };

    // V-phase mapping inside the quad (tensor cores, mma.m16n8k16): warp -> (local KV head
    // vkv, m-tiles [mt0, mt0 + MTW) of 16 channels); A = V codes (rows = channels, k = tokens)
    // through the pair table, B = fp16 weights (columns = the G query heads of vkv),
    // D = fp32 P.V accumulators (columns >= G unused).
    constexpr int WPK = QWARPS / HKV;           // warps per KV head
    constexpr int MTW = 8 / WPK;                // m-tiles per warp
    constexpr int FB = 2 * BITS;                // bits per A field (2 tokens x 1 channel)
    constexpr int NWV = (MTW * 16 * BITS + 31) / 32;   // code words per lane per tile
    constexpr bool SELF = (WPK == 1 && G == 1);        // warp w: softmax head w == V head w
    static_assert(HKV <= QWARPS && QWARPS % HKV == 0 && G <= 8, "V task mapping");
    const int vkv = w / WPK;
    const int mt0 = (w % WPK) * MTW;
    const int vbit0 = mt0 * 16 * BITS;
    const int vw0 = vbit0 >> 5, voff = vbit0 & 31;           // voff = 16 only for b=3, MTW=1
    const int vg = lane >> 2, vt = lane & 3;
    const int vq_lo = vkv * G + min(2 * vt, G - 1), vq_hi = vkv * G + min(2 * vt + 1, G - 1);
    const uint32_t vlut_base = smem_u32(vlut), vlane4 = 4u * lane;
    // this warp's K tables: base | (pair code << 2), + a constant per (head, pair)
    const uint32_t klut_w = smem_u32(klut) + (uint32_t)(w * KPW * NE * 4);
    if (klut_w & (NE * 4u - 1u)) __trap();
    float dacc[MTW][4];
#pragma unroll
    for (int x = 0; x < MTW; ++x) dacc[x][0] = dacc[x][1] = dacc[x][2] = dacc[x][3] = 0.f;
    float m_run = -CUDART_INF_F, l_lane = 0.f, z_lane = 0.f;   // softmax head w (w < HG)
    int E_cur = -126;      // dense V accumulator units: 2^E (uniform in the quad)
    long long tc0 = clock64(), tc1;
    tm[0] = tc0 - t_kernel0;

    for (int i = 0; i < nqt; ++i) {
        const int it = q + NQ * i;
        const int b = i & 1;
        const int st = q * SPQ + i % SPQ;
        if (SPQ >= 3) load_next(i);
        tc1 = clock64(); tm[5] += tc1 - tc0; tc0 = tc1;
        mbar_wait(full_b + st, (unsigned)((i / SPQ) & 1));
        tc1 = clock64(); tm[1] += tc1 - tc0; tc0 = tc1;
        unsigned char *sb = stage_ptr(st);
        const uint32_t *kw_s = reinterpret_cast<const uint32_t *>(sb + P.so_kw);
        const uint32_t *vw_s = reinterpret_cast<const uint32_t *>(sb + P.so_vw);
        const float2 *vsz_s = reinterpret_cast<const float2 *>(sb + P.so_vsz);
        const uint32_t *kit = reinterpret_cast<const uint32_t *>(sb + P.so_kit);
        const uint32_t *vit = reinterpret_cast<const uint32_t *>(sb + P.so_vit);
        const int *hdr = hdr_s + st * 4;
        const int64_t n0 = (int64_t)(t_begin + it) * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        const float2 *an32 = Q.anc + (i % NANC) * 64;
        int *kf = Q.kfix + b * HG * 32;

        // cis((n0 + j) theta_i) = anchor_i * cis(j theta_i), the second factor as a product of
        // the binary powers cis(2^k theta_i) (fp32 table) -- for items and heavy pairs
        auto cis_tok = [&](int ii, int j) -> float2 {
            float2 r = an32[ii];
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if ((j >> k) & 1) {
                    const float2 p = cisp[ii * 5 + k];
                    r = make_float2(r.x * p.x - r.y * p.y, r.x * p.y + r.y * p.x);
                }
            return r;
        };
        // K-outlier correction of one item: (x - K^(code)) * dscore/dK for query head
        // kvl*G + gg, in fp32
        auto k_corr = [&](uint32_t itm, int gg, int &j_out, int &g_out) -> float {
            const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x7ffu);
            const int kvl = chl >> 7, cc = chl & 127, ii = cc & 63, up = cc >> 6;
            const int bit = 2 * BITS * ii;
            const int wq = kvl * 4 * BITS + (bit >> 5);
            unsigned long long w64 = kw_s[wq * 32 + j];
            if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + j] << 32;
            const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
            const int code = (pc >> (up * BITS)) & CM;
            const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
            const float delta = xval - (cbKs[code] * ks_s[chl] + kz_s[chl]);
            const float2 cs = cis_tok(ii, j);
            const int g = kvl * G + gg;
            const float qa = qs[g * kHeadDim + ii], qb = qs[g * kHeadDim + ii + 64];
            j_out = j;
            g_out = g;
            return delta * (up ? (qb * cs.x - qa * cs.y) : (qa * cs.x + qb * cs.y));
        };

        // ------------------------------------------ a3: K outliers, heavy pairs
        {
            const int nk = hdr[0];
            for (int x = qtid; x < nk; x += QT) {
                const uint32_t itm = kit[x];
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    int j, g;
                    const float v = k_corr(itm, gg, j, g);
                    atomicAdd(&kf[g * 32 + j], kfix_of(v));
                }
            }
            if (hdr[2]) {
                // overflowed bucket: this tile's Key outliers from the CSC arrays (rare)
                for (int j = 0; j < ntok; ++j) {
                    const uint32_t r0 = __ldg(c.kptr + n0 + j), r1 = __ldg(c.kptr + n0 + j + 1);
                    for (uint32_t r = r0 + qtid; r < r1; r += QT) {
                        const uint32_t rec = __ldcg(c.kout + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < c_lo || ch >= c_hi) continue;
                        const uint32_t itm = (rec & 0xffff0000u) | ((uint32_t)j << 11) | (uint32_t)(ch - c_lo);
#pragma unroll
                        for (int gg = 0; gg < G; ++gg) {
                            int jj, g;
                            const float v = k_corr(itm, gg, jj, g);
                            atomicAdd(&kf[g * 32 + jj], kfix_of(v));
                        }
                    }
                }
            }
            // heavy RoPE pairs in fp32 (tables hlut): the (head, pair) list spread over the
            // quad's warps, lane = token
            for (int cb = w; cb < n_combo; cb += QWARPS) {
                const int g = hv_combo[cb] >> 3, hsl = hv_combo[cb] & 7;
                const int ii = hv_pair[g * 8 + hsl];
                const int bit = 2 * BITS * ii;
                const int wq = (g / G) * 4 * BITS + (bit >> 5);
                unsigned long long w64 = kw_s[wq * 32 + lane];
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + lane] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const float2 ab = hlut[(g * HMAX + hsl) * NE + pc];
                const float2 cs = cis_tok(ii, lane);
                atomicAdd(&kf[g * 32 + lane], kfix_of(cs.x * ab.x + cs.y * ab.y));
            }
        }
        // ------------------------------------------------------------ a2: K dense
        {
            float acc_c[HG], acc_s[HG];
#pragma unroll
            for (int g = 0; g < HG; ++g) { acc_c[g] = 0.f; acc_s[g] = 0.f; }
#pragma unroll
            for (int h = 0; h < HKV; ++h) {
                uint32_t wd[KWW];
#pragma unroll
                for (int x = 0; x < KWW; ++x) wd[x] = kw_s[(h * 4 * BITS + w * KWW + x) * 32 + lane];
#pragma unroll
                for (int k = 0; k < KPW; ++k) {
                    const float2 an = an32[w * KPW + k];
                    const float cc = an.x * t1c[k] - an.y * t1s[k];
                    const float ss = an.x * t1s[k] + an.y * t1c[k];
                    const uint32_t cs = pack_half2(cc, ss);
                    const int bsh = 2 * BITS * k - 2;   // bit of (pair code << 2) in the words
                    uint32_t off;
                    if (bsh < 0) off = wd[0] << 2;
                    else if ((bsh & 31) + 2 * BITS + 2 <= 32) off = wd[bsh >> 5] >> (bsh & 31);
                    else off = __funnelshift_r(wd[bsh >> 5], wd[(bsh >> 5) + 1], bsh & 31);
                    const uint32_t a = klut_w | (off & ((NE - 1) << 2));
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int g = h * G + gg;
                        const uint32_t ab = lds_u32(a + (uint32_t)((g * 64 + k) * NE * 4));
                        fma2_f16_f32(ab, cs, acc_c[g], acc_s[g]);
                    }
                }
            }
            float *rd = Q.red + (b * QWARPS + w) * HG * 32;
#pragma unroll
            for (int g = 0; g < HG; ++g) rd[g * 32 + lane] = acc_c[g] + acc_s[g];
        }
        tc1 = clock64(); tm[2] += tc1 - tc0; tc0 = tc1;
        bar_sync(1 + q, QT);   // the quad's scores of tile it are complete
        tc1 = clock64(); tm[3] += tc1 - tc0; tc0 = tc1;
        if (SPQ == 2) load_next(i);
        // anchors of the quad's tile two ahead (slot free: every warp is past K(i))
        if (w == 0 && i + 2 < nqt) {
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int ii = lane + 32 * h2;
                const double2 a = amaster[h2], r = rot128[ii];
                amaster[h2] = make_double2(a.x * r.x - a.y * r.y, a.x * r.y + a.y * r.x);
                Q.anc[((i + 2) % NANC) * 64 + ii] = make_float2((float)amaster[h2].x, (float)amaster[h2].y);
            }
        }

        // ------------------------------------------------------- a4: online softmax
        float smax = lane < ntok ? vsz_s[lane].x : 0.f;
        smax = warp_max_redux(smax);
        int E_new = E_cur;
        if (smax > 0.f) E_new = max(E_cur, ilog2f(smax) + 1);
        const float pe = pow2i(-E_new);
        float beta_w = 1.f;
        if (w < HG) {
            const int g = w, j = lane;
            const bool valid = j < ntok;
            const float *rd = Q.red + b * QWARPS * HG * 32;
            float s = 0.f;
#pragma unroll
            for (int x = 0; x < QWARPS; ++x) s += rd[(x * HG + g) * 32 + j];
            s = s * lut_inv[g] + (float)kf[g * 32 + j] * (1.f / kKfixScale);
            kf[g * 32 + j] = 0;
            s = valid ? s : -CUDART_INF_F;
            const float m_new = fmaxf(m_run, warp_max_redux(s));
            const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run - m_new);
            const float p = valid ? exp2f(s - m_new) : 0.f;
            const float2 sz = valid ? vsz_s[j] : make_float2(0.f, 0.f);
            l_lane = l_lane * alpha + p;
            z_lane = z_lane * alpha + p * sz.y;
            m_run = m_new;
            Q.p_s[g * 32 + j] = p;
            Q.w16[g * 32 + j] = __half_as_ushort(__float2half_rn(p * (sz.x * pe)));
            beta_w = alpha * pow2i(E_cur - E_new);
            if (!SELF && lane == 0) Q.beta[g] = beta_w;
        }
        const int E_prev = E_cur;
        E_cur = E_new;
        if (SELF) __syncwarp();
        else bar_sync(1 + q, QT);   // weights of other warps' heads

        // -------------------------------------------------------- a5: P.V dense
        {
            const float b_lo = SELF ? beta_w : Q.beta[vq_lo], b_hi = SELF ? beta_w : Q.beta[vq_hi];
            if (b_lo != 1.f || b_hi != 1.f) {
#pragma unroll
                for (int x = 0; x < MTW; ++x) {
                    dacc[x][0] *= b_lo; dacc[x][1] *= b_hi;
                    dacc[x][2] *= b_lo; dacc[x][3] *= b_hi;
                }
            }
            uint32_t vr[NWV + 1];
#pragma unroll
            for (int x = 0; x < NWV; ++x) vr[x] = vw_s[(vkv * 4 * BITS + vw0 + x) * 32 + lane];
            vr[NWV] = 0u;
            if (BITS == 3 && MTW == 1 && voff) { vr[0] = __funnelshift_r(vr[0], vr[1], 16); vr[1] >>= 16; }
            // B fragments (weights of query head vkv*G + g for tokens 16s + 2t.. / +8..)
            uint32_t bw[2][2];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const uint32_t *w32 = reinterpret_cast<const uint32_t *>(Q.w16 + (vkv * G + (vg < G ? vg : 0)) * 32 + 16 * s2 + 2 * vt);
                bw[s2][0] = vg < G ? w32[0] : 0u;
                bw[s2][1] = vg < G ? w32[4] : 0u;
            }
#pragma unroll
            for (int ml = 0; ml < MTW; ++ml) {
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    uint32_t a[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int bit = ((ml * 2 + s2) * 4 + r) * FB;
                        const int wi = bit >> 5, sh = bit & 31;
                        uint32_t off;
                        if (sh + FB <= 32) off = sh >= 7 ? (vr[wi] >> (sh - 7)) : (vr[wi] << (7 - sh));
                        else off = __funnelshift_r(vr[wi], vr[wi + 1], sh - 7);
                        a[r] = lds_u32(vlut_base + (vlane4 | (off & ((NE - 1) << 7))));
                    }
                    mma_f16_f32(dacc[ml], a, bw[s2]);
                }
            }
        }
        // ---------------------------------------------------- a6: V outliers
        {
            // this warp's items (its KV head, its m-tiles): sum_n p_n delta_{n,c} in fixed
            // point with |p delta| 2^(24-e) < 2^25, 2^e <= max|delta| < 2^(e+1), then folded
            // into the accumulators (units 2^-E)
            const int nvi = hdr[1];
            auto v_delta = [&](int j, int chl, uint16_t xbits) -> float {
                const int kvl = chl >> 7, cc = chl & 127;
                const int bit = vf_bit(j, cc, BITS);
                const uint32_t *vwp = vw_s + (kvl * 4 * BITS + (bit >> 5)) * 32 + vf_lane(j, cc);
                unsigned long long w64 = vwp[0];
                if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)vwp[32] << 32;
                const int code = (int)((w64 >> (bit & 31)) & CM);
                const float2 sz = vsz_s[j];
                return __half2float(__ushort_as_half(xbits)) - (cbVs[code] * sz.x + sz.y);
            };
            auto mine = [&](int chl) { return (chl >> 7) == vkv && (((chl & 127) >> 4) - mt0) >= 0 && (((chl & 127) >> 4) - mt0) < MTW; };
            float mx = 0.f;
            for (int x = lane; x < nvi; x += 32) {
                const uint32_t itm = vit[x];
                const int chl = (int)(itm & 0x7ffu);
                if (mine(chl)) mx = fmaxf(mx, fabsf(v_delta((int)((itm >> 11) & 31u), chl, (uint16_t)(itm >> 16))));
            }
            if (hdr[3]) {
                for (int r = lane; r < ntok * kv; r += 32) {
                    const uint32_t rec = __ldcg(c.vout + n0 * kv + r);
                    const int ch = (int)(rec & 0xffffu);
                    if (ch < c_lo || ch >= c_hi || !mine(ch - c_lo)) continue;
                    mx = fmaxf(mx, fabsf(v_delta(r / kv, ch - c_lo, (uint16_t)(rec >> 16))));
                }
            }
            mx = warp_max_redux(mx);
            if (mx > 0.f) {
                const int emx = ilog2f(mx);
                const float S = pow2i(24 - emx);
                int *vf = Q.vfix;
                for (int x = lane; x < nvi; x += 32) {
                    const uint32_t itm = vit[x];
                    const int chl = (int)(itm & 0x7ffu);
                    if (!mine(chl)) continue;
                    const int j = (int)((itm >> 11) & 31u), cc = chl & 127;
                    const float dS = v_delta(j, chl, (uint16_t)(itm >> 16)) * S;
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int g = vkv * G + gg;
                        atomicAdd(&vf[g * kHeadDim + cc], __float2int_rn(Q.p_s[g * 32 + j] * dS));
                    }
                }
                if (hdr[3]) {
                    for (int r = lane; r < ntok * kv; r += 32) {
                        const uint32_t rec = __ldcg(c.vout + n0 * kv + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < c_lo || ch >= c_hi || !mine(ch - c_lo)) continue;
                        const int j = r / kv, chl = ch - c_lo, cc = chl & 127;
                        const float dS = v_delta(j, chl, (uint16_t)(rec >> 16)) * S;
#pragma unroll
                        for (int gg = 0; gg < G; ++gg) {
                            const int g = vkv * G + gg;
                            atomicAdd(&vf[g * kHeadDim + cc], __float2int_rn(Q.p_s[g * 32 + j] * dS));
                        }
                    }
                }
                __syncwarp();
                // fold into the accumulators of the owner lanes (units 2^-E_cur) and clear
                const float unit = pow2i(emx - 24) * pow2i(-E_cur);
#pragma unroll
                for (int ml = 0; ml < MTW; ++ml) {
                    const int ch = (mt0 + ml) * 16 + vg;
#pragma unroll
                    for (int cl = 0; cl < 2; ++cl) {
                        if (2 * vt + cl < G) {
                            int *pv = vf + (vkv * G + 2 * vt + cl) * kHeadDim + ch;
                            dacc[ml][cl] += (float)pv[0] * unit;
                            dacc[ml][2 + cl] += (float)pv[8] * unit;
                            pv[0] = 0;
                            pv[8] = 0;
                        }
                    }
                }
            }
            (void)E_prev;
        }
        tc1 = clock64(); tm[4] += tc1 - tc0; tc0 = tc1;
    }
    // accumulators -> per-quad results (the ring is free once every quad is done)
    __syncthreads();
    float *osp = reinterpret_cast<float *>(smem_raw + P.st_base) + q * HG * kHeadDim;   // [NQ][HG][128]
    {
        const float sc = pow2i(E_cur);
#pragma unroll
        for (int ml = 0; ml < MTW; ++ml) {
            const int ch = (mt0 + ml) * 16 + vg;
#pragma unroll
            for (int cl = 0; cl < 2; ++cl) {
                if (2 * vt + cl < G) {
                    float *o = osp + (vkv * G + 2 * vt + cl) * kHeadDim + ch;
                    o[0] = dacc[ml][cl] * sc;
                    o[8] = dacc[ml][2 + cl] * sc;
                }
            }
        }
    }
    if (w < HG) {
        const float l = warp_sum(l_lane), z = warp_sum(z_lane);
        if (lane == 0) { Q.m_fin[w] = m_run; Q.l_fin[w] = l; Q.z_fin[w] = z; }
    }
    if (P.timers && qtid == 0) {
#pragma unroll
        for (int x = 0; x < 5; ++x) atomicAdd(P.timers + x, tm[x]);
        atomicAdd(P.timers + 5, (unsigned long long)nqt);
        atomicAdd(P.timers + 6, tm[5]);
    }
    __syncthreads();

    // ------------------------------------------------------ write partial (merge quads)
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    for (int x = tid; x < HG * (kHeadDim + 2); x += ATT_THREADS) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int qq = 0; qq < NQ; ++qq) {
            const Quad Qq = quad_at(qq);
            if (ntl > qq && Qq.l_fin[g] != 0.f) m = fmaxf(m, Qq.m_fin[g]);
        }
        float l = 0.f, o = 0.f;
        for (int qq = 0; qq < NQ; ++qq) {
            const Quad Qq = quad_at(qq);
            if (ntl <= qq || Qq.l_fin[g] == 0.f) continue;
            const float wq = exp2f(Qq.m_fin[g] - m);
            l += wq * Qq.l_fin[g];
            if (ch < kHeadDim) {
                const float *oq = reinterpret_cast<const float *>(smem_raw + P.st_base) + qq * HG * kHeadDim;
                o += wq * (oq[g * kHeadDim + ch] + Qq.z_fin[g]);
            }
        }
        part[(g0 + g) * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
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
    // outlier items a ring slot holds: ~2x the expected count (the bucket capacity is ~3x);
    // a tile with more uses the CSC / CSR fallback
    P.scap_k = (int)std::min<int64_t>(c.kcap_g, std::max<int64_t>(128, ((int64_t)c.kcap_g * 2 / 3 + 3) & ~3LL));
    P.scap_v = (int)std::min<int64_t>(c.vcap_g, std::max<int64_t>(128, ((int64_t)c.vcap_g * 2 / 3 + 3) & ~3LL));
    size_t off = 0;
    P.so_kw = (unsigned)off; off += 32 * qwc * 4;
    P.so_vw = (unsigned)off; off += 32 * qwc * 4;
    P.so_vsz = (unsigned)off; off += 256;
    P.so_kit = (unsigned)off; off += (size_t)P.scap_k * 4;
    P.so_vit = (unsigned)off; off += (size_t)P.scap_v * 4;
    const size_t stb = align128(off);
    const size_t base = align128(align128(C::fixed) + 128);   // + mbarriers
    P.st_base = (unsigned)base;
    const size_t limit = 227 * 1024;
    // 2..3 private slots per quad; the ring also holds the prologue's scratch and the final
    // per-quad results
    const size_t need = std::max<size_t>(C::t1 + 64 * 16 + HG * 64 * 5, (size_t)NQ * HG * kHeadDim * 4);
    for (int spq = 3; spq >= 2; --spq) {
        const size_t ring = std::max(NQ * spq * stb, need);
        if (base + ring <= limit) {
            P.spq = spq;
            P.st_bytes = (unsigned)stb;
            return base + ring;
        }
    }
    return 0;
}

template <int BITS, int HG, int G>
cudaError_t launch_t(const DevCache &c, Params &P, int grid, cudaStream_t s) {
    const size_t smem = layout<BITS, HG>(c, P);
    if (smem == 0) return cudaErrorInvalidConfiguration;
    static bool dbg = getenv("KVQ_DEBUG_LAYOUT") != nullptr;
    if (dbg) fprintf(stderr, "att_kernel<%d,%d,%d>: smem %zu fixed %zu slots/quad %d slot %u scap %d/%d\n",
                     BITS, HG, G, smem, Cfg<BITS, HG>::fixed, P.spq, P.st_bytes, P.scap_k, P.scap_v);
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
    // shared memory: K tables HG * 64 * 4^b * 4 bytes + 4 quads x 2-3 private ring slots
    const int cap = bits == 4 ? 1 : (G >= 4 ? 4 : 2);
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
    // one wave: every CTA needs a whole SM (launch_bounds(.., 1), ~200 KB smem)
    int S = sms / n_hg;
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
