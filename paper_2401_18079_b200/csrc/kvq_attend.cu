// kvq_attend.cu -- ATT: fused single-token decode attention over the compressed cache.
//
// One launch per attend.  grid = n_head_groups x splits (head group
// fastest), one CTA per SM, warp specialized:
//   warp 16 (producer)  TMA bulk copies (cp.async.bulk + mbarrier complete_tx) of every
//                       32-token tile of the CTA's head group -- K code words, V code words,
//                       per-token (s,z), CSC pointers, Value and Key outlier records -- into a
//                       STAGES-deep shared-memory ring; then compacts the tile's Key-outlier
//                       records of this head group into a self-contained item list.
//   warp 17 (producer)  compacts the tile's Value-outlier records of this head group.
//   warps 0..15         compute, synchronized among themselves with a named barrier:
//     a2+a3  K phase: RoPE-pair table lookups (lane = token, warp = 4 RoPE pairs, all
//            heads of the group; fp16 x fp16 -> fp32 FMAs), Key-outlier and heavy-pair
//            corrections in fp32 (flat over the item list, shared atomics);
//     a4     online softmax in base 2 (warp g = head g; per-lane deferred sums);
//     a5+a6  P.V: lane = CPL channels, sum_n (p_n s_n) Chat_V[code] + sum_n p_n z_n
//            (affine fold), Value-outlier corrections flat over the item list;
//     a7     the last CTA of each head group merges the split partials (log-sum-exp).
//   Tables (built per CTA, a1): q~ = RoPE(q, pos) with exact fp64 angles (R11, R12) times
//   log2(e)/sqrt(d); per (query head g, RoPE pair i) a 2^{2b}-entry table of fp16 pairs
//   (A, B), A = q~_i K^_i(a) + q~_i' K^_i'(b), B = q~_i' K^_i(a) - q~_i K^_i'(b) with
//   K^_c(a) = Chat_K[a] s_c + z_c: the paper's per-channel LUT with the query
//   and the affine folded in, so one lookup + 2 FMAs give cos(n' th_i) A + sin(n' th_i) B,
//   exactly the pair's share of q~ . RoPE(K^_n, n') (RoPE after dequantization, P:379,
//   P:730).  Pairs carrying a heavy Key channel use fp32 tables.  V: the
//   shared codebook as a pair table, one private copy per lane (conflict free).
#include "kvq_internal.cuh"

#include <math_constants.h>
#include <cstdlib>
#include <type_traits>

namespace kvq {
namespace {

constexpr int NHALF = 2;                      // independent compute halves (alternate tiles)
constexpr int HW = 8;                         // warps per half
constexpr int HT = HW * 32;                   // threads per half
constexpr int NCW = NHALF * HW;               // compute warps
constexpr int NCT = NCW * 32;                 // compute threads
constexpr int ATT_THREADS = NCT;              // 16 warps: 4 per SM sub-partition
constexpr int KPW = kPairs / HW;              // RoPE pairs per warp in the K phase

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
// named barrier among the warps of one compute half (ids 1, 2; the producer never joins)
__device__ __forceinline__ void half_sync(int half) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "n"(HT) : "memory");
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
// Score terms summed with shared 64-bit integer atomics (no native float atomics in shared
// memory): fixed point with 2^-16 resolution in log2-score units.  The 47 integer bits hold
// any sum of terms of finite fp16 data (|x q~| < 65504^2 * log2(e)/sqrt(d) < 2^30), so no
// clamp is needed and no sum can wrap.
constexpr float kKfixScale = 65536.f;
constexpr int WEXP = 14;   // fp16 P.V weights scaled into [0, 2^14]
__device__ __forceinline__ unsigned long long kfix_of(float v) {
    return (unsigned long long)__float2ll_rn(v * kKfixScale);
}
__device__ __forceinline__ float kfix_val(unsigned long long v) {
    return (float)(long long)v * (1.f / kKfixScale);
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

// G consecutive 32-bit shared words (G = 2 or 4) in one vector load
template <int G>
__device__ __forceinline__ void lds_vec(uint32_t addr, uint32_t (&v)[G]) {
    if constexpr (G == 2) {
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
    } else {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    }
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
    static constexpr int HMAX = BITS == 4 ? 4 : 8;   // fp32 "heavy" pairs per head
    static constexpr size_t klut = (size_t)HG * kPairs * NE * 4;
    static constexpr size_t vlut = (size_t)2 * NE * 32 * 4;   // hi and lo halves
    static constexpr size_t hlut = (size_t)HG * HMAX * NE * 8;
    static constexpr size_t t1 = (size_t)kPairs * 32 * 8;
    // per compute half: red, p, kcorr, hcorr, kbeg/kend, w16, osp, anchors, scalars
    static constexpr size_t half_bytes =
        HW * HG * 32 * 4 + HG * 32 * 4 * 3 + HG * 64 * 4 + HG * 32 * 4 + HG * kHeadDim * 4 * 2
        + 64 * 16 + 64 * 8 + 64 * 4 + HG * 4 * 4 + 16 + 64;
    static constexpr size_t small =
        HG * kHeadDim * 4              /* qs */
        + NHALF * half_bytes
        + 64 * 16 * 2                  /* rot64, qcis */
        + 64 * 4                       /* theta32 */
        + HG * 4 * 8                   /* per-head scalars */
        + HG * 64 * 4 + HG * 64        /* bound, heavy flags */
        + HG * 24 * 4                  /* heavy pair list, counts, flat list */
        + HG * kHeadDim * 4 * 2 + 64 * 4 /* staged s_c, z_c of the group, codebooks */
        + 8 * 16                       /* slot headers */
        + 256;
    static constexpr size_t fixed = klut + vlut + hlut + t1 + small;
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
    unsigned st_base, st_bytes, so_kw, so_vw, so_vsz, so_kit, so_vit, so_hdr, so_vdel;
    unsigned long long *timers;   // optional [8] phase cycle sums (diagnostics), may be null
};

template <int BITS, int HG, int G, bool TIMED>
__global__ void __launch_bounds__(ATT_THREADS, 1) att_kernel(DevCache c, Params P) {
    using C = Cfg<BITS, HG>;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int HKV = HG / G;
    constexpr int QWC = HKV * 4 * BITS;             // K (and V) words per token in the CTA
    constexpr int HMAX = C::HMAX;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sp = smem_raw;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += C::klut;
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += C::hlut;
    float2 *t1tab = reinterpret_cast<float2 *>(sp); sp += C::t1;   // cis(j theta_i) [i][j]
    float *qs = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    // per compute half h (alternate tiles): scratch of its own tile, at sp + h*half_bytes
    struct Half {
        float *red, *p_s, *osp, *beta_s, *m_fin, *l_fin, *z_fin;
        unsigned long long *kfix;   // [HG][32] Key-outlier + heavy-pair score terms, fixed point
        int *vfix;              // [HG][128] Value-outlier sums of the tile, fixed point
        int *vmax;              // [0] max |delta| of the tile's Value items (float bits)
        float *vscale;          // [0] fixed-point scale of the tile's V items
        float *vdel;            // [vcap_g] delta of each Value item of the tile
        uint16_t *w16;
        double2 *anc64;
        float2 *anc32;
        __half2 *anc16;         // fp16 copy of the anchors for the K dense phase
    };
    unsigned char *const half_base = sp;
    auto half_at = [&](int h) -> Half {
        Half H;
        unsigned char *q = half_base + h * C::half_bytes;
        H.red = reinterpret_cast<float *>(q); q += HW * HG * 32 * 4;
        H.p_s = reinterpret_cast<float *>(q); q += HG * 32 * 4;
        H.kfix = reinterpret_cast<unsigned long long *>(q); q += HG * 32 * 8;
        q += HG * 64 * 4;
        H.w16 = reinterpret_cast<uint16_t *>(q); q += HG * 32 * 4;   // hi [HG][32], then lo
        H.osp = reinterpret_cast<float *>(q); q += HG * kHeadDim * 4;
        H.vfix = reinterpret_cast<int *>(q); q += HG * kHeadDim * 4;
        q += (16 - ((HG * 32 * 2) % 16)) % 16;
        H.anc64 = reinterpret_cast<double2 *>(q); q += 64 * 16;
        H.anc32 = reinterpret_cast<float2 *>(q); q += 64 * 8;
        H.anc16 = reinterpret_cast<__half2 *>(q); q += 64 * 4;
        H.beta_s = reinterpret_cast<float *>(q); q += HG * 4;
        H.m_fin = reinterpret_cast<float *>(q); q += HG * 4;
        H.l_fin = reinterpret_cast<float *>(q); q += HG * 4;
        H.z_fin = reinterpret_cast<float *>(q); q += HG * 4;
        H.vmax = reinterpret_cast<int *>(q); q += 4;
        H.vscale = reinterpret_cast<float *>(q); q += 4;
        H.vdel = reinterpret_cast<float *>(smem_raw + P.so_vdel) + h * c.vcap_g;
        return H;
    };
    sp += NHALF * C::half_bytes;
    double2 *rot64 = reinterpret_cast<double2 *>(sp); sp += 64 * 16;   // rotation by 64 theta
    double2 *qcis = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    float *theta32 = reinterpret_cast<float *>(sp); sp += 64 * 4;
    float *lut_inv = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *lut_sc = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *bound_s = reinterpret_cast<float *>(sp); sp += HG * 64 * 4;
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(sp); sp += HG * 64;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_combo = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;   // flat (head, slot) list
    float *ks_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;   // s_c of the group
    float *kz_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;             // 4 codebooks
    int *flag_s = reinterpret_cast<int *>(sp); sp += 16;
    int *hdr_s = reinterpret_cast<int *>(sp); sp += 8 * 16;                // per ring slot
    // barriers just below the stage ring: full[S], empty[S]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + P.st_base - 128);
    uint64_t *full_b = bars;

    const long long t_kernel0 = clock64();
    const unsigned long long ns_kernel0 = TIMED ? gtimer_ns() : 0ull;
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

    auto stage_ptr = [&](int st) -> unsigned char * { return smem_raw + P.st_base + (size_t)st * P.st_bytes; };

    if (tid == 0) {
        for (int s = 0; s < P.stages; ++s) {
            mbar_init(full_b + s, 1);
        }
        mbar_fence_init();
    }

    // ---------------------------------------------------------------- prologue
    if (tid < 64) {
        const int i = tid;
        const double th = c.theta_tab[i];
        theta32[i] = (float)th;
        double s, co;
        sincos((double)P.pos * th, &s, &co);
        qcis[i] = make_double2(co, s);
        for (int h = 0; h < NHALF; ++h) {   // half h starts at tile t_begin + h
            const double a0 = (double)(c.pos_base + (int64_t)(t_begin + h) * kTileTokens) * th;
            sincos(a0, &s, &co);
            half_at(h).anc64[i] = make_double2(co, s);
            half_at(h).anc32[i] = make_float2((float)co, (float)s);
            half_at(h).anc16[i] = __floats2half2_rn((float)co, (float)s);
        }
        sincos((double)(NHALF * kTileTokens) * th, &s, &co);
        rot64[i] = make_double2(co, s);
    }
    for (int x = tid; x < kPairs * 32; x += ATT_THREADS) {
        const int i = x >> 5, j = x & 31;
        const double th = c.theta_tab[i];
        double s, co;
        sincos((double)j * th, &s, &co);
        t1tab[x] = make_float2((float)co, (float)s);
    }
    for (int x = tid; x < NHALF * HG * kHeadDim; x += ATT_THREADS) {
        const Half Hx = half_at(x / (HG * kHeadDim));
        Hx.osp[x % (HG * kHeadDim)] = 0.f;
        Hx.vfix[x % (HG * kHeadDim)] = 0;
    }
    if (tid < NHALF) { half_at(tid).vmax[0] = 0; half_at(tid).vscale[0] = 1.f; }
    for (int x = tid; x < HKV * kHeadDim; x += ATT_THREADS) {
        ks_s[x] = ks[c_lo + x];
        kz_s[x] = kz[c_lo + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
    for (int x = tid; x < NHALF * HG * 32; x += ATT_THREADS) half_at(x / (HG * 32)).kfix[x % (HG * 32)] = 0;
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
    // channel (bound > 1/2 of the head max, at most HMAX per head) get fp32 tables and
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
        float tau = 0.5f * M;
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
        // MHA: [g][i][pc]; GQA: the G query heads of a KV head interleaved per code,
        // [h][i][pc][G], so one vector load serves all G heads in the K phase
        uint32_t *dst = G == 1 ? klut + (size_t)(g * 64 + i) * NE + (bb << BITS)
                               : klut + ((size_t)((g / G) * 64 + i) * NE + (bb << BITS)) * G + (g % G);
        const bool heavy = heavy_s[gi] != 0;
        int hslot = 0;
        if (heavy)
            for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
#pragma unroll
        for (int a = 0; a <= CM; ++a) {
            const float xa = cbK[a] * ks_s[ci] + kz_s[ci];
            if (heavy) {
                dst[a * G] = 0u;
                hlut[(g * HMAX + hslot) * NE + (bb << BITS) + a] =
                    make_float2(qa1 * xa + qb1 * yb, qb1 * xa - qa1 * yb);
            } else {
                dst[a * G] = pack_half2(qa * xa + qb * yb, qb * xa - qa * yb);
            }
        }
    }
    // V table: lane-private copies (entry e for lane slot l at word e*32 + l), the fp16
    // codebook pair and, NE*32 words further, the fp16 residuals Chat - fp16(Chat): a diffuse
    // head averages ~10^4 tokens and the per-level fp16 rounding of Chat does not average out
    for (int x = tid; x < NE * 32; x += ATT_THREADS) {
        const int e = x >> 5;
        const float ca = cbV[e & CM], cb = cbV[e >> BITS];
        vlut[x] = pack_half2(ca, cb);
        vlut[NE * 32 + x] = pack_half2(ca - __half2float(__float2half_rn(ca)), cb - __half2float(__float2half_rn(cb)));
    }
    __syncthreads();

    // ====================================================== TMA issue (per half)
    // Each half owns SH = stages/2 ring slots and issues its own tiles: tiles of half h are
    // t_k = t_begin + h + 2k, slot k % SH.  The last warp of the half issues tile t_{k+SH-1}
    // at the top of iteration k, into the slot its half released at the end of k-1.
    // The five copies of a tile are issued by five different warps (HW-5..HW-1; a bulk copy
    // holds its warp ~150+ cycles), each from lane 0, with the tile's outlier counts read one
    // issue ahead (a global load on the issue path stalls the warp ~1 us).
    uint32_t cnt_nk = 0, cnt_nv = 0;
    auto read_counts = [&](int hh, int k) {
        const int ti = t_begin + hh + NHALF * k;
        cnt_nk = cnt_nv = 0;
        if (ti < t_end) {
            const uint32_t *gc = c.gcnt + ((int64_t)ti * c.NG + hg) * 2;
            cnt_nk = __ldg(gc);
            cnt_nv = __ldg(gc + 1);
        }
    };
    auto issue = [&](int hh, int k, int part) {   // lane 0 of issuing warp `part` (0..4)
        const int SH = P.stages / NHALF;
        const int ti = t_begin + hh + NHALF * k;
        if (ti >= t_end) return;
        const uint32_t nk = cnt_nk, nv = cnt_nv;
        read_counts(hh, k + 1);
        const int si = hh * SH + (SH == 2 ? (k & 1) : (k % SH));
        unsigned char *sb = stage_ptr(si);
        uint64_t *bar = full_b + si;
        const bool kov = nk > (uint32_t)c.kcap_g, vov = nv > (uint32_t)c.vcap_g;
        const uint32_t bk = kov ? 0u : ((nk + 3u) & ~3u) * 4u;
        const uint32_t bv = vov ? 0u : ((nv + 3u) & ~3u) * 4u;
        const unsigned b_kw = 32u * QWC * 4u;
        const int64_t bucket = (int64_t)ti * c.NG + hg;
        switch (part) {
            case 0: {
                // header in a generic-only array (no proxy fence); published by the
                // expect_tx arrival, read after the full-barrier wait (complete_tx of the
                // other parts may land first: the phase needs this arrival)
                int *hdr = hdr_s + si * 4;
                hdr[0] = kov ? 0 : (int)nk;
                hdr[1] = vov ? 0 : (int)nv;
                hdr[2] = kov;
                hdr[3] = vov;
                mbar_expect_tx(bar, 2u * b_kw + 256u + bk + bv);
                bulk_g2s(sb + P.so_kw, c.kcodes + ((int64_t)ti * c.QW + h0 * 4 * BITS) * 32, b_kw, bar);
                break;
            }
            case 1: bulk_g2s(sb + P.so_vw, c.vcodes + ((int64_t)ti * c.H_kv + h0) * 32 * 4 * BITS, b_kw, bar); break;
            case 2: bulk_g2s(sb + P.so_vsz, c.vsz + (int64_t)ti * 32, 256u, bar); break;
            case 3: if (bk) bulk_g2s(sb + P.so_kit, c.kit + bucket * c.kcap_g, bk, bar); break;
            default: if (bv) bulk_g2s(sb + P.so_vit, c.vit + bucket * c.vcap_g, bv, bar); break;
        }
    };

    // =========================================================== compute warps
    // Two independent halves of 8 warps process alternate tiles with their own scratch,
    // softmax state and named barrier; they share the read-only tables and hide each
    // other's latency.  Their partials are merged at the end.
    const int half = warp / HW, hw = warp % HW, htid = tid % HT;
    const int n_combo = flag_s[2];
    const Half H = half_at(half < NHALF ? half : 0);
    // V-phase task mapping inside a half (tensor cores, mma.m16n8k16): warp -> (local KV
    // head vkv, m-tiles [mt0, mt0 + MTW) of 16 channels); A = V codes (rows = channels,
    // k = tokens) through the pair table, B = fp16 weights (columns = the G query heads of
    // vkv), D = fp32 P.V accumulators (columns >= G unused).
    constexpr int WPK = HW / HKV;               // warps per KV head
    constexpr int MTW = 8 / WPK;                // m-tiles per warp
    constexpr int FB = 2 * BITS;                // bits per A field (2 tokens x 1 channel)
    constexpr int NWV = (MTW * 16 * BITS + 31) / 32;   // code words per lane per tile
    static_assert(HKV <= HW && HW % HKV == 0 && G <= 4, "V task mapping; hi/lo weight columns 2G <= 8");
    const int vkv = hw / WPK;                                // local KV head
    const int mt0 = (hw % WPK) * MTW;
    const int vbit0 = mt0 * 16 * BITS;
    const int vw0 = vbit0 >> 5, voff = vbit0 & 31;           // voff = 16 only for b=3, MTW=1
    const int vg = lane >> 2, vt = lane & 3;
    // D columns 2t, 2t+1 of lane (g, t): head t's hi and lo weight sums
    const int vq_lo = vkv * G + min(vt, G - 1), vq_hi = vq_lo;
    float dacc[MTW][4];
#pragma unroll
    for (int x = 0; x < MTW; ++x) dacc[x][0] = dacc[x][1] = dacc[x][2] = dacc[x][3] = 0.f;
    // lookup address = vlut + ((code << 7) | (lane << 2)): the OR is exact, the base add
    // folds into the load (uniform base register)
    const uint32_t vlane4 = 4u * lane;
    // lookups as byte offsets from the dynamic shared memory base: the table's offset (C::klut)
    // is a compile-time constant that folds into the LDS immediate
    const unsigned char *vlut_b = smem_raw + C::klut;
    float m_run = -CUDART_INF_F, l_lane = 0.f, z_lane = 0.f;
    int E_cur = -126;     // dense V accumulator units: 2^E_cur (uniform in a half)
    unsigned long long tm[6] = {0, 0, 0, 0, 0, 0};

    if (warp < NCW) {
        // per-lane constants for the K phase: cis(j * theta_i) for this warp's KPW pairs
        // as fp16 pairs t = (cos, sin) and t' = (-sin, cos): the tile rotation is then one
        // HMUL2 + one HFMA2 per pair: (a.x t + a.y t') = (a.x cos - a.y sin, a.x sin + a.y cos)
        // (fp32; the tile rotation anchor x cis(j th_i) is formed in fp32 and rounded once to
        // fp16)
        float2 t1v[KPW];
#pragma unroll
        for (int k = 0; k < KPW; ++k) t1v[k] = t1tab[(hw * KPW + k) * 32 + lane];
        // this warp's K tables: base | (pair code << 2), + a constant per (head, pair); the
        // base is a multiple of NE*4 bytes (dynamic shared memory is 1 KB aligned)
        const uint32_t klut_w = smem_u32(klut) + (uint32_t)(hw * KPW * NE * 4 * G);
        if (klut_w & (NE * 4u * G - 1u)) __trap();
        const int kbit0 = 2 * BITS * KPW * hw;
        const int kq0 = kbit0 >> 5, kshift = kbit0 & 31;
        const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
        long long tc0 = clock64(), tc1;
        tm[0] = tc0 - t_kernel0;   // prologue

        const int SH = P.stages / NHALF;
        const int ipart = hw - (HW - 5);   // issuing warps HW-5..HW-1 of the half
        if (ipart >= 0 && lane == 0) {
            read_counts(half, 0);
            for (int k = 0; k < SH - 1; ++k) issue(half, k, ipart);
        }
        int kk = 0, slot = 0, nv_prev = 0;
        unsigned par = 0;
        for (int t = t_begin + half; t < t_end; t += NHALF, ++kk) {
            const int st = half * SH + slot;
            if (ipart >= 0 && lane == 0) issue(half, kk + SH - 1, ipart);
            mbar_wait(full_b + st, par);
            if (++slot == SH) { slot = 0; par ^= 1u; }
            if (TIMED) { tc1 = clock64(); tm[1] += tc1 - tc0; tc0 = tc1; }
            unsigned char *sb = stage_ptr(st);
            const uint32_t *kw_s = reinterpret_cast<const uint32_t *>(sb + P.so_kw);
            const uint32_t *vw_s = reinterpret_cast<const uint32_t *>(sb + P.so_vw);
            const float2 *vsz_s = reinterpret_cast<const float2 *>(sb + P.so_vsz);
            const uint32_t *kit = reinterpret_cast<const uint32_t *>(sb + P.so_kit);
            const uint32_t *vit = reinterpret_cast<const uint32_t *>(sb + P.so_vit);
            const int *hdr = hdr_s + st * 4;
            const int64_t n0 = (int64_t)t * 32;
            const int ntok = (int)min((int64_t)32, P.T - n0);
            const float2 *anc32 = H.anc32;

            // K-outlier correction of one item: (x - K^(code)) * dscore/dK for query head
            // kvl*G + gg, in fp32
            auto k_corr = [&](uint32_t itm, int gg, int &j_out, int &g_out) -> float {
                const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x1ffu);
                const int kvl = chl >> 7, cc = chl & 127, i = cc & 63, up = cc >> 6;
                const int bit = 2 * BITS * i;
                const int wq = kvl * 4 * BITS + (bit >> 5);
                unsigned long long w64 = kw_s[wq * 32 + j];
                if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + j] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const int code = (pc >> (up * BITS)) & CM;
                const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                const float delta = xval - (cbKs[code] * ks_s[chl] + kz_s[chl]);
                const float2 an = anc32[i], tt = t1tab[i * 32 + j];
                const float co = an.x * tt.x - an.y * tt.y, si = an.x * tt.y + an.y * tt.x;
                const int g = kvl * G + gg;
                const float qa = qs[g * kHeadDim + i], qb = qs[g * kHeadDim + i + 64];
                j_out = j;
                g_out = g;
                return delta * (up ? (qb * co - qa * si) : (qa * co + qb * si));
            };

            // ------------------------------------------ a3: K outliers, heavy pairs
            {
                const int nk = hdr[0];
                // Key-outlier corrections straight into the (head, token) score term, in fixed
                // point (native shared integer atomics; see kfix_of)
                // items interleaved over the warps (item x -> warp x % HW) so every warp of the
                // half carries the same share and reaches the K barrier together
                const int ix = lane * HW + hw;
                for (int x = ix; x < nk; x += HT) {
                    const uint32_t itm = kit[x];
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        int j, g;
                        const float v = k_corr(itm, gg, j, g);
                        atomicAdd(&H.kfix[g * 32 + j], kfix_of(v));
                    }
                }
                // Value-outlier sums of this half's previous tile (fixed point) -> osp
                if (nv_prev) {
                    const float inv = H.vscale[0];
                    for (int x = htid; x < HG * kHeadDim; x += HT) {
                        const int v = H.vfix[x];
                        if (v) { H.osp[x] += (float)v * inv; H.vfix[x] = 0; }
                    }
                }
                if (htid == 0) H.vmax[0] = 0;
                nv_prev = hdr[1] | hdr[3];
                if (hdr[2]) {
                    // overflowed bucket: this tile's Key outliers from the CSC arrays (rare)
                    for (int j = 0; j < ntok; ++j) {
                        const uint32_t r0 = __ldg(c.kptr + n0 + j), r1 = __ldg(c.kptr + n0 + j + 1);
                        for (uint32_t r = r0 + htid; r < r1; r += HT) {
                            const uint32_t rec = __ldcg(c.kout + r);
                            const int ch = (int)(rec & 0xffffu);
                            if (ch < c_lo || ch >= c_hi) continue;
                            const uint32_t itm = (rec & 0xffff0000u) | ((uint32_t)j << 11) | (uint32_t)(ch - c_lo);
#pragma unroll
                            for (int gg = 0; gg < G; ++gg) {
                                int jj, g;
                                const float v = k_corr(itm, gg, jj, g);
                                atomicAdd(&H.kfix[g * 32 + jj], kfix_of(v));
                            }
                        }
                    }
                }
                // heavy RoPE pairs in fp32 (tables hlut): the (head, pair) list spread over the
                // half's warps, lane = token
                for (int cb = hw; cb < n_combo; cb += HW) {
                    const int g = hv_combo[cb] >> 3, hsl = hv_combo[cb] & 7;
                    const int i = hv_pair[g * 8 + hsl];
                    const int bit = 2 * BITS * i;
                    const int wq = (g / G) * 4 * BITS + (bit >> 5);
                    unsigned long long w64 = kw_s[wq * 32 + lane];
                    if ((bit & 31) + 2 * BITS > 32) w64 |= (unsigned long long)kw_s[(wq + 1) * 32 + lane] << 32;
                    const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                    const float2 ab = hlut[(g * HMAX + hsl) * NE + pc];
                    const float2 an = anc32[i], tt = t1tab[i * 32 + lane];
                    const float hc = (an.x * tt.x - an.y * tt.y) * ab.x + (an.x * tt.y + an.y * tt.x) * ab.y;
                    atomicAdd(&H.kfix[g * 32 + lane], kfix_of(hc));
                }
            }
            // ------------------------------------------------------------ a2: K dense
            {
                float acc_c[HG], acc_s[HG];
#pragma unroll
                for (int g = 0; g < HG; ++g) { acc_c[g] = 0.f; acc_s[g] = 0.f; }
                uint32_t wl[HKV], wh[HKV];
#pragma unroll
                for (int h = 0; h < HKV; ++h) {
                    unsigned long long w64 = kw_s[(h * 4 * BITS + kq0) * 32 + lane];
                    if (kshift + 2 * BITS * KPW > 32)
                        w64 |= (unsigned long long)kw_s[(h * 4 * BITS + kq0 + 1) * 32 + lane] << 32;
                    w64 >>= kshift;
                    wl[h] = (uint32_t)w64;
                    wh[h] = (uint32_t)(w64 >> 32);
                }
#pragma unroll
                for (int k = 0; k < KPW; ++k) {
                    const int i = hw * KPW + k;
                    const float2 an = H.anc32[i];
                    const __half2 csh = __floats2half2_rn(an.x * t1v[k].x - an.y * t1v[k].y, an.x * t1v[k].y + an.y * t1v[k].x);
                    const uint32_t cs = *reinterpret_cast<const uint32_t *>(&csh);
                    const int b = 2 * BITS * k - 2;   // bit of (pair code << 2) in the window
#pragma unroll
                    for (int h = 0; h < HKV; ++h) {
                        uint32_t off;
                        if (b < 0) off = wl[h] << 2;
                        else if (b + 2 * BITS + 2 <= 32) off = wl[h] >> b;
                        else if (b >= 32) off = wh[h] >> (b - 32);
                        else off = __funnelshift_r(wl[h], wh[h], b);
                        if constexpr (G == 1) {
                            const uint32_t a = klut_w | (off & ((NE - 1) << 2));
                            const uint32_t ab = lds_u32(a + (uint32_t)((h * 64 + k) * NE * 4));
                            fma2_f16_f32(ab, cs, acc_c[h], acc_s[h]);
                        } else {
                            // entries of the G heads are adjacent: (code << 2) << log2(G)
                            constexpr int LG = G == 2 ? 1 : 2;
                            const uint32_t a = klut_w | ((off << LG) & ((NE - 1) << (2 + LG)));
                            uint32_t ab[G];
                            lds_vec<G>(a + (uint32_t)((h * 64 + k) * NE * 4 * G), ab);
#pragma unroll
                            for (int gg = 0; gg < G; ++gg) fma2_f16_f32(ab[gg], cs, acc_c[h * G + gg], acc_s[h * G + gg]);
                        }
                    }
                }
#pragma unroll
                for (int g = 0; g < HG; ++g) H.red[(hw * HG + g) * 32 + lane] = acc_c[g] + acc_s[g];
            }
            half_sync(half);
            if (TIMED) { tc1 = clock64(); tm[2] += tc1 - tc0; tc0 = tc1; }

            // ------------------------------------------------------- a4: online softmax
            {
                float smax = lane < ntok ? vsz_s[lane].x : 0.f;
                smax = warp_max_redux(smax);
                int E_new = E_cur;
                if (smax > 0.f) E_new = max(E_cur, ilog2f(smax) + 1);
                // weights p s 2^(WEXP - E) <= 2^WEXP: normal fp16 down to p s 2^-E ~ 2^-28, so
                // the many small weights of a long context keep 11 significant bits
                const float pe = pow2i(WEXP - E_new);
                if (hw < HG) {
                    const int g = hw, j = lane;
                    const bool valid = j < ntok;
                    float s = 0.f;
#pragma unroll
                    for (int w = 0; w < HW; ++w) s += H.red[(w * HG + g) * 32 + j];
                    s = s * lut_inv[g] + kfix_val(H.kfix[g * 32 + j]);
                    H.kfix[g * 32 + j] = 0;
                    s = valid ? s : -CUDART_INF_F;
                    const float m_new = fmaxf(m_run, warp_max_redux(s));
                    const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run - m_new);
                    const float p = valid ? exp2f(s - m_new) : 0.f;
                    const float2 sz = valid ? vsz_s[j] : make_float2(0.f, 0.f);
                    l_lane = l_lane * alpha + p;
                    z_lane = z_lane * alpha + p * sz.y;
                    m_run = m_new;
                    H.p_s[g * 32 + j] = p;
                    {   // weight as fp16 hi + lo
                        const float wf = p * (sz.x * pe);
                        const __half wh = __float2half_rn(wf);
                        H.w16[g * 32 + j] = __half_as_ushort(wh);
                        H.w16[HG * 32 + g * 32 + j] = __half_as_ushort(__float2half_rn(wf - __half2float(wh)));
                    }
                    if (alpha != 1.f) {
#pragma unroll
                        for (int x = 0; x < kHeadDim / 32; ++x) H.osp[g * kHeadDim + x * 32 + lane] *= alpha;
                    }
                    if (lane == 0) H.beta_s[g] = alpha * pow2i(E_cur - E_new);
                } else {
                    // meanwhile the other warps compute the Value-outlier deltas
                    // x - (Chat_V[code] s_n + z_n) of the tile's items and their max |delta|
                    const int nvi = hdr[1];
                    float mx = 0.f;
                    for (int x = htid - HG * 32; x < nvi; x += HT - HG * 32) {
                        const uint32_t itm = vit[x];
                        const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x1ffu);
                        const int kvl = chl >> 7, cc = chl & 127;
                        const int bit = vf_bit(j, cc, BITS);
                        const uint32_t *vwp = vw_s + (kvl * 4 * BITS + (bit >> 5)) * 32 + vf_lane(j, cc);
                        unsigned long long w64 = vwp[0];
                        if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)vwp[32] << 32;
                        const int code = (int)((w64 >> (bit & 31)) & CM);
                        const float2 sz = vsz_s[j];
                        const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                        const float delta = xval - (cbVs[code] * sz.x + sz.y);
                        H.vdel[x] = delta;
                        mx = fmaxf(mx, fabsf(delta));
                    }
                    mx = warp_max_redux(mx);
                    if (lane == 0 && mx > 0.f) atomicMax(H.vmax, __float_as_int(mx));
                }
                E_cur = E_new;
            }
            half_sync(half);
            if (TIMED) { tc1 = clock64(); tm[3] += tc1 - tc0; tc0 = tc1; }

            // -------------------------------------------------------- a5: P.V dense
            {
                const float b_lo = H.beta_s[vq_lo], b_hi = H.beta_s[vq_hi];
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
                    // column vg: head vg / 2, its hi (vg even) or lo (vg odd) weight part
                    const int hb = vg >> 1;
                    const uint32_t *w32 = reinterpret_cast<const uint32_t *>(
                        H.w16 + ((vg & 1) ? HG * 32 : 0) + (vkv * G + (hb < G ? hb : 0)) * 32 + 16 * s2 + 2 * vt);
                    bw[s2][0] = hb < G ? w32[0] : 0u;
                    bw[s2][1] = hb < G ? w32[4] : 0u;
                }
                // the residual pass is skipped when the decode codebook is fp16-exact (R23)
                auto pv = [&](auto with_lo) {
#pragma unroll
                    for (int ml = 0; ml < MTW; ++ml) {
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            uint32_t a[4], alo[4];
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const int bit = ((ml * 2 + s2) * 4 + r) * FB;
                                const int wi = bit >> 5, sh = bit & 31;
                                // (field & (NE-1)) << 7 with one shift (funnel when it straddles)
                                uint32_t off;
                                if (sh + FB <= 32) off = sh >= 7 ? (vr[wi] >> (sh - 7)) : (vr[wi] << (7 - sh));
                                else off = __funnelshift_r(vr[wi], vr[wi + 1], sh - 7);
                                const uint32_t ad = vlane4 | (off & ((NE - 1) << 7));
                                a[r] = *reinterpret_cast<const uint32_t *>(vlut_b + ad);
                                if constexpr (decltype(with_lo)::value)
                                    alo[r] = *reinterpret_cast<const uint32_t *>(vlut_b + NE * 32 * 4 + ad);
                            }
                            mma_f16_f32(dacc[ml], a, bw[s2]);
                            if constexpr (decltype(with_lo)::value) mma_f16_f32(dacc[ml], alo, bw[s2]);
                        }
                    }
                };
                if (c.vcb_exact16) pv(std::false_type{});
                else pv(std::true_type{});
            }
            // ---------------------------------------------------- a6: V outliers
            {
                auto v_item = [&](uint32_t itm) {
                    const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x1ffu);
                    const int kvl = chl >> 7, cc = chl & 127;
                    const int bit = vf_bit(j, cc, BITS);
                    const uint32_t *vwp = vw_s + (kvl * 4 * BITS + (bit >> 5)) * 32 + vf_lane(j, cc);
                    unsigned long long w64 = vwp[0];
                    if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)vwp[32] << 32;
                    const int code = (int)((w64 >> (bit & 31)) & CM);
                    const float2 sz = vsz_s[j];
                    const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                    const float delta = xval - (cbVs[code] * sz.x + sz.y);
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int g = kvl * G + gg;
                        atomicAdd(&H.osp[g * kHeadDim + cc], H.p_s[g * 32 + j] * delta);
                    }
                };
                const int nvi = hdr[1];
                if (nvi) {
                    // sum_n p_n delta_{n,c} in fixed point: |p delta| 2^(24-e) < 2^25 with
                    // 2^e <= max|delta| < 2^(e+1); <= 32 items per (head, channel) and tile
                    const float mx = __int_as_float(H.vmax[0]);
                    const int emx = mx > 0.f ? ilog2f(mx) : 0;
                    const float S = pow2i(24 - emx);
                    if (htid == 0) H.vscale[0] = pow2i(emx - 24);   // 1/S
                    for (int x = htid; x < nvi; x += HT) {
                        const uint32_t itm = vit[x];
                        const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x1ffu);
                        const int kvl = chl >> 7, cc = chl & 127;
                        const float dS = H.vdel[x] * S;
#pragma unroll
                        for (int gg = 0; gg < G; ++gg) {
                            const int g = kvl * G + gg;
                            atomicAdd(&H.vfix[g * kHeadDim + cc], __float2int_rn(H.p_s[g * 32 + j] * dS));
                        }
                    }
                }
                if (hdr[3]) {
                    // overflowed bucket: this tile's Value outliers from the CSR rows (rare)
                    for (int r = htid; r < ntok * kv; r += HT) {
                        const uint32_t rec = __ldcg(c.vout + n0 * kv + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < c_lo || ch >= c_hi) continue;
                        v_item((rec & 0xffff0000u) | ((uint32_t)(r / kv) << 11) | (uint32_t)(ch - c_lo));
                    }
                }
            }
            // advance this half's anchors by two tiles (fp64 complex rotation by 64 theta_i)
            if (htid < 64) {
                const double2 a = H.anc64[htid], r = rot64[htid];
                const double2 b = make_double2(a.x * r.x - a.y * r.y, a.x * r.y + a.y * r.x);
                H.anc64[htid] = b;
                H.anc32[htid] = make_float2((float)b.x, (float)b.y);
                H.anc16[htid] = __floats2half2_rn((float)b.x, (float)b.y);
            }
            half_sync(half);
            if (TIMED) { tc1 = clock64(); tm[4] += tc1 - tc0; tc0 = tc1; }
        }
        if (nv_prev) {
            const float inv = H.vscale[0];
            for (int x = htid; x < HG * kHeadDim; x += HT) {
                const int v = H.vfix[x];
                if (v) H.osp[x] += (float)v * inv;
            }
        }
        half_sync(half);   // osp entries are updated by other threads below
        if (hw < HG) {
            const float l = warp_sum(l_lane), z = warp_sum(z_lane);
            if (lane == 0) { H.m_fin[hw] = m_run; H.l_fin[hw] = l; H.z_fin[hw] = z; }
        }
        {
            // dense P.V accumulators (units of 2^-E_cur): row g / g+8 = channel, column = head
            const float sc = pow2i(E_cur - WEXP);
#pragma unroll
            for (int ml = 0; ml < MTW; ++ml) {
                const int ch = (mt0 + ml) * 16 + vg;
                if (vt < G) {
                    float *o = H.osp + (vkv * G + vt) * kHeadDim + ch;
                    o[0] += (dacc[ml][0] + dacc[ml][1]) * sc;
                    o[8] += (dacc[ml][2] + dacc[ml][3]) * sc;
                }
            }
        }
        if (TIMED && tid == 0) {
#pragma unroll
            for (int x = 0; x < 5; ++x) atomicAdd(P.timers + x, tm[x]);
            atomicAdd(P.timers + 5, (unsigned long long)ntl);
            // wall-clock spread across CTAs: first start, last loop end, longest CTA loop
            atomicMax(P.timers + 6, ~ns_kernel0);
            const unsigned long long ns1 = gtimer_ns();
            atomicMax(P.timers + 7, ns1);
            atomicMax(P.timers + 8, ns1 - ns_kernel0);
        }
    }
    __syncthreads();

    // ------------------------------------------------ write partial (merge halves)
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    {
        const Half H0 = half_at(0), H1 = half_at(1);
        for (int x = tid; x < HG * (kHeadDim + 2); x += ATT_THREADS) {
            const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
            const bool u0 = ntl > 0 && H0.l_fin[g] != 0.f, u1 = ntl > 1 && H1.l_fin[g] != 0.f;
            const float m0 = u0 ? H0.m_fin[g] : -CUDART_INF_F, m1 = u1 ? H1.m_fin[g] : -CUDART_INF_F;
            const float m = fmaxf(m0, m1);
            const float w0 = u0 ? exp2f(m0 - m) : 0.f, w1 = u1 ? exp2f(m1 - m) : 0.f;
            const float l = w0 * (u0 ? H0.l_fin[g] : 0.f) + w1 * (u1 ? H1.l_fin[g] : 0.f);
            float o = 0.f;
            if (ch < kHeadDim) {
                if (u0) o += w0 * (H0.osp[g * kHeadDim + ch] + H0.z_fin[g]);
                if (u1) o += w1 * (H1.osp[g * kHeadDim + ch] + H1.z_fin[g]);
            }
            part[(g0 + g) * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
        }
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
        // partials in chunks of 8 independent L2 loads (one round trip per chunk)
        constexpr int MC = 8;
        const float *pbase = P.parts + (int64_t)gq * (kHeadDim + 2);
        const int64_t pstride = (int64_t)c.H_q * (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k)
                mv[k] = s0 + k < P.S ? __ldcg(pbase + (s0 + k) * pstride + kHeadDim) : -CUDART_INF_F;
#pragma unroll
            for (int k = 0; k < MC; ++k) m = fmaxf(m, mv[k]);
        }
        float l = 0.f, o = 0.f;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC], ov[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps + kHeadDim) : 0.f;
                lv[k] = in ? __ldcg(ps + kHeadDim + 1) : 0.f;
                ov[k] = (in && ch < kHeadDim) ? __ldcg(ps + ch) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                if (lv[k] == 0.f) continue;
                const float wgt = exp2f(mv[k] - m);
                l += wgt * lv[k];
                if (ch < kHeadDim) o += wgt * ov[k];
            }
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
    P.so_hdr = (unsigned)off; off = align128(off + 16);
    P.so_kit = (unsigned)off; off = align128(off + (size_t)c.kcap_g * 4);
    P.so_vit = (unsigned)off; off = align128(off + (size_t)c.vcap_g * 4);
    const size_t stb = off;
    // per-item Key-outlier contributions (one tile at a time), then the stage ring
    const size_t vdel = align128((size_t)NHALF * c.vcap_g * 4);
    P.so_vdel = (unsigned)align128(C::fixed);
    const size_t base = align128(P.so_vdel + vdel + 128);
    P.st_base = (unsigned)base;
    const size_t limit = 227 * 1024;
    for (int stages = 4; stages >= 2; stages -= 2) {
        const size_t total = base + stages * stb;
        if (total <= limit) {
            P.stages = stages;
            P.st_bytes = (unsigned)stb;
            return total;
        }
    }
    return 0;
}

template <int BITS, int HG, int G>
cudaError_t launch_t(const DevCache &c, Params &P, int grid, cudaStream_t s) {
    const size_t smem = layout<BITS, HG>(c, P);
    if (smem == 0) return cudaErrorInvalidConfiguration;
    if (P.timers) {   // diagnostics build of the kernel (phase clocks)
        cudaError_t e = cudaFuncSetAttribute(att_kernel<BITS, HG, G, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        att_kernel<BITS, HG, G, true><<<grid, ATT_THREADS, smem, s>>>(c, P);
        return cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(att_kernel<BITS, HG, G, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    att_kernel<BITS, HG, G, false><<<grid, ATT_THREADS, smem, s>>>(c, P);
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

// Query heads per outlier bucket group (the quantizer's (tile, group) item lists): the
// warp-autonomous MHA kernel reads one 2-head group per warp; the two-halves kernel uses
// CTAs of exactly one group.
int attend_bucket_heads(int bits, int H_q, int G, int vcb_exact16) {
    // MHA warp-autonomous kernel (4 bits only without the fp32-codebook residual pass)
    if (G == 1 && (bits == 2 || bits == 3 || (bits == 4 && vcb_exact16)) && H_q % 4 == 0) return 2;
    if ((G == 2 || G == 4 || G == 8) && bits >= 2 && bits <= 4) return G;   // GQA kernels: one KV head
    return attend_heads_per_cta(bits, H_q, G);
}

int attend_heads_per_cta(int bits, int H_q, int G) {
    if (G == 8 && (bits == 2 || bits == 3)) return 8;             // att_wgt_kernel: one CTA per KV head
    if (G > 1 && bits >= 2 && bits <= 4) return G < 4 ? G : 4;   // att_wgt_kernel (4-bit G = 8: two 4-head CTAs)
    const int cap = bits == 4 ? 1 : 4;   // K tables: HG * 64 * 4^b * 4 bytes of shared memory
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
    static const bool legacy = getenv("KVQ_ATT_LEGACY") != nullptr;
    const bool wa = !a.timers && !legacy && attend_wa_supported(c);
    const bool wag = !a.timers && !legacy && attend_wag_supported(c);
    // CTA heads: 4 for the warp-autonomous kernels, else one bucket group
    const int hg = wa ? 4 : (wag ? attend_heads_per_cta(c.bits, c.H_q, c.G) : (c.GW / kHeadDim) * c.G);
    if (hg == 0) return cudaErrorInvalidValue;
    if (a.kernel_out) *a.kernel_out = wa ? 1 : (wag ? 2 : 0);
    if (a.hg_out) *a.hg_out = hg;
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
    // MHA at 2-3 bits: the warp-autonomous kernel (kvq_attend_wa.cu); KVQ_ATT_LEGACY=1 or the
    // phase-timer diagnostics select the two-halves kernel below
    if (wa) return launch_attend_wa(c, a, S, s);
    if (wag) return launch_attend_wag(c, a, S, s);
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
