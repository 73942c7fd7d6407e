// kvq_attend_wa.cu -- ATT, warp-autonomous variant for multi-head attention (G = 1) at 2 and
// 3 bits: single-token decode attention over the compressed cache.
//
// Why a second kernel: the two-halves kernel (kvq_attend.cu) splits every 32-token tile over
// 8 warps (RoPE pairs over warps, then a cross-warp score reduction, a softmax phase on 4 of
// the 8 warps and a P.V phase), i.e. three barriers and ~2,000 bookkeeping instructions per
// tile; ncu showed it issue- and latency-bound at IPC ~2.1 (profiles/r1_att_kernel.md).  Here
// each warp owns whole tiles of the CTA's 4 query heads and runs the complete method on them
// with no block-level synchronisation in the tile loop:
//   a1   (prologue, per CTA) q~ = RoPE(q, pos) with exact fp64 angles (R11, R12) times
//        log2(e)/sqrt(d); per (head, RoPE pair i) a 2^{2b}-entry table of fp16 pairs
//        (A, B) = the paper's per-channel LUT with the query and the affine
//        folded in, so one lookup + 2 FMAs give cos(n' th_i) A + sin(n' th_i) B, the pair's
//        share of q~ . RoPE(K^_n, n') (RoPE after dequantization);
//   a2   lane = token: per pair one rotation cis(t0 th_i) x cis(j th_i) (fp16x2, shared by
//        the 4 heads) and per head one table lookup + 2 fp16 x fp16 -> fp32 FMAs;
//   a3   Key outliers (items bucketed per tile and head group by the quantizer) and the
//        few "heavy" pairs (fp32 tables) in fp32, lane-parallel;
//   a4   online softmax per head in base 2 with shuffles only;
//   a5   P.V on the tensor cores: mma.m16n8k16, A = Value codes (stored in A-fragment
//        order) through the shared codebook pair table, B = fp16 weights p s_n 2^(14-E)
//        (every column the same head, so each lane ends with rows g, g+8 of the product),
//        Sum_n p_n z_n as a per-lane scalar (affine fold);
//   a6   Value outliers p_n (x - V^(code)) lane-parallel into per-warp shared sums;
//   a7   warp partials -> CTA partial (log-sum-exp) -> split merge by the last CTA.
// Data reach the warp straight from HBM into registers (K words of the next tile during the
// current P.V, V words during the current K phase), so there is no shared staging ring and
// no producer warp.
#include "kvq_attend_common.cuh"

#include <cstdlib>

namespace kvq {
namespace {


template <int BITS, bool RESID, int WH>
struct WCfg {
    static constexpr int NWARP = NSTREAM * (HG / WH);
    static constexpr int NTHR = NWARP * 32;
    static constexpr int IPL = 4;                         // bucket items per lane in registers
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int KWH = 4 * BITS;                  // code words per head per token
    static constexpr int HMAX = 4;                        // fp32 "heavy" pairs per head (R24: 4 keep the error of 8)
    // K table entries per (head, RoPE pair): 2-3 bits, one entry per pair code (the query and
    // both channels folded in); 4 bits, per channel (16 + 16 entries, their two lookups summed
    // by the FMAs), since a 256-entry pair table per pair would need 64 KB per head
    static constexpr int NK = BITS == 4 ? 32 : NE;
    static constexpr size_t valign = (size_t)NE * 32 * 4;  // V table alignment (OR addressing)
    static constexpr size_t vlut = (size_t)(RESID ? 2 : 1) * NE * 32 * 4;
    static constexpr size_t klut = (size_t)HG * kPairs * NK * 4;
    static constexpr size_t hlut = (size_t)HG * HMAX * NK * 8;
    static constexpr size_t t1h = 0;
    static constexpr size_t t1f = 0;   // (round 2: token angles from MUFU sin/cos, no table)
    // per warp: K words of the tile (cp.async target), K-outlier fixed-point terms (then p),
    // V-outlier fixed-point sums, anchors (fp16 rotation pairs, fp32)
    static constexpr size_t w_kst = (size_t)WH * KWH * 32 * 4;
    static constexpr size_t w_bytes = w_kst + WH * 32 * 4 + WH * kHeadDim * 4 + 64 * 8;
    static constexpr int KCH = WH * KWH / 4;              // 16-byte K-word chunks per lane
    static constexpr size_t small = HG * kHeadDim * 4 /* qs */ + 64 * 16 /* rot */
        + HG * kHeadDim * 4 * 2 /* ks, kz */ + 64 * 4 /* cb */ + HG * 64 * 4 /* bound */
        + HG * 64 /* heavy flags */ + HG * 8 * 4 * 2 /* heavy lists */ + HG * 4 * 2 + 64
        + 64 * 40 /* theta, cis(pos theta), cis(first tile) */;
    static constexpr size_t total = valign + vlut + klut + hlut + t1h + t1f + NWARP * w_bytes + small;
};


// the kernel body; blk is the CTA's index within its own attend (one cache)
template <int BITS, bool RESID, int WH>
__device__ __forceinline__ void att_wa_body(const DevCache &c, const WParams &P, const int blk) {
    using C = WCfg<BITS, RESID, WH>;
    constexpr int NWARP = C::NWARP, NTHR = C::NTHR, IPL = C::IPL;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int KWH = C::KWH;
    constexpr int HMAX = C::HMAX;
    constexpr int FB = 2 * BITS;   // bits of one pair / A field

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // the V table starts at a multiple of its size in the shared window, so a lookup address
    // is (base | code << 7 | lane << 2) with one LOP3
    const uint32_t s0 = smem_u32(smem_raw);
    unsigned char *sp = smem_raw + ((C::valign - (s0 % C::valign)) % C::valign);
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += C::klut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += C::hlut;
    uint32_t *t1h = reinterpret_cast<uint32_t *>(sp); sp += C::t1h;
    float2 *t1f = reinterpret_cast<float2 *>(sp); sp += C::t1f;
    unsigned char *wbase = sp; sp += NWARP * C::w_bytes;
    float *qs = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    double2 *rot = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    float *ks_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *kz_s = reinterpret_cast<float *>(sp); sp += HG * kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;
    float *bound_s = reinterpret_cast<float *>(sp); sp += HG * 64 * 4;
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(sp); sp += HG * 64;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += HG * 8 * 4;
    float *lut_sc = reinterpret_cast<float *>(sp); sp += HG * 4;
    float *lut_inv = reinterpret_cast<float *>(sp); sp += HG * 4;
    int *flag_s = reinterpret_cast<int *>(sp); sp += 64;
    double2 *qcis = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double2 *cbase = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double *th64 = reinterpret_cast<double *>(sp); sp += 64 * 8;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_hg = c.H_q / HG;
    const int hg = blk % n_hg;
    const int split = blk / n_hg;
    const int g0 = hg * HG;               // first query head of the CTA = first KV head (G = 1)
    const int hw0 = (warp % (HG / WH)) * WH;   // this warp's first head within the CTA
    const int c_lo = g0 * kHeadDim;
    const int stream = warp / (HG / WH);
    // this warp's outlier buckets: the quantizer groups items per WH heads (c.GW = WH * 128)
    const int grp = (g0 + hw0) / WH;
    const int w_lo = c_lo + hw0 * kHeadDim;   // first channel of the warp's heads
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int D = c.D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;   // decode codebooks

    // per-warp scratch
    unsigned char *wp = wbase + warp * C::w_bytes;
    uint32_t *kst = reinterpret_cast<uint32_t *>(wp); wp += C::w_kst;
    int *kfix = reinterpret_cast<int *>(wp); wp += WH * 32 * 4;
    float *ps = reinterpret_cast<float *>(kfix);   // p of the tile, once the K terms are read
    int *vfix = reinterpret_cast<int *>(wp); wp += WH * kHeadDim * 4;
    // Key-outlier terms too large for the 32-bit fixed point (|term| >= 2^7 log2 units, only
    // extreme fp16 outliers): fp32 sums [WH][32] in the V-outlier scratch, which is free from
    // the K phase until the V-outlier phase (zeroed again at the end of every tile)
    float *kbig = reinterpret_cast<float *>(vfix);
    float2 *anc32 = reinterpret_cast<float2 *>(wp);

    // ------------------------------------------------------------- first tile's data
    // issued before the table build so the HBM latency overlaps the prologue
    const int t_first = t_begin + stream;
    uint32_t kitm[IPL], vitm[IPL];
    uint32_t cnt_k = 0, cnt_v = 0, ncnt_k = 0, ncnt_v = 0;
    float2 vsz = make_float2(0.f, 0.f);
    // K words of a tile (the warp's 2 heads: 3 KB contiguous in HBM) copied straight into kst
    // with cp.async: issued once the previous tile's readers of kst are done, in flight during
    // softmax, P.V and the V outliers, no registers held
    auto issue_k = [&](int t) {
        const unsigned char *src = reinterpret_cast<const unsigned char *>(
            c.kcodes + ((int64_t)t * c.QW + (g0 + hw0) * KWH) * 32);
        const uint32_t dst = smem_u32(kst);
#pragma unroll
        for (int k = 0; k < C::KCH; ++k) cp_async16(dst + (uint32_t)(lane + 32 * k) * 16u, src + (lane + 32 * k) * 16);
    };
    auto load_counts = [&](int t, uint32_t &nk, uint32_t &nv) {
        nk = nv = 0;
        if (t < t_end) {
            const uint32_t *gc = c.gcnt + ((int64_t)t * c.NG + grp) * 2;
            nk = __ldg(gc);
            nv = __ldg(gc + 1);
        }
    };
    // Items of a (tile, 4-head group) bucket are in (token, channel) order; a warp keeps the
    // whole bucket (IPL per lane) and skips the other heads' items.
    auto load_items = [&](int t) {
        const int64_t bucket = (int64_t)t * c.NG + grp;
        const uint32_t nk = cnt_k > (uint32_t)c.kcap_g ? 0u : cnt_k;
        const uint32_t nv = cnt_v > (uint32_t)c.vcap_g ? 0u : cnt_v;
#pragma unroll
        for (int k = 0; k < IPL; ++k) {
            const uint32_t x = lane + 32 * k;
            kitm[k] = x < nk ? __ldg(c.kit + bucket * c.kcap_g + x) : 0u;
            vitm[k] = x < nv ? __ldg(c.vit + bucket * c.vcap_g + x) : 0u;
        }
        vsz = (int64_t)t * 32 + lane < P.T ? __ldg(c.vsz + (int64_t)t * 32 + lane) : make_float2(0.f, 0.f);
    };

    // the first tile's K words and counts overlap the prologue unless the tile is the tail tile
    // (which a concurrent append may still be writing, see pdl_wait)
    const bool early = t_first < t_end && t_first != P.ntiles - 1;
    if (early) {
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ---------------------------------------------------------------- prologue (a1)
    // theta_i and cis(pos theta_i) for the query once per CTA (64 threads, exact fp64 angles,
    // R11, R12)
    if (tid < 64) {
        const int i = tid;
        const double th = c.theta_tab[i];
        th64[i] = th;
        double s, co;
        sincos(red2pi((double)P.pos * th), &s, &co);   // reduced first: fast-path sincos
        qcis[i] = make_double2(co, s);
    }
    __syncthreads();
    // Token angles.  Per warp and tile the anchor angle a_i = (pos_base + 32 t + 16) th_i,
    // reduced mod 2 pi in fp64 (register state, pairs lane and lane + 32, advanced per tile by
    // the stream stride), is published as (a_i, th_i) fp32; token j's angle is then
    // a_i + (j - 16) th_i (|.| < pi + 16) in fp32 and cis of it comes from the MUFU sin/cos
    // (abs error ~1e-6, far below the fp16 rounding of the factors).
    double ang64[2], step64[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int i = lane + 32 * k;
        const double th = th64[i];
        ang64[k] = red2pi((double)(c.pos_base + (int64_t)t_first * kTileTokens + 16) * th);
        step64[k] = red2pi((double)(NSTREAM * kTileTokens) * th);
        anc32[i] = make_float2((float)ang64[k], (float)th);
    }
    for (int x = lane; x < WH * 32; x += 32) { kfix[x] = 0; kbig[x] = 0.f; }
    for (int x = tid; x < HG * kHeadDim; x += NTHR) {
        ks_s[x] = c.kpar[c_lo + x];
        kz_s[x] = c.kpar[D + c_lo + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
    if (tid < 16) flag_s[tid] = 0;
    const double qscale = 1.4426950408889634 / sqrt((double)kHeadDim);
    for (int x = tid; x < HG * 64; x += NTHR) {
        const int g = x >> 6, i = x & 63;
        const __half *qg = P.q + (int64_t)(g0 + g) * kHeadDim;
        const double co = qcis[i].x, s = qcis[i].y;
        const double a = (double)__half2float(qg[i]), b = (double)__half2float(qg[i + 64]);
        qs[g * kHeadDim + i] = (float)((a * co - b * s) * qscale);
        qs[g * kHeadDim + i + 64] = (float)((b * co + a * s) * qscale);
    }
    __syncthreads();
    // per (head, pair) bound of |A|, |B|: pairs above 1/2 of the head maximum (at most HMAX)
    // get fp32 tables; the rest fp16 tables scaled so the largest entry is <= 2^14
    for (int x = tid; x < HG * 64; x += NTHR) {
        const int g = x >> 6, i = x & 63;
        const int ci = g * kHeadDim + i, cj = ci + 64;
        const float mx = fmaxf(fabsf(cbK[0] * ks_s[ci] + kz_s[ci]), fabsf(cbK[CM] * ks_s[ci] + kz_s[ci]));
        const float my = fmaxf(fabsf(cbK[0] * ks_s[cj] + kz_s[cj]), fabsf(cbK[CM] * ks_s[cj] + kz_s[cj]));
        const float qa = fabsf(qs[g * kHeadDim + i]), qb = fabsf(qs[g * kHeadDim + i + 64]);
        bound_s[x] = fmaxf(qa * mx + qb * my, qb * mx + qa * my);
    }
    __syncthreads();
    for (int g = warp; g < HG; g += NWARP) {
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
            int e = 0;
            if (rest > 0.f && isfinite(rest)) e = 14 - ilogbf(rest) - 1;
            e = max(-100, min(100, e));
            lut_sc[g] = ldexpf(1.f, e);
            lut_inv[g] = ldexpf(1.f, -e);
        }
    }
    __syncthreads();
    if constexpr (BITS == 4) {
        // per (head, pair): T1[a] = (qa x(a), qb x(a)) for channel i, T2[b] = (qb y(b), -qa y(b))
        // for channel i + 64, so T1[a] + T2[b] is the pair table entry of the 2-3 bit kernels
        for (int x = tid; x < HG * 64 * 32; x += NTHR) {
            const int e = x & 31, gi = x >> 5;
            const int g = gi >> 6, i = gi & 63;
            const int ch = g * kHeadDim + i + (e < 16 ? 0 : 64);
            const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
            const float v = cbK[e & 15] * ks_s[ch] + kz_s[ch];
            const float2 t = e < 16 ? make_float2(qa1 * v, qb1 * v) : make_float2(qb1 * v, -qa1 * v);
            const bool heavy = heavy_s[gi] != 0;
            if (heavy) {
                int hslot = 0;
                for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
                klut[(size_t)gi * 32 + e] = 0u;
                hlut[(g * HMAX + hslot) * 32 + e] = t;
            } else {
                const float sc = lut_sc[g];
                klut[(size_t)gi * 32 + e] = pack_half2(t.x * sc, t.y * sc);
            }
        }
    } else
    // K table entries [g][i][pair code], one (head, pair, second code) row per work item,
    // written as 16-byte vectors (the 2^b entries of a row are contiguous)
    for (int x = tid; x < HG * 64 * (CM + 1); x += NTHR) {
        const int bb = x % (CM + 1), gi = x / (CM + 1);
        const int g = gi >> 6, i = gi & 63;
        const int ci = g * kHeadDim + i, cj = ci + 64;
        const float *cbKsh = cb_s + 16;
        const float sc = lut_sc[g];
        const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
        const float qa = qa1 * sc, qb = qb1 * sc;
        const float ksi = ks_s[ci], kzi = kz_s[ci];
        const float yb = cbKsh[bb] * ks_s[cj] + kz_s[cj];
        const bool heavy = heavy_s[gi] != 0;
        int hslot = 0;
        if (heavy)
            for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
        uint32_t e[CM + 1];
#pragma unroll
        for (int a = 0; a <= CM; ++a) {
            const float xa = cbKsh[a] * ksi + kzi;
            e[a] = heavy ? 0u : pack_half2(qa * xa + qb * yb, qb * xa - qa * yb);
            if (heavy) hlut[(g * HMAX + hslot) * NE + (bb << BITS) + a] = make_float2(qa1 * xa + qb1 * yb, qb1 * xa - qa1 * yb);
        }
        uint4 *dst = reinterpret_cast<uint4 *>(klut + (size_t)(g * 64 + i) * NE + (bb << BITS));
#pragma unroll
        for (int v = 0; v < (CM + 1) / 4; ++v) dst[v] = make_uint4(e[4 * v], e[4 * v + 1], e[4 * v + 2], e[4 * v + 3]);
    }
    // V table: lane-private copies (entry e of lane l at word e*32 + l): the fp16 codebook
    // pair and (RESID) its fp16 residual Chat - fp16(Chat) (R23)
    for (int x = tid; x < NE * 32; x += NTHR) {
        const int e = x >> 5;
        const float ca = cbV[e & CM], cb = cbV[e >> BITS];
        vlut[x] = pack_half2(ca, cb);
        if constexpr (RESID)
            vlut[NE * 32 + x] = pack_half2(ca - __half2float(__float2half_rn(ca)), cb - __half2float(__float2half_rn(cb)));
    }
    __syncthreads();

    // The preceding append (programmatic dependent launch) writes only the tail tile (its
    // token's code words, (s, z), outlier records, bucket items and counts), so a warp waits
    // for it only before its first read of tail-tile data; every other tile streams while the
    // append is still running.  (Without the launch attribute the wait is a no-op.)
    auto tail_wait = [&](int tt) {
        if (tt == P.ntiles - 1) pdl_wait();
    };
    if (t_first < t_end && !early) {
        tail_wait(t_first);
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ================================================================ tile loop (per warp)
    // table bases, OR-ed with the shifted codes (the compiler must not turn the OR into an add)
    const uint32_t klut_u = opaque(smem_u32(klut) + (uint32_t)(hw0 * 64 * C::NK * 4));
    const uint32_t vlut_u = opaque(smem_u32(vlut) | (4u * lane));
    const int vg = lane >> 2, vt = lane & 3;
    const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
    float m_run[WH], l_lane[WH], z_lane[WH], acc[WH][4];
#pragma unroll
    for (int h = 0; h < WH; ++h) {
        m_run[h] = -CUDART_INF_F; l_lane[h] = 0.f; z_lane[h] = 0.f;
        acc[h][0] = acc[h][1] = acc[h][2] = acc[h][3] = 0.f;
    }
    // fp32 rotation cis(n' th_i) of token j of the tile: anchor angle + (j - 16) th_i
    auto rot32 = [&](int i, int j, float &co, float &si) {
        const float2 a = anc32[i];
        __sincosf(fmaf((float)(j - 16), a.y, a.x), &si, &co);
    };
    auto rot16 = [&](int i) -> uint32_t {
        float co, si;
        rot32(i, lane, co, si);
        return pack_half2(co, si);
    };

    for (int t = t_first; t < t_end; t += NSTREAM) {
        const int64_t n0 = (int64_t)t * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        const bool valid = lane < ntok;
        const bool kov = cnt_k > (uint32_t)c.kcap_g, vov = cnt_v > (uint32_t)c.vcap_g;
        const int nk = kov ? 0 : (int)cnt_k, nv = vov ? 0 : (int)cnt_v;
        // this tile's outlier items and (s, z) (consumed after the K loop), next tile's counts
        load_items(t);
        tail_wait(t + NSTREAM);
        load_counts(t + NSTREAM, ncnt_k, ncnt_v);

        // V words of this tile: in flight during the K phase
        // V words: issued halfway through the K loop, once the first half's K words are dead
        uint32_t vw[WH][KWH];
        auto load_v = [&]() {
#pragma unroll
            for (int h = 0; h < WH; ++h)
#pragma unroll
                for (int w = 0; w < KWH; ++w)
                    vw[h][w] = __ldg(c.vcodes + vf_word(t, c.H_kv, g0 + hw0 + h, w, lane, BITS));
        };

        cp_async_wait_all();
        __syncwarp();
        uint32_t kw[WH][BITS == 4 ? 1 : KWH];   // 4 bits: read from kst per word in the loop
        if constexpr (BITS != 4) {
#pragma unroll
            for (int h = 0; h < WH; ++h)
#pragma unroll
                for (int w = 0; w < KWH; ++w) kw[h][w] = kst[(h * KWH + w) * 32 + lane];
        }

        // ---------------------------------------------------------- a2: K dense
        // two accumulator pairs per head (even / odd pairs): shorter FMA dependency chains
        float acc_c[WH][2], acc_s[WH][2];
#pragma unroll
        for (int h = 0; h < WH; ++h) acc_c[h][0] = acc_s[h][0] = acc_c[h][1] = acc_s[h][1] = 0.f;
#pragma unroll
        for (int i = 0; i < kPairs; ++i) {
            if (i == kPairs / 2) load_v();
            // cis(n' th_i) from the MUFU, rounded once to fp16
            const uint32_t cs = rot16(i);
            if constexpr (BITS == 4) {
                // pair i = byte i % 4 of word i / 4: code a (low nibble, channel i) and b (high
                // nibble, channel i + 64), one lookup each in the pair's T1 / T2 halves
                const int sh = 8 * (i & 3);
#pragma unroll
                for (int h = 0; h < WH; ++h) {
                    if ((i & 3) == 0) kw[h][0] = kst[(h * KWH + (i >> 2)) * 32 + lane];
                    const uint32_t w = kw[h][0];
                    const uint32_t oa = (sh >= 2 ? (w >> (sh - 2)) : (w << 2)) & 0x3cu;
                    const uint32_t ob = (w >> (sh + 2)) & 0x3cu;
                    const uint32_t base = klut_u + (uint32_t)((h * 64 + i) * 32 * 4);
                    const uint32_t t1 = lds_u32(base | oa), t2 = lds_u32(base | 64u | ob);
                    fma2_f16_f32(t1, cs, acc_c[h][i & 1], acc_s[h][i & 1]);
                    fma2_f16_f32(t2, cs, acc_c[h][i & 1], acc_s[h][i & 1]);
                }
            } else {
            const int bit = FB * i, w = bit >> 5, sh = bit & 31;
#pragma unroll
            for (int h = 0; h < WH; ++h) {
                uint32_t off;
                if (sh + FB <= 32) off = sh >= 2 ? (kw[h][w] >> (sh - 2)) : (kw[h][w] << (2 - sh));
                else off = __funnelshift_r(kw[h][w], kw[h][w + 1], sh - 2);
                const uint32_t a = klut_u | (off & ((NE - 1) << 2));
                const uint32_t ab = lds_u32(a + (uint32_t)((h * 64 + i) * NE * 4));
                fma2_f16_f32(ab, cs, acc_c[h][i & 1], acc_s[h][i & 1]);
            }
            }
        }
        __syncwarp();

        // -------------------------------------------- a3: heavy pairs, Key outliers (fp32)
        float sco[WH];
#pragma unroll
        for (int h = 0; h < WH; ++h) {
            const int hc = hw0 + h;
            float hs = 0.f;
            const int nh = hv_n[hc];
            for (int u = 0; u < nh; ++u) {
                const int i = hv_pair[hc * 8 + u];
                const int bit = FB * i;
                const int wq = h * KWH + (bit >> 5);
                // the word after may be past the head's last (then unused): kst is followed by
                // the warp's other scratch, so the read stays in bounds
                const int pc = (int)(__funnelshift_r(kst[wq * 32 + lane], kst[(wq + 1) * 32 + lane], bit & 31) & (NE - 1));
                float2 ab;
                if constexpr (BITS == 4) {
                    const float2 t1 = hlut[(hc * HMAX + u) * 32 + (pc & 15)], t2 = hlut[(hc * HMAX + u) * 32 + 16 + (pc >> 4)];
                    ab = make_float2(t1.x + t2.x, t1.y + t2.y);
                } else {
                    ab = hlut[(hc * HMAX + u) * NE + pc];
                }
                float co, si;
                rot32(i, lane, co, si);
                hs += co * ab.x + si * ab.y;
            }
            sco[h] = ((acc_c[h][0] + acc_s[h][0]) + (acc_c[h][1] + acc_s[h][1])) * lut_inv[hc] + hs;
        }
        // item of the CTA's 4-head group -> (token, head of this warp or -1, correction)
        auto k_corr = [&](uint32_t itm, int &j, int &h) -> float {
            j = (int)((itm >> 11) & 31u);
            const int chl = (int)(itm & 0x1ffu), flag = (int)((itm >> 9) & 3u);
            h = chl >> 7;   // head of this warp
            const int cc = chl & 127, i = cc & 63, up = cc >> 6;
            const int ccta = hw0 * kHeadDim + chl;   // channel within the CTA's 4 heads
            int code = flag == 1 ? CM : 0;
            if (flag == 0) {   // code not named by the item: read it from the tile's words
                const int bit = FB * i;
                const int wq = h * KWH + (bit >> 5);
                unsigned long long w64 = kst[wq * 32 + j];
                if ((bit & 31) + FB > 32) w64 |= (unsigned long long)kst[(wq + 1) * 32 + j] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                code = (pc >> (up * BITS)) & CM;
            }
            const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
            const float delta = xval - (cbKs[code] * ks_s[ccta] + kz_s[ccta]);
            float co, si;
            rot32(i, j, co, si);
            const float qa = qs[(hw0 + h) * kHeadDim + i], qb = qs[(hw0 + h) * kHeadDim + i + 64];
            return delta * (up ? (qb * co - qa * si) : (qa * co + qb * si));
        };
        {
            const int64_t bucket = (int64_t)t * c.NG + grp;
#pragma unroll
            for (int k = 0; k < IPL; ++k) {
                if (32 * k < nk && lane + 32 * k < nk) {
                    int j, h;
                    const float v = k_corr(kitm[k], j, h);
                    kfix_add32(&kfix[h * 32 + j], &kbig[h * 32 + j], v);
                }
            }
            for (int x = 32 * IPL + lane; x < nk; x += 32) {
                int j, h;
                const float v = k_corr(__ldg(c.kit + bucket * c.kcap_g + x), j, h);
                kfix_add32(&kfix[h * 32 + j], &kbig[h * 32 + j], v);
            }
            if (kov) {   // overflowed bucket: this tile's Key outliers from the CSC arrays (rare)
                for (int j = 0; j < ntok; ++j) {
                    const uint32_t r0 = __ldg(c.kptr + n0 + j), r1 = __ldg(c.kptr + n0 + j + 1);
                    for (uint32_t r = r0 + lane; r < r1; r += 32) {
                        const uint32_t rec = __ldcg(c.kout + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < w_lo || ch >= w_lo + WH * kHeadDim) continue;
                        int jj, h;
                        const float v = k_corr((rec & 0xffff0000u) | ((uint32_t)j << 11) | (uint32_t)(ch - w_lo), jj, h);
                        kfix_add32(&kfix[h * 32 + jj], &kbig[h * 32 + jj], v);
                    }
                }
            }
        }
        __syncwarp();

        // kst is free (heavy pairs and Key items done): the next tile's K words
        const int tn = t + NSTREAM;
        if (tn < t_end) {
            tail_wait(tn);
            issue_k(tn);
        }

        // ------------------------------------------------------ a4: online softmax
        // weights p s_n 2^(WEXP - E) with E from the tile's largest s_n (fp16 normal range)
        const float smax = warp_max_redux(valid ? vsz.x : 0.f);
        const int E = smax > 0.f ? ilog2f(smax) + 1 : 0;
        const float pe = pow2i(WEXP - E), sc_out = pow2i(E - WEXP);
        uint32_t w2s[WH], w2l[WH];
#pragma unroll
        for (int h = 0; h < WH; ++h) {
            float s = sco[h] + (float)kfix[h * 32 + lane] * (1.f / kKfixScale) + kbig[h * 32 + lane];
            s = valid ? s : -CUDART_INF_F;
            const float m_new = fmaxf(m_run[h], warp_max_redux(s));
            const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run[h] - m_new);
            const float p = valid ? exp2f(s - m_new) : 0.f;
            l_lane[h] = l_lane[h] * alpha + p;
            z_lane[h] = z_lane[h] * alpha + p * vsz.y;
            m_run[h] = m_new;
            if (alpha != 1.f) {   // warp-uniform
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[h][r] *= alpha;
            }
            ps[h * 32 + lane] = p;   // over this lane's K term, just read
            // weight p s_n 2^(WEXP-E) as fp16 hi + lo (the lo part rides in the odd B columns,
            // so the mma sums both at no extra cost)
            const float wf = p * (vsz.x * pe);
            const __half wh = __float2half_rn(wf);
            const uint32_t hb = __half_as_ushort(wh), lb = __half_as_ushort(__float2half_rn(wf - __half2float(wh)));
            w2s[h] = hb | (__shfl_down_sync(0xffffffffu, hb, 1) << 16);   // tokens lane, lane+1
            w2l[h] = lb | (__shfl_down_sync(0xffffffffu, lb, 1) << 16);
        }
        // --------------------------------------------------------- a5: P.V dense
#pragma unroll
        for (int h = 0; h < WH; ++h) {
            // the next tile's K words, in flight during the rest of the tile (issued once the
            // first head's V words are consumed, to keep the register peak down)
            uint32_t bw[2][2];   // B fragments: weights of tokens 16 s2 + 2t (+1) and + 8;
                                 // column vg: hi part (vg even) or lo part (vg odd)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t xh = __shfl_sync(0xffffffffu, w2s[h], 16 * s2 + 2 * vt + 8 * r);
                    const uint32_t xl = __shfl_sync(0xffffffffu, w2l[h], 16 * s2 + 2 * vt + 8 * r);
                    bw[s2][r] = (vg & 1) ? xl : xh;
                }
            }
#pragma unroll
            for (int ml = 0; ml < 8; ++ml) {
                float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    uint32_t a[4], alo[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int bit = ((ml * 2 + s2) * 4 + r) * FB;
                        const int wi = bit >> 5, sh = bit & 31;
                        uint32_t off;
                        if (sh + FB <= 32) off = sh >= 7 ? (vw[h][wi] >> (sh - 7)) : (vw[h][wi] << (7 - sh));
                        else off = __funnelshift_r(vw[h][wi], vw[h][wi + 1], sh - 7);
                        const uint32_t ad = vlut_u | (off & ((NE - 1) << 7));
                        a[r] = lds_u32(ad);
                        if constexpr (RESID) alo[r] = lds_u32(ad + NE * 32 * 4);
                    }
                    mma_f16_f32(d, a, bw[s2]);
                    if constexpr (RESID) mma_f16_f32(d, alo, bw[s2]);
                }
                // columns 2t, 2t+1 hold head h's hi and lo sums: lane (g, t) keeps rows g, g+8
                // of m-tiles t, t+4
                if (vt == (ml & 3)) {
                    acc[h][(ml >> 2) * 2] += (d[0] + d[1]) * sc_out;
                    acc[h][(ml >> 2) * 2 + 1] += (d[2] + d[3]) * sc_out;
                }
            }
        }

        // ------------------------------------------------------ a6: V outliers
        // p_n (x - V^(code)) of this warp's items, summed in fixed point (native shared integer
        // atomics; scale from the tile's largest |term|) and folded into the lanes' accumulators
        if (nv > 0 || vov) {
#pragma unroll
            for (int h = 0; h < WH; ++h)
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int r = 0; r < 2; ++r) vfix[h * kHeadDim + 16 * (vt + 4 * k) + vg + 8 * r] = 0;
            __syncwarp();
            auto v_term = [&](uint32_t itm, bool act, int &h, int &cc) -> float {
                const int j = (int)((itm >> 11) & 31u), chl = (int)(itm & 0x1ffu), flag = (int)((itm >> 9) & 3u);
                h = chl >> 7;   // head of this warp
                cc = chl & 127;
                int code = flag == 1 ? CM : 0;
                if (act && flag == 0) {   // code not named by the item: read its word(s) (L2)
                    const int bit = vf_bit(j, cc, BITS);
                    const uint32_t *wq = c.vcodes + vf_word(t, c.H_kv, g0 + hw0 + h, bit >> 5, vf_lane(j, cc), BITS);
                    unsigned long long w64 = __ldg(wq);
                    if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)__ldg(wq + 32) << 32;
                    code = (int)((w64 >> (bit & 31)) & CM);
                }
                const float s_n = __shfl_sync(0xffffffffu, vsz.x, j), z_n = __shfl_sync(0xffffffffu, vsz.y, j);
                const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                return act ? ps[h * 32 + j] * (xval - (cbVs[code] * s_n + z_n)) : 0.f;
            };
            float vt_[IPL];
            int vix[IPL];   // h * 128 + channel
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < IPL; ++k) {
                vt_[k] = 0.f; vix[k] = 0;
                if (32 * k < nv) {
                    int h, cc;
                    vt_[k] = v_term(vitm[k], lane + 32 * k < nv, h, cc);
                    vix[k] = h * kHeadDim + cc;
                }
                mx = fmaxf(mx, fabsf(vt_[k]));
            }
            const bool slow = nv > 32 * IPL || vov;
            float ms = 0.f;
            const int64_t bucket = (int64_t)t * c.NG + grp;
            auto slow_term = [&](int x0, int &h, int &cc) -> float {   // item x0 + lane
                uint32_t itm = 0u;
                bool act = false;
                if (x0 < nv) {
                    act = x0 + lane < nv;
                    itm = act ? __ldg(c.vit + bucket * c.vcap_g + x0 + lane) : 0u;
                } else {   // CSR rows of the overflowed bucket, as items
                    const int kv = c.kv, r = x0 - nv + lane;
                    act = r < ntok * kv;
                    if (act) {
                        const uint32_t rec = __ldcg(c.vout + n0 * kv + r);
                        const int ch = (int)(rec & 0xffffu);
                        act = ch >= w_lo && ch < w_lo + WH * kHeadDim;
                        itm = (rec & 0xffff0000u) | ((uint32_t)(r / kv) << 11) | (uint32_t)(act ? ch - w_lo : 0);
                    }
                }
                return v_term(itm, act, h, cc);
            };
            const int x_end = (vov ? ntok * c.kv : 0) + nv;
            const int x_beg = vov ? 0 : 32 * IPL;   // overflow: every record from the CSR rows
            if (slow) {
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int h, cc;
                    ms = fmaxf(ms, fabsf(slow_term(x0, h, cc)));
                }
            }
            mx = warp_max(fmaxf(mx, ms));
            const int emx = mx > 0.f ? ilog2f(mx) : 0;
            const float S = pow2i(24 - emx);
#pragma unroll
            for (int k = 0; k < IPL; ++k)
                if (vt_[k] != 0.f) atomicAdd(&vfix[vix[k]], __float2int_rn(vt_[k] * S));
            if (slow) {
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int h, cc;
                    const float v = slow_term(x0, h, cc);
                    if (v != 0.f) atomicAdd(&vfix[h * kHeadDim + cc], __float2int_rn(v * S));
                }
            }
            __syncwarp();
            const float inv = pow2i(emx - 24);
#pragma unroll
            for (int h = 0; h < WH; ++h)
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int r = 0; r < 2; ++r)
                        acc[h][2 * k + r] += (float)vfix[h * kHeadDim + 16 * (vt + 4 * k) + vg + 8 * r] * inv;
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < WH; ++h) { kfix[h * 32 + lane] = 0; kbig[h * 32 + lane] = 0.f; }   // p read: done

        // advance the anchor angles by NSTREAM tiles (fp64, reduced mod 2 pi)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            ang64[k] = red2pi(ang64[k] + step64[k]);
            anc32[i].x = (float)ang64[k];
        }
        cnt_k = ncnt_k;
        cnt_v = ncnt_v;
        __syncwarp();
    }

    // ------------------------------------------- warp partials -> CTA partial (a7)
    cp_async_wait_all();
    __syncwarp();
    float *wpart = reinterpret_cast<float *>(kst);   // [WH][d + 2]
#pragma unroll
    for (int h = 0; h < WH; ++h) {
        const float l = warp_sum(l_lane[h]), z = warp_sum(z_lane[h]);
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ch = 16 * (vt + 4 * k) + vg + 8 * r;
                wpart[h * (kHeadDim + 2) + ch] = acc[h][2 * k + r] + z;
            }
        if (lane == 0) {
            wpart[h * (kHeadDim + 2) + kHeadDim] = m_run[h];
            wpart[h * (kHeadDim + 2) + kHeadDim + 1] = l;
        }
    }
    __syncthreads();
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    for (int x = tid; x < HG * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        const int wh = g / WH, hl = g % WH;   // warps with wh = warp % (HG/WH) hold head g
        float m = -CUDART_INF_F;
        for (int s = 0; s < NSTREAM; ++s) {
            const float *pw = reinterpret_cast<const float *>(wbase + (s * (HG / WH) + wh) * C::w_bytes) + hl * (kHeadDim + 2);
            if (pw[kHeadDim + 1] != 0.f) m = fmaxf(m, pw[kHeadDim]);
        }
        float l = 0.f, o = 0.f;
        for (int s = 0; s < NSTREAM; ++s) {
            const float *pw = reinterpret_cast<const float *>(wbase + (s * (HG / WH) + wh) * C::w_bytes) + hl * (kHeadDim + 2);
            const float lw = pw[kHeadDim + 1];
            if (lw == 0.f) continue;
            const float wt = exp2f(pw[kHeadDim] - m);
            l += wt * lw;
            if (ch < kHeadDim) o += wt * pw[ch];
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
    for (int x = tid; x < HG * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        const int gq = g0 + g;
        // the S partials in chunks of 8 independent L2 loads (one round trip per chunk, not per
        // split: the merge runs after every other CTA of the head group has finished)
        constexpr int MC = 8;
        const float *pbase = P.parts + (int64_t)gq * (kHeadDim + 2);
        const int64_t pstride = (int64_t)c.H_q * (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : -CUDART_INF_F;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k)
                if (lv[k] != 0.f) m = fmaxf(m, mv[k]);
        }
        float l = 0.f, o = 0.f;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC], ov[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : 0.f;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
                ov[k] = (in && ch < kHeadDim) ? __ldcg(ps2 + ch) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k) {   // fixed split order, as before
                if (lv[k] == 0.f) continue;
                const float wgt = exp2f(mv[k] - m);
                l += wgt * lv[k];
                if (ch < kHeadDim) o += wgt * ov[k];
            }
        }
        if (P.write_partial) {
            P.out[gq * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
        } else if (ch < kHeadDim) {
            P.out[gq * kHeadDim + ch] = o / l;
        }
    }
    if (tid == 0) P.tickets[hg] = 0;
}

template <int BITS, bool RESID, int WH>
__global__ void __launch_bounds__(WCfg<BITS, RESID, WH>::NTHR, 1) att_wa_kernel(DevCache c, WParams P) {
    att_wa_body<BITS, RESID, WH>(c, P, (int)blockIdx.x);
}

// Batched decode: one launch attends B independent caches of the same
// configuration (each its own context length, scratch and output).  The per-sequence
// descriptors travel in the kernel parameter space (constant bank, indexed by the CTA's
// sequence); CTA ranges are consecutive per sequence.
constexpr int kMaxBatch = 64;
struct WBatch {
    int n;
    int cta0[kMaxBatch + 1];
    DevCache c[kMaxBatch];
    WParams p[kMaxBatch];
};

template <int BITS, bool RESID, int WH>
__global__ void __launch_bounds__(WCfg<BITS, RESID, WH>::NTHR, 1) att_wa_batch_kernel(const __grid_constant__ WBatch b) {
    const int blk = (int)blockIdx.x;
    int s = 0;
    while (s + 1 < b.n && blk >= b.cta0[s + 1]) ++s;
    att_wa_body<BITS, RESID, WH>(b.c[s], b.p[s], blk - b.cta0[s]);
}

template <int BITS, bool RESID, int WH>
cudaError_t launch_wa_t(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    using C = WCfg<BITS, RESID, WH>;
    static_assert(C::total <= 227 * 1024, "shared memory");
    cudaError_t e = cudaFuncSetAttribute(att_wa_kernel<BITS, RESID, WH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    e = launch_maybe_pdl(att_wa_kernel<BITS, RESID, WH>, grid, C::NTHR, C::total, s, P.pdl != 0, c, P);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int BITS, bool RESID>
cudaError_t launch_wa_r(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    return launch_wa_t<BITS, RESID, 2>(c, P, grid, s);
}


// ===================================================================================
// Grouped-query attention (G = 4 query heads per KV head): att_wag_kernel.
// One CTA = one KV head and its G query heads; 16 warps = 16 tile streams, each warp runs
// whole tiles for all G heads.  Differences from the MHA kernel:
//   a2  one lookup per (token, pair) returns the G heads' (A, B) entries (vector LDS of the
//       code-interleaved tables) -> 2G FMAs, so the rotation and the extraction are shared;
//   a5  the contraction is dense over the G heads: B = the G heads' weights (columns 0..G-1)
//       and the mma accumulators persist across tiles (rescaled per head column when the
//       running max or the weight exponent grows);
//   a3/a6 every outlier item corrects all G heads.
constexpr int NSG = 16;    // tile streams (= warps) per GQA CTA (14 with the fp32-codebook
                           // second V table, which needs the shared memory of two warps)

template <int BITS, bool RESID, int G>
struct GCfg {
    static_assert(G <= 4, "hi/lo weight columns: 2 G <= 8 mma columns");
    static constexpr int NWARP = (RESID && BITS == 3 && G == 4) ? 14 : NSG;
    static constexpr int NTHR = NWARP * 32;
    static constexpr int IPL = 4;
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int KWH = 4 * BITS;
    static constexpr int HMAX = 8;
    static constexpr size_t valign = (size_t)NE * 32 * 4;
    static constexpr size_t vlut = (size_t)(RESID ? 2 : 1) * NE * 32 * 4;
    static constexpr size_t klut = (size_t)G * kPairs * NE * 4;   // [i][pair code][G]
    static constexpr size_t hlut = (size_t)G * HMAX * NE * 8;
    static constexpr size_t t1h = 0;
    static constexpr size_t t1f = 0;   // token angles from MUFU sin/cos (as the MHA kernel)
    // per warp: K words (cp.async target), K-outlier terms (then p) [G][32], V-outlier sums
    // fp32 [G][128], anchors
    static constexpr size_t w_kst = (size_t)KWH * 32 * 4;
    static constexpr size_t w_bytes = w_kst + G * 32 * 4 + G * kHeadDim * 4 * 2 + 64 * 8;
    static constexpr int KCH = KWH / 4;
    static constexpr size_t small = G * kHeadDim * 4 /* qs */ + 64 * 16 /* rot */
        + kHeadDim * 4 * 2 /* ks, kz */ + 64 * 4 /* cb */ + G * 64 * 4 /* bound */
        + G * 64 /* heavy flags */ + G * 8 * 4 * 2 /* heavy lists */ + G * 4 * 2 + 64
        + 64 * 40 /* theta, cis(pos theta), cis(first tile) */;
    static constexpr size_t total = valign + vlut + klut + hlut + t1h + t1f + NWARP * w_bytes + small;
};

template <int G>
__device__ __forceinline__ void lds_vecG(uint32_t addr, uint32_t (&v)[G]) {
    if constexpr (G == 2) {
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
    } else {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    }
}

template <int BITS, bool RESID, int G>
__global__ void __launch_bounds__(GCfg<BITS, RESID, G>::NTHR, 1) att_wag_kernel(DevCache c, WParams P) {
    using C = GCfg<BITS, RESID, G>;
    constexpr int NWARP = C::NWARP, NTHR = C::NTHR, IPL = C::IPL;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int KWH = C::KWH;
    constexpr int HMAX = C::HMAX;
    constexpr int FB = 2 * BITS;
    constexpr int LG = G == 2 ? 1 : 2;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s0 = smem_u32(smem_raw);
    unsigned char *sp = smem_raw + ((C::valign - (s0 % C::valign)) % C::valign);
    uint32_t *vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    uint32_t *klut = reinterpret_cast<uint32_t *>(sp); sp += C::klut;
    float2 *hlut = reinterpret_cast<float2 *>(sp); sp += C::hlut;
    uint32_t *t1h = reinterpret_cast<uint32_t *>(sp); sp += C::t1h;
    float2 *t1f = reinterpret_cast<float2 *>(sp); sp += C::t1f;
    unsigned char *wbase = sp; sp += NWARP * C::w_bytes;
    float *qs = reinterpret_cast<float *>(sp); sp += G * kHeadDim * 4;
    double2 *rot = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    float *ks_s = reinterpret_cast<float *>(sp); sp += kHeadDim * 4;
    float *kz_s = reinterpret_cast<float *>(sp); sp += kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;
    float *bound_s = reinterpret_cast<float *>(sp); sp += G * 64 * 4;
    uint8_t *heavy_s = reinterpret_cast<uint8_t *>(sp); sp += G * 64;
    int *hv_pair = reinterpret_cast<int *>(sp); sp += G * 8 * 4;
    int *hv_n = reinterpret_cast<int *>(sp); sp += G * 8 * 4;
    float *lut_sc = reinterpret_cast<float *>(sp); sp += G * 4;
    float *lut_inv = reinterpret_cast<float *>(sp); sp += G * 4;
    int *flag_s = reinterpret_cast<int *>(sp); sp += 64;
    double2 *qcis = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double2 *cbase = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double *th64 = reinterpret_cast<double *>(sp); sp += 64 * 8;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_hg = c.H_kv;   // one CTA per KV head
    const int hk = blockIdx.x % n_hg;
    const int split = blockIdx.x / n_hg;
    const int g0 = hk * G;     // first query head
    const int c_lo = hk * kHeadDim;
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int D = c.D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;

    unsigned char *wp = wbase + warp * C::w_bytes;
    uint32_t *kst = reinterpret_cast<uint32_t *>(wp); wp += C::w_kst;
    int *kfix = reinterpret_cast<int *>(wp); wp += G * 32 * 4;
    float *ps = reinterpret_cast<float *>(kfix);
    float *osp = reinterpret_cast<float *>(wp); wp += G * kHeadDim * 4;
    // Value-outlier sums of the tile in fixed point (native shared integer atomics; sm_100a
    // has no native shared fp32 add), folded into osp at the end of the tile; during the K
    // phase the same words hold the fp32 side sums of the Key-outlier terms too large for
    // the 32-bit fixed point (kfix_add32)
    int *vfix = reinterpret_cast<int *>(wp); wp += G * kHeadDim * 4;
    float *kbig = reinterpret_cast<float *>(vfix);
    float2 *anc32 = reinterpret_cast<float2 *>(wp);

    const int t_first = t_begin + warp;
    uint32_t kitm[IPL], vitm[IPL];
    uint32_t cnt_k = 0, cnt_v = 0, ncnt_k = 0, ncnt_v = 0;
    float2 vsz = make_float2(0.f, 0.f);
    auto issue_k = [&](int t) {
        const unsigned char *src = reinterpret_cast<const unsigned char *>(c.kcodes + ((int64_t)t * c.QW + hk * KWH) * 32);
        const uint32_t dst = smem_u32(kst);
#pragma unroll
        for (int k = 0; k < C::KCH; ++k) cp_async16(dst + (uint32_t)(lane + 32 * k) * 16u, src + (lane + 32 * k) * 16);
    };
    auto load_counts = [&](int t, uint32_t &nk, uint32_t &nv) {
        nk = nv = 0;
        if (t < t_end) {
            const uint32_t *gc = c.gcnt + ((int64_t)t * c.NG + hk) * 2;
            nk = __ldg(gc);
            nv = __ldg(gc + 1);
        }
    };
    auto load_items = [&](int t) {
        const int64_t bucket = (int64_t)t * c.NG + hk;
        const uint32_t nk = cnt_k > (uint32_t)c.kcap_g ? 0u : cnt_k;
        const uint32_t nv = cnt_v > (uint32_t)c.vcap_g ? 0u : cnt_v;
#pragma unroll
        for (int k = 0; k < IPL; ++k) {
            const uint32_t x = lane + 32 * k;
            kitm[k] = x < nk ? __ldg(c.kit + bucket * c.kcap_g + x) : 0u;
            vitm[k] = x < nv ? __ldg(c.vit + bucket * c.vcap_g + x) : 0u;
        }
        vsz = (int64_t)t * 32 + lane < P.T ? __ldg(c.vsz + (int64_t)t * 32 + lane) : make_float2(0.f, 0.f);
    };

    // the first tile's K words and counts overlap the prologue unless the tile is the tail tile
    // (which a concurrent append may still be writing, see pdl_wait)
    const bool early = t_first < t_end && t_first != P.ntiles - 1;
    if (early) {
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ---------------------------------------------------------------- prologue (a1)
    // theta_i and the large-argument angles once per CTA (64 threads): cis(pos theta_i) for the
    // query, cis((pos_base + 32 t_begin) theta_i) for the CTA's first tile (R11, R12)
    if (tid < 64) {
        const int i = tid;
        const double th = c.theta_tab[i];
        th64[i] = th;
        double s, co;
        sincos(red2pi((double)P.pos * th), &s, &co);   // reduced first: fast-path sincos
        qcis[i] = make_double2(co, s);
    }
    __syncthreads();
    // token angles as in the MHA kernel: per warp and tile (anchor angle a_i mod 2 pi, th_i) fp32,
    // token j's cis from the MUFU at a_i + (j - 16) th_i
    double ang64[2], step64[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int i = lane + 32 * k;
        const double th = th64[i];
        ang64[k] = red2pi((double)(c.pos_base + (int64_t)t_first * kTileTokens + 16) * th);
        step64[k] = red2pi((double)(C::NWARP * kTileTokens) * th);
        anc32[i] = make_float2((float)ang64[k], (float)th);
    }
    for (int x = lane; x < G * 32; x += 32) kfix[x] = 0;
    for (int x = lane; x < G * kHeadDim; x += 32) { osp[x] = 0.f; vfix[x] = 0; }
    for (int x = tid; x < kHeadDim; x += NTHR) {
        ks_s[x] = c.kpar[c_lo + x];
        kz_s[x] = c.kpar[D + c_lo + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
    if (tid < 16) flag_s[tid] = 0;
    const double qscale = 1.4426950408889634 / sqrt((double)kHeadDim);
    for (int x = tid; x < G * 64; x += NTHR) {
        const int g = x >> 6, i = x & 63;
        const __half *qg = P.q + (int64_t)(g0 + g) * kHeadDim;
        const double co = qcis[i].x, s = qcis[i].y;
        const double a = (double)__half2float(qg[i]), b = (double)__half2float(qg[i + 64]);
        qs[g * kHeadDim + i] = (float)((a * co - b * s) * qscale);
        qs[g * kHeadDim + i + 64] = (float)((b * co + a * s) * qscale);
    }
    __syncthreads();
    for (int x = tid; x < G * 64; x += NTHR) {
        const int g = x >> 6, i = x & 63;
        const int ci = i, cj = i + 64;
        const float mx = fmaxf(fabsf(cbK[0] * ks_s[ci] + kz_s[ci]), fabsf(cbK[CM] * ks_s[ci] + kz_s[ci]));
        const float my = fmaxf(fabsf(cbK[0] * ks_s[cj] + kz_s[cj]), fabsf(cbK[CM] * ks_s[cj] + kz_s[cj]));
        const float qa = fabsf(qs[g * kHeadDim + i]), qb = fabsf(qs[g * kHeadDim + i + 64]);
        bound_s[x] = fmaxf(qa * mx + qb * my, qb * mx + qa * my);
    }
    __syncthreads();
    for (int g = warp; g < G; g += NWARP) {
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
            int e = 0;
            if (rest > 0.f && isfinite(rest)) e = 14 - ilogbf(rest) - 1;
            e = max(-100, min(100, e));
            lut_sc[g] = ldexpf(1.f, e);
            lut_inv[g] = ldexpf(1.f, -e);
        }
    }
    __syncthreads();
    // K table entries [i][pair code][g]: the G heads of a code adjacent (one vector load);
    // one entry per work item, consecutive threads on consecutive words (conflict-free stores)
    {
        const float *cbKsh = cb_s + 16;
        for (int x = tid; x < G * 64 * NE; x += NTHR) {
            const int g = x % G, rest = x / G;
            const int code = rest % NE, i = rest / NE;
            const int a = code & CM, bb = code >> BITS;
            const int gi = g * 64 + i;
            const float qa1 = qs[g * kHeadDim + i], qb1 = qs[g * kHeadDim + i + 64];
            const float xa = cbKsh[a] * ks_s[i] + kz_s[i];
            const float yb = cbKsh[bb] * ks_s[i + 64] + kz_s[i + 64];
            const float A = qa1 * xa + qb1 * yb, B = qb1 * xa - qa1 * yb;
            uint32_t e = 0u;
            if (heavy_s[gi] != 0) {
                int hslot = 0;
                for (int u = 0; u < hv_n[g]; ++u) hslot = hv_pair[g * 8 + u] == i ? u : hslot;
                hlut[(g * HMAX + hslot) * NE + code] = make_float2(A, B);
            } else {
                const float sc = lut_sc[g];
                e = pack_half2(A * sc, B * sc);
            }
            klut[x] = e;
        }
    }
    for (int x = tid; x < NE * 32; x += NTHR) {
        const int e = x >> 5;
        const float ca = cbV[e & CM], cb = cbV[e >> BITS];
        vlut[x] = pack_half2(ca, cb);
        if constexpr (RESID)
            vlut[NE * 32 + x] = pack_half2(ca - __half2float(__float2half_rn(ca)), cb - __half2float(__float2half_rn(cb)));
    }
    __syncthreads();

    pdl_wait();
    if (t_first < t_end && !early) {
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ================================================================ tile loop (per warp)
    const uint32_t klut_u = opaque(smem_u32(klut));
    const uint32_t vlut_u = opaque(smem_u32(vlut) | (4u * lane));
    const int vg = lane >> 2, vt = lane & 3;
    const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
    // P.V accumulators (mma D fragments): column 2vt + (0|1) = query head, rows vg, vg + 8 of
    // m-tile ml; units 2^(E - WEXP) relative to the head's running max
    float dacc[8][4];
#pragma unroll
    for (int ml = 0; ml < 8; ++ml) dacc[ml][0] = dacc[ml][1] = dacc[ml][2] = dacc[ml][3] = 0.f;
    float m_run[G], l_lane[G], z_lane[G];
#pragma unroll
    for (int g = 0; g < G; ++g) { m_run[g] = -CUDART_INF_F; l_lane[g] = 0.f; z_lane[g] = 0.f; }
    int E_run = -126;
    // D columns 2t, 2t+1 of lane (g, t) are head t's hi and lo weight sums
    const int hcl = min(vt, G - 1);
    auto rot32 = [&](int i, int j, float &co, float &si) {
        const float2 a = anc32[i];
        __sincosf(fmaf((float)(j - 16), a.y, a.x), &si, &co);
    };
    auto rot16 = [&](int i) -> uint32_t {
        float co, si;
        rot32(i, lane, co, si);
        return pack_half2(co, si);
    };

    for (int t = t_first; t < t_end; t += C::NWARP) {
        const int64_t n0 = (int64_t)t * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        const bool valid = lane < ntok;
        const bool kov = cnt_k > (uint32_t)c.kcap_g, vov = cnt_v > (uint32_t)c.vcap_g;
        const int nk = kov ? 0 : (int)cnt_k, nv = vov ? 0 : (int)cnt_v;
        load_items(t);
        load_counts(t + C::NWARP, ncnt_k, ncnt_v);
        uint32_t vw[KWH];
#pragma unroll
        for (int w = 0; w < KWH; ++w) vw[w] = __ldg(c.vcodes + vf_word(t, c.H_kv, hk, w, lane, BITS));

        cp_async_wait_all();
        __syncwarp();
        uint32_t kw[KWH];
#pragma unroll
        for (int w = 0; w < KWH; ++w) kw[w] = kst[w * 32 + lane];

        // ---------------------------------------------------------- a2: K dense
        float acc_c[G], acc_s[G];
#pragma unroll
        for (int g = 0; g < G; ++g) { acc_c[g] = 0.f; acc_s[g] = 0.f; }
#pragma unroll
        for (int i = 0; i < kPairs; ++i) {
            const uint32_t cs = rot16(i);   // fp32 rotation rounded once
            const int bit = FB * i, w = bit >> 5, sh = bit & 31;
            // (pair code << 2) << log2(G): the G heads' entries of a code are adjacent
            uint32_t off;
            if (sh + FB <= 32) off = sh >= 2 + LG ? (kw[w] >> (sh - 2 - LG)) : (kw[w] << (2 + LG - sh));
            else off = __funnelshift_r(kw[w], kw[w + 1], sh - 2 - LG);
            const uint32_t a = klut_u | (off & ((NE - 1) << (2 + LG)));
            uint32_t ab[G];
            lds_vecG<G>(a + (uint32_t)(i * NE * 4 * G), ab);
#pragma unroll
            for (int g = 0; g < G; ++g) fma2_f16_f32(ab[g], cs, acc_c[g], acc_s[g]);
        }
        __syncwarp();

        // -------------------------------------------- a3: heavy pairs, Key outliers (fp32)
        // heavy pairs of each head (fp32 tables, fp32 rotation)
        float sco[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float hs = 0.f;
            const int nh = hv_n[g];
            for (int u = 0; u < nh; ++u) {
                const int i = hv_pair[g * 8 + u];
                const int bit = FB * i;
                const int wq = bit >> 5;
                unsigned long long w64 = kst[wq * 32 + lane];
                if ((bit & 31) + FB > 32) w64 |= (unsigned long long)kst[(wq + 1) * 32 + lane] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                const float2 ab = hlut[(g * HMAX + u) * NE + pc];
                float co, si;
                rot32(i, lane, co, si);
                hs += co * ab.x + si * ab.y;
            }
            sco[g] = (acc_c[g] + acc_s[g]) * lut_inv[g] + hs;
        }
        // item -> the G heads' corrections (x - K^(code)) * dscore/dK
        auto k_item = [&](uint32_t itm) {
            const int j = (int)((itm >> 11) & 31u);
            const int cc = (int)(itm & 0x7fu), flag = (int)((itm >> 9) & 3u);
            const int i = cc & 63, up = cc >> 6;
            int code = flag == 1 ? CM : 0;
            if (flag == 0) {
                const int bit = FB * i;
                const int wq = bit >> 5;
                unsigned long long w64 = kst[wq * 32 + j];
                if ((bit & 31) + FB > 32) w64 |= (unsigned long long)kst[(wq + 1) * 32 + j] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                code = (pc >> (up * BITS)) & CM;
            }
            const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
            const float delta = xval - (cbKs[code] * ks_s[cc] + kz_s[cc]);
            float co, si;
            rot32(i, j, co, si);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float qa = qs[g * kHeadDim + i], qb = qs[g * kHeadDim + i + 64];
                kfix_add32(&kfix[g * 32 + j], &kbig[g * 32 + j], delta * (up ? (qb * co - qa * si) : (qa * co + qb * si)));
            }
        };
        {
            const int64_t bucket = (int64_t)t * c.NG + hk;
#pragma unroll
            for (int k = 0; k < IPL; ++k)
                if (32 * k < nk && lane + 32 * k < nk) k_item(kitm[k]);
            for (int x = 32 * IPL + lane; x < nk; x += 32) k_item(__ldg(c.kit + bucket * c.kcap_g + x));
            if (kov) {
                for (int j = 0; j < ntok; ++j) {
                    const uint32_t r0 = __ldg(c.kptr + n0 + j), r1 = __ldg(c.kptr + n0 + j + 1);
                    for (uint32_t r = r0 + lane; r < r1; r += 32) {
                        const uint32_t rec = __ldcg(c.kout + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < c_lo || ch >= c_lo + kHeadDim) continue;
                        k_item((rec & 0xffff0000u) | ((uint32_t)j << 11) | (uint32_t)(ch - c_lo));
                    }
                }
            }
        }
        __syncwarp();
        const int tn = t + C::NWARP;
        if (tn < t_end) issue_k(tn);

        // ------------------------------------------------------ a4: online softmax
        // weights p s_n 2^(WEXP - E), E the running exponent bound of s_n (the accumulators
        // persist across tiles)
        const float smax = warp_max_redux(valid ? vsz.x : 0.f);
        const int E_new = smax > 0.f ? max(E_run, ilog2f(smax) + 1) : E_run;
        const float pe = pow2i(WEXP - E_new), rE = pow2i(E_run - E_new);
        E_run = E_new;
        uint32_t w2s[G], w2l[G];
        float al[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float s = sco[g] + (float)kfix[g * 32 + lane] * (1.f / kKfixScale) + kbig[g * 32 + lane];
            kbig[g * 32 + lane] = 0.f;   // the words are the V-outlier sums from here on
            s = valid ? s : -CUDART_INF_F;
            const float m_new = fmaxf(m_run[g], warp_max_redux(s));
            const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run[g] - m_new);
            const float p = valid ? exp2f(s - m_new) : 0.f;
            l_lane[g] = l_lane[g] * alpha + p;
            z_lane[g] = z_lane[g] * alpha + p * vsz.y;
            m_run[g] = m_new;
            al[g] = alpha;
            if (alpha != 1.f) {   // warp-uniform
#pragma unroll
                for (int x = 0; x < kHeadDim / 32; ++x) osp[g * kHeadDim + x * 32 + lane] *= alpha;
            }
            ps[g * 32 + lane] = p;
            const float wf = p * (vsz.x * pe);
            const __half wh = __float2half_rn(wf);
            const uint32_t hb = __half_as_ushort(wh), lb = __half_as_ushort(__float2half_rn(wf - __half2float(wh)));
            w2s[g] = hb | (__shfl_down_sync(0xffffffffu, hb, 1) << 16);
            w2l[g] = lb | (__shfl_down_sync(0xffffffffu, lb, 1) << 16);
        }
        {   // rescale the accumulators: per column (head) alpha, and the weight exponent
            float a0 = al[0];
#pragma unroll
            for (int g = 1; g < G; ++g) a0 = hcl == g ? al[g] : a0;
            a0 *= rE;
            const float a1 = a0;
            if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
                for (int ml = 0; ml < 8; ++ml) {
                    dacc[ml][0] *= a0; dacc[ml][2] *= a0;
                    dacc[ml][1] *= a1; dacc[ml][3] *= a1;
                }
            }
        }
        // B fragments: column vg = query head vg / 2, its hi (vg even) or lo (vg odd) weight
        // part; tokens 16 s2 + 2 vt (+1) and + 8
        uint32_t bw[2][2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t v = 0u;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t xh = __shfl_sync(0xffffffffu, w2s[g], 16 * s2 + 2 * vt + 8 * r);
                    const uint32_t xl = __shfl_sync(0xffffffffu, w2l[g], 16 * s2 + 2 * vt + 8 * r);
                    v = (vg >> 1) == g ? ((vg & 1) ? xl : xh) : v;
                }
                bw[s2][r] = v;
            }

        // --------------------------------------------------------- a5: P.V dense
#pragma unroll
        for (int ml = 0; ml < 8; ++ml) {
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                uint32_t a[4], alo[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int bit = ((ml * 2 + s2) * 4 + r) * FB;
                    const int wi = bit >> 5, sh = bit & 31;
                    uint32_t off;
                    if (sh + FB <= 32) off = sh >= 7 ? (vw[wi] >> (sh - 7)) : (vw[wi] << (7 - sh));
                    else off = __funnelshift_r(vw[wi], vw[wi + 1], sh - 7);
                    const uint32_t ad = vlut_u | (off & ((NE - 1) << 7));
                    a[r] = lds_u32(ad);
                    if constexpr (RESID) alo[r] = lds_u32(ad + NE * 32 * 4);
                }
                mma_f16_f32(dacc[ml], a, bw[s2]);
                if constexpr (RESID) mma_f16_f32(dacc[ml], alo, bw[s2]);
            }
        }

        // ------------------------------------------------------ a6: V outliers
        // p_g (x - V^(code)) of every item for the G heads, summed in fixed point (scale from
        // the tile's largest |term|) with native shared integer atomics, folded into osp
        __syncwarp();
        if (nv > 0 || vov) {
            // item -> (channel, delta); the G terms are ps[g][j] * delta
            auto v_delta = [&](uint32_t itm, bool act, int &j, int &cc) -> float {
                j = (int)((itm >> 11) & 31u);
                cc = (int)(itm & 0x7fu);
                const int flag = (int)((itm >> 9) & 3u);
                int code = flag == 1 ? CM : 0;
                if (act && flag == 0) {
                    const int bit = vf_bit(j, cc, BITS);
                    const uint32_t *wq = c.vcodes + vf_word(t, c.H_kv, hk, bit >> 5, vf_lane(j, cc), BITS);
                    unsigned long long w64 = __ldg(wq);
                    if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)__ldg(wq + 32) << 32;
                    code = (int)((w64 >> (bit & 31)) & CM);
                }
                const float s_n = __shfl_sync(0xffffffffu, vsz.x, j), z_n = __shfl_sync(0xffffffffu, vsz.y, j);
                const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                return act ? xval - (cbVs[code] * s_n + z_n) : 0.f;
            };
            const int64_t bucket = (int64_t)t * c.NG + hk;
            // the items beyond the registers (rare): x0 + lane for x0 >= 32 IPL, then (overflowed
            // bucket) every CSR record of the tile's tokens in this KV head
            const int kvn = c.kv;
            const int x_beg = vov ? 0 : 32 * IPL;
            const int x_end = (vov ? ntok * kvn : 0) + nv;
            auto slow_item = [&](int x0, int &j, int &cc) -> float {
                uint32_t itm = 0u;
                bool act = false;
                if (x0 < nv) {
                    act = x0 + lane < nv;
                    itm = act ? __ldg(c.vit + bucket * c.vcap_g + x0 + lane) : 0u;
                } else {
                    const int r = x0 - nv + lane;
                    act = r < ntok * kvn;
                    if (act) {
                        const uint32_t rec = __ldcg(c.vout + n0 * kvn + r);
                        const int ch = (int)(rec & 0xffffu);
                        act = ch >= c_lo && ch < c_lo + kHeadDim;
                        itm = (rec & 0xffff0000u) | ((uint32_t)(r / kvn) << 11) | (uint32_t)(act ? ch - c_lo : 0);
                    }
                }
                return v_delta(itm, act, j, cc);
            };
            const bool slow = nv > 32 * IPL || vov;
            float dl[IPL];
            int jx[IPL], cx[IPL];
            float pmax = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) pmax = fmaxf(pmax, ps[g * 32 + lane]);
            pmax = warp_max(pmax);   // every term is <= pmax |delta|
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < IPL; ++k) {
                dl[k] = 0.f; jx[k] = 0; cx[k] = 0;
                if (32 * k < nv && !vov) dl[k] = v_delta(vitm[k], lane + 32 * k < nv, jx[k], cx[k]);
                mx = fmaxf(mx, fabsf(dl[k]));
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    mx = fmaxf(mx, fabsf(slow_item(x0, j, cc)));
                }
            mx = warp_max(mx) * pmax;
            const int emx = mx > 0.f ? ilog2f(mx) : 0;
            const float S = pow2i(24 - emx);
            auto add = [&](float d, int j, int cc) {
                if (d == 0.f) return;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float v = ps[g * 32 + j] * d;
                    if (v != 0.f) atomicAdd(&vfix[g * kHeadDim + cc], __float2int_rn(v * S));
                }
            };
            if (!vov) {
#pragma unroll
                for (int k = 0; k < IPL; ++k) add(dl[k], jx[k], cx[k]);
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    const float d = slow_item(x0, j, cc);
                    add(d, j, cc);
                }
            __syncwarp();
            // fold only the entries this tile touched: the lanes re-walk their items and the
            // first to exchange an entry adds it (the others get 0)
            const float inv = pow2i(emx - 24);
            auto fold = [&](float d, int cc) {
                if (d == 0.f) return;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int v = atomicExch(&vfix[g * kHeadDim + cc], 0);
                    if (v) osp[g * kHeadDim + cc] += (float)v * inv;
                }
            };
            if (!vov) {
#pragma unroll
                for (int k = 0; k < IPL; ++k) fold(dl[k], cx[k]);
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    const float d = slow_item(x0, j, cc);
                    fold(d, cc);
                }
            __syncwarp();
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) kfix[g * 32 + lane] = 0;

#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            ang64[k] = red2pi(ang64[k] + step64[k]);
            anc32[i].x = (float)ang64[k];
        }
        cnt_k = ncnt_k;
        cnt_v = ncnt_v;
        __syncwarp();
    }

    // ------------------------------------------- warp partials -> CTA partial (a7)
    cp_async_wait_all();
    __syncwarp();
    // osp (V-outlier sums, real units) += the dense accumulators of the lane's columns
    {
        const float sc = pow2i(E_run - WEXP);
#pragma unroll
        for (int ml = 0; ml < 8; ++ml) {
            const int ch = ml * 16 + vg;
            if (vt < G) {
                osp[vt * kHeadDim + ch] += (dacc[ml][0] + dacc[ml][1]) * sc;
                osp[vt * kHeadDim + ch + 8] += (dacc[ml][2] + dacc[ml][3]) * sc;
            }
        }
    }
    __syncwarp();
    float *wpart = reinterpret_cast<float *>(osp);   // in place: [G][d] o, then m, l in kst
    float *wml = reinterpret_cast<float *>(kst);     // [G][2]
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float l = warp_sum(l_lane[g]), z = warp_sum(z_lane[g]);
#pragma unroll
        for (int x = 0; x < kHeadDim / 32; ++x) wpart[g * kHeadDim + x * 32 + lane] += z;
        if (lane == 0) { wml[g * 2] = m_run[g]; wml[g * 2 + 1] = l; }
    }
    __syncthreads();
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    for (int x = tid; x < G * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int w = 0; w < NWARP; ++w) {
            const float *ml = reinterpret_cast<const float *>(wbase + w * C::w_bytes) + g * 2;
            if (ml[1] != 0.f) m = fmaxf(m, ml[0]);
        }
        float l = 0.f, o = 0.f;
        for (int w = 0; w < NWARP; ++w) {
            const float *ml = reinterpret_cast<const float *>(wbase + w * C::w_bytes) + g * 2;
            if (ml[1] == 0.f) continue;
            const float wt = exp2f(ml[0] - m);
            l += wt * ml[1];
            if (ch < kHeadDim) {
                const float *ow = reinterpret_cast<const float *>(wbase + w * C::w_bytes + C::w_kst + G * 32 * 4);
                o += wt * ow[g * kHeadDim + ch];
            }
        }
        part[(g0 + g) * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
    }
    __threadfence();
    __syncthreads();
    int *s_last = flag_s + 1;
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.tickets[hk], 1u);
        *s_last = (prev == (unsigned)(P.S - 1));
    }
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    for (int x = tid; x < G * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        const int gq = g0 + g;
        // the S partials in chunks of 8 independent L2 loads (one round trip per chunk, not per
        // split: the merge runs after every other CTA of the head group has finished)
        constexpr int MC = 8;
        const float *pbase = P.parts + (int64_t)gq * (kHeadDim + 2);
        const int64_t pstride = (int64_t)c.H_q * (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : -CUDART_INF_F;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k)
                if (lv[k] != 0.f) m = fmaxf(m, mv[k]);
        }
        float l = 0.f, o = 0.f;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC], ov[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : 0.f;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
                ov[k] = (in && ch < kHeadDim) ? __ldcg(ps2 + ch) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k) {   // fixed split order, as before
                if (lv[k] == 0.f) continue;
                const float wgt = exp2f(mv[k] - m);
                l += wgt * lv[k];
                if (ch < kHeadDim) o += wgt * ov[k];
            }
        }
        if (P.write_partial) {
            P.out[gq * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
        } else if (ch < kHeadDim) {
            P.out[gq * kHeadDim + ch] = o / l;
        }
    }
    if (tid == 0) P.tickets[hk] = 0;
}

template <int BITS, bool RESID, int G>
cudaError_t launch_wag_t(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    using C = GCfg<BITS, RESID, G>;
    static_assert(C::total <= 227 * 1024, "shared memory");
    cudaError_t e = cudaFuncSetAttribute(att_wag_kernel<BITS, RESID, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    e = launch_maybe_pdl(att_wag_kernel<BITS, RESID, G>, grid, C::NTHR, C::total, s, P.pdl != 0, c, P);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
template <int BITS, bool RESID>
cudaError_t launch_wag_g(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    return c.G == 2 ? launch_wag_t<BITS, RESID, 2>(c, P, grid, s) : launch_wag_t<BITS, RESID, 4>(c, P, grid, s);
}


// ===================================================================================
// GQA with the K scores on the tensor cores: att_wgt_kernel.  Same structure as att_wag_kernel
// (one CTA per (KV head, split), 16 warps = 16 tile streams, every outlier item corrects the G
// heads, P.V on mma with persistent accumulators), but the K scores are a dense contraction
// here, so they run on mma.m16n8k16: A = RoPE(K^) of 16 tokens x 8 pairs, dequantized and
// rotated in fp32 and split into fp16 hi + lo (two mma), B = the G queries as fp16 hi / lo
// columns.  The products are exact and the sums fp32, so the scores are fp32-accurate and there
// is no heavy-pair pass; the Key codebook lookups are lane-private (conflict-free), the K-word
// reads swizzled (4 blocks -> 4 bank octets).
template <int WB>
__device__ __forceinline__ int kst_swz(int q, int j) {
    return q * 32 + (j ^ (8 * ((q / WB) & 3)));
}
// padded per-pair tables: the 4 lanes of a column read pairs 16 t + x (t = 0..3), which would
// share banks at a 16-entry stride
__device__ __forceinline__ int kpad(int p) { return p + (p >> 4); }        // 16-byte entries
__device__ __forceinline__ int apad(int p) { return p + 2 * (p >> 4); }    // 8-byte entries

#ifndef WGT_NW
#define WGT_NW 16
#endif
template <int BITS, bool RESID, int G>
struct TCfg {
    static_assert(G <= 4 || G == 8, "G <= 4: hi / lo query columns; G = 8: hi and lo B fragments");
    static constexpr int NWARP = G == 8 ? 12 : WGT_NW;   // G = 8: [8][128] outlier sums per warp
    static constexpr int NTHR = NWARP * 32;
    static constexpr int IPL = 4;
    static constexpr int NE = 1 << (2 * BITS);
    static constexpr int KWH = 4 * BITS;
    static constexpr size_t cpt = (size_t)NE * 32 * 8;    // lane-private (cb[a], cb[b]) fp32
    static constexpr size_t vlut = (size_t)(RESID ? 2 : 1) * NE * 32 * 4;
    static constexpr size_t valign = (size_t)NE * 32 * 4;
    // 2-3 bits: the codebook pair table first, aligned to its size (OR addressing), the V table
    // after it (aligned too); 4 bits (64 KB pair table, 32 KB V table): byte-aligned codes, PRMT +
    // add addressing, no alignment
    static constexpr size_t calign = BITS == 4 ? 16 : cpt;
    static_assert(BITS == 4 || cpt % valign == 0, "V table follows aligned");
    static_assert(BITS < 4 || !RESID, "4-bit GQA: fp16-exact Value decode codebook only");
    // per warp: K words (cp.async target, swizzled), K-outlier terms (then p) [G][32], V-outlier
    // sums fp32 [G][128] and fixed point [G][128], anchors, scores [G][32]
    static constexpr size_t w_kst = (size_t)KWH * 32 * 4;
    static constexpr size_t w_bytes = w_kst + G * 32 * 4 + G * kHeadDim * 4 * 2 + 72 * 8 + G * 32 * 4;
    static constexpr int KCH = KWH / 4;
    static constexpr size_t small = 68 * 16 /* kaf */ + 8 * 32 * 16 /* bqs */ + G * kHeadDim * 4 /* qs */ + kHeadDim * 4 * 2 /* ks, kz */
        + 64 * 4 /* cb */ + 64 /* flags */ + 64 * 16 /* cis(pos theta) */ + 64 * 8 /* theta */;
    static constexpr size_t total = calign + cpt + vlut + NWARP * w_bytes + small;
};

template <int BITS, bool RESID, int G>
__device__ __forceinline__ void att_wgt_body(const DevCache &c, const WParams &P, const int blk) {
    using C = TCfg<BITS, RESID, G>;
    constexpr int NWARP = C::NWARP, NTHR = C::NTHR, IPL = C::IPL;
    constexpr int NE = C::NE;
    constexpr int CM = (1 << BITS) - 1;
    constexpr int KWH = C::KWH;
    constexpr int FB = 2 * BITS;
    constexpr int WB = FB / 2;   // K words per 16-pair block

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // the lane-private codebook pair table first, at a multiple of its size (OR addressing),
    // then the V table (also aligned), then the per-warp regions and the small arrays
    const uint32_t s0 = smem_u32(smem_raw);
    unsigned char *sp = smem_raw + ((C::calign - (s0 % C::calign)) % C::calign);
    float2 *cpt;
    uint32_t *vlut;
    if constexpr (BITS == 4) {
        vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
        cpt = reinterpret_cast<float2 *>(sp); sp += C::cpt;
    } else {
        cpt = reinterpret_cast<float2 *>(sp); sp += C::cpt;
        vlut = reinterpret_cast<uint32_t *>(sp); sp += C::vlut;
    }
    unsigned char *wbase = sp; sp += NWARP * C::w_bytes;
    float4 *kaf = reinterpret_cast<float4 *>(sp); sp += 68 * 16;   // pair p at p + (p >> 4)
    uint4 *bqs = reinterpret_cast<uint4 *>(sp); sp += 8 * 32 * 16;   // score-mma B fragments [s][lane]
    constexpr bool G8 = G == 8;   // 8 query heads: columns = heads, hi and lo as two B fragments
    float *qs = reinterpret_cast<float *>(sp); sp += G * kHeadDim * 4;
    float *ks_s = reinterpret_cast<float *>(sp); sp += kHeadDim * 4;
    float *kz_s = reinterpret_cast<float *>(sp); sp += kHeadDim * 4;
    float *cb_s = reinterpret_cast<float *>(sp); sp += 64 * 4;
    int *flag_s = reinterpret_cast<int *>(sp); sp += 64;
    double2 *qcis = reinterpret_cast<double2 *>(sp); sp += 64 * 16;
    double *th64 = reinterpret_cast<double *>(sp); sp += 64 * 8;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // one CTA per (KV head, sub-group of G of its c.G query heads, split): G = 8 (LLaMA-2-70B)
    // runs as two sub-groups of 4 that read the same K / V words
    const int n_sub = c.G / G;
    const int n_hg = c.H_kv * n_sub;
    const int hgi = blk % n_hg;
    const int hk = hgi / n_sub;
    const int split = blk / n_hg;
    const int g0 = hk * c.G + (hgi % n_sub) * G;     // first query head of the CTA
    const int c_lo = hk * kHeadDim;
    const int t_begin = (int)((int64_t)split * P.ntiles / P.S);
    const int t_end = (int)((int64_t)(split + 1) * P.ntiles / P.S);
    const int D = c.D;
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;

    unsigned char *wp = wbase + warp * C::w_bytes;
    uint32_t *kst = reinterpret_cast<uint32_t *>(wp); wp += C::w_kst;
    int *kfix = reinterpret_cast<int *>(wp); wp += G * 32 * 4;
    float *ps = reinterpret_cast<float *>(kfix);
    float *osp = reinterpret_cast<float *>(wp); wp += G * kHeadDim * 4;
    // Value-outlier sums of the tile in fixed point (native shared integer atomics; sm_100a
    // has no native shared fp32 add), folded into osp at the end of the tile; during the K
    // phase the same words hold the fp32 side sums of the Key-outlier terms too large for
    // the 32-bit fixed point (kfix_add32)
    int *vfix = reinterpret_cast<int *>(wp); wp += G * kHeadDim * 4;
    float *kbig = reinterpret_cast<float *>(vfix);
    float2 *anc32 = reinterpret_cast<float2 *>(wp); wp += 72 * 8;   // pair p at p + 2 (p >> 4)
    float *sct = reinterpret_cast<float *>(wp);   // [G][32] scores of the tile (tensor cores)

    const int t_first = t_begin + warp;
    uint32_t kitm[IPL], vitm[IPL];
    uint32_t cnt_k = 0, cnt_v = 0, ncnt_k = 0, ncnt_v = 0;
    float2 vsz = make_float2(0.f, 0.f);
    auto issue_k = [&](int t) {
        const unsigned char *src = reinterpret_cast<const unsigned char *>(c.kcodes + ((int64_t)t * c.QW + hk * KWH) * 32);
        const uint32_t dst = smem_u32(kst);
#pragma unroll
        for (int k = 0; k < C::KCH; ++k) {
            const int x = lane + 32 * k;   // 16-byte chunk: word x / 8, tokens 4 (x % 8) ..
            cp_async16(dst + (uint32_t)kst_swz<WB>(x >> 3, (x & 7) * 4) * 4u, src + x * 16);
        }
    };
    auto load_counts = [&](int t, uint32_t &nk, uint32_t &nv) {
        nk = nv = 0;
        if (t < t_end) {
            const uint32_t *gc = c.gcnt + ((int64_t)t * c.NG + hk) * 2;
            nk = __ldg(gc);
            nv = __ldg(gc + 1);
        }
    };
    auto load_items = [&](int t) {
        const int64_t bucket = (int64_t)t * c.NG + hk;
        const uint32_t nk = cnt_k > (uint32_t)c.kcap_g ? 0u : cnt_k;
        const uint32_t nv = cnt_v > (uint32_t)c.vcap_g ? 0u : cnt_v;
#pragma unroll
        for (int k = 0; k < IPL; ++k) {
            const uint32_t x = lane + 32 * k;
            kitm[k] = x < nk ? __ldg(c.kit + bucket * c.kcap_g + x) : 0u;
            vitm[k] = x < nv ? __ldg(c.vit + bucket * c.vcap_g + x) : 0u;
        }
        vsz = (int64_t)t * 32 + lane < P.T ? __ldg(c.vsz + (int64_t)t * 32 + lane) : make_float2(0.f, 0.f);
    };

    // the first tile's K words and counts overlap the prologue unless the tile is the tail tile
    // (which a concurrent append may still be writing, see pdl_wait)
    const bool early = t_first < t_end && t_first != P.ntiles - 1;
    if (early) {
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ---------------------------------------------------------------- prologue (a1)
    // theta_i and the large-argument angles once per CTA (64 threads): cis(pos theta_i) for the
    // query, cis((pos_base + 32 t_begin) theta_i) for the CTA's first tile (R11, R12)
    if (tid < 64) {
        const int i = tid;
        const double th = c.theta_tab[i];
        th64[i] = th;
        double s, co;
        sincos(red2pi((double)P.pos * th), &s, &co);   // reduced first: fast-path sincos
        qcis[i] = make_double2(co, s);
    }
    __syncthreads();
    // token angles as in the MHA kernel: per warp and tile (anchor angle a_i mod 2 pi, th_i) fp32,
    // token j's cis from the MUFU at a_i + (j - 16) th_i
    double ang64[2], step64[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int i = lane + 32 * k;
        const double th = th64[i];
        ang64[k] = red2pi((double)(c.pos_base + (int64_t)t_first * kTileTokens + 16) * th);
        step64[k] = red2pi((double)(C::NWARP * kTileTokens) * th);
        anc32[apad(i)] = make_float2((float)ang64[k], (float)th);
    }
    for (int x = lane; x < G * 32; x += 32) kfix[x] = 0;
    for (int x = lane; x < G * kHeadDim; x += 32) { osp[x] = 0.f; vfix[x] = 0; }
    for (int x = tid; x < kHeadDim; x += NTHR) {
        ks_s[x] = c.kpar[c_lo + x];
        kz_s[x] = c.kpar[D + c_lo + x];
    }
    if (tid < 64) cb_s[tid] = c.cb[tid];
    if (tid < 16) flag_s[tid] = 0;
    const double qscale = 1.4426950408889634 / sqrt((double)kHeadDim);
    for (int x = tid; x < G * 64; x += NTHR) {
        const int g = x >> 6, i = x & 63;
        const __half *qg = P.q + (int64_t)(g0 + g) * kHeadDim;
        const double co = qcis[i].x, s = qcis[i].y;
        const double a = (double)__half2float(qg[i]), b = (double)__half2float(qg[i + 64]);
        qs[g * kHeadDim + i] = (float)((a * co - b * s) * qscale);
        qs[g * kHeadDim + i + 64] = (float)((b * co + a * s) * qscale);
    }
    __syncthreads();
    // Key dequantization tables: the lane-private pair table (cb[a], cb[b]) of every pair code
    // (entry e of lane l at e * 32 + l: conflict-free), and per RoPE pair the two channels'
    // (s, s', z, z') scaled by 2^-4 (A operand range)
    for (int x = tid; x < NE * 32; x += NTHR) {
        const int e = x >> 5;
        cpt[x] = make_float2(cbK[e & CM], cbK[e >> BITS]);
    }
    if (tid < 64) {
        const int i = tid;
        kaf[kpad(i)] = make_float4(ks_s[i] * 0.0625f, ks_s[i + 64] * 0.0625f, kz_s[i] * 0.0625f, kz_s[i + 64] * 0.0625f);
    }
    for (int x = tid; x < NE * 32; x += NTHR) {
        const int e = x >> 5;
        const float ca = cbV[e & CM], cb = cbV[e >> BITS];
        vlut[x] = pack_half2(ca, cb);
        if constexpr (RESID)
            vlut[NE * 32 + x] = pack_half2(ca - __half2float(__float2half_rn(ca)), cb - __half2float(__float2half_rn(cb)));
    }
    __syncthreads();

    pdl_wait();
    if (t_first < t_end && !early) {
        issue_k(t_first);
        load_counts(t_first, cnt_k, cnt_v);
    }

    // ================================================================ tile loop (per warp)
    const uint32_t vlut_u = BITS == 4 ? smem_u32(vlut) + 4u * lane : opaque(smem_u32(vlut) | (4u * lane));
    const uint32_t cpt_u = BITS == 4 ? smem_u32(cpt) + 8u * lane : opaque(smem_u32(cpt) | (8u * lane));
    const int vg = lane >> 2, vt = lane & 3;
    // B fragments of the score mma (constant): column vg = q~ of head vg (fp16 hi part) or of
    // head vg - 4 (lo part); k = 2 slot + (0: channel p, 1: channel p + 64); lane (vg, vt)
    // holds slot vt (pair 16 vt + 2 s) and slot vt + 4 (pair 16 vt + 2 s + 1) of k-step s
    // (a CTA-wide table in shared memory, one 8-byte load per k-step; written by warp 0)
    if (warp == 0) {
        const int hq = G8 ? vg : (vg < 4 ? vg : vg - 4);
#pragma unroll 1
        for (int s = 0; s < 8; ++s) {
            uint32_t v[2], vl[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int p = 16 * vt + 2 * s + j;
                v[j] = vl[j] = 0u;
                if (hq < G) {
                    const float qa = qs[hq * kHeadDim + p], qb = qs[hq * kHeadDim + p + 64];
                    const float ha = __half2float(__float2half_rn(qa)), hb = __half2float(__float2half_rn(qb));
                    if (G8) { v[j] = pack_half2(ha, hb); vl[j] = pack_half2(qa - ha, qb - hb); }
                    else v[j] = vg < 4 ? pack_half2(ha, hb) : pack_half2(qa - ha, qb - hb);
                }
            }
            bqs[s * 32 + lane] = make_uint4(v[0], v[1], vl[0], vl[1]);
        }
    }
    __syncthreads();
    const float *cbKs = cb_s + 16, *cbVs = cb_s + 48;
    // P.V accumulators (mma D fragments): column 2vt + (0|1) = query head, rows vg, vg + 8 of
    // m-tile ml; units 2^(E - WEXP) relative to the head's running max
    float dacc[8][4];
#pragma unroll
    for (int ml = 0; ml < 8; ++ml) dacc[ml][0] = dacc[ml][1] = dacc[ml][2] = dacc[ml][3] = 0.f;
    float m_run[G], l_lane[G], z_lane[G];
#pragma unroll
    for (int g = 0; g < G; ++g) { m_run[g] = -CUDART_INF_F; l_lane[g] = 0.f; z_lane[g] = 0.f; }
    int E_run = -126;
    // D columns 2t, 2t+1 of lane (g, t) are head t's hi and lo weight sums
    const int hcl = min(vt, G - 1);
    auto rot32 = [&](int i, int j, float &co, float &si) {
        const float2 a = anc32[apad(i)];
        __sincosf(fmaf((float)(j - 16), a.y, a.x), &si, &co);
    };
    auto rot16 = [&](int i) -> uint32_t {
        float co, si;
        rot32(i, lane, co, si);
        return pack_half2(co, si);
    };

    for (int t = t_first; t < t_end; t += C::NWARP) {
        const int64_t n0 = (int64_t)t * 32;
        const int ntok = (int)min((int64_t)32, P.T - n0);
        const bool valid = lane < ntok;
        const bool kov = cnt_k > (uint32_t)c.kcap_g, vov = cnt_v > (uint32_t)c.vcap_g;
        const int nk = kov ? 0 : (int)cnt_k, nv = vov ? 0 : (int)cnt_v;
        load_items(t);
        load_counts(t + C::NWARP, ncnt_k, ncnt_v);
        {   // this tile's V words (4b * 128 B) -> L2; read after the K scores
            const char *vb = reinterpret_cast<const char *>(c.vcodes + vf_word(t, c.H_kv, hk, 0, 0, BITS));
            if (lane < 4 * BITS) asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + lane * 128));
        }

        cp_async_wait_all();
        __syncwarp();
        // ---------------------------------------------------------- a2: K scores (tensor cores)
        // A = RoPE(K^_n) of the tile (rows = tokens, k = the pairs' two channels), dequantized
        // and rotated in fp32 and split into fp16 hi + lo (two mma), B = the G queries (hi / lo
        // columns): fp32-exact scores, no heavy-pair pass.  Lane (g, t) converts tokens
        // g + 8 m (m = 0..3) at the 16 pairs of block t.
        float dsc[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) dsc[mt][0] = dsc[mt][1] = dsc[mt][2] = dsc[mt][3] = 0.f;
        {
            uint32_t kwd[4][WB + 1];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
#pragma unroll
                for (int k = 0; k < WB; ++k) kwd[m][k] = kst[kst_swz<WB>(vt * WB + k, vg + 8 * m)];
                kwd[m][WB] = 0u;
            }
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int off = 2 * s * FB, wi = off >> 5, sh = off & 31;
                float4 af[2];
                float2 an[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    af[j] = kaf[kpad(16 * vt + 2 * s + j)];
                    an[j] = anc32[apad(16 * vt + 2 * s + j)];
                }
                uint32_t ahi[2][4], alo[2][4];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const uint32_t f = (sh + 2 * FB <= 32) ? (kwd[m][wi] >> sh) : __funnelshift_r(kwd[m][wi], kwd[m][wi + 1], sh);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        uint32_t ad;
                        if constexpr (BITS == 4) {   // byte j of the field, times 256, plus the lane base
                            uint32_t cj;
                            asm("prmt.b32 %0, %1, 0, %2;" : "=r"(cj) : "r"(f), "r"(0x4440u + (uint32_t)j));
                            ad = cpt_u + (cj << 8);
                        } else {
                            ad = cpt_u | ((f << (8 - FB * j)) & ((uint32_t)(NE - 1) << 8));
                        }
                        float2 x;
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(ad));
                        const float ka = fmaf(x.x, af[j].x, af[j].z), kb = fmaf(x.y, af[j].y, af[j].w);
                        float co, si;
                        __sincosf(fmaf((float)(vg + 8 * m - 16), an[j].y, an[j].x), &si, &co);
                        const float ra = ka * co - kb * si, rb = ka * si + kb * co;
                        const uint32_t h = pack_half2(ra, rb);
                        const __half2 h2 = *reinterpret_cast<const __half2 *>(&h);
                        // rows g (m even) / g + 8 (m odd) of m-tile m / 2; slot j: registers 0-1 / 2-3
                        ahi[m >> 1][2 * j + (m & 1)] = h;
                        alo[m >> 1][2 * j + (m & 1)] = pack_half2(ra - __low2float(h2), rb - __high2float(h2));
                    }
                }
                const uint4 bb = bqs[s * 32 + lane];
                const uint32_t b[2] = {bb.x, bb.y};
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    mma_f16_f32(dsc[mt], ahi[mt], b);
                    mma_f16_f32(dsc[mt], alo[mt], b);
                    if constexpr (G8) {   // + A_hi x q~_lo (A_lo x q~_lo is below fp32 rounding)
                        const uint32_t bl[2] = {bb.z, bb.w};
                        mma_f16_f32(dsc[mt], ahi[mt], bl);
                    }
                }
            }
        }
        // columns 2t, 2t+1 of lane (g, t): heads 2t, 2t+1 (hi part, t < 2) or their lo parts
        // (t >= 2): hi + lo via one shuffle, then scores (x 2^4) to lane = token
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int h = 2 * vt + (r & 1);
                if constexpr (G8) {   // column = head, hi and lo already summed by the mma
                    sct[h * 32 + 16 * mt + vg + 8 * (r >> 1)] = dsc[mt][r] * 16.f;
                } else {
                    const float v = dsc[mt][r] + __shfl_xor_sync(0xffffffffu, dsc[mt][r], 2);
                    if (vt < 2 && h < G) sct[h * 32 + 16 * mt + vg + 8 * (r >> 1)] = v * 16.f;
                }
            }
        // V words of this tile (L2 hits), used after the softmax
        uint32_t vw[KWH];
#pragma unroll
        for (int w = 0; w < KWH; ++w) vw[w] = __ldg(c.vcodes + vf_word(t, c.H_kv, hk, w, lane, BITS));
        __syncwarp();
        float sco[G];
#pragma unroll
        for (int g = 0; g < G; ++g) sco[g] = sct[g * 32 + lane];
        // item -> the G heads' corrections (x - K^(code)) * dscore/dK
        auto k_item = [&](uint32_t itm) {
            const int j = (int)((itm >> 11) & 31u);
            const int cc = (int)(itm & 0x7fu), flag = (int)((itm >> 9) & 3u);
            const int i = cc & 63, up = cc >> 6;
            int code = flag == 1 ? CM : 0;
            if (flag == 0) {
                const int bit = FB * i;
                const int wq = bit >> 5;
                unsigned long long w64 = kst[kst_swz<WB>(wq, j)];
                if ((bit & 31) + FB > 32) w64 |= (unsigned long long)kst[kst_swz<WB>(wq + 1, j)] << 32;
                const int pc = (int)((w64 >> (bit & 31)) & (NE - 1));
                code = (pc >> (up * BITS)) & CM;
            }
            const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
            const float delta = xval - (cbKs[code] * ks_s[cc] + kz_s[cc]);
            float co, si;
            rot32(i, j, co, si);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float qa = qs[g * kHeadDim + i], qb = qs[g * kHeadDim + i + 64];
                kfix_add32(&kfix[g * 32 + j], &kbig[g * 32 + j], delta * (up ? (qb * co - qa * si) : (qa * co + qb * si)));
            }
        };
        {
            const int64_t bucket = (int64_t)t * c.NG + hk;
#pragma unroll
            for (int k = 0; k < IPL; ++k)
                if (32 * k < nk && lane + 32 * k < nk) k_item(kitm[k]);
            for (int x = 32 * IPL + lane; x < nk; x += 32) k_item(__ldg(c.kit + bucket * c.kcap_g + x));
            if (kov) {
                for (int j = 0; j < ntok; ++j) {
                    const uint32_t r0 = __ldg(c.kptr + n0 + j), r1 = __ldg(c.kptr + n0 + j + 1);
                    for (uint32_t r = r0 + lane; r < r1; r += 32) {
                        const uint32_t rec = __ldcg(c.kout + r);
                        const int ch = (int)(rec & 0xffffu);
                        if (ch < c_lo || ch >= c_lo + kHeadDim) continue;
                        k_item((rec & 0xffff0000u) | ((uint32_t)j << 11) | (uint32_t)(ch - c_lo));
                    }
                }
            }
        }
        __syncwarp();
        const int tn = t + C::NWARP;
        if (tn < t_end) issue_k(tn);

        // ------------------------------------------------------ a4: online softmax
        // weights p s_n 2^(WEXP - E), E the running exponent bound of s_n (the accumulators
        // persist across tiles)
        const float smax = warp_max_redux(valid ? vsz.x : 0.f);
        const int E_new = smax > 0.f ? max(E_run, ilog2f(smax) + 1) : E_run;
        const float pe = pow2i(WEXP - E_new), rE = pow2i(E_run - E_new);
        E_run = E_new;
        uint32_t w2s[G], w2l[G];
        float al[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float s = sco[g] + (float)kfix[g * 32 + lane] * (1.f / kKfixScale) + kbig[g * 32 + lane];
            kbig[g * 32 + lane] = 0.f;   // the words are the V-outlier sums from here on
            s = valid ? s : -CUDART_INF_F;
            const float m_new = fmaxf(m_run[g], warp_max_redux(s));
            const float alpha = (m_new == -CUDART_INF_F) ? 1.f : exp2f(m_run[g] - m_new);
            const float p = valid ? exp2f(s - m_new) : 0.f;
            l_lane[g] = l_lane[g] * alpha + p;
            z_lane[g] = z_lane[g] * alpha + p * vsz.y;
            m_run[g] = m_new;
            al[g] = alpha;
            if (alpha != 1.f) {   // warp-uniform
#pragma unroll
                for (int x = 0; x < kHeadDim / 32; ++x) osp[g * kHeadDim + x * 32 + lane] *= alpha;
            }
            ps[g * 32 + lane] = p;
            const float wf = p * (vsz.x * pe);
            const __half wh = __float2half_rn(wf);
            const uint32_t hb = __half_as_ushort(wh), lb = __half_as_ushort(__float2half_rn(wf - __half2float(wh)));
            w2s[g] = hb | (__shfl_down_sync(0xffffffffu, hb, 1) << 16);
            w2l[g] = lb | (__shfl_down_sync(0xffffffffu, lb, 1) << 16);
        }
        {   // rescale the accumulators: per column (head) alpha, and the weight exponent
            // (G <= 4: columns 2t, 2t+1 are head t's hi / lo sums; G = 8: heads 2t, 2t+1)
            float a0 = al[0], a1 = al[0];
#pragma unroll
            for (int g = 1; g < G; ++g) {
                if constexpr (G8) { a0 = 2 * vt == g ? al[g] : a0; a1 = 2 * vt + 1 == g ? al[g] : a1; }
                else a0 = hcl == g ? al[g] : a0;
            }
            a0 *= rE;
            if constexpr (G8) a1 *= rE; else a1 = a0;
            if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
                for (int ml = 0; ml < 8; ++ml) {
                    dacc[ml][0] *= a0; dacc[ml][2] *= a0;
                    dacc[ml][1] *= a1; dacc[ml][3] *= a1;
                }
            }
        }
        // B fragments: G <= 4: column vg = query head vg / 2, its hi (vg even) or lo (vg odd)
        // weight part; G = 8: column vg = head vg, hi (bw) and lo (bwl) as two B fragments;
        // tokens 16 s2 + 2 vt (+1) and + 8
        uint32_t bw[2][2], bwl[2][2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t v = 0u, vl = 0u;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t xh = __shfl_sync(0xffffffffu, w2s[g], 16 * s2 + 2 * vt + 8 * r);
                    const uint32_t xl = __shfl_sync(0xffffffffu, w2l[g], 16 * s2 + 2 * vt + 8 * r);
                    if constexpr (G8) { v = vg == g ? xh : v; vl = vg == g ? xl : vl; }
                    else v = (vg >> 1) == g ? ((vg & 1) ? xl : xh) : v;
                }
                bw[s2][r] = v;
                bwl[s2][r] = vl;
            }

        // --------------------------------------------------------- a5: P.V dense
#pragma unroll
        for (int ml = 0; ml < 8; ++ml) {
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                uint32_t a[4], alo[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int bit = ((ml * 2 + s2) * 4 + r) * FB;
                    const int wi = bit >> 5, sh = bit & 31;
                    uint32_t ad;
                    if constexpr (BITS == 4) {   // byte-aligned fields: PRMT + add (no table alignment)
                        uint32_t cf;
                        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(cf) : "r"(vw[wi]), "r"(0x4440u + (uint32_t)(sh >> 3)));
                        ad = vlut_u + (cf << 7);
                    } else {
                        uint32_t off;
                        if (sh + FB <= 32) off = sh >= 7 ? (vw[wi] >> (sh - 7)) : (vw[wi] << (7 - sh));
                        else off = __funnelshift_r(vw[wi], vw[wi + 1], sh - 7);
                        ad = vlut_u | (off & ((NE - 1) << 7));
                    }
                    a[r] = lds_u32(ad);
                    if constexpr (RESID) alo[r] = lds_u32(ad + NE * 32 * 4);
                }
                mma_f16_f32(dacc[ml], a, bw[s2]);
                if constexpr (RESID) mma_f16_f32(dacc[ml], alo, bw[s2]);
                if constexpr (G8) {
                    mma_f16_f32(dacc[ml], a, bwl[s2]);
                    if constexpr (RESID) mma_f16_f32(dacc[ml], alo, bwl[s2]);
                }
            }
        }

        // ------------------------------------------------------ a6: V outliers
        // p_g (x - V^(code)) of every item for the G heads, summed in fixed point (scale from
        // the tile's largest |term|) with native shared integer atomics, folded into osp
        __syncwarp();
        if (nv > 0 || vov) {
            // item -> (channel, delta); the G terms are ps[g][j] * delta
            auto v_delta = [&](uint32_t itm, bool act, int &j, int &cc) -> float {
                j = (int)((itm >> 11) & 31u);
                cc = (int)(itm & 0x7fu);
                const int flag = (int)((itm >> 9) & 3u);
                int code = flag == 1 ? CM : 0;
                if (act && flag == 0) {
                    const int bit = vf_bit(j, cc, BITS);
                    const uint32_t *wq = c.vcodes + vf_word(t, c.H_kv, hk, bit >> 5, vf_lane(j, cc), BITS);
                    unsigned long long w64 = __ldg(wq);
                    if ((bit & 31) + BITS > 32) w64 |= (unsigned long long)__ldg(wq + 32) << 32;
                    code = (int)((w64 >> (bit & 31)) & CM);
                }
                const float s_n = __shfl_sync(0xffffffffu, vsz.x, j), z_n = __shfl_sync(0xffffffffu, vsz.y, j);
                const float xval = __half2float(__ushort_as_half((uint16_t)(itm >> 16)));
                return act ? xval - (cbVs[code] * s_n + z_n) : 0.f;
            };
            const int64_t bucket = (int64_t)t * c.NG + hk;
            // the items beyond the registers (rare): x0 + lane for x0 >= 32 IPL, then (overflowed
            // bucket) every CSR record of the tile's tokens in this KV head
            const int kvn = c.kv;
            const int x_beg = vov ? 0 : 32 * IPL;
            const int x_end = (vov ? ntok * kvn : 0) + nv;
            auto slow_item = [&](int x0, int &j, int &cc) -> float {
                uint32_t itm = 0u;
                bool act = false;
                if (x0 < nv) {
                    act = x0 + lane < nv;
                    itm = act ? __ldg(c.vit + bucket * c.vcap_g + x0 + lane) : 0u;
                } else {
                    const int r = x0 - nv + lane;
                    act = r < ntok * kvn;
                    if (act) {
                        const uint32_t rec = __ldcg(c.vout + n0 * kvn + r);
                        const int ch = (int)(rec & 0xffffu);
                        act = ch >= c_lo && ch < c_lo + kHeadDim;
                        itm = (rec & 0xffff0000u) | ((uint32_t)(r / kvn) << 11) | (uint32_t)(act ? ch - c_lo : 0);
                    }
                }
                return v_delta(itm, act, j, cc);
            };
            const bool slow = nv > 32 * IPL || vov;
            float dl[IPL];
            int jx[IPL], cx[IPL];
            float pmax = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) pmax = fmaxf(pmax, ps[g * 32 + lane]);
            pmax = warp_max(pmax);   // every term is <= pmax |delta|
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < IPL; ++k) {
                dl[k] = 0.f; jx[k] = 0; cx[k] = 0;
                if (32 * k < nv && !vov) dl[k] = v_delta(vitm[k], lane + 32 * k < nv, jx[k], cx[k]);
                mx = fmaxf(mx, fabsf(dl[k]));
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    mx = fmaxf(mx, fabsf(slow_item(x0, j, cc)));
                }
            mx = warp_max(mx) * pmax;
            const int emx = mx > 0.f ? ilog2f(mx) : 0;
            const float S = pow2i(24 - emx);
            auto add = [&](float d, int j, int cc) {
                if (d == 0.f) return;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float v = ps[g * 32 + j] * d;
                    if (v != 0.f) atomicAdd(&vfix[g * kHeadDim + cc], __float2int_rn(v * S));
                }
            };
            if (!vov) {
#pragma unroll
                for (int k = 0; k < IPL; ++k) add(dl[k], jx[k], cx[k]);
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    const float d = slow_item(x0, j, cc);
                    add(d, j, cc);
                }
            __syncwarp();
            // fold only the entries this tile touched: the lanes re-walk their items and the
            // first to exchange an entry adds it (the others get 0)
            const float inv = pow2i(emx - 24);
            auto fold = [&](float d, int cc) {
                if (d == 0.f) return;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int v = atomicExch(&vfix[g * kHeadDim + cc], 0);
                    if (v) osp[g * kHeadDim + cc] += (float)v * inv;
                }
            };
            if (!vov) {
#pragma unroll
                for (int k = 0; k < IPL; ++k) fold(dl[k], cx[k]);
            }
            if (slow)
                for (int x0 = x_beg; x0 < x_end; x0 += 32) {
                    int j, cc;
                    const float d = slow_item(x0, j, cc);
                    fold(d, cc);
                }
            __syncwarp();
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) kfix[g * 32 + lane] = 0;

#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            ang64[k] = red2pi(ang64[k] + step64[k]);
            anc32[apad(i)].x = (float)ang64[k];
        }
        cnt_k = ncnt_k;
        cnt_v = ncnt_v;
        __syncwarp();
    }

    // ------------------------------------------- warp partials -> CTA partial (a7)
    cp_async_wait_all();
    __syncwarp();
    // osp (V-outlier sums, real units) += the dense accumulators of the lane's columns
    {
        const float sc = pow2i(E_run - WEXP);
#pragma unroll
        for (int ml = 0; ml < 8; ++ml) {
            const int ch = ml * 16 + vg;
            if constexpr (G8) {   // columns 2t, 2t+1 = heads 2t, 2t+1
                osp[(2 * vt) * kHeadDim + ch] += dacc[ml][0] * sc;
                osp[(2 * vt + 1) * kHeadDim + ch] += dacc[ml][1] * sc;
                osp[(2 * vt) * kHeadDim + ch + 8] += dacc[ml][2] * sc;
                osp[(2 * vt + 1) * kHeadDim + ch + 8] += dacc[ml][3] * sc;
            } else if (vt < G) {
                osp[vt * kHeadDim + ch] += (dacc[ml][0] + dacc[ml][1]) * sc;
                osp[vt * kHeadDim + ch + 8] += (dacc[ml][2] + dacc[ml][3]) * sc;
            }
        }
    }
    __syncwarp();
    float *wpart = reinterpret_cast<float *>(osp);   // in place: [G][d] o, then m, l in kst
    float *wml = reinterpret_cast<float *>(kst);     // [G][2]
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float l = warp_sum(l_lane[g]), z = warp_sum(z_lane[g]);
#pragma unroll
        for (int x = 0; x < kHeadDim / 32; ++x) wpart[g * kHeadDim + x * 32 + lane] += z;
        if (lane == 0) { wml[g * 2] = m_run[g]; wml[g * 2 + 1] = l; }
    }
    __syncthreads();
    float *part = P.parts + (int64_t)split * c.H_q * (kHeadDim + 2);
    for (int x = tid; x < G * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int w = 0; w < NWARP; ++w) {
            const float *ml = reinterpret_cast<const float *>(wbase + w * C::w_bytes) + g * 2;
            if (ml[1] != 0.f) m = fmaxf(m, ml[0]);
        }
        float l = 0.f, o = 0.f;
        for (int w = 0; w < NWARP; ++w) {
            const float *ml = reinterpret_cast<const float *>(wbase + w * C::w_bytes) + g * 2;
            if (ml[1] == 0.f) continue;
            const float wt = exp2f(ml[0] - m);
            l += wt * ml[1];
            if (ch < kHeadDim) {
                const float *ow = reinterpret_cast<const float *>(wbase + w * C::w_bytes + C::w_kst + G * 32 * 4);
                o += wt * ow[g * kHeadDim + ch];
            }
        }
        part[(g0 + g) * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
    }
    __threadfence();
    __syncthreads();
    int *s_last = flag_s + 1;
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.tickets[hgi], 1u);
        *s_last = (prev == (unsigned)(P.S - 1));
    }
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    for (int x = tid; x < G * (kHeadDim + 2); x += NTHR) {
        const int g = x / (kHeadDim + 2), ch = x % (kHeadDim + 2);
        const int gq = g0 + g;
        // the S partials in chunks of 8 independent L2 loads (one round trip per chunk, not per
        // split: the merge runs after every other CTA of the head group has finished)
        constexpr int MC = 8;
        const float *pbase = P.parts + (int64_t)gq * (kHeadDim + 2);
        const int64_t pstride = (int64_t)c.H_q * (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : -CUDART_INF_F;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k)
                if (lv[k] != 0.f) m = fmaxf(m, mv[k]);
        }
        float l = 0.f, o = 0.f;
        for (int s0 = 0; s0 < P.S; s0 += MC) {
            float mv[MC], lv[MC], ov[MC];
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const bool in = s0 + k < P.S;
                const float *ps2 = pbase + (s0 + k) * pstride;
                mv[k] = in ? __ldcg(ps2 + kHeadDim) : 0.f;
                lv[k] = in ? __ldcg(ps2 + kHeadDim + 1) : 0.f;
                ov[k] = (in && ch < kHeadDim) ? __ldcg(ps2 + ch) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < MC; ++k) {   // fixed split order, as before
                if (lv[k] == 0.f) continue;
                const float wgt = exp2f(mv[k] - m);
                l += wgt * lv[k];
                if (ch < kHeadDim) o += wgt * ov[k];
            }
        }
        if (P.write_partial) {
            P.out[gq * (kHeadDim + 2) + ch] = ch < kHeadDim ? o : (ch == kHeadDim ? m : l);
        } else if (ch < kHeadDim) {
            P.out[gq * kHeadDim + ch] = o / l;
        }
    }
    if (tid == 0) P.tickets[hgi] = 0;
}


template <int BITS, bool RESID, int G>
__global__ void __launch_bounds__(TCfg<BITS, RESID, G>::NTHR, 1) att_wgt_kernel(DevCache c, WParams P) {
    att_wgt_body<BITS, RESID, G>(c, P, (int)blockIdx.x);
}

// Batched GQA decode: B independent caches of one configuration in one launch,
// per-sequence descriptors in the kernel parameter space (as att_wa_batch_kernel)
template <int BITS, bool RESID, int G>
__global__ void __launch_bounds__(TCfg<BITS, RESID, G>::NTHR, 1) att_wgt_batch_kernel(const __grid_constant__ WBatch b) {
    const int blk = (int)blockIdx.x;
    int s = 0;
    while (s + 1 < b.n && blk >= b.cta0[s + 1]) ++s;
    att_wgt_body<BITS, RESID, G>(b.c[s], b.p[s], blk - b.cta0[s]);
}

template <int BITS, bool RESID, int G>
cudaError_t launch_wgt_t(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    using C = TCfg<BITS, RESID, G>;
    static_assert(C::total <= 227 * 1024, "shared memory");
    cudaError_t e = cudaFuncSetAttribute(att_wgt_kernel<BITS, RESID, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    e = launch_maybe_pdl(att_wgt_kernel<BITS, RESID, G>, grid, C::NTHR, C::total, s, P.pdl != 0, c, P);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
template <int BITS, bool RESID, int G>
cudaError_t launch_wgt_batch_t(const WBatch &b, int grid, cudaStream_t s) {
    using C = TCfg<BITS, RESID, G>;
    cudaError_t e = cudaFuncSetAttribute(att_wgt_batch_kernel<BITS, RESID, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    att_wgt_batch_kernel<BITS, RESID, G><<<grid, C::NTHR, C::total, s>>>(b);
    return cudaGetLastError();
}
template <int BITS, bool RESID>
cudaError_t launch_wgt_batch_g(const WBatch &b, int G, int grid, cudaStream_t s) {
    if constexpr (BITS < 4)
        if (G == 8) return launch_wgt_batch_t<BITS, RESID, 8>(b, grid, s);
    return G == 2 ? launch_wgt_batch_t<BITS, RESID, 2>(b, grid, s) : launch_wgt_batch_t<BITS, RESID, 4>(b, grid, s);
}

template <int BITS, bool RESID>
cudaError_t launch_wgt_g(const DevCache &c, const WParams &P, int grid, cudaStream_t s) {
    // G = 8: one 8-head CTA per KV head at 2-3 bits; at 4 bits (shared memory) two CTAs of 4
    if constexpr (BITS < 4)
        if (c.G == 8) return launch_wgt_t<BITS, RESID, 8>(c, P, grid, s);
    return c.G == 2 ? launch_wgt_t<BITS, RESID, 2>(c, P, grid, s) : launch_wgt_t<BITS, RESID, 4>(c, P, grid * (c.G / 4), s);
}

}  // namespace

bool attend_wag_supported(const DevCache &c) {
    return (c.G == 2 || c.G == 4 || c.G == 8) && (c.bits == 2 || c.bits == 3 || (c.bits == 4 && c.vcb_exact16)) &&
           c.GW == kHeadDim;   // bucket per KV head
}

cudaError_t launch_attend_wag(const DevCache &c, const AttendArgs &a, int S, cudaStream_t s) {
    WParams P{};
    P.q = a.q; P.pos = a.pos; P.T = a.T; P.S = S; P.ntiles = (int)((a.T + 31) / 32);
    P.out = a.out; P.parts = a.parts; P.tickets = a.tickets; P.write_partial = a.write_partial;
    P.pdl = a.pdl;
    const int grid = c.H_kv * S;
    const bool resid = !c.vcb_exact16;
    static const bool lut = getenv("KVQ_WGT_OFF") != nullptr;   // A/B: the LUT kernel att_wag_kernel
    if (!lut || c.G == 8 || c.bits == 4) {   // (the LUT kernel has no G = 8 or 4-bit tiling)
        if (c.bits == 2) return resid ? launch_wgt_g<2, true>(c, P, grid, s) : launch_wgt_g<2, false>(c, P, grid, s);
        if (c.bits == 3) return resid ? launch_wgt_g<3, true>(c, P, grid, s) : launch_wgt_g<3, false>(c, P, grid, s);
        if (c.bits == 4 && !resid) return launch_wgt_g<4, false>(c, P, grid, s);
    }
    if (c.bits == 2) return resid ? launch_wag_g<2, true>(c, P, grid, s) : launch_wag_g<2, false>(c, P, grid, s);
    if (c.bits == 3) return resid ? launch_wag_g<3, true>(c, P, grid, s) : launch_wag_g<3, false>(c, P, grid, s);
    return cudaErrorInvalidValue;
}

template <int BITS, bool RESID>
cudaError_t launch_wa_batch_t(const WBatch &b, int grid, cudaStream_t s) {
    using C = WCfg<BITS, RESID, 2>;
    cudaError_t e = cudaFuncSetAttribute(att_wa_batch_kernel<BITS, RESID, 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    att_wa_batch_kernel<BITS, RESID, 2><<<grid, C::NTHR, C::total, s>>>(b);
    return cudaGetLastError();
}

int attend_batch_max() { return kMaxBatch; }

cudaError_t launch_attend_wa_batch(const DevCache *const *cs, const AttendArgs *as, int B, cudaStream_t s,
                                   int *splits_out) {
    if (B < 1 || B > kMaxBatch) return cudaErrorInvalidValue;
    static WBatch b;   // large: build on the host once per call (not thread-safe across host threads)
    WBatch &bb = b;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t tiles_all = 0;
    for (int i = 0; i < B; ++i) tiles_all += (as[i].T + 31) / 32;
    bb.n = B;
    int cta = 0;
    for (int i = 0; i < B; ++i) {
        const DevCache &c = *cs[i];
        const int n_hg = c.H_q / HG;
        const int ntiles = (int)((as[i].T + 31) / 32);
        // splits in proportion to the sequence's share of all tiles, so the launch fills one
        // wave of one CTA per SM (at least one split per head group)
        int S = (int)((int64_t)sms * ntiles / (tiles_all * n_hg));
        if (as[i].splits > 0) S = as[i].splits;
        S = S < 1 ? 1 : (S > ntiles ? ntiles : S);
        WParams &P = bb.p[i];
        P = WParams{};
        P.q = as[i].q; P.pos = as[i].pos; P.T = as[i].T; P.S = S; P.ntiles = ntiles;
        P.out = as[i].out; P.parts = as[i].parts; P.tickets = as[i].tickets; P.write_partial = as[i].write_partial;
        P.pdl = 0;
        bb.c[i] = c;
        bb.cta0[i] = cta;
        cta += n_hg * S;
        if (splits_out) splits_out[i] = S;
    }
    bb.cta0[B] = cta;
    const DevCache &c0 = *cs[0];
    const bool resid = !c0.vcb_exact16;
    if (c0.bits == 2) return resid ? launch_wa_batch_t<2, true>(bb, cta, s) : launch_wa_batch_t<2, false>(bb, cta, s);
    if (c0.bits == 3) return resid ? launch_wa_batch_t<3, true>(bb, cta, s) : launch_wa_batch_t<3, false>(bb, cta, s);
    if (c0.bits == 4 && !resid) return launch_wa_batch_t<4, false>(bb, cta, s);
    return cudaErrorInvalidValue;
}

// Batched GQA decode: one att_wgt_batch_kernel launch over B caches of one configuration (the
// GQA kernel's tiling: H_kv x G / Gs head groups of Gs = min(G, 4) query heads per sequence)
cudaError_t launch_attend_wgt_batch(const DevCache *const *cs, const AttendArgs *as, int B, cudaStream_t s,
                                    int *splits_out) {
    if (B < 1 || B > kMaxBatch) return cudaErrorInvalidValue;
    static WBatch b;   // large: built on the host per call (not thread-safe across host threads)
    WBatch &bb = b;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t tiles_all = 0;
    for (int i = 0; i < B; ++i) tiles_all += (as[i].T + 31) / 32;
    const DevCache &c0 = *cs[0];
    const int Gs = (c0.G == 8 && c0.bits < 4) ? 8 : (c0.G < 4 ? c0.G : 4);   // query heads per CTA
    bb.n = B;
    int cta = 0;
    for (int i = 0; i < B; ++i) {
        const DevCache &c = *cs[i];
        const int n_hg = c.H_kv * (c.G / Gs);
        const int ntiles = (int)((as[i].T + 31) / 32);
        int S = (int)((int64_t)sms * ntiles / (tiles_all * n_hg));
        if (as[i].splits > 0) S = as[i].splits;
        S = S < 1 ? 1 : (S > ntiles ? ntiles : S);
        WParams &P = bb.p[i];
        P = WParams{};
        P.q = as[i].q; P.pos = as[i].pos; P.T = as[i].T; P.S = S; P.ntiles = ntiles;
        P.out = as[i].out; P.parts = as[i].parts; P.tickets = as[i].tickets; P.write_partial = as[i].write_partial;
        P.pdl = 0;
        bb.c[i] = c;
        bb.cta0[i] = cta;
        cta += n_hg * S;
        if (splits_out) splits_out[i] = S;
    }
    bb.cta0[B] = cta;
    const bool resid = !c0.vcb_exact16;
    if (c0.bits == 2) return resid ? launch_wgt_batch_g<2, true>(bb, Gs, cta, s) : launch_wgt_batch_g<2, false>(bb, Gs, cta, s);
    if (c0.bits == 3) return resid ? launch_wgt_batch_g<3, true>(bb, Gs, cta, s) : launch_wgt_batch_g<3, false>(bb, Gs, cta, s);
    if (c0.bits == 4 && !resid) return launch_wgt_batch_g<4, false>(bb, Gs, cta, s);
    return cudaErrorInvalidValue;
}

bool attend_wa_supported(const DevCache &c) {
    return c.G == 1 && (c.bits == 2 || c.bits == 3 || (c.bits == 4 && c.vcb_exact16)) &&
           c.H_q % HG == 0 && c.GW == 2 * kHeadDim;   // outlier buckets per 2-head group (one per warp)
}

size_t attend_wa_smem_bytes(int bits, bool resid) {
    if (bits == 2) return resid ? WCfg<2, true, 2>::total : WCfg<2, false, 2>::total;  // WH = 2
    if (bits == 3) return resid ? WCfg<3, true, 2>::total : WCfg<3, false, 2>::total;
    if (bits == 4) return WCfg<4, false, 2>::total;
    return 0;
}

cudaError_t launch_attend_wa(const DevCache &c, const AttendArgs &a, int S, cudaStream_t s) {
    WParams P{};
    P.q = a.q; P.pos = a.pos; P.T = a.T; P.S = S; P.ntiles = (int)((a.T + 31) / 32);
    P.out = a.out; P.parts = a.parts; P.tickets = a.tickets; P.write_partial = a.write_partial;
    P.pdl = a.pdl;
    const int grid = (c.H_q / HG) * S;
    const bool resid = !c.vcb_exact16;
    if (c.bits == 2) return resid ? launch_wa_r<2, true>(c, P, grid, s) : launch_wa_r<2, false>(c, P, grid, s);
    if (c.bits == 3) return resid ? launch_wa_r<3, true>(c, P, grid, s) : launch_wa_r<3, false>(c, P, grid, s);
    if (c.bits == 4 && !resid) return launch_wa_r<4, false>(c, P, grid, s);
    return cudaErrorInvalidValue;
}

}  // namespace kvq
