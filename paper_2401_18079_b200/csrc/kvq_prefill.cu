// kvq_prefill.cu -- QZ: block prefill quantization (one CTA per 32-token tile)
// and quantize-on-append of one decode token (a8, append_kernel at the end of the file).
//
// Both compute exactly what T successive appends define (readings R2-R8):
//   Keys: outlier iff x < lo_c or x > hi_c (R4); code = ENC(clamp(x)).
//   Values (topk P:1028-1031): two-sided top-k, k = ceil(f D),
//         ceil(k/2) largest then floor(k/2) smallest of the rest, ties to the lower index,
//         -0 == +0 (R2, R3); (s, z) from the kept [lo, hi] in fp64, rounded once (R6, R7);
//         code = ENC(clamp(v)).
//
// ENC without per-element fp64 (R8).  The fp64 predicate P_j(y) = [2(y - z) > s m_j] that
// defines ENC is monotone in y, so for fp16 inputs it is fully described by its threshold
// T_j = the smallest fp16 value with P_j true, and ENC(y) = #{j : y >= T_j} (an IEEE fp16
// comparison; -0 == +0 on both sides).  The thresholds are found by a binary search over
// the fp16 values that evaluates exactly the oracle's fp64 expression:
//   * Keys: per channel, on the host at create time (kvq_api.cu, kenc table), with the
//     codes of the clamped values lo_c, hi_c (fp32, not fp16) precomputed the same way;
//   * Values: per token, by NM lanes of the token's warp after (s_n, z_n) are known.
// A whole channel pair or token pair is then encoded with fp16x2 compares (HSET2) and
// fp16x2 adds of the 0/1 results: integer decisions, bit-exact with the oracle.
//
// Work of a CTA (tile t, tokens [max(n0, 32t), min(n0 + T, 32t + 32))):
//   A  Value selection, warp per token: per-lane fp16 max/min over two channel groups, the
//      (k+1)-th largest group max bounds the outliers from below, so only elements at or
//      above it (typically ~40 of 4096) are ranked exactly by (value, index); same for the
//      lower tail.  A bit-by-bit exact selection over all elements handles inputs where the
//      bound admits too many candidates (ties, tiny D).  Writes (s, z), the CSR records
//      and the token's per-group outlier counts (its bitmask lives in the warp's scratch).
//   B  Keys, warp per KV head, lane = token: pair codes packed straight into the tile's
//      pair-stream words (coalesced 128-byte stores), outlier bitmask per (token, head).
//   C  Value codes, warp per KV head, lane = mma A-fragment lane: the head's V slice staged
//      transposed in shared memory, each field = one token pair of one channel.
//   D  Key CSC offsets by a decoupled look-back over the tiles of the launch (each CTA takes
//      its tile from a ticket, so every predecessor has started), CSC records, and the
//      outlier items of the (tile, head group) buckets in (token, channel) order (Value
//      items from the tokens' CSR rows).
// Order in the kernel: A, B, publish the tile's Key-outlier aggregate, C, resolve the
// look-back (so the wait for the predecessors overlaps C), D.
#include "kvq_internal.cuh"

namespace kvq {
namespace {

constexpr int PW = 8;              // warps per CTA
constexpr int PT = PW * 32;
constexpr int CANDMAX = 256;       // candidates per tail (fast path)
constexpr uint32_t LB_AGG = 1u, LB_INC = 2u;

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }
// fp16 bits -> order key (ascending value order), -0 merged with +0
__device__ __forceinline__ uint32_t okey(uint32_t h) {
    h &= 0xffffu;
    uint32_t k = h ^ ((h & 0x8000u) ? 0xffffu : 0x8000u);
    return k == 0x7fffu ? 0x8000u : k;
}
// fp16 bits of element e (0..7, run-time) of an 8-half vector, without indexing a register
// array (a dynamic index would put the array on the stack: a local-memory round trip per use)
__device__ __forceinline__ uint32_t half_at(const uint4 &u, int e) {
    const uint32_t w = (e & 4) ? ((e & 2) ? u.w : u.z) : ((e & 2) ? u.y : u.x);
    return (e & 1) ? (w >> 16) : (w & 0xffffu);
}
// order key -> fp16 bits (0x8000 -> +0)
__device__ __forceinline__ uint32_t key2h(uint32_t k) { return k >= 0x8000u ? (k ^ 0x8000u) : (k ^ 0xffffu); }

// counts of a half2 of {0,1} sums -> two small integers
__device__ __forceinline__ uint32_t h2codes(__half2 c2, int bits) {
    const uint32_t w = h2u(__hadd2(c2, __float2half2_rn(1024.f)));   // 0x6400 + code per half
    return (w & 0xfu) | ((w >> (16 - bits)) & (0xfu << bits));
}

template <int BITS>
struct PCfg {
    static constexpr int NM = (1 << BITS) - 1;             // ENC thresholds
    static constexpr int PS = ((4 + NM) + 3) & ~3;         // kenc words per channel pair
};

struct PParams {
    const __half *K, *V;       // chunk rows [T][D]
    int64_t n0, T;
    int64_t tile0;
    int ntile;
    unsigned long long *lb;    // [ntile] look-back words (zeroed before the launch)
    unsigned *ticket;          // zeroed before the launch
    unsigned long long *tm;    // diagnostics: per-phase clock sums [6] (tid 0 of every CTA), or null
};

// Dynamic shared memory layout (bytes), D channels, DW = D/32 mask words per token
struct PSmem {
    int DW, NG;
    size_t kmask, vmask, kcnt, cntK, cntV, posK, posV, tinfo, warp, total;
    __host__ __device__ PSmem(int D, int NG_) {
        DW = D / 32; NG = NG_;
        size_t o = 0;
        kmask = o; o += (size_t)32 * DW * 4;
        vmask = 0;   // (the Value outlier mask of a token lives in its warp's scratch during A)
        kcnt = o;  o += (size_t)32 * (D / 128) * 2;     // Key outliers per (token, head)
        cntK = o;  o += (size_t)32 * NG * 2;            // per (token, group)
        cntV = o;  o += (size_t)32 * NG * 2;
        posK = o;  o += (size_t)32 * NG * 2;            // bucket slot of (token, group)
        posV = o;  o += (size_t)32 * NG * 2;
        o = (o + 15) & ~(size_t)15;
        tinfo = o; o += (size_t)32 * 24 * 2;            // per token: lo, hi, T[15], code lo/hi
        o = (o + 15) & ~(size_t)15;
        warp = o;  o += (size_t)PW * 64 * 20 * 4;        // per warp: candidates + mask / V staging
        total = o;
    }
};
constexpr int TI_LO = 0, TI_HI = 1, TI_CLO = 2, TI_CHI = 3, TI_T = 4;   // tinfo fields (u16)

// ---------------------------------------------------------------- exact selection (slow)
// Marks in `mask` the `need` elements of `row` that come first in (value desc, index asc)
// (desc) or (value asc, index asc) order among elements not already in `mask`.  Bit-by-bit
// search of the order-key threshold, then ties at the threshold in index order.  Element
// ownership: lane l holds channels 256m + 8l + e.
__device__ __noinline__ void select_exact(const __half *row, int D, int need, bool desc, uint32_t *mask) {
    const int lane = threadIdx.x & 31;
    if (need <= 0) return;
    const int nch = (D + 255) / 256;
    auto kv = [&](uint32_t h) { const uint32_t k = okey(h); return desc ? k : 0xffffu - k; };
    auto count_ge = [&](uint32_t t, bool strict) {
        int cnt = 0;
        for (int m = 0; m < nch; ++m) {
            const int c0 = 256 * m + 8 * lane;
            if (c0 >= D) continue;
            const uint4 u = *reinterpret_cast<const uint4 *>(row + c0);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            const uint32_t mw = mask[c0 >> 5] >> (c0 & 31);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if ((mw >> e) & 1u) continue;
                const uint32_t k = kv(e & 1 ? w[e >> 1] >> 16 : w[e >> 1]);
                cnt += strict ? (k > t) : (k >= t);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        return cnt;
    };
    uint32_t t = 0;
    for (int b = 15; b >= 0; --b) {
        const uint32_t t2 = t | (1u << b);
        if (count_ge(t2, false) >= need) t = t2;
    }
    int take = need - count_ge(t, true);   // ties at t, lowest index first
    int run = 0;
    for (int m = 0; m < nch; ++m) {
        const int c0 = 256 * m + 8 * lane;
        uint32_t sel = 0, tie = 0;
        if (c0 < D) {
            const uint4 u = *reinterpret_cast<const uint4 *>(row + c0);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            const uint32_t mw = mask[c0 >> 5] >> (c0 & 31);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if ((mw >> e) & 1u) continue;
                const uint32_t k = kv(e & 1 ? w[e >> 1] >> 16 : w[e >> 1]);
                sel |= (uint32_t)(k > t) << e;
                tie |= (uint32_t)(k == t) << e;
            }
        }
        const int nt = __popc(tie);
        int ex = nt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ex, o);
            if (lane >= o) ex += y;
        }
        const int tot = __shfl_sync(0xffffffffu, ex, 31);
        ex -= nt;
        int r = run + ex;
        for (uint32_t x = tie; x; x &= x - 1, ++r)
            if (r < take) sel |= x & (~x + 1u);
        run += tot;
        if (sel) atomicOr(&mask[c0 >> 5], sel << (c0 & 31));
    }
    __syncwarp();
}

// Exact two-sided selection of one token by one warp (the slow path): the ku largest, then the kl
// smallest of the rest, into `vm` (zeroed here), and the kept min / max (lowest index attaining
// them, R7) as fp16 bits.
__device__ __noinline__ void vselect_exact_warp(const __half *row, int D, int ku, int kl, uint32_t *vm, uint32_t &lo_h,
                                   uint32_t &hi_h) {
    const int lane = threadIdx.x & 31, DW = D / 32, nch = (D + 255) / 256;
    for (int x = lane; x < DW; x += 32) vm[x] = 0;
    __syncwarp();
    select_exact(row, D, ku, true, vm);
    select_exact(row, D, kl, false, vm);
    uint32_t bh = 0, bl2 = 0xffffffffu;   // (key << 16 | 0xffff - idx) max; (key << 16 | idx) min
    for (int m = 0; m < nch; ++m) {
        const int c0 = 256 * m + 8 * lane;
        if (c0 >= D) continue;
        const uint4 u = *reinterpret_cast<const uint4 *>(row + c0);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        const uint32_t mw = vm[c0 >> 5] >> (c0 & 31);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if ((mw >> e) & 1u) continue;
            const uint32_t key = okey(e & 1 ? w[e >> 1] >> 16 : w[e >> 1]);
            bh = max(bh, (key << 16) | (0xffffu - (uint32_t)(c0 + e)));
            bl2 = min(bl2, (key << 16) | (uint32_t)(c0 + e));
        }
    }
    bh = __reduce_max_sync(0xffffffffu, bh);
    bl2 = __reduce_min_sync(0xffffffffu, bl2);
    hi_h = __half_as_ushort(row[0xffff - (bh & 0xffffu)]);
    lo_h = __half_as_ushort(row[bl2 & 0xffffu]);
}

// The rest of one token's Value quantization by one warp, after the selection: (s, z) in fp64
// rounded once (R6), the token's ENC thresholds and the codes of lo / hi (tinfo_row), the CSR
// records of its k outliers (ascending channel).
template <int NM>
__device__ void vfinish_warp(const DevCache &c, const __half *row, int D, const uint32_t *vm, uint32_t lo_h,
                             uint32_t hi_h, uint16_t *tinfo_row, int64_t n, const double *vmids) {
    const int lane = threadIdx.x & 31, DW = D / 32, k = c.kv;
    // (s, z) in fp64, rounded once (R6); ENC thresholds of the token (lanes 0..NM-1)
    const double lo = (double)__half2float(__ushort_as_half((uint16_t)lo_h));
    const double hi = (double)__half2float(__ushort_as_half((uint16_t)hi_h));
    const float s = __double2float_rn(__dsub_rn(hi, lo) / 2.0);
    const float z = __double2float_rn(__dadd_rn(hi, lo) / 2.0);
    uint16_t *ti = tinfo_row;
    if (lane == 0) {
        c.vsz[n] = make_float2(s, z);
        ti[TI_LO] = (uint16_t)lo_h;
        ti[TI_HI] = (uint16_t)hi_h;
    }
    uint32_t thr = 0x7c00u;   // +inf: never
    if (lane < NM) {
        // T_j = the smallest fp16 (order key in [0x0400, 0xfc00), else the +inf sentinel 0xfc00)
        // with 2(y - z) > s m_j in fp64 -- a monotone predicate.  Start at the fp16 nearest to
        // z + s m_j / 2 and walk to the boundary (one or two steps); a binary search if the walk
        // is long.
        const double mj = vmids[lane];
        const double sd = (double)s, zd = (double)z;
        auto pred = [&](uint32_t key) {
            const double y = (double)__half2float(__ushort_as_half((uint16_t)key2h(key)));
            return 2.0 * __dsub_rn(y, zd) > __dmul_rn(sd, mj);
        };
        unsigned short h0;
        asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h0) : "d"(__fma_rn(0.5 * sd, mj, zd)));
        uint32_t a = min(max(okey(h0), 0x0400u), 0xfbffu);
        int steps = 0;
        if (pred(a)) {
            while (a > 0x0400u && steps < 8 && pred(a - 1)) { --a; ++steps; }
        } else {
            while (a < 0xfc00u && steps < 8 && !pred(a)) { ++a; ++steps; }
        }
        if (steps == 8) {
            uint32_t lo = 0x0400u, hi = 0xfc00u;   // order keys of -65504 .. +inf (sentinel)
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (pred(mid)) hi = mid; else lo = mid + 1;
            }
            a = lo;
        }
        thr = key2h(a);
        ti[TI_T + lane] = (uint16_t)thr;
    }
    // codes of lo and hi (item flags of the outliers)
    const uint32_t klo = okey(lo_h), khi = okey(hi_h), kt = okey(thr);
    const int clo = __popc(__ballot_sync(0xffffffffu, lane < NM && klo >= kt));
    const int chi = __popc(__ballot_sync(0xffffffffu, lane < NM && khi >= kt));
    if (lane == 0) { ti[TI_CLO] = (uint16_t)clo; ti[TI_CHI] = (uint16_t)chi; }
    __syncwarp();
    // CSR records of the token's k outliers (ascending channel) and per-group counts
    if (k > 0) {
        const int wpl = (DW + 31) / 32;   // mask words per lane (ascending channels)
        int cnt = 0;
        for (int x = wpl * lane; x < wpl * lane + wpl && x < DW; ++x) cnt += __popc(vm[x]);
        int ex = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ex, o);
            if (lane >= o) ex += y;
        }
        ex -= cnt;
        uint32_t *vo = c.vout + n * (int64_t)k;
        for (int x = wpl * lane; x < wpl * lane + wpl && x < DW; ++x)
            for (uint32_t b = vm[x]; b; b &= b - 1) {
                const int ch = 32 * x + __ffs(b) - 1;
                vo[ex++] = (uint32_t)ch | ((uint32_t)__half_as_ushort(row[ch]) << 16);
            }
    }
}

// One token's Value quantization by one warp (reads R2, R3, R6, R7, R8): the two-sided top-k
// outliers (bitmask vm, [D/32] words, zeroed by the caller), kept range, (s, z) -> c.vsz[n],
// ENC thresholds and the codes of lo / hi -> tinfo_row, CSR records -> c.vout row n.
// cand: per-warp scratch [2][CANDMAX]; nc2: per-warp [2] counters.
template <int NM>
__device__ void vtoken_warp(const DevCache &c, const __half *row, int D, uint32_t *vm, uint32_t *cand,
                            int *nc2, uint16_t *tinfo_row, int64_t n, unsigned long long *tr = nullptr) {
    const int lane = threadIdx.x & 31;
    const int DW = D / 32;
    auto vstamp = [&](int i) {   // diagnostics (append trace only)
        if (tr && lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(tr + i, t);
        }
    };
    const int k = c.kv, ku = (k + 1) / 2, kl = k / 2;
    const int nch = (D + 255) / 256;
        // group maxima / minima (fp16 values; 2 groups per lane: even / odd chunks)
        // (scalars, chunk pairs per iteration: a run-time index into a register array would
        // live on the stack)
        __half2 mx0 = __float2half2_rn(-65504.f), mx1 = mx0, mn0 = __float2half2_rn(65504.f), mn1 = mn0;
        bool have0 = false, have1 = false;
#pragma unroll 4
        for (int m = 0; m < nch; m += 2) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int c0 = 256 * (m + q) + 8 * lane;
                if (m + q >= nch || c0 >= D) continue;
                const uint4 u = *reinterpret_cast<const uint4 *>(row + c0);
                const __half2 a = __hmax2(__hmax2(u2h(u.x), u2h(u.y)), __hmax2(u2h(u.z), u2h(u.w)));
                const __half2 b = __hmin2(__hmin2(u2h(u.x), u2h(u.y)), __hmin2(u2h(u.z), u2h(u.w)));
                if (q == 0) { mx0 = __hmax2(mx0, a); mn0 = __hmin2(mn0, b); have0 = true; }
                else        { mx1 = __hmax2(mx1, a); mn1 = __hmin2(mn1, b); have1 = true; }
            }
        }
        // (need+1)-th largest group max / smallest group min, bit search on order keys
        uint32_t gk[2], gl[2];
        gk[0] = have0 ? okey(h2u(__hmax2(mx0, __lowhigh2highlow(mx0)))) : 0u;
        gk[1] = have1 ? okey(h2u(__hmax2(mx1, __lowhigh2highlow(mx1)))) : 0u;
        gl[0] = have0 ? 0xffffu - okey(h2u(__hmin2(mn0, __lowhigh2highlow(mn0)))) : 0u;
        gl[1] = have1 ? 0xffffu - okey(h2u(__hmin2(mn1, __lowhigh2highlow(mn1)))) : 0u;
        vstamp(8);
        // both searches in one loop (two independent ballot chains in flight)
        uint32_t t_hi = 0, t_lo = 0;
        for (int b = 15; b >= 0; --b) {
            const uint32_t a2 = t_hi | (1u << b), b2 = t_lo | (1u << b);
            const int na = __popc(__ballot_sync(0xffffffffu, gk[0] >= a2)) + __popc(__ballot_sync(0xffffffffu, gk[1] >= a2));
            const int nb = __popc(__ballot_sync(0xffffffffu, gl[0] >= b2)) + __popc(__ballot_sync(0xffffffffu, gl[1] >= b2));
            if (na >= ku + 1) t_hi = a2;
            if (nb >= kl + 1) t_lo = b2;
        }
        const uint32_t tau_hi = t_hi;              // order key: (ku+1)-th largest group max
        const uint32_t tau_lo = 0xffffu - t_lo;    // order key: (kl+1)-th smallest group min
        vstamp(9);
        // candidates: value >= tau_hi (upper), value <= tau_lo (lower)
        if (lane < 2) nc2[lane] = 0;
        __syncwarp();
        const __half2 th2 = u2h(key2h(tau_hi) * 0x10001u), tl2 = u2h(key2h(tau_lo) * 0x10001u);
        bool ovf = false;
        // (chunks in batches of 4: their loads are in flight together)
        for (int m0 = 0; m0 < nch; m0 += 4) {
          uint4 ub[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c0 = 256 * (m0 + q) + 8 * lane;
            ub[q] = (m0 + q < nch && c0 < D) ? *reinterpret_cast<const uint4 *>(row + c0) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int m = m0 + q;
            if (m >= nch) break;
            const int c0 = 256 * m + 8 * lane;
            const uint4 u = ub[q];
            uint32_t fu = 0, fl = 0;
            if (c0 < D) {
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
                // the chunk's max / min first: per-element flags only where a candidate is
                const __half2 a = __hmax2(__hmax2(u2h(u.x), u2h(u.y)), __hmax2(u2h(u.z), u2h(u.w)));
                const __half2 b = __hmin2(__hmin2(u2h(u.x), u2h(u.y)), __hmin2(u2h(u.z), u2h(u.w)));
                if (__hbge2(__hmax2(a, __lowhigh2highlow(a)), th2) || __hble2(__hmin2(b, __lowhigh2highlow(b)), tl2)) {
                    // a true half compares to 1.0 (0x3c00: bits 10-13); word e2 keeps bit 10 + e2
                    // of each half: element 2 e2 -> flag bit 10 + e2, 2 e2 + 1 -> 26 + e2
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const uint32_t sel = 0x04000400u << e2;
                        fu |= h2u(__hge2(u2h(w[e2]), th2)) & sel;
                        fl |= h2u(__hle2(u2h(w[e2]), tl2)) & sel;
                    }
                }
            }
            if (__any_sync(0xffffffffu, (fu | fl) != 0u)) {
                const int nu = __popc(fu), nl = __popc(fl);
                int bu = 0, bl = 0;
                if (nu) bu = atomicAdd(&nc2[0], nu);
                if (nl) bl = atomicAdd(&nc2[1], nl);
                if (fu | fl) {
                    for (uint32_t x = fu; x; x &= x - 1) {
                        const int b = __ffs(x) - 1, e = b < 16 ? 2 * (b - 10) : 2 * (b - 26) + 1;
                        const uint32_t key = okey(half_at(u, e));
                        if (bu < CANDMAX) cand[bu] = (key << 13) | (8191u - (uint32_t)(c0 + e));
                        ++bu;
                    }
                    for (uint32_t x = fl; x; x &= x - 1) {
                        const int b = __ffs(x) - 1, e = b < 16 ? 2 * (b - 10) : 2 * (b - 26) + 1;
                        const uint32_t key = okey(half_at(u, e));
                        if (bl < CANDMAX) cand[CANDMAX + bl] = ((0xffffu - key) << 13) | (8191u - (uint32_t)(c0 + e));
                        ++bl;
                    }
                }
            }
          }
        }
        __syncwarp();
        vstamp(10);
        const int NU = nc2[0], NL = nc2[1];
        ovf = NU > CANDMAX || NL > CANDMAX || NU < ku + 1 || NL < kl + 1 || tau_lo >= tau_hi;
        uint32_t lo_h = 0, hi_h = 0;   // fp16 bits of the kept min / max
        if (!ovf) {
            // exact ranks among the candidates: rank = #candidates ordered before
            int hi_idx = -1, lo_idx = -1;
            for (int i = lane; i < NU; i += 32) {
                const uint32_t v = cand[i];
                int r = 0;
                for (int q = 0; q < NU; ++q) r += cand[q] > v;
                const int ch = 8191 - (int)(v & 8191u);
                if (r < ku) atomicOr(&vm[ch >> 5], 1u << (ch & 31));
                if (r == ku) hi_idx = ch;
            }
            for (int i = lane; i < NL; i += 32) {
                const uint32_t v = cand[CANDMAX + i];
                int r = 0;
                for (int q = 0; q < NL; ++q) r += cand[CANDMAX + q] > v;
                const int ch = 8191 - (int)(v & 8191u);
                if (r < kl) atomicOr(&vm[ch >> 5], 1u << (ch & 31));
                if (r == kl) lo_idx = ch;
            }
            hi_idx = __reduce_max_sync(0xffffffffu, hi_idx + 1) - 1;
            lo_idx = __reduce_max_sync(0xffffffffu, lo_idx + 1) - 1;
            hi_h = __half_as_ushort(row[hi_idx]);
            lo_h = __half_as_ushort(row[lo_idx]);
            __syncwarp();
        } else {
            vselect_exact_warp(row, D, ku, kl, vm, lo_h, hi_h);
        }
        vstamp(11);
        if (tr && lane == 0) atomicMax(tr + 15, (unsigned long long)(ovf ? 1000000 + NU * 1000 + NL : NU * 1000 + NL));
        vfinish_warp<NM>(c, row, D, vm, lo_h, hi_h, tinfo_row, n, c.mids + 16);

}

// ------------------------------------------------------------------------------ kernel
template <int BITS>
__global__ void __launch_bounds__(PT, BITS == 4 ? 2 : 3) prefill_kernel(DevCache c, PParams P) {
    using C = PCfg<BITS>;
    constexpr int NM = C::NM, PS = C::PS, CM = (1 << BITS) - 1, KWH = 4 * BITS;
    extern __shared__ __align__(16) unsigned char sm[];
    const int D = c.D, H = c.H_kv, NG = c.NG, GW = c.GW;
    const PSmem L(D, NG);
    const int DW = L.DW;
    uint32_t *kmask = reinterpret_cast<uint32_t *>(sm + L.kmask);
    uint16_t *kcnt = reinterpret_cast<uint16_t *>(sm + L.kcnt);
    uint16_t *cntK = reinterpret_cast<uint16_t *>(sm + L.cntK);
    uint16_t *cntV = reinterpret_cast<uint16_t *>(sm + L.cntV);
    uint16_t *posK = reinterpret_cast<uint16_t *>(sm + L.posK);
    uint16_t *posV = reinterpret_cast<uint16_t *>(sm + L.posV);
    uint16_t *tinfo = reinterpret_cast<uint16_t *>(sm + L.tinfo);
    __shared__ uint32_t s_tokbase[33], s_tile, s_kbase, s_gbase[64][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned char *wsc = sm + L.warp + (size_t)warp * 64 * 20 * 4;
    long long t_prev = clock64();
    int phase = 0;
    auto pmark = [&]() {   // diagnostics: CTA time per phase (sync to sync)
        if (P.tm && tid == 0) {
            const long long t = clock64();
            atomicAdd(P.tm + phase, (unsigned long long)(t - t_prev));
            t_prev = t;
        }
        ++phase;
    };

    if (tid == 0) s_tile = atomicAdd(P.ticket, 1u);
    for (int x = tid; x < 32 * DW; x += PT) kmask[x] = 0;
    __syncthreads();
    pmark();
    const int li = (int)s_tile;                       // logical tile of this CTA
    const int64_t tile = P.tile0 + li;
    const int64_t nt0 = tile * 32;                    // token of lane 0
    const int64_t nA = nt0 > P.n0 ? nt0 : P.n0, nB = (nt0 + 32 < P.n0 + P.T) ? nt0 + 32 : P.n0 + P.T;
    const int jA = (int)(nA - nt0), jB = (int)(nB - nt0);   // valid in-tile tokens [jA, jB)
    auto krow = [&](int j) { return P.K + (nt0 + j - P.n0) * (int64_t)D; };
    auto vrow = [&](int j) { return P.V + (nt0 + j - P.n0) * (int64_t)D; };
    if (tid < NG) {   // existing bucket counts (a chunk may start inside a tile of appended tokens)
        s_gbase[tid][0] = jA > 0 ? c.gcnt[(tile * NG + tid) * 2] : 0u;
        s_gbase[tid][1] = jA > 0 ? c.gcnt[(tile * NG + tid) * 2 + 1] : 0u;
    }

    // ====================================================== A: Value selection (warp/token)
    {
        uint32_t *cand = reinterpret_cast<uint32_t *>(wsc);   // [2][CANDMAX]
        uint32_t *vm = cand + 2 * CANDMAX;                      // [DW] the token's outlier mask
        static_assert(2 * CANDMAX * 4 + 8192 / 8 <= 64 * 20 * 4, "warp scratch: candidates + mask");
        __shared__ int s_nc[PW][2];
        for (int j = jA + warp; j < jB; j += PW) {
            const __half *row = vrow(j);
            for (int x = lane; x < DW; x += 32) vm[x] = 0;
            __syncwarp();
            vtoken_warp<NM>(c, row, D, vm, cand, s_nc[warp], tinfo + j * 24, nt0 + j);
            for (int g = lane; g < NG; g += 32) {
                int cnt = 0;
                for (int x = g * (GW / 32); x < (g + 1) * (GW / 32); ++x) cnt += __popc(vm[x]);
                cntV[j * NG + g] = (uint16_t)cnt;
            }
            __syncwarp();
        }
    }

    __syncthreads();   // per-token ENC thresholds of phase A
    pmark();
    // ============================================================ B: Keys (warp/KV head)
    {
        const uint4 *kenc = reinterpret_cast<const uint4 *>(c.kenc);
        const int j = lane;
        const bool valid = j >= jA && j < jB;
        const __half *row = valid ? krow(j) : nullptr;
        for (int h = warp; h < H; h += PW) {
            uint32_t kw[KWH];
#pragma unroll
            for (int w = 0; w < KWH; ++w) kw[w] = 0u;
            uint32_t mw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int a = 0; a < 8; ++a) {   // channels 8a..8a+7 and 64+8a..64+8a+7 of the head
                uint4 u0 = make_uint4(0, 0, 0, 0), u1 = make_uint4(0, 0, 0, 0);
                if (valid) {
                    u0 = *reinterpret_cast<const uint4 *>(row + h * kHeadDim + 8 * a);
                    u1 = *reinterpret_cast<const uint4 *>(row + h * kHeadDim + 64 + 8 * a);
                }
                const uint32_t w0[4] = {u0.x, u0.y, u0.z, u0.w}, w1[4] = {u1.x, u1.y, u1.z, u1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int p = 8 * a + e;   // RoPE pair (p, p + 64)
                    const uint32_t x2 = __byte_perm(w0[e >> 1], w1[e >> 1], (e & 1) ? 0x7632 : 0x5410);
                    const uint4 *te = kenc + ((size_t)(h * kPairs + p) * PS) / 4;
                    uint32_t tw[PS];
#pragma unroll
                    for (int q = 0; q < PS / 4; ++q) {
                        const uint4 t4 = __ldg(te + q);
                        tw[4 * q] = t4.x; tw[4 * q + 1] = t4.y; tw[4 * q + 2] = t4.z; tw[4 * q + 3] = t4.w;
                    }
                    const __half2 x = u2h(x2);
                    const __half2 olo = __hlt2(x, u2h(tw[0])), ohi = __hgt2(x, u2h(tw[1]));
                    __half2 cnt = __hge2(x, u2h(tw[4]));
#pragma unroll
                    for (int q = 1; q < NM; ++q) cnt = __hadd2(cnt, __hge2(x, u2h(tw[4 + q])));
                    cnt = __hfma2(olo, __hsub2(u2h(tw[2]), cnt), cnt);
                    cnt = __hfma2(ohi, __hsub2(u2h(tw[3]), cnt), cnt);
                    const uint32_t pc = h2codes(cnt, BITS);
                    const int bit = 2 * BITS * p, wi = bit >> 5, sh = bit & 31;
                    kw[wi] |= pc << sh;
                    if (sh + 2 * BITS > 32) kw[wi + 1] |= pc >> (32 - sh);
                    const uint32_t ob = h2u(__hadd2(olo, ohi));
                    mw[p >> 5] |= ((ob >> 13) & 1u) << (p & 31);
                    mw[2 + (p >> 5)] |= ((ob >> 29) & 1u) << (p & 31);
                }
            }
            if (valid) {
#pragma unroll
                for (int w = 0; w < KWH; ++w) c.kcodes[(tile * c.QW + h * KWH + w) * 32 + j] = kw[w];
#pragma unroll
                for (int w = 0; w < 4; ++w) kmask[j * DW + h * 4 + w] = mw[w];
            }
            kcnt[j * H + h] = (uint16_t)(valid ? __popc(mw[0]) + __popc(mw[1]) + __popc(mw[2]) + __popc(mw[3]) : 0);
        }
    }
    __syncthreads();
    pmark();

    // ================================ D1: Key-outlier totals, look-back aggregate, counts
    uint32_t lb_tot = 0, lb_agg = 0;   // warp 0: this lane's token total, the tile aggregate
    if (warp == 0) {
        int tot = 0;
        for (int h = 0; h < H; ++h) tot += kcnt[lane * H + h];
        int ex = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ex, o);
            if (lane >= o) ex += y;
        }
        lb_agg = (uint32_t)__shfl_sync(0xffffffffu, ex, 31);
        lb_tot = (uint32_t)tot;
        s_tokbase[lane] = (uint32_t)(ex - tot);
        // publish the aggregate now (decoupled look-back: word = flag << 32 | value); the
        // predecessors are resolved after phase C (next), when they have most likely published
        if (lane == 0) {
            if (li == 0) {
                s_kbase = c.kptr[nA];   // CSC offset of the chunk's first token (prior appends)
                atomicExch(&P.lb[0], ((unsigned long long)LB_INC << 32) | (s_kbase + lb_agg));
            } else {
                atomicExch(&P.lb[li], ((unsigned long long)LB_AGG << 32) | lb_agg);
            }
        }
    } else if (warp == 1) {
        // per (token, group) Key-outlier counts
        for (int g = 0; g < NG; ++g) {
            int cnt = 0;
            for (int h = g * (GW / kHeadDim); h < (g + 1) * (GW / kHeadDim); ++h) cnt += kcnt[lane * H + h];
            cntK[lane * NG + g] = (uint16_t)cnt;
        }
    }
    // ================================================ C: Value codes (warp/KV head, mma lanes)
    {
        // staging (warp scratch): the head's V slice for 64 channels, [token][channel] fp16
        const int vg = lane >> 2, vt = lane & 3;
        // per lane: its 4 token pairs (2u, 2u+1), u = vt + 4 * (2 s + r2), r2 = (j % 16) / 8
        __half2 T2[4][NM], lo2[4], hi2[4];
        uint32_t vmsk[4];
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
            const int ja = 2 * vt + 8 * pr, jb = ja + 1;   // pr = 2 s + r2
            const uint16_t *ta = tinfo + ja * 24, *tb2 = tinfo + jb * 24;
            const bool va = ja >= jA && ja < jB, vb = jb >= jA && jb < jB;
            lo2[pr] = u2h((uint32_t)(va ? ta[TI_LO] : 0) | ((uint32_t)(vb ? tb2[TI_LO] : 0) << 16));
            hi2[pr] = u2h((uint32_t)(va ? ta[TI_HI] : 0) | ((uint32_t)(vb ? tb2[TI_HI] : 0) << 16));
#pragma unroll
            for (int q = 0; q < NM; ++q)
                T2[pr][q] = u2h((uint32_t)(va ? ta[TI_T + q] : 0x7c00u) | ((uint32_t)(vb ? tb2[TI_T + q] : 0x7c00u) << 16));
            vmsk[pr] = (va ? (uint32_t)CM : 0u) | (vb ? (uint32_t)CM << BITS : 0u);
        }
        for (int h = warp; h < H; h += PW) {
            uint32_t vw[KWH];
#pragma unroll
            for (int w = 0; w < KWH; ++w) vw[w] = 0u;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                __syncwarp();
                // stage channels 64*half .. +63 of head h row-major: lane = token, row stride
                // 144 bytes (16-byte stores and ldmatrix row reads hit 8 distinct bank quads)
                {
                    const int j = lane;
                    const bool valid = j >= jA && j < jB;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        uint4 u = make_uint4(0, 0, 0, 0);
                        if (valid) u = *reinterpret_cast<const uint4 *>(vrow(j) + h * kHeadDim + 64 * half + 8 * a);
                        *reinterpret_cast<uint4 *>(wsc + j * 144 + 16 * a) = u;
                    }
                }
                __syncwarp();
#pragma unroll
                for (int mt2 = 0; mt2 < 4; ++mt2) {
                    const int mt = 4 * half + mt2;
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        // the 4 fields r of (mt2, s2) with one ldmatrix.x4.trans: matrix r = tokens
                        // 8 (2 s2 + r / 2) .. +7 x channels 16 mt2 + 8 (r % 2) .. +7; transposed, lane
                        // (g, t) receives tokens 2t, 2t+1 of the block at channel g (one half2)
                        uint32_t xr[4];
                        {
                            const int m = lane >> 3, tok = 8 * (2 * s2 + (m >> 1)) + (lane & 7);
                            const uint32_t ad = (uint32_t)__cvta_generic_to_shared(wsc + tok * 144 + 2 * (16 * mt2 + 8 * (m & 1)));
                            asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(xr[0]), "=r"(xr[1]), "=r"(xr[2]), "=r"(xr[3]) : "r"(ad));
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            // field f = (2 mt + s2) * 4 + r: channel 16 mt + g + 8 (r % 2),
                            // tokens 16 s2 + 2 vt + 8 (r / 2) (+1)
                            const int pr = 2 * s2 + (r >> 1);
                            const uint32_t x2 = xr[r];
                            __half2 x = __hmax2(__hmin2(u2h(x2), hi2[pr]), lo2[pr]);
                            __half2 cnt = __hge2(x, T2[pr][0]);
#pragma unroll
                            for (int q = 1; q < NM; ++q) cnt = __hadd2(cnt, __hge2(x, T2[pr][q]));
                            const uint32_t fv = h2codes(cnt, BITS) & vmsk[pr];
                            const int f = (2 * mt + s2) * 4 + r;
                            const int bit = f * 2 * BITS, wi = bit >> 5, sh = bit & 31;
                            vw[wi] |= fv << sh;
                            if (sh + 2 * BITS > 32) vw[wi + 1] |= fv >> (32 - sh);
                        }
                    }
                }
            }
            // a tile a chunk starts inside already holds codes of appended tokens: OR them in
#pragma unroll
            for (int w = 0; w < KWH; ++w) {
                uint32_t *dst = c.vcodes + vf_word(tile, H, h, w, lane, BITS);
                *dst = jA > 0 ? (*dst | vw[w]) : vw[w];
            }
        }
    }
    __syncthreads();
    pmark();

    // ============================ D1b: look-back resolution (warp 0), bucket slots (others)
    if (warp == 0) {
        if (li > 0) {
            uint32_t excl = 0;
            int jj = li - 1;
            while (true) {
                const int q = jj - lane;
                const unsigned long long v = q >= 0 ? *reinterpret_cast<volatile unsigned long long *>(&P.lb[q])
                                                    : ((unsigned long long)LB_INC << 32);
                const uint32_t fl = (uint32_t)(v >> 32);
                const unsigned inc = __ballot_sync(0xffffffffu, fl == LB_INC);
                const unsigned notready = __ballot_sync(0xffffffffu, fl == 0u);
                const int first = inc ? __ffs(inc) - 1 : 32;
                const unsigned need = first == 32 ? 0xffffffffu : ((2u << first) - 1u);
                if (notready & need) {   // a predecessor in the window has not published: back off
                    __nanosleep(128);      // (frees issue slots for the SM's other CTAs)
                    continue;
                }
                uint32_t val = (lane <= first) ? (uint32_t)v : 0u;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                excl += val;
                if (first < 32) break;
                jj -= 32;
            }
            if (lane == 0) {
                atomicExch(&P.lb[li], ((unsigned long long)LB_INC << 32) | (excl + lb_agg));
                s_kbase = excl;
            }
        }
        __syncwarp();
        // Key CSC column pointers kptr[n+1] of the tile's tokens
        if (lane >= jA && lane < jB) {
            const uint32_t end = s_kbase + s_tokbase[lane] + lb_tot;
            c.kptr[nt0 + lane + 1] = end;
            if ((int64_t)end > c.kcap) *(volatile int *)c.err |= kErrKeyCapacity;
        }
    } else {
        // bucket slots: exclusive prefix over the tile's tokens per group (warp per group)
        for (int g = warp - 1; g < NG; g += PW - 1) {
            const int ck = (lane >= jA && lane < jB) ? cntK[lane * NG + g] : 0;
            const int cv = (lane >= jA && lane < jB) ? cntV[lane * NG + g] : 0;
            int ek = ck, ev = cv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int yk = __shfl_up_sync(0xffffffffu, ek, o), yv = __shfl_up_sync(0xffffffffu, ev, o);
                if (lane >= o) { ek += yk; ev += yv; }
            }
            posK[lane * NG + g] = (uint16_t)(ek - ck);
            posV[lane * NG + g] = (uint16_t)(ev - cv);
            if (lane == 31) {
                c.gcnt[(tile * NG + g) * 2] = s_gbase[g][0] + (uint32_t)ek;
                c.gcnt[(tile * NG + g) * 2 + 1] = s_gbase[g][1] + (uint32_t)ev;
            }
        }
    }
    __syncthreads();
    pmark();

    // ================================ D2: Key CSC records + Key / Value items (warp/token)
    {
        const uint32_t *kenc32 = c.kenc;
        for (int j = jA + warp; j < jB; j += PW) {
            const __half *kr = krow(j);
            uint32_t tb = s_kbase + s_tokbase[j];   // CSC slot of the token's next head chunk
            for (int h0 = 0; h0 < H; h0 += 32) {
                const int h = h0 + lane;
                const int cnt = h < H ? kcnt[j * H + h] : 0;
                int ex = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, ex, o);
                    if (lane >= o) ex += y;
                }
                const int hsum = __shfl_sync(0xffffffffu, ex, 31);
                ex -= cnt;
                if (cnt) {
                    uint32_t pos = tb + (uint32_t)ex;
                    const int g = (h * kHeadDim) / GW;
                    int r = 0;   // rank inside the (token, group): outliers of earlier heads of the group
                    for (int h2 = g * (GW / kHeadDim); h2 < h; ++h2) r += kcnt[j * H + h2];
                    uint32_t bslot = s_gbase[g][0] + posK[j * NG + g] + (uint32_t)r;
                    uint32_t *dst = c.kit + (tile * NG + g) * (int64_t)c.kcap_g;
                    for (int w = 0; w < 4; ++w)
                        for (uint32_t b = kmask[j * DW + h * 4 + w]; b; b &= b - 1) {
                            const int cc = 32 * w + __ffs(b) - 1, ch = h * kHeadDim + cc;
                            // the value and the pair's (lo, code(lo), code(hi)) table words: four
                            // independent loads in flight together
                            const int pp = cc & 63, up = cc >> 6;
                            const uint32_t *te = kenc32 + (size_t)(h * kPairs + pp) * PS;
                            const uint32_t xh = __half_as_ushort(kr[ch]);
                            const uint32_t t0 = __ldg(te), t2 = __ldg(te + 2), t3 = __ldg(te + 3);
                            if ((int64_t)pos < c.kcap) c.kout[pos] = (uint32_t)ch | (xh << 16);
                            ++pos;
                            // dense code at the outlier: clamp to lo -> code_lo, to hi -> code_hi
                            const __half2 lo2 = u2h(t0);
                            const __half xv = __ushort_as_half((uint16_t)xh);
                            const bool below = __hlt(xv, up ? __high2half(lo2) : __low2half(lo2));
                            const uint32_t cw = h2u(__hadd2(u2h(below ? t2 : t3), __float2half2_rn(1024.f)));
                            const int code = (int)((up ? cw >> 16 : cw) & 0xfu);
                            if (bslot < (uint32_t)c.kcap_g)
                                dst[bslot] = (xh << 16) | ((uint32_t)j << 11) | item_code_flag<BITS>(code) |
                                             (uint32_t)(ch - g * GW);
                            ++bslot;
                        }
                }
                tb += (uint32_t)hsum;
            }
            // Value items of the token from its CSR row (phase A: k records in ascending channel
            // order), a lane per record: slot = the group's base + the record's rank in its group
            // (its index minus the token's outliers in earlier groups: a scan of cntV)
            const int kv = c.kv;
            if (kv > 0) {
                const uint16_t *ti = tinfo + j * 24;
                const uint32_t khi = okey(ti[TI_HI]);
                const int c0 = lane < NG ? cntV[j * NG + lane] : 0, c1 = lane + 32 < NG ? cntV[j * NG + 32 + lane] : 0;
                int s0 = c0, s1 = c1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y0 = __shfl_up_sync(0xffffffffu, s0, o), y1 = __shfl_up_sync(0xffffffffu, s1, o);
                    if (lane >= o) { s0 += y0; s1 += y1; }
                }
                const int e0 = s0 - c0, e1 = s1 - c1 + __shfl_sync(0xffffffffu, s0, 31);
                const uint32_t *vo = c.vout + (nt0 + j) * (int64_t)kv;
                for (int eb = 0; eb < kv; eb += 32) {
                    const int e = eb + lane;
                    const uint32_t rec = e < kv ? vo[e] : 0u;
                    const int ch = (int)(rec & 0xffffu), g = ch / GW;
                    const int st0 = __shfl_sync(0xffffffffu, e0, g & 31), st1 = __shfl_sync(0xffffffffu, e1, g & 31);
                    if (e < kv) {
                        const uint32_t bslot = s_gbase[g][1] + posV[j * NG + g] + (uint32_t)(e - (g < 32 ? st0 : st1));
                        const uint32_t xh = rec >> 16;
                        const int code = okey(xh) >= khi ? ti[TI_CHI] : ti[TI_CLO];
                        if (bslot < (uint32_t)c.vcap_g)
                            (c.vit + (tile * NG + g) * (int64_t)c.vcap_g)[bslot] =
                                (xh << 16) | ((uint32_t)j << 11) | item_code_flag<BITS>(code) | (uint32_t)(ch - g * GW);
                    }
                }
            }
        }
    }

    if (P.tm) { __syncthreads(); pmark(); }
}


// ============================================================================ append
// Quantize-on-append of ONE decode token, latency-oriented: one CTA of 32
// warps, every phase spread over the CTA (a single warp's serial selection took 14 of the
// 19 us of the round-2 kernel).
//   1  rows staged in shared memory; warp 31 fetches the CSC base kptr[n] and the bucket counts
//      of the tile at the same time (their latency hides under the staging)
//   2  Value selection by the whole CTA (vselect_block): per-thread groups of 8 elements, the
//      two candidate bounds by warps 0 / 1, candidates compacted by every warp, one rank per
//      thread -- the same bound argument and result as vtoken_warp
//   3  warp 0: (s, z), the token's ENC thresholds, CSR records (vfinish_warp); warps 1..31: Keys,
//      a KV head each: lane = RoPE pairs (lane, lane + 32), codes from the exact fp16 ENC
//      thresholds (kenc), pair-stream words, outlier bits by ballot
//   4  Key CSC slot; Key records + bucket items (warp per head; codes from the pair codes);
//      Value items (thread per mask word); Value codes OR-ed into the fragment-ordered tile
//      words (one OR per two codes)
// The kernel lets a dependent attend launch at once (programmatic dependent launch; its
// prologue reads no cache data).
constexpr int AT = 1024, AW = AT / 32;

// Block-wide selection of the token's ku largest and then kl smallest Values (R2, R3), into vm
// (D/32 words), and the kept min / max fp16 bits (lowest index attaining them, R7).  Groups of 8
// elements per thread: the (ku+1)-th largest group max tau bounds the ku + 1 largest elements
// from below for any grouping, so the candidates (elements >= tau) contain them; each candidate
// is ranked by (value desc, index asc) against the others.  The exact warp path takes over when
// the bound admits more than CANDMAX candidates (ties, tiny D).  sh: [8] shared ints.
__device__ void vselect_block(const __half *row, int D, int ku, int kl, uint32_t *vm, uint32_t *cand,
                              uint32_t *gk, uint32_t *gl, int *sh, uint32_t &lo_h, uint32_t &hi_h) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ng = D / 8, DW = D / 32;
    for (int x = tid; x < DW; x += AT) vm[x] = 0;
    if (tid < 8) sh[tid] = 0;
    const bool act = tid < ng;
    uint4 u = make_uint4(0, 0, 0, 0);
    uint32_t kmax = 0, kmin = 0xffffu;
    if (act) {
        u = *reinterpret_cast<const uint4 *>(row + 8 * tid);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t k = okey(e & 1 ? w[e >> 1] >> 16 : w[e >> 1]);
            kmax = max(kmax, k);
            kmin = min(kmin, k);
        }
    }
    // the bounds: a high-byte histogram of the group maxima (and of the mirrored minima); tau =
    // the lowest key of the bin holding the (ku+1)-th largest, a valid (slightly lower) bound
    uint32_t *hist = gk;   // [2][256]
    if (tid < 512) hist[tid] = 0;
    __syncthreads();
    if (act) {
        atomicAdd(&hist[kmax >> 8], 1u);
        atomicAdd(&hist[256 + ((0xffffu - kmin) >> 8)], 1u);
    }
    __syncthreads();
    if (warp < 2) {   // warp 0: upper side, warp 1: lower side (mirrored keys)
        const uint32_t *hh = hist + 256 * warp;
        const int need = warp == 0 ? ku + 1 : kl + 1;
        int cb[8], sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { cb[q] = (int)hh[255 - 8 * lane - q]; sum += cb[q]; }   // descending bins
        int inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const int exc = inc - sum;
        const bool mine = exc < need && need <= inc;
        int bin = 0;
        if (mine) {
            int run = exc;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (run < need && need <= run + cb[q]) bin = 255 - 8 * lane - q;
                run += cb[q];
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, mine);
        bin = bal ? __shfl_sync(0xffffffffu, bin, __ffs(bal) - 1) : 0;   // none: fewer groups than need
        if (lane == 0) sh[2 + warp] = (int)(warp == 0 ? ((uint32_t)bin << 8) : 0xffffu - ((uint32_t)bin << 8));
    }
    __syncthreads();
    const uint32_t tau_hi = (uint32_t)sh[2], tau_lo = (uint32_t)sh[3];
    // candidates, compacted per warp
    uint32_t fu = 0, fl = 0;
    if (act) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t k = okey(e & 1 ? w[e >> 1] >> 16 : w[e >> 1]);
            fu |= (uint32_t)(k >= tau_hi) << e;
            fl |= (uint32_t)(k <= tau_lo) << e;
        }
    }
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const uint32_t f = side ? fl : fu;
        const int cntl = __popc(f);
        int inc = cntl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        int base = 0;
        if (lane == 31 && inc) base = atomicAdd(&sh[side], inc);
        base = __shfl_sync(0xffffffffu, base, 31) + inc - cntl;
        for (uint32_t x = f; x; x &= x - 1) {
            const int e = __ffs(x) - 1, ch = 8 * tid + e;
            const uint32_t k = okey(half_at(u, e));
            if (base < CANDMAX)
                cand[side * CANDMAX + base] = ((side ? 0xffffu - k : k) << 13) | (8191u - (uint32_t)ch);
            ++base;
        }
    }
    __syncthreads();
    const int NU = sh[0], NL = sh[1];
    const bool ovf = NU > CANDMAX || NL > CANDMAX || NU < ku + 1 || NL < kl + 1 || tau_lo >= tau_hi;
    if (!ovf) {
        const int side = tid >= AT / 2 ? 1 : 0, i = tid - side * (AT / 2);
        const int nn = side ? NL : NU, kk = side ? kl : ku;
        if (i < nn) {
            const uint32_t *cs = cand + side * CANDMAX;
            const uint32_t v = cs[i];
            int r = 0;
            for (int q = 0; q < nn; ++q) r += cs[q] > v ? 1 : 0;
            const int ch = 8191 - (int)(v & 8191u);
            if (r < kk) atomicOr(&vm[ch >> 5], 1u << (ch & 31));
            if (r == kk) sh[4 + side] = ch;
        }
        __syncthreads();
        hi_h = __half_as_ushort(row[sh[4]]);
        lo_h = __half_as_ushort(row[sh[5]]);
    } else {
        if (warp == 0) {
            uint32_t l, h;
            vselect_exact_warp(row, D, ku, kl, vm, l, h);
            if (lane == 0) { sh[6] = (int)l; sh[7] = (int)h; }
        }
        __syncthreads();
        lo_h = (uint32_t)sh[6];
        hi_h = (uint32_t)sh[7];
    }
}

template <int BITS>
__global__ void __launch_bounds__(AT, 1) append_kernel(DevCache c, const __half *K, const __half *V, int64_t n,
                                                        unsigned long long *tr) {
    asm volatile("griddepcontrol.launch_dependents;");
    // diagnostics: %globaltimer at phase ends, max over the threads that reach them
    auto stamp = [&](int i) {
        if (tr) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(tr + i, t);
        }
    };
    if (threadIdx.x == 0) stamp(0);
    using Cf = PCfg<BITS>;
    constexpr int NM = Cf::NM, PS = Cf::PS, CM = (1 << BITS) - 1, KWH = 4 * BITS;
    __shared__ uint32_t vm[8192 / 32], cand[2 * CANDMAX], kmh[64 * 4];
    // group bounds of the selection, then (dead by then) the pair codes of the Keys
    __shared__ __align__(16) uint32_t gkl[2 * AT];
    uint32_t *gk = gkl, *gl = gkl + AT;
    uint8_t *pcs = reinterpret_cast<uint8_t *>(gkl);   // [64 heads][64 pairs]
    __shared__ int sh[8], kcnt[64], kbase[64], gslotK[64], gslotV[64];
    __shared__ uint16_t ti[24];
    __shared__ uint32_t s_kb0, s_ok;
    __shared__ double s_mids[16];
    __shared__ __align__(16) __half ks[8192], vs[8192];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = c.D, H = c.H_kv, NG = c.NG, GW = c.GW, DW = D / 32;
    const int64_t tile = n >> 5;
    const int jj = (int)(n & 31);
    const int k = c.kv, ku = (k + 1) / 2, kl = k / 2;
    // 1: rows -> shared; the CSC base and the tile's bucket counts fetched alongside
    for (int x = tid; x < D / 8; x += AT) {
        reinterpret_cast<uint4 *>(ks)[x] = reinterpret_cast<const uint4 *>(K)[x];
        reinterpret_cast<uint4 *>(vs)[x] = reinterpret_cast<const uint4 *>(V)[x];
    }
    if (warp == AW - 1) {
        if (lane == 0) s_kb0 = c.kptr[n];
        if (lane < 16) s_mids[lane] = c.mids[16 + lane];
        for (int g = lane; g < NG; g += 32) {
            gslotK[g] = (int)c.gcnt[(tile * NG + g) * 2];
            gslotV[g] = (int)c.gcnt[(tile * NG + g) * 2 + 1];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(1);
    K = ks;
    V = vs;

    // 2: Value selection, whole CTA
    uint32_t lo_h, hi_h;
    vselect_block(V, D, ku, kl, vm, cand, gk, gl, sh, lo_h, hi_h);
    if (threadIdx.x == 0) stamp(8);

    if (warp == 0) {
        // 3a: (s, z), thresholds, CSR records
        vfinish_warp<NM>(c, V, D, vm, lo_h, hi_h, ti, n, s_mids);
        if (lane == 0) stamp(2);
    } else {
        // 3b: Keys (warps 1..31)
        const uint4 *kenc = reinterpret_cast<const uint4 *>(c.kenc);
        for (int h = warp - 1; h < H; h += AW - 1) {
            uint32_t ob01[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int p = lane + 32 * q;
                const uint32_t x2 = (uint32_t)__half_as_ushort(K[h * kHeadDim + p]) |
                                    ((uint32_t)__half_as_ushort(K[h * kHeadDim + p + kPairs]) << 16);
                const uint4 *te = kenc + ((size_t)(h * kPairs + p) * PS) / 4;
                uint32_t tw[PS];
#pragma unroll
                for (int r = 0; r < PS / 4; ++r) {
                    const uint4 t4 = __ldg(te + r);
                    tw[4 * r] = t4.x; tw[4 * r + 1] = t4.y; tw[4 * r + 2] = t4.z; tw[4 * r + 3] = t4.w;
                }
                const __half2 x = u2h(x2);
                const __half2 olo = __hlt2(x, u2h(tw[0])), ohi = __hgt2(x, u2h(tw[1]));
                __half2 cnt = __hge2(x, u2h(tw[4]));
#pragma unroll
                for (int r = 1; r < NM; ++r) cnt = __hadd2(cnt, __hge2(x, u2h(tw[4 + r])));
                cnt = __hfma2(olo, __hsub2(u2h(tw[2]), cnt), cnt);
                cnt = __hfma2(ohi, __hsub2(u2h(tw[3]), cnt), cnt);
                pcs[h * 64 + p] = (uint8_t)h2codes(cnt, BITS);
                ob01[q] = h2u(__hadd2(olo, ohi));
            }
            // outlier bits of channels lane, lane + 32 (low halves) and lane + 64, + 96 (high)
            const uint32_t m0 = __ballot_sync(0xffffffffu, (ob01[0] >> 13) & 1u);
            const uint32_t m1 = __ballot_sync(0xffffffffu, (ob01[1] >> 13) & 1u);
            const uint32_t m2 = __ballot_sync(0xffffffffu, (ob01[0] >> 29) & 1u);
            const uint32_t m3 = __ballot_sync(0xffffffffu, (ob01[1] >> 29) & 1u);
            if (lane == 0) {
                kmh[h * 4 + 0] = m0; kmh[h * 4 + 1] = m1; kmh[h * 4 + 2] = m2; kmh[h * 4 + 3] = m3;
                kcnt[h] = __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3);
            }
            __syncwarp();
            // the head's pair-stream words: pair p occupies bits [2b p, 2b p + 2b)
            if (lane < KWH) {
                const int w = lane;
                uint32_t word = 0;
                const int p0 = (32 * w) / (2 * BITS), p1 = min(kPairs - 1, (32 * w + 31) / (2 * BITS));
                for (int p = p0; p <= p1; ++p) {
                    const int sh2 = 2 * BITS * p - 32 * w;
                    const uint32_t pc = pcs[h * 64 + p];
                    word |= sh2 >= 0 ? (pc << sh2) : (pc >> -sh2);
                }
                c.kcodes[(tile * c.QW + h * KWH + w) * 32 + jj] = word;
            }
        }
        if (lane == 0) stamp(3);
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(4);
    // 4a: Key CSC slot (warp 0)
    if (warp == 0) {
        int e0 = lane < H ? kcnt[lane] : 0, e1 = lane + 32 < H ? kcnt[lane + 32] : 0;
        int x0 = e0, x1 = e1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
            if (lane >= o) { x0 += y0; x1 += y1; }
        }
        const int t0 = __shfl_sync(0xffffffffu, x0, 31);
        if (lane < H) kbase[lane] = x0 - e0;
        if (lane + 32 < H) kbase[lane + 32] = t0 + x1 - e1;
        const int total = t0 + __shfl_sync(0xffffffffu, x1, 31);
        if (lane == 0) {
            const uint32_t base = s_kb0;
            const bool ok = (int64_t)base + total <= c.kcap;
            if (!ok) *(volatile int *)c.err |= kErrKeyCapacity;
            c.kptr[n + 1] = ok ? base + (uint32_t)total : base;
            s_ok = ok;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(5);
    // 4b: Key records + items (warps 1..31, a head each); Value items (thread per mask word of
    // warp 0, in channel order within each group)
    if (warp > 0) {
        for (int h = warp - 1; h < H; h += AW - 1) {
            if (kcnt[h] == 0) continue;
            const int g = (h * kHeadDim) / GW;
            int before = 0;   // the group's records of earlier heads (channel order)
            for (int h2 = (g * GW) / kHeadDim; h2 < h; ++h2) before += kcnt[h2];
            int rank = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t m = kmh[h * 4 + w];
                if ((m >> lane) & 1u) {
                    const int r = rank + __popc(m & ((1u << lane) - 1u));
                    const int cc = 32 * w + lane, ch = h * kHeadDim + cc;
                    const uint32_t xh = __half_as_ushort(K[ch]);
                    if (s_ok) c.kout[s_kb0 + (uint32_t)(kbase[h] + r)] = (uint32_t)ch | (xh << 16);
                    const uint32_t pc = pcs[h * 64 + (cc & 63)];
                    const int code = (int)((cc >> 6) ? (pc >> BITS) : (pc & CM));
                    const int slot = gslotK[g] + before + r;
                    if (slot < c.kcap_g)
                        c.kit[(tile * NG + g) * (int64_t)c.kcap_g + slot] =
                            (xh << 16) | ((uint32_t)jj << 11) | item_code_flag<BITS>(code) | (uint32_t)(ch - g * GW);
                }
                rank += __popc(m);
            }
        }
    } else {
        const uint32_t khi = okey(ti[TI_HI]);
        const int wpg = GW / 32;   // mask words per group
        for (int x = lane; x < DW; x += 32) {
            const int g = x / wpg;
            int slot = gslotV[g];
            for (int x2 = g * wpg; x2 < x; ++x2) slot += __popc(vm[x2]);
            for (uint32_t b = vm[x]; b; b &= b - 1) {
                const int ch = 32 * x + __ffs(b) - 1;
                const uint32_t xh = __half_as_ushort(V[ch]);
                const int code = okey(xh) >= khi ? ti[TI_CHI] : ti[TI_CLO];
                if (slot < c.vcap_g)
                    c.vit[(tile * NG + g) * (int64_t)c.vcap_g + slot] =
                        (xh << 16) | ((uint32_t)jj << 11) | item_code_flag<BITS>(code) | (uint32_t)(ch - g * GW);
                ++slot;
            }
        }
        // new counts (>= cap: the attend kernels use the CSC / CSR arrays for the tile)
        for (int g = lane; g < NG; g += 32) {
            int kc = 0, vc = 0;
            for (int h2 = (g * GW) / kHeadDim; h2 < ((g + 1) * GW) / kHeadDim; ++h2) kc += kcnt[h2];
            for (int x2 = g * wpg; x2 < (g + 1) * wpg; ++x2) vc += __popc(vm[x2]);
            c.gcnt[(tile * NG + g) * 2] = (uint32_t)(gslotK[g] + kc);
            c.gcnt[(tile * NG + g) * 2 + 1] = (uint32_t)(gslotV[g] + vc);
        }
    }
    if (lane == 0) stamp(6);
    // 4c: Value codes (every thread).  Channels cc and cc + 8 of a head share a lane of the
    // fragment layout and sit 2b bits apart: one OR per two codes (the words are shared with the
    // tile's other tokens)
    {
        const __half lo = __ushort_as_half(ti[TI_LO]), hi = __ushort_as_half(ti[TI_HI]);
        __half T[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) T[q] = __ushort_as_half(ti[TI_T + q]);
        for (int x = tid; x < H * 64; x += AT) {
            const int hh = x >> 6, mt = (x >> 3) & 7, g8 = x & 7;
            const int cc = mt * 16 + g8;
            uint32_t v = 0;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                __half y = V[hh * kHeadDim + cc + 8 * e];
                y = __hmax(__hmin(y, hi), lo);
                int code = 0;
#pragma unroll
                for (int q = 0; q < NM; ++q) code += __hge(y, T[q]) ? 1 : 0;
                v |= (uint32_t)code << (2 * BITS * e);
            }
            const int bit = vf_bit(jj, cc, BITS);
            const int ln = vf_lane(jj, cc), w = bit >> 5, off = bit & 31;
            uint32_t *dst = c.vcodes + vf_word(tile, H, hh, w, ln, BITS);
            atomicOr(dst, v << off);
            if (off + 3 * BITS > 32) atomicOr(dst + 32, v >> (32 - off));
        }
    }
    if (lane == 0) stamp(7);
}

}  // namespace

size_t prefill_smem_bytes(int D, int NG) { return PSmem(D, NG).total; }

cudaError_t launch_append(const DevCache &c, const __half *K, const __half *V, int64_t n, cudaStream_t s,
                          unsigned long long *tr) {
    switch (c.bits) {
        case 2: append_kernel<2><<<1, AT, 0, s>>>(c, K, V, n, tr); break;
        case 3: append_kernel<3><<<1, AT, 0, s>>>(c, K, V, n, tr); break;
        case 4: append_kernel<4><<<1, AT, 0, s>>>(c, K, V, n, tr); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_prefill(const DevCache &c, const __half *K, const __half *V, int64_t n0, int64_t T,
                           unsigned long long *lb, unsigned *ticket, cudaStream_t s, unsigned long long *tm) {
    if (T <= 0) return cudaSuccess;
    PParams P;
    P.K = K; P.V = V; P.n0 = n0; P.T = T;
    P.tile0 = n0 / 32;
    const int64_t tile1 = (n0 + T - 1) / 32;
    P.ntile = (int)(tile1 - P.tile0 + 1);
    P.lb = lb; P.ticket = ticket; P.tm = tm;
    cudaError_t e = cudaMemsetAsync(lb, 0, (size_t)P.ntile * 8, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ticket, 0, 4, s);
    if (e != cudaSuccess) return e;
    const size_t smem = prefill_smem_bytes(c.D, c.NG);
    switch (c.bits) {
        case 2:
            cudaFuncSetAttribute(prefill_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            prefill_kernel<2><<<P.ntile, PT, smem, s>>>(c, P);
            break;
        case 3:
            cudaFuncSetAttribute(prefill_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            prefill_kernel<3><<<P.ntile, PT, smem, s>>>(c, P);
            break;
        case 4:
            cudaFuncSetAttribute(prefill_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            prefill_kernel<4><<<P.ntile, PT, smem, s>>>(c, P);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace kvq
