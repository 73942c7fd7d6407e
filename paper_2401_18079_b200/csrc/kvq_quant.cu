// kvq_quant.cu -- QZ: quantize-on-append (decode) and block prefill quantization.
//
// One CTA per token (256 threads).  Per token:
//   Keys: outlier iff x < lo_c || x > hi_c (R4); code =
//         ENC(clamp(x); s_c, z_c) (R5, R8); outliers appended to the CSC tail in
//         ascending channel order.
//   Values (topk P:1028-1031): two-sided top-k with
//         k = ceil(f*D): ceil(k/2) largest then floor(k/2) smallest of the rest,
//         ties to the lower index, -0 == +0 (R2, R3), done as a CTA radix select on
//         order-preserving 16-bit keys; (s, z) from the kept [lo, hi] in fp64 rounded
//         once to fp32 (R6, R7); code = ENC(clamp(v)).
//   ENC: code = #{j : 2(y - z) > s (c_j + c_{j+1})} in fp64 with explicit round-to-
//         nearest intrinsics (no contraction), evaluated as a binary search since the
//         predicate is monotone in j for an ascending codebook (R8).  Taking this
//         integer decision in fp64 on both sides is what makes codes bit-exact.
//   Packing: Key tile layout / Value canonical rows (kvq_internal.cuh).
// Modes: 0 = single decode append (count, CTA scan, tail append, kptr[n+1]);
//        1 = prefill pass 1 (Key-outlier counts only);
//        2 = prefill pass 3 (everything, Key-outlier base from the scanned kptr).
#include "kvq_internal.cuh"

namespace kvq {
namespace {

constexpr int QZ_THREADS = 256;     // prefill: one CTA per token, many CTAs
constexpr int QZ_THREADS_1 = 1024;  // single decode append: one CTA does all the work

__device__ __forceinline__ uint16_t f16_order_key(uint16_t h) {
    if (h == 0x8000u) h = 0;                         // -0 == +0 (R3)
    return (h & 0x8000u) ? (uint16_t)(~h) : (uint16_t)(h | 0x8000u);
}

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// Exact ENC (R8): count of midpoints with 2(y-z) > s*m_j.
// The predicate 2(y-z) > s*m_j is true exactly for j < code (m ascending, s >= 0), so the
// count is found in log2(NLEV) steps: code += step when the predicate holds at code+step-1.
template <int NM>
__device__ __forceinline__ int enc_fp64(double y, double s, double z, const double *mids) {
    const double lhs = 2.0 * __dsub_rn(y, z);
    int code = 0;
#pragma unroll
    for (int step = (NM + 1) / 2; step >= 1; step >>= 1)
        if (lhs > __dmul_rn(s, mids[code + step - 1])) code += step;
    return code;
}

// Block-wide exclusive scan of one int per thread; returns exclusive prefix, *total.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int *total, int *sbuf /*[NT/32+1]*/) {
    constexpr int QZ_WARPS = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sbuf[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int w = 0; w < QZ_WARPS; ++w) { int t = sbuf[w]; sbuf[w] = acc; acc += t; }
        sbuf[QZ_WARPS] = acc;
    }
    __syncthreads();
    int res = sbuf[warp] + x - v;
    *total = sbuf[QZ_WARPS];
    return res;
}

// Histogram add with warp aggregation: lanes hitting the same bin are merged with
// match.any, so a concentrated value distribution does not serialize on one bank.
__device__ __forceinline__ void hist_add(int *hist, int bin, bool valid) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (valid) {
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
}

// Warp 0 finds, walking bins from 255 down, the bin `sel` where the running count reaches
// `need`, and the count strictly above it (`above`).  Parallel: 8 bins per lane + a
// warp scan, no serial 256-step walk.
__device__ __forceinline__ void select_bin(const int *hist, int need, int *out /*[2]*/) {
    const int lane = threadIdx.x & 31;
    int c[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k] = hist[255 - (8 * lane + k)]; sum += c[k]; }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int excl = incl - sum;
    if (excl < need && need <= incl) {
        int cum = excl;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (cum + c[k] >= need) { out[0] = 255 - (8 * lane + k); out[1] = cum; break; }
            cum += c[k];
        }
    }
}

// Radix select over 16-bit keys of the "candidate" elements: returns tau such that
// #(cand with key' > tau) < need <= #(cand with key' >= tau), where key' = key (desc=1)
// or 0xffff - key (desc=0, i.e. ascending order).  Also returns #(key' > tau).
// Loop trip counts are uniform across the CTA (E elements per thread).
template <int NT>
__device__ void radix_select16(const uint16_t *keys, const uint8_t *flags, int D, int c_begin,
                               int E, int o16, int o8, int need, bool desc, int *hist /*[256]*/,
                               int *shared_out /*[4]*/, int *tau_out, int *gt_out) {
    int prefix_hi = -1;   // selected high byte
    int gt = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int b = threadIdx.x; b < 256; b += NT) hist[b] = 0;
        __syncthreads();
        for (int e = 0; e < E; ++e) {
            const int c = c_begin + e;
            bool valid = c < D && !flags[c + o8];
            int kk = 0;
            if (valid) kk = desc ? keys[c + o16] : (0xffff - keys[c + o16]);
            if (pass == 0) {
                hist_add(hist, kk >> 8, valid);   // top bytes cluster: aggregate per warp
            } else if (valid && (kk >> 8) == prefix_hi) {
                atomicAdd(&hist[kk & 0xff], 1);   // few candidates, spread low bytes
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) select_bin(hist, need - gt, shared_out);
        __syncthreads();
        const int sel = shared_out[0];
        gt += shared_out[1];
        if (pass == 0) prefix_hi = sel;
        else *tau_out = (prefix_hi << 8) | sel;
        __syncthreads();
    }
    *gt_out = gt;
}

template <int BITS, int NT>
__global__ void __launch_bounds__(NT)
qz_kernel(DevCache c, const __half *__restrict__ Kin, const __half *__restrict__ Vin, int64_t n0,
          int mode, int part0) {
    // part: 0 = Keys and Values of the token; 1 = Keys only, 2 = Values only (a single decode
    // append runs the two halves as two CTAs, so its latency is the longer half, not the sum)
    const int part = part0 < 0 ? 1 + (int)blockIdx.x : part0;
    // a decode append lets a dependent attend launch now (its prologue reads no cache data)
    if (part0 < 0) asm volatile("griddepcontrol.launch_dependents;");
    constexpr int NLEV = 1 << BITS;
    constexpr int NM = NLEV - 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const int D = c.D;
    // Per-channel arrays, thread-contiguous ownership (E channels per thread).  Each thread's
    // segment is padded (2 halves / 4 bytes) when its stride in words would be even, so the
    // threads of a warp reading "their e-th channel" hit distinct banks (unpadded, E = 16 was
    // 8-way conflicted on the 16-bit arrays and 4-way on the byte arrays).
    const int E = (D + NT - 1) / NT;
    const int pad16 = (E % 4 == 0) ? 2 : 0;
    const int pad8 = (E % 8 == 0) ? 4 : 0;
    const int L16 = D + NT * pad16, L8 = D + NT * pad8;
    uint16_t *xk = reinterpret_cast<uint16_t *>(smem);          // [L16]
    uint16_t *xv = xk + L16;                                      // [L16]
    uint16_t *vkey = xv + L16;                                    // [L16]
    uint8_t *kc = reinterpret_cast<uint8_t *>(vkey + L16);        // [L8]
    uint8_t *vc = kc + L8;                                        // [L8]
    uint8_t *vflag = vc + L8;                                     // [L8]
    int *hist = reinterpret_cast<int *>(vflag + ((L8 + 15) & ~15));// [256]
    int *sbuf = hist + 256;                                       // [64]
    int *sout = sbuf + 64;                                        // [64]
    float *fred = reinterpret_cast<float *>(sout + 64);           // [64]
    constexpr int QZ_WARPS = NT / 32;
    __shared__ double s_mk[16], s_mv[16];

    const int64_t t = part0 < 0 ? 0 : blockIdx.x;
    const int64_t n = n0 + t;
    const int tid = threadIdx.x;
    // padded index of channel ch (any thread) and this thread's offsets for its own channels
    const unsigned long long einv = ((1ull << 20) + E - 1) / E;   // exact ch / E for ch < 8192
    auto seg = [&](int ch) -> int { return (int)(((unsigned long long)ch * einv) >> 20); };
    auto I16 = [&](int ch) -> int { return ch + seg(ch) * pad16; };
    auto I8 = [&](int ch) -> int { return ch + seg(ch) * pad8; };
    const int o16 = tid * pad16, o8 = tid * pad8;
    const __half *krow = Kin + t * (int64_t)D;
    const __half *vrow = Vin + t * (int64_t)D;
    const uint16_t *kr16 = reinterpret_cast<const uint16_t *>(krow);
    const uint16_t *vr16 = reinterpret_cast<const uint16_t *>(vrow);

    if (tid < NM) { s_mk[tid] = c.mids[tid]; s_mv[tid] = c.mids[16 + tid]; }
    // thread-contiguous channel ownership keeps ranks in ascending channel order
    const int cb0 = min(D, tid * E), cb1 = min(D, cb0 + E);
    for (int i = cb0; i < cb1; ++i) {
        if (part != 2) xk[i + o16] = kr16[i];
        if (mode != 1 && part != 1) { uint16_t v = vr16[i]; xv[i + o16] = v; vkey[i + o16] = f16_order_key(v); vflag[i + o8] = 0; }
    }
    __syncthreads();

    const float *ks = c.kpar, *kz = c.kpar + D, *klo = c.kpar + 2 * D, *khi = c.kpar + 3 * D;

    if (part != 2) {   // Keys (the whole Key half of the token)
    // ------------------------------------------------------------------ Keys
    int kcnt = 0;
    uint32_t kmask = 0;   // outlier flags of this thread's channels (E <= 32)
    for (int ch = cb0; ch < cb1; ++ch) {
        float x = h2f(xk[ch + o16]);
        float lo = klo[ch], hi = khi[ch];
        bool out = (x < lo) || (x > hi);
        kcnt += out;
        kmask |= (uint32_t)out << (ch - cb0);
        if (mode != 1) {
            float y = x < lo ? lo : (x > hi ? hi : x);
            kc[ch + o8] = (uint8_t)enc_fp64<NM>((double)y, (double)ks[ch], (double)kz[ch], s_mk);
        }
    }
    int ktotal;
    int krank = block_excl_scan<NT>(kcnt, &ktotal, sbuf);
    if (mode == 1) {
        if (tid == 0) c.counts[t] = ktotal;
        return;
    }
    {
        __shared__ uint32_t s_base;
        __shared__ int s_ok;
        if (tid == 0) {
            uint32_t base = c.kptr[n];
            uint32_t end;
            if (mode == 0) {
                end = base + (uint32_t)ktotal;
                bool ok = (int64_t)end <= c.kcap;
                if (!ok) { end = base; *(volatile int *)c.err |= kErrKeyCapacity; }
                c.kptr[n + 1] = end;
                s_ok = ok;
            } else {
                end = c.kptr[n + 1];
                bool ok = (int64_t)end <= c.kcap;
                if (!ok) *(volatile int *)c.err |= kErrKeyCapacity;
                s_ok = ok;
            }
            s_base = base;
        }
        __syncthreads();
        if (s_ok) {
            uint32_t pos = s_base + (uint32_t)krank;
            for (uint32_t m = kmask; m; m &= m - 1) {
                const int ch = cb0 + __ffs(m) - 1;
                c.kout[pos++] = (uint32_t)ch | ((uint32_t)xk[ch + o16] << 16);
            }
        }
    }
    // ---- Key outliers bucketed per (tile, attend head group).  The group is taken per record
    //      from its channel (a thread's channel chunk may straddle two groups, e.g. E = 20
    //      channels per thread against 256-channel groups at D = 5120); records of a group have
    //      contiguous ranks (ascending channel order), so a record's slot is the group's base
    //      plus its rank minus the group's first rank.  count > cap = overflow.
    {
        __shared__ int gk[64], gbk[64], gfirst[64];
        if (tid < 64) { gk[tid] = 0; gfirst[tid] = 0x7fffffff; }
        __syncthreads();
        {
            int r = krank;
            for (uint32_t m = kmask; m; m &= m - 1, ++r) {
                const int g = (cb0 + __ffs(m) - 1) / c.GW;
                atomicAdd(&gk[g], 1);
                atomicMin(&gfirst[g], r);
            }
        }
        __syncthreads();
        if (tid < c.NG) {
            const int tile0 = (int)(n >> 5);
            gbk[tid] = gk[tid] ? (int)atomicAdd(&c.gcnt[((int64_t)tile0 * c.NG + tid) * 2], (uint32_t)gk[tid]) : 0;
        }
        __syncthreads();
        if (kcnt) {
            const int tile0 = (int)(n >> 5), jj0 = (int)(n & 31);
            int r = krank;
            for (uint32_t m = kmask; m; m &= m - 1, ++r) {
                const int ch = cb0 + __ffs(m) - 1;
                const int g = ch / c.GW;
                const int pos = gbk[g] + (r - gfirst[g]);
                if (pos < c.kcap_g)
                    c.kit[((int64_t)tile0 * c.NG + g) * c.kcap_g + pos] =
                        ((uint32_t)xk[ch + o16] << 16) | ((uint32_t)jj0 << 11) | item_code_flag<BITS>(kc[ch + o8]) |
                        (uint32_t)(ch - g * c.GW);
            }
        }
    }

    }
    if (part != 1) {   // Values
    // ----------------------------------------------------------------- Values
    const int k = c.kv;
    const int ku = (k + 1) / 2, kl = k / 2;
    for (int sel = 0; sel < 2; ++sel) {
        const int need = sel == 0 ? ku : kl;
        if (need == 0) continue;
        const bool desc = (sel == 0);
        int tau, gt;
        radix_select16<NT>(vkey, vflag, D, tid * E, E, o16, o8, need, desc, hist, sout, &tau, &gt);
        // ties at tau: lowest channel index first
        int ties = 0;
        for (int ch = cb0; ch < cb1; ++ch) {
            if (vflag[ch + o8]) continue;
            int kk = desc ? vkey[ch + o16] : (0xffff - vkey[ch + o16]);
            ties += (kk == tau);
        }
        int tt;
        int trank = block_excl_scan<NT>(ties, &tt, sbuf);
        const int take = need - gt;
        for (int ch = cb0; ch < cb1; ++ch) {
            if (vflag[ch + o8]) continue;
            int kk = desc ? vkey[ch + o16] : (0xffff - vkey[ch + o16]);
            if (kk > tau) vflag[ch + o8] = 1 + sel;
            else if (kk == tau) { if (trank < take) vflag[ch + o8] = 1 + sel; ++trank; }
        }
        __syncthreads();
    }

    // kept range: value min/max, then the lowest-index element attaining it
    float vmin = INFINITY, vmax = -INFINITY;
    for (int ch = cb0; ch < cb1; ++ch) {
        if (vflag[ch + o8]) continue;
        float x = h2f(xv[ch + o16]);
        vmin = fminf(vmin, x);
        vmax = fmaxf(vmax, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    if ((tid & 31) == 0) { fred[tid >> 5] = vmin; fred[32 + (tid >> 5)] = vmax; }
    __syncthreads();
    if (tid == 0) {
        float a = fred[0], b = fred[32];
        for (int w = 1; w < QZ_WARPS; ++w) { a = fminf(a, fred[w]); b = fmaxf(b, fred[32 + w]); }
        fred[0] = a; fred[32] = b;
    }
    __syncthreads();
    vmin = fred[0]; vmax = fred[32];
    int imin = 0x7fffffff, imax = 0x7fffffff;
    for (int ch = cb0; ch < cb1; ++ch) {
        if (vflag[ch + o8]) continue;
        float x = h2f(xv[ch + o16]);
        if (x == vmin && imin == 0x7fffffff) imin = ch;
        if (x == vmax && imax == 0x7fffffff) imax = ch;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        imin = min(imin, __shfl_xor_sync(0xffffffffu, imin, o));
        imax = min(imax, __shfl_xor_sync(0xffffffffu, imax, o));
    }
    __syncthreads();
    if ((tid & 31) == 0) { sbuf[tid >> 5] = imin; sout[tid >> 5] = imax; }
    __syncthreads();
    __shared__ double s_lo, s_hi, s_s, s_z;
    if (tid == 0) {
        int a = sbuf[0], b = sout[0];
        for (int w = 1; w < QZ_WARPS; ++w) { a = min(a, sbuf[w]); b = min(b, sout[w]); }
        double lo = (double)h2f(xv[I16(a)]), hi = (double)h2f(xv[I16(b)]);
        float s = __double2float_rn(__dsub_rn(hi, lo) / 2.0);
        float z = __double2float_rn(__dadd_rn(hi, lo) / 2.0);
        s_lo = lo; s_hi = hi; s_s = (double)s; s_z = (double)z;
        c.vsz[n] = make_float2(s, z);
    }
    __syncthreads();
    {
        const double lo = s_lo, hi = s_hi, s = s_s, z = s_z;
        int vcnt = 0;
        for (int ch = cb0; ch < cb1; ++ch) {
            double x = (double)h2f(xv[ch + o16]);
            double y = x < lo ? lo : (x > hi ? hi : x);
            vc[ch + o8] = (uint8_t)enc_fp64<NM>(y, s, z, s_mv);
            vcnt += vflag[ch + o8] != 0;
        }
        int vtot;
        int vr = block_excl_scan<NT>(vcnt, &vtot, sbuf);
        uint32_t *vo = c.vout + n * (int64_t)k;
        // Value outliers bucketed per (tile, group) as for the Keys (group per record)
        __shared__ int gvc[64], gbv[64], gvf[64];
        if (tid < 64) { gvc[tid] = 0; gvf[tid] = 0x7fffffff; }
        __syncthreads();
        {
            int r = vr;
            for (int ch = cb0; ch < cb1; ++ch)
                if (vflag[ch + o8]) {
                    const int g = ch / c.GW;
                    atomicAdd(&gvc[g], 1);
                    atomicMin(&gvf[g], r);
                    ++r;
                }
        }
        __syncthreads();
        if (tid < c.NG)
            gbv[tid] = gvc[tid] ? (int)atomicAdd(&c.gcnt[((int64_t)(n >> 5) * c.NG + tid) * 2 + 1], (uint32_t)gvc[tid]) : 0;
        __syncthreads();
        for (int ch = cb0; ch < cb1; ++ch)
            if (vflag[ch + o8]) {
                const int g = ch / c.GW;
                const int vpos = gbv[g] + (vr - gvf[g]);
                if (vpos < c.vcap_g)
                    c.vit[((int64_t)(n >> 5) * c.NG + g) * c.vcap_g + vpos] =
                        ((uint32_t)xv[ch + o16] << 16) | ((uint32_t)(n & 31) << 11) | item_code_flag<BITS>(vc[ch + o8]) |
                        (uint32_t)(ch - g * c.GW);
                vo[vr++] = (uint32_t)ch | ((uint32_t)xv[ch + o16] << 16);
            }
    }
    __syncthreads();

    }
    // --------------------------------------------------------------- packing
    constexpr int PB = 2 * BITS;                 // bits per Key pair code
    const int tile = (int)(n >> 5), jj = (int)(n & 31);
    if (part != 2)
    for (int q = tid; q < c.QW; q += NT) {
        const int h = q / (4 * BITS), w = q % (4 * BITS);
        const int bit0 = 32 * w;
        const int p0 = bit0 / PB, off = bit0 - p0 * PB;
        unsigned long long acc = 0;
        for (int p = p0, sh = 0; sh < 32 + off && p < kPairs; ++p, sh += PB) {
            unsigned pc = (unsigned)kc[I8(h * kHeadDim + p)] | ((unsigned)kc[I8(h * kHeadDim + p + kPairs)] << BITS);
            acc |= (unsigned long long)pc << sh;
        }
        c.kcodes[((int64_t)tile * c.QW + q) * 32 + jj] = (uint32_t)(acc >> off);
    }
    if (part != 1)
    // Value codes into the fragment layout (kvq_internal.cuh): the two channels 16mt+g and
    // 16mt+g+8 of a head share a lane and sit 2b bits apart, so one OR per pair of codes.
    // Words are shared with the tile's other tokens (zeroed at create/reset).
    for (int x = tid; x < c.H_kv * 64; x += NT) {
        const int hh = x >> 6, mt = (x >> 3) & 7, g = x & 7;
        const int cc = mt * 16 + g;
        const int bit = vf_bit(jj, cc, BITS);
        const uint32_t v = (uint32_t)vc[I8(hh * kHeadDim + cc)] | ((uint32_t)vc[I8(hh * kHeadDim + cc + 8)] << (2 * BITS));
        const int lane = vf_lane(jj, cc), w = bit >> 5, off = bit & 31;
        uint32_t *dst = c.vcodes + vf_word(tile, c.H_kv, hh, w, lane, BITS);
        atomicOr(dst, v << off);
        if (off + 3 * BITS > 32) atomicOr(dst + 32, v >> (32 - off));
    }
}

// Prefill pass 2: kptr[n0+1+t] = kptr[n0] + inclusive_scan(counts)[t]  (one CTA).
__global__ void __launch_bounds__(1024) scan_counts_kernel(DevCache c, int64_t n0, int64_t T) {
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = c.kptr[n0];
    __syncthreads();
    for (int64_t b = 0; b < T; b += 1024) {
        int64_t i = b + tid;
        uint32_t v = i < T ? (uint32_t)c.counts[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t s = wsum[lane], t2 = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, t2, o);
                if (lane >= o) t2 += y;
            }
            wsum[lane] = t2 - s;   // exclusive warp offsets
        }
        __syncthreads();
        uint32_t incl = carry + wsum[warp] + x;
        if (i < T) c.kptr[n0 + 1 + i] = incl;
        __syncthreads();
        if (tid == 1023) carry = incl;
        __syncthreads();
    }
}

// Sort the bucketed items of (tile, group) lists touched by a prefill into (token, channel)
// order (the low 16 bits), i.e. the order T successive appends produce.  One CTA per list.
__global__ void __launch_bounds__(256) sort_buckets_kernel(DevCache c, int64_t tile0, int which) {
    const int64_t tile = tile0 + blockIdx.x / c.NG;
    const int g = blockIdx.x % c.NG;
    const int cap = which ? c.vcap_g : c.kcap_g;
    uint32_t *lst = (which ? c.vit : c.kit) + (tile * c.NG + g) * cap;
    const uint32_t cnt = c.gcnt[(tile * c.NG + g) * 2 + which];
    if (cnt > (uint32_t)cap || cnt < 2) return;   // overflowed lists are not used by attend
    extern __shared__ uint32_t sitem[];
    int n2 = 1;
    while (n2 < (int)cnt) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) sitem[i] = i < (int)cnt ? lst[i] : 0xffffffffu;
    __syncthreads();
    // bitonic sort on (token, channel) (the low 16 bits without the code flag); keys are
    // unique per list
    for (int k = 2; k <= n2; k <<= 1)
        for (int jv = k >> 1; jv > 0; jv >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ jv;
                if (ixj > i) {
                    const uint32_t a = sitem[i], b = sitem[ixj];
                    const uint32_t ka = a == 0xffffffffu ? 0xffffffffu : (a & 0xf9ffu);
                    const uint32_t kb = b == 0xffffffffu ? 0xffffffffu : (b & 0xf9ffu);
                    const bool up = (i & k) == 0;
                    if ((ka > kb) == up) { sitem[i] = b; sitem[ixj] = a; }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < (int)cnt; i += blockDim.x) lst[i] = sitem[i];
}

size_t qz_smem(int D, int NT) {
    const int E = (D + NT - 1) / NT;
    const size_t L16 = (size_t)D + (size_t)NT * ((E % 4 == 0) ? 2 : 0);
    const size_t L8 = (size_t)D + (size_t)NT * ((E % 8 == 0) ? 4 : 0);
    size_t b = L16 * 2 * 3 + L8 * 2 + ((L8 + 15) & ~size_t(15));
    b = (b + 15) & ~size_t(15);
    b += (256 + 64 + 64 + 64) * 4;
    return b;
}

template <int BITS>
cudaError_t launch_qz_bits(const DevCache &c, const __half *K, const __half *V, int64_t n0,
                           int64_t T, cudaStream_t s) {
    const size_t smem = qz_smem(c.D, QZ_THREADS), smem1 = qz_smem(c.D, QZ_THREADS_1);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(qz_kernel<BITS, QZ_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem1 > 48 * 1024)
        cudaFuncSetAttribute(qz_kernel<BITS, QZ_THREADS_1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    if (T == 1) {
        qz_kernel<BITS, QZ_THREADS_1><<<2, QZ_THREADS_1, smem1, s>>>(c, K, V, n0, 0, -1);
        return cudaGetLastError();
    }
    qz_kernel<BITS, QZ_THREADS><<<(unsigned)T, QZ_THREADS, smem, s>>>(c, K, V, n0, 1, 0);
    scan_counts_kernel<<<1, 1024, 0, s>>>(c, n0, T);
    qz_kernel<BITS, QZ_THREADS><<<(unsigned)T, QZ_THREADS, smem, s>>>(c, K, V, n0, 2, 0);
    const int64_t tile0 = n0 / 32, tile1 = (n0 + T - 1) / 32;
    const unsigned nl = (unsigned)((tile1 - tile0 + 1) * c.NG);
    int pk = 1, pv = 1;
    while (pk < c.kcap_g) pk <<= 1;
    while (pv < c.vcap_g) pv <<= 1;
    sort_buckets_kernel<<<nl, 256, pk * 4, s>>>(c, tile0, 0);
    sort_buckets_kernel<<<nl, 256, pv * 4, s>>>(c, tile0, 1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const DevCache &c, const __half *K, const __half *V, int64_t n0,
                            int64_t T, cudaStream_t s) {
    switch (c.bits) {
        case 2: return launch_qz_bits<2>(c, K, V, n0, T, s);
        case 3: return launch_qz_bits<3>(c, K, V, n0, T, s);
        case 4: return launch_qz_bits<4>(c, K, V, n0, T, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace kvq
