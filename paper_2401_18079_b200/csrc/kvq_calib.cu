// kvq_calib.cu -- SURVEY 8(f) f2, "Online for K" (tab:calibration): the
// per-channel Key outlier thresholds computed on the GPU from the Keys of a prefill block
// instead of offline calibration data.
//
// Per channel c over the block's T tokens: n = ceil(f T) outliers (integer ceil from ppm,
// reading R2), the ceil(n/2) largest and floor(n/2) smallest excluded (two-sided, R3), and
// lo_c / hi_c = the smallest / largest kept value, i.e. the floor(n/2)-th and (T-1-ceil(n/2))-th
// order statistics of the channel (ascending, 0-based); -0 is returned as +0.
//
// Two radix passes over order keys of the fp16 values (-0 merged with +0), HBM-bound:
//   pass 1  per (channel, high byte) counts, a CTA = 64 channels x a slice of the rows, rows
//           read as 128-byte segments; shared per-CTA histograms flushed with global atomics;
//   select  per channel (one warp): the high byte of both order statistics and their ranks
//           inside the bin;
//   pass 2  per (channel, low byte) counts of the elements in those two bins;
//   final   per channel: the two keys -> fp16 -> fp32 lo / hi.
#include "kvq_internal.cuh"

namespace kvq {
namespace {

constexpr int CC = 64;          // channels per CTA
constexpr int CT = 256;         // threads per CTA (4 row groups)
constexpr int HS = 257;         // padded histogram stride (bank spread)

__device__ __forceinline__ uint32_t okey16(uint16_t h) {
    const uint32_t k = (uint32_t)h ^ ((h & 0x8000u) ? 0xffffu : 0x8000u);
    return k == 0x7fffu ? 0x8000u : k;
}
__device__ __forceinline__ uint16_t key2h16(uint32_t k) {
    return (uint16_t)(k >= 0x8000u ? (k ^ 0x8000u) : (k ^ 0xffffu));
}

struct OnlineArgs {
    const uint16_t *K;     // [T][D] fp16 bits
    int64_t T;
    int D;
    int64_t rank_lo, rank_hi;   // ascending 0-based ranks of lo and hi
    uint32_t *hist1;       // [D][256]
    uint32_t *hist2;       // [D][2][256]
    uint32_t *sel;         // [D][4]: bin_lo, rank in bin, bin_hi, rank in bin
    float *lo, *hi;        // [D]
};

// pass = 1: high-byte counts; pass = 2: low-byte counts of the elements in the selected bins
template <int PASS>
__global__ void __launch_bounds__(CT) online_hist_kernel(OnlineArgs a) {
    extern __shared__ uint32_t h[];   // [CC (x2 in pass 2)][HS]
    const int tid = threadIdx.x, cl = tid & (CC - 1), rg = tid >> 6;
    const int c0 = blockIdx.x * CC, c = c0 + cl;
    const int R = gridDim.y;
    const int64_t r0 = a.T * blockIdx.y / R, r1 = a.T * (blockIdx.y + 1) / R;
    for (int x = tid; x < CC * HS * (PASS == 1 ? 1 : 2); x += CT) h[x] = 0;
    __syncthreads();
    const bool cv = c < a.D;
    uint32_t blo = 0, bhi = 0;
    if (PASS == 2 && cv) { blo = a.sel[c * 4 + 0]; bhi = a.sel[c * 4 + 2]; }
    if (cv) {
        for (int64_t r = r0 + rg; r < r1; r += CT / CC) {
            const uint32_t k = okey16(a.K[r * a.D + c]);
            if (PASS == 1) {
                atomicAdd(&h[cl * HS + (k >> 8)], 1u);
            } else {
                if ((k >> 8) == blo) atomicAdd(&h[(cl * 2) * HS + (k & 0xffu)], 1u);
                if ((k >> 8) == bhi) atomicAdd(&h[(cl * 2 + 1) * HS + (k & 0xffu)], 1u);
            }
        }
    }
    __syncthreads();
    const int nh = PASS == 1 ? 1 : 2;
    for (int x = tid; x < CC * nh * 256; x += CT) {
        const int row = x >> 8, b = x & 255;
        const int ch = c0 + row / nh;
        const uint32_t v = h[row * HS + b];
        if (v && ch < a.D) {
            uint32_t *g = PASS == 1 ? a.hist1 + (size_t)ch * 256 + b : a.hist2 + ((size_t)ch * 2 + row % nh) * 256 + b;
            atomicAdd(g, v);
        }
    }
}

// one warp per channel: the bin of a target rank in a 256-bin histogram and the rank inside it
__device__ __forceinline__ void find_bin(const uint32_t *hist, int64_t rank, uint32_t &bin, uint32_t &within) {
    const int lane = threadIdx.x & 31;
    uint32_t cnt[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { cnt[k] = hist[8 * lane + k]; s += cnt[k]; }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t exc = inc - s;
    const bool mine = (int64_t)exc <= rank && rank < (int64_t)inc;
    uint32_t b = 0, w = 0;
    if (mine) {
        uint32_t run = exc;
        bool found = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (!found && rank < (int64_t)(run + cnt[k])) { b = 8 * lane + k; w = (uint32_t)(rank - run); found = true; }
            run += cnt[k];
        }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;   // exactly one lane holds the rank
    bin = __shfl_sync(0xffffffffu, b, src);
    within = __shfl_sync(0xffffffffu, w, src);
}

template <int PASS>
__global__ void __launch_bounds__(256) online_select_kernel(OnlineArgs a) {
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= a.D) return;
    if (PASS == 1) {
        uint32_t b0, w0, b1, w1;
        find_bin(a.hist1 + (size_t)c * 256, a.rank_lo, b0, w0);
        find_bin(a.hist1 + (size_t)c * 256, a.rank_hi, b1, w1);
        if (lane == 0) { a.sel[c * 4 + 0] = b0; a.sel[c * 4 + 1] = w0; a.sel[c * 4 + 2] = b1; a.sel[c * 4 + 3] = w1; }
    } else {
        uint32_t l0, x0, l1, x1;
        find_bin(a.hist2 + ((size_t)c * 2) * 256, a.sel[c * 4 + 1], l0, x0);
        find_bin(a.hist2 + ((size_t)c * 2 + 1) * 256, a.sel[c * 4 + 3], l1, x1);
        if (lane == 0) {
            const float vlo = __half2float(__ushort_as_half(key2h16((a.sel[c * 4 + 0] << 8) | l0)));
            const float vhi = __half2float(__ushort_as_half(key2h16((a.sel[c * 4 + 2] << 8) | l1)));
            a.lo[c] = vlo == 0.f ? 0.f : vlo;
            a.hi[c] = vhi == 0.f ? 0.f : vhi;
        }
        (void)x0; (void)x1;
    }
}

// ---------------------------------------------------------------------------------------
// SURVEY 8(f) f4, mixed-precision sensitivity (sec:appendix-mp, eq:opt2 P:1336-1339):
//   Omega = (A - Q(A))^T F^D (A - Q(A)) = sum_{n,c} F[n][c] (A[n][c] - A^[n][c])^2
// over the tokens [n0, n0 + T) of a cache that holds them (quantized at the candidate, lower,
// precision), A^ the dequantized cache entry (R5, R6: outliers exact, else
// Chat_dec[code] s + z in fp64 from the stored fp32 s, z and codebook), separately for the
// Keys (pre-RoPE, as cached) and the Values.  One CTA per 32-token tile: the tile's outlier
// positions become a shared bitmap, then every (token, channel) element is visited once,
// channel-fastest, so K/V/F reads are coalesced rows and the tile's code words stay in L1.
struct SensArgs {
    DevCache c;
    const uint16_t *K, *V;     // [T][D] fp16 bits, row n - n0
    const float *FK, *FV;      // [T][D] or null (F = 1)
    int64_t n0, T;
    double *omega;             // [2] accumulated (zeroed by the caller)
};

__device__ __forceinline__ double h2d_dev(uint16_t h) { return (double)__half2float(__ushort_as_half(h)); }

__global__ void __launch_bounds__(256) sens_kernel(SensArgs a) {
    extern __shared__ uint32_t bm[];   // [2][32][D/32] outlier bitmaps (Key, Value)
    const DevCache &c = a.c;
    const int D = c.D, DW = D / 32, b = c.bits;
    const int64_t tile = a.n0 / 32 + blockIdx.x;
    const int64_t t0 = tile * 32;
    const int64_t lo = t0 > a.n0 ? t0 : a.n0;
    const int64_t hi = (t0 + 32 < a.n0 + a.T) ? t0 + 32 : a.n0 + a.T;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *kbm = bm, *vbm = bm + 32 * DW;
    for (int x = tid; x < 64 * DW; x += 256) bm[x] = 0;
    __syncthreads();
    for (int64_t n = lo + warp; n < hi; n += 8) {
        const int j = (int)(n - t0);
        const uint32_t r0 = c.kptr[n], r1 = c.kptr[n + 1];
        for (uint32_t r = r0 + lane; r < r1; r += 32) {
            const uint32_t ch = c.kout[r] & 0xffffu;
            atomicOr(&kbm[j * DW + (ch >> 5)], 1u << (ch & 31));
        }
        for (int r = lane; r < c.kv; r += 32) {
            const uint32_t ch = c.vout[n * c.kv + r] & 0xffffu;
            atomicOr(&vbm[j * DW + (ch >> 5)], 1u << (ch & 31));
        }
    }
    __syncthreads();
    const float *cbK = c.cb + 16, *cbV = c.cb + 48;
    const uint32_t m1 = (1u << b) - 1, m2 = (1u << (2 * b)) - 1;
    double ak = 0.0, av = 0.0;
    const int64_t ne = (hi - lo) * D;
    for (int64_t x = tid; x < ne; x += 256) {
        const int64_t n = lo + x / D;
        const int ch = (int)(x % D), j = (int)(n - t0);
        const int h = ch / kHeadDim, cc = ch % kHeadDim;
        const int64_t row = (n - a.n0) * D + ch;
        if (!((kbm[j * DW + (ch >> 5)] >> (ch & 31)) & 1u)) {
            const int p = cc & (kPairs - 1), bit = 2 * b * p, q = h * 4 * b + bit / 32;
            const uint32_t *wp = c.kcodes + ((size_t)tile * c.QW + q) * 32 + j;
            uint64_t w = __ldg(wp);
            if (bit % 32 + 2 * b > 32) w |= (uint64_t)__ldg(wp + 32) << 32;
            const uint32_t pc = (uint32_t)(w >> (bit % 32)) & m2;
            const uint32_t code = cc >= kPairs ? pc >> b : pc & m1;
            const double xh = (double)cbK[code] * (double)c.kpar[ch] + (double)c.kpar[D + ch];
            const double e = h2d_dev(a.K[row]) - xh;
            ak += (a.FK ? (double)a.FK[row] : 1.0) * e * e;
        }
        if (!((vbm[j * DW + (ch >> 5)] >> (ch & 31)) & 1u)) {
            const int bit = vf_bit(j, cc, b);
            const uint32_t *wp = c.vcodes + vf_word(tile, c.H_kv, h, bit / 32, vf_lane(j, cc), b);
            uint64_t w = __ldg(wp);
            if (bit % 32 + b > 32) w |= (uint64_t)__ldg(wp + 32) << 32;
            const uint32_t code = (uint32_t)(w >> (bit % 32)) & m1;
            const float2 sz = c.vsz[n];
            const double vh = (double)cbV[code] * (double)sz.x + (double)sz.y;
            const double e = h2d_dev(a.V[row]) - vh;
            av += (a.FV ? (double)a.FV[row] : 1.0) * e * e;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ak += __shfl_xor_sync(0xffffffffu, ak, o);
        av += __shfl_xor_sync(0xffffffffu, av, o);
    }
    __shared__ double red[8][2];
    if (lane == 0) { red[warp][0] = ak; red[warp][1] = av; }
    __syncthreads();
    if (tid == 0) {
        double sk = 0.0, sv = 0.0;
        for (int w = 0; w < 8; ++w) { sk += red[w][0]; sv += red[w][1]; }
        atomicAdd(a.omega, sk);
        atomicAdd(a.omega + 1, sv);
    }
}

// Diagonal Fisher information (F^D = diag(g (.) g); SPEC fisher_diag): F += g (.) g, one rounding (fmaf).
__global__ void fisher_kernel(float *F, const float *g, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = g[i];
        F[i] = fmaf(x, x, F[i]);
    }
}

// ---------------------------------------------------------------------------------------
// SURVEY 8(f) f3, offline calibration on the GPU (P:316-322 eq:fisher_kmeans, P:340, P:355-358
// eq:qnorm): the per-layer nuqX codebooks from calibration Keys / Values (readings R27,
// R28 in DESIGN.md):
//   points   Keys: x' = (x - z_c) / s_c for lo_c <= x <= hi_c (thresholds from the order-
//            statistics kernels above); Values: per token the two-sided top-k outliers removed
//            (R2, R3, ties to the lower index), x' = (v - z_n) / s_n over the kept range; fp64;
//            zero-width vectors contribute nothing
//   k-means  Lloyd, centroids initialised at the bin centres -1 + (2j+1)/k, nearest centroid with
//            ties to the lower index (2x' > c_j + c_{j+1}), per-element Fisher weights, empty
//            clusters keep their centroid, stop when the largest move < tol or after max_iter
//   Q-Norm   mean / population std of the points and of their encode-codebook values.
// Deterministic: a fixed grid (kCalG CTAs), per-CTA partials reduced in a fixed order.
constexpr int kCalG = 296;
constexpr int kCalT = 256;

struct CalArgs {
    const uint16_t *X[2];      // Keys, Values [N][D] fp16 bits
    const float *F[2];         // Fisher weights [N][D] or null
    int64_t N;
    int D, kv, k;
    const float *klo, *khi;    // [D] Key thresholds
    float *vlo, *vhi;          // [N] Value kept ranges (fp16 values)
    uint32_t *vmask;           // [N][D/32] Value outlier bits
    double *cent;              // [2][16] current centroids
    double *part;              // [2][kCalG][32] per-CTA sums
    int *done, *iters;         // [2]
    double tol;
    float *cb;                 // [4][16] outputs: Key enc, Key dec, Value enc, Value dec
    int fp16;
};

__device__ __forceinline__ uint16_t cal_d2h(double x) {
    unsigned short r;
    asm("cvt.rn.f16.f64 %0, %1;" : "=h"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ float cal_h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// one warp per token: the two-sided split of the token's Values, its kept range and outlier bits
__global__ void __launch_bounds__(128) cal_vrange_kernel(CalArgs a) {
    extern __shared__ uint4 rows[];   // [4][D/8]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = (int64_t)blockIdx.x * 4 + warp;
    if (n >= a.N) return;
    const int D = a.D, NC = D / 8, DW = D / 32;
    uint4 *r = rows + (size_t)warp * NC;
    const uint4 *src = reinterpret_cast<const uint4 *>(a.X[1] + n * D);
    for (int i = lane; i < NC; i += 32) r[i] = src[i];
    __syncwarp();
    const int ku = (a.kv + 1) / 2, kl = a.kv / 2;
    auto keys8 = [&](int i, uint32_t (&k8)[8]) {
        const uint4 u = r[i];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) k8[e] = okey16((uint16_t)(w[e >> 1] >> (16 * (e & 1))));
    };
    // count of elements with pred(key, idx), whole warp
    auto count = [&](auto pred) {
        int c = 0;
        for (int i = lane; i < NC; i += 32) {
            uint32_t k8[8];
            keys8(i, k8);
#pragma unroll
            for (int e = 0; e < 8; ++e) c += pred(k8[e], 8 * i + e) ? 1 : 0;
        }
        return (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    };
    // index (+1) of the need-th element (index order) with pred, 0 if need == 0
    auto cut_at = [&](auto pred, int need) {
        if (need <= 0) return 0;
        int run = 0;
        for (int m = 0; m * 32 < NC; ++m) {
            const int i = lane + 32 * m;
            uint32_t k8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            bool ok = i < NC;
            if (ok) keys8(i, k8);
            int c = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) c += (ok && pred(k8[e], 8 * i + e)) ? 1 : 0;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const int tot = __shfl_sync(0xffffffffu, inc, 31);
            if (run + tot >= need) {
                const int exc = inc - c;
                int idx = 0;
                const bool mine = run + exc < need && need <= run + inc;
                if (mine) {
                    int rr = need - run - exc;
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (pred(k8[e], 8 * i + e) && --rr == 0 && idx == 0) idx = 8 * i + e + 1;
                }
                const int src_l = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
                return __shfl_sync(0xffffffffu, idx, src_l);
            }
            run += tot;
        }
        return 0;
    };
    // upper outliers: the ku largest (value desc, index asc)
    uint32_t thi = 0;
    int cut_hi = 0;
    if (ku > 0) {
        for (int b = 15; b >= 0; --b) {
            const uint32_t t2 = thi | (1u << b);
            if (count([&](uint32_t k, int) { return k >= t2; }) >= ku) thi = t2;
        }
        const int above = count([&](uint32_t k, int) { return k > thi; });
        cut_hi = cut_at([&](uint32_t k, int) { return k == thi; }, ku - above);
    }
    auto upper = [&](uint32_t k, int idx) { return ku > 0 && (k > thi || (k == thi && idx < cut_hi)); };
    // lower outliers: the kl smallest of the rest (value asc, index asc)
    uint32_t tlo = 0;
    int cut_lo = 0;
    if (kl > 0) {
        for (int b = 15; b >= 0; --b) {
            const uint32_t t2 = tlo | (1u << b);
            if (count([&](uint32_t k, int idx) { return !upper(k, idx) && k < t2; }) < kl) tlo = t2;
        }
        const int below = count([&](uint32_t k, int idx) { return !upper(k, idx) && k < tlo; });
        cut_lo = cut_at([&](uint32_t k, int idx) { return !upper(k, idx) && k == tlo; }, kl - below);
    }
    auto lower = [&](uint32_t k, int idx) {
        return kl > 0 && !upper(k, idx) && (k < tlo || (k == tlo && idx < cut_lo));
    };
    uint32_t kmin = 0xffffffffu, kmax = 0;
    for (int m = 0; m * 32 < NC; ++m) {
        const int i = lane + 32 * m;
        uint32_t bits = 0;
        if (i < NC) {
            uint32_t k8[8];
            keys8(i, k8);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const bool out = upper(k8[e], 8 * i + e) || lower(k8[e], 8 * i + e);
                bits |= (out ? 1u : 0u) << e;
                if (!out) { kmin = min(kmin, k8[e]); kmax = max(kmax, k8[e]); }
            }
        }
        bits <<= 8 * (lane & 3);
        bits |= __shfl_xor_sync(0xffffffffu, bits, 1);
        bits |= __shfl_xor_sync(0xffffffffu, bits, 2);
        if (i < NC && (lane & 3) == 0) a.vmask[n * DW + i / 4] = bits;
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) {
        a.vlo[n] = cal_h2f(key2h16(kmin));
        a.vhi[n] = cal_h2f(key2h16(kmax));
    }
}

// MODE 0: per-cluster (sum w, sum w x') of a Lloyd step; MODE 1: Q-Norm moments (n, sum x',
// sum x'^2, sum q, sum q^2) with q the encode-codebook value.  blockIdx.y = 0 Keys, 1 Values.
template <int KC, int MODE>
__global__ void __launch_bounds__(kCalT) cal_km_kernel(CalArgs a) {
    extern __shared__ double acc[];   // MODE 0: [2 KC][kCalT]
    __shared__ double mid[16], cv[16];
    const int y = blockIdx.y, tid = threadIdx.x;
    if (MODE == 0 && a.done[y]) return;
    if (tid < KC) {
        if (MODE == 0) {
            cv[tid] = a.cent[y * 16 + tid];
        } else {
            cv[tid] = (double)a.cb[(2 * y) * 16 + tid];
        }
    }
    __syncthreads();
    if (tid + 1 < KC) mid[tid] = cv[tid] + cv[tid + 1];
    if (MODE == 0)
        for (int j = 0; j < 2 * KC; ++j) acc[j * kCalT + tid] = 0.0;
    __syncthreads();
    double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
    const int D = a.D, DW = D / 32;
    const uint16_t *X = a.X[y];
    const float *F = a.F[y];
    const int64_t nchunks = a.N * D / 8;
    for (int64_t ch = (int64_t)blockIdx.x * kCalT + tid; ch < nchunks; ch += (int64_t)gridDim.x * kCalT) {
        const int64_t e0 = ch * 8;
        const int64_t n = e0 / D;
        const int c0 = (int)(e0 - n * D);
        const uint4 u = *reinterpret_cast<const uint4 *>(X + e0);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
        float wt[8];
        if (F) {
            const float4 f0 = *reinterpret_cast<const float4 *>(F + e0), f1 = *reinterpret_cast<const float4 *>(F + e0 + 4);
            wt[0] = f0.x; wt[1] = f0.y; wt[2] = f0.z; wt[3] = f0.w; wt[4] = f1.x; wt[5] = f1.y; wt[6] = f1.z; wt[7] = f1.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) wt[e] = 1.f;
        }
        uint32_t vbits = 0;
        double vl = 0, vh = 0;
        if (y == 1) {
            vbits = (a.vmask[n * DW + c0 / 32] >> (c0 & 31)) & 0xffu;
            vl = (double)a.vlo[n];
            vh = (double)a.vhi[n];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const double x = (double)cal_h2f((uint16_t)(w4[e >> 1] >> (16 * (e & 1))));
            double lo, hi;
            bool kept;
            if (y == 0) {
                lo = (double)a.klo[c0 + e];
                hi = (double)a.khi[c0 + e];
                kept = lo <= x && x <= hi && hi > lo;
            } else {
                lo = vl; hi = vh;
                kept = !((vbits >> e) & 1u) && hi > lo;
            }
            if (!kept) continue;
            const double xn = (x - (hi + lo) / 2.0) / ((hi - lo) / 2.0);
            int lab = 0;
#pragma unroll
            for (int j = 0; j + 1 < KC; ++j) lab += (2.0 * xn > mid[j]) ? 1 : 0;
            if (MODE == 0) {
                const double w = (double)wt[e];
                acc[lab * kCalT + tid] += w;
                acc[(KC + lab) * kCalT + tid] += w * xn;
            } else {
                const double q = cv[lab];
                m0 += 1.0; m1 += xn; m2 += xn * xn; m3 += q; m4 += q * q;
            }
        }
    }
    if (MODE == 1) {
        acc[0 * kCalT + tid] = m0; acc[1 * kCalT + tid] = m1; acc[2 * kCalT + tid] = m2;
        acc[3 * kCalT + tid] = m3; acc[4 * kCalT + tid] = m4;
    }
    __syncthreads();
    const int NA = MODE == 0 ? 2 * KC : 5;
    if (tid < NA) {
        double s = 0.0;
        for (int t = 0; t < kCalT; ++t) s += acc[tid * kCalT + t];
        a.part[((size_t)y * kCalG + blockIdx.x) * 32 + tid] = s;
    }
}

__device__ float cal_store(double v, float prev, bool first, int fp16) {
    float r;
    if (fp16) {
        const uint16_t h = cal_d2h(v);
        r = cal_h2f(h);
        if (!first && !(r > prev)) {
            const uint16_t p = __half_as_ushort(__float2half_rn(prev));   // prev is an fp16 value
            const uint16_t nx = (p & 0x8000u) ? (p == 0x8000u ? (uint16_t)1 : (uint16_t)(p - 1)) : (uint16_t)(p + 1);
            r = cal_h2f(nx);
        }
    } else {
        r = (float)v;
        if (!first && !(r > prev)) r = nextafterf(prev, INFINITY);
    }
    return r;
}

// one Lloyd update per matrix: thread (y, j) reduces the partials, thread 0 of each half sorts
__global__ void cal_update_kernel(CalArgs a, int KC) {
    __shared__ double sums[2][32];
    const int y = threadIdx.x >> 5, t = threadIdx.x & 31;
    if (a.done[y]) return;
    if (t < 2 * KC) {
        double s = 0.0;
        for (int g = 0; g < kCalG; ++g) s += a.part[((size_t)y * kCalG + g) * 32 + t];
        sums[y][t] = s;
    }
    __syncwarp();
    if (t == 0) {
        double c[16];
        for (int j = 0; j < KC; ++j) {
            const double old = a.cent[y * 16 + j], sw = sums[y][j];
            c[j] = sw > 0.0 ? sums[y][KC + j] / sw : old;
        }
        for (int i = 1; i < KC; ++i)
            for (int j = i; j > 0 && c[j] < c[j - 1]; --j) { const double x = c[j]; c[j] = c[j - 1]; c[j - 1] = x; }
        double move = 0.0;
        for (int j = 0; j < KC; ++j) { move = fmax(move, fabs(c[j] - a.cent[y * 16 + j])); a.cent[y * 16 + j] = c[j]; }
        a.iters[y] += 1;
        if (move < a.tol) a.done[y] = 1;
    }
}

// MODE 0: store the encode codebooks (and copy them to the decode slots); MODE 1: Q-Norm'd
// decode codebooks from the moments
template <int MODE>
__global__ void cal_store_kernel(CalArgs a) {
    const int y = threadIdx.x;
    if (y >= 2) return;
    float *enc = a.cb + (2 * y) * 16, *dec = a.cb + (2 * y + 1) * 16;
    if (MODE == 0) {
        float prev = 0.f;
        for (int j = 0; j < a.k; ++j) { prev = cal_store(a.cent[y * 16 + j], prev, j == 0, a.fp16); enc[j] = prev; dec[j] = prev; }
    } else {
        double s[5];
        for (int t = 0; t < 5; ++t) {
            s[t] = 0.0;
            for (int g = 0; g < kCalG; ++g) s[t] += a.part[((size_t)y * kCalG + g) * 32 + t];
        }
        if (!(s[0] > 0.0)) return;
        const double mu1 = s[1] / s[0], mu2 = s[3] / s[0];
        const double sg1 = sqrt(fmax(s[2] / s[0] - mu1 * mu1, 0.0)), sg2 = sqrt(fmax(s[4] / s[0] - mu2 * mu2, 0.0));
        if (!(sg2 > 0.0)) return;
        float prev = 0.f;
        for (int j = 0; j < a.k; ++j) {
            prev = cal_store(((double)enc[j] - mu2) * sg1 / sg2 + mu1, prev, j == 0, a.fp16);
            dec[j] = prev;
        }
    }
}

template <int KC>
cudaError_t cal_run(CalArgs &a, int max_iter, int qnorm, cudaStream_t s) {
    const size_t sm0 = (size_t)2 * KC * kCalT * 8, sm1 = (size_t)5 * kCalT * 8;
    cudaFuncSetAttribute(cal_km_kernel<KC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0);
    const dim3 grid(kCalG, 2);
    for (int it = 0; it < max_iter; ++it) {
        cal_km_kernel<KC, 0><<<grid, kCalT, sm0, s>>>(a);
        cal_update_kernel<<<1, 64, 0, s>>>(a, KC);
    }
    cal_store_kernel<0><<<1, 32, 0, s>>>(a);
    if (qnorm) {
        cal_km_kernel<KC, 1><<<grid, kCalT, sm1, s>>>(a);
        cal_store_kernel<1><<<1, 32, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_layer_sensitivity(const DevCache &c, const __half *K, const __half *V, const float *FK,
                                     const float *FV, int64_t n0, int64_t T, double *omega, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(omega, 0, 2 * sizeof(double), s);
    if (e != cudaSuccess || T == 0) return e;
    SensArgs a;
    a.c = c;
    a.K = reinterpret_cast<const uint16_t *>(K);
    a.V = reinterpret_cast<const uint16_t *>(V);
    a.FK = FK; a.FV = FV; a.n0 = n0; a.T = T; a.omega = omega;
    const int64_t tiles = (n0 + T + 31) / 32 - n0 / 32;
    const size_t smem = (size_t)2 * 32 * (c.D / 32) * 4;
    cudaFuncSetAttribute(sens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sens_kernel<<<(unsigned)tiles, 256, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_calibrate(const __half *K, const __half *V, const float *FK, const float *FV, int64_t N, int D,
                             int bits, int ppm, int max_iter, double tol, int qnorm, int fp16, float *key_lo,
                             float *key_hi, float *cb, int *iters, cudaStream_t s) {
    cudaError_t e = launch_online_key_thresholds(K, N, D, ppm, key_lo, key_hi, s);
    if (e != cudaSuccess) return e;
    const int k = 1 << bits;
    const size_t DW = (size_t)D / 32;
    const size_t b_v = (size_t)N * 4, b_m = (size_t)N * DW * 4, b_c = 32 * 8, b_p = (size_t)2 * kCalG * 32 * 8;
    void *scratch = nullptr;
    e = cudaMallocAsync(&scratch, 2 * b_v + b_m + b_c + b_p + 64, s);
    if (e != cudaSuccess) return e;
    char *p = reinterpret_cast<char *>(scratch);
    CalArgs a;
    a.X[0] = reinterpret_cast<const uint16_t *>(K);
    a.X[1] = reinterpret_cast<const uint16_t *>(V);
    a.F[0] = FK; a.F[1] = FV;
    a.N = N; a.D = D; a.k = k;
    a.kv = (int)(((int64_t)ppm * D + 999999) / 1000000);
    a.klo = key_lo; a.khi = key_hi;
    a.cent = reinterpret_cast<double *>(p); p += b_c;
    a.part = reinterpret_cast<double *>(p); p += b_p;
    a.vlo = reinterpret_cast<float *>(p); p += b_v;
    a.vhi = reinterpret_cast<float *>(p); p += b_v;
    a.vmask = reinterpret_cast<uint32_t *>(p); p += b_m;
    a.done = iters + 2;    // iters: [2] counts + [2] done flags (caller's device scratch)
    a.iters = iters;
    a.tol = tol;
    a.cb = cb;
    a.fp16 = fp16;
    double c0[32];
    for (int y = 0; y < 2; ++y)
        for (int j = 0; j < 16; ++j) c0[y * 16 + j] = j < k ? -1.0 + (2.0 * j + 1.0) / k : 0.0;
    e = cudaMemcpyAsync(a.cent, c0, sizeof c0, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(iters, 0, 4 * sizeof(int), s);
    if (e != cudaSuccess) { cudaFreeAsync(scratch, s); return e; }
    const size_t smv = (size_t)4 * D * 2;
    cudaFuncSetAttribute(cal_vrange_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smv);
    cal_vrange_kernel<<<(unsigned)((N + 3) / 4), 128, smv, s>>>(a);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        if (k == 4) e = cal_run<4>(a, max_iter, qnorm, s);
        else if (k == 8) e = cal_run<8>(a, max_iter, qnorm, s);
        else e = cal_run<16>(a, max_iter, qnorm, s);
    }
    cudaFreeAsync(scratch, s);
    return e;
}

cudaError_t launch_fisher_accumulate(float *F, const float *g, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + 255) / 256;
    const unsigned grid = (unsigned)(want < 8 * sms ? want : 8 * sms);
    fisher_kernel<<<grid, 256, 0, s>>>(F, g, n);
    return cudaGetLastError();
}

cudaError_t launch_online_key_thresholds(const __half *K, int64_t T, int D, int ppm, float *lo, float *hi,
                                         cudaStream_t s) {
    const int64_t n = ((int64_t)ppm * T + 999999) / 1000000;
    const int64_t ku = (n + 1) / 2, kl = n / 2;
    OnlineArgs a;
    a.K = reinterpret_cast<const uint16_t *>(K);
    a.T = T; a.D = D;
    a.rank_lo = kl;
    a.rank_hi = T - 1 - ku;
    a.lo = lo; a.hi = hi;
    const size_t hb = (size_t)D * 256 * 4, sb = (size_t)D * 4 * 4;
    void *scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, hb * 3 + sb, s);
    if (e != cudaSuccess) return e;
    a.hist1 = reinterpret_cast<uint32_t *>(scratch);
    a.hist2 = a.hist1 + (size_t)D * 256;
    a.sel = a.hist2 + (size_t)D * 512;
    e = cudaMemsetAsync(scratch, 0, hb * 3, s);
    if (e != cudaSuccess) return e;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int cx = (D + CC - 1) / CC;
    int R = (3 * sms + cx - 1) / cx;                       // ~3 CTAs per SM
    if ((int64_t)R * (CT / CC) > T) R = (int)((T + (CT / CC) - 1) / (CT / CC));
    if (R < 1) R = 1;
    const dim3 grid((unsigned)cx, (unsigned)R);
    const size_t sm1 = (size_t)CC * HS * 4, sm2 = 2 * sm1;
    cudaFuncSetAttribute(online_hist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    cudaFuncSetAttribute(online_hist_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    online_hist_kernel<1><<<grid, CT, sm1, s>>>(a);
    online_select_kernel<1><<<(D + 7) / 8, 256, 0, s>>>(a);
    online_hist_kernel<2><<<grid, CT, sm2, s>>>(a);
    online_select_kernel<2><<<(D + 7) / 8, 256, 0, s>>>(a);
    e = cudaGetLastError();
    cudaFreeAsync(scratch, s);
    return e;
}

}  // namespace kvq
