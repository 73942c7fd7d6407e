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
