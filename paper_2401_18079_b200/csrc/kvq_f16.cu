// kvq_f16.cu -- F16: the fp16 KV-cache comparator of BASELINE config C3 ("4-bit vs 3-bit vs
// fp16 cache").  The paper's baseline is fp16 mat-vec against an fp16 cache of post-RoPE
// Keys ("Key fp16 Matvec", "Value fp16 Matvec", the ~1.4x of P:80); this is that
// baseline on B200: the same decode step as the quantized path (pre-RoPE q and its position
// in, o out) over a dense fp16 cache.
//
//   store  : K is rotated at append with exact fp64 angles (R11, R12; theta_i supplied by the
//            host) and rounded once to fp16 -- the cache holds RoPE(k) as an fp16 model cache
//            would; V is copied.
//   attend : q~ = RoPE(q, pos) log2(e)/sqrt(d) in fp64 then fp32; per 8-token tile a warp reads
//            the 8 Key rows of its head (lane = token sub-index x 32-channel group, 64
//            contiguous bytes per lane), scores in fp32 (Keys converted), base-2 online
//            softmax, and P.V in fp32 (Values converted, weights fp32).  Split over tokens:
//            warp partials -> CTA partial -> merge by the last CTA of the head (ticket).
// HBM-bound: 4 d bytes per token and head (K + V), read once.
#include "kvq_internal.cuh"

#include <math_constants.h>

namespace kvq {
namespace {

constexpr int FW = 8;              // warps per CTA
constexpr int FT = FW * 32;

// fp64 -> fp16, round to nearest even, one rounding
__device__ __forceinline__ __half d2h_rn(double x) {
    unsigned short r;
    asm("cvt.rn.f16.f64 %0, %1;" : "=h"(r) : "d"(x));
    return __ushort_as_half(r);
}

__device__ __forceinline__ float f_warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// one thread per (token, head, RoPE pair): fp64 rotation by (pos_base + n) theta_i, one rounding
__global__ void f16_store_kernel(F16Dev c, const __half *__restrict__ K, const __half *__restrict__ V,
                                 int64_t n0, int64_t T) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int PPT = c.D / 2;   // pairs per token
    if (x >= T * PPT) return;
    const int64_t t = x / PPT;
    const int r = (int)(x % PPT), h = r / kPairs, i = r % kPairs;
    const int64_t n = n0 + t;
    const __half *kr = K + t * c.D + h * kHeadDim;
    const double a = (double)__half2float(kr[i]), b = (double)__half2float(kr[i + kPairs]);
    double s, co;
    sincos((double)(c.pos_base + n) * c.theta_tab[i], &s, &co);
    __half *ko = c.K + n * c.D + h * kHeadDim;
    ko[i] = d2h_rn(a * co - b * s);
    ko[i + kPairs] = d2h_rn(b * co + a * s);
    const __half *vr = V + t * c.D + h * kHeadDim;
    __half *vo = c.V + n * c.D + h * kHeadDim;
    vo[i] = vr[i];
    vo[i + kPairs] = vr[i + kPairs];
}

struct FParams {
    const __half *q;
    int64_t pos, T;
    int S;
    float *out, *parts;
    unsigned *tickets;
};

__global__ void __launch_bounds__(FT, 2) f16_attend_kernel(F16Dev c, FParams P) {
    __shared__ float wpart[FW][kHeadDim + 2];
    __shared__ float qh[kHeadDim];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = blockIdx.x % c.H_q, split = blockIdx.x / c.H_q;
    const int h = g / c.G;
    const int64_t ntile = (P.T + 7) / 8;
    const int64_t t_begin = (int64_t)split * ntile / P.S, t_end = (int64_t)(split + 1) * ntile / P.S;

    // a1: q~ = RoPE(q, pos) * log2(e) / sqrt(d), fp64 angles, stored fp16
    if (tid < kPairs) {
        const int i = tid;
        const __half *qg = P.q + (int64_t)g * kHeadDim;
        double s, co;
        sincos((double)P.pos * c.theta_tab[i], &s, &co);
        const double a = (double)__half2float(qg[i]), b = (double)__half2float(qg[i + kPairs]);
        const double sc = 1.4426950408889634 / sqrt((double)kHeadDim);
        qh[i] = (float)((a * co - b * s) * sc);
        qh[i + kPairs] = (float)((b * co + a * s) * sc);
    }
    __syncthreads();
    const int ts = lane >> 2, cg = lane & 3;   // token of the tile, 32-channel group
    float2 qv[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) qv[k] = make_float2(qh[cg * 32 + 2 * k], qh[cg * 32 + 2 * k + 1]);
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.f;
    float m_run = -CUDART_INF_F, l_lane = 0.f;
    const size_t rowb = (size_t)c.D;
    for (int64_t t = t_begin + warp; t < t_end; t += FW) {
        const int64_t n = t * 8 + ts;
        const bool valid = n < P.T;
        const uint4 *kp = reinterpret_cast<const uint4 *>(c.K + n * rowb + h * kHeadDim + cg * 32);
        const uint4 *vp = reinterpret_cast<const uint4 *>(c.V + n * rowb + h * kHeadDim + cg * 32);
        uint4 kw[4], vw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            kw[k] = valid ? __ldcs(kp + k) : make_uint4(0, 0, 0, 0);
            vw[k] = valid ? __ldcs(vp + k) : make_uint4(0, 0, 0, 0);
        }
        // a2: score (fp16 x fp16 -> fp32), reduced over the token's 4 lanes
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w[4] = {kw[k].x, kw[k].y, kw[k].z, kw[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const __half2 kk = *reinterpret_cast<const __half2 *>(&w[e]);
                const float2 kf = __half22float2(kk), qf = qv[k * 4 + e];
                s0 = fmaf(kf.x, qf.x, s0);
                s1 = fmaf(kf.y, qf.y, s1);
            }
        }
        float s = s0 + s1;
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s = valid ? s : -CUDART_INF_F;
        // a4: base-2 online softmax over the tile's 8 tokens
        float mt = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, 4));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 8));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 16));
        const float m_new = fmaxf(m_run, mt);
        const float alpha = m_new == -CUDART_INF_F ? 1.f : exp2f(m_run - m_new);
        const float p = valid ? exp2f(s - m_new) : 0.f;
        m_run = m_new;
        l_lane = l_lane * alpha + (cg == 0 ? p : 0.f);
        if (alpha != 1.f) {
#pragma unroll
            for (int k = 0; k < 32; ++k) acc[k] *= alpha;
        }
        // a5: P.V in fp32
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w[4] = {vw[k].x, vw[k].y, vw[k].z, vw[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 vf = __half22float2(*reinterpret_cast<const __half2 *>(&w[e]));
                acc[k * 8 + 2 * e] = fmaf(p, vf.x, acc[k * 8 + 2 * e]);
                acc[k * 8 + 2 * e + 1] = fmaf(p, vf.y, acc[k * 8 + 2 * e + 1]);
            }
        }
    }
    // warp partial: reduce the 8 token lanes of each channel group
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        float v = acc[k];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        acc[k] = v;
    }
    const float l = f_warp_sum(l_lane);
    if (ts == 0) {
#pragma unroll
        for (int k = 0; k < 32; ++k) wpart[warp][cg * 32 + k] = acc[k];
    }
    if (lane == 0) { wpart[warp][kHeadDim] = m_run; wpart[warp][kHeadDim + 1] = l; }
    __syncthreads();
    float *part = P.parts + ((int64_t)split * c.H_q + g) * (kHeadDim + 2);
    if (tid < kHeadDim + 2) {
        float m = -CUDART_INF_F;
        for (int w = 0; w < FW; ++w)
            if (wpart[w][kHeadDim + 1] != 0.f) m = fmaxf(m, wpart[w][kHeadDim]);
        float lt = 0.f, o = 0.f;
        for (int w = 0; w < FW; ++w) {
            if (wpart[w][kHeadDim + 1] == 0.f) continue;
            const float wt = exp2f(wpart[w][kHeadDim] - m);
            lt += wt * wpart[w][kHeadDim + 1];
            if (tid < kHeadDim) o += wt * wpart[w][tid];
        }
        part[tid] = tid < kHeadDim ? o : (tid == kHeadDim ? m : lt);
    }
    // a7: the last CTA of the head merges the splits in fixed order
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&P.tickets[g], 1u) == (unsigned)(P.S - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid < kHeadDim) {
        const int64_t stride = (int64_t)c.H_q * (kHeadDim + 2);
        const float *pb = P.parts + (int64_t)g * (kHeadDim + 2);
        float m = -CUDART_INF_F;
        for (int s2 = 0; s2 < P.S; ++s2)
            if (__ldcg(pb + s2 * stride + kHeadDim + 1) != 0.f) m = fmaxf(m, __ldcg(pb + s2 * stride + kHeadDim));
        float lt = 0.f, o = 0.f;
        for (int s2 = 0; s2 < P.S; ++s2) {
            const float ls = __ldcg(pb + s2 * stride + kHeadDim + 1);
            if (ls == 0.f) continue;
            const float wt = exp2f(__ldcg(pb + s2 * stride + kHeadDim) - m);
            lt += wt * ls;
            o += wt * __ldcg(pb + s2 * stride + tid);
        }
        P.out[(int64_t)g * kHeadDim + tid] = o / lt;
    }
    __syncthreads();
    if (tid == 0) P.tickets[g] = 0;
}

}  // namespace

cudaError_t launch_f16_store(const F16Dev &c, const __half *K, const __half *V, int64_t n0, int64_t T,
                             cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    const int64_t work = T * (c.D / 2);
    f16_store_kernel<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(c, K, V, n0, T);
    return cudaGetLastError();
}

int f16_auto_splits(const F16Dev &c, int64_t T) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int S = 2 * sms / c.H_q;   // two CTAs per SM, one wave
    const int64_t ntile = (T + 7) / 8;
    if (S > ntile) S = (int)ntile;
    if (S < 1) S = 1;
    return S;
}

cudaError_t launch_f16_attend(const F16Dev &c, const __half *q, int64_t pos, int64_t T, float *out,
                              float *parts, unsigned *tickets, int S, cudaStream_t s) {
    FParams P;
    P.q = q; P.pos = pos; P.T = T; P.S = S; P.out = out; P.parts = parts; P.tickets = tickets;
    f16_attend_kernel<<<c.H_q * S, FT, 0, s>>>(c, P);
    return cudaGetLastError();
}

}  // namespace kvq
