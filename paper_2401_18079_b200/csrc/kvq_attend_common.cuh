// kvq_attend_common.cuh -- device helpers shared by the warp-level attend kernels
// (kvq_attend_wa.cu: MHA/GQA warp-autonomous kernels; kvq_attend_wd.cu: MHA with the K scores
// on the tensor cores).  Inline PTX wrappers, warp reductions, angle reduction, the fixed-point
// helpers of the outlier corrections and the launch helper with programmatic dependent launch.
#pragma once
#include "kvq_internal.cuh"

#include <math_constants.h>

namespace kvq {
namespace {

constexpr int WEXP = 14;   // fp16 P.V weights scaled into [0, 2^14]

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// 16-byte global -> shared copy (LDGSTS), completion by cp.async.wait_all
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
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
// warp max of floats with one REDUX via an order-preserving integer map
__device__ __forceinline__ float warp_max_redux(float v) {
    unsigned u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    u = __reduce_max_sync(0xffffffffu, u);
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(u);
}
// x mod 2 pi into [-pi, pi] in fp64 (x up to ~1e8: the fp64 product and the 2 pi constant err
// by < 1e-8 rad there)
__device__ __forceinline__ double red2pi(double x) {
    constexpr double kTwoPi = 6.283185307179586476925, kInv2Pi = 0.15915494309189533577;
    return fma(-kTwoPi, rint(x * kInv2Pi), x);
}
__device__ __forceinline__ float pow2i(int k) {
    k = max(-126, min(127, k));
    return __int_as_float((k + 127) << 23);
}
__device__ __forceinline__ int ilog2f(float x) { return ((__float_as_int(x) >> 23) & 255) - 127; }

constexpr int HG = 4;      // query heads per CTA (MHA: 4 KV heads, one outlier bucket group)
constexpr int NSTREAM = 8; // tile streams per CTA (warps sharing a stream take other heads)

// Key-outlier score terms in 64-bit fixed point: 2^-16 log2-score units; 47 integer bits
// hold any sum of finite fp16 terms (|x q~| < 2^30), so there is no clamp and no wrap
constexpr float kKfixScale = 65536.f;
__device__ __forceinline__ unsigned long long kfix_of(float v) {
    return (unsigned long long)__float2ll_rn(v * kKfixScale);
}
__device__ __forceinline__ float kfix_val(unsigned long long v) {
    return (float)(long long)v * (1.f / kKfixScale);
}
// 32-bit variant (MHA kernel): terms with |v| < 2^7 go to int32 fixed point -- at most 128
// Key-outlier items per (token, head), so |sum| < 2^7 * 2^7 * 2^16 = 2^30 cannot wrap --
// and larger terms (extreme fp16 outliers only) to an fp32 side sum.
constexpr float kKfixSmall = 128.f;
__device__ __forceinline__ void kfix_add32(int *fix, float *big, float v) {
    if (fabsf(v) < kKfixSmall) atomicAdd(fix, __float2int_rn(v * kKfixScale));
    else atomicAdd(big, v);
}
// a value the compiler cannot see through (keeps table bases OR-able instead of re-added)
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}

struct WParams {
    const __half *q;
    int64_t pos, T;
    int S, ntiles;
    float *out, *parts;
    unsigned *tickets;
    int write_partial;
    int pdl;
};

// Programmatic dependent launch: everything before pdl_wait() reads only the query and the
// cache's constant parameters (codebooks, Key thresholds), so it may overlap the preceding
// append kernel; cache contents are read after it.  A no-op without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename K, typename... Args>
cudaError_t launch_maybe_pdl(K kernel, int grid, int threads, size_t smem, cudaStream_t s, bool pdl,
                             Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace
}  // namespace kvq
