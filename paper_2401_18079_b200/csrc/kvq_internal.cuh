// kvq_internal.cuh -- device data layout and launch interfaces of libkvq (sm_100a).
//
// GPU layout of one layer cache:
//
//   kcodes  u32 [ntiles][QW][32]      Key codes, token tiles of 32 tokens.  For token
//           n = 32*t + j and KV head h, the head's pair stream (64 pairs, pair p packs
//           code(h, p) | code(h, p+64) << b in 2b bits at bit offset 2b*p, RoPE partners
//           adjacent) occupies words q = h*4b .. h*4b+4b-1, stored at [t][q][j] so a
//           warp with lane = token reads 128 contiguous bytes per word slot.
//   vcodes  u32 [ntiles][H_kv][4b][32] Value codes of a (tile, KV head) in the order of the
//           A operand of mma.m16n8k16 (rows = channels, k = tokens; see vf_lane/vf_bit):
//           lane l of word w holds bits 32w..32w+31 of lane l's 128b-bit string, which is
//           64 fields of 2b bits, field = (code of token 2u, code of token 2u+1) for one
//           channel -- exactly one f16x2 A register after the pair-table lookup.  One head
//           group's slice of a tile is one contiguous block (a single TMA bulk copy).
//   vsz     float2 [cap]              per-token Value (s_n, z_n), fp32 (reading R6).
//   vout    u32 [cap][kv]             Value outliers, exactly kv = ceil(f*D) per token
//           (implicit CSR row pointer n*kv), ascending channel; record =
//           channel | fp16(value) << 16  (16-bit index + 16-bit value).
//   kptr    u32 [cap+1]               Key-outlier CSC column pointers (32-bit per token,
//           P:1151), kout u32 [kcap] records as above.
//   kit/vit u32 [ntiles][NG][cap]     Key / Value outliers again, bucketed per (tile, attend
//           head group) as self-contained items (value, token, channel); gcnt counts.
//   kpar    float [4][D]              s_c, z_c, lo_c, hi_c of the Keys.
//   cb      float [4][16]             Key enc, Key dec, Value enc, Value dec codebooks.
//   mids    double [2][16]            encode midpoints c_j + c_{j+1} (fp64).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace kvq {

constexpr int kTileTokens = 32;
constexpr int kHeadDim = 128;
constexpr int kPairs = kHeadDim / 2;

struct DevCache {
    int H_q, H_kv, d, D, bits, nlev, kv;   // kv = value outliers per token
    int G;                                 // GQA group size
    int QW;                                // Key words per token (= H_kv * 4b)
    int VW;                                // Value words per token (= D*b/32)
    int64_t cap, kcap, pos_base;
    double theta;
    const double *theta_tab;   // [64] theta_i = base^(-2i/d) in fp64, host-computed at create
    uint32_t *kcodes, *vcodes, *vout, *kptr, *kout;
    float2 *vsz;
    float *kpar;    // [4][D]
    float *cb;      // [4][16]
    double *mids;   // [2][16]
    int *err;       // device view of the sticky error word (host mapped)
    int *counts;    // prefill scratch [cap]
    // Outliers bucketed per (32-token tile, attend head group) for the attend kernel:
    // item (see item_code_flag) in (token, channel) order.  Written by the quantizer next to the token-major CSC/CSR arrays
    // (which stay the canonical form for export and the overflow fallback).
    int NG, GW;             // head groups, channels per group
    int vcb_exact16;        // 1: every Value decode codebook entry is an fp16 value (R23)
    int kcap_g, vcap_g;     // items per (tile, group)
    uint32_t *kit, *vit;    // [ntiles][NG][cap]
    uint32_t *gcnt;         // [ntiles][NG][2] counts; bit 31 = overflowed (use CSC/CSR)
    uint16_t *gtmp;         // prefill scratch [cap][NG][2] per-token group counts
    uint32_t *gbase;        // prefill scratch [NG][2] counts of the first tile before
    // Key ENC table per (KV head, RoPE pair p): channels c1 = 128h + p, c2 = c1 + 64 as fp16x2
    // words [L, H, code(lo), code(hi), T_0 .. T_{NM-1}, pad] (kvq_prefill.cu): L = smallest
    // fp16 >= lo_c, H = largest fp16 <= hi_c, T_j = smallest fp16 y with 2(y - z_c) > s_c m_j
    // in the oracle's fp64 arithmetic (R8), codes of the clamped lo_c / hi_c as fp16 values
    uint32_t *kenc;         // [H_kv][64][PS]
    unsigned long long *lb; // prefill look-back words [cap/32 + 1]
    unsigned *ticket;       // prefill tile ticket
};

enum ErrBits { kErrKeyCapacity = 1 };

// Outlier item of a (tile, head group) bucket:
//   fp16 value << 16 | token-in-tile << 11 | code flag << 9 | channel - group start (9 bits)
// The code flag names the dense code the quantizer stored at the outlier position, which the
// attend kernel needs for the correction x - deq(code): 1 = the top code 2^b - 1, 2 = code 0
// (the usual case: an outlier is clamped to the range ends), 0 = read it from the code words.
template <int BITS>
__host__ __device__ inline uint32_t item_code_flag(int code) {
    return code == (1 << BITS) - 1 ? (1u << 9) : (code == 0 ? (2u << 9) : 0u);
}

// Value-code fragment layout.  Token j (0..31) of a tile, channel cc (0..127) of a head:
// m-tile mt = cc/16, k-step s = j/16, and the mma.m16n8k16 A-fragment coordinates
// (groupID g = cc%8, thread-in-group t = (j%8)/2, register a = 2*(j%16/8) + cc%16/8,
// half = j%2) give lane 4g+t and field f = (2mt+s)*4 + a of that lane's string.
__host__ __device__ inline int vf_lane(int j, int cc) { return (cc & 7) * 4 + ((j & 7) >> 1); }
__host__ __device__ inline int vf_bit(int j, int cc, int bits) {
    const int f = ((cc >> 4) * 2 + (j >> 4)) * 4 + ((j >> 3) & 1) * 2 + ((cc >> 3) & 1);
    return f * 2 * bits + (j & 1) * bits;
}
// word (tile, KV head h, word w, lane l) of vcodes
__host__ __device__ inline int64_t vf_word(int64_t tile, int H_kv, int h, int w, int lane, int bits) {
    return ((tile * H_kv + h) * (4 * bits) + w) * 32 + lane;
}


// ---- block prefill (kvq_prefill.cu): one CTA per 32-token tile ----
size_t prefill_smem_bytes(int D, int NG);
cudaError_t launch_prefill(const DevCache &c, const __half *K, const __half *V, int64_t n0, int64_t T,
                           unsigned long long *lb, unsigned *ticket, cudaStream_t s,
                           unsigned long long *tm = nullptr);   // tm: diagnostics (phase clocks) or null
cudaError_t launch_append(const DevCache &c, const __half *K, const __half *V, int64_t n, cudaStream_t s,
                          unsigned long long *trace = nullptr);   // trace: diagnostics (phase clocks) or null
inline int kenc_words_per_pair(int bits) { return ((4 + (1 << bits) - 1) + 3) & ~3; }

// ---- fp16 comparator cache (kvq_f16.cu): post-RoPE fp16 K, fp16 V ----
struct F16Dev {
    int H_q, H_kv, G, D;
    int64_t cap, pos_base;
    const double *theta_tab;   // [64] theta_i = base^(-2i/d), host-computed
    __half *K, *V;             // [cap][D]
};
cudaError_t launch_f16_store(const F16Dev &c, const __half *K, const __half *V, int64_t n0, int64_t T,
                             cudaStream_t s);
int f16_auto_splits(const F16Dev &c, int64_t T);
cudaError_t launch_f16_attend(const F16Dev &c, const __half *q, int64_t pos, int64_t T, float *out,
                              float *parts, unsigned *tickets, int S, cudaStream_t s);

// ---- online per-channel Key thresholds (kvq_calib.cu) ----
cudaError_t launch_online_key_thresholds(const __half *K, int64_t T, int D, int ppm, float *lo, float *hi,
                                         cudaStream_t s);
// ---- mixed-precision sensitivity (kvq_calib.cu) ----
cudaError_t launch_layer_sensitivity(const DevCache &c, const __half *K, const __half *V, const float *FK,
                                     const float *FV, int64_t n0, int64_t T, double *omega, cudaStream_t s);
cudaError_t launch_fisher_accumulate(float *F, const float *g, int64_t n, cudaStream_t s);
// ---- offline calibration (kvq_calib.cu) ----
// cb: device [4][16] (Key enc, Key dec, Value enc, Value dec); iters: device int [4] scratch
// (Lloyd updates run for Keys / Values, then two done flags)
cudaError_t launch_calibrate(const __half *K, const __half *V, const float *FK, const float *FV, int64_t N, int D,
                             int bits, int ppm, int max_iter, double tol, int qnorm, int fp16, float *key_lo,
                             float *key_hi, float *cb, int *iters, cudaStream_t s);

// ---- attention (kvq_attend.cu) ----
struct AttendArgs {
    const __half *q;
    int64_t pos;
    int64_t T;
    float *out;          // o [H_q][d] or merged partial [H_q][d+2]
    int write_partial;   // 0: normalized o; 1: partial
    float *parts;        // scratch [splits][H_q][d+2]
    unsigned *tickets;   // [n_head_groups], zero between launches
    int splits;          // 0 = auto
    unsigned long long *timers;   // diagnostics: phase cycle sums, or null
    int *kernel_out;     // optional: 1 = warp-autonomous kernel launched, 0 = two-halves
    int *hg_out;         // optional: query heads per CTA of the launch
    int pdl;             // 1: the previous kernel on the stream is this cache's append, so the
                         // warp-autonomous kernels launch with programmatic dependent launch
                         // (their q/table prologue overlaps the append; cache reads wait)
};
int attend_heads_per_cta(int bits, int H_q, int G);
int attend_bucket_heads(int bits, int H_q, int G, int vcb_exact16);
int attend_auto_splits(const DevCache &c, int64_t T, int hg);
cudaError_t launch_attend(const DevCache &c, const AttendArgs &a, int *splits_used,
                          cudaStream_t s);
cudaError_t launch_merge(const float *parts, int P, int H, int d, float *o, cudaStream_t s);
size_t attend_smem_bytes(int bits, int hg);
// warp-autonomous variant (kvq_attend_wa.cu): MHA at 2-3 bits
bool attend_wa_supported(const DevCache &c);
size_t attend_wa_smem_bytes(int bits, bool resid);
cudaError_t launch_attend_wa(const DevCache &c, const AttendArgs &a, int S, cudaStream_t s);
// batched decode over B caches of one configuration (all attend_wa_supported, same bits and
// codebook kind): one launch
int attend_batch_max();
cudaError_t launch_attend_wa_batch(const DevCache *const *cs, const AttendArgs *as, int B, cudaStream_t s,
                                   int *splits_out);
// batched GQA decode over B caches of one configuration (all attend_wag_supported): one launch
cudaError_t launch_attend_wgt_batch(const DevCache *const *cs, const AttendArgs *as, int B, cudaStream_t s,
                                    int *splits_out);
// warp-autonomous GQA variant (G = 4, 2-3 bits): one CTA per KV head
bool attend_wag_supported(const DevCache &c);
cudaError_t launch_attend_wag(const DevCache &c, const AttendArgs &a, int S, cudaStream_t s);

}  // namespace kvq
