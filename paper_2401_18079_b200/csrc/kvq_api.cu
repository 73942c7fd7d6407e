// kvq_api.cu -- C ABI of libkvq: validation, the cache object, staging, export.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/kvq.h"
#include "kvq_internal.cuh"

#include <nvtx3/nvToolsExt.h>

namespace {
// NVTX range around a public call (SURVEY 5 tracing): visible in Nsight / ncu timelines, a
// no-op without a tool attached
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace kvq;

struct kvq_cache {
    kvq_config cfg;
    DevCache dc;
    int64_t T = 0;             // host shadow of the token count
    int hg = 0;                // query heads per attend CTA (of the last launch)
    int last_kernel = -1;      // attend kernel of the last launch (kvq_info.attend_kernel)
    int pdl_ok = 0;            // the last op on pdl_stream was a single-token append
    void *pdl_stream = nullptr;
    int splits_forced = 0;
    int last_splits = 0;
    float *parts = nullptr;    // [max_splits][H_q][d+2]
    int max_splits = 0;
    unsigned *tickets = nullptr;
    unsigned long long *timers = nullptr;   // diagnostics (KVQ_PHASE_TIMERS=1)
    int *err_host = nullptr;   // host-mapped sticky error word
    void *stage = nullptr;     // device staging for host buffers
    size_t stage_bytes = 0;
    int64_t device_bytes = 0;
    std::vector<void *> allocs;
};

namespace {

thread_local std::string g_last_error;

kvq_status fail(kvq_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
kvq_status fail(kvq_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

kvq_status cuda_fail(cudaError_t e, const char *what) {
    return fail(KVQ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr)                                                     \
    do {                                                             \
        cudaError_t e__ = (expr);                                    \
        if (e__ != cudaSuccess) return cuda_fail(e__, #expr);        \
    } while (0)

bool finite_f(float x) { return std::isfinite(x); }

kvq_status check_sticky(kvq_cache *c) {
    if (c->err_host && *(volatile int *)c->err_host) {
        int e = *(volatile int *)c->err_host;
        if (e & kErrKeyCapacity)
            return fail(KVQ_ECAPACITY, "key-outlier capacity (%lld records) exceeded on device",
                        (long long)c->dc.kcap);
        return fail(KVQ_ECUDA, "sticky device error %d", e);
    }
    return KVQ_OK;
}

template <typename T>
kvq_status dev_alloc(kvq_cache *c, T **p, size_t bytes) {
    void *q = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    e = cudaMemset(q, 0, bytes);
    if (e != cudaSuccess) { cudaFree(q); return cuda_fail(e, "cudaMemset"); }
    c->allocs.push_back(q);
    c->device_bytes += (int64_t)bytes;
    *p = reinterpret_cast<T *>(q);
    return KVQ_OK;
}

// Classify a user pointer: 0 = device on `dev`, 1 = host, -1 = device elsewhere.
// page-locked (cudaHostAlloc / cudaHostRegister) host memory: device-to-host copies into it
// stay asynchronous (stream ordered, kvq.h); pageable host outputs make the call synchronous
bool host_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeHost;
}

int classify(const void *p, int dev, uint32_t flags) {
    if (flags & KVQ_FLAG_TRUST_DEVICE_PTRS) return 0;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) { cudaGetLastError(); return 1; }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged)
        return at.device == dev ? 0 : -1;
    return 1;
}

// ---- exact fp16 thresholds of the fp64 ENC predicate (R8), for the prefill Key table ----
uint16_t key2h(uint32_t k) { return (uint16_t)(k >= 0x8000u ? (k ^ 0x8000u) : (k ^ 0xffffu)); }
double h2d(uint16_t h) {
    const int e = (h >> 10) & 31, m = h & 1023;
    double v = e == 0 ? std::ldexp((double)m, -24) : (e == 31 ? INFINITY : std::ldexp((double)(m | 1024), e - 25));
    return (h & 0x8000u) ? -v : v;
}
// smallest order key in [0x0400, 0xFC00) (finite fp16, ascending) whose value satisfies the
// monotone predicate, else 0xFC00 (+inf)
template <typename F>
uint32_t first_key(F pred) {
    uint32_t a = 0x0400u, b = 0xfc00u;
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (pred(h2d(key2h(mid)))) b = mid; else a = mid + 1;
    }
    return a;
}
// the oracle's ENC (kvo_enc): #{j : 2(y - z) > s (c_j + c_{j+1})} in fp64, no contraction
int enc_exact(double y, float s, float z, const float *cb, int nlev) {
    const double lhs = 2.0 * (y - (double)z);
    int code = 0;
    for (int j = 0; j + 1 < nlev; ++j) {
        const volatile double rhs = (double)s * ((double)cb[j] + (double)cb[j + 1]);
        if (lhs > rhs) code++;
    }
    return code;
}
uint16_t f16_of_small_int(int v) {   // exact fp16 bits of 0..15
    if (v == 0) return 0;
    int e = 0;
    while ((v >> (e + 1)) != 0) ++e;
    return (uint16_t)(((e + 15) << 10) | ((v << (10 - e)) & 1023));
}

kvq_status ensure_stage(kvq_cache *c, size_t bytes) {
    if (c->stage_bytes >= bytes) return KVQ_OK;
    if (c->stage) { cudaFree(c->stage); c->device_bytes -= (int64_t)c->stage_bytes; c->stage = nullptr; }
    void *p = nullptr;
    CK(cudaMalloc(&p, bytes));
    c->stage = p;
    c->stage_bytes = bytes;
    c->device_bytes += (int64_t)bytes;
    return KVQ_OK;
}

}  // namespace

extern "C" {

int32_t kvq_version(void) { return 100; }

const char *kvq_last_error(void) { return g_last_error.c_str(); }

kvq_status kvq_cache_create(const kvq_config *cfg, const kvq_params *prm, kvq_cache **out) {
    if (!cfg || !prm || !out) return fail(KVQ_EINVAL, "null argument");
    const kvq_config &C = *cfg;
    if (C.bits < 2 || C.bits > 4) return fail(KVQ_EINVAL, "bits must be 2, 3 or 4 (got %d)", C.bits);
    if (C.outlier_ppm < 0 || C.outlier_ppm >= 500000)
        return fail(KVQ_EINVAL, "outlier_ppm must be in [0, 500000) (got %d)", C.outlier_ppm);
    if (C.n_q_heads < 1 || C.n_kv_heads < 1) return fail(KVQ_ESHAPE, "head counts must be >= 1");
    if (C.n_q_heads % C.n_kv_heads) return fail(KVQ_ESHAPE, "n_q_heads %% n_kv_heads != 0");
    if (C.head_dim != kHeadDim) return fail(KVQ_ESHAPE, "this build supports head_dim == 128 (got %d)", C.head_dim);
    const int G = C.n_q_heads / C.n_kv_heads;
    if (G != 1 && G != 2 && G != 4 && G != 8) return fail(KVQ_ESHAPE, "GQA group must be 1, 2, 4 or 8");
    const int64_t D = (int64_t)C.n_kv_heads * C.head_dim;
    if (D > 8192) return fail(KVQ_ESHAPE, "this build supports D = H_kv*d <= 8192 (got %lld)", (long long)D);
    if (C.capacity_tokens < 1) return fail(KVQ_EINVAL, "capacity_tokens must be >= 1");
    if (!(C.rope_theta > 0) || !std::isfinite(C.rope_theta)) return fail(KVQ_EINVAL, "rope_theta must be > 0");
    if (C.pos_base < 0) return fail(KVQ_EINVAL, "pos_base must be >= 0");
    const int hg = attend_heads_per_cta(C.bits, C.n_q_heads, G);
    if (hg == 0) return fail(KVQ_ESHAPE, "no attend tiling for bits=%d H_q=%d G=%d", C.bits, C.n_q_heads, G);
    const int64_t kv = ((int64_t)C.outlier_ppm * D + 999999) / 1000000;
    if (kv >= D) return fail(KVQ_EINVAL, "value outliers per token (%lld) must be < D", (long long)kv);
    const int nlev = 1 << C.bits;
    const float *cbs[4] = {prm->key_cb_enc, prm->key_cb_dec ? prm->key_cb_dec : prm->key_cb_enc,
                           prm->val_cb_enc, prm->val_cb_dec ? prm->val_cb_dec : prm->val_cb_enc};
    for (int k = 0; k < 4; ++k) {
        if (!cbs[k]) return fail(KVQ_EINVAL, "codebook %d is NULL", k);
        for (int j = 0; j < nlev; ++j) {
            if (!finite_f(cbs[k][j])) return fail(KVQ_EINVAL, "codebook %d has a non-finite entry", k);
            if ((k == 0 || k == 2) && j > 0 && !(cbs[k][j] > cbs[k][j - 1]))
                return fail(KVQ_EINVAL, "encode codebook %d is not strictly ascending", k);
        }
    }
    if (!prm->key_lo || !prm->key_hi) return fail(KVQ_EINVAL, "key thresholds are NULL");
    for (int64_t ch = 0; ch < D; ++ch) {
        float lo = prm->key_lo[ch], hi = prm->key_hi[ch];
        if (!finite_f(lo) || !finite_f(hi) || lo > hi)
            return fail(KVQ_EINVAL, "key thresholds of channel %lld invalid", (long long)ch);
    }

    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (C.device < 0 || C.device >= ndev) return fail(KVQ_EDEVICE, "device %d not present", C.device);
    CK(cudaSetDevice(C.device));

    kvq_cache *c = new (std::nothrow) kvq_cache();
    if (!c) return fail(KVQ_EINVAL, "out of host memory");
    c->cfg = C;
    c->hg = hg;
    DevCache &d = c->dc;
    d.H_q = C.n_q_heads; d.H_kv = C.n_kv_heads; d.d = C.head_dim; d.D = (int)D;
    d.bits = C.bits; d.nlev = nlev; d.kv = (int)kv; d.G = G;
    d.QW = C.n_kv_heads * 4 * C.bits;
    d.VW = (int)(D * C.bits / 32);
    d.cap = (C.capacity_tokens + 31) / 32 * 32;
    // default Key-outlier headroom: 2*ceil(f*D) per token (at least 8) + slack (R21)
    d.kcap = C.k_outlier_capacity > 0 ? C.k_outlier_capacity
                                      : d.cap * (2 * kv > 8 ? 2 * kv : 8) + 4096;
    if (d.kcap > 0xFFFFFFF0LL) d.kcap = 0xFFFFFFF0LL;
    d.pos_base = C.pos_base;
    d.theta = C.rope_theta;

    kvq_status st = KVQ_OK;
    auto A = [&](auto **p, size_t bytes) { if (st == KVQ_OK) st = dev_alloc(c, p, bytes); };
    A(&d.kcodes, (size_t)(d.cap / 32) * d.QW * 32 * 4);
    A(&d.vcodes, (size_t)d.cap * d.VW * 4 + 16);   // [cap/32][H_kv][4b][32]
    A(&d.vsz, (size_t)d.cap * sizeof(float2));
    A(&d.vout, (size_t)d.cap * (kv > 0 ? kv : 1) * 4);
    A(&d.kptr, (size_t)(d.cap + 64) * 4);   // +63: attend stages 48-word CSC slices
    A(&d.kout, (size_t)d.kcap * 4 + 16);
    A(&d.kpar, (size_t)4 * D * 4);
    A(&d.cb, 64 * 4);
    A(&d.mids, 32 * 8);
    A(&d.counts, (size_t)d.cap * 4);
    // outlier buckets per (tile, attend head group); capacity ~3x the expected count
    {
        // R23: an fp16-exact Value decode codebook lets the attend kernels skip their residual
        // pass (and selects the warp-autonomous kernel at 4 bits, which has no residual pass)
        d.vcb_exact16 = 1;
        for (int j = 0; j < nlev; ++j)
            if (__half2float(__float2half_rn(cbs[3][j])) != cbs[3][j]) d.vcb_exact16 = 0;
        // 4-bit GQA runs on att_wgt_kernel, which has no fp32-codebook residual pass (R23)
        if (G > 1 && C.bits == 4 && !d.vcb_exact16)
            st = fail(KVQ_ESHAPE, "4-bit GQA needs an fp16-exact Value decode codebook (R23)");
        const int hkv_g = attend_bucket_heads(C.bits, C.n_q_heads, G, d.vcb_exact16) / G;
        d.GW = hkv_g * kHeadDim;
        d.NG = C.n_kv_heads / hkv_g;
        const double f = C.outlier_ppm / 1e6;
        int kc = (int)std::ceil(3.0 * f * d.GW);
        kc = kc < 8 ? 8 : kc;
        int vc = (int)std::ceil(3.0 * (double)kv * d.GW / (double)D);
        vc = vc < 8 ? 8 : vc;
        if (vc > kv) vc = (int)kv;
        d.kcap_g = ((32 * kc) + 3) & ~3;
        d.vcap_g = ((32 * (vc > 0 ? vc : 1)) + 3) & ~3;
        const size_t ntiles = (size_t)(d.cap / 32);
        A(&d.kit, ntiles * d.NG * d.kcap_g * 4);
        A(&d.vit, ntiles * d.NG * d.vcap_g * 4);
        A(&d.gcnt, ntiles * d.NG * 2 * 4 + 16);
    }
    {
        const int ps = kenc_words_per_pair(C.bits);
        A(&d.kenc, (size_t)C.n_kv_heads * kPairs * ps * 4);
        A(&d.lb, (size_t)(d.cap / 32 + 2) * 8);
        A(&d.ticket, 64);
    }
    {
        double *tt = nullptr;
        A(&tt, 64 * 8);
        d.theta_tab = tt;
    }
    c->max_splits = 4 * 148;
    A(&c->parts, (size_t)c->max_splits * d.H_q * (kHeadDim + 2) * 4);
    A(&c->tickets, 1024 * 4);   // one per attend head group (<= H_q)
    if (getenv("KVQ_PHASE_TIMERS")) A(&c->timers, (16 + 4096) * 8);   // + trace of CTA 0
    if (st != KVQ_OK) { kvq_cache_destroy(c); return st; }
    {
        cudaError_t e = cudaHostAlloc(&c->err_host, 64, cudaHostAllocMapped);
        if (e != cudaSuccess) { kvq_cache_destroy(c); return cuda_fail(e, "cudaHostAlloc"); }
        memset(c->err_host, 0, 64);
        e = cudaHostGetDevicePointer((void **)&d.err, c->err_host, 0);
        if (e != cudaSuccess) { kvq_cache_destroy(c); return cuda_fail(e, "cudaHostGetDevicePointer"); }
    }
    // per-channel Key params: s = fp32((hi-lo)/2), z = fp32((hi+lo)/2) in fp64 (R6)
    std::vector<float> kpar(4 * D);
    for (int64_t ch = 0; ch < D; ++ch) {
        const double lo = prm->key_lo[ch], hi = prm->key_hi[ch];
        kpar[ch] = (float)((hi - lo) / 2.0);
        kpar[D + ch] = (float)((hi + lo) / 2.0);
        kpar[2 * D + ch] = prm->key_lo[ch];
        kpar[3 * D + ch] = prm->key_hi[ch];
    }
    float cb[64] = {0};
    double mids[32] = {0};
    for (int k = 0; k < 4; ++k)
        for (int j = 0; j < nlev; ++j) cb[16 * k + j] = cbs[k][j];
    for (int j = 0; j + 1 < nlev; ++j) {
        mids[j] = (double)cbs[0][j] + (double)cbs[0][j + 1];
        mids[16 + j] = (double)cbs[2][j] + (double)cbs[2][j + 1];
    }
    // Key ENC table of the prefill kernel: per channel the fp16 thresholds of the outlier test
    // and of every ENC midpoint predicate, found by binary search over fp16 values with the
    // oracle's exact fp64 predicate (monotone in y), and the codes of the clamped lo / hi
    std::vector<uint32_t> kenc;
    {
        const int ps = kenc_words_per_pair(C.bits);
        kenc.assign((size_t)C.n_kv_heads * kPairs * ps, 0u);
        std::vector<uint16_t> cw((size_t)D * 20);
        for (int64_t ch = 0; ch < D; ++ch) {
            const double lo = prm->key_lo[ch], hi = prm->key_hi[ch];
            const float s = kpar[ch], z = kpar[D + ch];
            uint16_t *w = &cw[(size_t)ch * 20];
            w[0] = key2h(first_key([&](double v) { return v >= lo; }));                 // L
            const uint32_t kg = first_key([&](double v) { return v > hi; });
            w[1] = key2h(kg - 1);                                                         // H
            w[2] = f16_of_small_int(enc_exact(lo, s, z, cbs[0], nlev));
            w[3] = f16_of_small_int(enc_exact(hi, s, z, cbs[0], nlev));
            for (int j = 0; j + 1 < nlev; ++j) {
                const double mj = (double)cbs[0][j] + (double)cbs[0][j + 1];
                w[4 + j] = key2h(first_key([&](double y) {
                    const volatile double rhs = (double)s * mj;
                    return 2.0 * (y - (double)z) > rhs;
                }));
            }
        }
        for (int h = 0; h < C.n_kv_heads; ++h)
            for (int p = 0; p < kPairs; ++p) {
                const uint16_t *a = &cw[(size_t)(h * kHeadDim + p) * 20];
                const uint16_t *b = &cw[(size_t)(h * kHeadDim + p + kPairs) * 20];
                uint32_t *o = &kenc[(size_t)(h * kPairs + p) * ps];
                for (int q = 0; q < 4 + nlev - 1; ++q) o[q] = (uint32_t)a[q] | ((uint32_t)b[q] << 16);
            }
    }
    cudaError_t e = cudaMemcpy(d.kpar, kpar.data(), kpar.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d.kenc, kenc.data(), kenc.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d.cb, cb, sizeof cb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d.mids, mids, sizeof mids, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        double th[64];
        for (int i = 0; i < 64; ++i) th[i] = std::pow(C.rope_theta, -2.0 * (double)i / (double)kHeadDim);
        e = cudaMemcpy(const_cast<double *>(d.theta_tab), th, sizeof th, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { kvq_cache_destroy(c); return cuda_fail(e, "upload parameters"); }
    *out = c;
    return KVQ_OK;
}

void kvq_cache_destroy(kvq_cache *c) {
    if (!c) return;
    cudaSetDevice(c->cfg.device);
    cudaDeviceSynchronize();
    for (void *p : c->allocs) cudaFree(p);
    if (c->stage) cudaFree(c->stage);
    if (c->err_host) cudaFreeHost(c->err_host);
    delete c;
}

int64_t kvq_num_tokens(const kvq_cache *c) { return c ? c->T : 0; }

kvq_status kvq_get_info(const kvq_cache *c, kvq_info *info) {
    if (!c || !info) return fail(KVQ_EINVAL, "null argument");
    info->heads_per_cta = c->hg;
    info->splits = c->last_splits;
    info->value_outliers = c->dc.kv;
    info->words_per_token = c->dc.VW;
    info->capacity_tokens = c->dc.cap;
    info->k_outlier_capacity = c->dc.kcap;
    info->device_bytes = c->device_bytes;
    info->attend_kernel = c->last_kernel;
    info->bucket_heads = c->dc.GW / kHeadDim * c->dc.G;
    return KVQ_OK;
}

// Diagnostics only (not in kvq.h): per-tile event clocks of CTA 0 of the last attend,
// [tile][4] = K scores done, SV past FULL, SV softmax done, SV P.V done (clock64).
extern "C" kvq_status kvq_debug_trace(kvq_cache *c, uint64_t *out, int n) {
    if (!c || !c->timers) return fail(KVQ_EINVAL, "phase timers disabled");
    if (n > 4096) n = 4096;
    CK(cudaMemcpy(out, c->timers + 16, (size_t)n * 8, cudaMemcpyDeviceToHost));
    return KVQ_OK;
}

kvq_status kvq_phase_timers(kvq_cache *c, uint64_t *out) {
    if (!c || !out) return fail(KVQ_EINVAL, "null argument");
    if (!c->timers) return fail(KVQ_EINVAL, "phase timers disabled (set KVQ_PHASE_TIMERS=1)");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, c->timers, 16 * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(c->timers, 0, (16 + 4096) * 8));
    return KVQ_OK;
}

kvq_status kvq_set_splits(kvq_cache *c, int32_t splits) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (splits < 0 || splits > c->max_splits) return fail(KVQ_EINVAL, "splits out of range [0, %d]", c->max_splits);
    c->splits_forced = splits;
    return KVQ_OK;
}

kvq_status kvq_sync(kvq_cache *c) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    return check_sticky(c);
}

// ---- snapshot / restore (SURVEY 5 checkpoint / resume; SPEC S:535-536 cache dump / load) ----
// The device state of tokens [0, T): the tile arrays of ceil(T/32) tiles (Key and Value code
// words, outlier buckets and their counts), the per-token arrays (Value (s, z), CSR records,
// CSC pointers) and the T_K Key-outlier records; everything else is derived from the create
// parameters.  Layout: a 16-word header, then the arrays in that order.
namespace {
struct SnapHdr {
    uint32_t magic, version, H_q, H_kv, bits, D, kv, NG, kcap_g, vcap_g, QW, VW;
    int64_t T, nnzK;
};
constexpr uint32_t kSnapMagic = 0x5351564bu;   // "KVQS"
struct SnapPart { void *dev; size_t bytes; };
std::vector<SnapPart> snap_parts(kvq_cache *c, int64_t T, int64_t nnzK) {
    const DevCache &d = c->dc;
    const size_t nt = (size_t)((T + 31) / 32);
    return {
        {d.kcodes, nt * d.QW * 32 * 4},
        {d.vcodes, nt * 32 * (size_t)d.VW * 4},
        {d.kit, nt * d.NG * (size_t)d.kcap_g * 4},
        {d.vit, nt * d.NG * (size_t)d.vcap_g * 4},
        {d.gcnt, nt * d.NG * 2 * 4},
        {d.vsz, (size_t)T * sizeof(float2)},
        {d.vout, (size_t)T * d.kv * 4},
        {d.kptr, (size_t)(T + 1) * 4},
        {d.kout, (size_t)nnzK * 4},
    };
}
SnapHdr snap_header(const kvq_cache *c, int64_t T, int64_t nnzK) {
    const DevCache &d = c->dc;
    return SnapHdr{kSnapMagic, 1u, (uint32_t)d.H_q, (uint32_t)d.H_kv, (uint32_t)d.bits, (uint32_t)d.D,
                   (uint32_t)d.kv, (uint32_t)d.NG, (uint32_t)d.kcap_g, (uint32_t)d.vcap_g, (uint32_t)d.QW,
                   (uint32_t)d.VW, T, nnzK};
}
}  // namespace

kvq_status kvq_snapshot_bytes(kvq_cache *c, int64_t *bytes) {
    if (!c || !bytes) return fail(KVQ_EINVAL, "null argument");
    kvq_status st = check_sticky(c);
    if (st != KVQ_OK) return st;
    CK(cudaSetDevice(c->cfg.device));
    uint32_t nnz = 0;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&nnz, c->dc.kptr + c->T, 4, cudaMemcpyDeviceToHost));
    size_t b = sizeof(SnapHdr);
    for (const SnapPart &x : snap_parts(c, c->T, nnz)) b += x.bytes;
    *bytes = (int64_t)b;
    return KVQ_OK;
}

kvq_status kvq_snapshot(kvq_cache *c, void *host, int64_t bytes) {
    NvtxRange r("kvq_snapshot");
    if (!c || !host) return fail(KVQ_EINVAL, "null argument");
    int64_t need = 0;
    kvq_status st = kvq_snapshot_bytes(c, &need);
    if (st != KVQ_OK) return st;
    if (bytes < need) return fail(KVQ_EINVAL, "snapshot needs %lld bytes (got %lld)", (long long)need, (long long)bytes);
    uint32_t nnz = 0;
    CK(cudaMemcpy(&nnz, c->dc.kptr + c->T, 4, cudaMemcpyDeviceToHost));
    const SnapHdr h = snap_header(c, c->T, nnz);
    char *p = (char *)host;
    memcpy(p, &h, sizeof h);
    p += sizeof h;
    for (const SnapPart &x : snap_parts(c, c->T, nnz)) {
        if (x.bytes) CK(cudaMemcpy(p, x.dev, x.bytes, cudaMemcpyDeviceToHost));
        p += x.bytes;
    }
    return KVQ_OK;
}

kvq_status kvq_restore(kvq_cache *c, const void *host, int64_t bytes) {
    NvtxRange r("kvq_restore");
    if (!c || !host) return fail(KVQ_EINVAL, "null argument");
    if (bytes < (int64_t)sizeof(SnapHdr)) return fail(KVQ_EINVAL, "snapshot too short");
    SnapHdr h;
    memcpy(&h, host, sizeof h);
    if (h.magic != kSnapMagic || h.version != 1u) return fail(KVQ_EINVAL, "not a kvq snapshot (magic / version)");
    const SnapHdr mine = snap_header(c, h.T, h.nnzK);
    if (memcmp(&h, &mine, offsetof(SnapHdr, T)) != 0)
        return fail(KVQ_ESHAPE, "snapshot of another cache configuration (heads, bits, D, outliers or buckets differ)");
    if (h.T < 0 || h.T > c->dc.cap) return fail(KVQ_ECAPACITY, "snapshot holds %lld tokens, capacity %lld",
                                                (long long)h.T, (long long)c->dc.cap);
    if (h.nnzK < 0 || h.nnzK > c->dc.kcap) return fail(KVQ_ECAPACITY, "snapshot Key outliers exceed the capacity");
    size_t need = sizeof h;
    const std::vector<SnapPart> parts = snap_parts(c, h.T, h.nnzK);
    for (const SnapPart &x : parts) need += x.bytes;
    if ((size_t)bytes < need) return fail(KVQ_EINVAL, "snapshot truncated (%lld of %zu bytes)", (long long)bytes, need);
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    // start from an empty cache (zeroed code words beyond the restored tiles)
    kvq_status st = kvq_reset(c, nullptr);
    if (st != KVQ_OK) return st;
    const char *p = (const char *)host + sizeof h;
    for (const SnapPart &x : parts) {
        if (x.bytes) CK(cudaMemcpy(x.dev, p, x.bytes, cudaMemcpyHostToDevice));
        p += x.bytes;
    }
    CK(cudaDeviceSynchronize());
    c->T = h.T;
    c->pdl_ok = 0;
    return KVQ_OK;
}

kvq_status kvq_set_pos_base(kvq_cache *c, int64_t pos_base) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (c->T != 0) return fail(KVQ_EINVAL, "set_pos_base needs an empty cache (it holds %lld tokens)", (long long)c->T);
    if (pos_base < 0) return fail(KVQ_EINVAL, "pos_base must be >= 0");
    c->cfg.pos_base = pos_base;
    c->dc.pos_base = pos_base;
    return KVQ_OK;
}

kvq_status kvq_reset(kvq_cache *c, void *stream) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaMemsetAsync(c->dc.kptr, 0, 4, (cudaStream_t)stream));
    CK(cudaMemsetAsync(c->dc.gcnt, 0, (size_t)(c->dc.cap / 32) * c->dc.NG * 2 * 4, (cudaStream_t)stream));
    // Value code words are OR-ed into by the quantizer (fragment layout)
    CK(cudaMemsetAsync(c->dc.vcodes, 0, (size_t)((c->T + 31) / 32) * 32 * c->dc.VW * 4, (cudaStream_t)stream));
    c->T = 0;
    return KVQ_OK;
}

static kvq_status append_tokens(kvq_cache *c, const void *K, const void *V, int64_t T, void *stream) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (T < 0) return fail(KVQ_EINVAL, "negative token count");
    if (T == 0) return KVQ_OK;
    if (!K || !V) return fail(KVQ_EINVAL, "null K or V");
    kvq_status st = check_sticky(c);
    if (st != KVQ_OK) return st;
    if (c->T + T > c->cfg.capacity_tokens)
        return fail(KVQ_ECAPACITY, "token capacity %lld exceeded (have %lld, adding %lld)",
                    (long long)c->cfg.capacity_tokens, (long long)c->T, (long long)T);
    CK(cudaSetDevice(c->cfg.device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)T * c->dc.D * 2;
    const int ck = classify(K, c->cfg.device, c->cfg.flags), cv = classify(V, c->cfg.device, c->cfg.flags);
    if (ck < 0 || cv < 0) return fail(KVQ_EDEVICE, "K/V device pointer is not on device %d", c->cfg.device);
    const __half *Kd = (const __half *)K, *Vd = (const __half *)V;
    if (ck == 1 || cv == 1) {
        st = ensure_stage(c, 2 * bytes);
        if (st != KVQ_OK) return st;
        char *sb = (char *)c->stage;
        if (ck == 1) { CK(cudaMemcpyAsync(sb, K, bytes, cudaMemcpyHostToDevice, s)); Kd = (const __half *)sb; }
        if (cv == 1) { CK(cudaMemcpyAsync(sb + bytes, V, bytes, cudaMemcpyHostToDevice, s)); Vd = (const __half *)(sb + bytes); }
    }
    // the quantize kernels read rows with 16-byte vector loads: stage unaligned device rows
    if (((uintptr_t)Kd | (uintptr_t)Vd) & 15u) {
        st = ensure_stage(c, 2 * bytes);
        if (st != KVQ_OK) return st;
        char *sb = (char *)c->stage;
        if ((const void *)Kd != (const void *)sb) { CK(cudaMemcpyAsync(sb, Kd, bytes, cudaMemcpyDeviceToDevice, s)); Kd = (const __half *)sb; }
        if ((const void *)Vd != (const void *)(sb + bytes)) { CK(cudaMemcpyAsync(sb + bytes, Vd, bytes, cudaMemcpyDeviceToDevice, s)); Vd = (const __half *)(sb + bytes); }
    }
    cudaError_t e = T == 1 ? launch_append(c->dc, Kd, Vd, c->T, s, c->timers ? c->timers + 16 : nullptr)
                           : launch_prefill(c->dc, Kd, Vd, c->T, T, c->dc.lb, c->dc.ticket, s,
                                            c->timers ? c->timers + 16 + 64 : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "quantize launch");
    c->T += T;
    c->pdl_ok = T == 1;
    c->pdl_stream = stream;
    return KVQ_OK;
}

kvq_status kvq_append(kvq_cache *c, const void *k, const void *v, void *stream) {
    NvtxRange r("kvq_append");
    return append_tokens(c, k, v, 1, stream);
}

kvq_status kvq_prefill_quantize(kvq_cache *c, const void *K, const void *V, int64_t T, void *stream) {
    NvtxRange r("kvq_prefill_quantize");
    return append_tokens(c, K, V, T, stream);
}

static kvq_status attend_impl(kvq_cache *c, const void *q, int64_t pos, float *out, int partial,
                              void *stream) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (!q || !out) return fail(KVQ_EINVAL, "null q or output");
    if (pos < 0) return fail(KVQ_EINVAL, "negative position");
    kvq_status st = check_sticky(c);
    if (st != KVQ_OK) return st;
    CK(cudaSetDevice(c->cfg.device));
    cudaStream_t s = (cudaStream_t)stream;
    const int H = c->dc.H_q;
    const size_t qbytes = (size_t)H * kHeadDim * 2;
    const size_t obytes = (size_t)H * (kHeadDim + (partial ? 2 : 0)) * 4;
    if (c->T == 0) {
        if (!partial) return fail(KVQ_EEMPTY, "attend on an empty cache");
        // empty partial: (0, -inf, 0)
        std::vector<float> h((size_t)H * (kHeadDim + 2), 0.f);
        for (int g = 0; g < H; ++g) h[(size_t)g * (kHeadDim + 2) + kHeadDim] = -INFINITY;
        const int co = classify(out, c->cfg.device, c->cfg.flags);
        if (co < 0) return fail(KVQ_EDEVICE, "output pointer not on device %d", c->cfg.device);
        if (co == 1) { memcpy(out, h.data(), obytes); return KVQ_OK; }
        CK(cudaMemcpyAsync(out, h.data(), obytes, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        return KVQ_OK;
    }
    const int cq = classify(q, c->cfg.device, c->cfg.flags), co = classify(out, c->cfg.device, c->cfg.flags);
    if (cq < 0 || co < 0) return fail(KVQ_EDEVICE, "q/output pointer not on device %d", c->cfg.device);
    const __half *qd = (const __half *)q;
    float *od = out;
    if (cq == 1 || co == 1) {
        st = ensure_stage(c, qbytes + obytes + 256);
        if (st != KVQ_OK) return st;
        char *sb = (char *)c->stage;
        if (cq == 1) { CK(cudaMemcpyAsync(sb, q, qbytes, cudaMemcpyHostToDevice, s)); qd = (const __half *)sb; }
        if (co == 1) od = (float *)(sb + ((qbytes + 255) / 256) * 256);
    }
    AttendArgs a;
    a.q = qd; a.pos = pos; a.T = c->T; a.out = od; a.write_partial = partial;
    a.parts = c->parts; a.tickets = c->tickets; a.splits = c->splits_forced;
    a.timers = c->timers;
    a.kernel_out = &c->last_kernel;
    a.hg_out = &c->hg;
    static const bool no_pdl = getenv("KVQ_NO_PDL") != nullptr;   // diagnostics switch
    a.pdl = (c->cfg.flags & KVQ_FLAG_DECODE_PDL) && c->pdl_ok && c->pdl_stream == stream && cq == 0 && !no_pdl;
    c->pdl_ok = 0;
    cudaError_t e = launch_attend(c->dc, a, &c->last_splits, s);
    if (e != cudaSuccess) return cuda_fail(e, "attend launch");
    if (co == 1) {
        CK(cudaMemcpyAsync(out, od, obytes, cudaMemcpyDeviceToHost, s));
        if (!host_pinned(out)) CK(cudaStreamSynchronize(s));
    }
    return KVQ_OK;
}

kvq_status kvq_decode_attend(kvq_cache *c, const void *q, int64_t pos, float *o, void *stream) {
    NvtxRange r("kvq_decode_attend");
    return attend_impl(c, q, pos, o, 0, stream);
}

kvq_status kvq_decode_attend_partial(kvq_cache *c, const void *q, int64_t pos, float *part, void *stream) {
    NvtxRange r("kvq_decode_attend_partial");
    return attend_impl(c, q, pos, part, 1, stream);
}

static kvq_status attend_batch_impl(kvq_cache *const *caches, int32_t B, const void *const *q, const int64_t *pos,
                                    float *const *o, int partial, void *stream) {
    if (!caches || !q || !pos || !o) return fail(KVQ_EINVAL, "null argument");
    if (B < 1) return fail(KVQ_EINVAL, "B must be >= 1");
    for (int i = 0; i < B; ++i) {
        if (!caches[i] || !q[i] || !o[i]) return fail(KVQ_EINVAL, "null cache, q or o at %d", i);
        if (pos[i] < 0) return fail(KVQ_EINVAL, "negative position at %d", i);
        if (caches[i]->T == 0) return fail(KVQ_EEMPTY, "attend on an empty cache (sequence %d)", i);
        if (caches[i]->cfg.device != caches[0]->cfg.device) return fail(KVQ_EDEVICE, "caches on different devices");
        kvq_status st = check_sticky(caches[i]);
        if (st != KVQ_OK) return st;
    }
    bool one_launch = B <= attend_batch_max();
    const DevCache &d0 = caches[0]->dc;
    // MHA: att_wa_batch_kernel; GQA: att_wgt_batch_kernel (getenv read once: KVQ_WGT_OFF keeps the
    // per-sequence LUT kernel for A/B)
    static const bool wgt_off = getenv("KVQ_WGT_OFF") != nullptr;
    const bool gqa = attend_wag_supported(d0) && !(wgt_off && d0.G != 8 && d0.bits != 4);
    for (int i = 0; i < B && one_launch; ++i) {
        const DevCache &d = caches[i]->dc;
        one_launch = (gqa ? attend_wag_supported(d) : attend_wa_supported(d)) && d.bits == d0.bits &&
                     d.vcb_exact16 == d0.vcb_exact16 && d.H_q == d0.H_q && d.H_kv == d0.H_kv;
    }
    if (!one_launch) {   // shapes the batched kernel does not cover: one attend per cache
        for (int i = 0; i < B; ++i) {
            kvq_status st = attend_impl(caches[i], q[i], pos[i], o[i], partial, stream);
            if (st != KVQ_OK) return st;
        }
        return KVQ_OK;
    }
    const int dev = caches[0]->cfg.device;
    CK(cudaSetDevice(dev));
    std::vector<const DevCache *> cs((size_t)B);
    std::vector<AttendArgs> as((size_t)B);
    std::vector<int> splits((size_t)B);
    for (int i = 0; i < B; ++i) {
        kvq_cache *c = caches[i];
        if (classify(q[i], dev, c->cfg.flags) != 0 || classify(o[i], dev, c->cfg.flags) != 0)
            return fail(KVQ_EDEVICE, "batched attend takes device q / o on device %d (sequence %d)", dev, i);
        cs[(size_t)i] = &c->dc;
        AttendArgs &a = as[(size_t)i];
        a = AttendArgs{};
        a.q = (const __half *)q[i]; a.pos = pos[i]; a.T = c->T; a.out = o[i]; a.write_partial = partial;
        a.parts = c->parts; a.tickets = c->tickets; a.splits = c->splits_forced;
    }
    cudaError_t e = gqa ? launch_attend_wgt_batch(cs.data(), as.data(), B, (cudaStream_t)stream, splits.data())
                        : launch_attend_wa_batch(cs.data(), as.data(), B, (cudaStream_t)stream, splits.data());
    if (e != cudaSuccess) return cuda_fail(e, "batched attend launch");
    for (int i = 0; i < B; ++i) {
        caches[i]->last_splits = splits[(size_t)i];
        caches[i]->last_kernel = gqa ? 2 : 1;
        caches[i]->pdl_ok = 0;
    }
    return KVQ_OK;
}

kvq_status kvq_decode_attend_batch(kvq_cache *const *caches, int32_t B, const void *const *q, const int64_t *pos,
                                   float *const *o, void *stream) {
    NvtxRange r("kvq_decode_attend_batch");
    return attend_batch_impl(caches, B, q, pos, o, 0, stream);
}

kvq_status kvq_decode_attend_batch_partial(kvq_cache *const *caches, int32_t B, const void *const *q,
                                           const int64_t *pos, float *const *part, void *stream) {
    NvtxRange r("kvq_decode_attend_batch_partial");
    return attend_batch_impl(caches, B, q, pos, part, 1, stream);
}

kvq_status kvq_merge_partials(const float *parts, int32_t P, int32_t H, int32_t d, float *o,
                              int32_t device, void *stream) {
    NvtxRange r("kvq_merge_partials");
    if (!parts || !o) return fail(KVQ_EINVAL, "null argument");
    if (P < 1 || H < 1 || d < 1) return fail(KVQ_EINVAL, "P, H_q, d must be >= 1");
    CK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    const int cp = classify(parts, device, 0), co = classify(o, device, 0);
    if (cp < 0 || co < 0) return fail(KVQ_EDEVICE, "pointer not on device %d", device);
    const size_t pb = (size_t)P * H * (d + 2) * 4, ob = (size_t)H * d * 4;
    const float *pd = parts;
    float *od = o;
    void *tmp = nullptr;
    if (cp == 1 || co == 1) {
        CK(cudaMallocAsync(&tmp, pb + ob, s));
        if (cp == 1) { CK(cudaMemcpyAsync(tmp, parts, pb, cudaMemcpyHostToDevice, s)); pd = (const float *)tmp; }
        if (co == 1) od = (float *)((char *)tmp + pb);
    }
    cudaError_t e = launch_merge(pd, P, H, d, od, s);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
    if (co == 1) { CK(cudaMemcpyAsync(o, od, ob, cudaMemcpyDeviceToHost, s)); }
    if (tmp) { CK(cudaFreeAsync(tmp, s)); }
    if (co == 1 && !host_pinned(o)) CK(cudaStreamSynchronize(s));
    return KVQ_OK;
}

kvq_status kvq_key_outlier_span(kvq_cache *c, int64_t t0, int64_t t1, int64_t *begin, int64_t *end) {
    if (!c || !begin || !end) return fail(KVQ_EINVAL, "null argument");
    if (t0 < 0 || t1 < t0 || t1 > c->T) return fail(KVQ_EINVAL, "bad token range");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    uint32_t a = 0, b = 0;
    CK(cudaMemcpy(&a, c->dc.kptr + t0, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&b, c->dc.kptr + t1, 4, cudaMemcpyDeviceToHost));
    *begin = a;
    *end = b;
    return check_sticky(c);
}

kvq_status kvq_export(kvq_cache *c, int64_t t0, int64_t t1, kvq_export_buf *buf) {
    if (!c || !buf) return fail(KVQ_EINVAL, "null argument");
    if (t0 < 0 || t1 < t0 || t1 > c->T) return fail(KVQ_EINVAL, "bad token range");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    kvq_status st = check_sticky(c);
    if (st != KVQ_OK) return st;
    const DevCache &d = c->dc;
    const int64_t n = t1 - t0;
    const int b = d.bits, D = d.D;
    if (n == 0) { if (buf->kptr) { uint32_t a; CK(cudaMemcpy(&a, d.kptr + t0, 4, cudaMemcpyDeviceToHost)); buf->kptr[0] = a; } return KVQ_OK; }
    if (buf->kcodes) {
        const int64_t tile0 = t0 / 32, tile1 = (t1 + 31) / 32;
        std::vector<uint32_t> kc((size_t)(tile1 - tile0) * d.QW * 32);
        CK(cudaMemcpy(kc.data(), d.kcodes + tile0 * d.QW * 32, kc.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t tl = t / 32 - tile0;
            const int j = (int)(t % 32);
            uint8_t *row = buf->kcodes + (t - t0) * D;
            for (int h = 0; h < d.H_kv; ++h) {
                for (int p = 0; p < kPairs; ++p) {
                    const int bit = 2 * b * p;
                    const int q = h * 4 * b + bit / 32;
                    uint64_t w = kc[((size_t)tl * d.QW + q) * 32 + j];
                    if (bit % 32 + 2 * b > 32) w |= (uint64_t)kc[((size_t)tl * d.QW + q + 1) * 32 + j] << 32;
                    const unsigned pc = (unsigned)(w >> (bit % 32)) & ((1u << (2 * b)) - 1);
                    row[h * kHeadDim + p] = (uint8_t)(pc & ((1u << b) - 1));
                    row[h * kHeadDim + p + kPairs] = (uint8_t)(pc >> b);
                }
            }
        }
    }
    if (buf->vcodes) {
        const int64_t tile0 = t0 / 32, tile1 = (t1 + 31) / 32;
        const int hw = 4 * b;   // words per (token, kv head)
        std::vector<uint32_t> vc((size_t)(tile1 - tile0) * d.H_kv * 32 * hw);
        CK(cudaMemcpy(vc.data(), d.vcodes + tile0 * d.H_kv * 32 * hw, vc.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t tl = t / 32 - tile0;
            const int j = (int)(t % 32);
            for (int ch = 0; ch < D; ++ch) {
                const int h = ch / kHeadDim, cc = ch % kHeadDim;
                const int bit = vf_bit(j, cc, b), lane = vf_lane(j, cc);
                const uint32_t *wp = vc.data() + vf_word(tl, d.H_kv, h, bit / 32, lane, b);
                uint64_t w = wp[0];
                if (bit % 32 + b > 32) w |= (uint64_t)wp[32] << 32;
                buf->vcodes[(t - t0) * D + ch] = (uint8_t)((w >> (bit % 32)) & ((1u << b) - 1));
            }
        }
    }
    if (buf->vs || buf->vz) {
        std::vector<float2> sz((size_t)n);
        CK(cudaMemcpy(sz.data(), d.vsz + t0, (size_t)n * sizeof(float2), cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < n; ++t) {
            if (buf->vs) buf->vs[t] = sz[t].x;
            if (buf->vz) buf->vz[t] = sz[t].y;
        }
    }
    if ((buf->vidx || buf->vval) && d.kv > 0) {
        std::vector<uint32_t> vo((size_t)n * d.kv);
        CK(cudaMemcpy(vo.data(), d.vout + t0 * d.kv, vo.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t r = 0; r < vo.size(); ++r) {
            if (buf->vidx) buf->vidx[r] = (uint16_t)(vo[r] & 0xffffu);
            if (buf->vval) buf->vval[r] = (uint16_t)(vo[r] >> 16);
        }
    }
    if (buf->kptr) {
        std::vector<uint32_t> kp((size_t)n + 1);
        CK(cudaMemcpy(kp.data(), d.kptr + t0, kp.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t r = 0; r < kp.size(); ++r) buf->kptr[r] = kp[r];
        if (buf->kidx || buf->kval) {
            const int64_t nnz = (int64_t)kp[n] - kp[0];
            if (nnz > 0) {
                std::vector<uint32_t> ko((size_t)nnz);
                CK(cudaMemcpy(ko.data(), d.kout + kp[0], ko.size() * 4, cudaMemcpyDeviceToHost));
                for (size_t r = 0; r < ko.size(); ++r) {
                    if (buf->kidx) buf->kidx[r] = (uint16_t)(ko[r] & 0xffffu);
                    if (buf->kval) buf->kval[r] = (uint16_t)(ko[r] >> 16);
                }
            }
        }
    }
    return KVQ_OK;
}

// ------------------------------------------------ online per-channel Key thresholds --
kvq_status kvq_key_thresholds_online(const void *K, int64_t T, int32_t D, int32_t ppm, float *key_lo,
                                     float *key_hi, int32_t device, void *stream) {
    if (!K || !key_lo || !key_hi) return fail(KVQ_EINVAL, "null argument");
    if (T < 1 || D < 1) return fail(KVQ_EINVAL, "T and D must be >= 1");
    if (ppm < 0 || ppm >= 500000) return fail(KVQ_EINVAL, "outlier_ppm must be in [0, 500000)");
    const int64_t n = ((int64_t)ppm * T + 999999) / 1000000;
    if ((n + 1) / 2 + n / 2 >= T) return fail(KVQ_EINVAL, "too many outliers (%lld) for %lld tokens", (long long)n, (long long)T);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(KVQ_EDEVICE, "device %d not present", device);
    CK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    const int ck = classify(K, device, 0), cl = classify(key_lo, device, 0), ch = classify(key_hi, device, 0);
    if (ck < 0 || cl < 0 || ch < 0) return fail(KVQ_EDEVICE, "pointer not on device %d", device);
    const size_t kb = (size_t)T * D * 2, ob = (size_t)D * 4;
    void *tmp = nullptr;
    const size_t need = (ck == 1 ? kb : 0) + 2 * ob + 256;
    CK(cudaMallocAsync(&tmp, need, s));
    char *tp = (char *)tmp;
    const __half *Kd = (const __half *)K;
    if (ck == 1) { CK(cudaMemcpyAsync(tp, K, kb, cudaMemcpyHostToDevice, s)); Kd = (const __half *)tp; tp += (kb + 255) / 256 * 256; }
    float *lo = cl == 1 ? (float *)tp : key_lo;
    float *hi = ch == 1 ? (float *)(tp + ob) : key_hi;
    cudaError_t e = launch_online_key_thresholds(Kd, T, D, ppm, lo, hi, s);
    if (e != cudaSuccess) { cudaFreeAsync(tmp, s); return cuda_fail(e, "online thresholds launch"); }
    if (cl == 1) CK(cudaMemcpyAsync(key_lo, lo, ob, cudaMemcpyDeviceToHost, s));
    if (ch == 1) CK(cudaMemcpyAsync(key_hi, hi, ob, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(tmp, s));
    if (cl == 1 || ch == 1) CK(cudaStreamSynchronize(s));
    return KVQ_OK;
}

// ------------------------------------------- mixed-precision sensitivity (f4) ----------
kvq_status kvq_layer_sensitivity(kvq_cache *c, const void *K, const void *V, const float *FK, const float *FV,
                                 int64_t t0, int64_t T, double *omega, void *stream) {
    if (!c || !K || !V || !omega) return fail(KVQ_EINVAL, "null argument");
    if (t0 < 0 || T < 0 || t0 + T > c->T) return fail(KVQ_EINVAL, "tokens [%lld, %lld) not cached (%lld)",
                                                     (long long)t0, (long long)(t0 + T), (long long)c->T);
    kvq_status st = check_sticky(c);
    if (st != KVQ_OK) return st;
    const int dev = c->cfg.device;
    CK(cudaSetDevice(dev));
    cudaStream_t s = (cudaStream_t)stream;
    const void *ins[4] = {K, V, FK, FV};
    int cls[4];
    for (int i = 0; i < 4; ++i) {
        cls[i] = ins[i] ? classify(ins[i], dev, 0) : 0;
        if (cls[i] < 0) return fail(KVQ_EDEVICE, "input pointer not on device %d", dev);
    }
    const int co = classify(omega, dev, 0);
    if (co < 0) return fail(KVQ_EDEVICE, "omega pointer not on device %d", dev);
    const size_t eb[4] = {(size_t)T * c->dc.D * 2, (size_t)T * c->dc.D * 2, (size_t)T * c->dc.D * 4,
                          (size_t)T * c->dc.D * 4};
    size_t need = 256;
    for (int i = 0; i < 4; ++i) if (cls[i] == 1) need += (eb[i] + 255) / 256 * 256;
    void *tmp = nullptr;
    CK(cudaMallocAsync(&tmp, need, s));
    char *tp = (char *)tmp;
    const void *dv[4];
    for (int i = 0; i < 4; ++i) {
        dv[i] = ins[i];
        if (cls[i] == 1 && eb[i]) {
            CK(cudaMemcpyAsync(tp, ins[i], eb[i], cudaMemcpyHostToDevice, s));
            dv[i] = tp;
            tp += (eb[i] + 255) / 256 * 256;
        }
    }
    double *od = co == 1 ? (double *)tp : omega;
    cudaError_t e = launch_layer_sensitivity(c->dc, (const __half *)dv[0], (const __half *)dv[1],
                                             (const float *)dv[2], (const float *)dv[3], t0, T, od, s);
    if (e != cudaSuccess) { cudaFreeAsync(tmp, s); return cuda_fail(e, "sensitivity launch"); }
    if (co == 1) CK(cudaMemcpyAsync(omega, od, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(tmp, s));
    if (co == 1) CK(cudaStreamSynchronize(s));
    return KVQ_OK;
}

kvq_status kvq_fisher_accumulate(float *F, const float *g, int64_t n, int32_t device, void *stream) {
    if (!F || !g) return fail(KVQ_EINVAL, "null argument");
    if (n < 0) return fail(KVQ_EINVAL, "negative element count");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(KVQ_EDEVICE, "device %d not present", device);
    CK(cudaSetDevice(device));
    if (classify(F, device, 0) != 0 || classify(g, device, 0) != 0)
        return fail(KVQ_EDEVICE, "F and g must be device pointers on device %d", device);
    cudaError_t e = launch_fisher_accumulate(F, g, n, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "fisher launch");
    return KVQ_OK;
}

kvq_status kvq_assign_bits(const double *omega, int32_t L, int32_t demote_count, int32_t bits_high,
                           int32_t bits_low, int32_t *bits_out) {
    if (!omega || !bits_out) return fail(KVQ_EINVAL, "null argument");
    if (L < 0 || demote_count < 0 || demote_count > L)
        return fail(KVQ_EINVAL, "demote_count %d out of [0, %d]", demote_count, L);
    for (int i = 0; i < L; ++i)
        if (!(omega[i] >= 0.0)) return fail(KVQ_EINVAL, "omega[%d] is negative or NaN", i);
    std::vector<int> idx((size_t)L);
    for (int i = 0; i < L; ++i) idx[(size_t)i] = i;
    // smallest omega first, ties to the lower layer index (a stable order)
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return omega[x] < omega[y]; });
    for (int i = 0; i < L; ++i) bits_out[i] = bits_high;
    for (int r = 0; r < demote_count; ++r) bits_out[idx[(size_t)r]] = bits_low;
    return KVQ_OK;
}

kvq_status kvq_calibrate_layer(const void *K, const void *V, const float *FK, const float *FV, int64_t N, int32_t D,
                               const kvq_calib_config *cfg, float *key_lo, float *key_hi, float *key_cb,
                               float *key_cb_dec, float *val_cb, float *val_cb_dec, int32_t *iters,
                               int32_t device, void *stream) {
    if (!K || !V || !cfg || !key_lo || !key_hi || !key_cb || !key_cb_dec || !val_cb || !val_cb_dec)
        return fail(KVQ_EINVAL, "null argument");
    const kvq_calib_config &C = *cfg;
    if (C.bits < 2 || C.bits > 4) return fail(KVQ_EINVAL, "bits must be 2, 3 or 4");
    if (C.outlier_ppm < 0 || C.outlier_ppm >= 500000) return fail(KVQ_EINVAL, "outlier_ppm must be in [0, 500000)");
    if (C.max_iter < 1) return fail(KVQ_EINVAL, "max_iter must be >= 1");
    if (!(C.tol >= 0.0)) return fail(KVQ_EINVAL, "tol must be >= 0");
    if (N < 1 || D < 128 || D % 128 || D > 8192) return fail(KVQ_EINVAL, "need N >= 1 and D a multiple of 128 <= 8192");
    const int64_t n = ((int64_t)C.outlier_ppm * N + 999999) / 1000000;
    if ((n + 1) / 2 + n / 2 >= N) return fail(KVQ_EINVAL, "too many Key outliers (%lld) for %lld tokens", (long long)n, (long long)N);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(KVQ_EDEVICE, "device %d not present", device);
    CK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    const void *ins[4] = {K, V, FK, FV};
    const size_t ib[4] = {(size_t)N * D * 2, (size_t)N * D * 2, (size_t)N * D * 4, (size_t)N * D * 4};
    void *outs[7] = {key_lo, key_hi, key_cb, key_cb_dec, val_cb, val_cb_dec, iters};
    const int nlev = 1 << C.bits;
    const size_t ob[7] = {(size_t)D * 4, (size_t)D * 4, (size_t)nlev * 4, (size_t)nlev * 4, (size_t)nlev * 4,
                          (size_t)nlev * 4, 2 * 4};
    int ci[4], co[7];
    for (int i = 0; i < 4; ++i) {
        ci[i] = ins[i] ? classify(ins[i], device, 0) : 0;
        if (ci[i] < 0) return fail(KVQ_EDEVICE, "input pointer not on device %d", device);
    }
    bool host_out = false;
    for (int i = 0; i < 7; ++i) {
        co[i] = outs[i] ? classify(outs[i], device, 0) : 0;
        if (co[i] < 0) return fail(KVQ_EDEVICE, "output pointer not on device %d", device);
        host_out |= outs[i] && co[i] == 1;
    }
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    size_t need = al((size_t)D * 4) * 2 + al(64 * 4) + al(4 * 4);
    for (int i = 0; i < 4; ++i) if (ci[i] == 1) need += al(ib[i]);
    void *tmp = nullptr;
    CK(cudaMallocAsync(&tmp, need, s));
    char *tp = (char *)tmp;
    float *lo_d = (float *)tp; tp += al((size_t)D * 4);
    float *hi_d = (float *)tp; tp += al((size_t)D * 4);
    float *cb_d = (float *)tp; tp += al(64 * 4);
    int *it_d = (int *)tp; tp += al(4 * 4);
    const void *dv[4];
    for (int i = 0; i < 4; ++i) {
        dv[i] = ins[i];
        if (ins[i] && ci[i] == 1) {
            CK(cudaMemcpyAsync(tp, ins[i], ib[i], cudaMemcpyHostToDevice, s));
            dv[i] = tp;
            tp += al(ib[i]);
        }
    }
    cudaError_t e = launch_calibrate((const __half *)dv[0], (const __half *)dv[1], (const float *)dv[2],
                                     (const float *)dv[3], N, D, C.bits, C.outlier_ppm, C.max_iter, C.tol, C.qnorm,
                                     C.fp16_codebooks, lo_d, hi_d, cb_d, it_d, s);
    if (e != cudaSuccess) { cudaFreeAsync(tmp, s); return cuda_fail(e, "calibration launch"); }
    const void *srcs[7] = {lo_d, hi_d, cb_d, cb_d + 16, cb_d + 32, cb_d + 48, it_d};
    for (int i = 0; i < 7; ++i) {
        if (!outs[i]) continue;
        CK(cudaMemcpyAsync(outs[i], srcs[i], ob[i], co[i] == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaFreeAsync(tmp, s));
    if (host_out) CK(cudaStreamSynchronize(s));
    return KVQ_OK;
}

// ------------------------------------------------------------- fp16 comparator cache --
struct kvq_f16_cache {
    kvq_config cfg;
    F16Dev dc;
    int64_t T = 0;
    double *theta = nullptr;
    float *parts = nullptr;
    unsigned *tickets = nullptr;
    void *stage = nullptr;
    size_t stage_bytes = 0;
    std::vector<void *> allocs;
};

static kvq_status f16_alloc(kvq_f16_cache *c, void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    e = cudaMemset(*p, 0, bytes ? bytes : 16);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset");
    c->allocs.push_back(*p);
    return KVQ_OK;
}

static kvq_status f16_stage(kvq_f16_cache *c, size_t bytes) {
    if (c->stage_bytes >= bytes) return KVQ_OK;
    if (c->stage) { cudaFree(c->stage); c->stage = nullptr; }
    CK(cudaMalloc(&c->stage, bytes));
    c->stage_bytes = bytes;
    return KVQ_OK;
}

void kvq_f16_cache_destroy(kvq_f16_cache *c) {
    if (!c) return;
    cudaSetDevice(c->cfg.device);
    cudaDeviceSynchronize();
    for (void *p : c->allocs) cudaFree(p);
    if (c->stage) cudaFree(c->stage);
    delete c;
}

kvq_status kvq_f16_cache_create(const kvq_config *cfg, kvq_f16_cache **out) {
    if (!cfg || !out) return fail(KVQ_EINVAL, "null argument");
    const kvq_config &C = *cfg;
    if (C.n_q_heads < 1 || C.n_kv_heads < 1 || C.n_q_heads % C.n_kv_heads)
        return fail(KVQ_ESHAPE, "head counts must be >= 1 with n_q_heads %% n_kv_heads == 0");
    if (C.n_q_heads != C.n_kv_heads) return fail(KVQ_ESHAPE, "the fp16 comparator supports MHA (G = 1)");
    if (C.head_dim != kHeadDim) return fail(KVQ_ESHAPE, "this build supports head_dim == 128");
    if ((int64_t)C.n_kv_heads * kHeadDim > 8192) return fail(KVQ_ESHAPE, "D = H_kv*d must be <= 8192");
    if (C.capacity_tokens < 1) return fail(KVQ_EINVAL, "capacity_tokens must be >= 1");
    if (!(C.rope_theta > 0) || !std::isfinite(C.rope_theta)) return fail(KVQ_EINVAL, "rope_theta must be > 0");
    if (C.pos_base < 0) return fail(KVQ_EINVAL, "pos_base must be >= 0");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (C.device < 0 || C.device >= ndev) return fail(KVQ_EDEVICE, "device %d not present", C.device);
    CK(cudaSetDevice(C.device));
    kvq_f16_cache *c = new (std::nothrow) kvq_f16_cache();
    if (!c) return fail(KVQ_EINVAL, "out of host memory");
    c->cfg = C;
    F16Dev &d = c->dc;
    d.H_q = C.n_q_heads; d.H_kv = C.n_kv_heads; d.G = C.n_q_heads / C.n_kv_heads;
    d.D = C.n_kv_heads * kHeadDim;
    d.cap = C.capacity_tokens;
    d.pos_base = C.pos_base;
    kvq_status st = KVQ_OK;
    void *p = nullptr;
    if (st == KVQ_OK && (st = f16_alloc(c, &p, (size_t)d.cap * d.D * 2)) == KVQ_OK) d.K = (__half *)p;
    if (st == KVQ_OK && (st = f16_alloc(c, &p, (size_t)d.cap * d.D * 2)) == KVQ_OK) d.V = (__half *)p;
    if (st == KVQ_OK && (st = f16_alloc(c, &p, 64 * 8)) == KVQ_OK) c->theta = (double *)p;
    if (st == KVQ_OK && (st = f16_alloc(c, &p, (size_t)4 * 148 * d.H_q * (kHeadDim + 2) * 4)) == KVQ_OK) c->parts = (float *)p;
    if (st == KVQ_OK && (st = f16_alloc(c, &p, (size_t)d.H_q * 4)) == KVQ_OK) c->tickets = (unsigned *)p;
    if (st != KVQ_OK) { kvq_f16_cache_destroy(c); return st; }
    double th[64];
    for (int i = 0; i < 64; ++i) th[i] = std::pow(C.rope_theta, -2.0 * (double)i / (double)kHeadDim);
    cudaError_t e = cudaMemcpy(c->theta, th, sizeof th, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { kvq_f16_cache_destroy(c); return cuda_fail(e, "upload theta"); }
    d.theta_tab = c->theta;
    *out = c;
    return KVQ_OK;
}

int64_t kvq_f16_num_tokens(const kvq_f16_cache *c) { return c ? c->T : 0; }

kvq_status kvq_f16_append(kvq_f16_cache *c, const void *K, const void *V, int64_t T, void *stream) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (T < 0) return fail(KVQ_EINVAL, "negative token count");
    if (T == 0) return KVQ_OK;
    if (!K || !V) return fail(KVQ_EINVAL, "null K or V");
    if (c->T + T > c->dc.cap) return fail(KVQ_ECAPACITY, "token capacity %lld exceeded", (long long)c->dc.cap);
    CK(cudaSetDevice(c->cfg.device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)T * c->dc.D * 2;
    const int ck = classify(K, c->cfg.device, c->cfg.flags), cv = classify(V, c->cfg.device, c->cfg.flags);
    if (ck < 0 || cv < 0) return fail(KVQ_EDEVICE, "K/V pointer not on device %d", c->cfg.device);
    const __half *Kd = (const __half *)K, *Vd = (const __half *)V;
    if (ck == 1 || cv == 1) {
        kvq_status st = f16_stage(c, 2 * bytes);
        if (st != KVQ_OK) return st;
        char *sb = (char *)c->stage;
        if (ck == 1) { CK(cudaMemcpyAsync(sb, K, bytes, cudaMemcpyHostToDevice, s)); Kd = (const __half *)sb; }
        if (cv == 1) { CK(cudaMemcpyAsync(sb + bytes, V, bytes, cudaMemcpyHostToDevice, s)); Vd = (const __half *)(sb + bytes); }
    }
    cudaError_t e = launch_f16_store(c->dc, Kd, Vd, c->T, T, s);
    if (e != cudaSuccess) return cuda_fail(e, "f16 store launch");
    c->T += T;
    return KVQ_OK;
}

kvq_status kvq_f16_decode_attend(kvq_f16_cache *c, const void *q, int64_t pos, float *o, void *stream) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (!q || !o) return fail(KVQ_EINVAL, "null q or output");
    if (pos < 0) return fail(KVQ_EINVAL, "negative position");
    if (c->T == 0) return fail(KVQ_EEMPTY, "attend on an empty cache");
    CK(cudaSetDevice(c->cfg.device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t qb = (size_t)c->dc.H_q * kHeadDim * 2, ob = (size_t)c->dc.H_q * kHeadDim * 4;
    const int cq = classify(q, c->cfg.device, c->cfg.flags), co = classify(o, c->cfg.device, c->cfg.flags);
    if (cq < 0 || co < 0) return fail(KVQ_EDEVICE, "q/output pointer not on device %d", c->cfg.device);
    const __half *qd = (const __half *)q;
    float *od = o;
    if (cq == 1 || co == 1) {
        kvq_status st = f16_stage(c, qb + ob + 256);
        if (st != KVQ_OK) return st;
        char *sb = (char *)c->stage;
        if (cq == 1) { CK(cudaMemcpyAsync(sb, q, qb, cudaMemcpyHostToDevice, s)); qd = (const __half *)sb; }
        if (co == 1) od = (float *)(sb + ((qb + 255) / 256) * 256);
    }
    const int S = f16_auto_splits(c->dc, c->T);
    cudaError_t e = launch_f16_attend(c->dc, qd, pos, c->T, od, c->parts, c->tickets, S, s);
    if (e != cudaSuccess) return cuda_fail(e, "f16 attend launch");
    if (co == 1) {
        CK(cudaMemcpyAsync(o, od, ob, cudaMemcpyDeviceToHost, s));
        if (!host_pinned(o)) CK(cudaStreamSynchronize(s));
    }
    return KVQ_OK;
}

kvq_status kvq_f16_export(kvq_f16_cache *c, int64_t t0, int64_t t1, uint16_t *k_out, uint16_t *v_out) {
    if (!c) return fail(KVQ_EINVAL, "null cache");
    if (t0 < 0 || t1 < t0 || t1 > c->T) return fail(KVQ_EINVAL, "bad token range");
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaDeviceSynchronize());
    const size_t n = (size_t)(t1 - t0) * c->dc.D * 2;
    if (k_out && n) CK(cudaMemcpy(k_out, c->dc.K + t0 * c->dc.D, n, cudaMemcpyDeviceToHost));
    if (v_out && n) CK(cudaMemcpy(v_out, c->dc.V + t0 * c->dc.D, n, cudaMemcpyDeviceToHost));
    return KVQ_OK;
}

}  // extern "C"
