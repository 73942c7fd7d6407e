"""KVQuant CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/kvq_oracle.c`` (plain fp64 C, see its header for the
paper passages each function follows).  Nothing in the product package
(``paper_2401_18079_b200``) imports this module; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs do.  The shared library is compiled with gcc on first use (or by
``__graft_entry__.build()``); building the checker is not using it.

Canonical cache form (the exchange format the GPU export is compared against):
    kcodes  uint16 [T, D]     Key codes, channel order
    kptr    int64  [T+1]      Key outlier CSC column pointers (tokens are columns)
    kidx    int32  [nnz]      Key outlier channel, ascending within a token
    kval    uint16 [nnz]      Key outlier original fp16 bits
    vcodes  uint16 [T, D]     Value codes
    vidx    int32  [T, k]     Value outlier channels (k = ceil(f*D) per token), ascending
    vval    uint16 [T, k]     Value outlier original fp16 bits
    vs, vz  float32 [T]       per-token Value scale / offset
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kvq_oracle.c")
_LIB = os.path.join(_HERE, "libkvq_oracle.so")
_lock = threading.Lock()
_lib = None

P_f64 = ctypes.POINTER(ctypes.c_double)
P_f32 = ctypes.POINTER(ctypes.c_float)
P_u16 = ctypes.POINTER(ctypes.c_uint16)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_u32 = ctypes.POINTER(ctypes.c_uint32)
P_u8 = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, -O2, OpenMP)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(
                ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                 "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB)
    lib.kvo_f16_to_f64.restype = ctypes.c_double
    lib.kvo_f16_to_f64.argtypes = [ctypes.c_uint16]
    lib.kvo_rope.argtypes = [P_f64, ctypes.c_int, ctypes.c_int64, ctypes.c_double, P_f64]
    lib.kvo_affine_from_range.argtypes = [ctypes.c_double, ctypes.c_double, P_f32, P_f32]
    lib.kvo_enc.restype = ctypes.c_int
    lib.kvo_enc.argtypes = [ctypes.c_double, ctypes.c_float, ctypes.c_float, P_f32, ctypes.c_int]
    lib.kvo_quantize_key.restype = ctypes.c_int
    lib.kvo_quantize_key.argtypes = [P_u16, ctypes.c_int, P_f32, P_f32, P_f32, ctypes.c_int,
                                     P_u16, P_i32, P_u16]
    lib.kvo_outlier_count.restype = ctypes.c_int
    lib.kvo_outlier_count.argtypes = [ctypes.c_int, ctypes.c_int]
    lib.kvo_select_outliers.argtypes = [P_u16, ctypes.c_int, ctypes.c_int, P_u8]
    lib.kvo_quantize_value.restype = ctypes.c_int
    lib.kvo_quantize_value.argtypes = [P_u16, ctypes.c_int, ctypes.c_int, P_f32, ctypes.c_int,
                                       ctypes.c_int, P_u16, P_i32, P_u16, P_f32, P_f32]
    lib.kvo_key_thresholds_online.restype = ctypes.c_int
    lib.kvo_key_thresholds_online.argtypes = [ctypes.c_int64, ctypes.c_int, P_u16, ctypes.c_int, P_f32, P_f32]
    lib.kvo_f64_to_f16.restype = ctypes.c_uint16
    lib.kvo_f64_to_f16.argtypes = [ctypes.c_double]
    lib.kvo_f16cache_key.argtypes = [P_u16, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_double, P_u16]
    lib.kvo_attend_dense.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P_u16, P_u16,
                                     P_u16, ctypes.c_int64, ctypes.c_double, P_f64]
    lib.kvo_prefill.restype = ctypes.c_int64
    lib.kvo_prefill.argtypes = [ctypes.c_int64, ctypes.c_int, P_u16, P_u16, P_f32, P_f32,
                                P_f32, P_f32, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                P_u16, P_i64, P_i32, P_u16, ctypes.c_int64,
                                P_u16, P_i32, P_u16, P_f32, P_f32]
    lib.kvo_attend.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               P_u16, P_i64, P_i32, P_u16, P_u16, ctypes.c_int, P_i32, P_u16,
                               P_f32, P_f32, P_f32, P_f32, P_f32, P_f32, P_u16,
                               ctypes.c_int64, ctypes.c_int64, ctypes.c_double, P_f64,
                               ctypes.c_int]
    lib.kvo_merge.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P_f64, P_f64]
    lib.kvo_pack.argtypes = [P_u16, ctypes.c_int64, ctypes.c_int, P_u32]
    lib.kvo_unpack.argtypes = [P_u32, ctypes.c_int64, ctypes.c_int, P_u16]
    _lib = lib
    return lib


def _p(a: np.ndarray, ptype):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ptype)


def _f16bits(x) -> np.ndarray:
    a = np.asarray(x)
    if a.dtype == np.uint16:
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(a.astype(np.float16)).view(np.uint16)


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


# ----------------------------------------------------------------- elementary ops ---
def f16_to_f64(h: int) -> float:
    return _load().kvo_f16_to_f64(int(h))


def rope(x, pos: int, theta_base: float = 10000.0) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty_like(x)
    _load().kvo_rope(_p(x, P_f64), x.shape[0], int(pos), float(theta_base), _p(out, P_f64))
    return out


def affine_from_range(lo: float, hi: float):
    s, z = ctypes.c_float(), ctypes.c_float()
    _load().kvo_affine_from_range(float(lo), float(hi), ctypes.byref(s), ctypes.byref(z))
    return s.value, z.value


def enc(y: float, s: float, z: float, cb) -> int:
    cb = _f32(cb)
    return _load().kvo_enc(float(y), float(s), float(z), _p(cb, P_f32), cb.shape[0])


def outlier_count(D: int, ppm: int) -> int:
    return _load().kvo_outlier_count(int(D), int(ppm))


def select_outliers(v, k: int) -> np.ndarray:
    v = _f16bits(v)
    mask = np.zeros(v.shape[0], dtype=np.uint8)
    _load().kvo_select_outliers(_p(v, P_u16), v.shape[0], int(k), _p(mask, P_u8))
    return mask.astype(bool)


def quantize_key(x, lo, hi, cb):
    x = _f16bits(x)
    lo, hi, cb = _f32(lo), _f32(hi), _f32(cb)
    D = x.shape[0]
    codes = np.zeros(D, dtype=np.uint16)
    idx = np.zeros(D, dtype=np.int32)
    val = np.zeros(D, dtype=np.uint16)
    n = _load().kvo_quantize_key(_p(x, P_u16), D, _p(lo, P_f32), _p(hi, P_f32), _p(cb, P_f32),
                                 cb.shape[0], _p(codes, P_u16), _p(idx, P_i32), _p(val, P_u16))
    return codes, idx[:n].copy(), val[:n].copy()


def quantize_value(v, ppm: int, cb, identity_affine: bool = False):
    v = _f16bits(v)
    cb = _f32(cb)
    D = v.shape[0]
    k = outlier_count(D, ppm)
    codes = np.zeros(D, dtype=np.uint16)
    idx = np.zeros(max(k, 1), dtype=np.int32)
    val = np.zeros(max(k, 1), dtype=np.uint16)
    s, z = ctypes.c_float(), ctypes.c_float()
    n = _load().kvo_quantize_value(_p(v, P_u16), D, int(ppm), _p(cb, P_f32), cb.shape[0],
                                   int(bool(identity_affine)), _p(codes, P_u16), _p(idx, P_i32),
                                   _p(val, P_u16), ctypes.byref(s), ctypes.byref(z))
    return codes, idx[:n].copy(), val[:n].copy(), s.value, z.value


# ------------------------------------------------------------------------- cache ---
@dataclass
class CanonCache:
    """Canonical quantized cache (one layer)."""
    kcodes: np.ndarray
    kptr: np.ndarray
    kidx: np.ndarray
    kval: np.ndarray
    vcodes: np.ndarray
    vidx: np.ndarray
    vval: np.ndarray
    vs: np.ndarray
    vz: np.ndarray

    @property
    def T(self) -> int:
        return int(self.kcodes.shape[0])


def prefill(K, V, key_lo, key_hi, cbK, cbV, ppm: int, value_identity_affine: bool = False,
            kcap: int | None = None) -> CanonCache:
    """Quantize T tokens as T successive appends (oracle step 5)."""
    K = _f16bits(K)
    V = _f16bits(V)
    T, D = K.shape
    assert V.shape == (T, D)
    cbK, cbV = _f32(cbK), _f32(cbV)
    assert cbK.shape == cbV.shape
    key_lo, key_hi = _f32(key_lo), _f32(key_hi)
    k = outlier_count(D, ppm)
    if kcap is None:
        kcap = T * D
    kcodes = np.zeros((T, D), dtype=np.uint16)
    vcodes = np.zeros((T, D), dtype=np.uint16)
    kptr = np.zeros(T + 1, dtype=np.int64)
    kidx = np.zeros(max(kcap, 1), dtype=np.int32)
    kval = np.zeros(max(kcap, 1), dtype=np.uint16)
    vidx = np.zeros((T, max(k, 1)), dtype=np.int32)
    vval = np.zeros((T, max(k, 1)), dtype=np.uint16)
    vs = np.zeros(T, dtype=np.float32)
    vz = np.zeros(T, dtype=np.float32)
    if k == 0:
        vidx_c = np.zeros(max(T, 1), dtype=np.int32)
        vval_c = np.zeros(max(T, 1), dtype=np.uint16)
    else:
        vidx_c, vval_c = vidx, vval
    nnz = _load().kvo_prefill(T, D, _p(K, P_u16), _p(V, P_u16), _p(key_lo, P_f32),
                              _p(key_hi, P_f32), _p(cbK, P_f32), _p(cbV, P_f32), cbK.shape[0],
                              int(ppm), int(bool(value_identity_affine)), _p(kcodes, P_u16),
                              _p(kptr, P_i64), _p(kidx, P_i32), _p(kval, P_u16), int(kcap),
                              _p(vcodes, P_u16), _p(vidx_c, P_i32), _p(vval_c, P_u16),
                              _p(vs, P_f32), _p(vz, P_f32))
    if nnz < 0:
        raise OverflowError("key outlier capacity exceeded")
    return CanonCache(kcodes, kptr, kidx[:nnz].copy(), kval[:nnz].copy(), vcodes,
                      vidx[:, :k].copy(), vval[:, :k].copy(), vs, vz)


def attend_partial(cache: CanonCache, q, pos: int, *, H_q: int, H_kv: int, d: int,
                   key_lo, key_hi, cbK_dec, cbV_dec, pos_base: int = 0,
                   theta_base: float = 10000.0, nthreads: int = 0) -> np.ndarray:
    """Partials [H_q, d+2] = (sum p V^, m, l) over the cache's tokens (oracle step 8)."""
    q = _f16bits(np.asarray(q).reshape(H_q, d))
    T = cache.T
    D = H_kv * d
    kper = int(cache.vidx.shape[1]) if cache.vidx.ndim == 2 else 0
    parts = np.zeros((H_q, d + 2), dtype=np.float64)
    kcodes = np.ascontiguousarray(cache.kcodes, dtype=np.uint16).reshape(T, D) if T else np.zeros((1, D), np.uint16)
    vcodes = np.ascontiguousarray(cache.vcodes, dtype=np.uint16).reshape(T, D) if T else np.zeros((1, D), np.uint16)
    kidx = np.ascontiguousarray(cache.kidx, dtype=np.int32) if cache.kidx.size else np.zeros(1, np.int32)
    kval = np.ascontiguousarray(cache.kval, dtype=np.uint16) if cache.kval.size else np.zeros(1, np.uint16)
    vidx = np.ascontiguousarray(cache.vidx, dtype=np.int32) if cache.vidx.size else np.zeros(1, np.int32)
    vval = np.ascontiguousarray(cache.vval, dtype=np.uint16) if cache.vval.size else np.zeros(1, np.uint16)
    kptr = np.ascontiguousarray(cache.kptr, dtype=np.int64)
    vs = _f32(cache.vs) if T else np.zeros(1, np.float32)
    vz = _f32(cache.vz) if T else np.zeros(1, np.float32)
    key_lo, key_hi = _f32(key_lo), _f32(key_hi)
    cbK_dec, cbV_dec = _f32(cbK_dec), _f32(cbV_dec)
    _load().kvo_attend(T, H_q, H_kv, d, _p(kcodes, P_u16), _p(kptr, P_i64), _p(kidx, P_i32),
                       _p(kval, P_u16), _p(vcodes, P_u16), kper, _p(vidx, P_i32), _p(vval, P_u16),
                       _p(vs, P_f32), _p(vz, P_f32), _p(key_lo, P_f32), _p(key_hi, P_f32),
                       _p(cbK_dec, P_f32), _p(cbV_dec, P_f32), _p(q, P_u16), int(pos),
                       int(pos_base), float(theta_base), _p(parts, P_f64), int(nthreads))
    return parts


def merge(parts) -> np.ndarray:
    """Log-sum-exp merge of partials [P, H, d+2] -> o [H, d] (oracle step 9)."""
    parts = np.ascontiguousarray(np.asarray(parts, dtype=np.float64))
    P, H, d2 = parts.shape
    d = d2 - 2
    o = np.zeros((H, d), dtype=np.float64)
    _load().kvo_merge(P, H, d, _p(parts, P_f64), _p(o, P_f64))
    return o


def attend(cache: CanonCache, q, pos: int, **kw) -> np.ndarray:
    """o [H_q, d] = merged single partial."""
    return merge(attend_partial(cache, q, pos, **kw)[None])


# --------------------------------------------- online per-channel Key thresholds (f2) ---
def key_thresholds_online(K, ppm: int):
    """Per-channel (lo, hi) fp32 from the Keys of a prefill block [T, D] ("Online for K",
    P:1036-1064): order statistics floor(n/2) and T-1-ceil(n/2), n = ceil(ppm T / 1e6)."""
    Kb = _f16bits(K)
    T, D = Kb.shape
    lo = np.zeros(D, np.float32)
    hi = np.zeros(D, np.float32)
    rc = _load().kvo_key_thresholds_online(T, D, _p(Kb, P_u16), int(ppm), _p(lo, P_f32), _p(hi, P_f32))
    if rc != 0:
        raise ValueError("too many outliers for the block")
    return lo, hi


# ------------------------------------------------------ fp16 comparator cache (F16) ---
def f64_to_f16(x: float) -> int:
    """IEEE binary16 bits of x, round to nearest even (one rounding)."""
    return int(_load().kvo_f64_to_f16(float(x)))


def f16cache_keys(K, H: int, d: int, pos_base: int = 0, theta_base: float = 10000.0) -> np.ndarray:
    """Stored Keys of the fp16 cache: fp16(RoPE(K_n, pos_base + n)) per head, [T, H d] bits."""
    Kb = _f16bits(K)
    T = Kb.shape[0]
    out = np.zeros_like(Kb)
    lib = _load()
    for n in range(T):
        row = np.ascontiguousarray(Kb[n])
        o = np.zeros_like(row)
        lib.kvo_f16cache_key(_p(row, P_u16), H, d, int(pos_base + n), float(theta_base), _p(o, P_u16))
        out[n] = o
    return out


def attend_dense(Kpost, V, q, pos: int, *, H_q: int, H_kv: int, d: int,
                 theta_base: float = 10000.0) -> np.ndarray:
    """o [H_q, d] of textbook attention over dense post-RoPE fp16 Keys (kvo_attend_dense)."""
    Kb, Vb = _f16bits(Kpost), _f16bits(V)
    qb = _f16bits(np.asarray(q).reshape(H_q, d))
    T = Kb.shape[0]
    o = np.zeros((H_q, d), np.float64)
    _load().kvo_attend_dense(T, H_q, H_kv, d, _p(Kb, P_u16), _p(Vb, P_u16), _p(qb, P_u16), int(pos),
                             float(theta_base), _p(o, P_f64))
    return o


def pack(codes, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(np.asarray(codes, dtype=np.uint16))
    n = codes.shape[0]
    words = np.zeros(max((n * bits + 31) // 32, 1), dtype=np.uint32)
    _load().kvo_pack(_p(codes, P_u16), n, int(bits), _p(words, P_u32))
    return words[: (n * bits + 31) // 32]


def unpack(words, n: int, bits: int) -> np.ndarray:
    words = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    if words.size == 0:
        words = np.zeros(1, np.uint32)
    codes = np.zeros(max(n, 1), dtype=np.uint16)
    _load().kvo_unpack(_p(words, P_u32), int(n), int(bits), _p(codes, P_u16))
    return codes[:n]


# ------------------------------------------ mixed-precision sensitivity (f4) -----------
def dequantize(cache: CanonCache, key_lo, key_hi, cbK_dec, cbV_dec):
    """K^, V^ [T, D] fp64 of a canonical cache, the plain definition the attend uses
    (readings R5, R6): an outlier entry is its stored fp16 value, every other
    entry Chat_dec[code] * s + z with s_c, z_c = fp32((hi-lo)/2), fp32((hi+lo)/2) for the
    Keys (per channel) and the stored fp32 (s_n, z_n) for the Values (per token)."""
    T, D = cache.kcodes.shape
    lo = np.asarray(key_lo, np.float32).astype(np.float64)
    hi = np.asarray(key_hi, np.float32).astype(np.float64)
    s = ((hi - lo) / 2.0).astype(np.float32).astype(np.float64)
    z = ((hi + lo) / 2.0).astype(np.float32).astype(np.float64)
    cK = np.asarray(cbK_dec, np.float32).astype(np.float64)
    cV = np.asarray(cbV_dec, np.float32).astype(np.float64)
    Kh = cK[cache.kcodes.astype(np.int64)] * s[None, :] + z[None, :]
    Vh = (cV[cache.vcodes.astype(np.int64)] * cache.vs.astype(np.float64)[:, None]
          + cache.vz.astype(np.float64)[:, None])
    for n in range(T):
        a, b = int(cache.kptr[n]), int(cache.kptr[n + 1])
        Kh[n, cache.kidx[a:b]] = cache.kval[a:b].view(np.float16).astype(np.float64)
        if cache.vidx.shape[1]:
            Vh[n, cache.vidx[n]] = cache.vval[n].view(np.float16).astype(np.float64)
    return Kh, Vh


def fisher_diag(grads) -> np.ndarray:
    """Diagonal Fisher information F^D = diag(g (.) g) summed over samples (SPEC
    fisher_diag: sum, not mean), fp64."""
    gs = [np.asarray(g, np.float64) for g in grads]
    if not gs:
        raise ValueError("no gradient samples")
    F = np.zeros_like(gs[0])
    for g in gs:
        if g.shape != F.shape:
            raise ValueError("gradient shapes differ")
        F = F + g * g
    return F


def layer_sensitivity(a, qa, f=None) -> float:
    """Omega = (A - Q(A))^T F^D (A - Q(A)) = sum F (A - Q(A))^2 (eq:opt2), fp64;
    f = None means F = 1 (the plain quantization error)."""
    a = np.asarray(a, np.float64)
    qa = np.asarray(qa, np.float64)
    if a.shape != qa.shape:
        raise ValueError("shape mismatch")
    e = a - qa
    if f is None:
        return float(np.sum(e * e))
    f = np.asarray(f, np.float64)
    if f.shape != a.shape:
        raise ValueError("shape mismatch")
    return float(np.sum(f * e * e))


def layer_omega(K, V, key_lo, key_hi, cbK, cbV, ppm: int, FK=None, FV=None, cbK_dec=None, cbV_dec=None):
    """(Omega_K, Omega_V) of one layer quantized with the given (lower-precision) codebooks and
    thresholds ("quantization error computed at the lower precision"; reading R26):
    prefill -> dequantize -> layer_sensitivity on the Keys and on the Values."""
    cbK_dec = cbK if cbK_dec is None else cbK_dec
    cbV_dec = cbV if cbV_dec is None else cbV_dec
    cache = prefill(K, V, key_lo, key_hi, cbK, cbV, ppm)
    Kh, Vh = dequantize(cache, key_lo, key_hi, cbK_dec, cbV_dec)
    Kf = _f16bits(K).view(np.float16).astype(np.float64)
    Vf = _f16bits(V).view(np.float16).astype(np.float64)
    return layer_sensitivity(Kf, Kh, FK), layer_sensitivity(Vf, Vh, FV)


def assign_mixed_precision(omegas, demote_count: int) -> list:
    """The demote_count layer ids with the smallest Omega, which get the lower bit width
    (one-shot assignment); ties to the lower layer id (SPEC
    assign_mixed_precision).  Plain selection: repeatedly take the smallest remaining."""
    om = [float(x) for x in omegas]
    if not 0 <= demote_count <= len(om):
        raise ValueError("demote_count out of range")
    left = list(range(len(om)))
    out = []
    for _ in range(demote_count):
        best = left[0]
        for i in left:
            if om[i] < om[best]:
                best = i
        out.append(best)
        left.remove(best)
    return sorted(out)


# --------------------------------------------- offline calibration on the GPU (f3) ------
# The readings these follow (R27, R28): normalized points of the kept values only
# ("the remaining numbers in the vector are normalized to the range [-1,1]"), Lloyd
# k-means for eq:fisher_kmeans with per-element Fisher weights on the normalized
# residual, centroids initialised at the k equal-width bin centres of [-1, 1], nearest
# centroid with ties to the lower index, empty clusters keep their centroid, stop when the
# largest move < tol or after max_iter updates; Q-Norm (eq:qnorm P:355-358) statistics over the
# same normalized points (unweighted, population std), post-quantization values from the
# encode codebook the cache will use.
def calib_key_points(Kcal, key_lo, key_hi, FK=None):
    """Normalized kept Key values and their weights, token-major order.  A value is kept when
    lo_c <= x <= hi_c (R4) and hi_c > lo_c; x' = (x - z_c) / s_c with s_c = (hi_c - lo_c)/2,
    z_c = (hi_c + lo_c)/2 in fp64."""
    K = _f16bits(Kcal).view(np.float16).astype(np.float64)
    lo = np.asarray(key_lo, np.float32).astype(np.float64)[None, :]
    hi = np.asarray(key_hi, np.float32).astype(np.float64)[None, :]
    s = (hi - lo) / 2.0
    z = (hi + lo) / 2.0
    kept = (K >= lo) & (K <= hi) & (hi > lo)
    xn = (K - z) / np.where(hi > lo, s, 1.0)
    w = np.ones_like(K) if FK is None else np.asarray(FK, np.float32).astype(np.float64)
    return xn[kept], w[kept]


def calib_value_points(Vcal, ppm: int, FV=None):
    """Normalized kept Value values per token: the k = ceil(f D) outliers of the two-sided
    split (R2, R3; the pinned select_outliers) removed, [lo_n, hi_n] the kept range, x' =
    (v - z_n) / s_n in fp64; tokens with hi_n == lo_n contribute nothing."""
    Vb = _f16bits(Vcal)
    N, D = Vb.shape
    k = outlier_count(D, ppm)
    V = Vb.view(np.float16).astype(np.float64)
    W = np.ones_like(V) if FV is None else np.asarray(FV, np.float32).astype(np.float64)
    xs, ws = [], []
    for n in range(N):
        kept = ~select_outliers(Vb[n], k)
        lo, hi = V[n, kept].min(), V[n, kept].max()
        if hi > lo:
            s, z = (hi - lo) / 2.0, (hi + lo) / 2.0
            xs.append((V[n, kept] - z) / s)
            ws.append(W[n, kept])
    if not xs:
        return np.zeros(0), np.zeros(0)
    return np.concatenate(xs), np.concatenate(ws)


def nearest_label(x, cb) -> np.ndarray:
    """Index of the nearest centroid, ties to the lower index: #{j : 2x > c_j + c_{j+1}}."""
    x = np.asarray(x, np.float64)
    c = np.asarray(cb, np.float64)
    lab = np.zeros(x.shape, np.int64)
    for j in range(c.size - 1):
        lab += (2.0 * x > c[j] + c[j + 1])
    return lab


def fisher_kmeans(x, w, k: int, max_iter: int = 100, tol: float = 1e-6):
    """Weighted Lloyd k-means in 1-D for eq:fisher_kmeans: returns (centroids
    ascending fp64, number of updates run)."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    c = -1.0 + (2.0 * np.arange(k) + 1.0) / k
    it = 0
    for it in range(1, max_iter + 1):
        lab = nearest_label(x, c)
        sw = np.bincount(lab, weights=w, minlength=k)          # sum of w per cluster
        sx = np.bincount(lab, weights=w * x, minlength=k)      # sum of w x per cluster
        new = np.where(sw > 0, sx / np.where(sw > 0, sw, 1.0), c)
        new = np.sort(new)
        move = np.max(np.abs(new - c))
        c = new
        if move < tol:
            break
    return c, it


def qnorm_stats(x, cb):
    """(mu1, sigma1, mu2, sigma2): mean / population std of the points and of their nearest
    codebook values (eq:qnorm P:355-358)."""
    x = np.asarray(x, np.float64)
    q = np.asarray(cb, np.float64)[nearest_label(x, cb)]
    return x.mean(), x.std(), q.mean(), q.std()


def apply_qnorm(cb, mu1, sigma1, mu2, sigma2) -> np.ndarray:
    """eq:qnorm: C^_i = (C_i - mu2) sigma1 / sigma2 + mu1."""
    c = np.asarray(cb, np.float64)
    return (c - mu2) * sigma1 / sigma2 + mu1


def _codebook_store(c, fp16: bool) -> np.ndarray:
    """fp32 (or fp16-valued, R23) storage of an ascending codebook, one rounding per entry;
    an entry that would not exceed its predecessor is bumped to the next representable value."""
    out = np.zeros(len(c), np.float32)
    for i, v in enumerate(np.asarray(c, np.float64)):
        r = np.float32(np.array([f64_to_f16(v)], np.uint16).view(np.float16)[0]) if fp16 else np.float32(v)
        if i and r <= out[i - 1]:
            if fp16:
                r = np.float32(np.nextafter(np.float16(out[i - 1]), np.float16(np.inf)))
            else:
                r = np.nextafter(out[i - 1], np.float32(np.inf))
        out[i] = r
    return out


def calibrate_layer(Kcal, Vcal, bits: int, ppm: int, FK=None, FV=None, max_iter: int = 100,
                    tol: float = 1e-6, qnorm: bool = False, fp16_codebooks: bool = True) -> dict:
    """Offline calibration of one layer: per-channel Key
    thresholds over the calibration tokens (the order statistics of key_thresholds_online),
    Key / Value codebooks by Fisher-weighted k-means on the normalized kept values, optional
    Q-Norm'd decode codebooks."""
    lo, hi = key_thresholds_online(Kcal, ppm)
    k = 1 << bits
    xk, wk = calib_key_points(Kcal, lo, hi, FK)
    xv, wv = calib_value_points(Vcal, ppm, FV)
    ck, itk = fisher_kmeans(xk, wk, k, max_iter, tol)
    cv, itv = fisher_kmeans(xv, wv, k, max_iter, tol)
    cbK, cbV = _codebook_store(ck, fp16_codebooks), _codebook_store(cv, fp16_codebooks)
    out = dict(key_lo=lo, key_hi=hi, cbK=cbK, cbV=cbV, cbK_dec=cbK.copy(), cbV_dec=cbV.copy(),
               iters=(itk, itv), centroids=(ck, cv))
    if qnorm:
        for key, x, cb in (("cbK_dec", xk, cbK), ("cbV_dec", xv, cbV)):
            if x.size == 0:
                continue                       # no points: decode = encode
            st = qnorm_stats(x, cb)
            if st[3] > 0:                      # sigma2 = 0 (one level used): decode = encode
                out[key] = _codebook_store(apply_qnorm(cb, *st), fp16_codebooks)
    return out
