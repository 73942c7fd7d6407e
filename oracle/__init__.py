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
