"""Thin Python binding of libkvq (ctypes).  Argument marshalling only.

Every call goes to the C ABI declared in include/kvq.h; every step of the hot path runs
in the sm_100a kernels of libkvq.so.  There is no CPU fallback: if the shared library
is missing or fails to load, importing the binding raises.

Buffers may be torch CUDA tensors (device pointers on the cache's device), torch CPU
tensors or numpy arrays (host memory: the library stages them on the call's stream).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvq.so")

KVQ_OK, KVQ_EINVAL, KVQ_ESHAPE, KVQ_EEMPTY, KVQ_ECAPACITY, KVQ_EDEVICE, KVQ_ECUDA = range(7)
_STATUS = {0: "KVQ_OK", 1: "KVQ_EINVAL", 2: "KVQ_ESHAPE", 3: "KVQ_EEMPTY",
           4: "KVQ_ECAPACITY", 5: "KVQ_EDEVICE", 6: "KVQ_ECUDA"}
KVQ_FLAG_TRUST_DEVICE_PTRS = 1
KVQ_FLAG_DECODE_PDL = 2

# Every symbol include/kvq.h declares (checked by tests/test_abi.py).
EXPORTED = ["kvq_cache_create", "kvq_cache_destroy", "kvq_append", "kvq_prefill_quantize",
            "kvq_decode_attend", "kvq_decode_attend_partial", "kvq_merge_partials",
            "kvq_num_tokens", "kvq_reset", "kvq_sync", "kvq_key_outlier_span", "kvq_export",
            "kvq_get_info", "kvq_set_splits", "kvq_phase_timers", "kvq_last_error", "kvq_version",
            "kvq_f16_cache_create", "kvq_f16_cache_destroy", "kvq_f16_append",
            "kvq_f16_decode_attend", "kvq_f16_export", "kvq_f16_num_tokens",
            "kvq_key_thresholds_online", "kvq_decode_attend_batch", "kvq_layer_sensitivity",
            "kvq_fisher_accumulate", "kvq_assign_bits", "kvq_calibrate_layer",
            "kvq_decode_attend_batch_partial", "kvq_set_pos_base", "kvq_snapshot_bytes", "kvq_snapshot",
            "kvq_restore"]


class KVQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class kvq_calib_config(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("outlier_ppm", ctypes.c_int32), ("max_iter", ctypes.c_int32),
                ("qnorm", ctypes.c_int32), ("fp16_codebooks", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("tol", ctypes.c_double)]


class kvq_config(ctypes.Structure):
    _fields_ = [("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("outlier_ppm", ctypes.c_int32), ("capacity_tokens", ctypes.c_int64),
                ("k_outlier_capacity", ctypes.c_int64), ("pos_base", ctypes.c_int64),
                ("rope_theta", ctypes.c_double), ("device", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


_PF = ctypes.POINTER(ctypes.c_float)


class kvq_params(ctypes.Structure):
    _fields_ = [("key_cb_enc", _PF), ("key_cb_dec", _PF), ("val_cb_enc", _PF),
                ("val_cb_dec", _PF), ("key_lo", _PF), ("key_hi", _PF)]


class kvq_export_buf(ctypes.Structure):
    _fields_ = [("kcodes", ctypes.c_void_p), ("kptr", ctypes.c_void_p), ("kidx", ctypes.c_void_p),
                ("kval", ctypes.c_void_p), ("vcodes", ctypes.c_void_p), ("vidx", ctypes.c_void_p),
                ("vval", ctypes.c_void_p), ("vs", ctypes.c_void_p), ("vz", ctypes.c_void_p)]


class kvq_info(ctypes.Structure):
    _fields_ = [("heads_per_cta", ctypes.c_int32), ("splits", ctypes.c_int32),
                ("value_outliers", ctypes.c_int32), ("words_per_token", ctypes.c_int32),
                ("capacity_tokens", ctypes.c_int64), ("k_outlier_capacity", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("attend_kernel", ctypes.c_int32),
                ("bucket_heads", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libkvq.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "kvq_cache_create": (i32, [ctypes.POINTER(kvq_config), ctypes.POINTER(kvq_params), ctypes.POINTER(vp)]),
        "kvq_cache_destroy": (None, [vp]),
        "kvq_append": (i32, [vp, vp, vp, vp]),
        "kvq_prefill_quantize": (i32, [vp, vp, vp, i64, vp]),
        "kvq_decode_attend": (i32, [vp, vp, i64, vp, vp]),
        "kvq_decode_attend_partial": (i32, [vp, vp, i64, vp, vp]),
        "kvq_merge_partials": (i32, [vp, i32, i32, i32, vp, i32, vp]),
        "kvq_num_tokens": (i64, [vp]),
        "kvq_reset": (i32, [vp, vp]),
        "kvq_sync": (i32, [vp]),
        "kvq_key_outlier_span": (i32, [vp, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "kvq_export": (i32, [vp, i64, i64, ctypes.POINTER(kvq_export_buf)]),
        "kvq_get_info": (i32, [vp, ctypes.POINTER(kvq_info)]),
        "kvq_set_splits": (i32, [vp, i32]),
        "kvq_phase_timers": (i32, [vp, ctypes.POINTER(ctypes.c_uint64)]),
        "kvq_last_error": (ctypes.c_char_p, []),
        "kvq_f16_cache_create": (i32, [ctypes.POINTER(kvq_config), ctypes.POINTER(vp)]),
        "kvq_f16_cache_destroy": (None, [vp]),
        "kvq_f16_append": (i32, [vp, vp, vp, i64, vp]),
        "kvq_f16_decode_attend": (i32, [vp, vp, i64, vp, vp]),
        "kvq_f16_export": (i32, [vp, i64, i64, vp, vp]),
        "kvq_f16_num_tokens": (i64, [vp]),
        "kvq_key_thresholds_online": (i32, [vp, i64, i32, i32, vp, vp, i32, vp]),
        "kvq_decode_attend_batch": (i32, [vp, i32, vp, vp, vp, vp]),
        "kvq_decode_attend_batch_partial": (i32, [vp, i32, vp, vp, vp, vp]),
        "kvq_set_pos_base": (i32, [vp, i64]),
        "kvq_snapshot_bytes": (i32, [vp, ctypes.POINTER(ctypes.c_int64)]),
        "kvq_snapshot": (i32, [vp, vp, i64]),
        "kvq_restore": (i32, [vp, vp, i64]),
        "kvq_layer_sensitivity": (i32, [vp, vp, vp, vp, vp, i64, i64, vp, vp]),
        "kvq_fisher_accumulate": (i32, [vp, vp, i64, i32, vp]),
        "kvq_assign_bits": (i32, [vp, i32, i32, i32, i32, vp]),
        "kvq_calibrate_layer": (i32, [vp, vp, vp, vp, i64, i32, ctypes.POINTER(kvq_calib_config), vp, vp, vp, vp,
                                      vp, vp, vp, i32, vp]),
        "kvq_version": (i32, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int):
    if status != KVQ_OK:
        raise KVQError(status, _lib.kvq_last_error().decode(errors="replace"))


def _ptr(x):
    """Raw pointer of a torch tensor (device or host) or numpy array (host)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(x)}")


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def version() -> int:
    return _lib.kvq_version()


class KVQCache:
    """One layer's compressed KV cache (wraps a kvq_cache handle)."""

    def __init__(self, *, n_q_heads: int, n_kv_heads: int, head_dim: int = 128, bits: int,
                 outlier_ppm: int, capacity_tokens: int, key_cb, val_cb, key_lo, key_hi,
                 key_cb_dec=None, val_cb_dec=None, k_outlier_capacity: int = 0,
                 pos_base: int = 0, rope_theta: float = 10000.0, device: int = 0,
                 trust_device_ptrs: bool = False, decode_pdl: bool = False):
        """decode_pdl: opt in to KVQ_FLAG_DECODE_PDL (kvq.h): the caller guarantees q is
        complete before each append that precedes an attend on the same stream."""
        flags = (KVQ_FLAG_TRUST_DEVICE_PTRS if trust_device_ptrs else 0) | (KVQ_FLAG_DECODE_PDL if decode_pdl else 0)
        cfg = kvq_config(n_q_heads, n_kv_heads, head_dim, bits, outlier_ppm, capacity_tokens,
                         k_outlier_capacity, pos_base, rope_theta, device, flags)
        keep = [_f32(key_cb), None if key_cb_dec is None else _f32(key_cb_dec), _f32(val_cb),
                None if val_cb_dec is None else _f32(val_cb_dec), _f32(key_lo), _f32(key_hi)]

        def fp(a):
            return None if a is None else a.ctypes.data_as(_PF)

        prm = kvq_params(*[fp(a) for a in keep])
        h = ctypes.c_void_p()
        _check(_lib.kvq_cache_create(ctypes.byref(cfg), ctypes.byref(prm), ctypes.byref(h)))
        self._h = h
        self.cfg = cfg
        self.D = n_kv_heads * head_dim
        self.H_q, self.H_kv, self.d, self.bits = n_q_heads, n_kv_heads, head_dim, bits

    # -- lifecycle -------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.kvq_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- hot path --------------------------------------------------------------------
    def append(self, k, v, stream=None):
        _check(_lib.kvq_append(self._h, _ptr(k), _ptr(v), _stream(stream)))

    def prefill(self, K, V, stream=None):
        T = int(K.shape[0])
        _check(_lib.kvq_prefill_quantize(self._h, _ptr(K), _ptr(V), T, _stream(stream)))

    def attend(self, q, pos: int, out, stream=None):
        _check(_lib.kvq_decode_attend(self._h, _ptr(q), int(pos), _ptr(out), _stream(stream)))
        return out

    def attend_partial(self, q, pos: int, out, stream=None):
        _check(_lib.kvq_decode_attend_partial(self._h, _ptr(q), int(pos), _ptr(out), _stream(stream)))
        return out

    # -- utilities -------------------------------------------------------------------
    @property
    def num_tokens(self) -> int:
        return int(_lib.kvq_num_tokens(self._h))

    def reset(self, stream=None):
        _check(_lib.kvq_reset(self._h, _stream(stream)))

    def snapshot(self) -> np.ndarray:
        """The cache contents as a host byte array (kvq_snapshot; synchronizes)."""
        n = ctypes.c_int64()
        _check(_lib.kvq_snapshot_bytes(self._h, ctypes.byref(n)))
        buf = np.empty(n.value, np.uint8)
        _check(_lib.kvq_snapshot(self._h, buf.ctypes.data, n.value))
        return buf

    def restore(self, buf: np.ndarray):
        """Replace the contents with a snapshot of a cache of the same configuration."""
        buf = np.ascontiguousarray(buf, np.uint8)
        _check(_lib.kvq_restore(self._h, buf.ctypes.data, buf.size))

    def set_pos_base(self, pos_base: int):
        """Reposition an EMPTY cache (token t -> position pos_base + t), kvq_set_pos_base."""
        _check(_lib.kvq_set_pos_base(self._h, int(pos_base)))

    def sync(self):
        _check(_lib.kvq_sync(self._h))

    def set_splits(self, splits: int):
        _check(_lib.kvq_set_splits(self._h, int(splits)))

    def phase_timers(self) -> list:
        out = (ctypes.c_uint64 * 16)()
        _check(_lib.kvq_phase_timers(self._h, out))
        return list(out)

    def info(self) -> dict:
        inf = kvq_info()
        _check(_lib.kvq_get_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in kvq_info._fields_}

    def key_outlier_span(self, t0: int, t1: int):
        b, e = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.kvq_key_outlier_span(self._h, t0, t1, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def export(self, t0: int = 0, t1: Optional[int] = None) -> dict:
        """Canonical cache contents of tokens [t0, t1) as numpy arrays."""
        if t1 is None:
            t1 = self.num_tokens
        n = t1 - t0
        kb, ke = self.key_outlier_span(t0, t1)
        kv = self.info()["value_outliers"]
        out = dict(kcodes=np.zeros((n, self.D), np.uint8), vcodes=np.zeros((n, self.D), np.uint8),
                   kptr=np.zeros(n + 1, np.int64), kidx=np.zeros(max(ke - kb, 1), np.uint16),
                   kval=np.zeros(max(ke - kb, 1), np.uint16), vidx=np.zeros((n, max(kv, 1)), np.uint16),
                   vval=np.zeros((n, max(kv, 1)), np.uint16), vs=np.zeros(n, np.float32),
                   vz=np.zeros(n, np.float32))
        buf = kvq_export_buf(*[out[k].ctypes.data for k in
                               ("kcodes", "kptr", "kidx", "kval", "vcodes", "vidx", "vval", "vs", "vz")])
        _check(_lib.kvq_export(self._h, t0, t1, ctypes.byref(buf)))
        out["kidx"] = out["kidx"][: ke - kb]
        out["kval"] = out["kval"][: ke - kb]
        out["vidx"] = out["vidx"][:, :kv]
        out["vval"] = out["vval"][:, :kv]
        return out


def attend_batch(caches, qs, positions, outs, stream=None):
    """Batched decode (kvq_decode_attend_batch): caches[i] attends qs[i] at positions[i] into
    outs[i] (device tensors), one launch when the caches share a configuration."""
    B = len(caches)
    hs = (ctypes.c_void_p * B)(*[c.handle.value for c in caches])
    qp = (ctypes.c_void_p * B)(*[_ptr(q).value for q in qs])
    op = (ctypes.c_void_p * B)(*[_ptr(o).value for o in outs])
    pp = (ctypes.c_int64 * B)(*[int(p) for p in positions])
    _check(_lib.kvq_decode_attend_batch(ctypes.cast(hs, ctypes.c_void_p), B, ctypes.cast(qp, ctypes.c_void_p),
                                        ctypes.cast(pp, ctypes.c_void_p), ctypes.cast(op, ctypes.c_void_p),
                                        _stream(stream)))
    return outs


def attend_batch_partial(caches, qs, positions, parts, stream=None):
    """Batched partials (kvq_decode_attend_batch_partial): caches[i] attends qs[i] at
    positions[i] into parts[i] ([H_q, d+2] fp32 device tensors), one launch when the caches share
    a configuration."""
    B = len(caches)
    hs = (ctypes.c_void_p * B)(*[c.handle.value for c in caches])
    qp = (ctypes.c_void_p * B)(*[_ptr(q).value for q in qs])
    op = (ctypes.c_void_p * B)(*[_ptr(o).value for o in parts])
    pp = (ctypes.c_int64 * B)(*[int(p) for p in positions])
    _check(_lib.kvq_decode_attend_batch_partial(ctypes.cast(hs, ctypes.c_void_p), B, ctypes.cast(qp, ctypes.c_void_p),
                                                ctypes.cast(pp, ctypes.c_void_p), ctypes.cast(op, ctypes.c_void_p),
                                                _stream(stream)))
    return parts


def key_thresholds_online(K, outlier_ppm: int, lo=None, hi=None, device: int = 0, stream=None):
    """Per-channel Key (lo, hi) from a prefill block K [T, D] fp16 on the GPU.
    Outputs default to host numpy arrays (the call then synchronizes)."""
    T, D = (int(x) for x in K.shape)
    if lo is None:
        lo = np.zeros(D, np.float32)
    if hi is None:
        hi = np.zeros(D, np.float32)
    _check(_lib.kvq_key_thresholds_online(_ptr(K), T, D, int(outlier_ppm), _ptr(lo), _ptr(hi), int(device),
                                          _stream(stream)))
    return lo, hi


def calibrate_layer(K, V, bits: int, outlier_ppm: int, FK=None, FV=None, max_iter: int = 100, tol: float = 1e-6,
                    qnorm: bool = False, fp16_codebooks: bool = True, device: int = 0, stream=None) -> dict:
    """Offline calibration of one layer on the GPU (kvq_calibrate_layer): Key
    thresholds and the four codebooks for KVQCache, from calibration K, V [N, D] fp16 (device or
    host) and optional fp32 Fisher diagonals.  Returns host numpy arrays (synchronizes)."""
    N, D = (int(x) for x in K.shape)
    k = 1 << int(bits)
    cfg = kvq_calib_config(int(bits), int(outlier_ppm), int(max_iter), int(bool(qnorm)), int(bool(fp16_codebooks)),
                           0, float(tol))
    out = dict(key_lo=np.zeros(D, np.float32), key_hi=np.zeros(D, np.float32), cbK=np.zeros(k, np.float32),
               cbK_dec=np.zeros(k, np.float32), cbV=np.zeros(k, np.float32), cbV_dec=np.zeros(k, np.float32),
               iters=np.zeros(2, np.int32))
    _check(_lib.kvq_calibrate_layer(_ptr(K), _ptr(V), _ptr(FK), _ptr(FV), N, D, ctypes.byref(cfg),
                                    _ptr(out["key_lo"]), _ptr(out["key_hi"]), _ptr(out["cbK"]), _ptr(out["cbK_dec"]),
                                    _ptr(out["cbV"]), _ptr(out["cbV_dec"]), _ptr(out["iters"]), int(device),
                                    _stream(stream)))
    return out


def layer_sensitivity(cache, K, V, FK=None, FV=None, t0: int = 0, omega=None, stream=None):
    """(Omega_K, Omega_V) of eq:opt2 over the cache's tokens [t0, t0 + len(K)).
    K, V: the [T, D] fp16 tensors that were quantized into `cache`; FK, FV: fp32 Fisher
    diagonals of the same shape or None (ones).  Returns a host numpy float64 [2] unless a
    device `omega` tensor is given (then asynchronous)."""
    T = int(K.shape[0])
    out = np.zeros(2, np.float64) if omega is None else omega
    _check(_lib.kvq_layer_sensitivity(cache.handle, _ptr(K), _ptr(V), _ptr(FK), _ptr(FV), int(t0), T, _ptr(out),
                                      _stream(stream)))
    return out


def fisher_accumulate(F, g, device: int = 0, stream=None):
    """F += g * g elementwise on the GPU (fp32 device tensors of equal size)."""
    if F.numel() != g.numel():
        raise ValueError("F and g differ in size")
    _check(_lib.kvq_fisher_accumulate(_ptr(F), _ptr(g), int(F.numel()), int(device), _stream(stream)))
    return F


def assign_bits(omega, demote_count: int, bits_high: int, bits_low: int) -> np.ndarray:
    """Per-layer bit widths: the demote_count least sensitive layers get bits_low (host)."""
    om = np.ascontiguousarray(np.asarray(omega, dtype=np.float64))
    out = np.zeros(om.shape[0], np.int32)
    _check(_lib.kvq_assign_bits(_ptr(om), int(om.shape[0]), int(demote_count), int(bits_high), int(bits_low),
                                _ptr(out)))
    return out


class F16Cache:
    """The fp16 comparator cache (kvq_f16_*): post-RoPE fp16 Keys, fp16 Values (C3's fp16 arm)."""

    def __init__(self, *, n_q_heads: int, n_kv_heads: int, head_dim: int = 128, capacity_tokens: int,
                 pos_base: int = 0, rope_theta: float = 10000.0, device: int = 0,
                 trust_device_ptrs: bool = False):
        cfg = kvq_config(n_q_heads, n_kv_heads, head_dim, 16, 0, capacity_tokens, 0, pos_base,
                         rope_theta, device, KVQ_FLAG_TRUST_DEVICE_PTRS if trust_device_ptrs else 0)
        h = ctypes.c_void_p()
        _check(_lib.kvq_f16_cache_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.D = n_kv_heads * head_dim
        self.H_q = n_q_heads

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.kvq_f16_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def append(self, K, V, stream=None):
        T = int(K.shape[0]) if K.ndim == 2 else 1
        _check(_lib.kvq_f16_append(self._h, _ptr(K), _ptr(V), T, _stream(stream)))

    def attend(self, q, pos: int, out, stream=None):
        _check(_lib.kvq_f16_decode_attend(self._h, _ptr(q), int(pos), _ptr(out), _stream(stream)))
        return out

    @property
    def num_tokens(self) -> int:
        return int(_lib.kvq_f16_num_tokens(self._h))

    def export(self, t0: int = 0, t1: Optional[int] = None):
        t1 = self.num_tokens if t1 is None else t1
        k = np.zeros((t1 - t0, self.D), np.uint16)
        v = np.zeros((t1 - t0, self.D), np.uint16)
        _check(_lib.kvq_f16_export(self._h, t0, t1, k.ctypes.data, v.ctypes.data))
        return k, v


def merge_partials(parts, out, device: int = 0, stream=None):
    """Log-sum-exp merge of [P, H_q, d+2] partials (m in log2 units) into o [H_q, d]."""
    P, H, d2 = (int(s) for s in parts.shape)
    _check(_lib.kvq_merge_partials(_ptr(parts), P, H, d2 - 2, _ptr(out), int(device), _stream(stream)))
    return out
