"""Offline calibration tooling (produces INPUTS to kvq_cache_create).

North star: "Codebook calibration (sensitivity-weighted k-means, Q-Norm) stays offline,
and its results are supplied as inputs."  This module is that offline step on
synthetic calibration tokens.  It is not on the hot path; the oracle and the CUDA
path both receive its outputs as plain numbers.

  * per-channel Key thresholds (tab:calibration P:1036-1064):
    two-sided split of each channel's calibration values with ceil(f*N_cal) outliers
    (ceil/2 largest, floor/2 smallest), lo_c/hi_c = min/max of the kept values.
  * nuqX codebook (eq:fisher_kmeans P:316-319): values normalized to [-1,1] per vector
    (P:321), pooled per layer, weighted 1-D Lloyd k-means.  The Fisher weights
    need model gradients (A7, OUT of scope), so the weights are uniform here.
    Deterministic init at weighted quantiles (2j+1)/2k; stop at max move < tol or
    max_iter; empty clusters keep their centroid (SPEC S:283-285 design decisions).
  * Q-Norm (eq:qnorm P:355-358): C^_i = (C_i - mu2) sigma1/sigma2 + mu1, per matrix,
    statistics in normalized space from one quantization pass with the raw codebook.
"""
from __future__ import annotations

import numpy as np


def two_sided_kept_range(x: np.ndarray, n_out: int, axis: int = 0):
    """min/max of the values kept after removing ceil(n/2) largest + floor(n/2) smallest."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[axis]
    ku, kl = (n_out + 1) // 2, n_out // 2
    if ku + kl >= n:
        raise ValueError("too many outliers for the calibration set")
    srt = np.sort(x, axis=axis)
    lo = np.take(srt, kl, axis=axis)
    hi = np.take(srt, n - 1 - ku, axis=axis)
    return lo, hi


def key_thresholds(Kcal, ppm: int):
    """Per-channel (lo_c, hi_c) fp32 from calibration Keys [N, D] (pre-RoPE)."""
    K = np.asarray(Kcal, dtype=np.float64)
    N = K.shape[0]
    n_out = (ppm * N + 999_999) // 1_000_000
    lo, hi = two_sided_kept_range(K, n_out, axis=0)
    return lo.astype(np.float32), hi.astype(np.float32)


def kmeans_1d(points, weights=None, k: int = 8, max_iter: int = 100, tol: float = 1e-6):
    """Weighted Lloyd k-means in 1-D; returns sorted centroids (float64)."""
    x = np.asarray(points, dtype=np.float64).ravel()
    w = np.ones_like(x) if weights is None else np.asarray(weights, dtype=np.float64).ravel()
    order = np.argsort(x, kind="stable")
    x, w = x[order], w[order]
    cw = np.cumsum(w)
    tot = cw[-1]
    qs = (2 * np.arange(k) + 1) / (2 * k) * tot
    c = x[np.minimum(np.searchsorted(cw, qs), x.size - 1)].copy()
    for _ in range(max_iter):
        mids = 0.5 * (c[:-1] + c[1:])
        lab = np.searchsorted(mids, x, side="right")
        sw = np.bincount(lab, weights=w, minlength=k)
        sx = np.bincount(lab, weights=w * x, minlength=k)
        new = np.where(sw > 0, sx / np.where(sw > 0, sw, 1), c)
        new.sort()
        move = np.max(np.abs(new - c))
        c = new
        if move < tol:
            break
    return c


def _strictly_ascending_f32(c: np.ndarray) -> np.ndarray:
    out = np.asarray(c, dtype=np.float32).copy()
    out.sort()
    for i in range(1, out.size):
        if out[i] <= out[i - 1]:
            out[i] = np.nextafter(out[i - 1], np.float32(np.inf))
    return out


def _subsample(v: np.ndarray, cap: int = 1 << 20) -> np.ndarray:
    if v.size <= cap:
        return v
    stride = int(np.ceil(v.size / cap))
    return v[::stride]


def key_codebook(Kcal, lo, hi, bits: int):
    K = np.asarray(Kcal, dtype=np.float64)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    s = (hi - lo) / 2.0
    z = (hi + lo) / 2.0
    kept = (K >= lo) & (K <= hi) & (s > 0)
    xn = ((K - z) / np.where(s > 0, s, 1.0))[kept]
    return _strictly_ascending_f32(kmeans_1d(_subsample(xn), k=1 << bits))


def value_normalized(Vcal, ppm: int):
    """Per-token two-sided split, normalized kept values (pooled)."""
    V = np.asarray(Vcal, dtype=np.float64)
    N, D = V.shape
    n_out = (ppm * D + 999_999) // 1_000_000
    lo, hi = two_sided_kept_range(V, n_out, axis=1)
    s = (hi - lo) / 2.0
    z = (hi + lo) / 2.0
    kept = (V >= lo[:, None]) & (V <= hi[:, None]) & (s[:, None] > 0)
    return ((V - z[:, None]) / np.where(s > 0, s, 1.0)[:, None])[kept]


def value_codebook(Vcal, ppm: int, bits: int):
    return _strictly_ascending_f32(kmeans_1d(_subsample(value_normalized(Vcal, ppm)), k=1 << bits))


def apply_qnorm(cb, mu1: float, sigma1: float, mu2: float, sigma2: float):
    """eq:qnorm."""
    c = np.asarray(cb, dtype=np.float64)
    return ((c - mu2) * sigma1 / sigma2 + mu1).astype(np.float32)


def qnorm_codebook(xn: np.ndarray, cb):
    """Q-Norm'd decode codebook from normalized calibration values (one pass)."""
    c = np.asarray(cb, dtype=np.float64)
    x = _subsample(np.asarray(xn, dtype=np.float64))
    mids = 0.5 * (c[:-1] + c[1:])
    q = c[np.searchsorted(mids, x, side="left")]
    return apply_qnorm(cb, x.mean(), x.std(), q.mean(), q.std())


def calibrate_layer(Kcal, Vcal, bits: int, ppm: int, qnorm: bool = False,
                    fp16_codebooks: bool = True):
    """Everything kvq_cache_create needs for one layer (offline)."""
    lo, hi = key_thresholds(Kcal, ppm)
    cbK = key_codebook(Kcal, lo, hi, bits)
    cbV = value_codebook(Vcal, ppm, bits)
    out = dict(key_lo=lo, key_hi=hi, cbK=cbK, cbV=cbV, cbK_dec=cbK.copy(), cbV_dec=cbV.copy())
    if qnorm:
        K = np.asarray(Kcal, np.float64)
        s = (hi.astype(np.float64) - lo) / 2.0
        z = (hi.astype(np.float64) + lo) / 2.0
        kept = (K >= lo) & (K <= hi) & (s > 0)
        xk = ((K - z) / np.where(s > 0, s, 1.0))[kept]
        out["cbK_dec"] = qnorm_codebook(xk, cbK)
        out["cbV_dec"] = qnorm_codebook(value_normalized(Vcal, ppm), cbV)
    if fp16_codebooks:
        # codebooks stored in fp16, as the paper's LUTs ("all arithmetic is performed in
        # fp16"); reading R23.  Strict ascent survives (k-means centroids are well separated).
        for key in ("cbK", "cbV", "cbK_dec", "cbV_dec"):
            cb = np.asarray(out[key], np.float32).astype(np.float16).astype(np.float32)
            assert np.all(np.diff(cb) > 0), key
            out[key] = cb
    return out
