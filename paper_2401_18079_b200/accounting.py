"""Algorithmic byte counts of the decode hot path for this build's layout.

Per decode step per layer, what the method itself must read/write (DESIGN.md
"Roofline"):
    T * (2*D*b/8            packed K and V codes
         + 4*k_V            Value outliers (16-bit channel + fp16 value)
         + 8                per-token Value (s, z) in fp32
         + 4)               32-bit Key CSC pointer per token
    + 4*nnz_K               Key outliers (16-bit channel + fp16 value)
    + H_q*d*2 + H_q*d*4     q in (fp16), o out (fp32)
    + D*16                  per-channel Key (s, z, lo, hi) fp32
"""
from __future__ import annotations


def attend_bytes(T: int, D: int, bits: int, kv: int, nnz_k: int, H_q: int, d: int = 128) -> int:
    return (T * (2 * D * bits // 8 + 4 * kv + 8 + 4) + 4 * nnz_k + H_q * d * 6 + D * 16)


def append_bytes(D: int, bits: int, kv: int, nnz_k_token: float) -> float:
    """Quantize-on-append of one token: read K, V (fp16), write codes/outliers/(s,z)."""
    return 2 * D * 2 + 2 * D * bits / 8 + 4 * kv + 4 * nnz_k_token + 8 + 4


def attend_flops(T: int, D: int, H_q: int, d: int = 128) -> int:
    """~2 flops per (query head, token, channel) for q.k and for p.V."""
    G = H_q // (D // d)
    return 4 * T * D * G
