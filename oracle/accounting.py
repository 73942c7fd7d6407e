"""Byte accounting under the paper's Appendix-I conventions -- TEST INFRASTRUCTURE.

PAPER.md "Memory Usage Estimation": for NUQ the scale and offset are
16-bit each; sparse matrices use 32-bit per-token pointers and 16-bit values and
per-element indices.  Keys are per-channel (affine amortized over the l tokens of a
channel), Values per-token (affine amortized over the D elements of a token).  The
per-token pointer exists only when outliers are kept (f > 0).

Pinned by the "Avg. Num. Bits" column of tab:models-wikitext2 and the
compression ratios 3.7x / 4.8x / 6.9x; see
tests/test_oracle_accounting.py.  Reading R1: the per-token Value vector is the whole
layer, D = H_kv * d (4096 for LLaMA-7B), which is the only reading that lands inside
the printed ranges.
"""
from __future__ import annotations


def avg_bits(bits: int, f: float, D: int, seq_len: int) -> float:
    """Average stored bits per cached element, averaged over the K and V halves."""
    key = bits + 32.0 / seq_len            # per-channel 16-bit scale + 16-bit offset
    val = bits + 32.0 / D                  # per-token 16-bit scale + 16-bit offset
    if f > 0:
        key += 32.0 * f + 32.0 / D         # 16-bit value + 16-bit row index; 32-bit col ptr per token
        val += 32.0 * f + 32.0 / D         # 16-bit value + 16-bit col index; 32-bit row ptr per token
    return 0.5 * (key + val)


def compression_ratio(bits: int, f: float, D: int, seq_len: int) -> float:
    return 16.0 / avg_bits(bits, f, D, seq_len)


def fp16_kv_bytes(n_layers: int, n_heads: int, head_dim: int, batch: int, seq_len: int) -> int:
    """2 * n * h * d * b * l elements, 2 bytes each."""
    return 2 * n_layers * n_heads * head_dim * batch * seq_len * 2
