"""Chunk-paged KV caches across sequences ("paged/blocked allocation across
sequences"; the paper's cache is one growing tensor copied on every append).

A `ChunkPool` owns fixed-size chunk caches of one layer configuration (each a kvq_cache with
capacity `chunk_tokens`, allocated once).  A `PagedSequence` is one sequence's cache of that
layer as a list of chunks taken from the pool as it grows: chunk i holds positions
[pos_base + i*chunk_tokens, ...), positioned with kvq_set_pos_base when taken, so RoPE sees the
global positions.  Releasing a sequence resets its chunks and returns them to the pool for the
next sequence -- memory is shared across sequences at chunk granularity instead of each
sequence reserving its maximum length.

Quantization is per token (per-token Values, per-channel Keys with fixed thresholds), so a
chunked sequence stores exactly the codes an unchunked cache would.  A decode step attends every
chunk (one kvq_decode_attend_batch_partial launch over the chunks of all sequences of the step)
and merges each sequence's chunk partials with kvq_merge_partials (exact log-sum-exp, fixed
chunk order) -- the same partial / merge arithmetic as the sequence sharding of sharding.py.

The chunk bookkeeping below is plain Python; every arithmetic step runs in the CUDA library.
"""
from __future__ import annotations

from typing import Callable, List, Sequence


class ChunkPool:
    """Fixed-size chunk caches of one layer configuration, shared by sequences."""

    def __init__(self, n_chunks: int, chunk_tokens: int, make_cache: Callable[[int], object]):
        """make_cache(capacity_tokens) -> a cache object (kvq.KVQCache or a test double) with
        append / prefill / num_tokens / reset / set_pos_base / attend / attend_partial."""
        if n_chunks < 1 or chunk_tokens < 1:
            raise ValueError("n_chunks and chunk_tokens must be >= 1")
        self.chunk_tokens = int(chunk_tokens)
        self._all = [make_cache(self.chunk_tokens) for _ in range(n_chunks)]
        self._free = list(reversed(self._all))

    @property
    def free_chunks(self) -> int:
        return len(self._free)

    def take(self, pos_base: int):
        if not self._free:
            raise MemoryError("chunk pool exhausted")
        c = self._free.pop()
        c.set_pos_base(pos_base)
        return c

    def give(self, chunks: Sequence[object], stream=None):
        for c in chunks:
            c.reset(stream)
            self._free.append(c)


class PagedSequence:
    """One sequence's cache of one layer, as chunks from a ChunkPool."""

    def __init__(self, pool: ChunkPool, pos_base: int = 0):
        self.pool = pool
        self.pos_base = int(pos_base)
        self.chunks: List[object] = []
        self.T = 0

    def _tail(self):
        if not self.chunks or self.chunks[-1].num_tokens == self.pool.chunk_tokens:
            self.chunks.append(self.pool.take(self.pos_base + self.T))
        return self.chunks[-1]

    def append(self, k, v, stream=None):
        self._tail().append(k, v, stream)
        self.T += 1

    def prefill(self, K, V, stream=None):
        n, a = int(K.shape[0]), 0
        while a < n:
            c = self._tail()
            b = min(n, a + self.pool.chunk_tokens - c.num_tokens)
            c.prefill(K[a:b], V[a:b], stream)
            self.T += b - a
            a = b

    def release(self, stream=None):
        self.pool.give(self.chunks, stream)
        self.chunks, self.T = [], 0


def attend_paged(seqs: Sequence[PagedSequence], qs, positions, outs, stream=None):
    """One decode step for several paged sequences: the chunks of all sequences in one batched
    partial launch (kvq_decode_attend_batch_partial, <= 64 chunks per launch), then one
    kvq_merge_partials per sequence into outs[i] ([H_q, d] fp32 device)."""
    import torch

    from . import kvq

    flat, fq, fp, owner = [], [], [], []
    for i, s in enumerate(seqs):
        if s.T == 0:
            raise ValueError(f"sequence {i} is empty")
        for c in s.chunks:
            if c.num_tokens:
                flat.append(c), fq.append(qs[i]), fp.append(int(positions[i])), owner.append(i)
    H, d = outs[0].shape
    parts = torch.empty((len(flat), H, d + 2), dtype=torch.float32, device=outs[0].device)
    B = 64   # kvq.h: at most 64 caches per batched launch
    for a in range(0, len(flat), B):
        b = min(len(flat), a + B)
        kvq.attend_batch_partial(flat[a:b], fq[a:b], fp[a:b], [parts[x] for x in range(a, b)], stream)
    dev = outs[0].device.index or 0
    start = 0
    for i, s in enumerate(seqs):
        n = sum(1 for o in owner if o == i)
        kvq.merge_partials(parts[start:start + n], outs[i], device=dev, stream=stream)
        start += n
    return outs
