"""Chunk bookkeeping of paged sequences (paper_2401_18079_b200/paged.py) on a
test double of the cache: chunk boundaries, positions, pool reuse and exhaustion (no GPU)."""
import numpy as np
import pytest

from paper_2401_18079_b200.paged import ChunkPool, PagedSequence


class FakeCache:
    def __init__(self, cap):
        self.cap, self.tokens, self.pos_base, self.resets = cap, [], None, 0

    @property
    def num_tokens(self):
        return len(self.tokens)

    def set_pos_base(self, p):
        assert not self.tokens, "repositioned while holding tokens"
        self.pos_base = p

    def reset(self, stream=None):
        self.tokens, self.resets = [], self.resets + 1

    def append(self, k, v, stream=None):
        assert len(self.tokens) < self.cap
        self.tokens.append(int(k[0]))

    def prefill(self, K, V, stream=None):
        assert len(self.tokens) + len(K) <= self.cap
        self.tokens += [int(x) for x in K[:, 0]]


def tok(a, b):
    return np.arange(a, b).reshape(-1, 1)


def test_chunks_positions_and_reuse():
    pool = ChunkPool(6, 128, FakeCache)
    s = PagedSequence(pool, pos_base=0)
    s.prefill(tok(0, 300), tok(0, 300))
    assert [c.num_tokens for c in s.chunks] == [128, 128, 44]
    assert [c.pos_base for c in s.chunks] == [0, 128, 256]
    for t in range(300, 390):
        s.append(tok(t, t + 1)[0], tok(t, t + 1)[0])
    assert [c.num_tokens for c in s.chunks] == [128, 128, 128, 6] and s.T == 390
    assert s.chunks[3].pos_base == 384
    # chunk i, slot j holds token pos_base_i + j: the sequence is the concatenation
    assert sum((c.tokens for c in s.chunks), []) == list(range(390))
    assert all(c.pos_base + j == t for c in s.chunks for j, t in enumerate(c.tokens))
    assert pool.free_chunks == 2
    s.release()
    assert pool.free_chunks == 6 and s.T == 0 and s.chunks == []
    # the next sequence reuses reset chunks at its own positions
    s2 = PagedSequence(pool, pos_base=5000)
    s2.prefill(tok(0, 200), tok(0, 200))
    assert [c.pos_base for c in s2.chunks] == [5000, 5128]
    assert all(c.resets >= 1 for c in s2.chunks)


def test_pool_exhaustion():
    pool = ChunkPool(2, 16, FakeCache)
    s = PagedSequence(pool)
    s.prefill(tok(0, 32), tok(0, 32))
    with pytest.raises(MemoryError):
        s.append(tok(32, 33)[0], tok(32, 33)[0])
    with pytest.raises(ValueError):
        ChunkPool(0, 16, FakeCache)
