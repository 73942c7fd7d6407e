"""Sequence sharding of one context across GPUs, torch.distributed glue.

Every rank holds a contiguous token range [start, end) of every layer's cache, created
with pos_base = start so RoPE positions stay global.  A decode step runs
kvq_decode_attend_partial on each rank, then ONE all-gather of the [H_q][d+2] fp32
partials (16,640 B for LLaMA-7B) over NCCL / NVLink, then the same fixed-order
log-sum-exp merge kernel (kvq_merge_partials) on every rank -> bitwise identical o
everywhere.  New decode tokens are appended by the rank that owns the tail.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    total_tokens: int      # prompt tokens at prefill time
    world: int
    rank: int

    def range_of(self, r: int):
        a = (self.total_tokens * r) // self.world
        b = (self.total_tokens * (r + 1)) // self.world
        return a, b

    @property
    def start(self) -> int:
        return self.range_of(self.rank)[0]

    @property
    def end(self) -> int:
        return self.range_of(self.rank)[1]

    @property
    def pos_base(self) -> int:
        return self.start

    @property
    def tail_owner(self) -> int:
        """Rank that appends decode tokens (the shard holding the newest positions)."""
        return self.world - 1

    def capacity(self, extra_tokens: int) -> int:
        n = self.end - self.start
        return n + (extra_tokens if self.rank == self.tail_owner else 0)


def gather_partials(part, group=None):
    """All-gather one [H_q, d+2] partial per rank -> [world, H_q, d+2] in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world * part.shape[0],) + tuple(part.shape[1:]), dtype=part.dtype,
                      device=part.device)
    dist.all_gather_into_tensor(out, part.contiguous(), group=group)
    return out.view((world,) + tuple(part.shape))


def gather_merge(part, out, group=None, stream=None):
    """All-gather partials and merge them with the CUDA merge kernel (device tensors)."""
    from .kvq import merge_partials

    parts = gather_partials(part, group)
    return merge_partials(parts, out, device=part.device.index or 0, stream=stream)
