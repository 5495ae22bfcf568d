"""KV-head sharding of a prefill attention layer across ranks.

Heads are independent (R/../SPEC.md sparse_exec "Rows and heads
independent"), so rank r of N owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and the
Hq/Hkv query heads that read them (GQA).  The path has no data exchange;
``gather_heads`` is the optional all-gather of O for a consumer that needs
every head on every rank (over NCCL/NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_begin: int
    kv_end: int
    q_begin: int
    q_end: int

    @property
    def kv_heads(self) -> int:
        return self.kv_end - self.kv_begin

    @property
    def q_heads(self) -> int:
        return self.q_end - self.q_begin


def shard_heads(hq: int, hkv: int, rank: int, world: int) -> HeadShard:
    """Contiguous KV-head blocks; query heads follow their KV head."""
    if hq % hkv:
        raise ValueError("hq must be a multiple of hkv")
    if hkv % world:
        raise ValueError(f"{hkv} KV heads cannot be split evenly over {world} ranks")
    rep = hq // hkv
    per = hkv // world
    kv0 = rank * per
    return HeadShard(rank, world, kv0, kv0 + per, kv0 * rep, (kv0 + per) * rep)


def local_slices(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, shard: HeadShard):
    """This rank's views of full-layer q [hq,n,d], k/v [hkv,n,d]."""
    return (q[shard.q_begin:shard.q_end], k[shard.kv_begin:shard.kv_end],
            v[shard.kv_begin:shard.kv_end])


def gather_heads(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-rank head blocks [hq/N, n, d] into [hq, n, d] (rank order)."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(out_local) for _ in range(world)]
    dist.all_gather(parts, out_local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Device-timed durations are reported as the max over ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
