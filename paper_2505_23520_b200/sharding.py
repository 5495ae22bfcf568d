"""Head sharding of a prefill attention layer across ranks.

Heads are independent (R/../SPEC.md sparse_exec "Rows and heads
independent").  With N <= Hkv ranks, rank r owns KV heads
[r*Hkv/N, (r+1)*Hkv/N) and the Hq/Hkv query heads that read them (GQA).  With
more ranks than KV heads (N a multiple of Hkv, e.g. Qwen2.5-7B's 4 KV heads
over 8 GPUs), each KV head's query heads are split into N/Hkv near-equal
runs and a rank owns one run plus its KV head (the KV head is replicated on
those ranks; query heads are independent given K/V).  The path has no data
exchange; ``gather_heads`` is the optional all-gather of O for a consumer that
needs every head on every rank (over NCCL/NVLink on GPUs, gloo in the CPU
tests).
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
    """Contiguous KV-head blocks (query heads follow their KV head), or, with
    more ranks than KV heads, contiguous query-head runs of one KV head."""
    if hq % hkv:
        raise ValueError("hq must be a multiple of hkv")
    rep = hq // hkv
    if world <= hkv:
        if hkv % world:
            raise ValueError(f"{hkv} KV heads cannot be split evenly over {world} ranks")
        per = hkv // world
        kv0 = rank * per
        return HeadShard(rank, world, kv0, kv0 + per, kv0 * rep, (kv0 + per) * rep)
    if world % hkv:
        raise ValueError(f"{world} ranks: not a multiple of the {hkv} KV heads")
    parts = world // hkv
    if parts > rep:
        raise ValueError(f"{world} ranks exceed the {hq} query heads")
    kvh, part = divmod(rank, parts)
    q0 = kvh * rep + (part * rep) // parts
    q1 = kvh * rep + ((part + 1) * rep) // parts
    return HeadShard(rank, world, kvh, kvh + 1, q0, q1)


def local_slices(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, shard: HeadShard):
    """This rank's views of full-layer q [hq,n,d], k/v [hkv,n,d]."""
    return (q[shard.q_begin:shard.q_end], k[shard.kv_begin:shard.kv_end],
            v[shard.kv_begin:shard.kv_end])


def gather_heads(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-rank head blocks [h_r, n, d] into [sum h_r, n, d] (rank
    order); blocks may differ in size (query-head runs), so they travel padded
    to the largest and are trimmed."""
    world = dist.get_world_size(group)
    sizes = [torch.zeros(1, dtype=torch.int64, device=out_local.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([out_local.shape[0]], dtype=torch.int64,
                                        device=out_local.device), group=group)
    sizes = [int(x.item()) for x in sizes]
    hmax = max(sizes)
    padded = out_local.new_zeros((hmax,) + tuple(out_local.shape[1:]))
    padded[:out_local.shape[0]] = out_local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Device-timed durations are reported as the max over ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
