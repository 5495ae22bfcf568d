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

``shard_work`` balances any rank count: the layer's (query head, query group)
units — groups are independent given the K/V prefix, so a head may be split
between ranks by group ranges (``aa_anchor_attention_groups``) — are ordered
KV head by KV head and cut into ``world`` contiguous runs of equal estimated
work (anchor-covered plus expected stripe positions per group).  For
Llama-3.1-8B's 32/8 heads over 1/2/4/8 ranks the cuts fall on KV-head
boundaries (the KV-head blocks of ``shard_heads``); Qwen2.5-7B's 28/4 over 8
ranks gives every rank 3.5 query heads of work instead of 4 or 3.
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


@dataclass(frozen=True)
class WorkUnit:
    """Query heads [q_begin, q_end) over the query groups [g_begin, g_end) —
    one call of the chain; the heads are either whole KV heads
    [kv_begin, kv_end) with all their query heads, or a run of the query heads
    of the single KV head kv_begin (kv_end = kv_begin + 1)."""

    kv_begin: int
    kv_end: int
    q_begin: int
    q_end: int
    g_begin: int
    g_end: int


def _series_min(r0: int, r1: int, b: int) -> int:
    """sum of min(b, i + 1) for i in [r0, r1)"""
    lo = min(max(r0, 0), r1)
    hi = min(r1, b)
    s = (lo + 1 + hi) * (hi - lo) // 2 if hi > lo else 0
    return s + b * (r1 - max(lo, hi))


def _series_over(r0: int, r1: int, ws: int) -> int:
    """sum of max(0, i + 1 - ws) for i in [r0, r1)"""
    a = max(r0, ws)
    if a >= r1:
        return 0
    return (a + 1 - ws + r1 - ws) * (r1 - a) // 2


def group_work(n: int, step: int = 16, b: int = 128, sel_frac: float = 0.15):
    """Estimated positions computed per head in each query group: the
    anchor-covered positions of its rows (R/src/detail/geometry.hpp:79-85)
    plus ``sel_frac`` of its stripe candidates (rows x middle-region keys)."""
    T = (n + b - 1) // b
    G = (T + step - 1) // step
    out = []
    for g in range(G):
        rb, re_ = g * step * b, min((g + 1) * step * b, n)
        wsb = 1 if rb < 2 * b else rb // b - 1
        ws = min(wsb * b, n)
        mid = max(0, max(ws, min(b, n)) - b)
        covered = _series_min(rb, re_, b) + _series_over(rb, re_, ws)
        out.append(covered + sel_frac * mid * (re_ - rb))
    return out


def shard_work(hq: int, hkv: int, rank: int, world: int, n: int, step: int = 16,
               sel_frac: float = 0.15) -> list:
    """This rank's WorkUnits: the (head, group) units in KV-head-major order cut
    into ``world`` runs of equal estimated work (each cut placed at the unit
    boundary nearest to the exact share)."""
    if hq % hkv:
        raise ValueError("hq must be a multiple of hkv")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    w = group_work(n, step, sel_frac=sel_frac)
    G = len(w)
    # prefix sums over the units in order (head-major, KV heads in order)
    head_total = sum(w)
    cum = [0.0]
    for g in range(G):
        cum.append(cum[-1] + w[g])
    total = hq * head_total

    def cut(r):
        """unit index (h * G + g) where run r starts"""
        if r <= 0:
            return 0
        if r >= world:
            return hq * G
        target = total * r / world
        h = min(hq - 1, int(target // head_total))
        rem = target - h * head_total
        # nearest group boundary inside head h
        g = min(range(G + 1), key=lambda x: abs(cum[x] - rem))
        return h * G + g

    u0, u1 = cut(rank), cut(rank + 1)
    rep = hq // hkv
    units = []
    u = u0
    while u < u1:
        h, g = divmod(u, G)
        if g == 0 and u + G <= u1:
            # whole heads: the rest of this KV head's heads inside the run, then
            # whole KV heads while the run covers them
            h_end = h + 1
            while h_end < hq and h_end % rep != 0 and (h_end + 1) * G <= u1:
                h_end += 1
            if h % rep == 0 and h_end % rep == 0:
                while h_end < hq and (h_end + rep) * G <= u1:
                    h_end += rep
                units.append(WorkUnit(h // rep, h_end // rep, h, h_end, 0, G))
            else:
                units.append(WorkUnit(h // rep, h // rep + 1, h, h_end, 0, G))
            u = h_end * G
        else:
            g_end = min(G, g + (u1 - u))
            units.append(WorkUnit(h // rep, h // rep + 1, h, h + 1, g, g_end))
            u = h * G + g_end
    return units


def work_of(units, n: int, step: int = 16, sel_frac: float = 0.15) -> float:
    """Estimated positions of a list of WorkUnits (for balance checks)."""
    w = group_work(n, step, sel_frac=sel_frac)
    return sum((x.q_end - x.q_begin) * sum(w[x.g_begin:x.g_end]) for x in units)


def unit_rows(unit: WorkUnit, n: int, step: int = 16, b: int = 128):
    """Row range [r0, r1) of the unit's query groups."""
    return unit.g_begin * step * b, min(unit.g_end * step * b, n)


def run_units(units, q, k, v, cfg, q_base: int = 0, kv_base: int = 0, out_dtype=None):
    """Run a rank's WorkUnits on its local tensors (q heads from global head
    ``q_base``, k/v heads from global KV head ``kv_base``) through the C ABI.
    Returns [(unit, out rows of the unit [q_end - q_begin, r1 - r0, d],
    computed [q_end - q_begin])]."""
    import torch

    from . import capi

    res = []
    for u in units:
        qs = q[u.q_begin - q_base:u.q_end - q_base]
        ks = k[u.kv_begin - kv_base:u.kv_end - kv_base]
        vs = v[u.kv_begin - kv_base:u.kv_end - kv_base]
        pipe = capi.Pipeline(qs, ks, vs, cfg)
        out, comp = pipe(qs, ks, vs, out_dtype=out_dtype or torch.float32,
                         groups=(u.g_begin, u.g_end))
        r0, r1 = unit_rows(u, q.shape[1], cfg.step, cfg.b_q)
        res.append((u, out[:, r0:r1], comp))
    return res


def assemble(pieces, hq: int, n: int, d: int, step: int = 16, b: int = 128):
    """The layer output [hq, n, d] and per-head computed counts [hq] from every
    rank's (unit, rows, computed) pieces (host tensors)."""
    import torch

    out = None
    computed = torch.zeros(hq, dtype=torch.int64)
    for u, rows, comp in pieces:
        if out is None:
            out = torch.empty((hq, n, d), dtype=rows.dtype)
        r0, r1 = unit_rows(u, n, step, b)
        out[u.q_begin:u.q_end, r0:r1] = rows
        computed[u.q_begin:u.q_end] += comp.to(torch.int64)
    return out, computed
