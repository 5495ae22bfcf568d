"""Multi-rank host logic of KV-head sharding (world_size 2, gloo, CPU) and the
sharded layer on one GPU (every rank's shard run in turn equals the full run)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_23520_b200.sharding import (gather_heads, local_slices, max_over_ranks,
                                            shard_heads)


def test_shard_assignment_covers_heads_once():
    for hq, hkv, world in [(32, 8, 1), (32, 8, 2), (32, 8, 4), (32, 8, 8), (28, 4, 2), (28, 4, 4),
                           (28, 4, 8), (32, 8, 16), (8, 2, 8)]:
        seen_q, seen_kv = [], []
        for r in range(world):
            s = shard_heads(hq, hkv, r, world)
            seen_q += list(range(s.q_begin, s.q_end))
            seen_kv += list(range(s.kv_begin, s.kv_end))
            for h in range(s.q_begin, s.q_end):  # GQA: query head reads a local KV head
                assert s.kv_begin <= h // (hq // hkv) < s.kv_end
        assert seen_q == list(range(hq))
        if world <= hkv:
            assert seen_kv == list(range(hkv))
        else:  # query-head runs: each KV head replicated on world / hkv ranks
            assert seen_kv == sorted(seen_kv) and sorted(set(seen_kv)) == list(range(hkv))
    # query-head runs: Qwen2.5-7B (28 Q / 4 KV) over 8 ranks -> 4 / 3 heads each
    assert [shard_heads(28, 4, r, 8).q_heads for r in range(8)] == [3, 4] * 4
    with pytest.raises(ValueError):
        shard_heads(28, 4, 0, 6)   # 6 ranks: neither divides nor is a multiple of 4 KV heads
    with pytest.raises(ValueError):
        shard_heads(8, 2, 0, 16)   # more ranks than query heads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, k, v, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = shard_heads(q.shape[0], k.shape[0], rank, world)
    ql, kl, vl = local_slices(q, k, v, shard)
    rep = q.shape[0] // k.shape[0]
    # stand-in per-head op with the same head->KV-head dependence as attention
    kv_of = torch.tensor([h // rep - shard.kv_begin for h in range(shard.q_begin, shard.q_end)])
    out_local = ql * kl[kv_of] + vl[kv_of]
    full = gather_heads(out_local)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        ret["full"] = full
        ret["max"] = t
    dist.destroy_process_group()


@pytest.mark.parametrize("world,hq,hkv", [(2, 8, 2), (4, 6, 2)])
def test_gloo_gather_and_max(world, hq, hkv):
    """world 2: KV-head blocks; world 4 over 2 KV heads: query-head runs of
    unequal length (3 query heads per KV head -> 1 / 2), gathered padded."""
    q = torch.randn(hq, 16, 4)
    k = torch.randn(hkv, 16, 4)
    v = torch.randn(hkv, 16, 4)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), q, k, v, ret), nprocs=world, join=True)
    rep = hq // hkv
    expect = q * k.repeat_interleave(rep, 0) + v.repeat_interleave(rep, 0)
    assert torch.equal(ret["full"], expect)
    assert ret["max"] == float(world)


@pytest.mark.gpu
def test_sharded_layer_equals_full_layer():
    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=8192, hq=8, hkv=4, seed=17), device="cuda")
    cfg = capi.BlockConfig()
    full, comp = capi.anchor_attention(q, k, v, cfg)
    for world in (2, 4, 8):  # 8 ranks over 4 KV heads: query-head runs
        parts, comps = [], []
        for r in range(world):
            s = shard_heads(8, 4, r, world)
            o, c = capi.anchor_attention(*local_slices(q, k, v, s), cfg)
            parts.append(o)
            comps.append(c)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(parts), full)
        assert torch.equal(torch.cat(comps), comp)


@pytest.mark.gpu
@pytest.mark.parametrize("world,hq,hkv", [(2, 32, 8), (8, 28, 4)])
def test_torchrun_sharded_chain(world, hq, hkv):
    """torchrun, one process per rank (all on the test box's one GPU, gloo
    for the gather): each rank runs the real chain on its balanced shard —
    KV-head blocks (Llama 32/8 over 2) or 3.5 query heads of work per rank
    (Qwen 28/4 over 8: one head split by query groups between two ranks) —
    and the assembled output and computed counts equal the single-rank layer
    bit for bit."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tests", "shard_worker.py"), "16384", str(hq), str(hkv)]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"SHARD_CHECK world={world} {hq}/{hkv} n=16384: OK" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("hq,hkv,world,n", [(32, 8, 1, 131072), (32, 8, 2, 131072), (32, 8, 4, 131072),
                                            (32, 8, 8, 131072), (28, 4, 8, 131072), (28, 4, 6, 131072),
                                            (32, 8, 3, 32768), (28, 4, 16, 131072), (8, 2, 5, 5000)])
def test_shard_work_covers_units_once_and_balances(hq, hkv, world, n):
    """Balanced (head, group) shards: every unit exactly once, each call either
    whole KV heads or a run of one KV head's query heads, estimated work
    within 1% of the mean (when units are plentiful), and the KV-head blocks
    of shard_heads for Llama 32/8 over 1/2/4/8 ranks."""
    from paper_2505_23520_b200.sharding import group_work, shard_work, work_of

    G = len(group_work(n))
    rep = hq // hkv
    seen = set()
    works = []
    for r in range(world):
        units = shard_work(hq, hkv, r, world, n)
        for u in units:
            assert 0 <= u.g_begin < u.g_end <= G
            if u.kv_end - u.kv_begin > 1 or (u.q_end - u.q_begin) == rep:
                assert (u.q_begin, u.q_end) == (u.kv_begin * rep, u.kv_end * rep)
            else:
                assert u.kv_begin * rep <= u.q_begin < u.q_end <= (u.kv_begin + 1) * rep
            for h in range(u.q_begin, u.q_end):
                for g in range(u.g_begin, u.g_end):
                    assert (h, g) not in seen
                    seen.add((h, g))
        works.append(work_of(units, n))
    assert len(seen) == hq * G
    if hq * G >= 20 * world:
        assert max(works) <= 1.01 * sum(works) / world
    if (hq, hkv) == (32, 8) and world in (1, 2, 4, 8):
        for r in range(world):
            s = shard_heads(hq, hkv, r, world)
            assert shard_work(hq, hkv, r, world, n) == [
                type(shard_work(hq, hkv, r, world, n)[0])(s.kv_begin, s.kv_end, s.q_begin, s.q_end, 0, G)]


@pytest.mark.gpu
@pytest.mark.parametrize("hq,hkv,world", [(28, 4, 8), (32, 8, 3), (8, 2, 5)])
def test_group_shards_equal_full_layer(hq, hkv, world):
    """Every rank's WorkUnits run in turn on one GPU (aa_anchor_attention_groups
    for split heads) and assembled equal the single-call layer bit for bit,
    computed counts included."""
    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.sharding import assemble, run_units, shard_work
    from paper_2505_23520_b200.workloads import gen_layer

    n = 16384
    q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda")
    cfg = capi.BlockConfig()
    full, comp = capi.anchor_attention(q, k, v, cfg)
    pieces = []
    for r in range(world):
        pieces += [(u, rows.cpu(), c.cpu()) for u, rows, c in
                   run_units(shard_work(hq, hkv, r, world, n), q, k, v, cfg)]
    out, computed = assemble(pieces, hq, n, 128)
    assert torch.equal(out, full.cpu())
    assert torch.equal(computed, comp.cpu())


def _units_worker(rank, world, port, hq, hkv, n, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_23520_b200.sharding import shard_work, unit_rows

    # stand-in per-row op: row i of head h combines its query with row i of
    # its KV head (the routing of heads, KV heads and group rows under test)
    g = torch.Generator().manual_seed(0)
    q = torch.randn(hq, n, 2, generator=g)
    kv = torch.randn(hkv, n, 2, generator=g)
    rep = hq // hkv
    pieces = []
    for u in shard_work(hq, hkv, rank, world, n, step=2):
        r0, r1 = unit_rows(u, n, step=2)
        heads = range(u.q_begin, u.q_end)
        rows = torch.stack([q[h, r0:r1] * kv[h // rep, r0:r1] for h in heads])
        pieces.append((u, rows, torch.full((len(heads),), r1 - r0, dtype=torch.int64)))
    gathered = [None] * world
    dist.all_gather_object(gathered, pieces)
    if rank == 0:
        from paper_2505_23520_b200.sharding import assemble

        out, cnt = assemble([p for ps in gathered for p in ps], hq, n, 2, step=2)
        ref = q * kv.repeat_interleave(rep, 0)
        ret["ok"] = torch.equal(out, ref) and bool((cnt == n).all())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,hq,hkv", [(2, 6, 2), (3, 7, 1)])
def test_gloo_group_shards_assemble(world, hq, hkv):
    """gloo, world 2 / 3: balanced (head, group) shards with split heads are
    computed per rank, all-gathered and assembled into the whole layer."""
    mgr = mp.Manager()
    ret = mgr.dict()
    n = 1000  # groups of step 2 x 128 = 256 rows, the last one partial
    mp.spawn(_units_worker, args=(world, _free_port(), hq, hkv, n, ret), nprocs=world, join=True)
    assert ret["ok"]
