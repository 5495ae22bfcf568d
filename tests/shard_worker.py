"""torchrun worker for tests/test_sharding.py::test_torchrun_sharded_chain:
every rank runs the real fused chain (C ABI, tcgen05 path) on its head shard
of one generated layer, the outputs are all-gathered (gather_heads; gloo,
since the ranks share the one GPU of the test box), and rank 0 checks the
gathered layer and per-head computed counts against the single-rank run
bit for bit.  Usage (from the repo root):
    python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 \\
        --master-port P tests/shard_worker.py N HQ HKV
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.sharding import gather_heads, shard_heads
    from paper_2505_23520_b200.workloads import gen_layer

    n, hq, hkv = (int(x) for x in sys.argv[1:4])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    shard = shard_heads(hq, hkv, rank, world)
    q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda", kv_heads=range(shard.kv_begin, shard.kv_end),
                        q_range=(shard.q_begin, shard.q_end))
    cfg = capi.BlockConfig()
    out, comp = capi.anchor_attention(q, k, v, cfg)
    torch.cuda.synchronize()
    full = gather_heads(out.cpu())
    comps = gather_heads(comp.cpu()[:, None, None])[:, 0, 0]
    if rank == 0:
        q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda")
        ref, ref_comp = capi.anchor_attention(q, k, v, cfg)
        torch.cuda.synchronize()
        ok = torch.equal(full, ref.cpu()) and torch.equal(comps, ref_comp.cpu())
        print(f"SHARD_CHECK world={world} {hq}/{hkv} n={n}: {'OK' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
