"""torchrun worker for tests/test_sharding.py::test_torchrun_sharded_chain:
every rank runs the real fused chain (C ABI, tcgen05 path) on its balanced
shard of one generated layer (sharding.shard_work: whole KV heads, or query
heads split by query-group ranges), the pieces are all-gathered (gloo, since
the ranks share the one GPU of the test box), and rank 0 checks the
assembled layer and per-head computed counts against the single-rank run
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
    from paper_2505_23520_b200.sharding import assemble, run_units, shard_work
    from paper_2505_23520_b200.workloads import gen_layer

    n, hq, hkv = (int(x) for x in sys.argv[1:4])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    # balanced (query head, query group) units; a head may be split between
    # ranks by group ranges (aa_anchor_attention_groups)
    units = shard_work(hq, hkv, rank, world, n)
    kv0, kv1 = min(u.kv_begin for u in units), max(u.kv_end for u in units)
    q0, q1 = min(u.q_begin for u in units), max(u.q_end for u in units)
    q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda", kv_heads=range(kv0, kv1), q_range=(q0, q1))
    cfg = capi.BlockConfig()
    pieces = [(u, rows.cpu(), c.cpu()) for u, rows, c in run_units(units, q, k, v, cfg, q0, kv0)]
    gathered = [None] * world
    dist.all_gather_object(gathered, pieces)
    if rank == 0:
        full, computed = assemble([p for ps in gathered for p in ps], hq, n, 128)
        q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda")
        ref, ref_comp = capi.anchor_attention(q, k, v, cfg)
        torch.cuda.synchronize()
        ok = torch.equal(full, ref.cpu()) and torch.equal(computed, ref_comp.cpu())
        print(f"SHARD_CHECK world={world} {hq}/{hkv} n={n}: {'OK' if ok else 'MISMATCH'} "
              f"(units per rank {[len(ps) for ps in gathered]})", flush=True)
        if not ok:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
