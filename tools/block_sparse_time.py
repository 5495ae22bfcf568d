"""Block-sparse baseline timing at matched budget (third
bullet): flashinfer's VariableBlockSparseAttentionWrapper (library code, the
container's flashinfer; a baseline here, never the product path) against this
repo's fused AnchorAttention chain on the bench layer.

Mask: per KV head (flashinfer shares one mask across a GQA group), per query
block, key blocks in descending true softmax mass summed over the group's
query heads (TILEMASS pass) until the group's mean stripe budget — covered
positions plus f_c(g)·rows, the positions AnchorAttention computes for that
query block — is spent; the diagonal block is always taken.  Recall of the
block selection per query head comes from the same tile masses.

    python tools/block_sparse_time.py [--seq-len 131072] > profiles/r1_sweeps/block_sparse_time.json
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_23520_b200 import capi  # noqa: E402
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload  # noqa: E402

B = 128


def time_ms(fn, reps):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--theta", type=float, default=12.0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n, hq, hkv = args.seq_len, args.hq, args.hkv
    rep = hq // hkv
    dev = torch.device("cuda", 0)
    qs, ks, vs = [], [], []
    for kvh in range(hkv):  # bench.py seeds
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=rep, hkv=1, seed=args.seed + kvh),
                                    device=dev)
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    del qs, ks, vs
    cfg = capi.BlockConfig(theta=args.theta)
    T = (n + B - 1) // B

    # this repo: the fused chain (K1 -> K2 -> K3), bf16 and f32 outputs
    pipe = capi.Pipeline(q, k, v, cfg)
    comp = torch.empty(hq, dtype=torch.int64, device=dev)
    res = {}
    for name, dt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
        o = torch.empty(q.shape, dtype=dt, device=dev)
        res[name] = time_ms(lambda: pipe(q, k, v, out=o, out_dtype=dt, computed=comp), args.reps)
        del o
    causal = n * (n + 1) / 2
    stripe_sparsity = 1.0 - float(comp.double().sum()) / (hq * causal)

    # stripe budget per (query head, query block) and stripe recall
    st = capi.compute_anchor(q, k, v, cfg)
    anchor, qbar = capi.pool(q, k, st, cfg)
    del st
    idx, cnt = capi.identify(q, k, qbar, anchor, cfg)
    rec_stripe = capi.union_recall(q, k, idx, cnt, cfg)
    c = cfg.c()
    covered_row = torch.tensor(
        [min(B, i + 1) + max(0, i + 1 - capi.lib().aa_window_start_token(i // (16 * B), C.byref(c), n))
         for i in range(n)], dtype=torch.float64, device=dev)
    covered_qb = torch.zeros(T, dtype=torch.float64, device=dev).index_add_(
        0, torch.arange(n, device=dev) // B, covered_row)
    rows_qb = torch.clamp(n - torch.arange(T, device=dev) * B, max=B).double()
    budget = covered_qb[None] + cnt.double()[:, torch.arange(T, device=dev) // 16] * rows_qb[None]
    del idx, cnt

    # block mask at the group's mean budget, by group-summed tile mass
    mass = capi.dense_tile_mass(q, k, cfg).double()                     # [hq, T, T]
    gmass = mass.view(hkv, rep, T, T).sum(1)                            # [hkv, T, T]
    gbudget = budget.view(hkv, rep, T).mean(1)                          # [hkv, T]
    qb = torch.arange(T, device=dev)
    cols = torch.clamp(n - qb * B, max=B).double()
    cost = rows_qb[:, None] * cols[None, :]
    cost[qb, qb] = rows_qb * (rows_qb + 1) / 2
    causal_b = qb[None, :] <= qb[:, None]
    key = torch.where(causal_b[None], gmass, torch.full_like(gmass, -1.0))
    key[:, qb, qb] = float("inf")                                       # diagonal first
    order = torch.argsort(key, dim=-1, descending=True)
    ks_ = torch.gather(key, -1, order)
    cs = torch.gather(cost[None].expand(hkv, T, T), -1, order)
    cs = torch.where(ks_ >= 0, cs, torch.zeros_like(cs))
    take = ((torch.cumsum(cs, -1) <= gbudget[..., None]) | (order == qb[None, :, None])) & (ks_ >= 0)
    mask = torch.zeros(hkv, T, T, dtype=torch.bool, device=dev).scatter_(-1, order, take)
    del key, ks_, cs, order, take, gmass
    block_positions = float((mask.double() * cost[None]).sum()) * rep
    block_sparsity = 1.0 - block_positions / (hq * causal)
    mh = mask.repeat_interleave(rep, 0)
    rec_block = (mass * mh).sum(dim=(-1, -2)) / n
    del mass, mh

    # flashinfer block-sparse (stock wrapper, fa2 backend on sm_100)
    import flashinfer
    from flashinfer.sparse import VariableBlockSparseAttentionWrapper
    ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    w = VariableBlockSparseAttentionWrapper(ws)
    rsz = torch.full((hkv, T), B, dtype=torch.int32, device=dev)
    rsz[:, -1] = n - (T - 1) * B
    w.plan(mask, rsz, rsz.clone(), hq, hkv, q.shape[-1], causal=True,
           q_data_type=torch.bfloat16)
    fi_out = torch.empty(n * hkv, rep, q.shape[-1], dtype=torch.bfloat16, device=dev)
    fi_ms = time_ms(lambda: w.run(q, k, v, out=fi_out), args.reps)
    full = torch.ones(hkv, T, T, dtype=torch.bool, device=dev)
    wd = VariableBlockSparseAttentionWrapper(ws)
    wd.plan(full, rsz, rsz.clone(), hq, hkv, q.shape[-1], causal=True, q_data_type=torch.bfloat16)
    fi_dense_ms = time_ms(lambda: wd.run(q, k, v, out=fi_out), max(2, args.reps // 2))
    dense_ms = time_ms(lambda: capi.dense_attention(q, k, v, out_dtype=torch.bfloat16), 2)

    row = {
        "workload": f"{hq}Q/{hkv}KV d=128 n={n}, b=128 step=16, theta={args.theta}, "
                    "synthetic sink/stripe heads (bench.py seeds), bf16 inputs resident",
        "anchor_attention_ms": {"out_bf16": res["bf16"], "out_f32": res["f32"]},
        "stripe": {"sparsity": stripe_sparsity, "recall_mean": float(rec_stripe.mean()),
                   "recall_min": float(rec_stripe.min())},
        "block_mask": {"sparsity": block_sparsity, "recall_mean": float(rec_block.mean()),
                       "recall_min": float(rec_block.min()),
                       "selector": "oracle top-mass per KV group at the group's mean stripe budget"},
        "flashinfer_block_sparse_ms": fi_ms,
        "flashinfer_block_sparse_dense_mask_ms": fi_dense_ms,
        "dense_attention_ms (this repo, fa_pair<DENSE>)": dense_ms,
        "flashinfer": flashinfer.__version__,
        "note": "flashinfer run() includes its own q/k/v re-layout copies (stock call path)",
    }
    print(json.dumps(row, indent=1))


if __name__ == "__main__":
    main()
