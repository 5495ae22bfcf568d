"""Stripe vs block granularity at matched sparsity (the
paper's Table 1 / §2.1.2 comparison, R/../PAPER.md:125-126; the block
selectors of R/src/baselines.cpp:62-133).

For the bench workload (synthetic Llama-shaped heads at 128k) and each theta:
* stripe: AnchorAttention's selection (anchor + window + stripes); recall from
  the GPU RECALL pass, budget = computed positions per query block;
* block oracle: per query block, key blocks taken in descending true softmax
  mass (from the two-pass TILEMASS kernel) until the same per-query-block
  budget of positions is spent — the best any block-granularity selector
  (top-k / top-cdf on the block map) could do with that budget.

    python tools/block_vs_stripe.py [--seq-len 131072] > profiles/r1_sweeps/block_vs_stripe.json
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


def block_oracle_recall(mass, budget, n):
    """mass [H, T, T] tile masses, budget [H, T] positions per query block."""
    H, T, _ = mass.shape
    dev = mass.device
    qb = torch.arange(T, device=dev)
    kb = torch.arange(T, device=dev)
    rows = (torch.clamp(n - qb * B, max=B)).to(torch.float64)          # rows per query block
    cols = (torch.clamp(n - kb * B, max=B)).to(torch.float64)          # keys per key block
    cost = rows[:, None] * cols[None, :]                                # full tiles
    diag = rows * (rows + 1) / 2                                        # causal diagonal tile
    cost[qb, qb] = diag
    causal = kb[None, :] <= qb[:, None]
    m = torch.where(causal[None], mass.double(), torch.full_like(mass.double(), -1.0))
    order = torch.argsort(m, dim=-1, descending=True)
    ms = torch.gather(m, -1, order)
    cs = torch.gather(cost[None].expand(H, T, T), -1, order)
    cs = torch.where(ms >= 0, cs, torch.zeros_like(cs))
    take = (torch.cumsum(cs, -1) <= budget[..., None]) & (ms >= 0)
    return (ms.clamp_min(0) * take).sum(dim=(-1, -2)) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--thetas", default="10,12,14")
    args = ap.parse_args()
    n, rep = args.seq_len, args.hq // args.hkv
    qs, ks, vs = [], [], []
    for kvh in range(args.hkv):  # bench.py seeds
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=rep, hkv=1, seed=args.seed + kvh),
                                    device="cuda")
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    del qs, ks, vs
    base = capi.BlockConfig()
    mass = capi.dense_tile_mass(q, k, base)
    st = capi.compute_anchor(q, k, v, base)
    anchor, qbar = capi.pool(q, k, st, base)
    del st
    T = (n + B - 1) // B
    c = base.c()
    G = capi.lib().aa_group_count(n, C.byref(c))
    covered_row = torch.tensor(
        [min(B, i + 1) + max(0, i + 1 - capi.lib().aa_window_start_token(i // (16 * B), C.byref(c), n))
         for i in range(n)], dtype=torch.float64, device="cuda")
    covered_qb = torch.zeros(T, dtype=torch.float64, device="cuda").index_add_(
        0, torch.arange(n, device="cuda") // B, covered_row)
    rows_qb = torch.clamp(n - torch.arange(T, device="cuda") * B, max=B).double()
    out = []
    for th in (float(t) for t in args.thetas.split(",")):
        cfg = capi.BlockConfig(theta=th)
        idx, cnt = capi.identify(q, k, qbar, anchor, cfg)
        rec = capi.union_recall(q, k, idx, cnt, cfg)
        # per-query-block budget: covered + f_c(g) * rows
        cnt_qb = cnt.double()[:, torch.arange(T, device="cuda") // 16]
        budget = covered_qb[None] + cnt_qb * rows_qb[None]
        brec = block_oracle_recall(mass, budget, n)
        causal = n * (n + 1) / 2
        row = {"theta": th, "sparsity": 1.0 - float(budget.sum()) / (args.hq * causal),
               "recall_stripe": float(rec.mean()), "recall_block_oracle": float(brec.mean()),
               "heads_stripe_ge_block": int((rec >= brec - 1e-9).sum()), "heads": args.hq}
        print(json.dumps(row), file=sys.stderr, flush=True)
        out.append(row)
        del idx, cnt
    print(json.dumps({"workload": f"{args.hq}Q/{args.hkv}KV d=128 n={n}, b=128 step=16, "
                                  "synthetic sink/stripe heads (bench.py seeds)",
                      "block_selector": "oracle: per query block, key blocks by descending true "
                                        "softmax mass within the same position budget",
                      "rows": out}, indent=1))


if __name__ == "__main__":
    main()
