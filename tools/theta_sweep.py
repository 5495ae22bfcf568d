"""Theta sweep at the bench workload (the paper's Table 6
shape, R/../PAPER.md:443-456): the anchor pass (K1) runs once, then for each
theta the identification (K2 + compaction) and the sparse fold (K3) run on
the same anchor state, with and without the anchor (zero-anchor arm,
R/src/stripe_identify.cpp:90-95).  Reports sparsity, recall (GPU RECALL pass
over the dense softmax) and device ms of K2 and K3 per theta.

    python tools/theta_sweep.py [--seq-len 131072] [--hq 32 --hkv 8] > profiles/theta_sweep.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_23520_b200 import capi  # noqa: E402
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload  # noqa: E402


def timed(fn, reps=3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--thetas", default="10,11,12,13,14,15")
    args = ap.parse_args()
    n, rep = args.seq_len, args.hq // args.hkv
    qs, ks, vs = [], [], []
    for kvh in range(args.hkv):  # same per-KV-head seeds as bench.py
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=rep, hkv=1, seed=args.seed + kvh),
                                    device="cuda")
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    del qs, ks, vs
    base = capi.BlockConfig()
    st, k1_ms = timed(lambda: capi.compute_anchor(q, k, v, base), reps=1)
    anchor, qbar = capi.pool(q, k, st, base)
    causal = n * (n + 1) // 2
    rows = []
    for zero in (False, True):
        for th in (float(t) for t in args.thetas.split(",")):
            cfg = capi.BlockConfig(theta=th)
            (idx, cnt), k2_ms = timed(lambda: capi.identify(q, k, qbar, anchor, cfg,
                                                            zero_anchor=zero))
            (out, comp), k3_ms = timed(lambda: capi.sparse(q, k, v, st, idx, cnt, cfg,
                                                           out_dtype=torch.bfloat16))
            rec = capi.union_recall(q, k, idx, cnt, cfg)
            torch.cuda.synchronize()
            rows.append({"theta": th, "zero_anchor": zero,
                         "sparsity": 1.0 - float(comp.sum()) / (args.hq * causal),
                         "recall": float(rec.mean()),
                         "k2_identify_ms": k2_ms, "k3_sparse_ms": k3_ms,
                         "layer_ms_est": k1_ms + k2_ms + k3_ms})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del idx, cnt, out, comp
    print(json.dumps({"workload": f"Llama-3.1-8B attention {args.hq}Q/{args.hkv}KV d=128, n={n}, "
                                  "b=128, step=16, synthetic sink/stripe heads (bench.py seeds)",
                      "k1_anchor_ms_once": k1_ms, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
