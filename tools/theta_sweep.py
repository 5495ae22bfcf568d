"""Theta sweep at the bench workload (the paper's Table 6
shape, R/../PAPER.md:443-456), with and without the anchor (zero-anchor arm,
R/src/stripe_identify.cpp:90-95).  Per theta: the fused chain (the bench
path, capi.Pipeline) timed with the library's stage events (K1, pool + K2 +
compaction, K3, the layer), sparsity from its computed counts, and recall
from a GPU RECALL pass over the dense softmax with the stripe lists of the
same configuration (stage API, untimed).

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
    causal = n * (n + 1) // 2
    out = torch.empty((args.hq, n, 128), dtype=torch.float32, device="cuda")
    computed = torch.empty(args.hq, dtype=torch.int64, device="cuda")
    base = capi.BlockConfig()
    st = capi.compute_anchor(q, k, v, base)
    anchor, qbar = capi.pool(q, k, st, base)
    del st
    rows = []
    k1_ms = None
    for zero in (False, True):
        for th in (float(t) for t in args.thetas.split(",")):
            cfg = capi.BlockConfig(theta=th)
            pipe = capi.Pipeline(q, k, v, cfg)
            pipe(q, k, v, zero_anchor=zero, out=out, computed=computed)  # warm-up
            reps = 3
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(reps)]
            for row in evs:
                for e in row:
                    e.record()
            torch.cuda.synchronize()
            for r in range(reps):
                capi.set_stage_events(evs[r])
                pipe(q, k, v, zero_anchor=zero, out=out, computed=computed)
            capi.set_stage_events(None)
            torch.cuda.synchronize()
            st_ms = [sum(evs[r][i].elapsed_time(evs[r][i + 1]) for r in range(reps)) / reps for i in range(5)]
            layer = sum(evs[r][0].elapsed_time(evs[r][5]) for r in range(reps)) / reps
            del pipe
            idx, cnt = capi.identify(q, k, qbar, anchor, cfg, zero_anchor=zero)
            rec = capi.union_recall(q, k, idx, cnt, cfg)
            torch.cuda.synchronize()
            k1_ms = st_ms[1]
            rows.append({"theta": th, "zero_anchor": zero,
                         "sparsity": 1.0 - float(computed.sum()) / (args.hq * causal),
                         "recall": float(rec.mean()),
                         "k1_anchor_ms": st_ms[1], "k2_stage_ms": st_ms[2], "k3_sparse_ms": st_ms[3],
                         "layer_ms": layer})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del idx, cnt, rec
    print(json.dumps({"workload": f"Llama-3.1-8B attention {args.hq}Q/{args.hkv}KV d=128, n={n}, "
                                  "b=128, step=16, synthetic sink/stripe heads (bench.py seeds)",
                      "timing": "fused chain (capi.Pipeline) per theta, library stage events, mean of 3",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
