#!/usr/bin/env python
"""Time the fused chain (bench workload) under runtime knobs read by the
library through getenv, e.g.

    python tools/knob_sweep.py --env AA_K3_CLUSTER=1,2,4

Prints one JSON line per setting with ms/layer and the per-stage device
times (CUDA events recorded by the library on its stream)."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", action="append", default=[], help="NAME=v1,v2,...")
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--theta", type=float, default=12.0)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--seed", type=int, default=2505)
    a = ap.parse_args()
    import torch

    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    dev = torch.device("cuda", 0)
    rep = a.hq // a.hkv
    qs, ks, vs = [], [], []
    for kvh in range(a.hkv):
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=a.n, hq=rep, hkv=1, seed=a.seed + kvh),
                                    device=dev)
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    cfg = capi.BlockConfig(128, 128, 16, a.theta)
    pipe = capi.Pipeline(q, k, v, cfg)
    out = torch.empty((a.hq, a.n, 128), dtype=torch.float32, device=dev)
    computed = torch.empty(a.hq, dtype=torch.int64, device=dev)
    ref = None
    settings = [[]]
    for spec in a.env:
        name, vals = spec.split("=", 1)
        settings = [s + [(name, v)] for s in settings for v in vals.split(",")]
    stream = torch.cuda.current_stream()
    for s in settings:
        for name, val in s:
            os.environ[name] = val
        for _ in range(3):
            pipe(q, k, v, out=out, computed=computed)
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(a.reps)]
        for row in evs:
            for e in row:
                e.record(stream)  # materialise the events (the library records them later)
        for r in range(a.reps):
            capi.set_stage_events(evs[r])
            pipe(q, k, v, out=out, computed=computed)
        capi.set_stage_events(None)
        torch.cuda.synchronize()
        tot = [evs[r][0].elapsed_time(evs[r][5]) for r in range(a.reps)]
        st = [statistics.median(evs[r][i].elapsed_time(evs[r][i + 1]) for r in range(a.reps))
              for i in range(5)]
        if ref is None:
            ref = out.clone()
            same = True
        else:
            same = bool(torch.equal(out, ref))
        k2k = statistics.median(evs[r][6].elapsed_time(evs[r][7]) for r in range(a.reps))
        print(json.dumps({"env": dict(s), "ms": statistics.median(tot), "min_ms": min(tot), "k2_kernel_ms": k2k,
                          "stages": dict(zip(capi.STAGES, st)), "out_equal_first": same}),
              flush=True)


if __name__ == "__main__":
    main()
