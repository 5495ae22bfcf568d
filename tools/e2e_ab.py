#!/usr/bin/env python
"""End-to-end host-entry timing for same-box A/B: AA_LIB_PATH=exp/libX.so python tools/e2e_ab.py
(Llama 32/8 at n=131072, pinned host buffers, min and median of 6 calls)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2505_23520_b200 import capi
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload
hq, hkv, n = 32, 8, 131072
rep = hq // hkv
qs, ks, vs = [], [], []
for kvh in range(hkv):
    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=rep, hkv=1, seed=2505 + kvh), device=torch.device("cuda", 0))
    qs.append(q), ks.append(k), vs.append(v)
q, k, v = torch.cat(qs).cpu().pin_memory(), torch.cat(ks).cpu().pin_memory(), torch.cat(vs).cpu().pin_memory()
del qs, ks, vs
cfg = capi.BlockConfig(128, 128, 16, 12.0)
o = torch.empty(q.shape, dtype=torch.float32).pin_memory()
c = torch.empty(q.shape[0], dtype=torch.int64).pin_memory()
capi.anchor_attention_host(q, k, v, cfg, out=o, computed=c)
ts = []
for i in range(6):
    t = time.perf_counter(); capi.anchor_attention_host(q, k, v, cfg, out=o, computed=c); ts.append((time.perf_counter() - t) * 1e3)
ts.sort()
print(os.environ.get("AA_LIB_PATH"), "min %.2f med %.2f" % (ts[0], ts[3]), flush=True)
