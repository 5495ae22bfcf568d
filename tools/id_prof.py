#!/usr/bin/env python
"""Cycle accounting of the K2 identify roles (-DAA_PROF build, see tools/fa_prof.py):
producer wait on a free K stage, MMA wait on K / on a free accumulator,
threshold-warp wait on S / work per tile, CTA cycles."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["AA_LIB_PATH"] = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "exp", "libanchorattn_b200_prof.so")
import torch  # noqa: E402

from paper_2505_23520_b200 import capi  # noqa: E402
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload  # noqa: E402

L = capi.lib()
L.aa_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 192)()
n, hq, hkv = 131072, 32, 8
dev = torch.device("cuda", 0)
qs, ks, vs = [], [], []
for kvh in range(hkv):
    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=hq // hkv, hkv=1, seed=2505 + kvh), device=dev)
    qs.append(q), ks.append(k), vs.append(v)
q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
cfg = capi.BlockConfig(128, 128, 16, 12.0)
st = capi.compute_anchor(q, k, v, cfg)
anchor, qbar = capi.pool(q, k, st, cfg)
for _ in range(3):
    L.aa_prof_read(buf, 1)
    capi.identify(q, k, qbar, anchor, cfg)
    assert L.aa_prof_read(buf, 1) == 0
    x = list(buf)[160:192]
    ctas, tiles, epi_tiles = max(1, x[7]), max(1, x[9]), max(1, x[5])
    print(json.dumps({"ctas": x[7], "k_tiles": x[9], "cta_cycles": x[6] // ctas,
                      "prod_wait_empty_per_tile": x[0] / tiles, "mma_wait_k_per_tile": x[1] / tiles,
                      "mma_wait_acc_per_cta": x[2] / ctas, "epi_wait_s_per_tile": x[3] / epi_tiles,
                      "epi_work_per_tile": x[4] / epi_tiles}))
