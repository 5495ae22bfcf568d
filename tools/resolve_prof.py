#!/usr/bin/env python
"""K2 ambiguity statistics from a -DAA_PROF build: keys k_resolve decides
exactly (listed), row spans that overflowed the shared-memory list, for the
stage API (key norms from K) and the fused chain (key norms from K1).
    python tools/resolve_prof.py exp/libB_prof.so"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["AA_LIB_PATH"] = sys.argv[1]
import torch  # noqa: E402

from paper_2505_23520_b200 import capi  # noqa: E402
from paper_2505_23520_b200.workloads import gen_layer  # noqa: E402

L = capi.lib()
L.aa_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 192)()
n, hq, hkv = 131072, 32, 8
q, k, v = gen_layer(n, hq, hkv, 2505, device="cuda")
cfg = capi.BlockConfig(128, 128, 16, 12.0)
st = capi.compute_anchor(q, k, v, cfg)
anchor, qbar = capi.pool(q, k, st, cfg)
del st
cand = sum(max(0, min(2048 * g - 128, n) - 128) if g > 0 else 0 for g in range(64)) * hq
for name, fn in (("stage identify", lambda: capi.identify(q, k, qbar, anchor, cfg)),
                 ("fused chain", lambda: capi.anchor_attention(q, k, v, cfg))):
    L.aa_prof_read(buf, 1)
    fn()
    torch.cuda.synchronize()
    assert L.aa_prof_read(buf, 1) == 0
    x = list(buf)[160:192]
    print(json.dumps({"path": name, "ambiguous": x[10], "candidates": cand,
                      "fraction": x[10] / cand, "overflow_spans": x[11], "spans": x[12]}))
