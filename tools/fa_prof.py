#!/usr/bin/env python
"""Cycle accounting of the fa_pair roles (K1 anchor, K3 sparse, dense) on the
bench workload.  Builds a -DAA_PROF copy of the library into exp/ (clock64
stamps around every barrier wait; never the shipped library) and prints, per
kernel, the mean cycles per CTA of each role:

    python tools/fa_prof.py [--n 131072] [--build-only]
"""
from __future__ import annotations

import argparse
import ctypes as C
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_LIB = os.path.join(ROOT, "exp", "libanchorattn_b200_prof.so")
SLOTS = ["smA_wait_s", "smA_compute", "smA_tiles", "mma_wait_p", "mma_wait_k", "mma_wait_v",
         "cta_cycles", "epilogue", "prologue", "ctas", "prod_wait_empty", "smB_wait_s",
         "smB_compute", "handoff_p_to_mma", "handoffs", "pv_issue"]


def build():
    from paper_2505_23520_b200 import build as b

    os.makedirs(os.path.dirname(PROF_LIB), exist_ok=True)
    objs = []
    for cu in sorted(glob.glob(os.path.join(b.CSRC, "*.cu"))):
        o = os.path.join(ROOT, "exp", os.path.basename(cu) + ".prof.o")
        subprocess.run([b.NVCC] + b.NVCC_FLAGS + ["-DAA_PROF", "-c", cu, "-o", o], check=True)
        objs.append(o)
    subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", PROF_LIB] + objs + ["-lcuda"], check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--build-only", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--sms", type=int, default=148, help="CTA slots (1 CTA / SM)")
    ap.add_argument("--lib", default=PROF_LIB, help="a -DAA_PROF build of the library")
    a = ap.parse_args()
    if a.build_only:
        build()
        return
    os.environ["AA_LIB_PATH"] = a.lib
    import torch

    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    L = capi.lib()
    L.aa_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 192)()

    def report(name, v):
        ctas = max(1, v[9])
        tiles = max(1, v[2])
        row = {"kernel": name, "ctas": v[9], "tiles_per_cta_A": v[2] / ctas}
        for i, s in enumerate(SLOTS):
            if s in ("ctas", "smA_tiles"):
                continue
            row[s + "_per_cta"] = round(v[i] / ctas)
        row["smA_compute_per_tile"] = round(v[1] / tiles)
        row["epi_wait_odone_per_cta"] = round(v[13] / ctas)
        row["smA_tmem_ld_per_tile"] = round(v[16] / tiles)
        row["epi_t_staged0"] = round(v[14] / ctas)
        row["epi_t_half0_done"] = round(v[15] / ctas)

        row["smA_wait_per_tile"] = round(v[0] / tiles)
        if v[21]:
            span = v[21] - ((1 << 64) - 1 - v[20])
            row["span_us"] = round(span / 1e3, 1)
            row["cta_us"] = round(v[22] / ctas / 1e3, 2)
            row["sm_busy"] = round(v[22] / (a.sms * span), 4)  # CTA-resident share (1 CTA / SM)
        row["lib"] = os.path.basename(a.lib)
        print(json.dumps(row), flush=True)

    dev = torch.device("cuda", 0)
    rep = a.hq // a.hkv
    qs, ks, vs = [], [], []
    for kvh in range(a.hkv):
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=a.n, hq=rep, hkv=1, seed=2505 + kvh),
                                    device=dev)
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    cfg = capi.BlockConfig(128, 128, 16, 12.0)
    pipe = capi.Pipeline(q, k, v, cfg)
    out = torch.empty((a.hq, a.n, 128), dtype=torch.float32, device=dev)
    for rnd in range(2):
        # the fused chain (f16 hand-off, the bench path): K1 and K3 rows
        L.aa_prof_read(buf, 1)
        pipe(q, k, v, out=out)
        torch.cuda.synchronize()
        assert L.aa_prof_read(buf, 1) == 0
        allv = list(buf)
        for name, mode in (("k1_anchor", 0), ("k3_sparse", 1)):
            report(name, allv[32 * mode:32 * mode + 32])
        if not a.no_dense and rnd == 0:
            nd = min(a.n, 32768)
            L.aa_prof_read(buf, 1)
            capi.dense_attention(q[:, :nd].contiguous(), k[:, :nd].contiguous(),
                                 v[:, :nd].contiguous(), out_dtype=torch.bfloat16)
            torch.cuda.synchronize()
            assert L.aa_prof_read(buf, 1) == 0
            report(f"dense n={nd}", list(buf)[64:96])


if __name__ == "__main__":
    main()
