#!/usr/bin/env python
"""One pass of the chain on the bench workload plus one dense launch at 32k —
a fixed launch sequence for ncu captures (fa_pair<0> K1, k_identify_tc K2,
fa_pair<1> K3, fa_pair<2> dense):

    ncu --set full --clock-control none --import-source on -k regex:fa_pair \
        -c 3 -o profiles/... python tools/ncu_target.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2505_23520_b200 import capi  # noqa: E402
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload  # noqa: E402


def main():
    n = int(os.environ.get("NCU_N", "131072"))
    hq, hkv = 32, 8
    dev = torch.device("cuda", 0)
    qs, ks, vs = [], [], []
    for kvh in range(hkv):
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=hq // hkv, hkv=1, seed=2505 + kvh),
                                    device=dev)
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    cfg = capi.BlockConfig(128, 128, 16, 12.0)
    pipe = capi.Pipeline(q, k, v, cfg)
    out = torch.empty((hq, n, 128), dtype=torch.float32, device=dev)
    pipe(q, k, v, out=out)
    nd = 32768
    capi.dense_attention(q[:, :nd].contiguous(), k[:, :nd].contiguous(), v[:, :nd].contiguous(),
                         out_dtype=torch.bfloat16)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
