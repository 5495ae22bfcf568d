"""Small cases of every fast / exact entry point for compute-sanitizer runs
(memcheck, synccheck):  compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Covers the fused chain (aligned and ragged n, GQA, zero-anchor arm), the
stage API with caller CSR lists, the dense and recall passes, the exact f64
path and the host-buffer entry."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2505_23520_b200 import capi as c  # noqa: E402
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload  # noqa: E402


def main():
    for n, hq, hkv, step in ((4096, 2, 1, 16), (5000, 4, 2, 16), (2300, 2, 1, 2)):
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=hq, hkv=hkv, seed=n))
        dq, dk, dv = q.cuda(), k.cuda(), v.cuda()
        cfg = c.BlockConfig(128, 128, step, 12.0)
        for za in (False, True):
            c.anchor_attention(dq, dk, dv, cfg, zero_anchor=za)
        st = c.compute_anchor(dq, dk, dv, cfg)
        anchor, qbar = c.pool(dq, dk, st, cfg)
        idx, counts = c.identify(dq, dk, qbar, anchor, cfg)
        c.sparse(dq, dk, dv, st, idx, counts, cfg)
        c.union_recall(dq, dk, idx, counts, cfg)
        c.dense_attention(dq, dk, dv)
        c.anchor_attention(dq.float(), dk.float(), dv.float(), cfg)  # exact path
        torch.cuda.synchronize()
        print("ok", n, hq, hkv, step, flush=True)
    # host-buffer entry (pinned copies pipelined against the chain)
    q, k, v = (x.pin_memory() for x in gen_sink_workload(SinkWorkloadSpec(n=4096, hq=4, hkv=2, seed=1)))
    out, computed = c.anchor_attention_host(q, k, v, c.BlockConfig())
    print("ok host", tuple(out.shape), flush=True)


if __name__ == "__main__":
    main()
