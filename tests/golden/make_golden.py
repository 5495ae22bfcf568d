"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists): ``python tests/golden/make_golden.py``.
Every output in the fixtures comes from oracle/_ref/libanchorref.so, i.e. the
unmodified reference sources (R/src/*.cpp) compiled by ``make -C oracle ref``
and called through their public API (``compute_anchor`` ->
``identify_stripes`` -> ``sparse_attention``).  The cases restate the
reference's own known-answer tests:

* lane_planted      R/tests/test_stripe_identify.cpp:103-123 (columns 300/500
                    at 9.5 vs anchor 10, theta 12 -> exactly {300, 500})
* lane_tie          R/tests/test_stripe_identify.cpp:146-157 (tie at theta kept)
* lane_zero_anchor  R/tests/test_stripe_identify.cpp:234-248 (zero-anchor arm)
* random_full       R/tests/test_sparse_exec.cpp:32-41 (theta=1e9 == dense)
* random_theta2     R/tests/test_sparse_exec.cpp:57-72 (union-mask equality)
* uneven_*          R/tests/test_sparse_exec.cpp:146-168 (uneven blockings)
* sink_theta*       R/tests/test_sparse_exec.cpp:214-236 (theta monotone)
* bf16_multigroup   d=128, b=128 bf16 inputs from the scalable generator, 8 groups
* bf16_c1           BASELINE config[0]: single head, 4k, d=128, theta=12
"""
from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Cfg, Reference  # noqa: E402


def lane_workload(n, d, sink, cols, bg):
    """R/tests/test_stripe_identify.cpp:27-45."""
    q = np.zeros((n, d), np.float32)
    k = np.zeros((n, d), np.float32)
    v = np.zeros((n, d), np.float32)
    sq = math.sqrt(d)
    q[:, 0] = 1.0
    v[:, 0] = np.arange(n, dtype=np.float32)
    k[:, 0] = np.float32(bg * sq)
    k[0, 0] = np.float32(sink * sq)
    for c, s in cols:
        k[c, 0] = np.float32(s * sq)
    return q, k, v


def sink_bf16(n, seed):
    import torch

    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=1, hkv=1, seed=seed))
    return [x[0].float().numpy() for x in (q, k, v)]


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ref = Reference()
    cases = []
    cases.append(("lane_planted", lane_workload(1024, 4, 10.0, [(300, 9.5), (500, 9.5)], -35.0),
                  Cfg(128, 128, 2, 12.0), False, True))
    cases.append(("lane_tie", lane_workload(512, 4, 10.0, [(200, 8.0)], -30.0),
                  Cfg(128, 128, 1, 2.0), False, True))
    lz = lane_workload(512, 4, 10.0, [(200, -1.0)], -30.0)
    cases.append(("lane_zero_anchor_real", lz, Cfg(128, 128, 1, 2.0), False, True))
    cases.append(("lane_zero_anchor_zero", lz, Cfg(128, 128, 1, 2.0), True, True))
    cases.append(("random_full", ref.gen_random(512, 8, 71), Cfg(64, 64, 2, 1e9), False, True))
    cases.append(("random_theta4", ref.gen_random(512, 8, 74), Cfg(64, 64, 2, 4.0), False, True))
    cases.append(("random_theta2", ref.gen_random(1024, 16, 73 + 1024), Cfg(64, 64, 2, 2.0),
                  False, True))
    for (n, d, bq, bkv, step) in [(777, 8, 32, 128, 2), (777, 8, 128, 32, 2), (515, 1, 64, 64, 3),
                                  (1030, 4, 128, 64, 5)]:
        for th in (1.5, 3.0):
            cases.append((f"uneven_{n}_{d}_{bq}_{bkv}_{step}_t{th}",
                          ref.gen_random(n, d, 83 + n + bq), Cfg(bq, bkv, step, th), False, True))
    sl = ref.gen_sink_local(1024, 16, 10.0, 128, 80)
    for th in (8.0, 10.0, 12.0, 14.0):
        cases.append((f"sink_theta{int(th)}", sl, Cfg(64, 64, 2, th), False, True))
    cases.append(("bf16_multigroup", sink_bf16(2048, 11), Cfg(128, 128, 2, 12.0), False, 11))
    cases.append(("bf16_c1", sink_bf16(4096, 12), Cfg(128, 128, 16, 12.0), False, 12))

    for name, (q, k, v), cfg, zero, store_inputs in cases:
        r = ref.pipeline(q, k, v, cfg, zero_anchor=zero)
        n, d = q.shape
        rec, spars = ref.recall(q, k, v, cfg, zero_anchor=zero) if n <= 4096 else (-1.0, -1.0)
        payload = dict(
            n=n, d=d, b_q=cfg.b_q, b_kv=cfg.b_kv, step=cfg.step, theta=cfg.theta,
            zero_anchor=int(zero), input_sha256=digest(q, k, v),
            m=r["m"], l=r["l"], pooled_anchor=r["pooled_anchor"], idx=r["idx"],
            counts=r["counts"], computed=r["computed"], recall=rec, sparsity=spars,
        )
        if store_inputs is True:
            payload.update(q=q, k=k, v=v, out=r["out"], anchor_out=r["anchor_out"])
        else:
            # inputs regenerate from paper_2505_23520_b200.workloads (sha-checked);
            # outputs stored on every 8th row to keep the fixture small.
            stride = 2 if n <= 2048 else 8
            payload.update(out_rows=np.arange(0, n, stride), out=r["out"][::stride],
                           anchor_out=r["anchor_out"][::stride], gen_seed=store_inputs,
                           gen="sink_bf16")
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **payload)
        print(f"{name:32s} n={n:5d} d={d:3d} computed={r['computed']:9d} "
              f"selected={int(r['counts'].sum()):7d} recall={rec:.4f}")


if __name__ == "__main__":
    main()
