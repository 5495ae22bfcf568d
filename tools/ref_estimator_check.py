"""Checks bench.py's stage-sampled reference timing (ReferenceTimer) against
the reference run whole on the same layer: oracle/_ref's anchor_attention for
every head through its own parallel_for, wall clock.  Usage:
    python tools/ref_estimator_check.py --seq-len 32768 --samples 3 [--full]
Prints one JSON line (estimate, measured, ratio)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--theta", type=float, default=12.0)
    ap.add_argument("--samples", type=int, default=3)
    ap.add_argument("--full", action="store_true", help="also run the whole layer")
    a = ap.parse_args()
    import torch

    import bench
    from oracle.oracle import Cfg, Reference
    from paper_2505_23520_b200.workloads import gen_layer

    args = argparse.Namespace(n=a.seq_len, hq=a.hq, hkv=a.hkv, step_blocks=16, theta=a.theta,
                              seed=2505)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    q, k, v = (x.float().cpu().numpy() for x in gen_layer(a.seq_len, a.hq, a.hkv, 2505, device=dev))
    t = time.perf_counter()
    est_ms, cpu = bench.reference_measurement(q, k, v, args, a.samples)
    est_wall = time.perf_counter() - t
    line = {"n": a.seq_len, "heads": f"{a.hq}/{a.hkv}", "estimate_ms": est_ms,
            "estimate_wall_s": est_wall, "sample": cpu["sample"], "cores": cpu["cores"],
            "cpu_model": cpu["cpu_model"]}
    if a.full:
        t = time.perf_counter()
        _, computed = Reference().layer(q, k, v, Cfg(128, 128, 16, a.theta))
        line["measured_ms"] = (time.perf_counter() - t) * 1e3
        line["ratio_estimate_over_measured"] = est_ms / line["measured_ms"]
        line["computed_positions"] = int(computed.sum())
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
