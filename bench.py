#!/usr/bin/env python
"""AnchorAttention prefill benchmark (BASELINE.json metric).

Workload (BASELINE.json configs[2]): Llama-3.1-8B attention shape at 128k
tokens — 32 query heads / 8 KV heads, d = 128, b_q = b_kv = 128, step = 16,
theta = 12 (the paper's operating point) — synthetic bf16 sink/stripe heads
(paper_2505_23520_b200.workloads), generated on the GPU.

One "step" = one prefill attention layer through the fused C-ABI chain
(V->f16, K1 anchor, pool, K2 identify + compaction, K3 sparse, stats) with
inputs resident in HBM.  value = ms per layer (lower is better).  With
--gpus N (torchrun) the layer's KV heads (and their query heads) are sharded
over the ranks with no data-path collective; ms/layer is the max over ranks
(strong scaling: the layer is fixed).

Also reported: per-stage device times (CUDA events recorded by the library
on its own stream), the dominant kernel's roofline, the dense tcgen05 kernel
on the same layer, e2e through the host-buffer C ABI entry
(aa_anchor_attention_host: H2D q/k/v + chain + D2H out), and the reference
CPU path timed on a bounded sample on this box's host cores.

``--impl reference`` times the reference CPU implementation itself
(oracle/_ref, the unmodified reference sources) on the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "128k prefill attention ms/layer & % roofline; sparsity at recall vs CPU ref"
UNIT = "ms/layer"
D = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq-len", dest="n", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--theta", type=float, default=12.0)
    ap.add_argument("--step-blocks", type=int, default=16)
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=32768, help="reference sample length")
    return ap.parse_args()


# --------------------------------------------------------------------------- utils
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, val in zip(names, r[5:9]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def model_name(hq, hkv):
    return {(32, 8): "Llama-3.1-8B", (28, 4): "Qwen2.5-7B"}.get((hq, hkv), "GQA")


def config_ref(args):
    """Which BASELINE.json config this run is."""
    if (args.hq, args.hkv) == (28, 4):
        return "BASELINE configs[4]"
    if (args.hq, args.hkv) == (32, 8):
        if args.n == 32768:
            return "BASELINE configs[1]"
        if args.n == 131072:
            return "BASELINE configs[3]" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else \
                "BASELINE configs[2]"
    return "off-baseline shape"


def workload_str(args):
    return (f"{model_name(args.hq, args.hkv)} attention {args.hq}Q/{args.hkv}KV d=128, n={args.n}, "
            f"theta={args.theta}, b=128, step={args.step_blocks} ({config_ref(args)})")


def layer_geometry(n, step):
    """covered positions and stripe candidates per head (closed form)."""
    from paper_2505_23520_b200 import capi

    cfg = capi.BlockConfig(128, 128, step, 12.0)
    c = cfg.c()
    import ctypes as C

    covered = capi.lib().aa_anchor_covered_count(n, C.byref(c))
    G = capi.lib().aa_group_count(n, C.byref(c))
    offs = capi.stripe_offsets(n, cfg)
    rows = [min((g + 1) * step * 128, n) - g * step * 128 for g in range(G)]
    cand = sum((offs[g + 1] - offs[g]) * rows[g] for g in range(G))
    return covered, cand


def layer_tiles(q, k, v, args, cfg):
    """128x128 tiles K1 and K3 execute on this rank's heads: K1 runs block 0
    plus the window [wsb(g), qb] for every query block (fa_pair<ANCHOR>'s
    loop bounds); K3 runs ceil(f_c(g) / 128) gathered tiles for each query
    block of group g (counts from one stage-API identify, outside the timed
    region)."""
    import torch

    from paper_2505_23520_b200 import capi

    n, step, hq = args.n, args.step_blocks, q.shape[0]
    T = (n + 127) // 128
    k1 = 0
    for qb in range(T):
        rb = (qb // step) * step * 128
        wsb = 1 if rb < 256 else rb // 128 - 1
        k1 += 1 + (qb - wsb + 1 if qb >= wsb else 0)
    st = capi.compute_anchor(q, k, v, cfg)
    anchor, qbar = capi.pool(q, k, st, cfg)
    del st
    _, cnt = capi.identify(q, k, qbar, anchor, cfg)
    G = cnt.shape[1]
    qtiles = [min(step, T - g * step) for g in range(G)]
    k3 = int(((cnt.long() + 127) // 128).cpu().sum(0).mul(torch.tensor(qtiles, dtype=torch.int64)).sum())
    return hq * k1, k3


def k2_mma_flops(args, kv_heads):
    """Executed MMA work of k_identify_tc: per KV head and 128-row M-tile of
    (group, head) rows, key tiles up to the widest middle region of its groups,
    two bf16 MMAs (q_bar hi and lo) of 2*128^3 FLOP per key tile."""
    import ctypes as C

    from paper_2505_23520_b200 import capi

    cfg = capi.BlockConfig(128, 128, args.step_blocks, args.theta)
    c = cfg.c()
    L = capi.lib()
    G = L.aa_group_count(args.n, C.byref(c))
    rep = args.hq // args.hkv
    n_mt = (G * rep + 127) // 128
    tiles = 0
    for mt in range(n_mt):
        g_last = min(G - 1, ((mt + 1) * 128 - 1) // rep)
        span = L.aa_middle_end_token(g_last, C.byref(c), args.n) - 128
        tiles += max(0, (span + 127) // 128)
    return kv_heads * tiles * 2 * 2.0 * 128 ** 3


def reference_sample(n_sample, heads, theta, step, seed, threads=None):
    """Run the reference (oracle/_ref) anchor_attention on `heads` heads of the
    synthetic workload at n_sample through its own parallel_for.  Returns
    (wall_s, computed per head, candidates per head, covered per head)."""
    import numpy as np

    from oracle.oracle import Cfg, Reference
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    ref = Reference()
    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n_sample, hq=heads, hkv=heads, seed=seed))
    qn, kn, vn = (x.float().numpy() for x in (q, k, v))
    if threads:
        os.environ["ANCHOR_ATTN_THREADS"] = str(threads)
    t0 = time.perf_counter()
    _, computed = ref.layer(qn, kn, vn, Cfg(128, 128, step, theta))
    wall = time.perf_counter() - t0
    covered, cand = layer_geometry(n_sample, step)
    return wall, computed, cand, covered


def cpu_estimate(args, n_sample, heads, threads):
    """Reference CPU ms/layer for the full workload, extrapolated by work:
    rate = computed positions / s on the sample; the full layer's computed
    positions use the sample's measured stripe-selection fraction."""
    wall, computed, cand_s, cov_s = reference_sample(n_sample, heads, args.theta,
                                                     args.step_blocks, args.seed, threads)
    sel_frac = float((computed - cov_s).sum()) / (heads * cand_s) if cand_s else 0.0
    rate = float(computed.sum()) / wall
    cov_L, cand_L = layer_geometry(args.n, args.step_blocks)
    layer_positions = args.hq * (cov_L + sel_frac * cand_L)
    ms = layer_positions / rate * 1e3
    sample = (f"reference anchor_attention (oracle/_ref) on {heads} synthetic heads at "
              f"n={n_sample} via its parallel_for ({threads} threads): {wall:.2f} s, "
              f"{rate:.3e} positions/s; extrapolated to the {args.hq}-head n={args.n} layer by "
              f"computed positions (selection fraction {sel_frac:.4f})")
    return ms, sample, wall


# ------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    # per-head reference seconds ~ 0.8 s at 4k, x ~2.2 per doubling (SURVEY probe)
    n_sample = 4096
    for cand in (8192, 16384, 32768):
        if 0.8 * (2.2 ** ((cand // 4096).bit_length() - 1)) <= per_step_budget:
            n_sample = cand
    heads = threads
    vals = []
    sample = ""
    for i in range(args.warmup + args.steps):
        ms, sample, _ = cpu_estimate(args, n_sample, heads, threads)
        if i >= args.warmup:
            vals.append(ms)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_str(args), "global_batch": 1,
                   "seq_len": args.n, "parallelism": "host threads over heads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2505_23520_b200 import capi
    from paper_2505_23520_b200.workloads import gen_layer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    # one process per GPU; if a test launches more ranks than GPUs, ranks share
    # devices and the control collectives run over gloo instead of NCCL
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    host_group = None
    if world > 1:
        if world <= ndev:
            dist.init_process_group("nccl", device_id=dev)
            host_group = dist.new_group(backend="gloo")
        else:
            dist.init_process_group("gloo")

    def reduce(vals, op="max"):
        """Host scalars reduced over ranks (max for device-timed durations)."""
        t = torch.tensor(vals, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                            group=host_group)
        return t.tolist()

    from paper_2505_23520_b200.sharding import shard_heads

    try:
        shard = shard_heads(args.hq, args.hkv, rank, world)
    except ValueError as exc:
        raise SystemExit(f"cannot shard {args.hq}/{args.hkv} heads over {world} ranks: {exc}")
    rep = args.hq // args.hkv
    kv_local = shard.kv_heads

    # this rank's KV heads and their query heads (KV-head blocks, or with more
    # ranks than KV heads a run of one KV head's query heads); each KV head is
    # generated from its own seed so the data does not depend on the rank count
    q, k, v = gen_layer(args.n, args.hq, args.hkv, args.seed, device=dev,
                        kv_heads=range(shard.kv_begin, shard.kv_end),
                        q_range=(shard.q_begin, shard.q_end))
    cfg = capi.BlockConfig(128, 128, args.step_blocks, args.theta)
    pipe = capi.Pipeline(q, k, v, cfg)
    hq_local = q.shape[0]
    out = torch.empty((hq_local, args.n, D), dtype=torch.float32, device=dev)
    computed = torch.empty(hq_local, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        pipe(q, k, v, out=out, computed=computed)
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    for row in evs:
        for e in row:
            e.record(stream)  # materialise the CUDA events
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0.record(stream)
    for s in range(args.steps):
        capi.set_stage_events(evs[s])
        pipe(q, k, v, out=out, computed=computed)
    capi.set_stage_events(None)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_local = t0.elapsed_time(t1) / args.steps
    stage_ms = [statistics.mean(evs[s][i].elapsed_time(evs[s][i + 1]) for s in range(args.steps))
                for i in range(5)]
    k2_kernel_ms = statistics.mean(evs[s][6].elapsed_time(evs[s][7]) for s in range(args.steps))

    print(f"[bench] rank {rank}: {ms_local:.3f} ms/layer-shard, stages "
          + ", ".join(f"{nm}={t:.3f}" for nm, t in zip(capi.STAGES, stage_ms)), file=sys.stderr,
          flush=True)
    comp_local = int(computed.sum().item())
    covered, cand = layer_geometry(args.n, args.step_blocks)
    ms = reduce([ms_local], "max")[0]
    comp_total = int(reduce([comp_local], "sum")[0])
    causal = args.n * (args.n + 1) // 2
    sparsity = 1.0 - comp_total / (args.hq * causal)

    # roofline of the dominant kernel (this rank's launches)
    peaks = measured_peaks()
    # K3 runs inside a long back-to-back step (the whole chain, K steps): the
    # sustained tensor peak is the denominator (B200_PROFILING.md); the burst
    # fraction is reported beside it
    tensor_peak_burst = peaks.get("bf16_tflops", 1590.0)
    tensor_peak = peaks.get("bf16_tflops_sustained", tensor_peak_burst)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    k1_flops = 4.0 * D * hq_local * covered
    k3_flops = 4.0 * D * (comp_local - hq_local * covered)
    # tile-executed work beside the algorithmic figures: every
    # 128x128 tile a kernel runs costs 4*128^3 FLOP (QK + PV) whatever the
    # causal / tail masks leave of it
    tile_fl = 4.0 * 128 ** 3
    k1_tiles, k3_tiles = layer_tiles(q, k, v, args, cfg)
    kernels = {
        "k1_anchor": {"ms": stage_ms[1], "flops": k1_flops,
                      "tflops": k1_flops / (stage_ms[1] * 1e-3) / 1e12,
                      "tiles": k1_tiles, "tile_tflops": k1_tiles * tile_fl / (stage_ms[1] * 1e-3) / 1e12},
        "k3_sparse": {"ms": stage_ms[3], "flops": k3_flops,
                      "tflops": k3_flops / (stage_ms[3] * 1e-3) / 1e12,
                      "tiles": k3_tiles, "tile_tflops": k3_tiles * tile_fl / (stage_ms[3] * 1e-3) / 1e12},
    }
    # K2 algorithmic bytes: K over the widest middle region once
    # per KV head + pooled q (f32) and anchor (f64) per (head, group)
    import ctypes as C

    c_cfg = cfg.c()
    G = capi.lib().aa_group_count(args.n, C.byref(c_cfg))
    max_mid = max(0, capi.lib().aa_middle_end_token(G - 1, C.byref(c_cfg), args.n) - 128)
    k2_bytes = kv_local * max_mid * D * 2 + hq_local * G * (D * 4 + 8)
    kernels["k2_identify"] = {"ms": k2_kernel_ms, "bytes": k2_bytes,
                              "gbs": k2_bytes / (k2_kernel_ms * 1e-3) / 1e9,
                              "frac_hbm": k2_bytes / (k2_kernel_ms * 1e-3) / 1e9 / hbm_peak,
                              "hbm_peak_gbs": hbm_peak,
                              "frac_spec_8tbs": k2_bytes / (k2_kernel_ms * 1e-3) / 1e9 / 8000.0,
                              "mma_tflops": k2_mma_flops(args, kv_local) / (k2_kernel_ms * 1e-3) / 1e12,
                              "note": "k_identify_tc alone (events 6->7); HBM bytes are the "
                                      "algorithmic figure; mma_tflops counts the executed hi + lo "
                                      "bf16 MMAs of the split q_bar (the other pipe it keeps busy)"}
    kernels["k2_stage"] = {"ms": stage_ms[2], "bytes": k2_bytes,
                           "gbs": k2_bytes / (stage_ms[2] * 1e-3) / 1e9,
                           "note": "pool + q_bar split + identify + offsets + compaction"}
    dom = max(("k1_anchor", "k3_sparse"), key=lambda kname: kernels[kname]["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    default_cfg = (args.n, args.hq, args.hkv, args.theta, args.step_blocks, world) == \
        (131072, 32, 8, 12.0, 16, 1)
    if default_cfg and os.path.exists(tpath):  # ncu capture of this exact configuration
        try:
            traffic = json.load(open(tpath)).get(dom)
        except ValueError:
            traffic = None
    roofline = {"bound": "tensor", "kernel": dom, "achieved": kernels[dom]["tflops"],
                "peak": tensor_peak, "unit": "TFLOP/s",
                "frac": kernels[dom]["tflops"] / tensor_peak, "traffic": traffic,
                "peak_source": ("measured sustained bf16 (MEASURED_PEAKS.json bf16_tflops_sustained; "
                                "the kernel runs inside a long back-to-back step)" if peaks else
                                "fallback (B200_PROFILING.md)"),
                "frac_of_burst_peak": kernels[dom]["tflops"] / tensor_peak_burst,
                "work": f"4*d*positions = {kernels[dom]['flops']:.4e} FLOP per launch"}

    # the same layer replayed from a CUDA graph (capi.GraphPipeline: every
    # launch of the chain captured once, no host work per step)
    graph = None
    try:
        del pipe
        torch.cuda.empty_cache()
        gp = capi.GraphPipeline(q, k, v, cfg)
        for _ in range(args.warmup):
            gp.replay()
        torch.cuda.synchronize()
        barrier()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        for _ in range(args.steps):
            gp.replay()
        gb.record(stream)
        torch.cuda.synchronize()
        graph = {"ms_per_layer": reduce([ga.elapsed_time(gb) / args.steps], "max")[0],
                 "note": "capi.GraphPipeline: the fused chain captured in a CUDA graph, replayed K times"}
        del gp
        torch.cuda.empty_cache()
        pipe = capi.Pipeline(q, k, v, cfg)
    except Exception as exc:  # noqa: BLE001 - reported, not fatal
        graph = {"error": str(exc)}

    # recall of the selection at 128k: one dense QK pass (RECALL kernel) over
    # this rank's heads with the stripe lists of the timed configuration
    recall = None
    try:
        st = capi.compute_anchor(q, k, v, cfg)
        anchor, qbar = capi.pool(q, k, st, cfg)
        idx, cnts = capi.identify(q, k, qbar, anchor, cfg)
        del st
        r = capi.union_recall(q, k, idx, cnts, cfg)
        torch.cuda.synchronize()
        rsum = reduce([float(r.sum().item())], "sum")[0]
        recall = rsum / args.hq
        del idx, cnts
    except Exception as exc:  # noqa: BLE001 - reported, not fatal
        print(f"[bench] recall pass failed: {exc}", file=sys.stderr)
    torch.cuda.empty_cache()

    # dense tcgen05 FlashAttention-style kernel on the same layer (baseline)
    dense_ms = None
    if not args.no_dense:
        dout = torch.empty((hq_local, args.n, D), dtype=torch.bfloat16, device=dev)
        capi.dense_attention(q, k, v, out=dout)
        torch.cuda.synchronize()
        reps = 2
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            capi.dense_attention(q, k, v, out=dout)
        b.record(stream)
        torch.cuda.synchronize()
        dense_ms = reduce([a.elapsed_time(b) / reps], "max")[0]
        del dout

    # e2e through the host-buffer C ABI entry (pinned host tensors)
    e2e = None
    if not args.no_e2e:
        try:
            hq_h = q.cpu().pin_memory()
            hk = k.cpu().pin_memory()
            hv = v.cpu().pin_memory()
            pipe = None
            torch.cuda.empty_cache()
            o_h = torch.empty(hq_h.shape, dtype=torch.float32).pin_memory()
            c_h = torch.empty(hq_h.shape[0], dtype=torch.int64).pin_memory()
            capi.anchor_attention_host(hq_h, hk, hv, cfg, out=o_h, computed=c_h)  # warm-up
            reps = max(2, min(args.steps, 5))
            barrier()
            tt = time.perf_counter()
            for _ in range(reps):
                capi.anchor_attention_host(hq_h, hk, hv, cfg, out=o_h, computed=c_h)
            # the host entry blocks until its own stream finishes: wall time of
            # the call is the end-to-end latency (max over ranks)
            e2e_ms = reduce([(time.perf_counter() - tt) * 1e3 / reps], "max")[0]
            h2d, d2h = (int(x) for x in reduce(
                [(hq_h.numel() + hk.numel() + hv.numel()) * 2, o_h.numel() * 4 + c_h.numel() * 8],
                "sum"))
            # the copy floor: the same bytes moved alone (H2D of q/k/v and
            # D2H of O on two streams at once, no kernels), best of 3
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            do = torch.empty(o_h.shape, dtype=torch.float32, device=dev)
            s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            floor = []
            for _ in range(3):
                torch.cuda.synchronize()
                tt = time.perf_counter()
                with torch.cuda.stream(s_in):
                    for d_, h_ in ((dq, hq_h), (dk, hk), (dv, hv)):
                        d_.copy_(h_, non_blocking=True)
                with torch.cuda.stream(s_out):
                    o_h.copy_(do, non_blocking=True)
                torch.cuda.synchronize()
                floor.append((time.perf_counter() - tt) * 1e3)
            del dq, dk, dv, do
            floor_ms = reduce([min(floor)], "max")[0]
            e2e = {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h,
                   "copy_floor_ms": floor_ms,
                   "copy_floor": "same H2D+D2H bytes alone on two streams, no kernels",
                   "path": "aa_anchor_attention_host (pinned host q/k/v -> device chain -> host out f32)"}
        except Exception as exc:  # noqa: BLE001 - reported in the line
            e2e = {"value": None, "unit": UNIT, "error": str(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            ms_cpu, sample, _ = cpu_estimate(args, args.cpu_n, threads, threads)
            cpu = {"value": ms_cpu, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": sample}
        except Exception as exc:  # noqa: BLE001 - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_str(args),
                       "global_batch": 1, "seq_len": args.n,
                       "parallelism": (f"kv-head shard x{world}" if world <= args.hkv else
                                       f"query-head runs of each KV head x{world}") if world > 1
                                      else "single GPU",
                       "l2": f"inputs larger than L2 (q/k/v {(args.hq + 2 * args.hkv) * args.n * D * 2 / 1e9:.2f} "
                             "GB per layer vs 126 MB L2), no flush"},
            "sparsity": sparsity, "recall": recall, "computed_positions": comp_total,
            "stage_ms": dict(zip(capi.STAGES, stage_ms)),
            "kernels": kernels,
            "dense_ms_per_layer": dense_ms,
            "speedup_vs_dense": (dense_ms / ms) if dense_ms else None,
            "graph": graph,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # per step: V->f16, K1, pool, q_bar split, K2 identify, offsets,
            # compaction, K3, computed counts
            "gpu_launches": 9 * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
