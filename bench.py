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
    ap.add_argument("--cpu-samples", type=int, default=6,
                    help="sparse_attention sample steps of the cpu_baseline reference timing")
    ap.add_argument("--no-dense-libs", action="store_true",
                    help="skip the cuDNN / flashinfer dense comparators")
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


def geometry(n, step, b=128):
    """Closed forms of the reference's blocking (R/src/detail/geometry.hpp:22-85,
    SURVEY.md Appendix A) in plain Python — shared by both arms, so the
    reference arm loads nothing of this repo's native code.  Returns dict(G,
    rows [G], covered (per head), cand [G] (middle-region keys per group))."""
    T = (n + b - 1) // b
    G = (T + step - 1) // step
    rows, cand = [], []
    covered = 0
    for g in range(G):
        rb = g * step * b
        re_ = min(rb + step * b, n)
        wsb = 1 if rb < 2 * b else rb // b - 1
        ws = min(wsb * b, n)
        mid_end = max(ws, min(b, n))
        rows.append(re_ - rb)
        cand.append(max(0, mid_end - b))
        # rows i in [rb, re_): covered = min(b, i + 1) + max(0, i + 1 - ws)
        lo = rb
        hi1 = min(re_, b)  # rows with i + 1 <= b
        if hi1 > lo:
            covered += (lo + 1 + hi1) * (hi1 - lo) // 2
            lo = hi1
        covered += b * (re_ - lo)
        w0 = max(rb, ws)  # rows with i + 1 > ws
        if re_ > w0:
            covered += (w0 + 1 - ws + re_ - ws) * (re_ - w0) // 2
    return {"G": G, "rows": rows, "covered": covered, "cand": cand}


def layer_geometry(n, step):
    """covered positions and stripe candidate positions per head."""
    g = geometry(n, step)
    return g["covered"], sum(c * r for c, r in zip(g["cand"], g["rows"]))


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


def sample_group(s, G):
    """Stripe group the reference times at sample step s: consecutive steps
    pair a heavy group with a light one (G-1-j, j), j striding over the
    lower half, so any two consecutive steps span the work distribution."""
    j = (s // 2) * 7 % max(1, G // 2)
    return G - 1 - j if s % 2 == 0 else j


class ReferenceTimer:
    """The reference CPU implementation (oracle/_ref: the unmodified
    reference sources compiled by oracle/Makefile) timed on THIS layer — the
    same GQA inputs, n, theta and step — through its own public API and its
    own parallel_for (one head per task, ANCHOR_ATTN_THREADS = host cores).

    * compute_anchor + identify_stripes run on every head of the layer once,
      timed as they are (no extrapolation): ``t12``.
    * sparse_attention is the bulk of the reference's time (SURVEY §8(a):
      21.3 of 55 s per head at sparsity 0.97, ~85% at 0.85).  A sample step
      runs it on one round of heads (one head per thread) with each head's
      StripeIndex cut to one group (sample_group), against the same round
      with every list emptied (``t0``: the per-head state copy and finalize
      the reference does regardless).  The per-position cost
      (t_step - t0) / positions is pooled over the steps (ratio estimator)
      and applied to the layer's own selected positions (the reference's
      identify output), round by round: rounds = ceil(H / threads).
    The layer estimate is t12 + rounds * (t0 + cost * mean selected positions
    per head of a round)."""

    def __init__(self, q, k, v, n, step, theta):
        import numpy as np

        from oracle.oracle import Cfg, Reference

        self.np = np
        self.ref = Reference()
        self.threads = self.ref.max_threads()
        self.H = q.shape[0]
        self.geo = geometry(n, step)
        self.layer = self.ref.open_layer(q, k, v, Cfg(128, 128, step, theta))
        t = time.perf_counter()
        self.layer.anchor_identify()
        self.t12 = time.perf_counter() - t
        G = self.geo["G"]
        self.counts = self.layer.counts(G)  # f_c per (head, group)
        self.rows = np.array(self.geo["rows"], np.int64)
        self.sel = (self.counts * self.rows[None, :]).sum(1)  # selected positions per head
        self.round = min(self.H, self.threads)
        self.rounds = (self.H + self.round - 1) // self.round
        self.t0 = []  # per round: the pass with every list emptied
        for r in range(self.rounds):
            t = time.perf_counter()
            self.layer.sparse_groups(self._groups(-2, r))
            self.t0.append(time.perf_counter() - t)
        self.num = 0.0  # sum of (t_step - t0[round])
        self.den = 0.0  # sum of the sampled positions of each pass's slowest head
        self.steps = []

    def _groups(self, g, r):
        """Group g kept on the heads of round r; the other heads sit out."""
        keep = self.np.full(self.H, -3, self.np.int64)
        keep[r * self.round:(r + 1) * self.round] = g
        return keep

    def sample(self, s):
        g = sample_group(s, self.geo["G"])
        r = s % self.rounds
        heads = self.np.arange(r * self.round, min((r + 1) * self.round, self.H))
        t = time.perf_counter()
        self.layer.sparse_groups(self._groups(g, r))
        dt = time.perf_counter() - t
        # the pass lasts as long as its slowest head (one head per thread)
        pos = float(self.counts[heads, g].max() * self.rows[g])
        self.steps.append((s, g, r, dt, pos))
        return dt - self.t0[r], pos

    def account(self, dt, pos):
        self.num += dt
        self.den += pos

    def layer_seconds(self):
        per_pos = self.num / self.den if self.den > 0 else 0.0
        k3 = 0.0
        for r in range(self.rounds):
            heads = self.sel[r * self.round:(r + 1) * self.round]
            k3 += self.t0[r] + per_pos * float(heads.mean())
        return self.t12 + k3, per_pos

    def describe(self, per_pos):
        return (f"reference anchor_attention stages (oracle/_ref, its own parallel_for over "
                f"{self.threads} threads) on this layer's {self.H} heads: compute_anchor + "
                f"identify_stripes measured whole ({self.t12:.1f} s); sparse_attention sampled on "
                f"{len(self.steps)} (round, group) steps of {self.round} heads x 1 group "
                f"(groups {sorted(set(g for _, g, _, _, _ in self.steps))}), "
                f"{per_pos * 1e9:.1f} ns per folded position per head-task, fixed cost "
                f"{sum(self.t0):.2f} s over the rounds, scaled by the layer's own selected positions "
                f"({float(self.sel.sum()):.4e}) over {self.rounds} round(s)")

    def close(self):
        self.layer.close()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_measurement(q, k, v, args, samples):
    """(ms/layer, cpu_baseline dict) of the reference on this layer."""
    rt = ReferenceTimer(q, k, v, args.n, args.step_blocks, args.theta)
    try:
        for s in range(samples):
            rt.account(*rt.sample(s))
        sec, per_pos = rt.layer_seconds()
        desc = rt.describe(per_pos)
        threads = rt.threads
    finally:
        rt.close()
    return sec * 1e3, {"value": sec * 1e3, "unit": UNIT, "cores": threads, "kind": "reference",
                       "cpu_model": cpu_model(), "sample": desc}


def layer_config(args):
    """The `config` object both arms print (identical for the same run)."""
    return {"workload": workload_str(args), "global_batch": 1, "seq_len": args.n,
            "heads": f"{args.hq}Q/{args.hkv}KV",
            "parallelism": "heads sharded over ranks" if int(os.environ.get("WORLD_SIZE", "1")) > 1
                           else "one device",
            "l2": f"inputs larger than L2 (q/k/v {(args.hq + 2 * args.hkv) * args.n * D * 2 / 1e9:.2f} "
                  "GB per layer vs 126 MB L2), no flush"}


# ------------------------------------------------------------------------ reference arm
def run_reference(args):
    """--impl reference: the reference CPU implementation on this layer (the
    same inputs as our arm, generated by workloads.gen_layer), rank 0 only.
    One step = one sparse_attention sample of ReferenceTimer; warm-up steps
    are run and discarded; the line's value is the layer estimate from the
    K timed steps."""
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2505_23520_b200.workloads import gen_layer

    dev = "cuda" if torch.cuda.is_available() else "cpu"  # the bench's generator stream
    q, k, v = gen_layer(args.n, args.hq, args.hkv, args.seed, device=dev)
    qn, kn, vn = (x.float().cpu().numpy() for x in (q, k, v))
    del q, k, v
    t_start = time.perf_counter()
    rt = ReferenceTimer(qn, kn, vn, args.n, args.step_blocks, args.theta)
    del qn, kn, vn
    try:
        for s in range(args.warmup):
            rt.sample(s)
        for s in range(args.warmup, args.warmup + args.steps):
            rt.account(*rt.sample(s))
        sec, per_pos = rt.layer_seconds()
        desc = rt.describe(per_pos)
        threads = rt.threads
    finally:
        rt.close()
    value = sec * 1e3
    wall = time.perf_counter() - t_start
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": layer_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_wall_s": wall,
        "note": ("a step is a bounded sample (one sparse_attention group per head of a round); "
                 "value is the whole-layer estimate, not the sample's wall time"),
    }
    print(json.dumps(line), flush=True)


def dense_library_baselines(q, k, v, barrier, reduce, reps=2):
    """Dense causal GQA attention of the same layer through library kernels
    (the comparators of the north-star bar, semantics R/src/oracle.cpp:66-94):
    torch SDPA on its cuDNN backend and flashinfer's single-prefill kernels
    (cutlass = the sm100 FMHA, fa2), each timed with CUDA events after one
    warm-up call; an entry holds the error when a backend is unavailable."""
    import torch
    import torch.nn.functional as F

    hq, n, d = q.shape
    hkv = k.shape[0]
    res = {}
    stream = torch.cuda.current_stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return reduce([a.elapsed_time(b) / reps], "max")[0]

    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        q4, k4, v4 = q[None], k[None], v[None]
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            try:
                res["torch_sdpa_cudnn"] = timed(
                    lambda: F.scaled_dot_product_attention(q4, k4, v4, is_causal=True,
                                                           enable_gqa=True))
            except Exception:  # noqa: BLE001 - cuDNN without native GQA: K/V expanded
                rep = hq // hkv
                ke, ve = (x.repeat_interleave(rep, dim=1) for x in (k4, v4))
                res["torch_sdpa_cudnn"] = timed(
                    lambda: F.scaled_dot_product_attention(q4, ke, ve, is_causal=True))
                res["torch_sdpa_cudnn_note"] = "K/V expanded to the query heads (no GQA entry)"
                del ke, ve
    except Exception as exc:  # noqa: BLE001 - reported in the line
        res["torch_sdpa_cudnn"] = f"unavailable: {str(exc).splitlines()[0][:160]}"
    torch.cuda.empty_cache()
    try:
        import flashinfer

        qn = q.transpose(0, 1).contiguous()  # NHD
        kn = k.transpose(0, 1).contiguous()
        vn = v.transpose(0, 1).contiguous()
        # the ragged-batch prefill wrapper carries flashinfer's Blackwell
        # kernels: "cutlass" (the sm100 CUTLASS FMHA) and "cute-dsl" (the
        # CuTe-DSL sm100 attention kernel); fa2 through the single-prefill entry
        ind = torch.tensor([0, n], dtype=torch.int32, device=q.device)
        for backend in ("cutlass", "cute-dsl"):
            try:
                ws = torch.empty(256 << 20, dtype=torch.uint8, device=q.device)
                w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, kv_layout="NHD",
                                                                    backend=backend)
                w.plan(ind, ind, hq, hkv, d, causal=True, q_data_type=q.dtype,
                       kv_data_type=k.dtype)
                res[f"flashinfer_{backend}"] = timed(lambda: w.run(qn, kn, vn))
                del w, ws
            except Exception as exc:  # noqa: BLE001
                res[f"flashinfer_{backend}"] = f"unavailable: {str(exc).splitlines()[0][:160]}"
        try:
            res["flashinfer_fa2"] = timed(
                lambda: flashinfer.single_prefill_with_kv_cache(qn, kn, vn, causal=True,
                                                                backend="fa2"))
        except Exception as exc:  # noqa: BLE001
            res["flashinfer_fa2"] = f"unavailable: {str(exc).splitlines()[0][:160]}"
        del qn, kn, vn
    except Exception as exc:  # noqa: BLE001
        res["flashinfer"] = f"unavailable: {str(exc).splitlines()[0][:160]}"
    return res


def best_dense(ours, libs):
    vals = [x for x in [ours] + list((libs or {}).values()) if isinstance(x, (int, float))]
    return min(vals) if vals else None


def run_units_timing(args, units, q, k, v, q0, kv0, dev, world, rank, reduce, gather_all):
    """A rank whose share holds split heads (query-group ranges): every step
    runs its WorkUnits through the C ABI (aa_anchor_attention_groups); the
    line reports ms/layer (max over ranks), the per-rank times and the
    imbalance.  Per-kernel metrics need a whole-head shard and are omitted."""
    import torch
    import torch.distributed as dist

    from paper_2505_23520_b200 import capi

    cfg = capi.BlockConfig(128, 128, args.step_blocks, args.theta)
    calls = []
    for u in units:
        qs = q[u.q_begin - q0:u.q_end - q0]
        ks, vs = k[u.kv_begin - kv0:u.kv_end - kv0], v[u.kv_begin - kv0:u.kv_end - kv0]
        calls.append((u, qs, ks, vs, capi.Pipeline(qs, ks, vs, cfg),
                      torch.empty((qs.shape[0], args.n, D), dtype=torch.float32, device=dev),
                      torch.empty(qs.shape[0], dtype=torch.int64, device=dev)))

    def step():
        for u, qs, ks, vs, pipe, out, comp in calls:
            pipe(qs, ks, vs, out=out, computed=comp, groups=(u.g_begin, u.g_end))

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_local = t0.elapsed_time(t1) / args.steps
    rank_ms = gather_all(ms_local)
    ms = max(rank_ms)
    comp_total = int(reduce([float(sum(int(c.sum()) for *_, c in calls))], "sum")[0])
    print(f"[bench] rank {rank}: {ms_local:.3f} ms/layer-shard over {len(units)} units", file=sys.stderr,
          flush=True)
    if rank == 0:
        causal = args.n * (args.n + 1) // 2
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": layer_config(args),
            "placement": f"balanced (query head, query group) units x{world} (sharding.shard_work)",
            "rank_ms": rank_ms, "imbalance": max(rank_ms) / (sum(rank_ms) / len(rank_ms)),
            "sparsity": 1.0 - comp_total / (args.hq * causal), "computed_positions": comp_total,
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "note": "a rank holds split heads: per-kernel metrics, e2e and the CPU baseline are "
                    "reported by whole-head shards (the default configurations)",
            "gpu_launches": sum(9 for _ in units) * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


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

    from paper_2505_23520_b200.sharding import shard_work

    def gather_all(x):
        """one host float from every rank (rank order)"""
        if world == 1:
            return [x]
        t = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(t, torch.tensor([x], dtype=torch.float64), group=host_group)
        return [float(v[0]) for v in t]

    # this rank's balanced share of the layer's (query head, query group)
    # units (sharding.shard_work): whole KV heads when they split evenly
    # (Llama 32/8 over 1/2/4/8 ranks), else query heads split by query-group
    # ranges; each KV head is generated from its own seed so the data does not
    # depend on the rank count
    G_all = geometry(args.n, args.step_blocks)["G"]
    units = shard_work(args.hq, args.hkv, rank, world, args.n, args.step_blocks)
    kv0, kv1 = min(u.kv_begin for u in units), max(u.kv_end for u in units)
    q0, q1 = min(u.q_begin for u in units), max(u.q_end for u in units)
    q, k, v = gen_layer(args.n, args.hq, args.hkv, args.seed, device=dev,
                        kv_heads=range(kv0, kv1), q_range=(q0, q1))
    if not (len(units) == 1 and (units[0].g_begin, units[0].g_end) == (0, G_all)):
        return run_units_timing(args, units, q, k, v, q0, kv0, dev, world, rank, reduce,
                                gather_all)
    rep = args.hq // args.hkv
    kv_local = kv1 - kv0
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
    rank_ms = gather_all(ms_local)
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
    dense_libs = None
    if not args.no_dense and not args.no_dense_libs:
        dense_libs = dense_library_baselines(q, k, v, barrier, reduce)
        torch.cuda.empty_cache()

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
            del pipe
        except NameError:
            pass
        torch.cuda.empty_cache()
        try:
            qn, kn, vn = (x.float().cpu().numpy() for x in (q, k, v))
            _, cpu = reference_measurement(qn, kn, vn, args, args.cpu_samples)
            del qn, kn, vn
        except Exception as exc:  # noqa: BLE001 - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": layer_config(args),
            "placement": f"whole KV heads per rank x{world} (sharding.shard_work)" if world > 1
                         else "single GPU",
            "rank_ms": rank_ms,
            "imbalance": max(rank_ms) / (sum(rank_ms) / len(rank_ms)),
            "sparsity": sparsity, "recall": recall, "computed_positions": comp_total,
            "stage_ms": dict(zip(capi.STAGES, stage_ms)),
            "kernels": kernels,
            "dense_ms_per_layer": dense_ms,
            "speedup_vs_dense": (dense_ms / ms) if dense_ms else None,
            "dense_library_ms": dense_libs,
            "dense_best_ms": best_dense(dense_ms, dense_libs),
            "speedup_vs_best_dense": (best_dense(dense_ms, dense_libs) / ms)
                                     if best_dense(dense_ms, dense_libs) else None,
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
