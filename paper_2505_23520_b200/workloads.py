"""Scalable synthetic prefill workloads (O(N*d), no dense verification pass).

The reference's generators verify their structure with an O(N^2) dense score
map (``gen_sink_local``, R/src/workloads.cpp:116-196, checks argmax
concentration with ``dense_scores``), which is infeasible at 128k tokens.
This module builds the same *shape* of head directly:

* one shared scale direction ``u`` per KV head; query row ``i`` carries
  ``sink_mult(band(i)) * u`` with ``sink_mult`` in [0.7, 1.3] per 256-row band
  (workloads.cpp:133-143, 152-155);
* key ``j`` carries ``(a - depth_j) * sqrt(d) * u`` (workloads.cpp:172-183):
  the sink column has depth 0, ``N/32`` spread "strong" columns sit at depth
  U(3, 7.8) and the remaining columns are buried at depths drawn from a
  piecewise-linear CDF (``_DEEP_CDF``) calibrated so that the selected
  fraction at theta = 10..15 follows the paper's Table 6 sparsities
  (R/../PAPER.md:443-448: 97/93/89/81/72/61 %);
* a near-diagonal boost through a per-token "personality" direction shared by
  the KV head and all its query heads (the GQA analogue of the residual boost,
  workloads.cpp:185-190), gain ``min(0.3*sqrt(d), a/4)``;
* N(0, 0.015^2) noise on q/k, N(0, 1) values; everything rounded to bf16.

Scores are therefore ``s(i, j) ~= sink_mult_i * (a - depth_j)`` and the
difference-aware test ``anchor - s <= theta`` keeps columns with
``depth <~ theta``: theta sweeps move sparsity the way the paper's Table 6
does (recall on these synthetic heads is higher than on real LLM heads
because the strong columns carry most of the off-anchor mass).

Layout: head-major ``q [Hq, N, d]``, ``k, v [Hkv, N, d]``, bf16.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class SinkWorkloadSpec:
    n: int
    d: int = 128
    hq: int = 32
    hkv: int = 8
    sink_strength: float = 12.0
    seed: int = 0


def _unit_rows(x: torch.Tensor) -> torch.Tensor:
    return x / x.norm(dim=-1, keepdim=True).clamp_min(1e-12)


# (depth, CDF) knots for the buried columns: F(theta) ~ (selected fraction at
# theta - 3.1% strong columns) / 96.9% for the paper's Table 6 operating points.
_DEEP_CDF = ((10.0, 0.0), (11.0, 0.04), (12.0, 0.085), (13.0, 0.165), (14.0, 0.26),
             (15.0, 0.37), (16.0, 0.48), (20.0, 0.8), (30.0, 1.0))


def _sample_deep(u: torch.Tensor) -> torch.Tensor:
    """Inverse-CDF sample of buried-column depths from uniforms ``u``."""
    xs = torch.tensor([c for _, c in _DEEP_CDF], device=u.device, dtype=u.dtype)
    ys = torch.tensor([dpt for dpt, _ in _DEEP_CDF], device=u.device, dtype=u.dtype)
    i = torch.searchsorted(xs, u.contiguous()).clamp(1, len(_DEEP_CDF) - 1)
    x0, x1, y0, y1 = xs[i - 1], xs[i], ys[i - 1], ys[i]
    return y0 + (u - x0) / (x1 - x0) * (y1 - y0)


def gen_sink_workload(spec: SinkWorkloadSpec, device="cpu", dtype=torch.bfloat16):
    """Returns (q [Hq,N,d], k [Hkv,N,d], v [Hkv,N,d]) in ``dtype``.

    Deterministic for a given (spec, device type): CPU generation is used for
    parity fixtures, CUDA generation for full-size benchmarks.
    """
    n, d, hq, hkv = spec.n, spec.d, spec.hq, spec.hkv
    if hq % hkv:
        raise ValueError("hq must be a multiple of hkv")
    g = torch.Generator(device=device)
    g.manual_seed(spec.seed)
    f32 = torch.float32
    sqrt_d = math.sqrt(d)
    a = spec.sink_strength
    noise = 0.015
    rep = hq // hkv

    # Per KV head: scale direction u, personalities p_j orthogonal to u.
    u = _unit_rows(torch.randn(hkv, 1, d, generator=g, device=device, dtype=f32))
    pers = torch.randn(hkv, n, d, generator=g, device=device, dtype=f32)
    pers = _unit_rows(pers - (pers * u).sum(-1, keepdim=True) * u)

    # Key depths: sink (j=0) at 0, N/32 strong columns spread over
    # [192, 7N/8) (workloads.cpp:158-167), the rest buried.
    depth = _sample_deep(torch.rand(hkv, n, generator=g, device=device, dtype=f32))
    if n >= 512:
        n_strong = n // 32
        lo, hi = 192, (n * 7) // 8
        cols = lo + ((hi - lo) * torch.arange(n_strong, device=device, dtype=torch.int64)) // n_strong
        depth[:, cols] = 3.0 + 4.8 * torch.rand(hkv, n_strong, generator=g, device=device,
                                                dtype=f32)
    depth[:, 0] = 0.0
    local_gain = min(0.3 * sqrt_d, a / 4.0)

    k = noise * torch.randn(hkv, n, d, generator=g, device=device, dtype=f32)
    k += ((a - depth) * sqrt_d).unsqueeze(-1) * u
    # personality boost: q_i . k_j picks up gain*sqrt(d)*(p_i.p_j) -> +gain on the diagonal
    k[:, 1:] += local_gain * pers[:, 1:]
    v = torch.randn(hkv, n, d, generator=g, device=device, dtype=f32)

    n_bands = (n + 255) // 256
    sink_mult = 0.7 + 0.6 * torch.rand(hq, n_bands, generator=g, device=device, dtype=f32)
    sm_rows = sink_mult.repeat_interleave(256, dim=1)[:, :n]  # [hq, n]
    q = noise * torch.randn(hq, n, d, generator=g, device=device, dtype=f32)
    u_q = u.repeat_interleave(rep, dim=0)
    q += sm_rows.unsqueeze(-1) * u_q
    q += sqrt_d * pers.repeat_interleave(rep, dim=0)
    return q.to(dtype), k.to(dtype), v.to(dtype)


def gen_random_workload(n, d=128, hq=1, hkv=1, seed=0, device="cpu", dtype=torch.bfloat16):
    """Unit Gaussian heads (the shape of gen_random, R/src/workloads.cpp:98-114)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = torch.randn(hq, n, d, generator=g, device=device)
    k = torch.randn(hkv, n, d, generator=g, device=device)
    v = torch.randn(hkv, n, d, generator=g, device=device)
    return q.to(dtype), k.to(dtype), v.to(dtype)
