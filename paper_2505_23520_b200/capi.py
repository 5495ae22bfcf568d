"""ctypes binding of the C ABI (include/anchorattn_capi.h) for device tensors.

This is the batched, device-resident entry used by bench.py and the GPU
tests: torch supplies device memory and the stream (plumbing only); every
computation runs in ``lib/libanchorattn_b200.so``.  Loading fails loudly when
the library is missing — there is no Python or CPU fallback.

Tensor layouts (head-major, contiguous): q [hq, n, d], k / v [hkv, n, d].
dtype torch.bfloat16 selects the tcgen05 path, torch.float32 the exact path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AA_LIB_PATH") or os.path.join(PKG, "lib", "libanchorattn_b200.so")

AA_F32, AA_BF16, AA_F64 = 0, 1, 2
_STATUS = {0: "AA_OK", 1: "AA_ERR_INVALID_ARGUMENT", 2: "AA_ERR_OUT_OF_RANGE",
           3: "AA_ERR_UNSUPPORTED", 4: "AA_ERR_CUDA"}


class _Cfg(C.Structure):
    _fields_ = [("b_q", C.c_int64), ("b_kv", C.c_int64), ("step", C.c_int64),
                ("theta", C.c_double)]


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int64), ("hq", C.c_int64), ("hkv", C.c_int64),
                ("cfg", _Cfg), ("dtype", C.c_int), ("q_row_stride", C.c_int64),
                ("q_head_stride", C.c_int64), ("kv_row_stride", C.c_int64),
                ("kv_head_stride", C.c_int64)]


class _Plan(C.Structure):
    _fields_ = [("q_blocks", C.c_int64), ("groups", C.c_int64), ("state_dtype", C.c_int),
                ("stripe_capacity", C.c_int64), ("covered_positions", C.c_int64),
                ("workspace_bytes", C.c_size_t)]


class AnchorAttnError(RuntimeError):
    pass


class InvalidArgument(AnchorAttnError, ValueError):
    pass


class OutOfRange(AnchorAttnError, IndexError):
    pass


_lib = None


def lib():
    """Load the native library (builds it first when sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2505_23520_b200/build.py "
                              "(anchorattn has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.aa_last_error.restype = C.c_char_p
        L.aa_version.restype = C.c_char_p
        p = C.c_void_p
        P = C.POINTER(_Problem)
        sigs = {
            "aa_make_plan": [P, C.POINTER(_Plan)],
            "aa_compute_anchor": [P, p, p, p, p, p, p, p, p, p],
            "aa_pool": [P, p, p, p, p, p, p, p],
            "aa_identify": [P, p, p, p, C.c_int, p, p, p, C.c_size_t, p],
            "aa_sparse_attention": [P, p, p, p, p, p, p, p, p, p, C.c_int64, p, C.c_int, p, p],
            "aa_finalize_anchor": [P, p, p, p, C.c_int, p],
            "aa_anchor_attention": [P, p, p, p, C.c_int, p, C.c_int, p, p, C.c_size_t, p],
            "aa_anchor_attention_groups": [P, C.c_int64, C.c_int64, p, p, p, C.c_int, p, C.c_int, p, p,
                                           C.c_size_t, p],
            "aa_anchor_attention_host": [P, p, p, p, C.c_int, p, C.c_int, p],
            "aa_dense_attention": [P, p, p, p, p, C.c_int, p],
            "aa_union_recall": [P, p, p, p, p, p, p],
            "aa_stream_sync": [p],
            "aa_set_stage_events": [C.POINTER(C.c_void_p), C.c_int],
            "aa_dense_tile_mass": [P, p, p, p, p],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        for name in ("aa_group_count", "aa_anchor_covered_count"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.c_int64, C.POINTER(_Cfg)]
        for name in ("aa_window_start_token", "aa_middle_end_token", "aa_stripe_offset"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.c_int64, C.POINTER(_Cfg), C.c_int64]
        _lib = L
    return _lib


def _check(status: int):
    if status == 0:
        return
    msg = lib().aa_last_error().decode()
    if status == 1:
        raise InvalidArgument(msg)
    if status == 2:
        raise OutOfRange(msg)
    raise AnchorAttnError(f"{_STATUS.get(status, status)}: {msg}")


@dataclass(frozen=True)
class BlockConfig:
    """BlockConfig (R/include/anchorattn/matrix.hpp:53-62), paper defaults."""

    b_q: int = 128
    b_kv: int = 128
    step: int = 16
    theta: float = 12.0

    def c(self) -> _Cfg:
        return _Cfg(self.b_q, self.b_kv, self.step, float(self.theta))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return AA_BF16
    if t.dtype == torch.float32:
        return AA_F32
    raise TypeError(f"q/k/v must be bfloat16 (fast path) or float32 (exact path), got {t.dtype}")


def make_problem(q: torch.Tensor, k: torch.Tensor, cfg: BlockConfig,
                 v: torch.Tensor | None = None) -> _Problem:
    """The C-ABI problem for q [hq, n, d] and k (and v) [hkv, n, d].

    The ABI reads v with k's strides and q's dtype, so v (when given) must
    match k in shape, strides, dtype and device, and k must share q's dtype
    and device."""
    if q.dim() != 3 or k.dim() != 3:
        raise ValueError("expected q [hq, n, d] and k/v [hkv, n, d]")
    hq, n, d = q.shape
    hkv = k.shape[0]
    if k.shape[1:] != (n, d):
        raise ValueError("q and k/v must share (n, d)")
    if q.stride(2) != 1 or k.stride(2) != 1:
        raise ValueError("head dim must be contiguous")
    if k.dtype != q.dtype:
        raise TypeError(f"q and k must share a dtype, got {q.dtype} and {k.dtype}")
    if k.device != q.device:
        raise ValueError("q and k must be on the same device")
    if v is not None:
        if v.shape != k.shape:
            raise ValueError(f"v shape {tuple(v.shape)} != k shape {tuple(k.shape)}")
        if v.dtype != k.dtype:
            raise TypeError(f"v dtype {v.dtype} != k dtype {k.dtype}")
        if v.device != k.device:
            raise ValueError("v must be on k's device")
        if v.stride() != k.stride():
            raise ValueError(f"v strides {v.stride()} != k strides {k.stride()} (the ABI reads "
                             "v with k's kv strides)")
    return _Problem(n, d, hq, hkv, cfg.c(), _dtype_code(q), q.stride(1), q.stride(0),
                    k.stride(1), k.stride(0))


def _same_layout(p: _Problem, q, k, v) -> None:
    """Re-check tensors handed to a Pipeline built for problem ``p``."""
    p2 = make_problem(q, k, BlockConfig(p.cfg.b_q, p.cfg.b_kv, p.cfg.step, p.cfg.theta), v)
    for f in ("n", "d", "hq", "hkv", "dtype", "q_row_stride", "q_head_stride", "kv_row_stride",
              "kv_head_stride"):
        if getattr(p2, f) != getattr(p, f):
            raise ValueError(f"tensors do not match the Pipeline's problem ({f}: "
                             f"{getattr(p2, f)} != {getattr(p, f)})")


def plan(p: _Problem) -> _Plan:
    pl = _Plan()
    _check(lib().aa_make_plan(C.byref(p), C.byref(pl)))
    return pl


def stripe_offsets(n: int, cfg: BlockConfig) -> list:
    c = cfg.c()
    G = lib().aa_group_count(n, C.byref(c))
    return [lib().aa_stripe_offset(g, C.byref(c), n) for g in range(G + 1)]


def _out_code(dt):
    return AA_BF16 if dt == torch.bfloat16 else AA_F32


class Pipeline:
    """Reusable device workspace for repeated calls on one problem shape."""

    def __init__(self, q, k, v, cfg: BlockConfig):
        self.cfg = cfg
        self.p = make_problem(q, k, cfg, v)
        self.plan = plan(self.p)
        self.workspace = torch.empty(self.plan.workspace_bytes, dtype=torch.uint8, device=q.device)

    def __call__(self, q, k, v, zero_anchor=False, out=None, out_dtype=torch.float32,
                 computed=None, groups=None):
        """The chain (aa_anchor_attention); ``groups=(g0, g1)`` runs only the
        query groups [g0, g1) of every head (aa_anchor_attention_groups: the
        other rows of ``out`` are left untouched)."""
        _same_layout(self.p, q, k, v)
        hq, n, d = q.shape
        if out is None:
            out = torch.empty((hq, n, d), dtype=out_dtype, device=q.device)
        elif out.shape != q.shape or not out.is_contiguous() or out.device != q.device:
            raise ValueError("out must be a contiguous [hq, n, d] tensor on q's device")
        if computed is None:
            computed = torch.empty(hq, dtype=torch.int64, device=q.device)
        if groups is None:
            _check(lib().aa_anchor_attention(C.byref(self.p), _ptr(q), _ptr(k), _ptr(v),
                                             int(zero_anchor), _ptr(out), _out_code(out.dtype),
                                             _ptr(computed), _ptr(self.workspace),
                                             self.plan.workspace_bytes, _stream()))
        else:
            _check(lib().aa_anchor_attention_groups(C.byref(self.p), int(groups[0]), int(groups[1]),
                                                    _ptr(q), _ptr(k), _ptr(v), int(zero_anchor),
                                                    _ptr(out), _out_code(out.dtype), _ptr(computed),
                                                    _ptr(self.workspace),
                                                    self.plan.workspace_bytes, _stream()))
        return out, computed


class GraphPipeline:
    """The fused chain captured once into a CUDA graph on fixed device
    buffers (q, k, v, out, computed): ``replay()`` re-runs every launch of
    aa_anchor_attention (V->f16, K1, pool, K2, compaction, K3, stats) with no
    host work per step.  Write new inputs into ``q``/``k``/``v`` in place
    between replays."""

    def __init__(self, q, k, v, cfg: BlockConfig, out_dtype=torch.float32, zero_anchor=False):
        self.q, self.k, self.v = q, k, v
        self.pipe = Pipeline(q, k, v, cfg)
        hq, n, d = q.shape
        self.out = torch.empty((hq, n, d), dtype=out_dtype, device=q.device)
        self.computed = torch.empty(hq, dtype=torch.int64, device=q.device)
        # warm-up outside the capture (one-time attributes, allocator pools)
        s = torch.cuda.Stream(device=q.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.pipe(q, k, v, zero_anchor=zero_anchor, out=self.out, computed=self.computed)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.pipe(q, k, v, zero_anchor=zero_anchor, out=self.out, computed=self.computed)

    def replay(self):
        self.graph.replay()
        return self.out, self.computed


STAGES = ("v_to_f16", "k1_anchor", "pool_k2_identify", "k3_sparse", "stats")


def set_stage_events(events):
    """Record ``events`` (6 torch.cuda.Event, or None) at the fused chain's
    stage boundaries on the next calls from this thread (aa_set_stage_events)."""
    if events is None:
        _check(lib().aa_set_stage_events(None, 0))
        return
    arr = (C.c_void_p * len(events))(*[e.cuda_event for e in events])
    set_stage_events._keep = arr  # keep alive while registered
    _check(lib().aa_set_stage_events(arr, len(events)))


def anchor_attention(q, k, v, cfg=BlockConfig(), zero_anchor=False, out_dtype=torch.float32):
    """anchor_attention (R/src/sparse_exec.cpp:126-133) over all heads.

    Returns (out [hq, n, d], computed_positions [hq] int64)."""
    return Pipeline(q, k, v, cfg)(q, k, v, zero_anchor=zero_anchor, out_dtype=out_dtype)


def compute_anchor(q, k, v, cfg=BlockConfig()):
    """Alg. 1: returns dict(m, l, acc, qsum, msum) (state f64 on the exact path)."""
    p = make_problem(q, k, cfg, v)
    pl = plan(p)
    hq, n, d = q.shape
    sdt = torch.float64 if pl.state_dtype == AA_F64 else torch.float32
    m = torch.empty((hq, n), dtype=sdt, device=q.device)
    l = torch.empty_like(m)
    acc = torch.empty((hq, n, d), dtype=sdt, device=q.device)
    qsum = torch.empty((hq, pl.q_blocks, d), dtype=torch.float32, device=q.device)
    msum = torch.empty((hq, pl.q_blocks), dtype=torch.float64, device=q.device)
    fast = p.dtype == AA_BF16
    _check(lib().aa_compute_anchor(C.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(l),
                                   _ptr(acc), _ptr(qsum) if fast else None,
                                   _ptr(msum) if fast else None, _stream()))
    return dict(m=m, l=l, acc=acc, qsum=qsum if fast else None, msum=msum if fast else None)


def pool(q, k, state, cfg=BlockConfig(), use_partials=True):
    """pooled_anchor + avgpool_rows(Q): returns (anchor [hq, G] f64, qbar [hq, G, d] f32)."""
    p = make_problem(q, k, cfg)
    pl = plan(p)
    hq, n, d = q.shape
    anchor = torch.empty((hq, pl.groups), dtype=torch.float64, device=q.device)
    qbar = torch.empty((hq, pl.groups, d), dtype=torch.float32, device=q.device)
    qsum = state.get("qsum") if use_partials else None
    msum = state.get("msum") if use_partials else None
    _check(lib().aa_pool(C.byref(p), _ptr(q), _ptr(state["m"]), _ptr(qsum), _ptr(msum),
                         _ptr(anchor), _ptr(qbar), _stream()))
    return anchor, qbar


def identify(q, k, qbar, anchor, cfg=BlockConfig(), zero_anchor=False, out=None, workspace=None):
    """Alg. 2: returns (indices [hq, capacity] u32-as-int32, counts [hq, G] int32).
    ``out=(indices, counts)`` and a ``workspace`` (uint8, >= plan.workspace_bytes)
    may be passed to keep allocations out of timed loops."""
    p = make_problem(q, k, cfg)
    pl = plan(p)
    hq = q.shape[0]
    cap = max(pl.stripe_capacity, 1)
    if out is None:
        idx = torch.zeros((hq, cap), dtype=torch.int32, device=q.device)
        counts = torch.zeros((hq, pl.groups), dtype=torch.int32, device=q.device)
    else:
        idx, counts = out
    ws = workspace if workspace is not None else None
    _check(lib().aa_identify(C.byref(p), _ptr(k), _ptr(qbar), _ptr(anchor), int(zero_anchor),
                             _ptr(idx), _ptr(counts), _ptr(ws), ws.numel() if ws is not None else 0,
                             _stream()))
    return idx, counts


def sparse(q, k, v, state, idx, counts, cfg=BlockConfig(), offsets=None, fold_chunk=64,
           out_dtype=torch.float32):
    """Alg. 3: returns (out [hq, n, d], computed [hq])."""
    p = make_problem(q, k, cfg, v)
    hq, n, d = q.shape
    out = torch.empty((hq, n, d), dtype=out_dtype, device=q.device)
    computed = torch.empty(hq, dtype=torch.int64, device=q.device)
    _check(lib().aa_sparse_attention(C.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(state["m"]),
                                     _ptr(state["l"]), _ptr(state["acc"]), _ptr(idx),
                                     _ptr(counts), _ptr(offsets), fold_chunk, _ptr(out),
                                     _out_code(out_dtype), _ptr(computed), _stream()))
    return out, computed


def finalize(q, k, state, cfg=BlockConfig(), out_dtype=torch.float32):
    p = make_problem(q, k, cfg)
    out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    _check(lib().aa_finalize_anchor(C.byref(p), _ptr(state["l"]), _ptr(state["acc"]), _ptr(out),
                                    _out_code(out_dtype), _stream()))
    return out


def dense_attention(q, k, v, out_dtype=torch.float32, out=None):
    """Dense causal attention (the baseline; exact or tcgen05 by dtype)."""
    p = make_problem(q, k, BlockConfig(), v)
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    _check(lib().aa_dense_attention(C.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                    _out_code(out.dtype), _stream()))
    return out


def union_recall(q, k, idx, counts, cfg=BlockConfig()):
    """Per-head recall of covered ∪ stripes under dense softmax (metrics.cpp:8-19)."""
    p = make_problem(q, k, cfg)
    r = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
    _check(lib().aa_union_recall(C.byref(p), _ptr(q), _ptr(k), _ptr(idx), _ptr(counts), _ptr(r),
                                 _stream()))
    return r


def dense_tile_mass(q, k, cfg=BlockConfig()):
    """Softmax mass per (query block, key block) tile, [hq, T_m, T_n] f32."""
    p = make_problem(q, k, cfg)
    hq, n, _ = q.shape
    T = (n + 127) // 128
    m = torch.zeros((hq, T, T), dtype=torch.float32, device=q.device)
    _check(lib().aa_dense_tile_mass(C.byref(p), _ptr(q), _ptr(k), _ptr(m), _stream()))
    return m


def anchor_attention_host(q, k, v, cfg=BlockConfig(), zero_anchor=False,
                          out_dtype=torch.float32, out=None, computed=None):
    """The chain on HOST (pinned) tensors through aa_anchor_attention_host."""
    p = make_problem(q, k, cfg, v)
    for t in (q, k, v):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("anchor_attention_host takes contiguous host tensors")
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, pin_memory=q.is_pinned())
    out_dtype = out.dtype
    if computed is None:
        computed = torch.empty(q.shape[0], dtype=torch.int64, pin_memory=q.is_pinned())
    _check(lib().aa_anchor_attention_host(C.byref(p), _ptr(q), _ptr(k), _ptr(v),
                                          int(zero_anchor), _ptr(out), _out_code(out_dtype),
                                          _ptr(computed)))
    return out, computed
