"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU parity oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference arm may import this module; the product path never does.

* :class:`Oracle` wraps ``oracle/liboracle.so``: the plain-C restatement of the
  reference algorithm (``oracle/anchor_oracle.c``; each function cites the
  reference file:line it restates).
* :class:`Reference` wraps ``oracle/_ref/libanchorref.so``: the UNMODIFIED
  reference library compiled from its own sources by ``make -C oracle ref``
  (only possible where ``/root/reference`` exists; the built ``.so`` travels to
  the GPU box).

Stripe indices use the capacity layout of ``include/anchorattn_capi.h``: group
``g`` owns slots ``[offset(g), offset(g) + middle_len(g))`` of which
``counts[g]`` are valid.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libanchorref.so")

_i64 = C.c_int64
_f64 = C.c_double
_p = C.c_void_p


class _Cfg(C.Structure):
    _fields_ = [("b_q", _i64), ("b_kv", _i64), ("step", _i64), ("theta", _f64)]


@dataclass(frozen=True)
class Cfg:
    """Mirror of ``BlockConfig`` (R/include/anchorattn/matrix.hpp:53-62)."""

    b_q: int = 128
    b_kv: int = 128
    step: int = 16
    theta: float = 12.0

    def c(self) -> _Cfg:
        return _Cfg(self.b_q, self.b_kv, self.step, float(self.theta))


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def build(force: bool = False) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    if os.path.isdir("/root/reference/proj/src") and (force or not os.path.exists(REF_PATH)):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, stdout=subprocess.DEVNULL)


class Oracle:
    """The plain-C restatement (f64 arithmetic over f32 inputs)."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        for name in ("ao_group_count", "ao_anchor_covered_count", "ao_stripe_capacity"):
            getattr(L, name).restype = _i64
            getattr(L, name).argtypes = [_i64, C.POINTER(_Cfg)]
        for name in ("ao_window_start_token", "ao_middle_end_token", "ao_stripe_offset"):
            getattr(L, name).restype = _i64
            getattr(L, name).argtypes = [_i64, C.POINTER(_Cfg), _i64]
        L.ao_window_start_block.restype = _i64
        L.ao_window_start_block.argtypes = [_i64, C.POINTER(_Cfg)]
        L.ao_covered_count_for_row.restype = _i64
        L.ao_covered_count_for_row.argtypes = [_i64, C.POINTER(_Cfg), _i64]
        L.ao_anchor_region.restype = _i64
        L.ao_anchor_region.argtypes = [_i64, C.POINTER(_Cfg), _i64, _p, _i64]
        L.ao_validate.restype = C.c_int
        L.ao_validate.argtypes = [C.POINTER(_Cfg)]
        L.ao_compute_anchor.argtypes = [_i64, _i64, _p, _p, _p, C.POINTER(_Cfg), _p, _p, _p]
        L.ao_avgpool_rows.argtypes = [_i64, _i64, _p, _i64, _p]
        L.ao_avgpool_vector.argtypes = [_i64, _p, _i64, _p]
        L.ao_identify.argtypes = [_i64, _i64, _p, _p, _p, C.POINTER(_Cfg), _p, _p, _p]
        L.ao_sparse_attention.restype = _i64
        L.ao_sparse_attention.argtypes = [_i64, _i64, _p, _p, _p, C.POINTER(_Cfg), _p, _p, _p,
                                          _p, _p, _i64, _p]
        L.ao_sparse_attention_lists.restype = _i64
        L.ao_sparse_attention_lists.argtypes = [_i64, _i64, _p, _p, _p, C.POINTER(_Cfg), _p, _p,
                                                _p, _p, _p, _p, _i64, _p]
        L.ao_anchor_attention.restype = _i64
        L.ao_anchor_attention.argtypes = [_i64, _i64, _p, _p, _p, C.POINTER(_Cfg), C.c_int, _p,
                                          _p, _p, _p, _p]
        L.ao_finalize.argtypes = [_i64, _i64, _p, _p, _p]
        L.ao_dense_attention.argtypes = [_i64, _i64, _p, _p, _p, _p]
        L.ao_union_recall.restype = _f64
        L.ao_union_recall.argtypes = [_i64, _i64, _p, _p, C.POINTER(_Cfg), _p, _p]

    # geometry -------------------------------------------------------------
    def validate(self, cfg: Cfg) -> bool:
        c = cfg.c()
        return self.L.ao_validate(C.byref(c)) == 0

    def group_count(self, n, cfg):
        c = cfg.c()
        return self.L.ao_group_count(n, C.byref(c))

    def window_start_token(self, g, cfg, n):
        c = cfg.c()
        return self.L.ao_window_start_token(g, C.byref(c), n)

    def middle_end_token(self, g, cfg, n):
        c = cfg.c()
        return self.L.ao_middle_end_token(g, C.byref(c), n)

    def anchor_covered_count(self, n, cfg):
        c = cfg.c()
        return self.L.ao_anchor_covered_count(n, C.byref(c))

    def stripe_capacity(self, n, cfg):
        c = cfg.c()
        return self.L.ao_stripe_capacity(n, C.byref(c))

    def stripe_offsets(self, n, cfg) -> np.ndarray:
        c = cfg.c()
        G = self.group_count(n, cfg)
        return np.array([self.L.ao_stripe_offset(g, C.byref(c), n) for g in range(G + 1)],
                        dtype=np.int64)

    def anchor_region(self, qb, cfg, n):
        c = cfg.c()
        buf = np.zeros(4096, dtype=np.int64)
        cnt = self.L.ao_anchor_region(qb, C.byref(c), n, _ptr(buf), buf.size)
        return [int(x) for x in buf[:cnt]]

    # stages ---------------------------------------------------------------
    def compute_anchor(self, q, k, v, cfg):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        m = np.empty(n, np.float64)
        l = np.empty(n, np.float64)
        acc = np.empty((n, d), np.float64)
        c = cfg.c()
        self.L.ao_compute_anchor(n, d, _ptr(q), _ptr(k), _ptr(v), C.byref(c), _ptr(m), _ptr(l),
                                 _ptr(acc))
        return m, l, acc

    def avgpool_rows(self, x, block):
        x = _f32(x)
        rows, cols = x.shape
        out = np.empty(((rows + block - 1) // block, cols), np.float32)
        self.L.ao_avgpool_rows(rows, cols, _ptr(x), block, _ptr(out))
        return out

    def avgpool_vector(self, x, block):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((x.size + block - 1) // block, np.float64)
        self.L.ao_avgpool_vector(x.size, _ptr(x), block, _ptr(out))
        return out

    def pooled_anchor(self, m, cfg):
        return self.avgpool_vector(m, cfg.step * cfg.b_q)

    def identify(self, q, k, anchor, cfg, want_margin=False):
        q, k = _f32(q), _f32(k)
        n, d = q.shape
        G = self.group_count(n, cfg)
        anchor = np.ascontiguousarray(anchor, dtype=np.float64)
        assert anchor.size == G
        cap = max(self.stripe_capacity(n, cfg), 1)
        idx = np.zeros(cap, np.uint32)
        counts = np.zeros(G, np.int64)
        margin = np.zeros(cap, np.float64) if want_margin else None
        c = cfg.c()
        self.L.ao_identify(n, d, _ptr(q), _ptr(k), _ptr(anchor), C.byref(c), _ptr(idx),
                           _ptr(counts), _ptr(margin))
        return (idx, counts, margin) if want_margin else (idx, counts)

    def sparse(self, q, k, v, cfg, m, l, acc, idx, counts, chunk=64):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        m = np.ascontiguousarray(m, np.float64)
        l = np.ascontiguousarray(l, np.float64)
        acc = np.ascontiguousarray(acc, np.float64)
        idx = np.ascontiguousarray(idx, np.uint32)
        counts = np.ascontiguousarray(counts, np.int64)
        c = cfg.c()
        computed = self.L.ao_sparse_attention(n, d, _ptr(q), _ptr(k), _ptr(v), C.byref(c),
                                              _ptr(m), _ptr(l), _ptr(acc), _ptr(idx),
                                              _ptr(counts), chunk, _ptr(out))
        if computed < 0:
            raise IndexError("sparse_attention: stripe index out of range")
        return out, int(computed)

    def sparse_lists(self, q, k, v, cfg, m, l, acc, lists, chunk=64):
        """sparse_attention over a StripeIndex given as per-group lists of any
        length and content (the reference filters them per row)."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        starts = np.zeros(len(lists), np.int64)
        counts = np.array([len(x) for x in lists], np.int64)
        if len(lists):
            starts[1:] = np.cumsum(counts)[:-1]
        flat = np.zeros(max(int(counts.sum()), 1), np.uint32)
        for s0, x in zip(starts, lists):
            flat[s0:s0 + len(x)] = np.asarray(x, dtype=np.uint64).astype(np.uint32)
        out = np.empty((n, d), np.float32)
        c = cfg.c()
        computed = self.L.ao_sparse_attention_lists(
            n, d, _ptr(q), _ptr(k), _ptr(v), C.byref(c), _ptr(np.ascontiguousarray(m, np.float64)),
            _ptr(np.ascontiguousarray(l, np.float64)), _ptr(np.ascontiguousarray(acc, np.float64)),
            _ptr(flat), _ptr(starts), _ptr(counts), chunk, _ptr(out))
        if computed < 0:
            raise IndexError("sparse_attention: stripe index out of range")
        return out, int(computed)

    def anchor_attention(self, q, k, v, cfg, zero_anchor=False):
        """Full chain. Returns dict(out, m, l, idx, counts, computed)."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        G = self.group_count(n, cfg)
        cap = max(self.stripe_capacity(n, cfg), 1)
        out = np.empty((n, d), np.float32)
        m = np.empty(n, np.float64)
        l = np.empty(n, np.float64)
        idx = np.zeros(cap, np.uint32)
        counts = np.zeros(G, np.int64)
        c = cfg.c()
        computed = self.L.ao_anchor_attention(n, d, _ptr(q), _ptr(k), _ptr(v), C.byref(c),
                                              int(zero_anchor), _ptr(out), _ptr(m), _ptr(l),
                                              _ptr(idx), _ptr(counts))
        return dict(out=out, m=m, l=l, idx=idx, counts=counts, computed=int(computed))

    def finalize(self, l, acc):
        acc = np.ascontiguousarray(acc, np.float64)
        n, d = acc.shape
        out = np.empty((n, d), np.float32)
        self.L.ao_finalize(n, d, _ptr(np.ascontiguousarray(l, np.float64)), _ptr(acc), _ptr(out))
        return out

    def dense_attention(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        self.L.ao_dense_attention(n, d, _ptr(q), _ptr(k), _ptr(v), _ptr(out))
        return out

    def union_recall(self, q, k, cfg, idx, counts):
        q, k = _f32(q), _f32(k)
        n, d = q.shape
        c = cfg.c()
        return float(self.L.ao_union_recall(n, d, _ptr(q), _ptr(k), C.byref(c),
                                            _ptr(np.ascontiguousarray(idx, np.uint32)),
                                            _ptr(np.ascontiguousarray(counts, np.int64))))

    # helpers -------------------------------------------------------------
    def groups_from_capacity(self, n, cfg, idx, counts):
        """Capacity layout -> list of per-group lists (StripeIndex.groups)."""
        offs = self.stripe_offsets(n, cfg)
        return [list(map(int, idx[offs[g]:offs[g] + counts[g]])) for g in range(len(counts))]


class Reference:
    """The reference library itself (oracle/_ref), for golden vectors and timing."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: build it with `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_pipeline.restype = C.c_int
        L.ref_pipeline.argtypes = [_i64, _i64, _p, _p, _p, _i64, _i64, _i64, _f64, C.c_int,
                                   _p, _p, _p, _p, _p, _p, _p, _p, _p]
        L.ref_layer.restype = C.c_int
        L.ref_layer.argtypes = [_i64, _i64, _i64, _i64, _p, _p, _p, _i64, _i64, _i64, _f64,
                                C.c_int, _p, _p]
        L.ref_dense_attention.restype = C.c_int
        L.ref_dense_attention.argtypes = [_i64, _i64, _p, _p, _p, _p]
        L.ref_recall.restype = C.c_int
        L.ref_recall.argtypes = [_i64, _i64, _p, _p, _p, _i64, _i64, _i64, _f64, C.c_int,
                                 C.POINTER(_f64), C.POINTER(_f64)]
        L.ref_gen_random.restype = C.c_int
        L.ref_gen_random.argtypes = [_i64, _i64, C.c_uint64, _p, _p, _p]
        L.ref_gen_sink_local.restype = C.c_int
        L.ref_gen_sink_local.argtypes = [_i64, _i64, _f64, _i64, C.c_uint64, _p, _p, _p]
        L.ref_max_threads.restype = _i64
        L.ref_layer_open.restype = _p
        L.ref_layer_open.argtypes = [_i64, _i64, _i64, _i64, _p, _p, _p, _i64, _i64, _i64, _f64]
        L.ref_layer_close.restype = None
        L.ref_layer_close.argtypes = [_p]
        L.ref_layer_anchor_identify.restype = C.c_int
        L.ref_layer_anchor_identify.argtypes = [_p, C.c_int]
        L.ref_layer_counts.restype = C.c_int
        L.ref_layer_counts.argtypes = [_p, _p]
        L.ref_layer_sparse_groups.restype = C.c_int
        L.ref_layer_sparse_groups.argtypes = [_p, _p, _p]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def pipeline(self, q, k, v, cfg: Cfg, zero_anchor=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        o = Oracle()
        G = o.group_count(n, cfg)
        cap = max(o.stripe_capacity(n, cfg), 1)
        res = dict(out=np.empty((n, d), np.float32), m=np.empty(n), l=np.empty(n),
                   acc=np.empty((n, d)), anchor_out=np.empty((n, d), np.float32),
                   pooled_anchor=np.empty(G), idx=np.zeros(cap, np.uint32),
                   counts=np.zeros(G, np.int64), computed=np.zeros(1, np.int64))
        self._check(self.L.ref_pipeline(
            n, d, _ptr(q), _ptr(k), _ptr(v), cfg.b_q, cfg.b_kv, cfg.step, float(cfg.theta),
            int(zero_anchor), _ptr(res["out"]), _ptr(res["m"]), _ptr(res["l"]), _ptr(res["acc"]),
            _ptr(res["anchor_out"]), _ptr(res["pooled_anchor"]), _ptr(res["idx"]),
            _ptr(res["counts"]), _ptr(res["computed"])))
        res["computed"] = int(res["computed"][0])
        return res

    def layer(self, q, k, v, cfg: Cfg, zero_anchor=False):
        """q [H, n, d], k/v [Hkv, n, d] -> (out [H, n, d], computed [H])."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        H, n, d = q.shape
        out = np.empty_like(q)
        computed = np.zeros(H, np.int64)
        self._check(self.L.ref_layer(H, k.shape[0], n, d, _ptr(q), _ptr(k), _ptr(v), cfg.b_q,
                                     cfg.b_kv, cfg.step, float(cfg.theta), int(zero_anchor),
                                     _ptr(out), _ptr(computed)))
        return out, computed

    def dense_attention(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        self._check(self.L.ref_dense_attention(n, d, _ptr(q), _ptr(k), _ptr(v), _ptr(out)))
        return out

    def recall(self, q, k, v, cfg: Cfg, zero_anchor=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        r, s = _f64(), _f64()
        self._check(self.L.ref_recall(n, d, _ptr(q), _ptr(k), _ptr(v), cfg.b_q, cfg.b_kv,
                                      cfg.step, float(cfg.theta), int(zero_anchor), C.byref(r),
                                      C.byref(s)))
        return r.value, s.value

    def gen_random(self, n, d, seed):
        q, k, v = (np.empty((n, d), np.float32) for _ in range(3))
        self._check(self.L.ref_gen_random(n, d, seed, _ptr(q), _ptr(k), _ptr(v)))
        return q, k, v

    def gen_sink_local(self, n, d, sink_strength, window, seed):
        q, k, v = (np.empty((n, d), np.float32) for _ in range(3))
        self._check(self.L.ref_gen_sink_local(n, d, sink_strength, window, seed, _ptr(q),
                                              _ptr(k), _ptr(v)))
        return q, k, v

    def max_threads(self) -> int:
        return int(self.L.ref_max_threads())

    def open_layer(self, q, k, v, cfg: Cfg) -> "RefLayer":
        return RefLayer(self, q, k, v, cfg)


class RefLayer:
    """A GQA layer (q [H, n, d], k/v [Hkv, n, d]) resident in the reference's
    own types, for stage-by-stage timing (oracle/ref_driver.cpp ref_layer_*)."""

    def __init__(self, ref: Reference, q, k, v, cfg: Cfg):
        self.ref = ref
        q, k, v = _f32(q), _f32(k), _f32(v)
        self.H, self.n, self.d = q.shape
        self.cfg = cfg
        self.h = ref.L.ref_layer_open(self.H, k.shape[0], self.n, self.d, _ptr(q), _ptr(k), _ptr(v),
                                      cfg.b_q, cfg.b_kv, cfg.step, float(cfg.theta))
        if not self.h:
            raise RuntimeError(ref.L.ref_last_error().decode())

    def close(self):
        if self.h:
            self.ref.L.ref_layer_close(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def anchor_identify(self, zero_anchor=False):
        """compute_anchor + identify_stripes on every head (parallel_for)."""
        self.ref._check(self.ref.L.ref_layer_anchor_identify(self.h, int(zero_anchor)))

    def counts(self, groups: int) -> np.ndarray:
        c = np.zeros((self.H, groups), np.int64)
        self.ref.L.ref_layer_counts(self.h, _ptr(c))
        return c

    def sparse_groups(self, group_of_head) -> np.ndarray:
        """sparse_attention per head keeping only group group_of_head[h] of its
        StripeIndex (-1: all groups, -2: none, -3: head left out of the pass).
        Returns computed positions."""
        g = np.ascontiguousarray(group_of_head, np.int64)
        out = np.zeros(self.H, np.int64)
        self.ref._check(self.ref.L.ref_layer_sparse_groups(self.h, _ptr(g), _ptr(out)))
        return out
