"""CPU-side checks of the C ABI boundary: the library loads, exports every
symbol include/anchorattn_capi.h declares, validates like the reference and
refuses to compute without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest
import torch

from conftest import ROOT
from paper_2505_23520_b200 import capi

HEADER = os.path.join(ROOT, "include", "anchorattn_capi.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(aa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name


def test_geometry_matches_oracle(oracle):
    from oracle.oracle import Cfg

    L = capi.lib()
    for n, cfg in [(4096, (128, 128, 16)), (1000, (64, 32, 3)), (777, (32, 128, 2)),
                   (131072, (128, 128, 16))]:
        c = capi._Cfg(*cfg, 12.0)
        oc = Cfg(*cfg, 12.0)
        assert L.aa_group_count(n, C.byref(c)) == oracle.group_count(n, oc)
        assert L.aa_anchor_covered_count(n, C.byref(c)) == oracle.anchor_covered_count(n, oc)
        G = oracle.group_count(n, oc)
        offs = oracle.stripe_offsets(n, oc)
        for g in range(G):
            assert L.aa_window_start_token(g, C.byref(c), n) == oracle.window_start_token(g, oc, n)
            assert L.aa_middle_end_token(g, C.byref(c), n) == oracle.middle_end_token(g, oc, n)
            assert L.aa_stripe_offset(g, C.byref(c), n) == offs[g]


def test_plan_validation_messages():
    q = torch.zeros(1, 256, 16)
    with pytest.raises(capi.InvalidArgument, match="one of b_q, b_kv must divide the other"):
        capi.plan(capi.make_problem(q, q, capi.BlockConfig(96, 64, 1, 1.0)))
    with pytest.raises(capi.InvalidArgument, match="theta must be finite"):
        capi.plan(capi.make_problem(q, q, capi.BlockConfig(64, 64, 1, float("inf"))))
    with pytest.raises(capi.InvalidArgument, match="b_q, b_kv, step must be >= 1"):
        capi.plan(capi.make_problem(q, q, capi.BlockConfig(64, 64, 0, 1.0)))
    with pytest.raises(capi.AnchorAttnError, match="requires b_q == b_kv == 128 and d == 128"):
        capi.plan(capi.make_problem(q.bfloat16(), q.bfloat16(), capi.BlockConfig(128, 128, 1)))
    pl = capi.plan(capi.make_problem(torch.zeros(32, 131072, 128, dtype=torch.bfloat16),
                                     torch.zeros(8, 131072, 128, dtype=torch.bfloat16),
                                     capi.BlockConfig()))
    assert pl.groups == 64 and pl.q_blocks == 1024
    assert pl.stripe_capacity == 4112640
    assert pl.covered_positions == 167313408


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device failure mode")
def test_no_cpu_fallback():
    q = torch.zeros(1, 256, 16)
    p = capi.make_problem(q, q, capi.BlockConfig(64, 64, 2, 1.0))
    st = capi.lib().aa_dense_attention(C.byref(p), None, None, None, None, 0, None)
    assert st == 4  # AA_ERR_CUDA
    assert "no CPU fallback" in capi.lib().aa_last_error().decode()


def test_pybind_module_surface():
    from paper_2505_23520_b200 import anchorattn as aa

    for name in ["BlockConfig", "HeadWorkload", "SelectionMask", "RunStats", "StripeIndex",
                 "anchor_attention", "identify_stripes", "union_mask", "anchor_mask",
                 "compute_anchor", "sparse_attention", "finalize_anchor", "pooled_anchor",
                 "identify_stripes_zero_anchor", "dense_attention", "union_recall"]:
        assert hasattr(aa, name), name
    cfg = aa.BlockConfig()
    assert (cfg.b_q, cfg.b_kv, cfg.step, cfg.theta) == (128, 128, 16, 12.0)
    with pytest.raises(ValueError):
        aa.BlockConfig(b_q=96, b_kv=64)
    assert aa.anchor_region(16, aa.BlockConfig(128, 128, 16), 4096) == [0, 15, 16]
    assert aa.anchor_region(2, aa.BlockConfig(128, 64, 1), 4096) == [0, 3, 4, 5]
    with pytest.raises(ValueError):
        aa.anchor_region(99, aa.BlockConfig(128, 128, 16), 256)
    mask = aa.anchor_mask(512, aa.BlockConfig(64, 32, 2))
    assert mask.total_selected() == aa.anchor_covered_count(512, aa.BlockConfig(64, 32, 2))


def test_make_problem_checks_v_and_dtypes():
    """The ABI reads v with k's strides and q's dtype: mismatches are refused
    before any call (capi.make_problem)."""
    q = torch.zeros(4, 256, 128, dtype=torch.bfloat16)
    k = torch.zeros(2, 256, 128, dtype=torch.bfloat16)
    cfg = capi.BlockConfig()
    capi.make_problem(q, k, cfg, k.clone())
    with pytest.raises(TypeError):
        capi.make_problem(q, k, cfg, k.half())
    with pytest.raises(TypeError):
        capi.make_problem(q, k.float(), cfg)
    with pytest.raises(ValueError):
        capi.make_problem(q, k, cfg, torch.zeros(2, 255, 128, dtype=torch.bfloat16))
    # same shape, different layout (a transposed view of a [n, hkv, d] buffer)
    v = torch.zeros(256, 2, 128, dtype=torch.bfloat16).transpose(0, 1)
    with pytest.raises(ValueError, match="strides"):
        capi.make_problem(q, k, cfg, v)


def test_oracle_sparse_lists_equals_capacity_layout(oracle):
    """The oracle's arbitrary-list sparse_attention (the checker of the
    unfiltered-list GPU test) equals its capacity-layout form bit for bit."""
    import numpy as np

    from oracle.oracle import Cfg
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    n, cfg = 3000, Cfg(128, 128, 4, 12.0)
    q, k, v = (x[0].float().numpy() for x in gen_sink_workload(SinkWorkloadSpec(n=n, hq=1, hkv=1, seed=4)))
    m, l, acc = oracle.compute_anchor(q, k, v, cfg)
    idx, cnt = oracle.identify(q, k, oracle.pooled_anchor(m, cfg), cfg)
    offs = oracle.stripe_offsets(n, cfg)
    lists = [idx[offs[g]:offs[g] + cnt[g]] for g in range(len(cnt))]
    a = oracle.sparse(q, k, v, cfg, m, l, acc, idx, cnt)
    b = oracle.sparse_lists(q, k, v, cfg, m, l, acc, lists)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    # and it skips what the reference skips: covered / out-of-window entries
    # change nothing, duplicates count twice
    wide = [list(x) + [0, 5, n - 1] for x in lists]
    c = oracle.sparse_lists(q, k, v, cfg, m, l, acc, wide)
    assert np.array_equal(a[0], c[0]) and a[1] == c[1]
    with pytest.raises(IndexError):
        oracle.sparse_lists(q, k, v, cfg, m, l, acc, [list(x) + [n] for x in lists])
