"""GPU parity of the EXACT path (f32 in, f64 state) through the reference-named
pybind module and the C ABI, against the reference's own outputs (golden
fixtures from oracle/_ref) and the restated reference unit tests.

The exact path mirrors the reference's operation order, so selection sets and
computed-position counts are identical and values agree to f64 round-off.
"""
import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aa():
    from paper_2505_23520_b200 import anchorattn

    anchorattn.set_precision(anchorattn.Precision.Exact)
    return anchorattn


def cfg_of(aa, z):
    return aa.BlockConfig(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))


def lists(z, oracle):
    from oracle.oracle import Cfg

    c = Cfg(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))
    return oracle.groups_from_capacity(int(z["n"]), c, z["idx"], z["counts"])


@pytest.mark.parametrize("name", golden_names())
def test_pipeline_matches_reference(aa, oracle, name):
    z = load_golden(name)
    w = aa.HeadWorkload(z["q"], z["k"], z["v"])
    cfg = cfg_of(aa, z)
    out, stats = aa.anchor_attention(w, cfg, bool(z["zero_anchor"]))
    rows = z["out_rows"]
    assert np.abs(out[rows] - z["out"]).max() <= 1e-6
    assert stats.computed_positions == int(z["computed"])
    n = int(z["n"])
    assert stats.causal_positions == n * (n + 1) // 2

    st = aa.compute_anchor(w, cfg)
    np.testing.assert_allclose(st.m, z["m"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st.l, z["l"], rtol=1e-11)
    np.testing.assert_allclose(aa.pooled_anchor(st, cfg), z["pooled_anchor"], rtol=1e-12)
    fin = aa.finalize_anchor(st)
    assert np.abs(fin[rows] - z["anchor_out"]).max() <= 1e-6
    if bool(z["zero_anchor"]):
        idx = aa.identify_stripes_zero_anchor(w, cfg)
    else:
        idx = aa.identify_stripes_from_state(w, st, cfg)
    assert idx.groups == lists(z, oracle)


def test_fold_plans_do_not_change_result(aa):
    """R/tests/test_sparse_exec.cpp:74-89."""
    z = load_golden("random_theta4")
    w = aa.HeadWorkload(z["q"], z["k"], z["v"])
    cfg = cfg_of(aa, z)
    st = aa.compute_anchor(w, cfg)
    idx = aa.identify_stripes_from_state(w, st, cfg)
    assert idx.total_selected() > 0
    base, bstats = aa.sparse_attention(w, st, idx, cfg)
    for chunk, seed in [(1, 0), (7, 1), (64, 2), (1000, 3), (13, 99), (5000, 4), (10**6, 5)]:
        alt, astats = aa.sparse_attention(w, st, idx, cfg, aa.FoldPlan(chunk, seed))
        assert np.abs(base - alt).max() <= 1e-6
        assert astats.computed_positions == bstats.computed_positions
    # chunks longer than the kernel's score staging (4096) fold in two passes
    # with the same scores in the same order: bit-identical to one staged chunk
    longest = max(len(g) for g in idx.groups)
    assert longest <= 4096
    staged, _ = aa.sparse_attention(w, st, idx, cfg, aa.FoldPlan(4096, 0))
    for chunk in (4097, 10**6):
        two_pass, _ = aa.sparse_attention(w, st, idx, cfg, aa.FoldPlan(chunk, 0))
        assert np.array_equal(staged, two_pass), chunk


def test_covered_stripes_are_skipped(aa, oracle):
    """R/tests/test_sparse_exec.cpp:123-144: {200, 300} in group 3 -> only 200 folds."""
    rng = np.random.default_rng(77)
    n, d = 512, 8
    q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(3))
    w = aa.HeadWorkload(q, k, v)
    cfg = aa.BlockConfig(128, 128, 1, 12.0)
    st = aa.compute_anchor(w, cfg)
    groups = [[] for _ in range(aa.group_count(n, cfg))]
    groups[3] = [200, 300]
    idx = aa.StripeIndex(n, cfg, groups)
    out, stats = aa.sparse_attention(w, st, idx, cfg)
    assert stats.computed_positions == aa.anchor_covered_count(n, cfg) + 128
    mask = aa.union_mask(idx, cfg, n)
    assert stats.computed_positions == mask.total_selected()


def test_error_paths(aa):
    """R/tests/test_sparse_exec.cpp:170-190."""
    rng = np.random.default_rng(78)
    q, k, v = (rng.standard_normal((256, 4)).astype(np.float32) for _ in range(3))
    w = aa.HeadWorkload(q, k, v)
    small, big = aa.BlockConfig(32, 32, 2, 12.0), aa.BlockConfig(64, 64, 2, 12.0)
    st = aa.compute_anchor(w, small)
    with pytest.raises(ValueError, match="another blocking"):
        aa.identify_stripes_from_state(w, st, big)
    idx = aa.identify_stripes_from_state(w, st, small)
    with pytest.raises(ValueError, match="another blocking"):
        aa.sparse_attention(w, st, idx, big)
    cfg = aa.BlockConfig(64, 64, 1, 12.0)
    st = aa.compute_anchor(w, cfg)
    groups = [[] for _ in range(aa.group_count(256, cfg))]
    groups[2] = [9999]
    with pytest.raises(IndexError, match="stripe index 9999 out of range"):
        aa.sparse_attention(w, st, aa.StripeIndex(256, cfg, groups), cfg)
    with pytest.raises(ValueError, match="index_chunk must be >= 1"):
        aa.sparse_attention(w, st, aa.StripeIndex(256, cfg, [[]] * 4), cfg, aa.FoldPlan(0, 0))


def test_empty_index_equals_finalized_anchor(aa):
    """R/tests/test_sparse_exec.cpp:43-55."""
    rng = np.random.default_rng(72)
    q, k, v = (rng.standard_normal((400, 8)).astype(np.float32) for _ in range(3))
    w = aa.HeadWorkload(q, k, v)
    cfg = aa.BlockConfig(64, 64, 2, -1e9)
    st = aa.compute_anchor(w, cfg)
    idx = aa.identify_stripes_from_state(w, st, cfg)
    assert idx.total_selected() == 0
    out, stats = aa.sparse_attention(w, st, idx, cfg)
    assert np.abs(out - aa.finalize_anchor(st)).max() <= 1e-12
    assert stats.computed_positions == aa.anchor_covered_count(400, cfg)


def test_determinism(aa):
    """R/tests/test_sparse_exec.cpp:192-199 (bitwise)."""
    z = load_golden("sink_theta12")
    w = aa.HeadWorkload(z["q"], z["k"], z["v"])
    a, sa = aa.anchor_attention(w, cfg_of(aa, z))
    b, sb = aa.anchor_attention(w, cfg_of(aa, z))
    assert np.array_equal(a, b) and sa.computed_positions == sb.computed_positions


def test_dense_and_recall_match_oracle(aa, oracle):
    from oracle.oracle import Cfg

    z = load_golden("sink_theta10")
    w = aa.HeadWorkload(z["q"], z["k"], z["v"])
    dense = aa.dense_attention(w)
    assert np.abs(dense - oracle.dense_attention(z["q"], z["k"], z["v"])).max() <= 1e-6
    cfg = cfg_of(aa, z)
    idx = aa.identify_stripes(w, cfg)
    r = aa.union_recall(w, idx, cfg)
    assert abs(r - float(z["recall"])) <= 1e-9


def test_capi_multihead_gqa_exact(oracle):
    """4 query heads over 2 KV heads through the C ABI, each head vs the oracle."""
    from oracle.oracle import Cfg
    from paper_2505_23520_b200 import capi

    rng = np.random.default_rng(5)
    n, d = 600, 16
    q = rng.standard_normal((4, n, d)).astype(np.float32)
    k = rng.standard_normal((2, n, d)).astype(np.float32)
    v = rng.standard_normal((2, n, d)).astype(np.float32)
    cfg = capi.BlockConfig(64, 64, 2, 3.0)
    out, computed = capi.anchor_attention(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                          torch.from_numpy(v).cuda(), cfg)
    out = out.cpu().numpy()
    for h in range(4):
        r = oracle.anchor_attention(q[h], k[h // 2], v[h // 2], Cfg(64, 64, 2, 3.0))
        assert np.abs(out[h] - r["out"]).max() <= 1e-6
        assert int(computed[h]) == r["computed"]
