"""Pin the plain-C oracle restatement against the reference's own outputs.

Fixtures come from oracle/_ref (the reference library compiled from its own
sources, tests/golden/make_golden.py).  The restatement must reproduce them
exactly for index/count work and to f64 round-off for values, and must pass
the reference's known-answer tests restated here (file:line cited per test).
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle.oracle import Cfg

NAMES = golden_names()


def cfg_of(z):
    return Cfg(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_fixture(oracle, name):
    z = load_golden(name)
    cfg = cfg_of(z)
    r = oracle.anchor_attention(z["q"], z["k"], z["v"], cfg, zero_anchor=bool(z["zero_anchor"]))
    np.testing.assert_array_equal(r["counts"], z["counts"])
    np.testing.assert_array_equal(r["idx"], z["idx"])
    assert r["computed"] == int(z["computed"])
    np.testing.assert_allclose(r["m"], z["m"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r["l"], z["l"], rtol=1e-12)
    rows = z["out_rows"]
    assert np.abs(r["out"][rows] - z["out"]).max() <= 1e-6
    pooled = oracle.pooled_anchor(r["m"], cfg)
    np.testing.assert_allclose(pooled, z["pooled_anchor"], rtol=1e-13)


def test_lane_planted_exact_columns(oracle):
    """R/tests/test_stripe_identify.cpp:103-123: exactly {300, 500} per group."""
    z = load_golden("lane_planted")
    cfg = cfg_of(z)
    n = int(z["n"])
    groups = oracle.groups_from_capacity(n, cfg, z["idx"], z["counts"])
    for g, sel in enumerate(groups):
        end = oracle.middle_end_token(g, cfg, n)
        expect = [c for c in (300, 500) if cfg.b_kv <= c < end]
        assert sel == expect
    assert sum(map(len, groups)) > 0


def test_tie_at_theta_included():
    """R/tests/test_stripe_identify.cpp:146-157."""
    z = load_golden("lane_tie")
    assert 200 in z["idx"][: int(z["counts"].sum())]


def test_zero_anchor_arm():
    """R/tests/test_stripe_identify.cpp:234-248."""
    assert int(load_golden("lane_zero_anchor_real")["counts"].sum()) == 0
    z = load_golden("lane_zero_anchor_zero")
    assert 200 in z["idx"][: int(z["counts"].sum())]


def test_full_coverage_equals_dense(oracle):
    """R/tests/test_sparse_exec.cpp:32-41: theta=1e9 reproduces dense attention."""
    z = load_golden("random_full")
    dense = oracle.dense_attention(z["q"], z["k"], z["v"])
    assert np.abs(dense - z["out"]).max() <= 1e-5
    n = int(z["n"])
    assert int(z["computed"]) == n * (n + 1) // 2


def test_anchor_region_lists(oracle):
    """R/tests/test_anchor_pass.cpp:28-47."""
    assert oracle.anchor_region(0, Cfg(128, 128, 16), 4096) == [0]
    assert oracle.anchor_region(16, Cfg(128, 128, 16), 4096) == [0, 15, 16]
    assert oracle.anchor_region(2, Cfg(128, 64, 1), 4096) == [0, 3, 4, 5]
    assert oracle.anchor_region(16, Cfg(128, 128, 16), 2100) == [0, 15, 16]


@pytest.mark.parametrize("n", [129, 256, 1000, 2048])
@pytest.mark.parametrize("cfg", [Cfg(128, 128, 16), Cfg(128, 64, 1), Cfg(64, 128, 2),
                                 Cfg(32, 32, 3)])
def test_regions_tile_causal_rows(oracle, n, cfg):
    """R/tests/test_stripe_identify.cpp:191-215: init + middle + window == causal row."""
    for i in range(n):
        g = i // (cfg.step * cfg.b_q)
        wstart = oracle.window_start_token(g, cfg, n)
        mid_end = min(oracle.middle_end_token(g, cfg, n), i + 1)
        init = min(cfg.b_kv, i + 1)
        window = max(0, i + 1 - wstart)
        middle = max(0, mid_end - cfg.b_kv)
        assert init + middle + window == i + 1


def test_anchor_state_matches_restricted_softmax(oracle):
    """R/tests/test_anchor_pass.cpp:100-114 (m, l vs a one-shot softmax)."""
    rng = np.random.default_rng(35)
    n, d = 300, 8
    q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(3))
    cfg = Cfg(32, 32, 3)
    m, l, acc = oracle.compute_anchor(q, k, v, cfg)
    s = (q.astype(np.float64) @ k.astype(np.float64).T) / np.sqrt(d)
    for i in range(n):
        g = i // (cfg.step * cfg.b_q)
        ws = oracle.window_start_token(g, cfg, n)
        cols = [j for j in range(min(cfg.b_kv, i + 1))] + list(range(ws, i + 1))
        ref_m = s[i, cols].max()
        assert abs(m[i] - ref_m) <= 1e-9 * max(1.0, abs(ref_m))
        assert abs(l[i] - np.exp(s[i, cols] - ref_m).sum()) <= 1e-6 * l[i]


def test_covered_count_closed_form(oracle):
    """BASELINE/SURVEY §8 counts: covered + candidates == causal exactly."""
    for n, cov, cand in [(4096, 4720640, 3670016), (32768, 41435136, 495452160),
                         (131072, 167313408, 8422686720)]:
        cfg = Cfg(128, 128, 16, 12.0)
        assert oracle.anchor_covered_count(n, cfg) == cov
        G = oracle.group_count(n, cfg)
        rows = [min((g + 1) * 2048, n) - g * 2048 for g in range(G)]
        offs = oracle.stripe_offsets(n, cfg)
        mids = np.diff(offs)
        assert int((mids * np.array(rows)).sum()) == cand
        assert cov + cand == n * (n + 1) // 2
