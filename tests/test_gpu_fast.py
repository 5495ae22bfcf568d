"""GPU parity of the tcgen05 fast path (bf16 Q/K/V, b = 128, d = 128) against
the CPU oracle on identical bf16-rounded inputs, with the north-star
tolerances (BASELINE.json north_star):

* stripe sets identical except keys whose oracle margin |anchor - s - theta|
  is within 1e-3 (BAND);
* attention output: max-abs <= 2e-2 and relative L2 <= 1e-3 (O in f32);
* anchor state m and l within 1e-5 relative;
* computed_positions exact whenever the selected sets agree.
"""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle.oracle import Cfg

pytestmark = pytest.mark.gpu

BAND = 1e-3
MAX_ABS = 2e-2
REL_L2 = 1e-3


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def assert_out_close(got, ref, what=""):
    err = np.abs(got - ref).max()
    rel = rel_l2(got, ref)
    assert err <= MAX_ABS and rel <= REL_L2, f"{what}: max-abs {err:.3e} rel-l2 {rel:.3e}"


def gen(n, hq=1, hkv=1, seed=0):
    from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload

    return gen_sink_workload(SinkWorkloadSpec(n=n, hq=hq, hkv=hkv, seed=seed))


def capi():
    from paper_2505_23520_b200 import capi as c

    return c


def band_equal(oracle, q, k, cfg, m_gpu_anchor_src, idx_gpu, counts_gpu):
    """Selection sets equal outside the +-BAND margin (oracle margins)."""
    n = q.shape[0]
    m_o, _, _ = oracle.compute_anchor(q, k, np.zeros_like(q), cfg)
    anchor = oracle.pooled_anchor(m_o, cfg)
    idx_o, cnt_o, margin = oracle.identify(q, k, anchor, cfg, want_margin=True)
    offs = oracle.stripe_offsets(n, cfg)
    same = True
    for g in range(len(cnt_o)):
        a = set(idx_o[offs[g]:offs[g] + cnt_o[g]].tolist())
        b = set(idx_gpu[offs[g]:offs[g] + counts_gpu[g]].tolist())
        for j in a ^ b:
            same = False
            assert abs(margin[offs[g] + j - cfg.b_kv]) <= BAND, (g, j, margin[offs[g] + j - cfg.b_kv])
    return same


@pytest.mark.parametrize("n,step", [(4096, 16), (2048, 2), (4000, 4), (640, 1), (130, 16)])
def test_anchor_pass_matches_oracle(oracle, n, step):
    c = capi()
    q, k, v = gen(n, seed=n + step)
    cfg = c.BlockConfig(128, 128, step, 12.0)
    st = c.compute_anchor(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    qn, kn, vn = (x[0].float().numpy() for x in (q, k, v))
    m, l, acc = oracle.compute_anchor(qn, kn, vn, Cfg(128, 128, step, 12.0))
    mg = st["m"][0].double().cpu().numpy()
    assert np.max(np.abs(mg - m) / np.maximum(np.abs(m), 1.0)) <= 1e-5
    lg = st["l"][0].double().cpu().numpy()
    assert np.max(np.abs(lg - l) / l) <= 1e-5
    fin = (st["acc"][0] / st["l"][0, :, None]).cpu().numpy()
    assert_out_close(fin, oracle.finalize(l, acc), "finalize_anchor")
    # pooled partials -> anchor / qbar
    anchor, qbar = c.pool(q.cuda(), k.cuda(), st, cfg)
    ref_anchor = oracle.pooled_anchor(m, Cfg(128, 128, step, 12.0))
    assert np.max(np.abs(anchor[0].cpu().numpy() - ref_anchor)) <= 1e-4
    ref_qbar = oracle.avgpool_rows(qn, step * 128)
    assert np.max(np.abs(qbar[0].cpu().numpy() - ref_qbar)) <= 1e-5


@pytest.mark.parametrize("n,step,theta", [(4096, 16, 12.0), (2048, 2, 12.0), (4000, 4, 13.0),
                                          (8192, 16, 10.0), (1100, 1, 14.0),
                                          # ragged last groups (K3 clusters with gather-only pairs)
                                          (5000, 16, 12.0), (6444, 16, 11.0), (2300, 2, 12.0)])
def test_pipeline_matches_oracle(oracle, n, step, theta):
    c = capi()
    q, k, v = gen(n, seed=7 * n + step)
    cfg = c.BlockConfig(128, 128, step, theta)
    out, computed = c.anchor_attention(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    qn, kn, vn = (x[0].float().numpy() for x in (q, k, v))
    ocfg = Cfg(128, 128, step, theta)
    r = oracle.anchor_attention(qn, kn, vn, ocfg)
    assert_out_close(out[0].cpu().numpy(), r["out"], f"n={n}")
    # selection: recompute the GPU stripe lists through the stage API
    st = c.compute_anchor(q.cuda(), k.cuda(), v.cuda(), cfg)
    anchor, qbar = c.pool(q.cuda(), k.cuda(), st, cfg)
    idx, counts = c.identify(q.cuda(), k.cuda(), qbar, anchor, cfg)
    idx = idx[0].cpu().numpy().view(np.uint32)
    counts = counts[0].cpu().numpy()
    same = band_equal(oracle, qn, kn, ocfg, None, idx, counts)
    if same:
        assert int(computed[0]) == r["computed"]


def test_golden_fixtures_bf16():
    """The reference's own outputs (oracle/_ref fixtures) on bf16 inputs."""
    c = capi()
    for name in ("bf16_c1", "bf16_multigroup"):
        z = load_golden(name)
        q, k, v = (torch.from_numpy(z[x]).bfloat16()[None].cuda() for x in ("q", "k", "v"))
        cfg = c.BlockConfig(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))
        out, computed = c.anchor_attention(q, k, v, cfg)
        got = out[0].cpu().numpy()[z["out_rows"]]
        assert_out_close(got, z["out"], name)
        assert int(computed[0]) == int(z["computed"]), name


@pytest.mark.parametrize("hq,hkv,heads", [(8, 2, (1, 6)), (28, 4, (0, 13, 27))])
def test_gqa_multihead_and_sharded_heads(oracle, hq, hkv, heads):
    """GQA through the fused chain (Llama-like 4:1 and Qwen2.5-like 7:1
    ratios); spot-check heads of different KV groups against the oracle."""
    c = capi()
    n = 4096
    rep = hq // hkv
    q, k, v = gen(n, hq=hq, hkv=hkv, seed=21 + hq)
    cfg = c.BlockConfig()
    out, computed = c.anchor_attention(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    for h in heads:
        r = oracle.anchor_attention(q[h].float().numpy(), k[h // rep].float().numpy(),
                                    v[h // rep].float().numpy(), Cfg())
        assert_out_close(out[h].cpu().numpy(), r["out"], f"head {h}")


def test_dense_matches_oracle(oracle):
    c = capi()
    n = 2048 + 77
    q, k, v = gen(n, seed=5)
    out = c.dense_attention(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    ref = oracle.dense_attention(*(x[0].float().numpy() for x in (q, k, v)))
    assert_out_close(out[0].cpu().numpy(), ref, "dense")
    # random (diffuse) heads too
    from paper_2505_23520_b200.workloads import gen_random_workload

    q, k, v = gen_random_workload(1024, seed=9)
    out = c.dense_attention(q.cuda(), k.cuda(), v.cuda())
    ref = oracle.dense_attention(*(x[0].float().numpy() for x in (q, k, v)))
    assert_out_close(out[0].cpu().numpy(), ref, "dense-random")


def test_theta_extremes_at_32k():
    """Size-independent properties at 32k (Llama GQA shape, 4 query heads):
    theta = +1e9 reproduces dense attention with computed == causal;
    theta = -1e9 reproduces the finalized anchor state."""
    c = capi()
    n = 32768
    q, k, v = gen(n, hq=4, hkv=1, seed=2)
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    full, comp = c.anchor_attention(q, k, v, c.BlockConfig(theta=1e9))
    dense = c.dense_attention(q, k, v)
    torch.cuda.synchronize()
    assert int(comp.min()) == n * (n + 1) // 2 == int(comp.max())
    assert_out_close(full.cpu().numpy(), dense.cpu().numpy(), "theta=+1e9 vs dense")
    none, comp = c.anchor_attention(q, k, v, c.BlockConfig(theta=-1e9))
    st = c.compute_anchor(q, k, v, c.BlockConfig())
    fin = c.finalize(q, k, st, c.BlockConfig())
    torch.cuda.synchronize()
    pl = c.plan(c.make_problem(q, k, c.BlockConfig()))
    assert int(comp.max()) == pl.covered_positions
    # the fused chain hands the anchor state to K3 as f16 acc / l (f16 carries
    # 11 significant bits: relative rounding <= 2^-11)
    assert torch.allclose(none, fin, atol=1e-5, rtol=2 ** -10)


def test_selection_monotone_in_theta():
    """R/tests/test_stripe_identify.cpp:125-144 at 16k on the fast path."""
    c = capi()
    n = 16384
    q, k, v = gen(n, hq=2, hkv=1, seed=4)
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    cfg = c.BlockConfig()
    st = c.compute_anchor(q, k, v, cfg)
    anchor, qbar = c.pool(q, k, st, cfg)
    prev = None
    offs = c.stripe_offsets(n, cfg)
    for theta in (8.0, 10.0, 12.0, 14.0, 16.0):
        idx, counts = c.identify(q, k, qbar, anchor, c.BlockConfig(theta=theta))
        idx, counts = idx.cpu().numpy(), counts.cpu().numpy()
        if prev is not None:
            pidx, pcounts = prev
            assert (counts >= pcounts).all()
            for h in range(2):
                for g in range(len(offs) - 1):
                    a = set(pidx[h, offs[g]:offs[g] + pcounts[h, g]].tolist())
                    b = set(idx[h, offs[g]:offs[g] + counts[h, g]].tolist())
                    assert a <= b
        prev = (idx, counts)


def test_stage_api_equals_fused_chain():
    c = capi()
    n = 8192
    q, k, v = gen(n, hq=2, hkv=1, seed=8)
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    cfg = c.BlockConfig()
    fused, comp = c.anchor_attention(q, k, v, cfg)
    st = c.compute_anchor(q, k, v, cfg)
    anchor, qbar = c.pool(q, k, st, cfg)
    idx, counts = c.identify(q, k, qbar, anchor, cfg)
    out, comp2 = c.sparse(q, k, v, st, idx, counts, cfg)
    torch.cuda.synchronize()
    assert torch.equal(comp, comp2)
    # the fused chain hands K1's state to K3 as f16 acc / l (half the bytes);
    # the stage API keeps AnchorState's f32 acc: same selection, outputs equal
    # to f16 rounding of the anchor part
    err = (fused - out).abs().max().item()
    rel = ((fused - out).norm() / out.norm()).item()
    assert err <= 5e-3 and rel <= 3e-4, (err, rel)


@pytest.mark.parametrize("n,step,theta", [(4096, 16, 12.0), (2048, 2, 10.0), (3000, 4, 14.0)])
def test_recall_pass_matches_oracle(oracle, n, step, theta):
    """GPU recall (one dense QK pass keeping total and selected softmax mass per
    row) == recall(union_mask(stripes), dense_probs) on the same stripe lists."""
    c = capi()
    q, k, v = gen(n, hq=2, hkv=1, seed=31 + n)
    dq, dk, dv = q.cuda(), k.cuda(), v.cuda()
    cfg = c.BlockConfig(128, 128, step, theta)
    st = c.compute_anchor(dq, dk, dv, cfg)
    anchor, qbar = c.pool(dq, dk, st, cfg)
    idx, counts = c.identify(dq, dk, qbar, anchor, cfg)
    rec = c.union_recall(dq, dk, idx, counts, cfg).cpu().numpy()
    ocfg = Cfg(128, 128, step, theta)
    for h in range(2):
        ref = oracle.union_recall(q[h].float().numpy(), k[0].float().numpy(), ocfg,
                                  idx[h].cpu().numpy().view(np.uint32),
                                  counts[h].cpu().numpy().astype(np.int64))
        assert abs(rec[h] - ref) <= 1e-4, (h, rec[h], ref)


@pytest.mark.parametrize("n", [1024, 1100])
def test_dense_tile_mass_matches_softmax(n):
    """Two-pass TILEMASS map == tile sums of the f64 causal softmax (numpy)."""
    c = capi()
    q, k, v = gen(n, hq=2, hkv=1, seed=5 + n)
    mass = c.dense_tile_mass(q.cuda(), k.cuda()).cpu().numpy()
    T = (n + 127) // 128
    for h in range(2):
        qh = q[h].double().numpy()
        kh = k[0].double().numpy()
        s = qh @ kh.T / np.sqrt(128.0)
        s[np.triu_indices(n, 1)] = -np.inf
        p = np.exp(s - s.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        ref = np.zeros((T, T))
        for a in range(T):
            for b in range(T):
                ref[a, b] = p[a * 128:(a + 1) * 128, b * 128:(b + 1) * 128].sum()
        assert np.abs(mass[h] - ref).max() <= 2e-4
        assert abs(mass[h].sum() - n) <= 1e-2 * n / 1000


@pytest.mark.parametrize("hq,hkv,pinned", [(8, 2, True), (36, 12, True), (4, 4, False), (7, 1, True),
                                           (66, 33, True)])
def test_host_entry_pipelined_equals_device_chain(hq, hkv, pinned):
    """aa_anchor_attention_host (KV-head chunks pipelined over three streams)
    returns exactly the device chain's output and per-head computed counts —
    including head counts that do not split evenly into chunks and pageable
    host buffers."""
    c = capi()
    n = 2048
    q, k, v = gen(n, hq=hq, hkv=hkv, seed=hq + hkv)
    cfg = c.BlockConfig()
    ref, comp = c.anchor_attention(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    if pinned:
        q, k, v = q.pin_memory(), k.pin_memory(), v.pin_memory()
    out, comp_h = c.anchor_attention_host(q, k, v, cfg)
    assert torch.equal(out, ref.cpu())
    assert torch.equal(comp_h, comp.cpu())
    out16, _ = c.anchor_attention_host(q, k, v, cfg, out_dtype=torch.bfloat16)
    assert torch.equal(out16.float(), ref.cpu().bfloat16().float())


def test_graph_replay_equals_eager():
    """The fused chain captured in a CUDA graph (capi.GraphPipeline) replays
    the eager result exactly, also after the inputs are rewritten in place."""
    c = capi()
    n = 8192
    q, k, v = (x.cuda() for x in gen(n, hq=4, hkv=1, seed=31))
    cfg = c.BlockConfig()
    g = c.GraphPipeline(q, k, v, cfg)
    out, comp = g.replay()
    torch.cuda.synchronize()
    ref, ref_comp = c.anchor_attention(q, k, v, cfg)
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(comp, ref_comp)
    q2, k2, v2 = (x.cuda() for x in gen(n, hq=4, hkv=1, seed=32))
    g.q.copy_(q2), g.k.copy_(k2), g.v.copy_(v2)
    out, comp = g.replay()
    torch.cuda.synchronize()
    ref, ref_comp = c.anchor_attention(q2, k2, v2, cfg)
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(comp, ref_comp)


@pytest.mark.parametrize("hq,step", [(12, 2), (7, 4), (3, 16)])
def test_identify_mtile_pairs_all_heads(oracle, hq, step):
    """K2 assigns one CTA per (KV head, pair of 128-row M-tiles of (group,
    head) rows): 12 heads x 32 groups (step 2) = 3 M-tiles (an odd pair), 7
    heads x 16 groups = 1 M-tile, 3 heads x 4 groups.  Every head's stripe
    sets match the oracle outside the +-1e-3 band, and the fused chain's
    outputs match the oracle for every head."""
    c = capi()
    n = 8192
    q, k, v = gen(n, hq=hq, hkv=1, seed=100 + hq)
    cfg = c.BlockConfig(128, 128, step, 12.0)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    st = c.compute_anchor(qd, kd, vd, cfg)
    anchor, qbar = c.pool(qd, kd, st, cfg)
    idx, counts = c.identify(qd, kd, qbar, anchor, cfg)
    out, computed = c.anchor_attention(qd, kd, vd, cfg)
    torch.cuda.synchronize()
    ocfg = Cfg(128, 128, step, 12.0)
    kn, vn = k[0].float().numpy(), v[0].float().numpy()
    idx = idx.cpu().numpy().view(np.uint32)
    counts = counts.cpu().numpy()
    for h in range(hq):
        qn = q[h].float().numpy()
        same = band_equal(oracle, qn, kn, ocfg, None, idx[h], counts[h])
        r = oracle.anchor_attention(qn, kn, vn, ocfg)
        assert_out_close(out[h].cpu().numpy(), r["out"], f"head {h}")
        if same:
            assert int(computed[h]) == r["computed"], h


@pytest.mark.parametrize("n", [1, 5, 64, 127, 128, 129, 255])
def test_tiny_sequences(oracle, n):
    """Sequences shorter than / around one 128-row block: partial tiles, no
    middle region, a single group — the fused chain and the stage API agree
    with the oracle."""
    c = capi()
    q, k, v = gen(n, hq=2, hkv=1, seed=n)
    cfg = c.BlockConfig(128, 128, 16, 12.0)
    out, computed = c.anchor_attention(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    for h in range(2):
        r = oracle.anchor_attention(q[h].float().numpy(), k[0].float().numpy(), v[0].float().numpy(),
                                    Cfg(128, 128, 16, 12.0))
        assert_out_close(out[h].cpu().numpy(), r["out"], f"n={n} head {h}")
        assert int(computed[h]) == r["computed"]


def test_fast_path_deterministic_and_recall_at_32k():
    """R/tests/test_sparse_exec.cpp:192-212 on the tcgen05 path at 32k (4 query
    heads / 1 KV head): two runs are bitwise identical, and on the sink /
    stripe heads the selection keeps recall >= 0.99 (GPU recall pass over
    covered ∪ stripes) at sparsity > 0.5."""
    c = capi()
    n = 32768
    q, k, v = (x.cuda() for x in gen(n, hq=4, hkv=1, seed=77))
    cfg = c.BlockConfig()
    o1, c1 = c.anchor_attention(q, k, v, cfg)
    o2, c2 = c.anchor_attention(q, k, v, cfg)
    st = c.compute_anchor(q, k, v, cfg)
    anchor, qbar = c.pool(q, k, st, cfg)
    idx, counts = c.identify(q, k, qbar, anchor, cfg)
    rec = c.union_recall(q, k, idx, counts, cfg)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(c1, c2)
    sparsity = 1.0 - c1.double() / (n * (n + 1) / 2)
    assert float(rec.min()) >= 0.99, rec
    assert float(sparsity.min()) > 0.5, sparsity
