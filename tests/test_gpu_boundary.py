"""The drop-in boundary on the tcgen05 path.

* The reference-named pybind module (R/python/bindings.cpp:122-136) under its
  default precision (Bf16: the tcgen05 kernels) on the reference's own bf16
  golden outputs (oracle/_ref fixtures): anchor_attention, the stage chain
  compute_anchor -> identify_stripes_from_state -> sparse_attention, and
  identify_stripes_zero_anchor.
* aa_sparse_attention on caller lists (R/src/sparse_exec.cpp:51-56, 79-82):
  an index >= n is AA_ERR_OUT_OF_RANGE with the reference's text on both
  paths; unfiltered lists (covered, out-of-window and duplicate entries, any
  order) fold exactly the entries the reference folds.
* The host entry refuses V outside the f16 range of the PV operand.
"""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle.oracle import Cfg

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
REL_L2 = 1e-3
BAND = 1e-3


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def close(got, ref, what):
    err = float(np.abs(got - ref).max())
    rel = rel_l2(got, ref)
    assert err <= MAX_ABS and rel <= REL_L2, f"{what}: max-abs {err:.3e} rel-l2 {rel:.3e}"


@pytest.fixture()
def aa_bf16():
    from paper_2505_23520_b200 import anchorattn

    prev = anchorattn.precision()
    anchorattn.set_precision(anchorattn.Precision.Bf16)
    yield anchorattn
    anchorattn.set_precision(prev)


def test_default_precision_is_tcgen05():
    """A reference user who swaps in the module gets the tcgen05 path by
    default (ANCHORATTN_PRECISION=exact opts into the f64 kernels)."""
    import os
    import subprocess
    import sys

    code = ("from paper_2505_23520_b200 import anchorattn as a; "
            "print(a.precision() == a.Precision.Bf16)")
    env = dict(os.environ)
    env.pop("ANCHORATTN_PRECISION", None)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, check=True).stdout.strip()
    assert out == "True"


def band_equal_lists(oracle, z, cfg_o, got_groups, zero_anchor=False):
    q, k = z["q"], z["k"]
    n = int(z["n"])
    m, _, _ = oracle.compute_anchor(q, k, np.zeros_like(q), cfg_o)
    G = oracle.group_count(n, cfg_o)
    anchor = np.zeros(G) if zero_anchor else oracle.pooled_anchor(m, cfg_o)
    idx_o, cnt_o, margin = oracle.identify(q, k, anchor, cfg_o, want_margin=True)
    offs = oracle.stripe_offsets(n, cfg_o)
    same = True
    for g in range(G):
        a = set(idx_o[offs[g]:offs[g] + cnt_o[g]].tolist())
        b = set(got_groups[g])
        assert got_groups[g] == sorted(got_groups[g])
        for j in a ^ b:
            same = False
            assert abs(margin[offs[g] + j - cfg_o.b_kv]) <= BAND, (g, j)
    return same


@pytest.mark.parametrize("name", ["bf16_c1", "bf16_multigroup"])
def test_pybind_bf16_on_reference_goldens(aa_bf16, oracle, name):
    aa = aa_bf16
    z = load_golden(name)
    w = aa.HeadWorkload(z["q"], z["k"], z["v"])
    cfg = aa.BlockConfig(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))
    cfg_o = Cfg(int(z["b_q"]), int(z["b_kv"]), int(z["step"]), float(z["theta"]))
    rows = z["out_rows"]
    # whole chain (bindings.cpp:122-128)
    out, stats = aa.anchor_attention(w, cfg, False)
    close(out[rows], z["out"], f"{name} anchor_attention")
    assert stats.computed_positions == int(z["computed"])
    # stage chain
    st = aa.compute_anchor(w, cfg)
    m = np.asarray(st.m)
    assert np.max(np.abs(m - z["m"]) / np.maximum(np.abs(z["m"]), 1.0)) <= 1e-5
    assert np.max(np.abs(np.asarray(st.l) - z["l"]) / z["l"]) <= 1e-5
    np.testing.assert_allclose(aa.pooled_anchor(st, cfg), z["pooled_anchor"], rtol=0, atol=1e-4)
    close(aa.finalize_anchor(st)[rows], z["anchor_out"], f"{name} finalize_anchor")
    idx = aa.identify_stripes_from_state(w, st, cfg)
    same = band_equal_lists(oracle, z, cfg_o, idx.groups)
    out2, stats2 = aa.sparse_attention(w, st, idx, cfg)
    close(out2[rows], z["out"], f"{name} sparse_attention")
    if same:
        assert stats2.computed_positions == int(z["computed"])
    # zero-anchor arm (R/src/stripe_identify.cpp:90-95)
    zi = aa.identify_stripes_zero_anchor(w, cfg)
    band_equal_lists(oracle, z, cfg_o, zi.groups, zero_anchor=True)
    outz, statsz = aa.anchor_attention(w, cfg, True)
    rz = oracle.anchor_attention(z["q"], z["k"], z["v"], cfg_o, zero_anchor=True)
    close(outz, rz["out"], f"{name} zero-anchor chain")


def _gen(n, hq, hkv, seed):
    from paper_2505_23520_b200.workloads import gen_sink_workload, SinkWorkloadSpec

    return gen_sink_workload(SinkWorkloadSpec(n=n, hq=hq, hkv=hkv, seed=seed))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_sparse_out_of_range_index(dtype):
    """An index >= n is std::out_of_range with the reference's text on the
    C ABI itself (not only in the C++ shim), for both paths."""
    from paper_2505_23520_b200 import capi

    n = 4096
    q, k, v = (x.cuda().to(dtype) for x in _gen(n, 2, 1, 3))
    cfg = capi.BlockConfig()
    st = capi.compute_anchor(q, k, v, cfg)
    anchor, qbar = capi.pool(q, k, st, cfg)
    idx, counts = capi.identify(q, k, qbar, anchor, cfg)
    torch.cuda.synchronize()
    offs = capi.stripe_offsets(n, cfg)
    h, g = 1, 1
    assert int(counts[h, g]) >= 3
    bad = idx.clone()
    bad[h, offs[g] + 2] = n + 5  # first bad entry in (head, group, position) order
    bad[h, offs[g] + 1] = 128  # an in-range entry stays valid
    with pytest.raises(IndexError, match=f"sparse_attention: stripe index {n + 5} out of range"):
        capi.sparse(q, k, v, st, bad, counts, cfg)
    # a later bad entry does not mask the first one
    bad[h, offs[g] + 3] = -5  # 4294967291 as uint32
    with pytest.raises(IndexError, match=f"stripe index {n + 5} out of range"):
        capi.sparse(q, k, v, st, bad, counts, cfg)


def test_fast_sparse_unfiltered_csr_lists(oracle):
    """CSR lists with anchor-covered, out-of-window, non-causal and duplicate
    entries in arbitrary order: the fast path folds exactly what
    sparse_exec.cpp:79-82 folds (oracle on the same lists), computed counts
    included."""
    from paper_2505_23520_b200 import capi

    n, hq = 6144, 2
    q, k, v = _gen(n, hq, 1, 17)
    cfg = capi.BlockConfig(128, 128, 4, 12.0)
    ocfg = Cfg(128, 128, 4, 12.0)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    st = capi.compute_anchor(qd, kd, vd, cfg)
    rng = np.random.default_rng(5)
    G = (n // 128 + 3) // 4
    lists, counts, starts = [], [], []
    pos = 7  # lists need not be packed
    for h in range(hq):
        for g in range(G):
            L = list(rng.integers(0, n, size=int(rng.integers(0, 300))))
            L += L[:5]  # duplicates fold twice
            lists.append(L)
            starts.append(pos)
            counts.append(len(L))
            pos += len(L) + 3
    flat = np.zeros(pos + 1, np.uint32)
    for s, L in zip(starts, lists):
        flat[s:s + len(L)] = L
    offsets = torch.tensor(starts + [pos], dtype=torch.int64, device="cuda")
    idx_t = torch.from_numpy(flat.view(np.int32)).cuda()
    cnt_t = torch.tensor(counts, dtype=torch.int32, device="cuda")
    out, comp = capi.sparse(qd, kd, vd, st, idx_t, cnt_t, cfg, offsets=offsets)
    torch.cuda.synchronize()
    for h in range(hq):
        qn, kn, vn = q[h].float().numpy(), k[0].float().numpy(), v[0].float().numpy()
        m, l, acc = oracle.compute_anchor(qn, kn, vn, ocfg)
        ref_out, ref_comp = oracle.sparse_lists(qn, kn, vn, ocfg, m, l, acc, lists[h * G:(h + 1) * G])
        close(out[h].cpu().numpy(), ref_out, f"head {h}")
        assert int(comp[h]) == ref_comp


def test_host_entry_rejects_v_outside_f16():
    from paper_2505_23520_b200 import capi

    n = 1024
    q, k, v = _gen(n, 2, 1, 2)
    v = v.clone()
    v[0, 700, 3] = 1e6
    with pytest.raises(capi.AnchorAttnError, match="65504"):
        capi.anchor_attention_host(q, k, v, capi.BlockConfig())
    # in range: fine
    v[0, 700, 3] = 6e4
    out, _ = capi.anchor_attention_host(q, k, v, capi.BlockConfig())
    assert torch.isfinite(out).all()
