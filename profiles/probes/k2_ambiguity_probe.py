import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_23520_b200 import capi
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload
n, hq, hkv, rep = 131072, 32, 8, 4
dev = torch.device("cuda", 0)
tot = amb = 0
for kvh in range(2):
    q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=rep, hkv=1, seed=2505 + kvh), device=dev)
    cfg = capi.BlockConfig(128, 128, 16, 12.0)
    st = capi.compute_anchor(q, k, v, cfg)
    anchor, qbar = capi.pool(q, k, st, cfg)       # [rep, G] f64, [rep, G, d] f32
    G = qbar.shape[1]
    hi = qbar.bfloat16().float(); lo = qbar - hi
    kf = k[0].float()                              # [n, d]
    knorm = kf.norm(dim=1)                         # [n]
    tile_max = knorm.view(-1, 128).max(dim=1).values.repeat_interleave(128)
    for g in range(G):
        mend = max(128, min(2048 * g - 128, n)) if g > 0 else 128
        if mend <= 128: continue
        keys = slice(128, mend)
        for hh in range(rep):
            thr = (anchor[hh, g].item() - 12.0) * (128 ** 0.5)
            s_hi = kf[keys] @ hi[hh, g]
            bound = lo[hh, g].norm() * tile_max[keys] + 2 ** -16 * hi[hh, g].norm() * tile_max[keys]
            a = ((s_hi - thr).abs() <= bound).sum().item()
            amb += a; tot += s_hi.numel()
print(f"ambiguous {amb} of {tot} = {amb / tot:.2e}")
