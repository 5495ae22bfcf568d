import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle.oracle import Cfg, Oracle
from paper_2505_23520_b200 import capi as c
from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload, gen_random_workload
orc = Oracle()
for n, step, kind in [(4096, 16, 'sink'), (2048, 2, 'sink'), (4000, 4, 'sink'), (640, 1, 'sink'), (8192, 16, 'sink'), (2048, 16, 'random')]:
    if kind == 'sink':
        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=n, hq=1, hkv=1, seed=n + step))
    else:
        q, k, v = gen_random_workload(n, seed=3)
    cfg = c.BlockConfig(128, 128, step, 12.0)
    st = c.compute_anchor(q.cuda(), k.cuda(), v.cuda(), cfg)
    torch.cuda.synchronize()
    qn, kn, vn = (x[0].float().numpy() for x in (q, k, v))
    m, l, acc = orc.compute_anchor(qn, kn, vn, Cfg(128, 128, step, 12.0))
    lg = st["l"][0].double().cpu().numpy()
    rel = np.abs(lg - l) / l
    mg = st["m"][0].double().cpu().numpy()
    print(kind, n, step, "l max rel %.3e mean %.3e" % (rel.max(), rel.mean()), "m max rel %.3e" % (np.abs(mg - m) / np.maximum(np.abs(m), 1)).max())
