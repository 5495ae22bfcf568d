import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_2505_23520_b200 import capi
from paper_2505_23520_b200.workloads import gen_layer
q, k, v = gen_layer(131072, 32, 8, 2505, device="cuda")
cfg = capi.BlockConfig()
pipe = capi.Pipeline(q, k, v, cfg)
out = torch.empty((32, 131072, 128), dtype=torch.float32, device="cuda")
for _ in range(2):
    pipe(q, k, v, out=out)
torch.cuda.synchronize()
