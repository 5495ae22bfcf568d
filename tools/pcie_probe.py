"""PCIe copy rates for the e2e bytes (2.15 GB D2H, 1.61 GB H2D; pinned): D2H over
1 / 2 / 4 streams alone and with the H2D concurrent, and the H2D alone."""
import torch, time
dev = torch.device("cuda", 0)
nb = 2147483648
d = torch.empty(nb, dtype=torch.uint8, device=dev)
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
hi = torch.empty(1610612736, dtype=torch.uint8).pin_memory()
di = torch.empty(1610612736, dtype=torch.uint8, device=dev)
def run(ns, with_h2d=False):
    ss = [torch.cuda.Stream(dev) for _ in range(ns)]
    s_in = torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        if with_h2d:
            with torch.cuda.stream(s_in):
                di.copy_(hi, non_blocking=True)
        ch = nb // (ns * 8)
        for i in range(ns * 8):
            with torch.cuda.stream(ss[i % ns]):
                h[i*ch:(i+1)*ch].copy_(d[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best * 1e3
for ns in (1, 2, 4):
    print("d2h streams", ns, "ms %.2f" % run(ns), "with concurrent h2d %.2f" % run(ns, True), flush=True)
torch.cuda.synchronize(); t = time.perf_counter(); di.copy_(hi, non_blocking=True); torch.cuda.synchronize(); print("h2d alone %.2f" % ((time.perf_counter()-t)*1e3))
