"""Contiguous SGEMM through the tcgen05 tiled kernel vs the k-run kernel (forced)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
for n in (2048, 4096):
    a = torch.rand(n * n, device="cuda") - 0.5
    b = torch.rand(n * n, device="cuda") - 0.5
    for mode in ("off", "force"):
        g.set_kr(mode)
        c = torch.zeros(n * n, device="cuda")
        args = (2, (n, n), (n, 1), a, 2, (n, n), (n, 1), b, 1, (1,), (0,), (0, 1), (n, 1), c)
        for _ in range(2): sgett_device(*args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): sgett_device(*args)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(n, mode, g.last_kernel(), round(ms, 4), "TF", round(2 * n**3 / ms / 1e9, 1), flush=True)
g.set_kr("auto")
