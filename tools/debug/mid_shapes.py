"""Mid-size contiguous SGEMM shapes: the automatic choice vs the wide kernel
forced (with split-K factors), device time per call (queued)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
def run(M, N, K, reps=40):
    gen = torch.Generator(device="cuda").manual_seed(1)
    a = torch.rand(M * K, device="cuda", generator=gen); b = torch.rand(K * N, device="cuda", generator=gen)
    c = torch.zeros(M * N, device="cuda")
    args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (N, 1), c)
    for _ in range(3): assert sgett_device(*args) == []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): sgett_device(*args)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2.0 * M * N * K / ms / 1e9, g.last_kernel()
for shape in [(1024, 1024, 1024), (1536, 1536, 1536), (1024, 1024, 4096), (512, 512, 8192), (2048, 1024, 2048), (768, 768, 3072), (3072, 3072, 3072)]:
    out = []
    g.set_wide("auto"); g.set_split_k(0)
    out.append(("auto",) + run(*shape))
    for sp in (0, 2, 4, 8):
        g.set_wide("force"); g.set_split_k(sp)
        try:
            out.append((f"wide sp{sp}",) + run(*shape))
        except Exception as e:
            out.append((f"wide sp{sp}", 0, 0, str(e)[:40]))
    g.set_wide("auto"); g.set_split_k(0)
    print(shape, " | ".join(f"{n}: {ms*1e3:.1f}us {tf:.0f}TF {k.replace('sgett_tc3xtf32_','')}" for n, ms, tf, k in out), flush=True)
