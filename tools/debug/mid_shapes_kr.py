"""Mid-size contiguous SGEMM shapes (row-major A[m,k], B[k,n]): the automatic
choice vs the k-run kernel forced."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
def run(M, N, K, reps=200):
    gen = torch.Generator(device="cuda").manual_seed(1)
    a = torch.rand(M * K, device="cuda", generator=gen); b = torch.rand(K * N, device="cuda", generator=gen)
    c = torch.zeros(M * N, device="cuda")
    args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (N, 1), c)
    for _ in range(3): assert sgett_device(*args) == []
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        sgett_device(*args); s.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(10): sgett_device(*args)
        gr.replay(); s.synchronize()
        e0.record(s)
        for _ in range(reps // 10): gr.replay()
        e1.record(s); s.synchronize()
    ms = e0.elapsed_time(e1) / (reps // 10 * 10)
    return ms, 2.0 * M * N * K / ms / 1e9, g.last_kernel()
for shape in [(1024, 1024, 1024), (768, 768, 3072), (512, 512, 8192), (256, 256, 16384), (1024, 128, 4096), (2048, 96, 4096), (1536, 1536, 1536), (1024, 1024, 4096)]:
    out = []
    for mode in ("auto", "force"):
        g.set_kr(mode)
        try:
            out.append((mode,) + run(*shape))
        except Exception as e:
            out.append((mode, 0.0, 0.0, "ERR " + str(e)[:60]))
    g.set_kr("auto")
    print(shape, " | ".join(f"kr {n}: {ms*1e3:.1f}us {tf:.0f}TF {k.replace('sgett_','')}" for n, ms, tf, k in out), flush=True)
