"""Is c5 back to back host-bound?  Host issue time per call vs GPU time per
call, and the GPU time per call when 20 calls are replayed from one CUDA graph
(no per-call host work)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
from paper_2410_06770_b200.workloads import C5
a, b, c = (torch.from_numpy(x).cuda() for x in C5.buffers())
pos, kw = C5.args(a, b, c)
for _ in range(20): sgett_device(*pos, **kw)
torch.cuda.synchronize()
n = 5000
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(n): sgett_device(*pos, **kw)
t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
print(g.last_kernel(), "host issue us/call %.1f  gpu us/call %.1f" % ((t1 - t0) / n * 1e6, e0.elapsed_time(e1) / n * 1e3))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): sgett_device(*pos, **kw)
    s.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20): sgett_device(*pos, **kw)
    for _ in range(5): gr.replay()
    s.synchronize()
    e0.record(s)
    for _ in range(200): gr.replay()
    e1.record(s); s.synchronize()
print("graph of 20 calls: gpu us/call %.2f" % (e0.elapsed_time(e1) / 4000 * 1e3))
