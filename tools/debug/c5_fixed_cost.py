"""c5 with its contracted mode A1/B2 cut to 24, 18, 12, 6 (K = 30720 ... 7680;
same tiles and splits, 16 ... 4 k-blocks per CTA pair): GPU time per call from
a CUDA graph of 20 calls -> per-k-block cost (slope) and fixed cost (intercept)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from dataclasses import replace
import numpy as np, torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
from paper_2410_06770_b200.workloads import C5
pts = []
for k1 in (24, 18, 12, 6):
    ea = list(C5.ext_a); ea[1] = k1
    eb = list(C5.ext_b); eb[2] = k1
    w = replace(C5, ext_a=tuple(ea), ext_b=tuple(eb))
    a, b, c = (torch.from_numpy(x).cuda() for x in w.buffers())
    pos, kw = w.args(a, b, c)
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(3): assert sgett_device(*pos, **kw) == []
        s.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(20): sgett_device(*pos, **kw)
        for _ in range(5): gr.replay()
        s.synchronize()
        e0.record(s)
        for _ in range(100): gr.replay()
        e1.record(s); s.synchronize()
    us = e0.elapsed_time(e1) / 2000 * 1e3
    pts.append((k1 * 32 * 40 // 24 // 80, us))
    print(k1, g.last_kernel(), "k-blocks per CTA pair", pts[-1][0], "us/call %.2f" % us, flush=True)
x, y = np.array(pts).T
sl, ic = np.polyfit(x, y, 1)
print("per k-block %.3f us, fixed %.2f us" % (sl, ic))
