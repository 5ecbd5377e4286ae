"""c5 per-call time, back to back (20000 calls) and with an L2 flush before
each call (201 calls, median), for the k-run kernel single / pair and the tiled kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
from paper_2410_06770_b200.workloads import C5
a, b, c = (torch.from_numpy(x).cuda() for x in C5.buffers())
pos, kw = C5.args(a, b, c)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name, kr, pair in (("pair", "auto", True), ("single", "auto", False), ("tiled", "off", True), ("pair", "auto", True)):
    g.set_kr(kr, False, pair)
    for _ in range(50): sgett_device(*pos, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20000): sgett_device(*pos, **kw)
    e1.record(); torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 20000 * 1e3
    ts = []
    for _ in range(201):
        flush.zero_()
        e0.record(); sgett_device(*pos, **kw); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, g.last_kernel(), "back-to-back us %.1f" % b2b, "flushed median us %.1f p10 %.1f" % (np.median(ts), np.percentile(ts, 10)), flush=True)
