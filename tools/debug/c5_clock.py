"""c5 back to back for ~2 s under nvidia-smi sampling: SM clock and power
while the k-run SGETT runs (is the kernel power-throttled?)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device, dgett_device
from paper_2410_06770_b200.workloads import C5, C2
for w, fn, n in ((C5, sgett_device, 40000), (C2, dgett_device, 500)):
    a, b, c = (torch.from_numpy(x).cuda() for x in w.buffers())
    pos, kw = w.args(a, b, c)
    fn(*pos, **kw); torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn(*pos, **kw)
    e1.record(); torch.cuda.synchronize()
    time.sleep(0.2); smi.terminate()
    lines = [l.strip() for l in smi.stdout.read().splitlines() if l.strip()]
    print(w.name, g.last_kernel(), "ms per call", e0.elapsed_time(e1) / n)
    print("\n".join(lines[2:-2][::4]))
