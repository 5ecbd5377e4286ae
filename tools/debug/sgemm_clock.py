"""SGEMM n^3 back to back for ~1.5 s under nvidia-smi sampling: SM clock and
power for the current GETT_WIDE_* settings."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
gen = torch.Generator(device="cuda").manual_seed(1)
a = torch.rand(n * n, device="cuda", generator=gen) * 2 - 1
b = torch.rand(n * n, device="cuda", generator=gen) * 2 - 1
c = torch.zeros(n * n, device="cuda")
args = (2, (n, n), (n, 1), a, 2, (n, n), (n, 1), b, 1, (1,), (0,), (0, 1), (n, 1), c)
sgett_device(*args); torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
reps = 2500
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    sgett_device(*args)
e1.record(); torch.cuda.synchronize()
time.sleep(0.2); smi.terminate()
lines = [l.strip() for l in smi.stdout.read().splitlines() if l.strip()]
ms = e0.elapsed_time(e1) / reps
print(n, g.last_kernel(), "ms per call %.4f  TF %.1f" % (ms, 2 * n ** 3 / ms / 1e9))
print(" | ".join(lines[4:-3][::3]))
