"""Run one BASELINE config through the zero-copy device entry a few times
(for ncu / compute-sanitizer captures; the kernel mode comes from GETT_*
environment variables).   python tools/run_one.py c5 [calls]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import dgett_device, sgett_device  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402

name = sys.argv[1]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = CONFIGS[name]
a, b, c = (torch.from_numpy(x).cuda() for x in w.buffers())
pos, kw = w.args(a, b, c)
fn = dgett_device if w.dtype == "d" else sgett_device
for _ in range(calls):
    assert fn(*pos, **kw) == []
torch.cuda.synchronize()
print(name, g.last_kernel(), g.launch_count())
