"""Run a contiguous fp32 GEMM-shaped SGETT (row-major A[m,k], B[k,n] or, with
`kk`, B[n,k]) a few times through the zero-copy device entry (for ncu).
    python tools/run_sgemm.py 4096 [calls] [kk]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import sgett_device  # noqa: E402

n = int(sys.argv[1])
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kk = len(sys.argv) > 3 and sys.argv[3] == "kk"
gen = torch.Generator(device="cuda").manual_seed(1)
a = torch.rand(n * n, device="cuda", generator=gen) * 2 - 1
b = torch.rand(n * n, device="cuda", generator=gen) * 2 - 1
c = torch.zeros(n * n, device="cuda")
if kk:
    args = (2, (n, n), (n, 1), a, 2, (n, n), (n, 1), b, 1, (1,), (1,), (0, 1), (n, 1), c)
else:
    args = (2, (n, n), (n, 1), a, 2, (n, n), (n, 1), b, 1, (1,), (0,), (0, 1), (n, 1), c)
for _ in range(calls):
    assert sgett_device(*args) == []
torch.cuda.synchronize()
print(n, g.last_kernel(), g.launch_count())
