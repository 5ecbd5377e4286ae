import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
g.set_kr("force")
for (M, N, K) in [(1024, 128, 4096), (2048, 96, 4096), (1024, 1024, 1024), (512, 512, 8192)]:
    a = torch.rand(M * K, device="cuda"); b = torch.rand(K * N, device="cuda"); c = torch.zeros(M * N, device="cuda")
    print("shape", (M, N, K), file=sys.stderr, flush=True)
    assert sgett_device(2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (N, 1), c) == []
    print("->", g.last_kernel(), file=sys.stderr, flush=True)
