"""Wide kernel under the current GETT_WIDE_* environment (no setter calls):
error vs fp64 for both B' orientations and a few shapes, then timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
for (M, N, K) in [(2048, 2048, 512), (2048, 2304, 528), (2500, 2100, 1040), (4096, 4096, 1024)]:
    for bkf in (False, True):
        gen = torch.Generator(device="cuda").manual_seed(M + K + bkf)
        a = torch.rand(M * K, device="cuda", generator=gen) * 2 - 1
        b = torch.rand(N * K, device="cuda", generator=gen) * 2 - 1
        c0 = torch.rand(M * N, device="cuda", generator=gen) * 2 - 1
        c = c0.clone()
        if bkf:
            args = (2, (M, K), (K, 1), a, 2, (N, K), (K, 1), b, 1, (1,), (1,), (0, 1), (N, 1), c)
            bm = b.view(N, K).double().t()
        else:
            args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (N, 1), c)
            bm = b.view(K, N).double()
        assert sgett_device(*args) == []
        want = c0.view(M, N).double() + a.view(M, K).double() @ bm
        err = ((c.view(M, N).double() - want).abs().max() / K).item()
        print((M, N, K), "bkf" if bkf else "brm", g.last_kernel(), "err_k %.2e" % err, "OK" if err <= 1e-5 else "FAIL", flush=True)
