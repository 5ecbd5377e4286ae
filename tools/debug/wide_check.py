"""Wide CTA-pair SGETT: K-normalised error vs an fp64 product, kernel, time.
GETT_WIDE=2 forces the kernel, 0 turns it off.   python tools/debug/wide_check.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import sgett_device  # noqa: E402


def case(M, N, K, bkf, seed=0):
    """C[m,n] += sum_k A[m,k] B'[n,k]; A row-major (K-major); B either [k][n]
    (rows-major B') or [n][k] (K-major B')."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.rand(M * K, device="cuda", generator=gen) * 2 - 1
    b = torch.rand(N * K, device="cuda", generator=gen) * 2 - 1
    c = torch.rand(M * N, device="cuda", generator=gen) * 2 - 1
    c0 = c.clone()
    if bkf:
        args = (2, (M, K), (K, 1), a, 2, (N, K), (K, 1), b, 1, (1,), (1,), (0, 1), (N, 1), c)
        bm = b.view(N, K).double()
    else:
        args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (N, 1), c)
        bm = b.view(K, N).double().t()
    assert sgett_device(*args) == []
    want = c0.view(M, N).double() + a.view(M, K).double() @ bm.t()
    err = ((c.view(M, N).double() - want).abs().max() / K).item()
    kname = g.last_kernel()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sgett_device(*args)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = sorted(times)[2]
    return {"M": M, "N": N, "K": K, "bkf": bkf, "kernel": kname, "err_k": err, "ms": round(ms, 4),
            "tflops": round(2 * M * N * K / ms / 1e9, 1), "wide": os.environ.get("GETT_WIDE")}


if __name__ == "__main__":
    shapes = [(256, 256, 64), (512, 384, 256), (300, 520, 128), (2048, 2048, 2048), (4096, 4096, 4096),
              (1000, 1800, 512), (4096, 1024, 8192)]
    for (M, N, K) in shapes:
        for bkf in (False, True):
            print(json.dumps(case(M, N, K, bkf)), flush=True)
