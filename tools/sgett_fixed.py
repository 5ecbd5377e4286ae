"""Fixed vs per-k-block cost of the SGETT tcgen05 kernel at c5's tile grid
(M' 96 x N' 768 -> 6 tiles, split-K 24 -> 144 CTAs): a rows-major A' and a
K-major B' (TMA-fed), each CTA given kb k-blocks of 16; device time per call
(CUDA events over back-to-back calls) for several kb -> linear fit."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import sgett_device  # noqa: E402


def main():
    g.set_kernel("tiled")
    g.set_split_k(24)
    res = []
    kbs = [int(x) for x in sys.argv[1:]] or [1, 5, 20, 40, 80]
    for kb in kbs:
        K = 24 * 16 * kb
        M, N = 96, 768
        # A'(orig B) rows-major: A[k][m] (m contiguous); B'(orig A) K-major: B[n][k]
        a = torch.rand(K * M, device="cuda")
        b = torch.rand(N * K, device="cuda")
        c = torch.zeros(M * N, device="cuda")
        # C[n][m] with m fastest -> M group holds C's fast mode -> planner roles:
        # contract A(k, m) with B(n, k): C = (m, n) with inc (1, M)
        args = (2, (K, M), (M, 1), a, 2, (N, K), (K, 1), b, 1, (0,), (1,), (0, 1), (1, M), c)
        for _ in range(3):
            assert sgett_device(*args) == []
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sgett_device(*args)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.append((kb, ms))
        print(json.dumps({"kblocks_per_cta": kb, "K": K, "ms": round(ms, 4), "kernel": g.last_kernel()}))
    if len(res) < 2:
        return
    x = np.array([r[0] for r in res], float)
    y = np.array([r[1] for r in res])
    slope, icpt = np.polyfit(x, y, 1)
    print(json.dumps({"fixed_us": round(icpt * 1e3, 2), "per_kblock_ns": round(slope * 1e6, 1)}))


if __name__ == "__main__":
    main()
