"""Random-shape campaign for the round-2 SGETT kernels: the k-run kernel
(single / pair, 1 or 2 runs per k-block, mixed / 3xTF32 split, fused /
separate reduce, forced splits, PDL on / off) and the wide kernel (both B'
orientations, mixed / 3xTF32, tail split, split-K, ragged edges), each against
an fp64 product with the K-normalised 1e-5 bar and untouched padding.
    python tools/debug/fuzz_new.py [seconds] [seed]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import sgett_device
from tests.test_gpu_kr import _case, _check

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t_end = time.time() + budget
n_kr = n_wide = 0
kernels = {}
while time.time() < t_end:
    if rng.random() < 0.5:
        kr = int(rng.choice([8, 16, 24, 32, 40, 48, 56, 64, 128]))
        m1, m2 = int(rng.integers(1, 7)), int(rng.choice([16, 32, 33, 50, 64, 100, 128, 200]))
        k2 = int(rng.integers(1, 33)) * (1 if rng.random() < 0.5 else 2)
        n = int(rng.choice([16, 40, 64, 96, 128, 189, 200, 320]))
        cmf = bool(rng.integers(0, 2))
        split = int(rng.choice([0, 0, 1, 2, 3, 5, 8]))
        pair, fused, mixed, pdl = (bool(rng.integers(0, 2)) for _ in range(4))
        pos, kw = _case(m1, m2, kr, k2, n, cmf, seed=int(rng.integers(1 << 30)))
        c0 = pos[13].copy()
        g.set_kernel("tiled"); g.set_split_k(split); g.set_kr("force", fused, pair, mixed); g.set_pdl(pdl)
        try:
            assert g.sgett(*pos, **kw) == []
            _check(pos, kw, c0)
        except Exception:
            print("FAIL kr", (m1, m2, kr, k2, n, cmf, split, pair, fused, mixed, pdl), g.last_kernel(), flush=True)
            raise
        kernels[g.last_kernel()] = kernels.get(g.last_kernel(), 0) + 1
        n_kr += 1
    else:
        M = int(rng.choice([256, 300, 512, 640, 1000, 1280, 2048, 2560, 4096]))
        N = int(rng.choice([256, 260, 512, 520, 768, 1152, 2048, 2100, 4096]))
        K = 16 * int(rng.integers(2, 130))
        bkf, mixed, tail = (bool(rng.integers(0, 2)) for _ in range(3))
        split = int(rng.choice([0, 0, 0, 1, 2, 3]))
        gen = torch.Generator(device="cuda").manual_seed(int(rng.integers(1 << 30)))
        a = torch.rand(M * K, device="cuda", generator=gen) * 2 - 1
        b = torch.rand(N * K, device="cuda", generator=gen) * 2 - 1
        ldc = N + 5
        c0 = torch.rand(M * ldc + 4, device="cuda", generator=gen) * 2 - 1
        c = c0.clone()
        if bkf:
            args = (2, (M, K), (K, 1), a, 2, (N, K), (K, 1), b, 1, (1,), (1,), (0, 1), (ldc, 1), c)
            bm = b.view(N, K).double()
        else:
            args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (ldc, 1), c)
            bm = b.view(K, N).double().t()
        g.set_kernel("tiled"); g.set_split_k(split); g.set_kr("off"); g.set_wide("force", mixed, tail)
        try:
            assert sgett_device(*args) == []
            want = c0[:M * ldc].view(M, ldc).double()
            want[:, :N] += a.view(M, K).double() @ bm.t()
            got = c[:M * ldc].view(M, ldc)
            err = ((got.double() - want).abs().max() / K).item()
            assert err <= 1e-5, err
            assert torch.equal(got[:, N:], c0[:M * ldc].view(M, ldc)[:, N:]) and torch.equal(c[M * ldc:], c0[M * ldc:])
        except Exception:
            print("FAIL wide", (M, N, K, bkf, mixed, tail, split), g.last_kernel(), flush=True)
            raise
        kernels[g.last_kernel()] = kernels.get(g.last_kernel(), 0) + 1
        n_wide += 1
g.set_kernel("auto"); g.set_split_k(0); g.set_kr("auto"); g.set_wide("auto"); g.set_pdl(True)
print("ok: k-run cases", n_kr, "wide cases", n_wide)
for k, v in sorted(kernels.items()):
    print("  ", k, v)
