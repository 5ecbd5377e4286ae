"""Wide CTA-pair SGETT (sgett_tc.cu wide::sgett_tc_wide_kernel): a 256 x 256
output tile per cluster of two CTAs (tcgen05.mma.cta_group::2, M = N = 256),
each CTA holding 128 A' rows in TMEM and 128 B' rows in shared memory.

Bars: without split-K it issues the same MMAs in the same k order as the
128 x 128 kernel, so the results are bitwise equal; with split-K (partials +
reduce) within the K-normalised 3xTF32 bar of an fp64 product.  Shapes cover
both B' orientations (K-major boxes used in place, rows-major transposed),
pair tiles whose second CTA holds no A' rows or no B' rows (its boxes are
skipped), ragged edges, strided C with padding left untouched, and the
automatic choice."""
import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu


def _operands(M, N, K, bkf, seed, pad_c=0):
    import torch

    gen = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.rand(M * K, device="cuda", generator=gen) * 2 - 1
    b = torch.rand(N * K, device="cuda", generator=gen) * 2 - 1
    ldc = N + pad_c
    c = torch.rand(M * ldc + 4, device="cuda", generator=gen) * 2 - 1
    if bkf:
        args = (2, (M, K), (K, 1), a, 2, (N, K), (K, 1), b, 1, (1,), (1,), (0, 1), (ldc, 1), c)
        bm = b.view(N, K).double()
    else:
        args = (2, (M, K), (K, 1), a, 2, (K, N), (N, 1), b, 1, (1,), (0,), (0, 1), (ldc, 1), c)
        bm = b.view(K, N).double().t()
    return args, a.view(M, K).double(), bm


def _run(args, c0, mode, split, kernel_mode, mixed=False, tail=True):
    from paper_2410_06770_b200.device import sgett_device

    kernel_mode("tiled", wide=mode, split=split, wide_mixed=mixed, wide_tail=tail)
    c = c0.clone()
    args = args[:13] + (c,)
    assert sgett_device(*args) == []
    return c, g.last_kernel()


SHAPES = [(256, 256, 64), (512, 768, 256), (300, 520, 128), (384, 200, 96), (640, 1152, 512), (2048, 2048, 512)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("bkf", [False, True])
def test_wide_bitwise_equals_single_cta(shape, bkf, kernel_mode):
    M, N, K = shape
    args, am, bm = _operands(M, N, K, bkf, sum(shape), pad_c=5)
    c0 = args[13].clone()
    wide, kw = _run(args, c0, "force", 1, kernel_mode)
    if N < 256:
        assert "wide" not in kw, kw  # needs two 128-row B' halves
        return
    assert kw == "sgett_tc3xtf32_wide", kw
    single, ks = _run(args, c0, "off", 1, kernel_mode)
    assert "wide" not in ks
    assert wide.cpu().numpy().tobytes() == single.cpu().numpy().tobytes()
    ldc = N + 5
    got = wide[:M * ldc].view(M, ldc).double()
    want = c0[:M * ldc].view(M, ldc).double()
    want[:, :N] += am @ bm.t()
    assert ((got - want).abs().max() / K).item() <= 1e-5
    # padding columns and the tail untouched
    assert torch_equal(wide[:M * ldc].view(M, ldc)[:, N:], c0[:M * ldc].view(M, ldc)[:, N:])
    assert torch_equal(wide[M * ldc:], c0[M * ldc:])


def torch_equal(x, y):
    return x.cpu().numpy().tobytes() == y.cpu().numpy().tobytes()


@pytest.mark.parametrize("split", [2, 5])
@pytest.mark.parametrize("bkf", [False, True])
def test_wide_split_k(split, bkf, kernel_mode):
    M, N, K = 768, 512, 1024
    args, am, bm = _operands(M, N, K, bkf, split)
    c0 = args[13].clone()
    c, kname = _run(args, c0, "force", split, kernel_mode)
    assert kname == "sgett_tc3xtf32_wide_splitk", kname
    want = c0[:M * N].view(M, N).double() + am @ bm.t()
    err = ((c[:M * N].view(M, N).double() - want).abs().max() / K).item()
    assert err <= 1e-5, err


def test_wide_auto_choice(kernel_mode):
    """Automatic: a 2048^3 GEMM (64 pair tiles) takes the wide kernel; a
    512 x 384 x 256 one (4 pair tiles, split-K territory) does not."""
    from paper_2410_06770_b200.device import sgett_device

    for (M, N, K), want in (((2048, 2048, 2048), True), ((512, 384, 256), False)):
        args, _, _ = _operands(M, N, K, False, 1)
        kernel_mode("auto")
        assert sgett_device(*args) == []
        assert ("wide" in g.last_kernel()) == want, (M, N, K, g.last_kernel())


def test_wide_strided_views(kernel_mode):
    """Non-contiguous affine views (row pitch > K, C column-major with
    padding): the TMA boxes and the epilogue offset tables follow the views."""
    import torch

    from paper_2410_06770_b200.device import sgett_device

    M, N, K = 512, 512, 128
    rng = np.random.default_rng(3)
    a = torch.from_numpy(rng.uniform(-1, 1, M * (K + 16)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.uniform(-1, 1, K * (N + 32)).astype(np.float32)).cuda()
    ldc = M + 7
    c0 = torch.from_numpy(rng.uniform(-1, 1, N * ldc).astype(np.float32)).cuda()
    outs = []
    for mode in ("force", "off"):
        kernel_mode("tiled", wide=mode, split=1, wide_mixed=False)
        c = c0.clone()
        assert sgett_device(2, (M, K), (K + 16, 1), a, 2, (K, N), (N + 32, 1), b, 1, (1,), (0,), (0, 1),
                            (1, ldc), c) == []
        outs.append((c, g.last_kernel()))
    assert outs[0][0].cpu().numpy().tobytes() == outs[1][0].cpu().numpy().tobytes(), [k for _, k in outs]
    am = a.view(M, K + 16)[:, :K].double()
    bm = b.view(K, N + 32)[:, :N].double()
    got = outs[0][0].view(N, ldc)[:, :M].double().t()
    want = c0.view(N, ldc)[:, :M].double().t() + am @ bm
    assert ((got - want).abs().max() / K).item() <= 1e-5


@pytest.mark.parametrize("shape", SHAPES + [(1024, 1024, 2048)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("bkf", [False, True])
@pytest.mark.parametrize("split", [1, 3])
def test_wide_mixed_split(shape, bkf, split, kernel_mode):
    """The mixed split (one tf32 MMA of the hi parts + one bf16 MMA carrying
    both cross terms per 8 k) in the wide kernel, both B' orientations, with
    and without split-K: within the bar of an fp64 product, as accurate as the
    three-MMA truncation split (<= 1.5x its error; smaller for long K), padding
    untouched, and exact on small-integer data."""
    import torch

    M, N, K = shape
    if N < 256:
        pytest.skip("needs two 128-row B' halves")
    args, am, bm = _operands(M, N, K, bkf, sum(shape) + split, pad_c=5)
    c0 = args[13].clone()
    ldc = N + 5
    want = c0[:M * ldc].view(M, ldc).double()
    want[:, :N] += am @ bm.t()
    errs = {}
    for mixed in (True, False):
        c, kname = _run(args, c0, "force", split, kernel_mode, mixed=mixed)
        assert kname.startswith("sgett_tctf32bf16_wide" if mixed else "sgett_tc3xtf32_wide"), kname
        assert ("splitk" in kname) == (split > 1), kname
        errs[mixed] = ((c[:M * ldc].view(M, ldc).double() - want).abs().max() / K).item()
        assert errs[mixed] <= 1e-5, (mixed, errs)
        assert torch_equal(c[:M * ldc].view(M, ldc)[:, N:], c0[:M * ldc].view(M, ldc)[:, N:])
        assert torch_equal(c[M * ldc:], c0[M * ldc:])
    assert errs[True] <= 1.5 * errs[False] + 1e-9, errs
    # integers |x| <= 8: hi parts exact, lo parts zero
    ai = torch.round(args[3] * 8)
    bi = torch.round(args[7] * 8)
    ci = torch.round(c0 * 8)
    iargs = args[:3] + (ai,) + args[4:7] + (bi,) + args[8:13] + (ci,)
    outs = [_run(iargs, ci, "force", split, kernel_mode, mixed=m)[0] for m in (True, False)]
    assert torch_equal(outs[0], outs[1])


@pytest.mark.parametrize("shape", [(2560, 2048, 1024), (2500, 2100, 1040), (4096, 4096, 1024)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("bkf", [False, True])
@pytest.mark.parametrize("mixed", [False, True])
def test_wide_tail_split(shape, bkf, mixed, kernel_mode):
    """More pair tiles than pair slots (74 on 148 SMs) with a partial last wave
    of at most half the slots (80 -> 6, 90 -> 16, 256 -> 34 tiles): those tiles
    run as two K halves whose compact partials a small reduce adds to C.
    Within the bar of an fp64 product; every tile the whole-K CTAs wrote is
    bitwise what the launch without a tail split writes; padding untouched."""
    import torch

    M, N, K = shape
    args, am, bm = _operands(M, N, K, bkf, sum(shape), pad_c=3)
    c0 = args[13].clone()
    ldc = N + 3
    c, kname = _run(args, c0, "force", 0, kernel_mode, mixed=mixed)
    assert kname.endswith("_wide_tail"), kname
    plain, kplain = _run(args, c0, "force", 0, kernel_mode, mixed=mixed, tail=False)
    assert kplain.endswith("_wide"), kplain
    want = c0[:M * ldc].view(M, ldc).double()
    want[:, :N] += am @ bm.t()
    got = c[:M * ldc].view(M, ldc)
    assert ((got.double() - want).abs().max() / K).item() <= 1e-5
    assert torch_equal(got[:, N:], c0[:M * ldc].view(M, ldc)[:, N:])
    assert torch_equal(c[M * ldc:], c0[M * ldc:])
    same = (got == plain[:M * ldc].view(M, ldc))[:, :N]
    tiles_m, tiles_n = -(-M // 256), -(-N // 256)
    rem = (tiles_m * tiles_n) % 74
    pad = torch.zeros(tiles_m * 256, tiles_n * 256, dtype=torch.bool, device=same.device)
    pad[:M, :N] = ~same
    differing = pad.view(tiles_m, 256, tiles_n, 256).any(dim=3).any(dim=1).sum().item()
    assert differing <= rem, (differing, rem)
