"""DGETT bulk-add epilogue (dgett_ws.cu, p.c_bulk; capi.cu c_bulk_rows/cols):
C += acc as one cp.reduce.async.bulk .add.f64 per 32-element C row run,
staged in the ring slot after the tile's last k-block, instead of one
red.global.add.f64 per element.  Both perform exactly one IEEE add per element
at L2, so results are bitwise equal; the cases cover one CTA per tile,
persistent stream-K with FULL/HEAD tiles (including shares shorter than a
tile, where a CTA's last segment is a FULL tile right after a TAIL — the case
that exposed a staging-slot race), split-K (not bulk), both producers (TMA
and cp.async gathers), negated accumulation (complex), and the layouts that
must fall back (C's N run not a multiple of 32, odd offsets, unaligned C)."""
import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu


def _gemm(M, N, K, seed, inc_c=None, off_c=0, data="int"):
    rng = np.random.default_rng(seed)
    if data == "int":
        A = rng.integers(-3, 4, M * K).astype(np.float64)
        B = rng.integers(-3, 4, N * K).astype(np.float64)
        C = rng.integers(-3, 4, off_c + M * (inc_c or N) + 8).astype(np.float64)
    else:
        A = rng.standard_normal(M * K)
        B = rng.standard_normal(N * K)
        C = rng.standard_normal(off_c + M * (inc_c or N) + 8)
    return A, B, C


def _run(M, N, K, A, B, C, inc_c, off_c, bulk, tma, kernel_mode):
    kernel_mode("tiled", tma=tma, bulk=bulk)
    c = C.copy()
    assert g.dgett(2, (M, K), (K, 1), A, 2, (N, K), (K, 1), B, 1, (1,), (1,), (0, 1), (inc_c, 1), c,
                   offset_c=off_c) == []
    return c, g.last_kernel()


SHAPES = [(128, 256, 96), (1024, 2048, 64), (1920, 1664, 128), (1152, 1152, 64), (384, 8192, 512),
          (2048, 2048, 256), (200, 4000, 320)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("tma", [True, False])
def test_bulk_equals_red_bitwise(shape, tma, kernel_mode):
    M, N, K = shape
    A, B, C = _gemm(M, N, K, sum(shape), inc_c=N + 32, off_c=2, data="normal")
    got, kname = _run(M, N, K, A, B, C, N + 32, 2, True, tma, kernel_mode)
    want, _ = _run(M, N, K, A, B, C, N + 32, 2, False, tma, kernel_mode)
    assert kname.startswith("dgett_dmma_ws"), kname
    assert kname.endswith("_bulk") or "splitk" in kname, kname
    assert got.tobytes() == want.tobytes()
    # and right: integer data is exact
    Ai, Bi, Ci = _gemm(M, N, K, 7, inc_c=N + 32, off_c=2)
    got, _ = _run(M, N, K, Ai, Bi, Ci, N + 32, 2, True, tma, kernel_mode)
    ref = Ci.copy()
    view = ref[2:2 + M * (N + 32)].reshape(M, N + 32)
    view[:, :N] += Ai.reshape(M, K) @ Bi.reshape(N, K).T
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("inc_c,off_c,why", [(1000, 2, "N run 1000 not a multiple of 32"),
                                             (1056, 1, "odd C offset"), (1057, 0, "odd row stride")])
def test_bulk_falls_back_bitwise(inc_c, off_c, why, kernel_mode):
    """Layouts the bulk requests cannot take run the red.add epilogue: same
    bits.  (Device entry: the host entry re-bases C's footprint on the device,
    so an odd host offset is even there.)"""
    import torch

    from paper_2410_06770_b200.device import dgett_device

    M, K = 640, 96
    N = 1000 if inc_c == 1000 else 1024
    A, B, C = _gemm(M, N, K, 3, inc_c=inc_c, off_c=off_c, data="normal")
    ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = []
    for bulk in (True, False):
        kernel_mode("tiled", bulk=bulk)
        tc = torch.from_numpy(C).cuda()
        assert dgett_device(2, (M, K), (K, 1), ta, 2, (N, K), (K, 1), tb, 1, (1,), (1,), (0, 1), (inc_c, 1), tc,
                            offset_c=off_c) == []
        assert not g.last_kernel().endswith("_bulk"), (g.last_kernel(), why)
        outs.append(tc.cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes(), why


def test_bulk_negated_complex(kernel_mode):
    """zgett's embedded real GETT subtracts the a.im*b.im term (p.neg)."""
    rng = np.random.default_rng(11)
    M, N, K = 384, 512, 64
    a = (rng.standard_normal(M * K) + 1j * rng.standard_normal(M * K))
    b = (rng.standard_normal(N * K) + 1j * rng.standard_normal(N * K))
    c0 = (rng.standard_normal(M * N) + 1j * rng.standard_normal(M * N))
    outs = []
    for bulk in (True, False):
        kernel_mode("tiled", bulk=bulk)
        c = c0.copy()
        assert g.zgett(2, (M, K), (K, 1), a, 2, (N, K), (K, 1), b, 1, (1,), (1,), (0, 1), (N, 1), c) == []
        outs.append(c)
    assert outs[0].tobytes() == outs[1].tobytes()
    want = c0.reshape(M, N) + a.reshape(M, K) @ b.reshape(N, K).T
    assert np.abs(outs[0].reshape(M, N) - want).max() <= 1e-12 * K * 4


def test_bulk_c3_equals_red(kernel_mode):
    """c3 through the device entry (one stream-K launch; the host entry cuts
    it into pipelined slabs)."""
    import torch

    from paper_2410_06770_b200.device import dgett_device
    from paper_2410_06770_b200.workloads import C3

    a, b, c = C3.buffers()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    outs = []
    for bulk in (True, False):
        kernel_mode("auto", bulk=bulk)
        tc = torch.from_numpy(c).cuda()
        pos, kw = C3.args(ta, tb, tc)
        assert dgett_device(*pos, **kw) == []
        assert g.last_kernel().endswith("_bulk") == bulk, g.last_kernel()
        outs.append(tc.cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes()
