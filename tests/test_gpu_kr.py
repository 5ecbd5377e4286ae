"""The SGETT k-run kernel (sgett_kr.cu): one k-block = the TMEM operand's
whole contiguous inner k run (<= 64 floats; longer runs are cut into 64-or-
smaller pieces), dense [rows][KR+4] TMA boxes, the rows-major operand
transposed into K-major hi/lo tiles, and split-K partials reduced either
inside the kernel (tile counters, generations, slice claims) or by the
separate reduce kernel.

Every case: within the K-normalised fp32 bar of an fp64 contraction, bytes
outside C's view untouched, and the fused and separate reduces bitwise equal
(same partials, same order).  Shapes cover both operand orientations (C's
fast mode in either operand), run lengths 8..64 and a cut 128-run, output
widths that need N padding (40 -> 48) or several column tiles (200, 300),
row counts off the 128 grid, and forced split counts."""
import numpy as np
import pytest

import paper_2410_06770_b200 as g
from paper_2410_06770_b200.workloads import C5

pytestmark = pytest.mark.gpu


def _strided(buf, ext, inc, off):
    return np.lib.stride_tricks.as_strided(buf[off:], shape=ext, strides=[i * buf.itemsize for i in inc])


def _case(m1, m2, kr, k2, n, c_m_fast, seed):
    """A[m1][m2][k2][kr] (kr contiguous, padded rows), B[kr][k2][n] (n
    contiguous), contract (k2, kr); C[m1][m2][n] with m2 or n fastest."""
    rng = np.random.default_rng(seed)
    ext_a = (m1, m2, k2, kr)
    a_inc = (m2 * k2 * kr + 8, k2 * kr, kr, 1)
    ext_b = (kr, k2, n)
    nb = n + (4 - n % 4) % 4 + 4
    b_inc = (k2 * nb, nb, 1)
    if c_m_fast:
        c_inc = (m2 + 4, 1, m1 * (m2 + 4) + 4)
    else:
        c_inc = (m2 * (n + 4), n + 4, 1)
    span = lambda e, i: sum((x - 1) * y for x, y in zip(e, i)) + 1  # noqa: E731
    a = rng.uniform(-1, 1, span(ext_a, a_inc) + 8).astype(np.float32)
    b = rng.uniform(-1, 1, span(ext_b, b_inc) + 8).astype(np.float32)
    off_c = 4
    c = rng.uniform(-1, 1, off_c + span((m1, m2, n), c_inc) + 8).astype(np.float32)
    pos = (4, ext_a, a_inc, a, 3, ext_b, b_inc, b, 2, (2, 3), (1, 0), (0, 1, 2), c_inc, c)
    return pos, {"offset_c": off_c}


def _check(pos, kw, c0):
    (ra, ext_a, inc_a, a, rb, ext_b, inc_b, b, _, _, _, _, inc_c, c) = pos
    A = _strided(a, ext_a, inc_a, 0).astype(np.float64)
    B = _strided(b, ext_b, inc_b, 0).astype(np.float64)
    ext_c = (ext_a[0], ext_a[1], ext_b[2])
    want = _strided(c0, ext_c, inc_c, kw["offset_c"]).astype(np.float64) + np.einsum("abjk,kjn->abn", A, B)
    got = _strided(c, ext_c, inc_c, kw["offset_c"]).astype(np.float64)
    K = ext_a[2] * ext_a[3]
    err = np.max(np.abs(got - want)) / (K * np.abs(a).max() * np.abs(b).max())
    assert err <= 1e-5, err
    mask = np.ones(len(c0), bool)
    idx = kw["offset_c"] + sum(np.ix_(*[np.arange(e) * i for e, i in zip(ext_c, inc_c)]))
    mask[np.asarray(idx).ravel()] = False
    assert c[mask].tobytes() == c0[mask].tobytes()


SHAPES = [
    # (m1, m2, kr, k2, n)
    (6, 16, 40, 24, 96),     # c5-like
    (3, 50, 8, 64, 128),
    (2, 64, 16, 30, 40),     # N padded 40 -> 48
    (5, 40, 24, 20, 200),    # two column tiles
    (1, 200, 32, 12, 300),   # three column tiles, 200 rows
    (4, 32, 48, 10, 64),
    (2, 48, 56, 9, 80),
    (3, 33, 64, 8, 64),
    (2, 64, 128, 6, 96),     # a 128-run cut into 64-float k-blocks
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("c_m_fast", [True, False])
@pytest.mark.parametrize("split", [0, 1, 5])
@pytest.mark.parametrize("mixed", [True, False], ids=["tf32bf16", "3xtf32"])
def test_kr_kernel_matches_fp64_fused_equals_separate(shape, c_m_fast, split, mixed, kernel_mode):
    """single CTAs and CTA pairs (where the tiling allows; pairs may take two
    k runs per k-block, which moves the split-K cuts), fused and separate
    reduce, the mixed (tf32 + bf16) and the 3xTF32 split: each within the bar,
    fused == separate bitwise for each form."""
    m1, m2, kr, k2, n = shape
    names = []
    for pair in (True, False):
        outs = []
        for fused in (True, False):
            pos, kw = _case(m1, m2, kr, k2, n, c_m_fast, seed=sum(shape) + split)
            c0 = pos[13].copy()
            kernel_mode("tiled", split=split, kr="force", kr_fused=fused, kr_pair=pair, kr_mixed=mixed)
            assert g.sgett(*pos, **kw) == []
            kname = g.last_kernel()
            assert kname.startswith("sgett_tctf32bf16_kr" if mixed else "sgett_tc3xtf32_kr"), kname
            _check(pos, kw, c0)
            outs.append(pos[13])
            names.append(kname)
        assert outs[0].tobytes() == outs[1].tobytes(), names
    assert not any("pair" in k for k in names[2:]), names


def test_kr_auto_on_c5_and_off_for_large_tilings(kernel_mode):
    """Automatic choice: c5 (a 40-float run, 6 output tiles) takes the
    k-run kernel; a 1024^3 GEMM (64 tiles, 64-float k-blocks) does not."""
    kernel_mode("auto")
    a, b, c = C5.buffers()
    pos, kw = C5.args(a, b, c)
    assert g.sgett(*pos, **kw) == []
    assert g.last_kernel().startswith(("sgett_tc3xtf32_kr", "sgett_tctf32bf16_kr"))
    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, 1024 * 1024).astype(np.float32)
    B = rng.uniform(-1, 1, 1024 * 1024).astype(np.float32)
    C = np.zeros(1024 * 1024, np.float32)
    assert g.sgett(2, (1024, 1024), (1024, 1), A, 2, (1024, 1024), (1024, 1), B, 1, (1,), (0,), (0, 1),
                   (1024, 1), C) == []
    assert "kr" not in g.last_kernel()


def test_kr_c5_equals_tiled_bitwise(kernel_mode):
    """On c5 both tcgen05 kernels (one-CTA form, three tf32 MMAs) cut K at the same points
    (1280 = 32 runs of 40 = 80 blocks of 16) and issue the same MMAs in the
    same k order: the results are bit-identical."""
    outs = []
    for kr in ("force", "off"):
        kernel_mode("tiled", kr=kr, kr_pair=False, kr_mixed=False)
        a, b, c = C5.buffers()
        pos, kw = C5.args(a, b, c)
        assert g.sgett(*pos, **kw) == []
        outs.append(c)
    assert outs[0].tobytes() == outs[1].tobytes()


def test_kr_graph_replay_fused(kernel_mode):
    """The fused reduce's counters reset themselves: a CUDA graph of a k-run
    split-K call replays to the same bits as direct calls."""
    import torch

    from paper_2410_06770_b200.device import sgett_device
    from paper_2410_06770_b200.graph import GettGraph

    kernel_mode("tiled", kr="force")
    w = C5.slice_free("A", 0, 0, 16)
    a, b, c = w.buffers()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    direct = torch.from_numpy(c).cuda()
    pos, kw = w.args(ta, tb, direct)
    for _ in range(3):
        assert sgett_device(*pos, **kw) == []
    tc = torch.from_numpy(c).cuda()
    pos, kw = w.args(ta, tb, tc)
    gg = GettGraph(sgett_device, *pos, **kw)
    assert g.last_kernel().startswith(("sgett_tc3xtf32_kr", "sgett_tctf32bf16_kr"))
    for _ in range(2):
        gg.replay()
    torch.cuda.synchronize()
    assert torch.equal(tc, direct)


def test_kr_pair_taken_on_c5(kernel_mode):
    kernel_mode("auto")
    a, b, c = C5.buffers()
    pos, kw = C5.args(a, b, c)
    assert g.sgett(*pos, **kw) == []
    assert g.last_kernel().startswith("sgett_tctf32bf16_kr_pair"), g.last_kernel()


@pytest.mark.parametrize("ny", [189, 193, 320])
def test_kr_pair_second_column_tile_half_out_of_range(ny, kernel_mode):
    """CTA pairs split each 128-column tile in two halves; with NY = 189 the
    second tile's second half (rows 192..255) is wholly past the tensor — its
    box is not loaded (a fully out-of-bounds box faults) and its columns are
    never stored."""
    kernel_mode("tiled", kr="force")
    rng = np.random.default_rng(ny)
    na, nb, k = ny, 175, 16
    inc_a, inc_b = (1, na + 7 + (4 - (na + 7) % 4) % 4), (k + 4, 1)
    a = rng.uniform(-1, 1, inc_a[1] * k + 8).astype(np.float32)
    b = rng.uniform(-1, 1, (k + 4) * nb + 8).astype(np.float32)
    c0 = rng.uniform(-1, 1, 3 + (nb + 1) * na + 8).astype(np.float32)
    c = c0.copy()
    assert g.sgett(2, (na, k), inc_a, a, 2, (nb, k), inc_b, b, 1, (1,), (1,), (0, 1), (nb + 1, 1), c,
                   offset_c=3) == []
    assert g.last_kernel().startswith(("sgett_tc3xtf32_kr", "sgett_tctf32bf16_kr")), g.last_kernel()
    A = _strided(a, (na, k), inc_a, 0).astype(np.float64)
    B = _strided(b, (nb, k), inc_b, 0).astype(np.float64)
    want = _strided(c0, (na, nb), (nb + 1, 1), 3).astype(np.float64) + A @ B.T
    got = _strided(c, (na, nb), (nb + 1, 1), 3).astype(np.float64)
    assert np.abs(got - want).max() / (k * np.abs(a).max() * np.abs(b).max()) <= 1e-5


def test_kr_mixed_split_at_least_as_accurate_as_3xtf32(kernel_mode):
    """The mixed split (one tf32 MMA of tf32-rounded hi parts + one bf16 MMA
    carrying both cross terms) against the three-MMA truncation split on c5
    and on a short-K case: its error against fp64 is no larger than 1.25x the
    3xTF32 error (it is smaller on c5: rounding the hi parts removes the
    truncation split's one-signed lo*lo term), and on integer data both are
    exact."""
    from oracle import oracle

    def err_of(w, mixed):
        a, b, c = w.buffers()
        ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                                  w.conts, w.cont_a, w.cont_b, w.perm)
        ref = ref + oracle.strided(c, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
        kernel_mode("tiled", kr="force", kr_mixed=mixed)
        pos, kw = w.args(a, b, c)
        assert g.sgett(*pos, **kw) == []
        assert ("tf32bf16" in g.last_kernel()) == mixed, g.last_kernel()
        return np.max(np.abs(oracle.strided(c, w.ext_c, w.inc_c, w.off_c) - ref))

    for w in (C5, C5.slice_free("A", 0, 0, 16)):
        e_mix, e_3x = err_of(w, True), err_of(w, False)
        assert e_mix <= 1.25 * e_3x, (w.name, e_mix, e_3x)
    # integer data (|x| <= 8): hi parts exact, lo parts zero -> exact sums
    pos, kw = _case(3, 50, 8, 64, 128, True, seed=5)
    pos = list(pos)
    for i in (3, 7, 13):
        pos[i] = np.rint(pos[i] * 8).astype(np.float32)
    outs = []
    for mixed in (True, False):
        c = pos[13].copy()
        kernel_mode("tiled", kr="force", kr_mixed=mixed)
        assert g.sgett(*pos[:13], c, **kw) == []
        outs.append(c)
    assert outs[0].tobytes() == outs[1].tobytes()


def test_kr_pdl_on_off_bitwise(kernel_mode):
    """Programmatic dependent launch only changes when the k-run kernel and the
    reduce are scheduled: back-to-back calls on one stream (each a dependent of
    the previous call's reduce, whose workspace it reuses) give the same bits as
    ordinary launches, for the separate and the fused reduce."""
    import torch

    from paper_2410_06770_b200.device import sgett_device

    w = C5.slice_free("A", 0, 0, 24)
    a, b, c = w.buffers()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for fused in (False, True):
        outs = []
        for pdl in (True, False):
            g.set_pdl(pdl)
            try:
                kernel_mode("tiled", kr="force", kr_fused=fused)
                tc = torch.from_numpy(c).cuda()
                pos, kw = w.args(ta, tb, tc)
                for _ in range(5):  # C accumulates: 5 dependent calls
                    assert sgett_device(*pos, **kw) == []
                torch.cuda.synchronize()
                outs.append(tc.cpu().numpy())
            finally:
                g.set_pdl(True)
        assert outs[0].tobytes() == outs[1].tobytes(), fused
