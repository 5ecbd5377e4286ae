"""TMA-fed SGETT operands (sgett_tc.cu, capi.cu tma_layout): when both kernel
operands are affine boxes (rank <= 5, positive strides, K a multiple of 16,
inner k extent a multiple of 8) they are loaded by cp.async.bulk.tensor —
K-major operands as SWIZZLE_32B 8-float boxes, rows-major ones as
[8 k][128 rows] boxes, rows past the view zero-filled.  Every case runs twice,
TMA on and off: the two paths feed the same values to the same MMAs in the
same k order, so C must be bitwise identical, and within the K-normalised
fp32 bar of test_gpu_parity.py of an fp64 contraction.  Bytes outside C's view
never change; non-affine or negative-stride views fall back to the gathers."""
import itertools

import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu


def _inc(dims, order):
    """Increments with `order` fastest first; every stride a multiple of 4
    (16-byte TMA strides), padded so that adjacent modes do not merge."""
    inc = [0] * len(dims)
    step = 1
    for d in order:
        inc[d] = step
        step *= dims[d] + (4 - dims[d] % 4) % 4 + 4
    return inc, step


def _run(a_dims, a_inc, b_dims, b_inc, cont_a, cont_b, M, N, c_row, seed, sign_a=1):
    rng = np.random.default_rng(seed)
    span = lambda ext, inc: sum((e - 1) * abs(i) for e, i in zip(ext, inc)) + 1  # noqa: E731
    a = rng.uniform(-1, 1, span(a_dims, a_inc) + 8).astype(np.float32)
    b = rng.uniform(-1, 1, span(b_dims, b_inc) + 8).astype(np.float32)
    c_inc = (N + 4, 1) if c_row else (1, M + 4)
    off_c = 4
    c = rng.uniform(-1, 1, off_c + (M - 1) * c_inc[0] + (N - 1) * c_inc[1] + 8).astype(np.float32)
    a_inc = [sign_a * i for i in a_inc]
    off_a = 0 if sign_a > 0 else span(a_dims, a_inc) - 1
    return a, a_inc, off_a, b, c, c_inc, off_c


def _strided(buf, ext, inc, off):
    return np.lib.stride_tricks.as_strided(buf[off:], shape=ext,
                                           strides=[i * buf.itemsize for i in inc])


def _c_modes(a_dims, b_dims, cont_a, cont_b, c_inc):
    """C's per-mode increments: the output modes (free A modes, then free B
    modes) flattened row-major into the M x N matrix with increments c_inc."""
    fa = [a_dims[d] for d in range(len(a_dims)) if d not in cont_a]
    fb = [b_dims[d] for d in range(len(b_dims)) if d not in cont_b]
    inc = []
    for ext, step in ((fa, c_inc[0]), (fb, c_inc[1])):
        part = []
        for e in reversed(ext):
            part.append(step)
            step *= e
        inc += list(reversed(part))
    return tuple(inc)


def _contract(a, a_dims, a_inc, off_a, b, b_dims, b_inc, c, c_inc, off_c, nc, cont_a, cont_b):
    ra, rb = len(a_dims), len(b_dims)
    inc_c = _c_modes(a_dims, b_dims, cont_a, cont_b, c_inc)
    errs = g.sgett(ra, a_dims, a_inc, a, rb, b_dims, b_inc, b, nc, cont_a, cont_b,
                   tuple(range(ra + rb - 2 * nc)), inc_c, c, offset_a=off_a, offset_c=off_c)
    assert errs == []
    return g.last_kernel()


CASES = {
    # name: (A dims, B dims, contracted A modes, contracted B modes, free-row modes of A)
    "gemm": ((200, 16, 40), (16, 40, 136), (1, 2), (0, 1)),
    "c5like": ((96, 16, 40), (16, 40, 300), (1, 2), (0, 1)),
    "narrow_n": ((300, 8, 24), (8, 24, 40), (1, 2), (0, 1)),
    "two_row_modes": ((16, 13, 32, 8), (32, 8, 136), (2, 3), (0, 1)),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("a_kf,b_kf,c_row", list(itertools.product([True, False], repeat=3)))
@pytest.mark.parametrize("split", [0, 3])
def test_tma_matches_gathers_and_fp64(name, a_kf, b_kf, c_row, split, kernel_mode):
    a_dims, b_dims, cont_a, cont_b = CASES[name]
    ra = len(a_dims)
    a_free = [d for d in range(ra) if d not in cont_a]
    b_free = [d for d in range(len(b_dims)) if d not in cont_b]
    # K-major: contracted modes fastest (last pair innermost); rows-major: free modes fastest
    a_order = list(reversed(cont_a)) + a_free if a_kf else a_free + list(reversed(cont_a))
    b_order = list(reversed(cont_b)) + b_free if b_kf else b_free + list(reversed(cont_b))
    a_inc, _ = _inc(a_dims, a_order)
    b_inc, _ = _inc(b_dims, b_order)
    M = int(np.prod([a_dims[d] for d in a_free]))
    N = int(np.prod([b_dims[d] for d in b_free]))
    K = int(np.prod([a_dims[d] for d in cont_a]))
    a, a_inc, off_a, b, c0, c_inc, off_c = _run(a_dims, a_inc, b_dims, b_inc, cont_a, cont_b, M, N,
                                                c_row, 7)
    outs, kernels = [], []
    for tma in (True, False):
        kernel_mode("tiled", split=split, tma=tma, kr="off")
        c = c0.copy()
        kernels.append(_contract(a, a_dims, a_inc, off_a, b, b_dims, b_inc, c, c_inc, off_c,
                                 len(cont_a), cont_a, cont_b))
        outs.append(c)
    assert "tma" in kernels[0] and "tma" not in kernels[1], kernels
    assert outs[0].tobytes() == outs[1].tobytes(), kernels
    # fp64 reference (C's view is [free A modes..., free B modes...] flattened to M x N)
    A = _strided(a, a_dims, a_inc, off_a).astype(np.float64)
    B = _strided(b, b_dims, b_inc, 0).astype(np.float64)
    letters = "abcdefgh"
    la = [letters[i] for i in range(ra)]
    lb = [None] * len(b_dims)
    for ca, cb in zip(cont_a, cont_b):
        lb[cb] = la[ca]
    nxt = iter(letters[ra:])
    lb = [x if x is not None else next(nxt) for x in lb]
    out = "".join(la[d] for d in a_free) + "".join(lb[d] for d in b_free)
    prod = np.einsum("".join(la) + "," + "".join(lb) + "->" + out, A, B).reshape(M, N)
    got = _strided(outs[0], (M, N), c_inc, off_c).astype(np.float64)
    want = _strided(c0, (M, N), c_inc, off_c).astype(np.float64) + prod
    err = np.max(np.abs(got - want)) / (K * np.abs(a).max() * np.abs(b).max())
    assert err <= 1e-5, (kernels, err)
    mask = np.ones(len(c0), bool)
    mask[off_c + np.add.outer(np.arange(M) * c_inc[0], np.arange(N) * c_inc[1]).ravel()] = False
    assert outs[0][mask].tobytes() == c0[mask].tobytes()


def test_tma_taken_for_affine_views(kernel_mode):
    """The gemm-shaped affine case runs the TMA kernel (evidence of the path)."""
    kernel_mode("tiled", kr="off")
    a_dims, b_dims, cont_a, cont_b = CASES["gemm"]
    a_inc, _ = _inc(a_dims, [2, 1, 0])
    b_inc, _ = _inc(b_dims, [2, 1, 0])
    a, a_inc, off_a, b, c, c_inc, off_c = _run(a_dims, a_inc, b_dims, b_inc, cont_a, cont_b, 200,
                                               136, True, 3)
    assert "tma" in _contract(a, a_dims, a_inc, off_a, b, b_dims, b_inc, c, c_inc, off_c, 2,
                              cont_a, cont_b)


def test_tma_falls_back_on_negative_strides(kernel_mode):
    """A negative-stride A view is not a TMA box: the gathers run, and the
    result still matches fp64."""
    kernel_mode("tiled", kr="off")
    a_dims, b_dims, cont_a, cont_b = CASES["gemm"]
    a_inc, _ = _inc(a_dims, [2, 1, 0])
    b_inc, _ = _inc(b_dims, [2, 1, 0])
    a, a_inc, off_a, b, c, c_inc, off_c = _run(a_dims, a_inc, b_dims, b_inc, cont_a, cont_b, 200,
                                               136, True, 5, sign_a=-1)
    c0 = c.copy()
    kern = _contract(a, a_dims, a_inc, off_a, b, b_dims, b_inc, c, c_inc, off_c, 2, cont_a, cont_b)
    assert kern.startswith("sgett_tc3xtf32") and "tma" not in kern
    A = _strided(a, a_dims, a_inc, off_a).astype(np.float64)
    B = _strided(b, b_dims, b_inc, 0).astype(np.float64)
    want = _strided(c0, (200, 136), c_inc, off_c) + np.einsum("mij,ijn->mn", A, B)
    got = _strided(c, (200, 136), c_inc, off_c).astype(np.float64)
    assert np.max(np.abs(got - want)) / (640 * np.abs(a).max() * np.abs(b).max()) <= 1e-5


@pytest.mark.parametrize("M,N,K1,K2", [(96, 768, 24, 40), (64, 300, 16, 32), (128, 512, 8, 40)])
def test_pair_kernel_matches_single_cta(M, N, K1, K2, kernel_mode):
    """The CTA-pair kernel (tcgen05.mma.cta_group::2: B' rows 256 per pair in
    the two CTAs' TMEM, the narrow operand split N-wise across the pair's
    shared memory) computes the same products in the same k order as the
    single-CTA TMA kernel: C bitwise equal, and within the fp64 bar."""
    rng = np.random.default_rng(M + N + K1)
    # A (m, k1, k2) rows-major (m fastest); B (n, k1, k2) K-major; C[m, n] m fastest
    a_dims, b_dims = (M, K1, K2), (N, K1, K2)
    a_inc = (1, M + 4, (M + 4) * K1)
    b_inc = (K1 * K2 + 4, K2, 1)
    a = rng.uniform(-1, 1, (M + 4) * K1 * K2 + 8).astype(np.float32)
    b = rng.uniform(-1, 1, N * (K1 * K2 + 4) + 8).astype(np.float32)
    c0 = rng.uniform(-1, 1, (M + 4) * N + 8).astype(np.float32)
    outs, kernels = [], []
    for pair in (True, False):
        kernel_mode("tiled", pair=pair, kr="off")
        c = c0.copy()
        assert g.sgett(3, a_dims, a_inc, a, 3, b_dims, b_inc, b, 2, (1, 2), (1, 2), (0, 1), (1, M + 4), c,
                       offset_c=2) == []
        kernels.append(g.last_kernel())
        outs.append(c)
    assert kernels[0] == "sgett_tc3xtf32_pair_splitk" and "pair" not in kernels[1], kernels
    assert outs[0].tobytes() == outs[1].tobytes(), kernels
    A = _strided(a, a_dims, a_inc, 0).astype(np.float64)
    B = _strided(b, b_dims, b_inc, 0).astype(np.float64)
    want = _strided(c0, (M, N), (1, M + 4), 2).astype(np.float64) + np.einsum("mij,nij->mn", A, B)
    got = _strided(outs[0], (M, N), (1, M + 4), 2).astype(np.float64)
    assert np.max(np.abs(got - want)) / (K1 * K2 * np.abs(a).max() * np.abs(b).max()) <= 1e-5
