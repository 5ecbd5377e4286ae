"""TMA-fed DGETT (dgett_ws.cu TMA path, capi.cu dgett_tma_layout): when both
operands' row and k groups are affine boxes (K and the inner k run multiples
of 32; a 128-row tile = one box) each k-block arrives as one box per operand,
issued by one thread, into the gathers' padded layouts (4 zero-filled
out-of-bounds columns).  Every case runs with TMA on and off: the
same values reach the same DMMAs in the same order, so C must be bitwise
identical, within the fp64 K-normalised bar of an fp64 contraction, and bytes
outside C's view untouched."""
import itertools

import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu


def _inc(dims, order, pad):
    inc = [0] * len(dims)
    step = 1
    for d in order:
        inc[d] = step
        step *= dims[d] + pad
    return inc, step


def _run(M, N, K1, K2, a_kfast, b_kfast, c_nfast, seed, kernel_mode, tma, split=0, stream_k=True):
    rng = np.random.default_rng(seed)
    # A [M, K2, K1], B [K2, K1, N]; contract (1, 2) with (0, 1)
    a_dims, b_dims = (M, K2, K1), (K2, K1, N)
    a_inc, sa = _inc(a_dims, (2, 1, 0) if a_kfast else (0, 2, 1), 2)
    b_inc, sb = _inc(b_dims, (1, 0, 2) if b_kfast else (2, 1, 0), 2)
    c_inc = (N + 2, 1) if c_nfast else (1, M + 2)
    a = rng.uniform(-1, 1, sa + 4)
    b = rng.uniform(-1, 1, sb + 4)
    c0 = rng.uniform(-1, 1, (M + 2) * (N + 2) + 4)
    c = c0.copy()
    kernel_mode("tiled", split=split, stream_k=stream_k, tma=tma)
    assert g.dgett(3, a_dims, tuple(a_inc), a, 3, b_dims, tuple(b_inc), b, 2, (1, 2), (0, 1), (0, 1),
                   c_inc, c) == []
    kname = g.last_kernel()
    A = np.lib.stride_tricks.as_strided(a, a_dims, [8 * i for i in a_inc])
    B = np.lib.stride_tricks.as_strided(b, b_dims, [8 * i for i in b_inc])
    want = np.lib.stride_tricks.as_strided(c0, (M, N), [8 * i for i in c_inc]) + np.einsum("mjk,jkn->mn", A, B)
    got = np.lib.stride_tricks.as_strided(c, (M, N), [8 * i for i in c_inc])
    err = np.max(np.abs(got - want)) / (K1 * K2 * np.abs(a).max() * np.abs(b).max())
    assert err <= 1e-12, err
    mask = np.ones(len(c0), bool)
    mask[(np.arange(M)[:, None] * c_inc[0] + np.arange(N)[None, :] * c_inc[1]).ravel()] = False
    assert c[mask].tobytes() == c0[mask].tobytes()
    return c, kname


@pytest.mark.parametrize("a_kfast,b_kfast,c_nfast", list(itertools.product([True, False], repeat=3)))
@pytest.mark.parametrize("shape", [(384, 256, 32, 5), (128, 384, 64, 2), (640, 128, 96, 3), (100, 90, 32, 2)])
def test_dgett_tma_equals_gathers(shape, a_kfast, b_kfast, c_nfast, kernel_mode):
    M, N, K1, K2 = shape
    seed = M + N + K1
    c_tma, k_tma = _run(M, N, K1, K2, a_kfast, b_kfast, c_nfast, seed, kernel_mode, True)
    c_g, k_g = _run(M, N, K1, K2, a_kfast, b_kfast, c_nfast, seed, kernel_mode, False)
    assert "_tma" in k_tma and "_tma" not in k_g, (k_tma, k_g)
    assert c_tma.tobytes() == c_g.tobytes()


@pytest.mark.parametrize("split,stream_k", [(3, True), (0, False), (0, True)])
def test_dgett_tma_split_and_stream_k(split, stream_k, kernel_mode):
    """split-K partials and persistent stream-K segments (a 1200-tile grid)
    through the TMA producer: bitwise equal to the gather path."""
    M, N, K1, K2 = (1536, 1280, 64, 4) if split == 0 else (256, 256, 32, 12)
    outs = []
    for tma in (True, False):
        c, k = _run(M, N, K1, K2, True, False, True, 7, kernel_mode, tma, split=split, stream_k=stream_k)
        outs.append(c)
        assert ("_tma" in k) == tma, k
    assert outs[0].tobytes() == outs[1].tobytes()


def test_dgett_tma_not_taken_for_k_tails_or_ragged_rows(kernel_mode):
    """K not a multiple of 32 (a -0.0-padded K tail), or a rows-fast operand
    of more than 128 rows whose inner row extent is not a multiple of 128 (its
    padded 132-row box lines would run into the next rows), stays on the
    gathers."""
    _, k = _run(200, 200, 24, 3, True, True, True, 3, kernel_mode, True)
    assert "_tma" not in k, k
    _, k = _run(300, 200, 32, 5, True, False, True, 3, kernel_mode, True)
    assert "_tma" not in k, k
