"""Layout matrix for the tiled product kernels (tcgen05 SGETT, DMMA DGETT):
every gather path — k-contiguous or rows-contiguous operands, 16-byte vector
or scalar copies, C row- or column-major (which decides the A/B role swap),
K split across two modes with long (40) and short (2 < BK) inner runs, the
K-table slice in smem or the global-table fallback — on ragged M, N, K,
against an fp64 numpy contraction with the K-normalised bar of
test_gpu_parity.py.  Bytes outside C's view must not change."""
import itertools

import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu

TOL = {"s": 1e-5, "d": 1e-12}


def _view(order, dims, vec, rng_pad):
    """Increments for a rank-len(dims) view with the dims in `order`
    (fastest first); vec pads every stride to a multiple of 4, otherwise the
    padded strides are odd."""
    inc = [0] * len(dims)
    step = 1
    for d in order:
        inc[d] = step
        e = dims[d]
        # vec: +4 keeps strides multiples of 4 but stops adjacent modes merging
        pad = (4 - e % 4) % 4 + 4 if vec else (1 if (e + 1) % 2 else 2)
        step *= e + pad + rng_pad
    return inc, step


def _case(dtype, a_kf, a_vec, b_kf, b_vec, c_rowmajor, kmodes, seed, M, N):
    rng = np.random.default_rng(seed)
    k1, k2 = kmodes
    # A (m, k1, k2); B (k1, k2, n); contract A1-B0, A2-B1; C[m, n]
    a_dims, b_dims = (M, k1, k2), (k1, k2, N)
    a_inc, _ = _view((2, 1, 0) if a_kf else (0, 2, 1), a_dims, a_vec, 0)
    b_inc, _ = _view((1, 0, 2) if b_kf else (2, 1, 0), b_dims, b_vec, 0)
    off_a = 0 if a_vec else 1
    off_b = 0 if b_vec else 3
    c_inc = (N + 5, 1) if c_rowmajor else (1, M + 3)
    off_c = 7
    span = lambda ext, inc: sum((e - 1) * i for e, i in zip(ext, inc)) + 1  # noqa: E731
    np_t = np.float32 if dtype == "s" else np.float64
    a = rng.uniform(-1, 1, off_a + span(a_dims, a_inc) + 2).astype(np_t)
    b = rng.uniform(-1, 1, off_b + span(b_dims, b_inc) + 2).astype(np_t)
    c = rng.uniform(-1, 1, off_c + span((M, N), c_inc) + 4).astype(np_t)
    return a, a_dims, a_inc, off_a, b, b_dims, b_inc, off_b, c, c_inc, off_c


def _strided(buf, ext, inc, off):
    return np.lib.stride_tricks.as_strided(buf[off:], shape=ext,
                                           strides=[i * buf.itemsize for i in inc])


LAYOUTS = list(itertools.product([True, False], repeat=5))


@pytest.mark.parametrize("dtype", ["s", "d"])
@pytest.mark.parametrize("kmodes,split", [((25, 40), 0), ((500, 2), 1)])
# (200, 136): square-ish tiles; (24, 300) and (300, 40): one narrow operand
# (mostly-padded tiles, C row-major vs column-major flips the role swap)
@pytest.mark.parametrize("M,N", [(200, 136), (24, 300), (300, 40)])
def test_layout_matrix(dtype, kmodes, split, M, N, kernel_mode):
    kernel_mode("tiled", split=split)
    entry = g.sgett if dtype == "s" else g.dgett
    for i, (a_kf, a_vec, b_kf, b_vec, c_row) in enumerate(LAYOUTS):
        (a, a_dims, a_inc, off_a, b, b_dims, b_inc, off_b, c, c_inc,
         off_c) = _case(dtype, a_kf, a_vec, b_kf, b_vec, c_row, kmodes, 100 + i, M, N)
        c0 = c.copy()
        errs = entry(3, a_dims, a_inc, a, 3, b_dims, b_inc, b, 2, (1, 2), (0, 1), (0, 1), c_inc, c,
                     offset_a=off_a, offset_b=off_b, offset_c=off_c)
        assert errs == []
        A = _strided(a, a_dims, a_inc, off_a).astype(np.float64)
        B = _strided(b, b_dims, b_inc, off_b).astype(np.float64)
        want = _strided(c0, (M, N), c_inc, off_c).astype(np.float64) + np.einsum(
            "mij,ijn->mn", A, B, optimize=True)
        got = _strided(c, (M, N), c_inc, off_c).astype(np.float64)
        k = kmodes[0] * kmodes[1]
        err = np.max(np.abs(got - want)) / (k * np.abs(a).max() * np.abs(b).max())
        assert err <= TOL[dtype], (a_kf, a_vec, b_kf, b_vec, c_row, err)
        # bytes outside the view untouched
        mask = np.ones(len(c), bool)
        idx = off_c + np.add.outer(np.arange(M) * c_inc[0], np.arange(N) * c_inc[1]).ravel()
        mask[idx] = False
        assert c[mask].tobytes() == c0[mask].tobytes()
        assert g.last_kernel().startswith(("sgett_tc3xtf32", "sgett_tctf32bf16") if dtype == "s" else "dgett_dmma")
