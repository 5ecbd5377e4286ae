"""Randomised descriptors through the tiled kernels: ranks 2-4, one to three
contracted pairs, random mode orders and paddings (strides multiples of 4, so
the TMA SGETT path is eligible whenever K is a multiple of 16), random C
layouts and offsets.  Each case is checked against an fp64 contraction with
the K-normalised bar of test_gpu_parity.py, bytes outside C's view must not
change, and for fp32 the TMA and gather paths must agree bitwise."""
import numpy as np
import pytest

import paper_2410_06770_b200 as g

pytestmark = pytest.mark.gpu

TOL = {"s": 1e-5, "d": 1e-12}


def _case(rng):
    while True:
        c = _draw(rng)
        size_c = int(np.prod(c[10]))
        k = int(np.prod([c[0][d] for d in c[7]]))
        if size_c <= 400_000 and k <= 2048:
            return c


def _draw(rng):
    conts = int(rng.integers(1, 4))
    fa, fb = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    kext = [int(rng.choice([2, 4, 8, 16, 24, 40])) for _ in range(conts)]
    fea = [int(rng.integers(8, 200)) for _ in range(fa)]
    feb = [int(rng.integers(8, 200)) for _ in range(fb)]
    # positions of contracted modes inside A and B
    ra, rb = fa + conts, fb + conts
    pos_a = list(rng.permutation(ra))
    pos_b = list(rng.permutation(rb))
    cont_a = tuple(int(x) for x in pos_a[:conts])
    cont_b = tuple(int(x) for x in pos_b[:conts])
    ext_a, ext_b = [0] * ra, [0] * rb
    for k, (ia, ib) in enumerate(zip(cont_a, cont_b)):
        ext_a[ia] = ext_b[ib] = kext[k]
    for d, e in zip(pos_a[conts:], fea):
        ext_a[d] = e
    for d, e in zip(pos_b[conts:], feb):
        ext_b[d] = e

    def incs(ext):
        order = rng.permutation(len(ext))
        inc, step = [0] * len(ext), 1
        for d in order:
            inc[d] = step
            pad = int(rng.choice([0, 4, 8]))
            step *= ext[d] + pad + (4 - ext[d] % 4) % 4
        return tuple(inc), step

    inc_a, span_a = incs(ext_a)
    inc_b, span_b = incs(ext_b)
    rc = fa + fb
    perm = tuple(int(x) for x in rng.permutation(rc))
    ext_c = [0] * rc
    free = [ext_a[d] for d in range(ra) if d not in cont_a] + [ext_b[d] for d in range(rb) if d not in cont_b]
    for i, e in enumerate(free):
        ext_c[perm[i]] = e
    inc_c, span_c = incs(ext_c)
    return (ext_a, inc_a, span_a, ext_b, inc_b, span_b, conts, cont_a, cont_b, perm, ext_c, inc_c, span_c)


def _strided(buf, ext, inc, off):
    return np.lib.stride_tricks.as_strided(buf[off:], shape=ext, strides=[i * buf.itemsize for i in inc])


@pytest.mark.parametrize("dtype", ["s", "d"])
def test_random_descriptors(dtype, kernel_mode):
    rng = np.random.default_rng(2024 if dtype == "s" else 2025)
    np_t = np.float32 if dtype == "s" else np.float64
    entry = g.sgett if dtype == "s" else g.dgett
    letters = "abcdefghijklmnop"
    n_tma = 0
    for case_i in range(150):
        (ext_a, inc_a, span_a, ext_b, inc_b, span_b, conts, cont_a, cont_b, perm, ext_c, inc_c,
         span_c) = _case(rng)
        off_a, off_b, off_c = (int(rng.integers(0, 3)) * 4 for _ in range(3))
        a = rng.uniform(-1, 1, off_a + span_a + 4).astype(np_t)
        b = rng.uniform(-1, 1, off_b + span_b + 4).astype(np_t)
        c0 = rng.uniform(-1, 1, off_c + span_c + 4).astype(np_t)
        outs = []
        for tma in ((True, False) if dtype == "s" else (True,)):
            # (the tcgen05 kernel's TMA and gather paths: same MMAs, same k
            # order; the k-run kernel has its own tests, test_gpu_kr.py)
            kernel_mode("tiled", tma=tma, kr="off")
            c = c0.copy()
            assert entry(len(ext_a), tuple(ext_a), inc_a, a, len(ext_b), tuple(ext_b), inc_b, b, conts, cont_a,
                         cont_b, perm, inc_c, c, offset_a=off_a, offset_b=off_b, offset_c=off_c) == []
            if tma and "tma" in g.last_kernel():
                n_tma += 1
            outs.append(c)
        if dtype == "s":
            assert outs[0].tobytes() == outs[1].tobytes(), case_i
        # fp64 reference
        la = [letters[i] for i in range(len(ext_a))]
        lb = [None] * len(ext_b)
        for ia, ib in zip(cont_a, cont_b):
            lb[ib] = la[ia]
        nxt = iter(letters[len(ext_a):])
        lb = [x if x is not None else next(nxt) for x in lb]
        free_l = [la[d] for d in range(len(ext_a)) if d not in cont_a] + \
                 [lb[d] for d in range(len(ext_b)) if d not in cont_b]
        out_l = [None] * len(free_l)
        for i, l in enumerate(free_l):
            out_l[perm[i]] = l
        A = _strided(a, ext_a, inc_a, off_a).astype(np.float64)
        B = _strided(b, ext_b, inc_b, off_b).astype(np.float64)
        prod = np.einsum("".join(la) + "," + "".join(lb) + "->" + "".join(out_l), A, B, optimize=True)
        want = _strided(c0, ext_c, inc_c, off_c).astype(np.float64) + prod
        got = _strided(outs[0], ext_c, inc_c, off_c).astype(np.float64)
        K = int(np.prod([ext_a[d] for d in cont_a]))
        err = np.max(np.abs(got - want)) / (K * np.abs(a).max() * np.abs(b).max())
        assert err <= TOL[dtype], (case_i, g.last_kernel(), err)
        mask = np.ones(len(c0), bool)
        idx = off_c + sum(np.ix_(*[np.arange(e) * i for e, i in zip(ext_c, inc_c)]))
        mask[np.asarray(idx).ravel()] = False
        assert outs[0][mask].tobytes() == c0[mask].tobytes(), case_i
    if dtype == "s":
        assert n_tma > 0  # the TMA path was exercised


@pytest.mark.parametrize("dtype", ["s", "d"])
def test_random_descriptors_auto_mode_negative_strides(dtype, kernel_mode):
    """The same generator in auto mode (ref / dot / tiled / split-K chosen by
    size) with some increments negated (base offsets moved to the high end)."""
    rng = np.random.default_rng(7 if dtype == "s" else 8)
    np_t = np.float32 if dtype == "s" else np.float64
    entry = g.sgett if dtype == "s" else g.dgett
    letters = "abcdefghijklmnop"
    kernel_mode("auto")
    kernels = set()
    for case_i in range(120):
        (ext_a, inc_a, span_a, ext_b, inc_b, span_b, conts, cont_a, cont_b, perm, ext_c, inc_c,
         span_c) = _case(rng)
        # shrink some cases so the ref / dot kernels are chosen too
        if case_i % 3 == 0:
            ext_a = [min(e, 6) if d not in cont_a else e for d, e in enumerate(ext_a)]
            ext_b = [min(e, 6) if d not in cont_b else e for d, e in enumerate(ext_b)]
            free = [ext_a[d] for d in range(len(ext_a)) if d not in cont_a] + \
                   [ext_b[d] for d in range(len(ext_b)) if d not in cont_b]
            ext_c = [0] * len(free)
            for i, e in enumerate(free):
                ext_c[perm[i]] = e
        sign = lambda inc: tuple(i if rng.random() < 0.7 else -i for i in inc)  # noqa: E731
        inc_a, inc_b = sign(inc_a), sign(inc_b)
        low = lambda ext, inc: -sum((e - 1) * i for e, i in zip(ext, inc) if i < 0)  # noqa: E731
        off_a, off_b, off_c = low(ext_a, inc_a), low(ext_b, inc_b), 3
        a = rng.uniform(-1, 1, span_a + 8).astype(np_t)
        b = rng.uniform(-1, 1, span_b + 8).astype(np_t)
        c0 = rng.uniform(-1, 1, off_c + span_c + 4).astype(np_t)
        c = c0.copy()
        assert entry(len(ext_a), tuple(ext_a), inc_a, a, len(ext_b), tuple(ext_b), inc_b, b, conts, cont_a,
                     cont_b, perm, inc_c, c, offset_a=off_a, offset_b=off_b, offset_c=off_c) == []
        kernels.add(g.last_kernel())
        la = [letters[i] for i in range(len(ext_a))]
        lb = [None] * len(ext_b)
        for ia, ib in zip(cont_a, cont_b):
            lb[ib] = la[ia]
        nxt = iter(letters[len(ext_a):])
        lb = [x if x is not None else next(nxt) for x in lb]
        free_l = [la[d] for d in range(len(ext_a)) if d not in cont_a] + \
                 [lb[d] for d in range(len(ext_b)) if d not in cont_b]
        out_l = [None] * len(free_l)
        for i, l in enumerate(free_l):
            out_l[perm[i]] = l
        A = _strided(a, ext_a, inc_a, off_a).astype(np.float64)
        B = _strided(b, ext_b, inc_b, off_b).astype(np.float64)
        prod = np.einsum("".join(la) + "," + "".join(lb) + "->" + "".join(out_l), A, B, optimize=True)
        want = _strided(c0, ext_c, inc_c, off_c).astype(np.float64) + prod
        got = _strided(c, ext_c, inc_c, off_c).astype(np.float64)
        K = int(np.prod([ext_a[d] for d in cont_a]))
        err = np.max(np.abs(got - want)) / (K * np.abs(a).max() * np.abs(b).max())
        assert err <= TOL[dtype], (case_i, g.last_kernel(), err)
        mask = np.ones(len(c0), bool)
        idx = off_c + sum(np.ix_(*[np.arange(e) * i for e, i in zip(ext_c, inc_c)]))
        mask[np.asarray(idx).ravel()] = False
        assert c[mask].tobytes() == c0[mask].tobytes(), case_i
    assert len(kernels) >= 2, kernels


@pytest.mark.parametrize("dtype", ["c", "z"])
def test_random_complex_descriptors_embedded_and_4x(dtype, kernel_mode):
    """cgett/zgett on the tiled kernels through both complex schemes: the one
    real GETT on an embedding of the smaller operand (default) and the four
    real GETTs on re/im sub-views.  Both against a complex128 contraction,
    bytes outside C's view unchanged."""
    rng = np.random.default_rng(31 if dtype == "c" else 32)
    np_t = np.complex64 if dtype == "c" else np.complex128
    entry = g.cgett if dtype == "c" else g.zgett
    tol = TOL["s" if dtype == "c" else "d"] * 2
    letters = "abcdefghijklmnop"
    names = set()
    for case_i in range(40):
        (ext_a, inc_a, span_a, ext_b, inc_b, span_b, conts, cont_a, cont_b, perm, ext_c, inc_c,
         span_c) = _case(rng)
        off_a, off_b, off_c = (int(rng.integers(0, 3)) for _ in range(3))
        draw = lambda n: (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np_t)  # noqa: E731
        a, b, c0 = draw(off_a + span_a + 2), draw(off_b + span_b + 2), draw(off_c + span_c + 2)
        la = [letters[i] for i in range(len(ext_a))]
        lb = [None] * len(ext_b)
        for ia, ib in zip(cont_a, cont_b):
            lb[ib] = la[ia]
        nxt = iter(letters[len(ext_a):])
        lb = [x if x is not None else next(nxt) for x in lb]
        free_l = [la[d] for d in range(len(ext_a)) if d not in cont_a] + \
                 [lb[d] for d in range(len(ext_b)) if d not in cont_b]
        out_l = [None] * len(free_l)
        for i, l in enumerate(free_l):
            out_l[perm[i]] = l
        A = _strided(a, ext_a, inc_a, off_a).astype(np.complex128)
        B = _strided(b, ext_b, inc_b, off_b).astype(np.complex128)
        prod = np.einsum("".join(la) + "," + "".join(lb) + "->" + "".join(out_l), A, B, optimize=True)
        want = _strided(c0, ext_c, inc_c, off_c).astype(np.complex128) + prod
        K = int(np.prod([ext_a[d] for d in cont_a]))
        mask = np.ones(len(c0), bool)
        idx = off_c + sum(np.ix_(*[np.arange(e) * i for e, i in zip(ext_c, inc_c)]))
        mask[np.asarray(idx).ravel()] = False
        for embed in (True, False):
            kernel_mode("tiled", complex_embed=embed)
            c = c0.copy()
            assert entry(len(ext_a), tuple(ext_a), inc_a, a, len(ext_b), tuple(ext_b), inc_b, b, conts, cont_a,
                         cont_b, perm, inc_c, c, offset_a=off_a, offset_b=off_b, offset_c=off_c) == []
            names.add(g.last_kernel())
            got = _strided(c, ext_c, inc_c, off_c).astype(np.complex128)
            err = np.max(np.abs(got - want)) / (K * np.abs(a).max() * np.abs(b).max())
            assert err <= tol, (case_i, embed, g.last_kernel(), err)
            assert c[mask].tobytes() == c0[mask].tobytes(), (case_i, embed)
    assert any("embedded" in n for n in names) and any("4x" in n for n in names), names


@pytest.mark.parametrize("embed", [True, False])
def test_complex_edge_shapes(embed, kernel_mode):
    """The complex schemes on edge shapes: a stride-0 (broadcast) mode in the
    expanded operand, the smaller operand on either side, a matrix-vector
    contraction (C rank 1), a scalar output (C rank 0) and a K of one."""
    kernel_mode("tiled", complex_embed=embed)
    rng = np.random.default_rng(77)
    draw = lambda n, dt: (rng.integers(-3, 4, n) + 1j * rng.integers(-3, 4, n)).astype(dt)  # noqa: E731
    for dt, entry in ((np.complex64, g.cgett), (np.complex128, g.zgett)):
        # B (300 x 20, its column mode of stride 0) smaller than A (600 x 300):
        # the broadcast operand is the one the embedded scheme expands
        a = draw(600 * 300, dt)
        b = draw(300, dt)
        c = draw(600 * 20, dt)
        want = c.astype(np.complex128).reshape(600, 20) + \
            (a.astype(np.complex128).reshape(600, 300) @ np.repeat(b.astype(np.complex128)[:, None], 20, 1))
        assert entry(2, (600, 300), (300, 1), a, 2, (300, 20), (1, 0), b, 1, (1,), (0,), (0, 1), (20, 1), c) == []
        assert np.array_equal(c.reshape(600, 20), want.astype(dt)), (dt, g.last_kernel())
        assert ("embedded" in g.last_kernel()) == embed, g.last_kernel()
        # B smaller than A: (600 x 64) x (64 x 8)
        a = draw(600 * 64, dt)
        b = draw(64 * 8, dt)
        c = draw(600 * 8, dt)
        want = c.astype(np.complex128).reshape(600, 8) + a.astype(np.complex128).reshape(600, 64) @ \
            b.astype(np.complex128).reshape(64, 8)
        assert entry(2, (600, 64), (64, 1), a, 2, (64, 8), (8, 1), b, 1, (1,), (0,), (0, 1), (8, 1), c) == []
        assert np.array_equal(c.reshape(600, 8), want.astype(dt)), (dt, g.last_kernel())
        # matrix-vector: C rank 1
        a = draw(700 * 90, dt)
        b = draw(90, dt)
        c = draw(700, dt)
        want = c.astype(np.complex128) + a.astype(np.complex128).reshape(700, 90) @ b.astype(np.complex128)
        assert entry(2, (700, 90), (90, 1), a, 1, (90,), (1,), b, 1, (1,), (0,), (0,), (1,), c) == []
        assert np.array_equal(c, want.astype(dt)), (dt, g.last_kernel())
        # scalar output: full contraction of two 30 x 40 tensors
        a = draw(1200, dt)
        b = draw(1200, dt)
        c = draw(1, dt)
        want = c.astype(np.complex128) + np.sum(a.astype(np.complex128).reshape(30, 40) *
                                                b.astype(np.complex128).reshape(40, 30).T)
        assert entry(2, (30, 40), (40, 1), a, 2, (40, 30), (30, 1), b, 2, (0, 1), (1, 0), (), (), c) == []
        assert np.array_equal(c, want.astype(dt)), (dt, g.last_kernel())
        # K of one (outer product)
        a = draw(200, dt)
        b = draw(300, dt)
        c = draw(200 * 300, dt)
        want = c.astype(np.complex128).reshape(200, 300) + np.outer(a, b).astype(np.complex128)
        assert entry(2, (200, 1), (1, 1), a, 2, (1, 300), (300, 1), b, 1, (1,), (0,), (0, 1), (300, 1), c) == []
        assert np.array_equal(c.reshape(200, 300), want.astype(dt)), (dt, g.last_kernel())
