"""Multi-device xGETT in one call (include/gett_b200.h
gett_{d,s}gett_multi): slabs of C's outermost free mode across devices with
the replicated operand exchanged over NVLink, or split-K with one reduce on
devices[0] loading the peers' partials.

A device listed twice is two lanes (own streams, staging, partial buffers),
so the whole path — chunked replicated-operand upload + peer exchange, per
lane pipelined slabs, partial buffers and the ordered reduce — runs on the
single GPU a test box has, with devices=(0, 0) / (0, 0, 0).

Bars: golden suite (reference outputs) bitwise on integer data and within
err_K otherwise, for both strategies; full BASELINE configs within err_K of
fp64 with the padding untouched; slabs bitwise equal to a one-device call
when per-slab schedules match (ref-order kernel).
"""
import numpy as np
import pytest

import paper_2410_06770_b200 as g
from oracle import oracle
from tests.golden_util import load_suite, view_offsets
from tests.test_gpu_parity import ENTRY, TOL_K, k_norm_err

pytestmark = pytest.mark.gpu

SUITE = [c for c in load_suite() if c.dtype in "ds"]


@pytest.fixture
def multi():
    def use(strategy="auto", staged=False):
        g.set_multi(strategy, staged)
    yield use
    g.set_multi("auto")
    g.set_devices(None)


def _suite_case(case, devices):
    a, b, c = case.buffers()
    before = c.copy()
    pos, kw = case.args(a, b, c)
    errs = ENTRY[case.dtype](*pos, **kw, devices=devices)
    assert errs == [], errs
    offs = case.c_offsets()
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == before[mask].tobytes(), "bytes outside the C view changed"
    got = c[offs]
    if case.data == "int":
        assert got.tobytes() == case.want.tobytes(), "not bitwise equal to the reference"
    else:
        k = int(np.prod([case.a["ext"][d] for d in case.cont_a])) if case.conts else 1
        assert k_norm_err(got, case.want, k) <= TOL_K[case.dtype]


@pytest.mark.parametrize("strategy,devices", [("slabs", (0, 0)), ("slabs", (0, 0, 0)),
                                              ("splitk", (0, 0)), ("splitk", (0, 0, 0))])
def test_golden_suite_multi(strategy, devices, multi, kernel_mode):
    kernel_mode("auto")
    multi(strategy)
    fails, used = [], 0
    for case in SUITE:
        try:
            _suite_case(case, devices)
            used += g.last_multi() != "none"
        except AssertionError as e:
            fails.append(f"{case.id}: {e}")
    assert not fails, f"{len(fails)} failures, first: {fails[:5]}"
    assert used > len(SUITE) // 4, (used, len(SUITE))  # the forced strategy ran on most cases


def test_golden_suite_splitk_staged_reduce(multi, kernel_mode):
    kernel_mode("auto")
    multi("splitk", staged=True)
    fails = []
    for case in SUITE[::3]:
        try:
            _suite_case(case, (0, 0, 0))
        except AssertionError as e:
            fails.append(f"{case.id}: {e}")
    assert not fails, fails[:5]


def test_validation_errors_unchanged_by_devices(multi):
    a, b, c = np.ones(6), np.ones(6), np.zeros(4)
    want = g.dgett(2, (2, 3), (3, 1), a, 2, (2, 3), (3, 1), b, 1, (1,), (0,), (0, 1), (2, 1), c)
    got = g.dgett(2, (2, 3), (3, 1), a, 2, (2, 3), (3, 1), b, 1, (1,), (0,), (0, 1), (2, 1), c,
                  devices=(0, 0))
    assert [(e.code, e.message) for e in got] == [(e.code, e.message) for e in want] != []
    assert c.tolist() == [0.0] * 4


def _full(name, devices):
    from paper_2410_06770_b200.workloads import CONFIGS as W

    w = W[name]
    a, b, c = w.buffers()
    c0 = c.copy()
    pos, kw = w.args(a, b, c)
    assert ENTRY[w.dtype](*pos, **kw, devices=devices) == []
    sched = g.last_multi()
    offs = view_offsets(w.ext_c, w.inc_c, w.off_c)
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == c0[mask].tobytes()
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    ref = ref + oracle.strided(c0, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
    got = oracle.strided(c, w.ext_c, w.inc_c, w.off_c)
    err = k_norm_err(got, ref, w.size_k, float(np.abs(a).max()), float(np.abs(b).max()))
    assert err <= TOL_K[w.dtype], (name, err)
    return sched


@pytest.mark.parametrize("name,devices,expect", [
    ("c2", (0, 0), "slabs x2"), ("c3", (0, 0, 0), "slabs x3"), ("c4", (0, 0), "slabs x2"),
    ("c5", (0, 0), "split-K x2"), ("c5", (0, 0, 0, 0), "split-K x4"), ("c1", (0, 0), "none")])
def test_full_configs_multi_auto(name, devices, expect, multi, kernel_mode):
    """Automatic schedule: the free-mode configs shard by slabs, c5 (6 output
    tiles) splits K, c1 (1.2 M MACs) stays on one device."""
    kernel_mode("auto")
    multi("auto")
    sched = _full(name, devices)
    assert sched.startswith(expect), sched


def test_c5_splitk_staged_equals_peer_load(multi, kernel_mode):
    """The two reduce forms read the same partials in the same order."""
    from paper_2410_06770_b200.workloads import C5

    kernel_mode("auto")
    out = []
    for staged in (False, True):
        multi("splitk", staged)
        a, b, c = C5.buffers()
        pos, kw = C5.args(a, b, c)
        assert g.sgett(*pos, **kw, devices=(0, 0, 0)) == []
        assert ("staged" if staged else "peer-load") in g.last_multi()
        out.append(c)
    assert out[0].tobytes() == out[1].tobytes()


def test_slabs_bitwise_equal_one_device_ref_order(multi, kernel_mode):
    """With the reference-order kernel each element's sum does not depend on
    the tiling, so the slab schedule equals a one-device call bit for bit."""
    from paper_2410_06770_b200.workloads import C3

    w = C3.slice_free("A", 0, 0, 24)
    kernel_mode("ref")
    multi("slabs")
    a, b, c = w.buffers()
    one = c.copy()
    pos, kw = w.args(a, b, one)
    assert g.dgett(*pos, **kw) == []
    pos, kw = w.args(a, b, c)
    assert g.dgett(*pos, **kw, devices=(0, 0, 0)) == []
    assert g.last_multi().startswith("slabs x3")
    assert c.tobytes() == one.tobytes()


def test_set_devices_default_applies_to_drop_in_signature(multi, kernel_mode):
    """set_devices() makes the unchanged reference signature multi-device."""
    from paper_2410_06770_b200.workloads import C3

    kernel_mode("auto")
    w = C3.slice_free("A", 0, 0, 64)
    a, b, c = w.buffers()
    want = c.copy()
    pos, kw = w.args(a, b, want)
    assert g.dgett(*pos, **kw) == []
    g.set_devices((0, 0))
    multi("slabs")
    pos, kw = w.args(a, b, c)
    assert g.dgett(*pos, **kw) == []
    assert g.last_multi().startswith("slabs x2")
    g.set_devices(None)
    assert k_norm_err(c, want, w.size_k) <= 1e-12


def test_bad_device_ordinal_raises(multi):
    a, b, c = np.ones(4), np.ones(4), np.zeros(1)
    with pytest.raises(g.GettRuntimeError):
        g.dgett(1, (4,), (1,), a, 1, (4,), (1,), b, 1, (0,), (0,), (), (), c, devices=(0, 63))
    assert c[0] == 0.0


# ---------------------------------------------------------------------------
# pack (testkit.py:101-103) on the device


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.complex64, np.complex128])
def test_pack_equals_fancy_index(dtype):
    rng = np.random.default_rng(5)
    buf = rng.standard_normal(5000).astype(dtype)
    if np.iscomplexobj(buf):
        buf = buf + 1j * rng.standard_normal(5000).astype(dtype)
    buf[7] = -0.0
    for ext, inc, off in [((3, 4, 5), (1, 3, 12), 0), ((6, 7), (-9, 1), 60), ((5, 1, 4), (200, 0, -30), 100),
                          ((), (), 17), ((0, 3), (1, 1), 0), ((8, 8, 8, 4), (2, 16, 128, 1024), 1)]:
        v = g.TensorView(len(ext), ext, inc, off, len(buf))
        got = g.pack(v, buf)
        want = buf[view_offsets(ext, inc, off)] if ext else buf[off:off + 1]
        assert got.tobytes() == want.tobytes(), (ext, inc, off)


def test_pack_device_and_bounds():
    import torch

    from paper_2410_06770_b200.device import pack_device

    buf = torch.arange(1000, dtype=torch.float64, device="cuda")
    v = g.TensorView(2, (10, 7), (3, 100), 5, 1000)
    got = pack_device(v, buf).cpu().numpy()
    assert np.array_equal(got, np.arange(1000.0)[view_offsets((10, 7), (3, 100), 5)])
    with pytest.raises(IndexError):
        g.pack(g.TensorView(1, (10,), (200,), 0, 5000), np.zeros(1000))
