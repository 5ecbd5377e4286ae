"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden vectors were produced by running the reference gett.kernel.dgett /
sgett (tests/golden/make_golden.py); the oracle must reproduce them BITWISE,
since it restates the same sequential, unfused loop (kernel.py:48-78).
"""
import numpy as np
import pytest

from oracle import oracle
from tests.golden_util import load_configs, load_suite, load_validation, sliced_workload

SUITE = load_suite()


def test_suite_covers_every_category():
    cats = {c.category for c in SUITE}
    assert len(cats) == 23
    assert {c.dtype for c in SUITE} == {"d", "s", "c", "z"}


@pytest.mark.parametrize("case", SUITE, ids=lambda c: c.id)
def test_oracle_matches_reference_bitwise(case):
    a, b, c = case.buffers()
    before = c.copy()
    pos, kw = case.args(a, b, c)
    oracle.ORACLE[case.dtype](*pos, **kw)
    offs = case.c_offsets()
    assert c[offs].tobytes() == case.want.tobytes()
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == before[mask].tobytes()


@pytest.mark.parametrize("key", ["c1_0", "c2_0", "c2_1", "c3_0", "c4_0", "c5_0"])
def test_oracle_matches_reference_configs(key):
    meta, want = load_configs()[key]
    w = sliced_workload(meta)
    a, b, c = w.buffers()
    pos, kw = w.args(a, b, c)
    fn = oracle.oracle_dgett if w.dtype == "d" else oracle.oracle_sgett
    fn(*pos, **kw, threads=8)
    from tests.golden_util import view_offsets

    got = c[view_offsets(w.ext_c, w.inc_c, w.off_c)]
    assert got.tobytes() == want.tobytes()


def test_oracle_threads_bitwise_equal_serial():
    w = load_configs()["c1_0"][0]
    w = sliced_workload(w)
    a, b, c1 = w.buffers()
    c8 = c1.copy()
    pos, kw = w.args(a, b, c1)
    oracle.oracle_dgett(*pos, **kw, threads=1)
    pos, kw = w.args(a, b, c8)
    oracle.oracle_dgett(*pos, **kw, threads=7)
    assert c1.tobytes() == c8.tobytes()


@pytest.mark.parametrize("case", load_validation(), ids=lambda c: c["label"])
def test_validation_restatement_matches_reference(case):
    if "raises" in case:
        pytest.skip("structural (raised) case: checked against the product in test_abi.py")
    args, kw = case["args"], case["kw"]
    (ra, ea, ia, a, rb, eb, ib, b, conts, ca, cb, perm, inc_c, c) = args
    if len(ca) != conts or len(cb) != conts or len(ea) != ra or len(eb) != rb:
        pytest.skip("structural")
    got = oracle.validate_codes(ra, ea, ia, len(a), kw.get("offset_a", 0), rb, eb, ib, len(b),
                                kw.get("offset_b", 0), conts, ca, cb, perm, inc_c, len(c),
                                kw.get("offset_c", 0))
    assert got == [e[0] for e in case["errors"]]


def test_einsum_crosscheck_agrees_with_oracle():
    w = sliced_workload(load_configs()["c1_0"][0])
    a, b, c = w.buffers()
    c0 = c.copy()
    pos, kw = w.args(a, b, c)
    oracle.oracle_dgett(*pos, **kw)
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b, w.conts,
                              w.cont_a, w.cont_b, w.perm)
    got = oracle.strided(c, w.ext_c, w.inc_c, w.off_c) - oracle.strided(c0, w.ext_c, w.inc_c, w.off_c)
    assert np.max(np.abs(got - ref)) < 1e-12 * w.size_k
