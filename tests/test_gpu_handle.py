"""Plan handles (handle.py; gett_plan_create / gett_execute[_device]): a
plan made from dgett's arguments executes bitwise like dgett on the golden
suite (host and device buffers), repeats on new contents, and rejects buffers
of another length or dtype."""
import numpy as np
import pytest

import paper_2410_06770_b200 as g
from tests.golden_util import load_suite

pytestmark = pytest.mark.gpu

SUITE = [c for c in load_suite() if c.dtype in "ds"]


@pytest.mark.parametrize("where", ["host", "device"])
def test_plan_equals_entry_on_golden_suite(where, kernel_mode):
    import torch

    kernel_mode("auto")
    fails = []
    for case in SUITE:
        a, b, c = case.buffers()
        want = c.copy()
        pos, kw = case.args(a, b, want)
        entry = g.dgett if case.dtype == "d" else g.sgett
        assert entry(*pos, **kw) == []
        got = c.copy()
        pos, kw = case.args(a, b, got)
        plan = (g.dgett_plan if case.dtype == "d" else g.sgett_plan)(*pos, **kw)
        assert plan.errors == []
        if where == "host":
            assert plan(a, b, got) == []
        else:
            ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, got))
            assert plan.device(ta, tb, tc) == []
            got = tc.cpu().numpy()
        plan.close()
        if got.tobytes() != want.tobytes():
            fails.append(case.id)
    assert not fails, fails[:5]


def test_plan_repeats_and_checks_buffers(kernel_mode):
    from paper_2410_06770_b200.workloads import C1

    kernel_mode("auto")
    a, b, c = C1.buffers()
    pos, kw = C1.args(a, b, c)
    plan = g.dgett_plan(*pos, **kw)
    ref = c.copy()
    rpos, rkw = C1.args(a, b, ref)
    for step in range(3):
        a[:] = np.random.default_rng(step).uniform(-1, 1, a.size)
        assert g.dgett(*rpos, **rkw) == []
        assert plan(a, b, c) == []
        assert c.tobytes() == ref.tobytes()
    with pytest.raises(TypeError):
        plan(a[:-1], b, c)
    with pytest.raises(TypeError):
        plan(a.astype(np.float32), b, c)
