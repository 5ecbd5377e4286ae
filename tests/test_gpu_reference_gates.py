"""The reference's OWN gates, run against this backend on the GPU (SURVEY
§8f #3): with the reference installed under baseline/_ref (the
git-ignored install that travels to the GPU box), its 221-test pytest suite
passes with gett.kernel.{s,d,c,z}gett / zero_view replaced by this package,
and its verification harness testkit.run_suite over all 23 categories x 1000
cases (seed 1) reports no failure — each case checked by the reference's own
wide oracle and check_case (bitwise after the cast, bytes outside C's view
unchanged, commutativity).  Skipped when baseline/_ref is absent."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "pkg")
needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_PKG, "tests")),
                               reason="reference not installed under baseline/_ref/pkg")


def _run(args, timeout):
    env = dict(os.environ, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/gett_numba_cache"))
    return subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


@needs_ref
def test_reference_pytest_suite_on_gpu_backend():
    r = _run([os.path.join("tools", "run_reference_suite.py"), REF_PKG], 900)
    tail = (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail


@needs_ref
@pytest.mark.parametrize("kernel", ["auto", "tiled"])
def test_reference_run_suite_23x1000_seed1(kernel):
    r = _run([os.path.join("tools", "run_reference_verify.py"), REF_PKG, "--cases", "1000",
              "--seed", "1", "--kernel", kernel], 1200)
    tail = (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, tail
    assert "23 categories, 23000 cases, 0 failures" in r.stdout, tail
