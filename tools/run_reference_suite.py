"""Run the REFERENCE package's own pytest suite with our GPU backend installed
as gett.kernel.dgett / sgett / zero_view.

    python tools/run_reference_suite.py [REF_PKG_DIR] [pytest args...]

REF_PKG_DIR defaults to /root/reference/pkg, else baseline/_ref/pkg (a
git-ignored copy that travels to the GPU box with gpurun).  The reference's
tests are copied to a temp dir with a conftest.py that installs the backend
before any test module imports gett.kernel's names (all of s/d/c/z gett and
zero_view are the GPU backend's).  Verification tool only:
not part of the product, the GPU test suite or bench.py.
"""
import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFTEST = '''
import sys
sys.path.insert(0, {src!r})
sys.path.insert(0, {repo!r})
import gett.kernel as _k
import gett.plan as _p
import paper_2410_06770_b200 as _b

def _adapt(entry):
    def call(*args, **kw):
        errs = entry(*args, **kw)
        return [_p.ValidationError(_p.ErrorCode[e.code.name], e.message) for e in errs]
    call.__name__ = entry.__name__
    return call

_k.dgett = _adapt(_b.dgett)
_k.sgett = _adapt(_b.sgett)
_k.cgett = _adapt(_b.cgett)
_k.zgett = _adapt(_b.zgett)

def _zero_view(view, buf):
    _b.zero_view(_b.TensorView(view.rank, view.extents, view.increments, view.base_offset,
                               view.buffer_len), buf)
_k.zero_view = _zero_view
'''


def main():
    args = sys.argv[1:]
    ref = None
    if args and os.path.isdir(args[0]):
        ref = args.pop(0)
    for cand in (ref, "/root/reference/pkg", os.path.join(REPO, "baseline", "_ref", "pkg")):
        if cand and os.path.isdir(os.path.join(cand, "tests")):
            ref = cand
            break
    else:
        print("reference package not found", file=sys.stderr)
        return 2
    tmp = tempfile.mkdtemp(prefix="gett_refsuite_")
    shutil.copytree(os.path.join(ref, "tests"), os.path.join(tmp, "tests"))
    with open(os.path.join(tmp, "tests", "conftest.py"), "w") as f:
        f.write(CONFTEST.format(src=os.path.join(os.path.abspath(ref), "src"), repo=REPO))
    env = dict(os.environ, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/numba_cache"))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", os.path.join(tmp, "tests")] + args
    return subprocess.call(cmd, cwd=tmp, env=env)


if __name__ == "__main__":
    sys.exit(main())
