"""Run the REFERENCE's own verification harness (gett.testkit.run_suite, the
`gett verify` command, cli.py:86-109) with this package's GPU backend
installed as gett.kernel.{s,d,c,z}gett / zero_view.

    python tools/run_reference_verify.py [REF_PKG_DIR] [--cases N] [--seed S] [--suite all|cat,...]

Every case is checked by the reference's check_case (testkit.py:543-605):
kernel vs the reference's wide oracle bitwise after the cast, bytes outside
C's view unchanged, commutativity bit-identical, etc.  SPEC.md:403's gate is
--cases 1000 --seed 1 over all 23 categories.  Verification tool only: not
part of the product, the GPU test suite or bench.py.
"""
import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ref", nargs="?", default=None)
    ap.add_argument("--cases", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--suite", default="all")
    ap.add_argument("--kernel", default="auto", help="auto|ref|tiled (GETT_KERNEL family)")
    args = ap.parse_args()
    for cand in (args.ref, "/root/reference/pkg", os.path.join(REPO, "baseline", "_ref", "pkg")):
        if cand and os.path.isdir(os.path.join(cand, "src", "gett")):
            ref = cand
            break
    else:
        print("reference package not found", file=sys.stderr)
        return 2
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, os.path.join(os.path.abspath(ref), "src"))
    sys.path.insert(0, REPO)
    import gett.kernel as rk
    import gett.plan as rp
    from gett import testkit

    import paper_2410_06770_b200 as b

    def adapt(entry):
        def call(*a, **kw):
            return [rp.ValidationError(rp.ErrorCode[e.code.name], e.message) for e in entry(*a, **kw)]
        call.__name__ = entry.__name__
        return call

    for name in ("sgett", "dgett", "cgett", "zgett"):
        setattr(rk, name, adapt(getattr(b, name)))

    def zero_view(view, buf):
        b.zero_view(b.TensorView(view.rank, view.extents, view.increments, view.base_offset,
                                 view.buffer_len), buf)

    rk.zero_view = zero_view
    b.set_kernel(args.kernel)
    cats = None if args.suite == "all" else args.suite.split(",")
    width = max(len(c) for c in testkit.CATEGORIES) + 2
    launches0 = b.launch_count()
    t0 = time.time()

    def progress(res):
        print(f"{res.category:<{width}}{res.passed}/{res.passed + res.failed}", flush=True)

    report = testkit.run_suite(categories=cats, cases=args.cases, seed=args.seed, progress=progress)
    total = sum(r.passed + r.failed for r in report.results)
    failed = sum(r.failed for r in report.results)
    print(f"{len(report.results)} categories, {total} cases, {failed} failures, "
          f"{time.time() - t0:.1f} s, backend kernel family {args.kernel}, "
          f"{b.launch_count() - launches0} GPU kernel launches")
    for res in report.results:
        for seed, msg in res.failures:
            print(f"FAIL {res.category} seed={seed}: {msg}")
    return 1 if failed else 0


if __name__ == "__main__":
    sys.exit(main())
