"""CPU tests of the drop-in boundary: the C ABI library loads, exports every
symbol include/gett_b200.h declares, and reproduces the reference's
validation behaviour (codes, order, messages, raises) through the C ABI —
none of which needs a GPU, because validation and the empty-space early
return happen before any CUDA call (kernel.py:146-153, :93-94)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2410_06770_b200 as g
from paper_2410_06770_b200 import _native
from tests.golden_util import load_validation, load_zero_view

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "gett_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gett_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 17
    lib = ctypes.CDLL(_native.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)


def test_abi_version():
    assert _native.LIB.gett_abi_version() == 107


@pytest.mark.parametrize("case", load_validation(), ids=lambda c: c["label"])
def test_validation_through_abi_matches_reference(case):
    args, kw = case["args"], case["kw"]
    c = args[13]
    c[:] = 7.0
    if "raises" in case:
        with pytest.raises({"TypeError": TypeError, "ValueError": ValueError}[case["raises"]]):
            g.dgett(*args, **kw)
        return
    if not case["errors"]:
        pytest.skip("valid call: needs the GPU (tests/test_gpu_parity.py)")
    errs = g.dgett(*args, **kw)
    assert [(e.code.value, e.message) for e in errs] == [tuple(e) for e in case["errors"]]
    assert np.all(c == 7.0), "C must be untouched when validation fails"


def test_validate_with_explicit_c_view():
    a, b = g.TensorView.contiguous((2, 3)), g.TensorView.contiguous((3, 4))
    spec = g.ContractionSpec(1, (1,), (0,), (0, 1))
    assert g.validate(a, b, spec, (1, 2)) == []
    assert g.validate(a, b, spec, (1, 2), g.TensorView.contiguous((2, 4))) == []
    small = g.TensorView(2, (2, 4), (1, 2), 0, 7)
    errs = g.validate(a, b, spec, (1, 2), small)
    assert [e.code for e in errs] == [g.ErrorCode.FootprintOutOfBounds]
    assert "C addresses" in errs[0].message
    neg = g.TensorView(1, (-1,), (1,), 0, 4)
    errs = g.validate(a, b, spec, (1, 2), neg)
    assert errs[0].code == g.ErrorCode.NegativeExtent and errs[0].message.startswith("C ")


def test_messages_match_reference_text():
    a, b = g.TensorView.contiguous((2, 3)), g.TensorView.contiguous((4, 4))
    errs = g.validate(a, b, g.ContractionSpec(1, (1,), (0,), (0, 1)), (1, 2))
    assert "pair 0" in str(errs[0])
    fa = g.TensorView(1, (5,), (1,), 0, 4)
    errs = g.validate(fa, g.TensorView.contiguous((5,)), g.ContractionSpec(1, (0,), (0,), ()), ())
    assert "A" in str([e for e in errs if e.code == g.ErrorCode.FootprintOutOfBounds][0])


def test_type_and_structure_raises():
    a = np.zeros(1, dtype=np.float32)
    with pytest.raises(TypeError):
        g.dgett(0, (), (), a, 0, (), (), a, 0, (), (), (), (), a)
    a = np.zeros(2)
    with pytest.raises(ValueError):
        g.dgett(2, (2,), (1,), a, 1, (2,), (1,), a, 0, (), (), (0, 1), (1, 2), a)
    with pytest.raises(TypeError):
        g.dgett(1, (2,), (1,), a, 1, (2,), (1,), a, 1, (0,), (0,), (), (), [0.0])
    with pytest.raises(TypeError):
        g.dgett(1, (2,), (1,), np.zeros((2, 1)), 1, (2,), (1,), a, 1, (0,), (0,), (), (), np.zeros(1))
    with pytest.raises(ValueError):
        g.ContractionSpec(2, (0,), (0, 1), ())
    with pytest.raises(ValueError):
        g.ContractionSpec(-1, (), (), ())


def test_empty_iteration_writes_nothing_without_device():
    c = np.full(4, 3.0)
    errs = g.dgett(1, (0,), (1,), np.array([1.0]), 1, (1,), (1,), np.array([2.0]),
                   0, (), (), (0, 1), (1, 1), c)
    assert errs == [] and np.all(c == 3.0)


def test_multi_device_call_validates_without_device():
    """gett_dgett_multi validates (and returns the empty-space early exit)
    before touching any device, exactly like the one-device entry."""
    a, b, c = np.ones(6), np.ones(6), np.zeros(4)
    args = (2, (2, 3), (3, 1), a, 2, (2, 3), (3, 1), b, 1, (1,), (0,), (0, 1), (2, 1), c)
    want = g.dgett(*args)
    got = g.dgett(*args, devices=(0, 1, 0))
    assert want and [(e.code, e.message) for e in got] == [(e.code, e.message) for e in want]
    c = np.full(4, 3.0)
    assert g.dgett(1, (0,), (1,), np.array([1.0]), 1, (1,), (1,), np.array([2.0]),
                   0, (), (), (0, 1), (1, 1), c, devices=(0, 1)) == [] and np.all(c == 3.0)
    with pytest.raises(ValueError):
        g.dgett(*args, devices=())
    with pytest.raises(TypeError):
        g.zgett(1, (1,), (1,), np.ones(1, np.complex128), 1, (1,), (1,), np.ones(1, np.complex128),
                1, (0,), (0,), (), (), np.zeros(1, np.complex128), devices=(0,))


def test_multi_device_setters():
    from paper_2410_06770_b200 import _native

    assert _native.LIB.gett_set_multi(3) == _native.E_INVALID_ARG
    assert _native.LIB.gett_set_multi(-1) == _native.E_INVALID_ARG
    assert _native.LIB.gett_set_devices(1, _native.i32([-1])) == _native.E_INVALID_ARG
    for s in ("auto", "slabs", "splitk"):
        g.set_multi(s)
    g.set_multi("splitk", staged=True)
    g.set_multi("auto")
    g.set_devices((0, 0))
    g.set_devices(None)
    assert g.last_multi() == "none"


def test_kernel_switch_setters():
    """The tuning switches validate their argument and leave the defaults
    restorable (no CUDA call involved)."""
    from paper_2410_06770_b200 import _native

    L = _native.LIB
    for bad in (-1, 3, 7, 32):            # (mode & 3) == 3 or out of range
        assert L.gett_set_kr(bad) == _native.E_INVALID_ARG
    for bad in (-1, 3, 16):
        assert L.gett_set_wide(bad) == _native.E_INVALID_ARG
    for bad in (-1, 2):
        assert L.gett_set_pdl(bad) == _native.E_INVALID_ARG
        assert L.gett_set_bulk(bad) == _native.E_INVALID_ARG
    for mixed in (False, True):
        g.set_kr("force", fused=True, pair=False, mixed=mixed)
        g.set_wide("force", mixed=mixed, tail=not mixed)
    g.set_pdl(False)
    g.set_pdl(True)
    g.set_kr("auto")
    g.set_wide("auto")
    with pytest.raises(ValueError):
        g.set_wide("sometimes")


def test_derive_output_extents():
    a, b = g.TensorView.contiguous((2, 3)), g.TensorView.contiguous((3, 4))
    assert g.derive_output_extents(a, b, g.ContractionSpec(1, (1,), (0,), (1, 0))) == (4, 2)
    c5a = g.TensorView.contiguous((48, 24, 32, 16, 40))
    c5b = g.TensorView.contiguous((40, 32, 24, 96))
    assert g.derive_output_extents(c5a, c5b, g.ContractionSpec(3, (1, 2, 4), (2, 1, 0), (1, 2, 0))) == (96, 48, 16)


def test_fastdiv_formula():
    """The device FastDiv (csrc/device.cuh): q = umulhi(n, mul) >> shr with
    mul = ceil(2^(31+l) / d), l = ceil(log2 d), exact for n < 2^31."""
    rng = np.random.default_rng(0)
    ds = [1, 2, 3, 5, 7, 24, 40, 96, 127, 128, 129, 768, 4096, 5184, 65536, 1 << 20, (1 << 31) - 1]
    ds += [int(x) for x in rng.integers(1, 1 << 31, 200)]
    for d in ds:
        if d == 1:
            continue
        l = (d - 1).bit_length()
        p = 31 + l
        mul = ((1 << p) + d - 1) // d
        assert mul < (1 << 32)
        shr = p - 32
        ns = [0, 1, d - 1, d, d + 1, (1 << 31) - 1] + [int(x) for x in rng.integers(0, 1 << 31, 200)]
        for n in ns:
            assert ((n * mul) >> 32) >> shr == n // d, (n, d)


def test_zero_view_golden_cpu_checks():
    # structure of the fixture; device results are checked in test_gpu_parity.py
    cases = load_zero_view()
    assert len(cases) == 6
    empty = [c for c in cases if 0 in c["ext"] or any(e < 0 for e in c["ext"])]
    for c in empty:
        assert c["result"] == list(np.arange(1, c["n"] + 1, dtype=float))


# ---------------------------------------------------------------------------
# a plain C caller (tools/abi_c_example.c) links libgett_b200.so through
# include/gett_b200.h alone


def _build_c_example(tmp_path):
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2410_06770_b200")
    exe = str(tmp_path / "abi_c_example")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tools", "abi_c_example.c"), "-L", pkg, "-lgett_b200",
                    f"-Wl,-rpath,{pkg}", "-o", exe], check=True)
    return exe


def test_c_caller_gets_coded_validation_errors(tmp_path):
    """Validation needs no GPU: a C program gets the reference-ordered error
    codes back with C untouched."""
    import subprocess

    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe, "validate"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"c_untouched": 1' in r.stdout


@pytest.mark.gpu
def test_c_caller_contracts_on_the_gpu(tmp_path):
    import subprocess

    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe, "run"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"bitwise_equal": 1' in r.stdout


def test_readonly_c_returns_phase_two_errors():
    """A read-only C whose only problem is its footprint: the reference runs
    output_view_errors before its first store (kernel.py:149-153) and returns
    [FootprintOutOfBounds C]; a clean read-only call raises ValueError."""
    a = np.ones(6)
    b = np.ones(12)
    c = np.zeros(7)  # C [2,4] contiguous needs 8 elements
    c.flags.writeable = False
    errs = g.dgett(2, (2, 3), (3, 1), a, 2, (3, 4), (4, 1), b, 1, (1,), (0,), (0, 1), (4, 1), c)
    assert [e.code for e in errs] == [g.ErrorCode.FootprintOutOfBounds]
    assert "C" in errs[0].message
    c = np.zeros(8)
    c.flags.writeable = False
    with pytest.raises(ValueError):
        g.dgett(2, (2, 3), (3, 1), a, 2, (3, 4), (4, 1), b, 1, (1,), (0,), (0, 1), (4, 1), c)


def test_plan_handle_validates_like_the_entry_without_device():
    """dgett_plan reports exactly dgett's validation errors (no GPU needed),
    and an empty iteration space plans to a no-op."""
    n = 0
    for case in load_validation():
        if "raises" in case or not case["errors"]:
            continue
        args, kw = case["args"], case["kw"]
        want = g.dgett(*args, **kw)
        p = g.dgett_plan(*args, **kw)
        assert [(e.code, e.message) for e in p.errors] == [(e.code, e.message) for e in want]
        assert p(args[3] if isinstance(args[3], np.ndarray) else np.asarray(args[3]),
                 np.asarray(args[7]), args[13]) == p.errors
        p.close()
        n += 1
    assert n > 100
    c = np.full(4, 3.0)
    p = g.dgett_plan(1, (0,), (1,), np.array([1.0]), 1, (1,), (1,), np.array([2.0]), 0, (), (), (0, 1),
                     (1, 1), c)
    assert p.errors == [] and p(np.array([1.0]), np.array([2.0]), c) == [] and np.all(c == 3.0)
    with pytest.raises(TypeError):
        g.GettPlan("z", 0, (), (), 1, 0, (), (), 1, 0, (), (), (), (), 1)
