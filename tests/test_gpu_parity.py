"""GPU parity: the sm_100a kernels, called through the C ABI (dgett/sgett host
entry points and the zero-copy device entry points), against the reference's
golden outputs and the CPU oracle.

Bars (north_star / SURVEY §8d):
  * ref-order kernel: BITWISE equal to the reference on every golden case.
  * tiled kernels: BITWISE on integer data (exact sums); otherwise
    err_K = max|C - C_ref| / (|K|·max|A|·max|B|) <= 1e-12 (f64) / 1e-5 (f32),
    and for SGETT the error vs an fp64 oracle within 2x the reference's own.
  * nothing outside the C view changes (testkit.py:568-573).
"""
import numpy as np
import pytest

import paper_2410_06770_b200 as g
from oracle import oracle
from tests.golden_util import (load_configs, load_suite, load_zero_view, sliced_workload,
                               view_offsets)

pytestmark = pytest.mark.gpu

SUITE = load_suite()
TOL_K = {"d": 1e-12, "s": 1e-5, "z": 1e-12, "c": 1e-5}
ENTRY = {"d": g.dgett, "s": g.sgett, "z": g.zgett, "c": g.cgett}


def run(entry, pos, kw):
    errs = entry(*pos, **kw)
    assert errs == [], errs


def k_norm_err(got, want, w_or_k, amax=1.0, bmax=1.0):
    k = max(1, w_or_k)
    wide = np.complex128 if np.iscomplexobj(got) or np.iscomplexobj(want) else np.float64
    d = np.max(np.abs(got.astype(wide) - want.astype(wide))) if got.size else 0.0
    return d / (k * max(amax, 1e-300) * max(bmax, 1e-300))


# ---------------------------------------------------------------------------
# known answers (restating the reference's test_kernel.py cases)

MODES = ["auto", "ref", "tiled", "dot"]


@pytest.mark.parametrize("mode", MODES)
def test_known_answers(mode, kernel_mode):
    kernel_mode(mode)
    dg = g.dgett
    a, b, c = np.array([1.0, 2, 3]), np.array([4.0, 5, 6]), np.zeros(1)
    assert dg(1, (3,), (1,), a, 1, (3,), (1,), b, 1, (0,), (0,), (), (), c) == [] and c[0] == 32.0
    eye, m, c = np.eye(3).ravel(order="F"), np.arange(9, dtype=np.float64), np.zeros(9)
    assert dg(2, (3, 3), (1, 3), eye, 2, (3, 3), (1, 3), m, 1, (1,), (0,), (0, 1), (1, 3), c) == []
    assert np.array_equal(c, m)
    c = np.zeros(4)
    assert dg(1, (2,), (1,), np.array([1.0, 2]), 1, (2,), (1,), np.array([3.0, 4]), 0, (), (), (0, 1), (1, 2), c) == []
    assert c.tolist() == [3.0, 6.0, 4.0, 8.0]
    b6, c = np.arange(6, dtype=np.float64), np.zeros(6)
    assert dg(0, (), (), np.array([2.5]), 2, (2, 3), (1, 2), b6, 0, (), (), (0, 1), (1, 2), c) == []
    assert np.array_equal(c, 2.5 * b6)
    a, b, c = np.array([1.0, 2, 3]), np.array([1.0, 2, 3]), np.zeros(1)
    assert dg(1, (3,), (-1,), a, 1, (3,), (1,), b, 1, (0,), (0,), (), (), c, offset_a=2) == [] and c[0] == 10
    c = np.full(16, 9.0)
    assert dg(1, (2,), (1,), np.array([1.0, 2]), 1, (2,), (1,), np.array([3.0, 4]), 0, (), (), (0, 1), (1, 4), c, offset_c=5) == []
    assert [c[5], c[6], c[9], c[10]] == [12, 15, 13, 17]
    assert all(c[i] == 9.0 for i in set(range(16)) - {5, 6, 9, 10})
    c = np.zeros(4)
    assert dg(2, (2, 2), (0, 1), np.array([5.0, 7]), 1, (2,), (1,), np.array([1.0, 1]), 1, (1,), (0,), (0,), (1,), c[:2]) == []
    assert c[:2].tolist() == [12.0, 12.0]
    cs = np.zeros(1, np.float32)
    assert g.sgett(1, (3,), (1,), np.array([1, 2, 3], np.float32), 1, (3,), (1,), np.array([4, 5, 6], np.float32),
                   1, (0,), (0,), (), (), cs) == [] and cs[0] == np.float32(32)
    # complex known answers (test_kernel.py:184-198)
    cz = np.zeros(1, np.complex128)
    assert g.zgett(1, (1,), (1,), np.array([1 + 2j]), 1, (1,), (1,), np.array([3 + 4j]),
                   1, (0,), (0,), (), (), cz) == [] and cz[0] == (-5 + 10j)
    cc = np.zeros(1, np.complex64)
    assert g.cgett(1, (2,), (1,), np.array([2 - 1j, 1 + 1j], np.complex64), 1, (2,), (1,),
                   np.array([1 + 1j, 3 + 0j], np.complex64), 1, (0,), (0,), (), (), cc) == []
    assert cc[0] == np.complex64(6 + 4j)
    # zero_view on complex buffers zeroes both parts of the addressed elements only
    zb = np.arange(1, 9, dtype=np.complex128) * (1 + 1j)
    g.zero_view(g.TensorView(2, (2, 2), (1, 4), 1, 8), zb)
    assert [zb[i] == 0 for i in range(8)] == [False, True, True, False, False, True, True, False]


@pytest.mark.parametrize("mode", ["ref", "tiled"])
def test_complex_gemm_against_numpy(mode, kernel_mode):
    """zgett/cgett at tiled sizes: integer data exact, uniform within tolerance."""
    kernel_mode(mode)
    rng = np.random.default_rng(9)
    for dt, tol in ((np.complex128, 1e-12), (np.complex64, 1e-5)):
        for m, k, n in [(3, 5, 2), (130, 70, 129), (256, 600, 64)]:
            for data in ("int", "uniform"):
                draw = (lambda s: rng.integers(-4, 5, s) + 1j * rng.integers(-4, 5, s)) if data == "int" \
                    else (lambda s: rng.uniform(-1, 1, s) + 1j * rng.uniform(-1, 1, s))
                A, B, C = draw((m, k)).astype(dt), draw((k, n)).astype(dt), draw((m, n)).astype(dt)
                c = C.ravel(order="F").copy()
                entry = g.zgett if dt == np.complex128 else g.cgett
                assert entry(2, (m, k), (1, m), A.ravel(order="F"), 2, (k, n), (1, k), B.ravel(order="F"),
                             1, (1,), (0,), (0, 1), (1, m), c) == []
                want = C.astype(np.complex128) + A.astype(np.complex128) @ B.astype(np.complex128)
                got = c.reshape((m, n), order="F")
                if data == "int":
                    assert np.array_equal(got, want.astype(dt)), (dt, m, k, n, mode)
                else:
                    assert np.max(np.abs(got - want)) <= tol * k * 2, (dt, m, k, n, mode)


@pytest.mark.parametrize("mode", MODES)
def test_accumulation_and_gemm(mode, kernel_mode):
    kernel_mode(mode)
    rng = np.random.default_rng(5)
    for m, k, n in [(1, 1, 1), (5, 3, 2), (33, 65, 17), (129, 40, 131), (256, 300, 64)]:
        A = rng.integers(-4, 5, (m, k)).astype(np.float64)
        B = rng.integers(-4, 5, (k, n)).astype(np.float64)
        c = np.zeros(m * n)
        args = (2, (m, k), (1, m), A.ravel(order="F"), 2, (k, n), (1, k), B.ravel(order="F"),
                1, (1,), (0,), (0, 1), (1, m), c)
        assert g.dgett(*args) == []
        assert np.array_equal(c.reshape((m, n), order="F"), A @ B)
        assert g.dgett(*args) == []
        assert np.array_equal(c.reshape((m, n), order="F"), 2 * (A @ B))


def test_kernel_selection_evidence(kernel_mode):
    c = np.zeros(128 * 128)
    A = np.ones(128 * 512)
    kernel_mode("tiled")
    g.dgett(2, (128, 512), (512, 1), A, 2, (512, 128), (128, 1), A, 1, (1,), (0,), (0, 1), (128, 1), c)
    assert g.last_kernel().startswith("dgett_dmma")
    kernel_mode("ref")
    g.dgett(2, (128, 512), (512, 1), A, 2, (512, 128), (128, 1), A, 1, (1,), (0,), (0, 1), (128, 1), c)
    assert g.last_kernel() == "dgett_ref_order"
    n0 = g.launch_count()
    g.dgett(2, (128, 512), (512, 1), A, 2, (512, 128), (128, 1), A, 1, (1,), (0,), (0, 1), (128, 1), c)
    assert g.launch_count() == n0 + 1


# ---------------------------------------------------------------------------
# golden suite (reference-generated descriptors, reference outputs)


def _check_suite_case(case, mode, kernel_mode):
    kernel_mode(mode)
    a, b, c = case.buffers()
    before = c.copy()
    pos, kw = case.args(a, b, c)
    run(ENTRY[case.dtype], pos, kw)
    offs = case.c_offsets()
    got = c[offs]
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == before[mask].tobytes(), "bytes outside the C view changed"
    if mode == "ref" or case.data == "int":
        # integer data: every partial sum is exact, so any order/precision split agrees
        assert got.tobytes() == case.want.tobytes(), "not bitwise equal to the reference"
    else:
        k = int(np.prod([case.a["ext"][d] for d in case.cont_a])) if case.conts else 1
        assert k_norm_err(got, case.want, k) <= TOL_K[case.dtype]


@pytest.mark.parametrize("mode", ["ref", "tiled", "auto", "ffma", "dot"])
def test_golden_suite(mode, kernel_mode):
    failures = []
    for case in SUITE:
        try:
            _check_suite_case(case, mode, kernel_mode)
        except AssertionError as e:
            failures.append(f"{case.id}: {e}")
    assert not failures, f"{len(failures)} failures, first: {failures[:5]}"


@pytest.mark.parametrize("split", [2, 3, 7])
def test_golden_suite_forced_split_k(split, kernel_mode):
    failures = []
    for case in SUITE[::5]:
        try:
            kernel_mode("tiled", split)
            _check_suite_case(case, "tiled", lambda m, s=split: kernel_mode(m, s))
        except AssertionError as e:
            failures.append(f"{case.id}: {e}")
    assert not failures, failures[:5]


@pytest.mark.parametrize("slabs", [2, 3])
def test_golden_suite_pipelined_host_path(slabs, kernel_mode):
    """Host path with H2D/compute/D2H overlapped over C-disjoint slabs."""
    failures = []
    for case in SUITE:
        try:
            _check_suite_case(case, "tiled", lambda m: kernel_mode(m, 0, slabs))
        except AssertionError as e:
            failures.append(f"{case.id}: {e}")
    assert not failures, f"{len(failures)} failures, first: {failures[:5]}"


def test_commutativity_bit_identical(kernel_mode):
    """Swapping A and B with a rotated perm writes a bit-identical buffer
    (testkit.py:476-495, :575-581) on the integer-data cases."""
    kernel_mode("tiled")
    for case in SUITE:
        if case.data != "int":
            continue
        a, b, c = case.buffers()
        pos, kw = case.args(a, b, c.copy())
        c1 = pos[13]
        run(ENTRY[case.dtype], pos, kw)
        fa = case.a["rank"] - case.conts
        perm = tuple(case.perm[fa:]) + tuple(case.perm[:fa])
        c2 = c.copy()
        pos2 = (case.b["rank"], tuple(case.b["ext"]), tuple(case.b["inc"]), b,
                case.a["rank"], tuple(case.a["ext"]), tuple(case.a["inc"]), a,
                case.conts, tuple(case.cont_b), tuple(case.cont_a), perm, tuple(case.c["inc"]), c2)
        kw2 = dict(offset_a=case.b["off"], offset_b=case.a["off"], offset_c=case.c["off"])
        run(ENTRY[case.dtype], pos2, kw2)
        assert c1.tobytes() == c2.tobytes(), case.id


# ---------------------------------------------------------------------------
# BASELINE configs


CONFIGS = load_configs()


@pytest.mark.parametrize("key", sorted(CONFIGS))
def test_config_slices_ref_bitwise(key, kernel_mode):
    kernel_mode("ref")
    meta, want = CONFIGS[key]
    w = sliced_workload(meta)
    a, b, c = w.buffers()
    pos, kw = w.args(a, b, c)
    run(ENTRY[w.dtype], pos, kw)
    assert c[view_offsets(w.ext_c, w.inc_c, w.off_c)].tobytes() == want.tobytes()


@pytest.mark.parametrize("key", sorted(CONFIGS))
def test_config_slices_tiled(key, kernel_mode):
    kernel_mode("auto")
    meta, want = CONFIGS[key]
    w = sliced_workload(meta)
    a, b, c = w.buffers()
    pos, kw = w.args(a, b, c)
    run(ENTRY[w.dtype], pos, kw)
    got = c[view_offsets(w.ext_c, w.inc_c, w.off_c)]
    assert k_norm_err(got, want, w.size_k, np.abs(a).max(), np.abs(b).max()) <= TOL_K[w.dtype]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_full_config(name, kernel_mode):
    """Full-size run: golden slices (reference) + fp64 einsum over the whole
    output + padding untouched."""
    from paper_2410_06770_b200.workloads import CONFIGS as W

    kernel_mode("auto")
    w = W[name]
    a, b, c = w.buffers()
    c0 = c.copy()
    pos, kw = w.args(a, b, c)
    run(ENTRY[w.dtype], pos, kw)
    offs = view_offsets(w.ext_c, w.inc_c, w.off_c)
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == c0[mask].tobytes()
    amax, bmax = float(np.abs(a).max()), float(np.abs(b).max())
    # reference golden slices
    for key, (meta, want) in CONFIGS.items():
        if meta["workload"] != name:
            continue
        ws = sliced_workload(meta)
        got = c[view_offsets(ws.ext_c, ws.inc_c, ws.off_c)]
        assert k_norm_err(got, want, w.size_k, amax, bmax) <= TOL_K[w.dtype], key
    # whole output vs fp64
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    ref = ref + oracle.strided(c0, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
    got = oracle.strided(c, w.ext_c, w.inc_c, w.off_c)
    assert k_norm_err(got, ref, w.size_k, amax, bmax) <= TOL_K[w.dtype]
    if name == "c5":
        # secondary gate: error vs fp64 no worse than 2x the reference's own
        _, want = CONFIGS["c5_0"]
        ref_flat = ref.ravel(order="F")  # view order: dimension 0 fastest
        e_ref = np.max(np.abs(want.astype(np.float64) - ref_flat))
        e_new = np.max(np.abs(c[offs].astype(np.float64) - ref_flat))
        assert e_new <= 2 * e_ref, (e_new, e_ref)


# ---------------------------------------------------------------------------
# other entry points


def test_device_entry_matches_host_bitwise():
    import torch

    from paper_2410_06770_b200.device import dgett_device
    from paper_2410_06770_b200.workloads import C3

    w = C3.slice_free("A", 0, 0, 8)
    a, b, c = w.buffers()
    ch = c.copy()
    pos, kw = w.args(a, b, ch)
    run(g.dgett, pos, kw)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    pos, kw = w.args(ta, tb, tc)
    assert dgett_device(*pos, **kw) == []
    torch.cuda.synchronize()
    assert tc.cpu().numpy().tobytes() == ch.tobytes()


def test_zero_view_golden():
    for z in load_zero_view():
        buf = np.arange(1, z["n"] + 1, dtype=np.float64)
        g.zero_view(g.TensorView(z["rank"], z["ext"], z["inc"], z["off"], z["n"]), buf)
        assert buf.tolist() == z["result"]
        bs = np.arange(1, z["n"] + 1, dtype=np.float32)
        g.zero_view(g.TensorView(z["rank"], z["ext"], z["inc"], z["off"], z["n"]), bs)
        assert bs.tolist() == z["result"]


def test_aliasing_output_uses_serial_kernel_and_matches_oracle():
    """Distinct output coordinates sharing a C element (legal: only inc 0 is
    rejected, plan.py:220-227) — the serial kernel reproduces the sequential
    reference order bitwise."""
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, 12)
    b = rng.uniform(-1, 1, 20)
    args = (2, (3, 4), (1, 3), a, 2, (4, 5), (1, 4), b, 1, (1,), (0,), (0, 1), (1, 1))
    c = rng.uniform(-1, 1, 10)
    want = c.copy()
    oracle.oracle_dgett(*args, want)
    assert g.dgett(*args, c) == []
    assert g.last_kernel() == "dgett_serial"
    assert c.tobytes() == want.tobytes()


@pytest.mark.parametrize("mode", ["tiled", "ref"])
def test_plan_cache_is_offset_independent(mode, kernel_mode):
    """Plans are cached by descriptor; offsets (and so copied spans) are per
    call.  Same descriptor, different offsets, back to back."""
    kernel_mode(mode)
    rng = np.random.default_rng(11)
    a = rng.integers(-4, 5, 40).astype(np.float64)
    b = rng.integers(-4, 5, 40).astype(np.float64)
    for off_a, off_b, off_c in [(0, 0, 0), (7, 3, 2), (30, 0, 5), (1, 31, 0)]:
        c = rng.integers(-4, 5, 12).astype(np.float64)
        want = c.copy()
        args = (1, (5,), (1,), a, 1, (5,), (-1,), b, 1, (0,), (0,), (), ())
        kw = dict(offset_a=off_a, offset_b=off_b + 4, offset_c=off_c)
        oracle.oracle_dgett(*args, want, **kw)
        assert g.dgett(*args, c, **kw) == []
        assert c.tobytes() == want.tobytes(), (off_a, off_b, off_c)


def test_signed_zero_semantics(kernel_mode):
    for mode in ("ref", "tiled"):
        kernel_mode(mode)
        a = np.array([-0.0, 0.0, -4.0])
        b = np.array([1.0, -0.0, 0.0])
        for c0 in (0.0, -0.0):
            c = np.array([c0])
            want = np.array([c0])
            oracle.oracle_dgett(1, (3,), (1,), a, 1, (3,), (1,), b, 1, (0,), (0,), (), (), want)
            assert g.dgett(1, (3,), (1,), a, 1, (3,), (1,), b, 1, (0,), (0,), (), (), c) == []
            assert c.tobytes() == want.tobytes(), (mode, c0)
        # all products -0 with C = -0 stays -0
        c = np.array([-0.0])
        assert g.dgett(1, (3,), (1,), np.array([-0.0, -0.0, -0.0]),
                       1, (3,), (1,), np.ones(3), 1, (0,), (0,), (), (), c) == []
        assert np.signbit(c[0])


# ---------------------------------------------------------------------------
# split-K across ranks (shard.splitk_contract): the device sub-calls


def _emulated_splitk(w, world, ta, tb, tc):
    """`world` ranks run one after another on this GPU; reduce() emulates
    ncclReduce(sum) onto rank 0 (non-roots deposit, the root sums last)."""
    import torch

    from paper_2410_06770_b200.device import dgett_device, sgett_device
    from paper_2410_06770_b200.shard import splitk_contract

    entry = sgett_device if w.dtype == "s" else dgett_device
    acc = []

    def reduce_for(rank):
        def red(p):
            if rank != 0:
                acc.append(p.clone())
            else:
                for q in acc:
                    p.add_(q)
        return red

    for rank in reversed(range(world)):
        ci = tc if rank == 0 else tc.clone()
        pos, kw = w.args(ta, tb, ci)
        errs = splitk_contract(entry, pos, kw, rank, world,
                               zeros=lambda n: torch.zeros(n, dtype=tc.dtype, device=tc.device),
                               ones=lambda: torch.ones(1, dtype=tc.dtype, device=tc.device),
                               reduce=reduce_for(rank))
        assert errs == []
        if rank != 0:
            torch.cuda.synchronize()
            assert torch.equal(ci, tc)  # only the owner writes C


@pytest.mark.parametrize("name,world", [("c1", 3), ("c5", 4), ("c5", 8)])
def test_splitk_ranks_on_device(name, world):
    import torch

    from paper_2410_06770_b200.workloads import CONFIGS as W

    w = W[name]
    a, b, c = w.buffers()
    c0 = c.copy()
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    _emulated_splitk(w, world, ta, tb, tc)
    got_flat = tc.cpu().numpy()
    offs = view_offsets(w.ext_c, w.inc_c, w.off_c)
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert got_flat[mask].tobytes() == c0[mask].tobytes()
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    ref = ref + oracle.strided(c0, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
    got = oracle.strided(got_flat, w.ext_c, w.inc_c, w.off_c)
    assert k_norm_err(got, ref, w.size_k, np.abs(a).max(), np.abs(b).max()) <= TOL_K[w.dtype]


def test_splitk_device_nccl_group():
    """splitk_device through a real NCCL process group (world size 1 here:
    one GPU per gpurun box) — wiring, validation and the owner write."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2410_06770_b200.shard import splitk_device
    from paper_2410_06770_b200.workloads import C5

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        w = C5.slice_free("A", 0, 0, 8)
        a, b, c = w.buffers()
        want = c.copy()
        pos, kw = w.args(a, b, want)
        run(g.sgett, pos, kw)
        ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
        pos, kw = w.args(ta, tb, tc)
        assert splitk_device("s", pos, kw) == []
        assert tc.cpu().numpy().tobytes() == want.tobytes()
        bad = list(pos)
        bad[12] = (0,) + tuple(bad[12][1:])  # zero output increment
        errs = splitk_device("s", tuple(bad), kw)
        assert errs and errs[0].code == g.ErrorCode.OutputWriteAliasing
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# SURVEY §8d variants: column-major (the reference's canonical layout) and the
# zeroed-C reading "C = contract(A, B)"


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_config_column_major(name, kernel_mode):
    from paper_2410_06770_b200.workloads import CONFIGS as W
    from paper_2410_06770_b200.workloads import colmajor

    kernel_mode("auto")
    w = colmajor(W[name])
    a, b, c = w.buffers()
    c0 = c.copy()
    pos, kw = w.args(a, b, c)
    run(ENTRY[w.dtype], pos, kw)
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    ref = ref + oracle.strided(c0, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
    got = oracle.strided(c, w.ext_c, w.inc_c, w.off_c)
    assert k_norm_err(got, ref, w.size_k, np.abs(a).max(), np.abs(b).max()) <= TOL_K[w.dtype]
    assert g.last_kernel().split("_")[0] in ("dgett", "sgett")


@pytest.mark.parametrize("name", ["c1", "c4", "c5"])
def test_zeroed_c_then_contract(name, kernel_mode):
    """zero_view on C's view, then xGETT: C = contract(A, B); padding keeps its
    bytes through both steps."""
    from paper_2410_06770_b200.workloads import CONFIGS as W

    kernel_mode("auto")
    w = W[name]
    a, b, c = w.buffers()
    c0 = c.copy()
    g.zero_view(g.TensorView(len(w.ext_c), w.ext_c, w.inc_c, w.off_c, len(c)), c)
    offs = view_offsets(w.ext_c, w.inc_c, w.off_c)
    assert not np.any(c[offs])
    pos, kw = w.args(a, b, c)
    run(ENTRY[w.dtype], pos, kw)
    mask = np.ones(len(c), bool)
    mask[offs] = False
    assert c[mask].tobytes() == c0[mask].tobytes()
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    got = oracle.strided(c, w.ext_c, w.inc_c, w.off_c)
    assert k_norm_err(got, ref, w.size_k, np.abs(a).max(), np.abs(b).max()) <= TOL_K[w.dtype]


# ---------------------------------------------------------------------------
# DGETT persistent stream-K schedule (tiles split between two CTAs: the head
# adds the tail's published partial) — deterministic, and equal in accuracy
# to the one-CTA-per-tile launch


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_stream_k_deterministic_and_accurate(name, kernel_mode):
    from paper_2410_06770_b200.workloads import CONFIGS as W

    w = W[name]
    a, b, c = w.buffers()
    outs = {}
    for sk in (True, False):
        kernel_mode("auto", pipeline=0, stream_k=sk)
        for rep in range(2):
            cc = c.copy()
            pos, kw = w.args(a, b, cc)
            run(ENTRY[w.dtype], pos, kw)
            kname = g.last_kernel()
            if rep:
                assert cc.tobytes() == outs[sk].tobytes(), "run-to-run difference"
            outs[sk] = cc
        assert kname.replace("_tma", "").replace("_bulk", "") == ("dgett_dmma_ws_sk" if sk else "dgett_dmma_ws")
    ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                              w.conts, w.cont_a, w.cont_b, w.perm)
    ref = ref + oracle.strided(c, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
    for sk, cc in outs.items():
        got = oracle.strided(cc, w.ext_c, w.inc_c, w.off_c)
        assert k_norm_err(got, ref, w.size_k, np.abs(a).max(), np.abs(b).max()) <= TOL_K["d"], sk


@pytest.mark.parametrize("rows", [256, 384, 512, 640, 1152])
def test_stream_k_below_two_waves(rows, kernel_mode):
    """Tiles below two waves run stream-K over all tiles — between one and two
    waves (640 x 4096 -> 160 tiles, 1152 x 4096 -> 288 tiles on 148 SMs) and
    below one wave (384 -> 96, 512 -> 128 tiles: shares shorter than a tile,
    heads adding several parts; 256 -> 64 tiles with K 512, where stream-K
    replaces split-K): deterministic, within the fp64 K-normalised bar of an
    fp64 contraction, and C's padding intact."""
    rng = np.random.default_rng(rows)
    M, N, K = rows, 4096, (512 if rows == 256 else 256)
    a = rng.uniform(-1, 1, M * (K + 8)).astype(np.float64)
    b = rng.uniform(-1, 1, K * (N + 4)).astype(np.float64)
    c0 = rng.uniform(-1, 1, M * (N + 2)).astype(np.float64)
    args = lambda cc: (2, (M, K), (K + 8, 1), a, 2, (K, N), (N + 4, 1), b, 1, (1,), (0,),  # noqa: E731
                       (0, 1), (N + 2, 1), cc)
    outs = []
    for sk in (True, True, False):
        kernel_mode("tiled", pipeline=0, stream_k=sk)
        cc = c0.copy()
        assert g.dgett(*args(cc)) == []
        assert g.last_kernel().replace("_tma", "").replace("_bulk", "") == ("dgett_dmma_ws_sk" if sk else
                                                       "dgett_dmma_ws_splitk" if rows == 256 else "dgett_dmma_ws")
        outs.append(cc)
    assert outs[0].tobytes() == outs[1].tobytes(), "run-to-run difference"
    A = oracle.strided(a, (M, K), (K + 8, 1), 0).astype(np.float64)
    B = oracle.strided(b, (K, N), (N + 4, 1), 0).astype(np.float64)
    ref = oracle.strided(c0, (M, N), (N + 2, 1), 0) + A @ B
    mask = np.ones(len(c0), bool)
    mask[np.add.outer(np.arange(M) * (N + 2), np.arange(N)).ravel()] = False
    for cc in (outs[0], outs[2]):
        got = oracle.strided(cc, (M, N), (N + 2, 1), 0)
        assert k_norm_err(got, ref, K, np.abs(a).max(), np.abs(b).max()) <= TOL_K["d"]
        assert cc[mask].tobytes() == c0[mask].tobytes()


def test_concurrent_streams_keep_separate_workspaces(kernel_mode):
    """Two device calls in flight on two streams at once — a split-K SGETT (c5)
    and a stream-K DGETT (c3), twice each — must not share partial-sum
    workspaces: results equal the same calls run alone."""
    import torch

    from paper_2410_06770_b200.device import dgett_device, sgett_device
    from paper_2410_06770_b200.workloads import CONFIGS as W

    kernel_mode("auto")
    jobs = []
    for name, fn in (("c5", sgett_device), ("c3", dgett_device)):
        w = W[name]
        a, b, c = w.buffers()
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        alone = torch.from_numpy(c).cuda()
        pos, kw = w.args(ta, tb, alone)
        assert fn(*pos, **kw) == []
        torch.cuda.synchronize()
        jobs.append((w, fn, ta, tb, c, alone))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    work = [(job, st, torch.from_numpy(job[4]).cuda()) for _ in range(2)
            for job, st in zip(jobs, streams)]
    torch.cuda.synchronize()  # inputs in place; the launches below overlap
    outs = []
    for (w, fn, ta, tb, c, alone), st, tc in work:
        with torch.cuda.stream(st):
            pos, kw = w.args(ta, tb, tc)
            assert fn(*pos, **kw) == []
        outs.append((tc, alone))
    torch.cuda.synchronize()
    for tc, alone in outs:
        assert torch.equal(tc, alone)


@pytest.mark.parametrize("mode", ["auto", "tiled", "ref"])
def test_offsets_beyond_32_bits(mode, kernel_mode):
    """Views whose offsets pass 2**31 elements (int64
    offsets): A lives at element 2**31 + 17 of a 8.6 GB fp32 buffer, C near
    2**31 of another; checked against the same contraction at offset 0."""
    import torch

    from paper_2410_06770_b200.device import sgett_device

    kernel_mode(mode)
    big = (1 << 31) + 70000
    rng = np.random.default_rng(7)
    M, K, N = 200, 300, 136
    a_small = rng.uniform(-1, 1, M * K).astype(np.float32)
    b = torch.from_numpy(rng.uniform(-1, 1, K * N).astype(np.float32)).cuda()
    ta = torch.zeros(big, dtype=torch.float32, device="cuda")
    tc = torch.zeros(big, dtype=torch.float32, device="cuda")
    off_a, off_c = (1 << 31) + 17, (1 << 31) - 5
    ta[off_a:off_a + M * K] = torch.from_numpy(a_small).cuda()
    args = lambda A, C, oa, oc: ((2, (M, K), (K, 1), A, 2, (K, N), (N, 1), b, 1, (1,), (0,),  # noqa: E731
                                  (0, 1), (N, 1), C), dict(offset_a=oa, offset_c=oc))
    pos, kw = args(ta, tc, off_a, off_c)
    assert sgett_device(*pos, **kw) == []
    ref_c = torch.zeros(M * N, dtype=torch.float32, device="cuda")
    pos, kw = args(torch.from_numpy(a_small).cuda(), ref_c, 0, 0)
    assert sgett_device(*pos, **kw) == []
    torch.cuda.synchronize()
    assert torch.equal(tc[off_c:off_c + M * N], ref_c)
    assert int(torch.count_nonzero(tc[:off_c])) == 0 and int(torch.count_nonzero(tc[off_c + M * N:])) == 0
    del ta, tc
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# dot mode (few outputs, long K): the staged-row kernel up to K = 4096, the
# warp-per-output kernel above; both operand orders of the streamed / staged
# roles, negative increments and non-affine K tables


@pytest.mark.parametrize("K1,K2", [(32, 40), (64, 64), (17, 241)])
@pytest.mark.parametrize("neg", [False, True])
@pytest.mark.parametrize("a_kfast", [True, False])
def test_dot_kernels_match_fp64(K1, K2, neg, a_kfast, kernel_mode):
    kernel_mode("dot")
    rng = np.random.default_rng(K1 * 1000 + K2 + 7 * neg + a_kfast)
    M, N = 24, 20
    # A (m, k1, k2), B (k1, k2, n): the K-fast operand streams, the other is staged
    a_dims, b_dims = (M, K1, K2), (K1, K2, N)
    if a_kfast:
        a_inc = (K1 * K2 + 3, K2, 1)
        b_inc = (1, K1 + 2, (K1 + 2) * K2)
    else:
        a_inc = (1, M + 1, (M + 1) * K1)
        b_inc = (K2 * N + 5, N, 1)
    sign = -1 if neg else 1
    a_inc = tuple(sign * i for i in a_inc)
    span = lambda ext, inc: sum((e - 1) * abs(i) for e, i in zip(ext, inc)) + 1  # noqa: E731
    a = rng.uniform(-1, 1, span(a_dims, a_inc) + 4)
    b = rng.uniform(-1, 1, span(b_dims, b_inc) + 4)
    off_a = span(a_dims, a_inc) - 1 if neg else 0
    c0 = rng.uniform(-1, 1, M * N + 8)
    c = c0.copy()
    assert g.dgett(3, a_dims, a_inc, a, 3, b_dims, b_inc, b, 2, (1, 2), (0, 1), (0, 1), (N, 1), c,
                   offset_a=off_a, offset_c=3) == []
    assert g.last_kernel() == "dgett_dot"
    A = oracle.strided(a, a_dims, a_inc, off_a).astype(np.float64)
    B = oracle.strided(b, b_dims, b_inc, 0).astype(np.float64)
    want = oracle.strided(c0, (M, N), (N, 1), 3) + np.einsum("mij,ijn->mn", A, B)
    got = oracle.strided(c, (M, N), (N, 1), 3)
    assert k_norm_err(got, want, K1 * K2, np.abs(a).max(), np.abs(b).max()) <= TOL_K["d"]
    mask = np.ones(len(c0), bool)
    mask[3:3 + M * N] = False
    assert c[mask].tobytes() == c0[mask].tobytes()


# ---------------------------------------------------------------------------
# CUDA-graph replay of a device call (graph.py)


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_graph_replay_equals_direct_calls(name, kernel_mode):
    """Replaying a captured call twice gives C bitwise equal to three direct
    calls (the construction runs the call once), for the dot, DGETT and
    split-K SGETT paths (DGETT direct calls with stream-K off: a captured DGETT
    runs one CTA per tile)."""
    import torch

    from paper_2410_06770_b200.device import dgett_device, sgett_device
    from paper_2410_06770_b200.graph import GettGraph
    from paper_2410_06770_b200.workloads import CONFIGS as W

    kernel_mode("auto", stream_k=False)
    w = W[name]
    a, b, c = w.buffers()
    fn = dgett_device if w.dtype == "d" else sgett_device
    outs = []
    for use_graph in (True, False):
        ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
        pos, kw = w.args(ta, tb, tc)
        if use_graph:
            gg = GettGraph(fn, *pos, **kw)
            gg.replay()
            gg.replay()
        else:
            for _ in range(3):
                assert fn(*pos, **kw) == []
        torch.cuda.synchronize()
        outs.append(tc.cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes()


@pytest.mark.gpu
def test_graph_capture_sub_wave_stream_k_shape(kernel_mode):
    """A DGETT of 64 output tiles (1024 x 1024, K 4096): the eager call runs the
    sub-wave stream-K schedule; the captured one must still need no new
    workspace and give exactly the direct calls' result on integer
    data.  Then >512 other descriptors churn the plan LRU: the captured plan is
    pinned, so the replay still reads valid offset tables."""
    import torch

    from paper_2410_06770_b200.device import dgett_device
    from paper_2410_06770_b200.graph import GettGraph

    kernel_mode("auto", stream_k=True)
    rng = np.random.default_rng(5)
    M = N = 1024
    K = 4096
    a = rng.integers(-3, 4, M * K).astype(np.float64)
    b = rng.integers(-3, 4, K * N).astype(np.float64)
    c = rng.integers(-3, 4, M * N).astype(np.float64)
    args = (2, (M, K), (K, 1), None, 2, (K, N), (N, 1), None, 1, (1,), (0,), (0, 1), (N, 1), None)

    def call_args(ta, tb, tc):
        x = list(args)
        x[3], x[7], x[13] = ta, tb, tc
        return x

    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    gg = GettGraph(dgett_device, *call_args(ta, tb, tc))
    # churn: 600 distinct small descriptors
    sa = torch.ones(600, dtype=torch.float64, device="cuda")
    sc = torch.zeros(1, dtype=torch.float64, device="cuda")
    for e in range(1, 601):
        assert dgett_device(1, (e,), (1,), sa, 1, (e,), (1,), sa, 1, (0,), (0,), (), (), sc) == []
    gg.replay()
    gg.replay()
    torch.cuda.synchronize()
    want = c + 3 * (a.reshape(M, K) @ b.reshape(K, N)).ravel()
    assert tc.cpu().numpy().tobytes() == want.tobytes()
