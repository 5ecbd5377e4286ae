"""Where does the DGETT bulk-add epilogue go wrong? small GEMMs, error map."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402

g.set_kernel("tiled")
for (M, N, K) in [(128, 256, 96), (1024, 2048, 64), (2048, 2048, 256), (1920, 1664, 128), (384, 8192, 512), (1152, 1152, 64)]:
    rng = np.random.default_rng(0)
    A = rng.integers(-3, 4, (M, K)).astype(np.float64)
    B = rng.integers(-3, 4, (N, K)).astype(np.float64)
    C = rng.integers(-3, 4, (M, N)).astype(np.float64)
    want = C + A @ B.T
    c = C.ravel().copy()
    assert g.dgett(2, (M, K), (K, 1), A.ravel(), 2, (N, K), (K, 1), B.ravel(), 1, (1,), (1,), (0, 1), (N, 1), c) == []
    got = c.reshape(M, N)
    bad = got != want
    print(M, N, K, g.last_kernel(), "bad", int(bad.sum()), "of", M * N)
    if bad.any():
        r, cidx = np.nonzero(bad)
        print("  rows", np.unique(r)[:20], "cols", np.unique(cidx)[:40])
        i, j = r[0], cidx[0]
        print("  first", i, j, "got", got[i, j], "want", want[i, j], "C0", C[i, j], "acc", (A @ B.T)[i, j])
        d = got - C
        acc = A @ B.T
        # is got-C a permuted acc?
        print("  row of got-C:", d[i, :8], "acc:", acc[i, :8])
        tm, tn = (M + 127) // 128, (N + 127) // 128
        cnt = np.zeros((tm, tn), int)
        for a_, b_ in zip(r, cidx):
            cnt[a_ // 128, b_ // 128] += 1
        print("  bad per tile (tile rows x tile cols):")
        for row in cnt:
            print("   ", " ".join(f"{x:5d}" for x in row))
        t = np.nonzero(cnt)
        ti, tj = t[0][0], t[1][0]
        blk = bad[ti * 128:(ti + 1) * 128, tj * 128:(tj + 1) * 128]
        print("  tile", ti, tj, "bad rows", np.nonzero(blk.any(1))[0][:64], "bad col chunks", np.unique(np.nonzero(blk)[1] // 32))
        ex = (got - want)[ti * 128:(ti + 1) * 128, tj * 128:(tj + 1) * 128]
        print("  extra sample", ex[blk][:8])
        sl = (slice(ti * 128, (ti + 1) * 128), slice(tj * 128, (tj + 1) * 128))
        dd = (got - C)[sl][blk]
        for k0 in range(0, K // 32):
            for k1 in range(k0 + 1, K // 32 + 1):
                part = (A[:, 32 * k0:32 * k1] @ B[:, 32 * k0:32 * k1].T)[sl][blk]
                full = acc[sl][blk]
                for name, cand in (("part", part), ("full+part", full + part), ("2full-part", 2 * full - part)):
                    if np.array_equal(cand, dd):
                        print("  MATCH", name, "kb", k0, k1)
