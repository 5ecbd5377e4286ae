"""cuBLAS comparators (through torch) for the GETT rooflines: DGEMM and SGEMM
(fp32, TF32 off) at 4096^3 and the c2-shaped problem.  Plumbing only — not a
product path.  Prints one JSON object per measurement."""
import json

import torch


def bench(dtype, n, reps=10, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n ** 3 / best / 1e9


if __name__ == "__main__":
    for n in (4096, 8192):
        print(json.dumps({"op": "cublas_dgemm", "n": n, "tflops": round(bench(torch.float64, n), 3)}))
    print(json.dumps({"op": "cublas_sgemm_fp32", "n": 4096, "tflops": round(bench(torch.float32, 4096), 3)}))
    print(json.dumps({"op": "cublas_sgemm_tf32", "n": 4096, "tflops": round(bench(torch.float32, 4096, tf32=True), 3)}))
