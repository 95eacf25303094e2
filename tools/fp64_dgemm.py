"""cuBLAS DGEMM / ZGEMM throughput via torch (the library FP64 reference point).

Measured once per box so the PSCA roofline has an FP64 denominator; the
driver's MEASURED_PEAKS.json records only bf16 and HBM.
"""
import json

import torch


def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    mult = 8 if dtype.is_complex else 2
    return mult * n ** 3 / (ms * 1e-3) / 1e12, ms


if __name__ == "__main__":
    for dt, n in ((torch.float64, 8192), (torch.float64, 16384), (torch.complex128, 8192)):
        tf, ms = bench(dt, n)
        print(json.dumps({"kernel": f"torch.matmul {dt} {n}^3", "tflops": round(tf, 3), "ms": round(ms, 3)}))
