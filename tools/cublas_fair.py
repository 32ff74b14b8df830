"""cuBLAS on the same operation as the bench (fp16/bf16 A,B; fp32 C,D; D = A*B + C) for a
like-for-like library comparison (torch.addmm with out_dtype=float32 -> cublasLt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import tools.bench_variants as bv  # noqa: E402

n = int(os.environ.get("N", "8192"))
for dt in (torch.float16, torch.bfloat16):
    a = torch.randn(n, n, device="cuda").to(dt)
    b = torch.randn(n, n, device="cuda").to(dt)
    c = torch.randn(n, n, device="cuda")
    d = torch.empty(n, n, device="cuda")
    try:
        sec = bv.timeit(lambda: torch.addmm(c, a, b, out_dtype=torch.float32))
        bv.report(f"cuBLAS addmm {dt}->fp32 (C fp32) {n}^3", sec, 2.0 * n ** 3, "TFLOPS", "cublas")
    except Exception as e:
        print("addmm out_dtype failed:", e)
    try:
        sec = bv.timeit(lambda: torch.mm(a, b, out_dtype=torch.float32))
        bv.report(f"cuBLAS mm {dt}->fp32 (no C) {n}^3", sec, 2.0 * n ** 3, "TFLOPS", "cublas")
    except Exception as e:
        print("mm out_dtype failed:", e)
    sec = bv.timeit(lambda: torch.matmul(a, b))
    bv.report(f"cuBLAS matmul {dt}->{dt} {n}^3", sec, 2.0 * n ** 3, "TFLOPS", "cublas")
