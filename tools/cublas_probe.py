"""One cuBLAS fp16 8192^3 GEMM (for ncu comparisons with our kernel)."""
import torch
n = 8192
a = torch.randn(n, n, device='cuda').half()
b = torch.randn(n, n, device='cuda').half()
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
