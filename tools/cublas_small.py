"""cuBLASLt's same-operation kernel for small squares (context for the small-shape study):
torch.addmm(C_fp32, A_half, B_half, out_dtype=float32), a few launches per size, for ncu."""
import sys

import torch

for n in [int(x) for x in (sys.argv[1:] or ["1024"])]:
    a = torch.randn(n, n, device="cuda").half()
    b = torch.randn(n, n, device="cuda").half()
    c = torch.randn(n, n, device="cuda")
    for _ in range(4):
        torch.addmm(c, a, b, out_dtype=torch.float32)
    torch.cuda.synchronize()
