import os, sys, dataclasses
sys.path.insert(0, os.getcwd())
import torch, paper_2009_12263_b200 as tk
from paper_2009_12263_b200 import components, kernel
n = 8192
dev = torch.device("cuda")
bias = torch.randn(n, device=dev)
cfg = dataclasses.replace(tk.build_dense_config(n, n, n, tk.FLOAT16, trans_b=True),
    transform_g2s_c=components.scale(1/3), transform_r2s_d=components.scale(1.5),
    epilogue=components.BiasEpilogue(bias), transform_s2g_d=components.relu)
a = torch.randn(n*n, device=dev).half(); b = torch.randn(n*n, device=dev).half()
c = torch.randn(n*n, device=dev); d = torch.empty(n*n, device=dev)
for _ in range(4):
    tk.gemm_execute(cfg, a, b, c, d, synchronize=False)
torch.cuda.synchronize()
