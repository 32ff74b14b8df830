"""A/B of single-wave (small) dense shapes: whole-K pair tiles vs the on-chip split-K kernel
(TK_KSPLIT=0 / 2, two or one K-blocks per stage) vs cuBLASLt on the same operation.
Graph-replayed (10 launches per replay, no host overhead), CUDA events, device time per GEMM.

    python tools/small_ab.py [m,n,k ...]
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib, kernel  # noqa: E402

dev = torch.device("cuda")


def graph_time(f, reps=20):
    f()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / (10 * reps) * 1e3)  # us per GEMM
    return best


def main():
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [
        (1024, 1024, 1024), (1024, 1024, 2048), (1024, 1024, 4096), (1024, 1024, 8192),
        (768, 768, 768), (512, 512, 512), (512, 1024, 2048), (1024, 2048, 1024), (1536, 1536, 1536)]
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for (m, n, k) in shapes:
        a = torch.randn(m * k, generator=g, device=dev).half()
        b = torch.randn(k * n, generator=g, device=dev).half()
        c = torch.randn(m * n, generator=g, device=dev)
        cfg = kernel.resolve_config(tk.build_dense_config(m, n, k, tk.FLOAT16))
        row = []
        ref = None
        for label, ks, kps, pdl in (("pair", "0", None, None), ("ks-nt1", "2", "1", None), ("ks-nt2", "2", "2", None),
                                    ("ks-w256", "2", "w", None), ("auto", None, None, None)):
            _lib.tune_reset()
            if ks is not None:
                _lib.tune("TK_KSPLIT", ks)
            if kps == "w":
                _lib.tune("TK_KSPLIT_BNI", "256")
            elif kps is not None:
                _lib.tune("TK_KSPLIT_NT", kps)
            if pdl is not None:
                _lib.tune("TK_PDL", pdl)
            d = torch.empty(m * n, device=dev)
            f = lambda: tk.gemm_execute(cfg, a, b, c, d, synchronize=False)
            us = graph_time(f)
            kern = tk.last_run()["plan"]["kernel"]
            if ref is None:
                ref = d.clone()
            err = ((d - ref).abs().max() / ref.abs().max()).item()
            row.append(f"{label}[{kern}] {us:6.2f} us {2 * m * n * k / us * 1e-6:6.1f} TF err {err:.1e}")
        _lib.tune_reset()
        A = a.view(k, m).t()
        B = b.view(n, k).t()
        C = c.view(n, m).t()
        out = torch.empty(n, m, device=dev).t()
        us = graph_time(lambda: torch.addmm(C, A, B, out_dtype=torch.float32, out=out))
        row.append(f"cublasLt {us:6.2f} us {2 * m * n * k / us * 1e-6:6.1f} TF")
        print(f"{m}x{n}x{k}: " + " | ".join(row), flush=True)


if __name__ == "__main__":
    main()
