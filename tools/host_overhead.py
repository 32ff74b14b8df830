"""Per-call host overhead of the drop-in path (no graph replay): CPU wall time per call of
`tk.matmul(cfg, <device tensors>, synchronize=False)` and of the bare C ABI `tk_gemm` (ctypes,
the plan lowered once) on a problem whose device time is a few microseconds, so the loop is
host-bound; and, at 1024^3, the stream period of back-to-back calls vs the graph-replayed
device time.  Prints one JSON line."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib, kernel  # noqa: E402


def bufs(n):
    a = torch.randn(n * n, device="cuda").half()
    b = torch.randn(n * n, device="cuda").half()
    c = torch.randn(n * n, device="cuda")
    return a, b, c, torch.empty_like(c)


def host_loop(fn, reps):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / reps * 1e6, (t2 - t0) / reps * 1e6  # us issue, us period


out = {}
for n in (256, 1024):
    cfg = kernel.resolve_config(tk.build_dense_config(n, n, n, tk.FLOAT16))
    a, b, c, d = bufs(n)
    issue, period = host_loop(lambda: tk.matmul(cfg, a, b, c, d, synchronize=False), 2000)
    out[f"matmul_{n}"] = {"host_us_per_call": round(issue, 2), "stream_period_us": round(period, 2)}
    # the C ABI alone: the same lowered plan, one ctypes call per GEMM
    prep = kernel.prepare(cfg, None)
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    args = (prep.plan_ref, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
            ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(d.data_ptr()), None, None, None, 0,
            ctypes.c_void_p(s))
    issue, period = host_loop(lambda: lib.tk_gemm(*args), 2000)
    out[f"tk_gemm_{n}"] = {"host_us_per_call": round(issue, 2), "stream_period_us": round(period, 2)}
    # graph-replayed device time for reference
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            tk.matmul(cfg, a, b, c, d, synchronize=False)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    out[f"graph_{n}"] = {"device_us_per_gemm": round(e0.elapsed_time(e1) * 1e3 / 500, 2)}
print(json.dumps(out))
