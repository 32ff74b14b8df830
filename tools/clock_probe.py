"""SM clock under load: a 1-CTA probe kernel records clock64 vs globaltimer while a GEMM loop
runs concurrently (ours vs cuBLAS).  Tuning aid; prints TFLOPS and the probe's MHz."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib, kernel  # noqa: E402

lib = _lib.load()
lib.tk_debug_clock_probe.argtypes = [ctypes.c_double, ctypes.c_void_p]
lib.tk_debug_clock_probe_mhz.restype = ctypes.c_double
n = int(os.environ.get("N", "8192"))
reps = 40
side = torch.cuda.Stream()


def probe(name, fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(reps):
        fn()
        if i == 5:
            lib.tk_debug_clock_probe(ctypes.c_double(10000.0), ctypes.c_void_p(side.cuda_stream))
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{name:40s} {ms:8.3f} ms {flops / ms / 1e9:8.1f} TFLOPS  probe {lib.tk_debug_clock_probe_mhz():7.1f} MHz",
          flush=True)


g = torch.Generator(device="cuda")
g.manual_seed(0)
for dt, tdt in ((tk.FLOAT16, torch.float16), (tk.BFLOAT16, torch.bfloat16)):
    a = torch.randn(n * n, generator=g, device="cuda").to(tdt)
    b = torch.randn(n * n, generator=g, device="cuda").to(tdt)
    c = torch.randn(n * n, generator=g, device="cuda")
    d = torch.empty(n * n, device="cuda")
    cfg = kernel.resolve_config(tk.build_dense_config(n, n, n, dt))
    for env in ({}, {"TK_PAIR_NSUB": "2"}, {"TK_PAIR_CSTREAM": "0", "TK_DBG_SKIP_EPI": "1"}):
        os.environ.pop("TK_PAIR_NSUB", None)
        os.environ.pop("TK_PAIR_CSTREAM", None)
        os.environ.pop("TK_DBG_SKIP_EPI", None)
        os.environ.update(env)
        probe(f"ours {tdt} {env}", lambda: tk.gemm_execute(cfg, a, b, c, d, synchronize=False), 2.0 * n ** 3)
    for k in ("TK_PAIR_NSUB", "TK_PAIR_CSTREAM", "TK_DBG_SKIP_EPI"):
        os.environ.pop(k, None)
    A, B = a.view(n, n), b.view(n, n)
    probe(f"cuBLAS {tdt}", lambda: torch.matmul(A, B), 2.0 * n ** 3)
    C = c.view(n, n)
    probe(f"cuBLAS addmm fp32-out-free {tdt}", lambda: torch.matmul(A, B).float().add_(C), 2.0 * n ** 3)
