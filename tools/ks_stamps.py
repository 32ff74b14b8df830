"""Timeline of one small GEMM inside a graph-replayed stream of them (stamps build:
tools/build_variants.sh stamps "-DTK_STAMPS=1", TK_SM100_LIB=build/var_stamps/libtk_sm100.so).
CTA-0 globaltimer stamps in us after its entry; `prev exit` is the previous launch's exit
(negative: this CTA entered before it -- programmatic dependent launch)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TK_DBG_CTA", "0")
import torch  # noqa: E402

import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib, kernel  # noqa: E402

lib = _lib.load()
NAMES = {"ksplit": ["entry", "inputs ok", "1st full", "sent", "acc full", "partial in", "D issued", "exit",
                    "D read", "max exit", "max D issued", "max acc full", "max inputs ok", "max 1st full",
                    "pre-math"],
         "pair": ["entry", "prologue", "1st full", "last MMA issued", "last acc full", "epilogue done",
                  "stores drained", "exit", "epi:tmem", "epi:math", "epi:store", "epi:C ready"]}
SHAPES = [tuple(int(x) for x in s.split("x")) for s in
          os.environ.get("SHAPES", "512x512x512,1024x1024x1024,1024x1024x8192").split(",")]
for (m, n, k) in SHAPES:
    for ks in ("2", "0"):
        _lib.tune("TK_KSPLIT", ks)
        cfg = kernel.resolve_config(tk.build_dense_config(m, n, k, tk.FLOAT16))
        a = torch.randn(m * k, device="cuda").half()
        b = torch.randn(k * n, device="cuda").half()
        c = torch.randn(m * n, device="cuda")
        d = torch.empty(m * n, device="cuda")
        f = lambda: tk.gemm_execute(cfg, a, b, c, d, synchronize=False)
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
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 100 * 1e3
        kern = tk.last_run()["plan"]["kernel"]
        out = (ctypes.c_double * 16)()
        lib.tk_debug_pair_ts(out)
        names = NAMES.get(kern, NAMES["pair"])
        line = "  ".join(f"{nm}={out[i]:.2f}" for i, nm in enumerate(names))
        prev = f"  prev exit={out[15]:.2f}" if kern == "ksplit" else ""
        print(f"{m}x{n}x{k} [{kern}] {us:.2f} us/GEMM: {line}{prev}", flush=True)
    _lib.tune_reset()
