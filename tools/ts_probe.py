"""Where does a small pair-kernel launch spend its time: CTA-0 globaltimer stamps (us).
Needs a build with the stamps compiled in: tools/build_variants.sh stamps "-DTK_STAMPS=1" and
TK_SM100_LIB=build/var_stamps/libtk_sm100.so."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TK_DBG_CTA", "0")
import torch  # noqa: E402

import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib, kernel  # noqa: E402

lib = _lib.load()
names = ["entry", "prologue", "1st full", "last MMA issued", "last acc full", "epilogue done", "stores drained",
         "exit", "epi:tmem", "epi:math", "epi:store", "epi:C ready", "1st issue", "max 1st issue"]
SHAPES = [tuple(int(x) for x in s.split("x")) for s in
          os.environ.get("SHAPES", "1024x1024x320,1024x1024x1024,1024x1024x4096,2048x2048x2048").split(",")]
for (m, n, k) in SHAPES:
    cfg = kernel.resolve_config(tk.build_dense_config(m, n, k, tk.FLOAT16))
    a = torch.randn(m * k, device="cuda").half()
    b = torch.randn(k * n, device="cuda").half()
    c = torch.randn(m * n, device="cuda")
    d = torch.empty(m * n, device="cuda")
    for _ in range(5):
        tk.gemm_execute(cfg, a, b, c, d)
    torch.cuda.synchronize()
    for i in range(16):
        pass
    out = (ctypes.c_double * 16)()
    lib.tk_debug_pair_ts(out)
    print(f"{m}x{n}x{k}: " + "  ".join(f"{nm}={v:.2f}" for nm, v in zip(names, out) if nm != "-"))
