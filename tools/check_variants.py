"""Bitwise cross-check of kernel variants selected by env knobs (tuning safety net):
every variant must reproduce the default kernel's D exactly (same k order per element)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import kernel  # noqa: E402

VARIANTS = [dict(TK_PAIR_BNI="256"), dict(TK_PAIR_BNI="128"), dict(TK_PAIR_BNI="64"),
            dict(TK_PAIR_BNI="128", TK_PAIR_CSTREAM="0"), dict(TK_PAIR_BNI="64", TK_PAIR_CSTREAM="0"),
            dict(TK_PAIR_NSUB="2"), dict(TK_PAIR_CSTREAM="0")]
if os.environ.get("VARIANTS"):
    VARIANTS = [dict(kv.split("=") for kv in v.split("+")) for v in os.environ["VARIANTS"].split(",")]
KEYS = {k for v in VARIANTS for k in v}
os.environ["TK_SERPENTINE"] = "0"  # same k order in every tile, so variants must agree bitwise
shapes = [(1024, 1024, 1024), (4096, 4096 + 256, 4096), (3000, 5000, 1000), (8192, 2048, 512),
          (2048, 8192 + 64, 2048), (640, 200, 704)]
g = torch.Generator(device="cuda")
g.manual_seed(1)
bad = 0
for (m, n, k) in shapes:
    for trans in ("nn", "tt"):
        cfg = kernel.resolve_config(tk.build_dense_config(m, n, k, tk.FLOAT16, trans_a=trans[0] == "t",
                                                          trans_b=trans[1] == "t"))
        a = torch.randn(m * k, generator=g, device="cuda").half()
        b = torch.randn(k * n, generator=g, device="cuda").half()
        c = torch.randn(m * n, generator=g, device="cuda")
        for key in KEYS:
            os.environ.pop(key, None)
        d0 = torch.full((m * n,), float("nan"), device="cuda")
        tk.gemm_execute(cfg, a, b, c, d0)
        A = a.view(k, m).t() if trans[0] == "n" else a.view(m, k)
        B = b.view(n, k).t() if trans[1] == "n" else b.view(k, n)
        ref = (A.double() @ B.double()).t().reshape(-1) + c.double() if True else None
        err = ((d0.double() - ref).abs().max() / ref.abs().max()).item()
        print(f"{m}x{n}x{k} {trans} default: rel err vs f64 {err:.2e}", flush=True)
        for v in VARIANTS:
            for key in KEYS:
                os.environ.pop(key, None)
            os.environ.update(v)
            d1 = torch.full((m * n,), float("nan"), device="cuda")
            tk.gemm_execute(cfg, a, b, c, d1)
            same = torch.equal(d0, d1)
            bad += not same
            print(f"   {v}: {'bitwise equal' if same else 'MISMATCH max %g' % (d0 - d1).abs().max().item()}",
                  flush=True)
print("FAILURES", bad)
