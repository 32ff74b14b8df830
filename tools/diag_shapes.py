"""Mainloop diagnostics across shapes (L2-resident vs DRAM-streaming operands), tuning only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("COOLDOWN", "0.5")
import torch  # noqa: E402

import tools.bench_variants as bv  # noqa: E402

KN = ("TK_PAIR_CSTREAM", "TK_DBG_SKIP_EPI", "TK_DBG_NO_LOAD", "TK_DBG_NO_MMA", "TK_PAIR_NSUB",
      "TK_GROUP_M", "TK_DBG_C_ZERO", "TK_POL_A", "TK_POL_B")
CASES = {
    "full": {},
    "mainloop": dict(TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1),
    "loads": dict(TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_MMA=1),
    "mma": dict(TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_LOAD=1),
    "czero": dict(TK_DBG_C_ZERO=1),
    "regepi": dict(TK_PAIR_CSTREAM=0),
    "regepi_czero": dict(TK_PAIR_CSTREAM=0, TK_DBG_C_ZERO=1),
}
shapes = [tuple(int(x) for x in s.split("x")) for s in
          os.environ.get("SHAPES", "8192x8192x2048,8192x8192x4096,8192x8192x8192").split(",")]
cases = os.environ.get("CASES", "full,mainloop,loads,mma").split(",")
extras = [dict(kv.split("=") for kv in e.split("+") if kv)
          for e in os.environ.get("EXTRAS", os.environ.get("EXTRA", "").replace(",", "+")).split(",")]
for (m, n, k) in shapes:
    for extra in extras:
        for c in cases:
            for key in KN:
                os.environ.pop(key, None)
            os.environ.update({a: str(b) for a, b in {**CASES[c], **extra}.items()})
            bv.dense(n, m=m, k=k, name=f"{m}x{n}x{k} {c} {extra}")
    for key in KN:
        os.environ.pop(key, None)
    if os.environ.get("CUBLAS", "1") == "1":
        a = torch.randn(m, k, device="cuda").half()
        b = torch.randn(k, n, device="cuda").half()
        sec = bv.timeit(lambda: torch.matmul(a, b))
        bv.report(f"{m}x{n}x{k} cuBLAS fp16", sec, 2.0 * m * n * k, "TFLOPS", "cublas")
