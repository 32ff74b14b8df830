"""Diagnose the dense 8192^3 pair kernel: which part of the step limits throughput.

Cases (env knobs read per call by libtk_sm100.so): default streamed-C epilogue, register
epilogue, C = Zero, mainloop only (epilogue skipped), MMA issue only (no operand loads),
the 4-CTA multicast kernel, and cuBLAS (torch.matmul) for reference.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("COOLDOWN", "1.0")
import torch  # noqa: E402

import tools.bench_variants as bv  # noqa: E402

n = int(os.environ.get("N", "8192"))
KN = ("TK_PAIR_CSTREAM", "TK_DBG_SKIP_EPI", "TK_DBG_NO_LOAD", "TK_TC_KERNEL", "TK_GROUP_M",
      "TK_POLICY_AB", "TK_DBG_NO_MMA", "TK_L2_PROMO", "TK_PAIR_NSUB")


SEL = os.environ.get("CASES")  # comma-separated subset of case tags (default: all)


def case(name, tag=None, **env):
    if SEL and (tag or name) not in SEL.split(","):
        return
    for k in KN:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    bv.dense(n, name=name)


case("default (streamed C)", "default")
case("register epilogue", "regepi", TK_PAIR_CSTREAM=0)
case("mainloop only", "mainloop", TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1)
case("MMA issue only", "mmaonly", TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_LOAD=1)
case("loads only (no MMA)", "loadsonly", TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_MMA=1)
case("nsub2 (256x512) streamed C", "nsub2", TK_PAIR_NSUB=2)
case("nsub2 register epilogue", "nsub2", TK_PAIR_NSUB=2, TK_PAIR_CSTREAM=0)
case("nsub2 mainloop only", "nsub2", TK_PAIR_NSUB=2, TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1)
case("nsub2 loads only", "nsub2", TK_PAIR_NSUB=2, TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_MMA=1)
case("nsub2 MMA only", "nsub2", TK_PAIR_NSUB=2, TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1, TK_DBG_NO_LOAD=1)
case("quad multicast", "quad", TK_TC_KERNEL="quad")
case("quad mainloop only", "quadml", TK_TC_KERNEL="quad", TK_DBG_SKIP_EPI=1)
for g in (4, 16):
    case(f"group_m {g}", "group", TK_GROUP_M=g)
case("policy normal", "policy", TK_POLICY_AB=0)
for k in KN:
    os.environ.pop(k, None)

for p in (0, 128):
    case(f"L2 promotion {p}", "promo", TK_L2_PROMO=p)
    case(f"L2 promotion {p} mainloop", "promo", TK_L2_PROMO=p, TK_PAIR_CSTREAM=0, TK_DBG_SKIP_EPI=1)
for k in KN:
    os.environ.pop(k, None)
for dt in ((torch.float16, torch.bfloat16) if not SEL or "cublas" in SEL else ()):
    a = torch.randn(n, n, device="cuda").to(dt)
    b = torch.randn(n, n, device="cuda").to(dt)
    sec = bv.timeit(lambda: torch.matmul(a, b))
    bv.report(f"cuBLAS torch.matmul {dt}", sec, 2.0 * n ** 3, "TFLOPS", "cublas")
