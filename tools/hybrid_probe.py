"""Premise check for a GPC-aware hybrid launch: the 4-CTA multicast kernel (33 clusters fit)
and the CTA-pair kernel run concurrently on two streams over disjoint column slabs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import kernel  # noqa: E402

m = k = 8192
nq = int(os.environ.get("NQ", "7424"))
np_ = 8192 - nq
a = torch.randn(m * k, device="cuda").half()
b = torch.randn(k * 8192, device="cuda").half()
c = torch.randn(m * 8192, device="cuda")
d = torch.empty(m * 8192, device="cuda")
cq = kernel.resolve_config(tk.build_dense_config(m, nq, k, tk.FLOAT16))
cp = kernel.resolve_config(tk.build_dense_config(m, np_, k, tk.FLOAT16))
bq, bp = b[: k * nq], b[k * nq:]
cq_, cp_ = c[: m * nq], c[m * nq:]
dq, dp = d[: m * nq], d[m * nq:]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def step(mode):
    if mode in ("both", "quad"):
        os.environ["TK_TC_KERNEL"] = "quad"
        tk.gemm_execute(cq, a, bq, cq_, dq, synchronize=False, stream=s1)
    if mode in ("both", "pair"):
        os.environ["TK_TC_KERNEL"] = "pair"
        if mode == "both":
            os.environ["TK_PAIR_GRID"] = os.environ.get("PGRID", "8")
        tk.gemm_execute(cp, a, bp, cp_, dp, synchronize=False, stream=s2)
        os.environ.pop("TK_PAIR_GRID", None)


for mode in ("quad", "pair", "both"):
    for _ in range(3):
        step(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        step(mode)
        ev = torch.cuda.Event()
        # join: each rep starts when both streams finished the previous one
        ev.record(s2)
        s1.wait_event(ev)
        ev2 = torch.cuda.Event()
        ev2.record(s1)
        s2.wait_event(ev2)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    n = {"quad": nq, "pair": np_, "both": 8192}[mode]
    print(f"{mode:5s} n={n:5d}: {ms:.3f} ms  {2.0 * m * n * k / ms / 1e9:.1f} TFLOPS", flush=True)
