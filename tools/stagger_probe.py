"""Staggered 256x512 schedule (TK_STAGGER=1): bitwise check against the default schedule (with
serpentine K off, both accumulate in the same order) and graph-replayed timing, tuning only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("COOLDOWN", "0.5")
os.environ.setdefault("GRAPH", "1")
import torch  # noqa: E402

import tools.bench_variants as bv  # noqa: E402
from paper_2009_12263_b200 import kernel  # noqa: E402
import paper_2009_12263_b200 as tk  # noqa: E402

shapes = [tuple(int(x) for x in s.split("x")) for s in
          os.environ.get("SHAPES", "8192x8192x8192,16384x16384x16384,8192x16384x8192").split(",")]
for (m, n, k) in shapes:
    cfg = kernel.resolve_config(tk.build_dense_config(m, n, k, tk.FLOAT16))
    a, b = bv.rnd(m * k, torch.float16), bv.rnd(k * n, torch.float16)
    c = bv.rnd(m * n, torch.float32)
    outs = []
    for st in ("0", "1"):
        os.environ["TK_STAGGER"], os.environ["TK_SERPENTINE"] = st, "0"
        d = torch.full((m * n,), float("nan"), device="cuda")
        tk.gemm_execute(cfg, a, b, c, d)
        outs.append(d)
    os.environ.pop("TK_SERPENTINE")
    same = torch.equal(outs[0], outs[1])
    print(f"{m}x{n}x{k}: staggered == default bitwise: {same}", flush=True)
    del outs
    for st in ("0", "1", "0", "1"):
        os.environ["TK_STAGGER"] = st
        d = torch.empty(m * n, device="cuda")
        sec = bv.timeit(bv.run(cfg, a, b, c, d))
        bv.report(f"{m}x{n}x{k} stagger={st}", sec, 2.0 * m * n * k, "TFLOPS", tk.last_run()["lane"])
    os.environ.pop("TK_STAGGER")
    del a, b, c
    torch.cuda.empty_cache()
