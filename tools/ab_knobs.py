"""A/B timing of tuning-knob settings on one GEMM (CUDA events, in-kernel clock).

    python tools/ab_knobs.py dense 8192 "TK_NSUB2_OVERLAP=0" "TK_NSUB2_OVERLAP=16" [--reps 20 --rounds 3]

Each setting is timed `--rounds` times, interleaved (A B A B ...) with a cool-down between runs,
so box-to-box power state drifts hit every setting alike.  Prints TFLOPS (2MNK) and the SM clock
seen inside the kernel (tk_debug_pair_mhz) per run, then the median per setting.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=["dense", "dense_c0", "fused", "complex_il", "complex_split"])
    ap.add_argument("n", type=int)
    ap.add_argument("settings", nargs="+")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--cool", type=float, default=1.0)
    ap.add_argument("--graph", action="store_true", help="replay a CUDA graph of 10 launches (no host overhead)")
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    a = torch.randn(n * n, generator=g, device=dev).half()
    b = torch.randn(n * n, generator=g, device=dev).half()
    c = torch.randn(n * n, generator=g, device=dev)
    d = torch.empty(n * n, device=dev)
    flops = 2.0 * n ** 3
    if args.case.startswith("complex"):
        split = args.case == "complex_split"
        a = torch.randn(2 * n * n, generator=g, device=dev).half()
        b = torch.randn(2 * n * n, generator=g, device=dev).half()
        c = torch.randn(2 * n * n, generator=g, device=dev)
        d = torch.empty(2 * n * n, device=dev)
        cfg = tk.build_complex_config(n, n, n, tk.COMPLEX32, split=split)
        flops = 8.0 * n ** 3
    elif args.case == "fused":
        cfg = tk.build_fused_config(n, n, n, np.float16, bias=torch.randn(n, generator=g, device=dev),
                                    relu_on_c=True, relu_on_d=True, add_a=0.5, add_b=-0.25)
    else:
        cfg = tk.build_dense_config(n, n, n, tk.FLOAT16)
    if args.case == "dense_c0":
        c.zero_()
    mhz = _lib.load().tk_debug_pair_mhz
    mhz.restype = ctypes.c_double
    res = {s: [] for s in args.settings}
    for r in range(args.rounds):
        for setting in args.settings:
            _lib.tune_reset()
            for kv in filter(None, setting.split(",")):
                k, v = kv.split("=")
                _lib.tune(k, v)
            for _ in range(3):
                tk.matmul(cfg, a, b, c, d, synchronize=False)
            torch.cuda.synchronize()
            step, per = (lambda: tk.matmul(cfg, a, b, c, d, synchronize=False)), 1
            if args.graph:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for _ in range(10):
                        tk.matmul(cfg, a, b, c, d, synchronize=False)
                step, per = gr.replay, 10
                step()
                torch.cuda.synchronize()
            time.sleep(args.cool)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(args.reps):
                step()
            s1.record()
            torch.cuda.synchronize()
            ms = s0.elapsed_time(s1) / (args.reps * per)
            tf = flops / (ms * 1e-3) / 1e12
            us = ms * 1e3
            res[setting].append((tf, mhz()))
            print(f"round {r} {setting:40s} {us:8.2f} us {tf:8.1f} TF  {mhz():7.1f} MHz  plan={tk.last_run()['plan']['kernel']}"
                  f"/{tk.last_run()['plan']['tile_n']}/ovl{tk.last_run()['plan']['overlap_kb']}", flush=True)
    out = {s: {"tflops_median": float(np.median([x[0] for x in v])),
               "mhz_median": float(np.median([x[1] for x in v])),
               "per_clock": float(np.median([x[0] * 1e12 / (148 * 8192 * x[1] * 1e6) for x in v]))}
           for s, v in res.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
