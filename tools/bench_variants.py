"""Measure every SURVEY 8d configuration on one B200 (CUDA events, warm-up excluded).

Prints one line per case and writes gpurun_out/variants.json.  Units: TFLOPS with the
reference's flop conventions (real 2MNK, complex 8MNK, dual 6MNK, TC 2*Na*Nb*Nc*Nd) or GB/s
of algorithmic bytes for the HBM-bound diagonal / skinny cases.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_12263_b200 as tk  # noqa: E402
from paper_2009_12263_b200 import components, kernel  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(0)


def rnd(n, dt):
    return torch.randn(n, generator=g, device=dev).to(dt)


from paper_2009_12263_b200.clocks import ClockSampler  # noqa: E402

_clock = {}


def timeit(fn, reps=10, warm=3):
    import time

    torch.cuda.synchronize()
    time.sleep(float(os.environ.get("COOLDOWN", "1.0")))  # let the power/clock state settle
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as cs:
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
    _clock.update(cs.summary())
    try:  # effective SM clock of the last pair-kernel launch, measured in-kernel
        import ctypes as _ct
        from paper_2009_12263_b200 import _lib as _l
        f = _l.load().tk_debug_pair_mhz
        f.restype = _ct.c_double
        _clock["kernel_mhz"] = round(f(), 1)
    except Exception:
        pass
    return s.elapsed_time(e) / reps * 1e-3 / getattr(fn, "per_call", 1)


results = []


def report(name, sec, work, unit, lane, extra=None):
    val = work / sec / (1e12 if unit == "TFLOPS" else 1e9)
    row = {"case": name, "ms": sec * 1e3, "value": val, "unit": unit, "lane": lane,
           "launches": tk.last_run()["launches"], "sm_mhz": _clock.get("sm_mhz"),
           "reasons": _clock.get("reasons"), **(extra or {})}
    results.append(row)
    print(f"{name:48s} {sec * 1e3:9.3f} ms  {val:9.1f} {unit:6s} lane={lane} "
          f"launches={row['launches']} sm={row['sm_mhz']} kmhz={_clock.get('kernel_mhz')} W={_clock.get('power_w')} {row['reasons']}", flush=True)


def run(cfg, a, b, c, d):
    cfg = kernel.resolve_config(cfg)
    f = lambda: tk.gemm_execute(cfg, a, b, c, d, synchronize=False)
    if os.environ.get("GRAPH") == "1":  # replay a CUDA graph of 10 launches (no host overhead)
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
        launches = tk.last_run()["launches"]

        def replay():
            g.replay()
            kernel._LAST["launches"] = launches
        replay.per_call = 10
        return replay
    return f


def dense(n, m=None, k=None, dtype="fp16", trans="nn", name=None):
    m = m or n
    k = k or n
    dt = tk.FLOAT16 if dtype == "fp16" else tk.BFLOAT16
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    cfg = tk.build_dense_config(m, n, k, dt, trans_a=trans[0] == "t", trans_b=trans[1] == "t")
    a, b, c, d = rnd(m * k, tdt), rnd(k * n, tdt), rnd(m * n, torch.float32), \
        torch.empty(m * n, device=dev)
    f = run(cfg, a, b, c, d)
    sec = timeit(f)
    report(name or f"dense {dtype} {trans} {m}x{n}x{k}", sec, 2.0 * m * n * k, "TFLOPS",
           tk.last_run()["lane"])
    return sec


def simt_f32(n):
    """The reference's default dtype (build_dense_config(..., np.float32), api.py:166) on the exact
    CUDA-core lane (reference operation order, bitwise): device buffers, no graph."""
    cfg = tk.build_dense_config(n, n, n, np.float32)
    a, b, c, d = rnd(n * n, torch.float32), rnd(n * n, torch.float32), rnd(n * n, torch.float32), \
        torch.empty(n * n, device=dev)
    cfg = kernel.resolve_config(cfg)
    sec = timeit(lambda: tk.gemm_execute(cfg, a, b, c, d, synchronize=False), reps=3, warm=1)
    report(f"simt f32 {n}^3 (exact lane)", sec, 2.0 * n ** 3, "TFLOPS", tk.last_run()["lane"])


def host_numpy(n):
    """The drop-in call a reference user makes: tk.matmul on numpy host buffers (fp16 A/B,
    fp32 C/D) -- staging copies to the device and D back to the host inside the call."""
    import time

    rng = np.random.default_rng(0)
    a = rng.standard_normal(n * n).astype(np.float16)
    b = rng.standard_normal(n * n).astype(np.float16)
    c = rng.standard_normal(n * n).astype(np.float32)
    d = np.empty(n * n, np.float32)
    cfg = tk.build_dense_config(n, n, n, tk.FLOAT16)
    for _ in range(2):
        tk.matmul(cfg, a, b, c, d)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        tk.matmul(cfg, a, b, c, d)
    sec = (time.perf_counter() - t0) / reps
    report(f"host numpy matmul {n}^3 (wall clock, copies included)", sec, 2.0 * n ** 3, "TFLOPS",
           tk.last_run()["lane"])


def cublas_ref(n, dtype=torch.float16):
    """cuBLAS on the same operation (fp16/bf16 A,B; fp32 C,D; D = A*B + C) via torch.addmm with
    out_dtype=float32 -- the library baseline for the sweep (graph-replayed when GRAPH=1)."""
    a = torch.randn(n, n, generator=g, device=dev).to(dtype)
    b = torch.randn(n, n, generator=g, device=dev).to(dtype)
    c = torch.randn(n, n, generator=g, device=dev)
    f = lambda: torch.addmm(c, a, b, out_dtype=torch.float32)
    if os.environ.get("GRAPH") == "1":
        f()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(10):
                f()

        def replay():
            gr.replay()
        replay.per_call = 10
        fn = replay
    else:
        fn = f
    sec = timeit(fn)
    report(f"cuBLAS addmm {dtype} {n}^3 (same op)", sec, 2.0 * n ** 3, "TFLOPS", "cublas")


def skinny(n, k):
    m = n
    cfg = tk.build_dense_config(m, n, k, tk.FLOAT16)
    a, b, c, d = rnd(m * k, torch.float16), rnd(k * n, torch.float16), \
        rnd(m * n, torch.float32), torch.empty(m * n, device=dev)
    sec = timeit(run(cfg, a, b, c, d))
    byts = 2 * (m * k + k * n) + 8 * m * n
    report(f"skinny fp16 {m}x{n}x{k} (C read, D write)", sec, byts, "GB/s", tk.last_run()["lane"],
           {"tflops": 2.0 * m * n * k / sec / 1e12})


def fused_c3(n):
    m = k = n
    al, be = 1.5, 0.5
    bias = rnd(n, torch.float32)
    for trans in ("nn", "nt", "tn", "tt"):
        cfg = dataclasses.replace(
            tk.build_dense_config(m, n, k, tk.FLOAT16, trans_a=trans[0] == "t",
                                  trans_b=trans[1] == "t"),
            transform_g2s_c=components.scale(be / al), transform_r2s_d=components.scale(al),
            epilogue=components.BiasEpilogue(bias), transform_s2g_d=components.relu)
        a, b, c, d = rnd(m * k, torch.float16), rnd(k * n, torch.float16), \
            rnd(m * n, torch.float32), torch.empty(m * n, device=dev)
        sec = timeit(run(cfg, a, b, c, d))
        report(f"C3 {trans} alpha/beta+bias+relu {n}^3", sec, 2.0 * m * n * k, "TFLOPS",
               tk.last_run()["lane"])


def fused_builder(n):
    m = k = n
    bias = rnd(n, torch.float32)
    cfg = tk.build_fused_config(m, n, k, tk.FLOAT16, bias=bias, relu_on_c=True, relu_on_d=True,
                                add_a=0.5, add_b=-0.25)
    a, b, c, d = rnd(m * k, torch.float16), rnd(k * n, torch.float16), \
        rnd(m * n, torch.float32), torch.empty(m * n, device=dev)
    sec = timeit(run(cfg, a, b, c, d))
    report(f"build_fused_config add_a/add_b/relu/bias {n}^3", sec, 2.0 * m * n * k, "TFLOPS",
           tk.last_run()["lane"])


def pair_op(kind, n, split):
    m = k = n
    half = tk.COMPLEX32 if kind == "complex" else tk.DUAL16
    build = tk.build_complex_config if kind == "complex" else tk.build_dual_config
    cfg = build(m, n, k, half, split=split)
    a, b = rnd(2 * m * k, torch.float16), rnd(2 * k * n, torch.float16)
    c, d = rnd(2 * m * n, torch.float32), torch.empty(2 * m * n, device=dev)
    sec = timeit(run(cfg, a, b, c, d), reps=5)
    flops = (8.0 if kind == "complex" else 6.0) * m * n * k
    report(f"{kind} fp16 {'split' if split else 'interleaved'} {n}^3", sec, flops, "TFLOPS",
           tk.last_run()["lane"])


def diagonal(n):
    cfg = tk.build_diagonal_config(n, tk.FLOAT16)
    a, b, c, d = rnd(n, torch.float16), rnd(n * n, torch.float16), rnd(n * n, torch.float32), \
        torch.empty(n * n, device=dev)
    sec = timeit(run(cfg, a, b, c, d))
    byts = 2 * n + 2 * n * n + 4 * n * n + 4 * n * n
    report(f"diagonal fp16 {n}", sec, byts, "GB/s", tk.last_run()["lane"])


def contraction(na, nb, nc, nd):
    cfg = tk.build_tc_config(na, nb, nc, nd, tk.FLOAT16)
    m, n, k = nb * na, nc, nd
    a, b = rnd(m * k, torch.float16), rnd(k * n, torch.float16)
    d = torch.empty(m * n, device=dev)
    c = torch.empty(0, device=dev)
    sec = timeit(run(cfg, a, b, c, d), reps=3, warm=1)
    report(f"TC D_abc=A_bda*B_dc ({na},{nb},{nc},{nd})", sec, 2.0 * m * n * k, "TFLOPS",
           tk.last_run()["lane"])


def gett_case(spec, sizes):
    d_idx, a_idx, b_idx = spec.split("-")
    cfg = tk.build_gett_config(spec, sizes, tk.FLOAT16)
    m, n, k = cfg.params.gemm_shape
    a = rnd(int(np.prod([sizes[i] for i in a_idx])), torch.float16)
    b = rnd(int(np.prod([sizes[i] for i in b_idx])), torch.float16)
    d = torch.empty(m * n, device=dev)
    c = torch.empty(0, device=dev)
    sec = timeit(run(cfg, a, b, c, d), reps=5, warm=2)
    report(f"GETT {spec} M={m} N={n} K={k}", sec, 2.0 * m * n * k, "TFLOPS", tk.last_run()["lane"])


if __name__ == "__main__":
    which = sys.argv[1:] or ["dense", "sweep", "fused", "pair", "diag", "skinny", "tc", "gett"]
    if "dense" in which:
        dense(8192)
        dense(8192, dtype="bf16")
        for t in ("nt", "tn", "tt"):
            dense(8192, trans=t)
    if "sweep" in which:
        for n in (1024, 2048, 4096, 16384):
            dense(n)
    if "simt" in which:
        for n in (1024, 2048):
            simt_f32(n)
    if "host" in which:
        for n in (2048, 8192):
            host_numpy(n)
    if "cublas" in which:
        for n in (1024, 2048, 4096, 8192, 16384):
            cublas_ref(n)
    if "fused" in which:
        fused_c3(8192)
        fused_builder(8192)
    if "pair" in which:
        for kind in ("complex", "dual"):
            for n in (4096, 8192):
                for split in (True, False):
                    pair_op(kind, n, split)
    if "diag" in which:
        for n in (4096, 8192, 16384):
            diagonal(n)
    if "skinny" in which:
        skinny(8192, 128)
        skinny(8192, 256)
    if "gett" in which:
        gett_case("abcd-aebf-dfce", dict(a=128, b=64, c=128, d=64, e=128, f=64))
        gett_case("abcd-aebf-fdec", dict(a=128, b=64, c=128, d=64, e=128, f=64))
        gett_case("abc-acd-db", dict(a=128, b=8192, c=64, d=8192))
        gett_case("abc-bda-dc", dict(a=64, b=128, c=8192, d=8192))
    if "tc" in which:
        contraction(64, 32, 2048, 2048)
        contraction(64, 128, 8192, 8192)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w") as f:
        json.dump(results, f, indent=1)
