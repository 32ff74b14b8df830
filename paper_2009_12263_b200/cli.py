"""``python -m paper_2009_12263_b200.cli {check,bench,sweep}`` -- the reference CLI on the B200.

Same subcommands, flags, CSV schema and exit codes as the reference harness
(``pkg/src/tilekit/bench.py:1-558``: ``check`` exits 0 within tolerance / 1 otherwise / 2 on a
configuration error; ``bench`` emits one CSV row, best-of-R GFLOP/s with the warm-up excluded;
``sweep`` reads a ``key=value`` file whose keys are CSV column names).  The CSV keeps the
reference's 21 columns and appends GPU columns: ``tflops``, ``gbs`` (algorithmic bytes),
``pct_peak`` (of the measured bf16 peak in MEASURED_PEAKS.json, or GB/s of the measured copy
bandwidth for the HBM-bound variants), ``sm_mhz``, ``lane`` and ``launches``.

Timing is on the device (CUDA events, synchronised).  ``check`` compares against a float64
(complex128) numpy product computed here -- the reference's brute-force oracle semantics
(``reference.py:15-122``) -- and, for the diagonal variant, also against the enumerated
executed/skipped iteration counts (``bench.py:168-193``).
"""

from __future__ import annotations

import argparse
import dataclasses
import itertools
import json
import os
import statistics
import sys

import numpy as np

from . import api, dtypes, kernel
from .clocks import ClockSampler
from .components import ConfigError

CSV_COLUMNS = [
    "variant", "m", "n", "k", "block_m", "block_n", "block_k",
    "op_m", "op_n", "op_k", "threads", "reps", "sec_mean", "sec_std",
    "gflops", "max_rel_err", "global_loads", "global_stores",
    "operator_invocations", "iters_executed", "iters_skipped",
]
GPU_COLUMNS = ["tflops", "gbs", "pct_peak", "sm_mhz", "lane", "launches"]

DTYPES = {
    "f32": np.dtype(np.float32), "f64": np.dtype(np.float64),
    "c64": np.dtype(np.complex64), "c128": np.dtype(np.complex128),
    "dual32": dtypes.DUAL32, "dual64": dtypes.DUAL64,
    "f16": dtypes.FLOAT16, "bf16": dtypes.BFLOAT16,
    "c32": dtypes.COMPLEX32, "dual16": dtypes.DUAL16,
}
# normwise tolerance: reference values for its own dtypes (bench.py:57-60); half storage is
# judged against the fp16/bf16-rounded inputs with the FP32-accumulation bound 8*2^-24*sqrt(K)
TOLERANCES = {"f32": 1e-5, "f64": 1e-12, "c64": 1e-5, "c128": 1e-12, "dual32": 1e-5,
              "dual64": 1e-12}


def _tolerance(name, k):
    return TOLERANCES.get(name, 8.0 * 2.0 ** -24 * np.sqrt(k))


def _peaks():
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 1590.0, 6650.0


class Case:
    """Prepared device buffers, a runner and an oracle check for one variant."""

    def __init__(self, variant, shape, config, bufs, flops, nbytes, want, read_d, tol,
                 extra_checks=None, hbm=False):
        self.variant, self.gemm_shape, self.config = variant, shape, config
        self.bufs, self.flops, self.nbytes, self.want = bufs, flops, nbytes, want
        self.read_d, self.tol, self.hbm = read_d, tol, hbm
        self.extra_checks = extra_checks or (lambda c: [])
        res = kernel.resolve_config(config)
        self.block = res.params.block_tile
        self.op = res.params.operator_shape

    def run(self, synchronize=True):
        return kernel.gemm_execute(self.config, *self.bufs, synchronize=synchronize)

    def rel_err(self):
        got = np.asarray(self.read_d(), dtype=np.complex128 if np.iscomplexobj(self.want)
                         else np.float64)
        denom = float(np.max(np.abs(self.want))) or 1.0
        return float(np.max(np.abs(got - self.want)) / denom)


def _torch():
    import torch

    return torch


def _dev(x):
    torch = _torch()
    x = np.asarray(x)
    flat = np.ascontiguousarray(x.ravel(order="F"))
    if x.dtype == dtypes.BFLOAT16:
        return torch.from_numpy(flat.view(np.uint16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(flat).cuda()


def _draw(rng, shape, dt):
    """Random values representable in ``dt`` (returned widened for the f64 check)."""
    if dtypes.pair_kind(dt):
        sc = dtypes.storage_scalar(dt)
        p0 = rng.standard_normal(shape).astype(sc)
        p1 = rng.standard_normal(shape).astype(sc)
        return p0, p1
    return rng.standard_normal(shape).astype(dt)


def _wide(x):
    return np.asarray(x).astype(np.float64)


def prepare(args, rng) -> Case:
    name = args.dtype
    # like the reference CLI (bench.py:223-254): a pair variant given a real dtype takes the
    # matching pair type of the same storage width
    if args.variant == "complex" and not name.startswith("c"):
        name = {"f16": "c32", "bf16": "c32", "f32": "c64"}.get(name, "c128")
    elif args.variant == "dual" and not name.startswith("dual"):
        name = {"f16": "dual16", "bf16": "dual16", "f32": "dual32"}.get(name, "dual64")
    args.dtype = name
    dt = DTYPES[name]
    v = args.variant
    half = dtypes.is_half(dt)
    acc = api.accumulator_dtype(dt)
    if v in ("dense", "fused", "diagonal"):
        if dtypes.pair_kind(dt):
            raise ConfigError(f"{v} variant expects a real dtype")
        m, n, k = (args.n, args.n, args.n) if v == "diagonal" else (args.m, args.n, args.k)
        ta, tb = args.trans[0] == "t", args.trans[1] == "t"
        a = _draw(rng, (m,) if v == "diagonal" else (m, k), dt)
        b = _draw(rng, (k, n), dt)
        c = rng.standard_normal((m, n)).astype(acc)
        if v == "dense":
            cfg = api.build_dense_config(m, n, k, dt, trans_a=ta, trans_b=tb,
                                         wide_accumulate=args.wide, block_tile=args.block,
                                         operator_shape=args.op, shared_pad=args.pad,
                                         worker_threads=args.threads)
            kernel.resolve_config(cfg)
            want = _wide(a) @ _wide(b) + _wide(c)
            abuf = _dev(a.T if ta else a) if ta else _dev(a)
            bbuf = _dev(b.T if tb else b) if tb else _dev(b)
        elif v == "fused":
            bias = rng.standard_normal(n).astype(acc)
            cfg = api.build_fused_config(m, n, k, dt, bias=bias, relu_on_c=True, relu_on_d=True,
                                         add_a=0.5, add_b=-0.25, block_tile=args.block,
                                         operator_shape=args.op, worker_threads=args.threads)
            kernel.resolve_config(cfg)
            want = np.maximum((_wide(a) + 0.5) @ (_wide(b) - 0.25) + np.maximum(_wide(c), 0)
                              + _wide(bias)[None, :], 0)
            abuf, bbuf = _dev(a), _dev(b)
        else:
            cfg = api.build_diagonal_config(n, dt, block_tile=args.block, operator_shape=args.op,
                                            worker_threads=args.threads)
            kernel.resolve_config(cfg)
            want = _wide(a)[:, None] * _wide(b) + _wide(c)
            abuf, bbuf = _dev(a), _dev(b)
        d = _torch().zeros(m * n, dtype=dtypes.torch_scalar(acc), device="cuda")
        flops = 2.0 * m * n * k
        nbytes = (2 * n if v == "diagonal" else dt.itemsize * m * k) + dt.itemsize * k * n \
            + 2 * acc.itemsize * m * n
        read = lambda: d.cpu().numpy().reshape((m, n), order="F")

        def extra(counters):
            if v != "diagonal":
                return []
            bm, bn, bk = kernel.resolve_config(cfg).params.block_tile
            exe = sum(1 for i0 in range(0, n, bm) for _ in range(0, n, bn)
                      for k0 in range(0, n, bk) if max(i0, k0) < min(i0 + bm, k0 + bk))
            out = []
            if counters.inner_iterations_executed != exe:
                out.append(f"executed iterations {counters.inner_iterations_executed} != "
                           f"enumerated {exe}")
            return out

        return Case(v, (m, n, k), cfg, (abuf, bbuf, _dev(c), d), flops, nbytes, want, read,
                    _tolerance(name, k), extra, hbm=(v == "diagonal"))
    if v in ("complex", "dual"):
        kind = dtypes.pair_kind(dt)
        if kind != ("complex" if v == "complex" else "dual"):
            raise ConfigError(f"{v} variant expects a {v} dtype")
        m, n, k = args.m, args.n, args.k
        a0, a1 = _draw(rng, (m, k), dt)
        b0, b1 = _draw(rng, (k, n), dt)
        cs = dtypes.storage_scalar(acc)
        c0, c1 = (rng.standard_normal((m, n)).astype(cs) for _ in range(2))
        build = api.build_complex_config if v == "complex" else api.build_dual_config
        cfg = build(m, n, k, dt, block_tile=args.block, operator_shape=args.op,
                    worker_threads=args.threads)
        inter = lambda p0, p1: np.stack([np.asarray(p0).ravel(order="F"),
                                         np.asarray(p1).ravel(order="F")], axis=1).ravel()
        torch = _torch()
        kernel.resolve_config(cfg)  # configuration errors before any device work
        abuf, bbuf = _dev(inter(a0, a1)), _dev(inter(b0, b1))
        cbuf = _dev(inter(c0, c1))
        d = torch.zeros_like(cbuf)
        A0, A1, B0, B1 = (_wide(x) for x in (a0, a1, b0, b1))
        if v == "complex":
            want = (A0 + 1j * A1) @ (B0 + 1j * B1) + (_wide(c0) + 1j * _wide(c1))
            flops = 8.0 * m * n * k
        else:
            want = (A0 @ B0 + _wide(c0)) + 1j * (A0 @ B1 + A1 @ B0 + _wide(c1))
            flops = 6.0 * m * n * k

        def read():
            x = d.cpu().numpy().astype(np.float64)
            return (x[0::2] + 1j * x[1::2]).reshape((m, n), order="F")

        nbytes = 2 * dtypes.storage_scalar(dt).itemsize * (m * k + k * n) + 4 * cs.itemsize * m * n
        return Case(v, (m, n, k), cfg, (abuf, bbuf, cbuf, d), flops, nbytes, want, read,
                    _tolerance(name, k) * 2)
    if v == "tc":
        na, nb, nc, nd = args.na, args.nb, args.nc, args.nd
        a = _draw(rng, (nb, nd, na), dt)
        b = _draw(rng, (nd, nc), dt)
        cfg = api.build_tc_config(na, nb, nc, nd, dt, block_tile=args.block,
                                  operator_shape=args.op, worker_threads=args.threads)
        kernel.resolve_config(cfg)
        torch = _torch()
        d = torch.zeros(na * nb * nc, dtype=dtypes.torch_scalar(acc), device="cuda")
        want = np.einsum("bda,dc->abc", _wide(a), _wide(b))
        read = lambda: d.cpu().numpy().reshape((na, nb, nc), order="F")
        cbuf = torch.empty(0, dtype=dtypes.torch_scalar(acc), device="cuda")
        m, n, k = nb * na, nc, nd
        return Case(v, (m, n, k), cfg, (_dev(a), _dev(b), cbuf, d), 2.0 * m * n * k,
                    dt.itemsize * (m * k + k * n) + acc.itemsize * m * n, want, read,
                    _tolerance(name, k))
    raise ConfigError(f"unknown variant {v!r}")


VARIANTS = ("complex", "dense", "diagonal", "dual", "fused", "tc")


def _counters_row(c):
    return [c.global_loads, c.global_stores, c.operator_invocations,
            c.inner_iterations_executed, c.inner_iterations_skipped]


def _lane_ctx(lane):
    import contextlib

    return kernel.force_lane(lane) if lane not in (None, "auto") else contextlib.nullcontext()


def cmd_check(args) -> int:
    rng = np.random.default_rng(args.seed)
    case = prepare(args, rng)
    with _lane_ctx(args.lane):
        counters = case.run()
    err = case.rel_err()
    m, n, k = case.gemm_shape
    print(f"variant={case.variant} m={m} n={n} k={k} dtype={args.dtype} "
          f"lane={kernel.last_run()['lane']}")
    print(f"max_rel_err = {err:.3e} (tolerance {case.tol:.0e})")
    print("counters: " + " ".join(f"{f.name}={getattr(counters, f.name)}"
                                  for f in dataclasses.fields(counters)))
    failures = case.extra_checks(counters)
    for f in failures:
        print(f"counter check FAILED: {f}")
    if err > case.tol or failures:
        print("FAIL")
        return 1
    print("PASS")
    return 0


def _bench_case(args, case, out):
    torch = _torch()

    with _lane_ctx(args.lane):
        counters = case.run()          # warm-up, excluded
        times = []
        with ClockSampler(torch.cuda.current_device()) as cs:
            for _ in range(args.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                counters = case.run(synchronize=False)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e) * 1e-3)
    err = case.rel_err()
    best = min(times)
    mean = statistics.fmean(times)
    std = statistics.stdev(times) if len(times) > 1 else 0.0
    m, n, k = case.gemm_shape
    peak_tf, peak_gbs = _peaks()
    tflops = case.flops / best / 1e12
    gbs = case.nbytes / best / 1e9
    pct = 100 * (gbs / peak_gbs if case.hbm else tflops / peak_tf)
    row = [case.variant, m, n, k, *case.block, *case.op, args.threads, args.reps,
           f"{mean:.6f}", f"{std:.6f}", f"{case.flops / best / 1e9:.3f}", f"{err:.3e}",
           *_counters_row(counters), f"{tflops:.2f}", f"{gbs:.1f}", f"{pct:.1f}",
           cs.summary().get("sm_mhz"), kernel.last_run()["lane"], kernel.last_run()["launches"]]
    out.write(",".join(str(x) for x in row) + "\n")
    out.flush()


def cmd_bench(args) -> int:
    rng = np.random.default_rng(args.seed)
    out = open(args.out, "w") if args.out else sys.stdout
    try:
        out.write(",".join(CSV_COLUMNS + GPU_COLUMNS) + "\n")
        lanes = list(kernel.available_lanes()) if args.lane == "both" else [args.lane]
        for lane in lanes:
            args.lane = lane
            _bench_case(args, prepare(args, rng), out)
    finally:
        if args.out:
            out.close()
    return 0


def _parse_sweep_file(path):
    axes = {}
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if "=" not in line:
                raise ConfigError(f"sweep line is not key=value: {line!r}")
            key, _, value = line.partition("=")
            key = key.strip()
            if key not in CSV_COLUMNS + ["dtype", "trans"]:
                raise ConfigError(f"unknown sweep key {key!r}; keys are CSV column names")
            axes[key] = [x.strip() for x in value.split(",") if x.strip()]
    return axes


def _apply_sweep_key(ns, key, value):
    if key in ("m", "n", "k", "threads"):
        setattr(ns, key, int(value))
    elif key in ("dtype", "trans"):
        setattr(ns, key, value)
    elif key.startswith("block_"):
        block = list(ns.block or (0, 0, 0))
        block["mnk".index(key[-1])] = int(value)
        ns.block = tuple(block)
    elif key.startswith("op_"):
        op = list(ns.op or (8, 8, 8))
        op["mnk".index(key[-1])] = int(value)
        ns.op = tuple(op)
    else:
        raise ConfigError(f"sweep key {key!r} is not sweepable")


def cmd_sweep(args) -> int:
    axes = _parse_sweep_file(args.config)
    variants = axes.pop("variant", ["dense"])
    reps = int(axes.pop("reps", ["3"])[0])
    keys = sorted(axes)
    out = open(args.out, "w") if args.out else sys.stdout
    try:
        out.write(",".join(CSV_COLUMNS + GPU_COLUMNS) + "\n")
        for variant in variants:
            for values in itertools.product(*(axes[k] for k in keys)):
                ns = argparse.Namespace(m=256, n=256, k=256, na=8, nb=4, nc=16, nd=16,
                                        dtype=args.dtype, trans="nn", wide=False, pad=0,
                                        block=None, op=None, threads=args.threads,
                                        seed=args.seed, lane=args.lane, reps=reps,
                                        variant=variant)
                for key, value in zip(keys, values):
                    _apply_sweep_key(ns, key, value)
                for flag, val in (("block", ns.block), ("op", ns.op)):
                    if val is not None and 0 in val:
                        raise ConfigError(f"sweep must set all three {flag}_* keys together")
                _bench_case(ns, prepare(ns, np.random.default_rng(ns.seed)), out)
    finally:
        if args.out:
            out.close()
    return 0


def _split3(text):
    parts = tuple(int(p) for p in text.split(","))
    if len(parts) != 3:
        raise argparse.ArgumentTypeError("expects three comma-separated integers")
    return parts


def _add_common(p):
    p.add_argument("--variant", required=True, choices=VARIANTS)
    for dim, default in (("m", 256), ("n", 256), ("k", 256), ("na", 8), ("nb", 4), ("nc", 16),
                         ("nd", 16)):
        p.add_argument(f"--{dim}", type=int, default=default)
    p.add_argument("--dtype", default="f16", choices=sorted(DTYPES))
    p.add_argument("--trans", default="nn", choices=["nn", "nt", "tn", "tt"])
    p.add_argument("--wide", action="store_true", help="f64 accumulation (exact lane)")
    p.add_argument("--pad", type=int, default=0)
    p.add_argument("--block", type=_split3, default=None, metavar="BM,BN,BK")
    p.add_argument("--op", type=_split3, default=None, metavar="OM,ON,OK")
    p.add_argument("--threads", type=int, default=int(os.environ.get("TILEKIT_THREADS", "1")),
                   help="accepted for compatibility; the device schedule ignores it")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--lane", default="auto", choices=["auto", "tcgen05", "simt", "both"])


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tk-b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    pc = sub.add_parser("check", help="verify a variant against the float64 product")
    _add_common(pc)
    pc.set_defaults(fn=cmd_check)
    pb = sub.add_parser("bench", help="time a variant on the device, emit CSV")
    _add_common(pb)
    pb.add_argument("--reps", type=int, default=5)
    pb.add_argument("--out", default=None)
    pb.set_defaults(fn=cmd_bench)
    ps = sub.add_parser("sweep", help="run a key=value sweep file")
    ps.add_argument("--config", required=True)
    ps.add_argument("--out", default=None)
    ps.add_argument("--dtype", default="f16", choices=sorted(DTYPES))
    ps.add_argument("--threads", type=int, default=int(os.environ.get("TILEKIT_THREADS", "1")))
    ps.add_argument("--seed", type=int, default=0)
    ps.add_argument("--lane", default="auto", choices=["auto", "tcgen05", "simt"])
    ps.set_defaults(fn=cmd_sweep)
    args = ap.parse_args(argv)
    if args.command == "check" and args.lane == "both":
        ap.error("--lane both is only valid for bench")
    try:
        return args.fn(args)
    except ConfigError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
