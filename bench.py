"""Benchmark: FP16 -> FP32 GEMM TFLOPS on B200 (BASELINE.json metric), one JSON line.

Workload (BASELINE.json configs[1]): D = A*B + C, column-major, fp16 A/B, fp32 C/D,
reference `build_dense_config` semantics.

* N = 1 GPU: the north-star point, M = N = K = 8192.
* N > 1 GPUs (BASELINE configs[1]'s "N=16384 column-sharded at 2/4/8 GPUs", the default):
  one process per GPU, the fixed 16384^3 problem split into G column slabs of B/C/D with A
  replicated -- no data-path collective, `scaling` "strong".  `--weak` instead gives every
  rank its own n-column slab of an M x (n*G) x K problem.  The NCCL all-gather of the D
  slabs (the north star's optional collective) is timed separately, never in `value`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n N] [--dtype fp16|bf16] [--weak]
  python bench.py --impl reference ...   # the reference's own CPU implementation
  python bench.py --gpus 2 --dry-run     # launcher/rank plumbing only (gloo, no GPU work)

`--gpus N` without a torchrun environment re-launches this script under
`torch.distributed.run` with N ranks (127.0.0.1 rendezvous); the line's `n_gpus` must equal
`--gpus` or the run fails.

Timing: W untimed steps, then K steps bracketed by barrier + cuda synchronize, CUDA events
on the launching stream, max over ranks.  Inputs (768 MiB at n=8192) exceed the 126 MB L2.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GEMM TFLOPS (FP16/BF16 in, FP32 acc) vs N; % of B200 dense tensor-core peak"
UNIT = "TFLOPS"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0) or 0), \
            float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


from paper_2009_12263_b200.clocks import ClockSampler  # noqa: E402


# ---- reference CPU implementation -------------------------------------------------------

def _reference_module():
    """The reference package (oracle/_ref, built from /root/reference by oracle/Makefile)."""
    path = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(path, "tilekit")):
        sys.path.insert(0, path)
        import tilekit

        return tilekit, "reference"
    return None, "port"


_CPU_INPUTS = {}


def _cpu_inputs(m, k, s):
    """fp16-valued float32 inputs for the CPU slab (generated once per process)."""
    key = (m, k, s)
    if key not in _CPU_INPUTS:
        rng = np.random.default_rng(0)
        a = np.asfortranarray(rng.standard_normal((m, k), dtype=np.float32)
                              .astype(np.float16).astype(np.float32))
        b = np.asfortranarray(rng.standard_normal((k, s), dtype=np.float32)
                              .astype(np.float16).astype(np.float32))
        c = np.asfortranarray(rng.standard_normal((m, s), dtype=np.float32))
        _CPU_INPUTS[key] = (a, b, c)
    return _CPU_INPUTS[key]


def cpu_sample(m, k, threads):
    """Time the reference CPU path on an m x s x k column slab of the workload.

    The reference (oracle/_ref: tilekit with its compiled Cython lane) runs its own
    ``matmul(build_dense_config(...))`` on fp16-valued float32 inputs (it has no fp16 type;
    SURVEY 8c protocol).  The slab width s bounds the run to a few seconds on the host cores.
    """
    tilekit, kind = _reference_module()
    s = 1024 * max(1, min(8, -(-threads // 8)))  # one 1024-column block per 8 host threads
    if m > 8192:  # keep a step's CPU work at the 8192^3 sample's size (a few seconds)
        s = max(256, s * 8192 * 8192 // (m * k))
    a, b, c = _cpu_inputs(m, k, s)
    flops = 2.0 * m * s * k
    if tilekit is not None:
        cfg = tilekit.build_dense_config(m, s, k, np.float32, worker_threads=threads)
        d = np.zeros(m * s, np.float32)
        fa, fb, fc = a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F")
        run = lambda: tilekit.matmul(cfg, fa, fb, fc, d)
        lane = tilekit.active_lane()
        cfgr = tilekit.kernel.resolve_config(cfg)
        blocks = (m // cfgr.params.block_tile[0]) * (s // cfgr.params.block_tile[1])
        used = tilekit.kernel._effective_workers(threads, blocks)
    else:
        from oracle import oracle as O

        run = lambda: O.gemm_real(a, b, c, threads=threads)
        lane, used = "oracle-port", threads
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    return {"value": flops / dt / 1e12, "unit": UNIT, "cores": int(used), "kind": kind,
            "seconds": dt,
            "sample": f"{m}x{s}x{k} column slab of the {m}x{m}x{k} workload, fp16-valued f32, "
                      f"{'tilekit.matmul(build_dense_config)' if tilekit else 'oracle C port'} "
                      f"lane={lane}, {used} of {threads} host threads"}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    n = args.n
    for _ in range(args.warmup):
        cpu_sample(n, n, threads)
    samples = [cpu_sample(n, n, threads) for _ in range(args.steps)]
    value = float(np.median([s["value"] for s in samples]))
    ms = float(np.median([s["seconds"] for s in samples])) * 1e3
    s0 = samples[0]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f32 (fp16-valued inputs)", "data": "synthetic",
            "config": {"workload": f"dense GEMM D=A*B+C, M=N=K={n} column-major "
                                   "(bounded column-slab sample per step)", "n": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": s0["cores"],
                             "kind": s0["kind"], "sample": s0["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- our implementation -------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2009_12263_b200 as tk
    from paper_2009_12263_b200 import api

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m = k = args.n
    # per-rank column slab: N/G columns of the fixed N x N x N problem (strong: the default at
    # N > 1 GPUs, SURVEY 8e's "N=16384 over 2/4/8 GPUs") or n columns each (--weak)
    n = args.n // world if args.strong else args.n
    if n * (world if args.strong else 1) != args.n or n % 8:
        raise SystemExit(f"strong scaling needs N divisible by 8 x world size (N={args.n}, G={world})")
    dt = tk.FLOAT16 if args.dtype == "fp16" else tk.BFLOAT16
    tdt = torch.float16 if args.dtype == "fp16" else torch.bfloat16
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    a = torch.randn(m * k, generator=g, device=dev).to(tdt)          # replicated A (same seed
    if world > 1:                                                     # on every rank)
        dist.broadcast(a, 0)
    b = torch.randn(k * n, generator=g, device=dev).to(tdt)          # this rank's slab of B
    c = torch.randn(m * n, generator=g, device=dev)
    d = torch.empty(m * n, device=dev)
    cfg = tk.kernel.resolve_config(tk.build_dense_config(m, n, k, dt))
    stream = torch.cuda.current_stream(dev)

    def step():
        tk.gemm_execute(cfg, a, b, c, d, stream=stream, synchronize=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 1)):
        step()
    launches_per_step = tk.last_run()["launches"]
    barrier()
    sampler = ClockSampler(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ms = start.elapsed_time(end) / args.steps
    # SM clock the kernel actually ran at (clock64 vs globaltimer in CTA 0 of the last timed
    # launch): NVML reports the boost clock while the tensor-core step is power/current-limited
    kernel_mhz = None
    try:
        import ctypes

        f = tk._lib.load().tk_debug_pair_mhz
        f.restype = ctypes.c_double
        kernel_mhz = round(f(), 1) or None
    except Exception:
        pass
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops_rank = 2.0 * m * n * k
    value = flops_rank * world / (ms * 1e-3) / 1e12

    # roofline of the dominant (only) kernel: one tcgen05 launch per step
    burst, sustained_peak, hbm, src = _peaks()
    kernel_ms = ms / launches_per_step
    achieved = flops_rank / (kernel_ms * 1e-3) / 1e12
    traffic = args.traffic
    if traffic is None:  # dram bytes per launch from the committed ncu --set full capture
        try:
            with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
                traffic = json.load(f).get(f"{args.dtype}_{m}")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                "frac": achieved / burst, "traffic": traffic,
                "traffic_unit": "bytes/launch (dram read+write, ncu --set full)",
                "algorithmic_flops_per_launch": flops_rank,
                "algorithmic_bytes_per_launch": 2 * (m * k + k * n) + 8 * m * n,
                "peak_source": ("measured bf16 burst (MEASURED_PEAKS.json)" if src == "measured" else
                                "fallback 1590 TF/s bf16 burst (B200_PROFILING.md; MEASURED_PEAKS.json absent)"),
                "frac_of_sustained": achieved / sustained_peak if sustained_peak else None,
                "frac_of_spec_2250": achieved / 2250.0}

    # optional collective, timed separately (north star: "an optional NCCL all-gather of C over
    # NVLink is timed separately"): every rank's D slab gathered into the full M x (n*G) D
    allgather = None
    if world > 1:
        try:
            full = torch.empty(m * n * world, device=dev)
            for _ in range(2):
                dist.all_gather_into_tensor(full, d)
            barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, min(args.steps, 10))
            g0.record(stream)
            for _ in range(reps):
                dist.all_gather_into_tensor(full, d)
            g1.record(stream)
            torch.cuda.synchronize(dev)
            gms = torch.tensor([g0.elapsed_time(g1) / reps], device=dev)
            dist.all_reduce(gms, op=dist.ReduceOp.MAX)
            gms = float(gms.item())
            recv = (world - 1) * m * n * 4  # bytes each rank receives
            allgather = {"ms": gms, "bytes_received_per_rank": recv,
                         "GB_per_s_per_rank": recv / (gms * 1e-3) / 1e9,
                         "collective": "torch.distributed.all_gather_into_tensor (NCCL)",
                         "in_value": False}
            if args.fused_allgather:
                allgather["fused"] = fused_allgather(args, tk, torch, dist, dev, stream, a, b, c,
                                                     m, n, k, world, rank, d)
            del full
        except Exception as exc:
            allgather = {"unavailable": str(exc)[:160]}

    # sustained window (not `value`): the same step back to back for ~--sustain-s seconds with
    # NVML sampling throughout, so clocks / power are observed under a long load and the
    # sustained rate can be set beside MEASURED_PEAKS' bf16_tflops_sustained
    sustained = None
    if args.sustain_s > 0:
        reps = max(1, int(args.sustain_s * 1e3 / ms))
        long_sampler = ClockSampler(local)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with long_sampler:
            s0.record(stream)
            for _ in range(reps):
                step()
            s1.record(stream)
            torch.cuda.synchronize(dev)
        barrier()
        sms = torch.tensor([s0.elapsed_time(s1) / reps], device=dev)
        if world > 1:
            dist.all_reduce(sms, op=dist.ReduceOp.MAX)
        sms = float(sms.item())
        sus_tf = flops_rank * world / (sms * 1e-3) / 1e12
        sustained = {"steps": reps, "seconds": sms * reps * 1e-3, "ms_per_step": sms,
                     "value": sus_tf, "unit": UNIT,
                     "per_gpu_vs_bf16_sustained_peak": (sus_tf / world) / sustained_peak
                     if sustained_peak else None,
                     "clocks": long_sampler.summary()}

    # e2e through the C ABI with host (pinned) buffers: H2D of A, B, C and D2H of C each step
    e2e = run_e2e(args, tk, api, torch, dev, m, n, k, world)

    # context only (not the product, not in `value`): cuBLASLt on the same operation
    # (fp16/bf16 A,B; fp32 C,D; D = A*B + C) timed the same way on this GPU
    library = None
    if rank == 0 and world == 1 and not args.no_library:
        try:
            # column-major D = A B + C is row-major D^T = B^T A^T + C^T: all operands contiguous
            At, Bt, Ct = a.view(k, m), b.view(n, k), c.view(n, m)
            f = lambda: torch.addmm(Ct, Bt, At, out_dtype=torch.float32)
            for _ in range(3):
                f()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                f()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            lms = e0.elapsed_time(e1) / args.steps
            library = {"cublas_same_op_tflops": flops_rank / (lms * 1e-3) / 1e12,
                       "call": "torch.addmm(C_fp32, A_half, B_half, out_dtype=float32)"}
        except Exception as exc:  # older torch without out_dtype
            library = {"unavailable": str(exc)[:120]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(m, k, len(os.sched_getaffinity(0)))
        cpu.pop("seconds", None)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic",
                "config": {"workload": f"dense GEMM D=A*B+C, fp16/bf16 A,B -> fp32 C,D, "
                                       f"column-major, M=K={m}, N={n} per GPU (column slab; "
                                       f"A replicated)",
                           "m": m, "n_per_gpu": n, "k": k, "accumulate": "fp32",
                           "parallelism": f"column-slab x{world}",
                           "l2": "inputs (A+B+C+D) exceed the 126 MB L2; no flush",
                           "lane": tk.last_run()["lane"]},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                # sm_mhz_in_kernel (clock64 / globaltimer inside the GEMM) is the clock the
                # kernel ran at; NVML's sm_mhz over a short timed region can miss the load
                "clocks": {"sm_mhz_in_kernel": kernel_mhz, **sampler.summary(),
                           "note": "sm_mhz_in_kernel = clock64 / %globaltimer inside the GEMM (the effective "
                                   "clock); NVML's sm_mhz / power_w over a short region report the requested "
                                   "clock and a lagging power average ('sustained' holds a seconds-long run)"},
                "sustained": sustained,
                "library_baseline": library,
                "allgather_d": allgather,
                "gpu_launches": launches_per_step * args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def fused_allgather(args, tk, torch, dist, dev, stream, a, b, c, m, n, k, world, rank, d):
    """Opt-in (--fused-allgather): the GEMM whose epilogue TMA-stores every D tile into all
    ranks' full-D buffers over peer memory (CUDA IPC mappings; NVLink on an NVSwitch box),
    timed per step as GEMM + gather, checked against the NCCL-gathered D."""
    from paper_2009_12263_b200 import shard

    try:
        full = torch.empty(m * n * world, device=dev)
        peers = shard.PeerBuffers(full)
        big_b = torch.empty(k * n * world, device=dev, dtype=a.dtype)  # this rank's slab = the
        big_c = torch.empty(m * n * world, device=dev)                  # bench step's B and C
        big_b.view(world, -1)[rank].copy_(b)
        big_c.view(world, -1)[rank].copy_(c)
        cfg = tk.kernel.resolve_config(tk.build_dense_config(m, n * world, k,
                                                             tk.FLOAT16 if args.dtype == "fp16" else tk.BFLOAT16))
        step = lambda: shard.sharded_gemm(cfg, a, big_b, big_c, None, rank=rank, world=world,
                                          allgather_into=full, fused=True, peers=peers,
                                          stream=stream, synchronize=False)
        for _ in range(2):
            step()
        reps = max(3, min(args.steps, 10))
        dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(reps):
            step()  # includes the device sync + barrier that publish the gathered D
        ms = (time.perf_counter() - t0) * 1e3 / reps
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = bool(torch.equal(full.view(world, -1)[rank], d))  # this rank's slab, as computed
        mode = tk.last_run().get("peer_mode")
        peers.close()
        return {"ms_per_step_gemm_plus_gather": float(t.item()), "peer_mode": mode,
                "own_slab_matches_bench_step": ok,
                "how": "tk_gemm_peers: epilogue TMA stores to local + peer slabs (wall clock "
                       "incl. device sync + barrier per step)"}
    except Exception as exc:
        return {"unavailable": str(exc)[:200]}


def run_e2e(args, tk, api, torch, dev, m, n, k, world):
    """Same metric through tk_gemm_ex_raw (the reference-facing C ABI) on host buffers."""
    tag = api.TAG_F16F32 if args.dtype == "fp16" else api.TAG_BF16F32
    hd = torch.float16 if args.dtype == "fp16" else torch.bfloat16
    ha = torch.randn(m * k).to(hd).pin_memory()
    hb = torch.randn(k * n).to(hd).pin_memory()
    hc = torch.randn(m * n).pin_memory()
    h2d = (ha.numel() + hb.numel()) * 2 + hc.numel() * 4
    d2h = hc.numel() * 4

    def call():
        rc = api.gemm_ex_raw(tag, 0, 0, m, n, k, 1.0, 0.0, ha.data_ptr(), hb.data_ptr(), 1.0,
                             0.0, hc.data_ptr())
        if rc != 0:
            raise RuntimeError(f"tk_gemm_ex_raw returned {rc}: {tk._lib.last_error()}")

    reps = max(1, min(args.steps, args.e2e_steps))
    call()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    torch.cuda.synchronize(dev)
    sec = (time.perf_counter() - t0) / reps
    t = torch.tensor([sec], device=dev)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item())
    return {"value": 2.0 * m * n * k * world / sec / 1e12, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": sec * 1e3, "steps": reps,
            "path": "tk_gemm_ex_raw(TAG_F16F32) on pinned host buffers (C updated in place)"}


def run_dry(args):
    """--dry-run: the launcher and rank plumbing without GPU work (gloo process group; the
    CPU test of `--gpus N`).  Prints the line rank 0 would print, minus the measurements."""
    import torch
    import torch.distributed as dist

    world, rank, _ = _dist()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(rank)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        seen = int(t.item()) + 1
        dist.destroy_process_group()
    else:
        seen = 1
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "ranks_seen": seen, "dry_run": True,
                          "scaling": "strong" if args.strong else "weak",
                          "config": {"n": args.n, "n_per_gpu": args.n // world if args.strong else args.n}}),
              flush=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _self_launch(args):
    """`--gpus N` outside torchrun: re-run this script as N ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=None,
                    help="problem size (default 8192 on 1 GPU, 16384 strong-sharded on N > 1)")
    ap.add_argument("--dtype", choices=["fp16", "bf16"], default="fp16")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sustain-s", type=float, default=3.0,
                    help="seconds of back-to-back steps for the sustained clocks/TFLOPS figure")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the N x N x N problem split into G column slabs "
                         "(the default when N > 1 GPUs)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank owns an n-column slab (n = --n, default 8192)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rank plumbing only: gloo process group, no GPU work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-library", action="store_true", help="skip the cuBLAS same-op context line")
    ap.add_argument("--fused-allgather", action="store_true",
                    help="N>1: also time the GEMM with the all-gather fused into its epilogue")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    world = _dist()[0]
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but {world} rank(s) launched (WORLD_SIZE)")
    if args.strong and args.weak:
        raise SystemExit("--strong and --weak are exclusive")
    args.strong = args.strong or (world > 1 and not args.weak)
    if args.n is None:
        args.n = 16384 if args.strong and world > 1 else 8192
    if world > 1:  # let the driver see NCCL's own report of the ranks / transports
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
