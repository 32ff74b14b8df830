"""Column-slab sharding across ranks.

CPU: world_size-2 gloo processes each compute their slab (the oracle stands in for the
device GEMM) and all-gather D; the result must be bit-identical to the unsharded oracle.
GPU: every slab computed by the device equals the same columns of the single-GPU run.
"""

import os
import socket

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from paper_2009_12263_b200 import shard
from paper_2009_12263_b200.components import ConfigError


def _problem(m=64, n=96, k=32, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    bias = rng.standard_normal(n).astype(np.float32)
    return a, b, c, bias


def test_slab_geometry_and_bias():
    m, n, k = 64, 96, 32
    a, b, c, bias = _problem(m, n, k)
    cfg = tk.build_fused_config(m, n, k, np.float32, bias=bias, block_tile=(16, 16, 8))
    slab, off, (j0, j1) = shard.shard_config(cfg, 1, 3)
    assert (j0, j1) == (32, 64)
    assert slab.params.gemm_shape == (m, 32, k) and slab.params.block_tile == (16, 16, 8)
    assert off == {"B": 32 * k, "C": 32 * m, "D": 32 * m}
    assert np.array_equal(slab.epilogue.bias, bias[32:64])
    with pytest.raises(ConfigError, match="divisible"):
        shard.column_slab(96, 5, 0)
    with pytest.raises(ConfigError, match="column-major"):
        shard.shard_config(tk.build_dense_config(m, n, k, np.float32, trans_b=True), 0, 2)


def _worker(rank, world, port, result):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    m, n, k = 64, 96, 32
    a, b, c, bias = _problem(m, n, k)
    cfg = tk.build_fused_config(m, n, k, np.float32, bias=bias, relu_on_c=True,
                                block_tile=(16, 16, 8))
    slab, off, (j0, j1) = shard.shard_config(cfg, rank, world)
    fb, fc = b.ravel(order="F"), c.ravel(order="F")
    sb = fb[off["B"]:off["B"] + slab.global_b_layout.physical_size()].reshape(
        (k, j1 - j0), order="F")
    sc = fc[off["C"]:off["C"] + slab.global_c_layout.physical_size()].reshape(
        (m, j1 - j0), order="F")
    # the oracle stands in for the device GEMM on CPU
    d_slab = O.fused_reference(a, sb, sc, slab.epilogue.bias, relu_on_c=True, relu_on_d=True,
                               threads=1)
    full = torch.empty(m * n, dtype=torch.float32)
    dist.all_gather_into_tensor(full, torch.from_numpy(d_slab.ravel(order="F").copy()))
    if rank == 0:
        want = O.fused_reference(a, b, c, bias, relu_on_c=True, relu_on_d=True, threads=1)
        result.put(bool(np.array_equal(full.numpy().reshape((m, n), order="F"), want)))
    dist.destroy_process_group()


def test_gloo_world2_allgather_equals_unsharded():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.gpu
def test_device_slabs_match_single_gpu_columns(knob):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    knob("TK_TC_KERNEL", "pair")
    knob("TK_SERPENTINE", "0")  # same k order in every tile of every slab
    m, n, k = 1024, 2048, 512
    rng = np.random.default_rng(3)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(np.asarray(x).ravel(order="F"))).cuda()
    a = dev(rng.standard_normal((m, k)).astype(np.float16))
    b = dev(rng.standard_normal((k, n)).astype(np.float16))
    c = dev(rng.standard_normal((m, n)).astype(np.float32))
    cfg = tk.build_dense_config(m, n, k, np.float16)
    full = torch.zeros(m * n, device="cuda")
    tk.matmul(cfg, a, b, c, full)
    world = 4
    d = torch.zeros(m * n, device="cuda")
    total = 0
    for r in range(world):
        total += shard.sharded_gemm(cfg, a, b, c, d, rank=r, world=world).global_stores
    assert torch.equal(d, full)
    assert total == m * n


def _fused_worker(rank, world, port, result, shape):
    """One rank of a fused GEMM + all-gather: both processes share cuda:0 (the only GPU of the
    test box), peer buffers are mapped with CUDA IPC exactly as across NVLink peers."""
    import torch
    import torch.distributed as dist

    os.environ["TK_SERPENTINE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        m, n, k = shape
        rng = np.random.default_rng(11)
        a = rng.integers(-4, 5, (m, k)).astype(np.float16)
        b = rng.integers(-4, 5, (k, n)).astype(np.float16)
        c = rng.integers(-4, 5, (m, n)).astype(np.float32)
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(np.asarray(x).ravel(order="F"))).cuda()
        A, B, C = dev(a), dev(b), dev(c)
        cfg = tk.build_dense_config(m, n, k, np.float16)
        # the gathered D sits 4 KB into its allocation: IPC maps allocations, not tensors
        store = torch.full((m * n + 1024,), float("nan"), device="cuda")
        full = store[1024:]
        peers = shard.PeerBuffers(full)
        try:
            shard.sharded_gemm(cfg, A, B, C, None, rank=rank, world=world, allgather_into=full,
                               fused=True, peers=peers)
            mode = tk.last_run().get("peer_mode")
            want = torch.zeros(m * n, device="cuda")
            tk.matmul(cfg, A, B, C, want)
            ok = bool(torch.equal(full, want))
            if not ok:
                bad = (full != want).view(n, m)
                cols = torch.nonzero(bad.any(dim=1)).flatten()
                ok = (f"mismatch: nan={int(torch.isnan(full).sum())} cols {int(cols.min())}..{int(cols.max())} "
                      f"n={len(cols)} maxdiff={float((full - want).abs().nan_to_num(0).max())}")
            result.put((rank, mode, ok))
            dist.barrier()
        finally:
            peers.close()
    except Exception as exc:  # report instead of hanging the parent
        result.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("shape,mode", [((1024, 2048, 1024), 1),   # streamed epilogue: peer TMA stores
                                        ((512, 1024, 256), 2)])     # K <= 256: copies after the GEMM
def test_fused_allgather_two_ranks_one_gpu(shape, mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, q, shape)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(60)
    for rank, got_mode, ok in res:
        if isinstance(ok, str) and "cudaIpc" in ok:
            pytest.skip(f"CUDA IPC unavailable in this sandbox: {ok}")
        assert ok is True, (rank, ok)
        assert got_mode == mode, (rank, got_mode)


def test_bench_self_launch_dry_run():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself with two ranks
    (gloo dry run: rank plumbing only) and reports n_gpus == 2 seen by both ranks."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=240, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2 and line["dry_run"], line
