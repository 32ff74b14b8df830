"""Multi-GPU column-slab sharding (one process per GPU).

The output blocks of the reference schedule are independent (reference
``kernel.py:320-340`` deals them to worker threads with no reduction).  Across GPUs the
B200 path shards the same way along N: rank ``g`` of ``G`` owns columns
``[g*N/G, (g+1)*N/G)`` -- a column slab of B, C, D and the bias -- and A is replicated.
With column-major B/C/D every slab is a contiguous sub-buffer, so sharding is pointer
arithmetic: no repacking and no collective on the data path.  An optional all-gather of
the D slabs (NCCL over NVLink; gloo in the CPU tests) reassembles the full column-major D
because the slabs are contiguous column blocks in rank order.
"""

from __future__ import annotations

import dataclasses

from . import kernel, layouts
from .components import BiasEpilogue, ConfigError


def column_slab(n: int, world: int, rank: int) -> tuple:
    """[start, stop) columns of rank ``rank`` (equal slabs; ``world`` must divide ``n``)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world of {world}")
    if n % world:
        raise ConfigError(f"N={n} is not divisible by the {world} ranks; zero-pad the problem")
    w = n // world
    return rank * w, (rank + 1) * w


def _slab_layout(layout, j0, j1, label):
    if isinstance(layout, layouts.Zero):
        return dataclasses.replace(layout, extents=(layout.extents[0], j1 - j0)), 0
    if type(layout) is layouts.ColMajor or (isinstance(layout, layouts.InterleavedComplex)
                                            and layout.order == "F"):
        rows = layout.extents[0]
        per_elem = 2 if isinstance(layout, layouts.InterleavedComplex) else 1
        return dataclasses.replace(layout, extents=(rows, j1 - j0)), j0 * rows * per_elem
    raise ConfigError(f"{label}: column-slab sharding needs a column-major layout, got "
                      f"{type(layout).__name__}")


def shard_config(config, rank: int, world: int):
    """(slab KernelConfig, scalar offsets {'B','C','D'}, (j0, j1)) for one rank."""
    config = kernel.resolve_config(config)
    m, n, k = config.params.gemm_shape
    j0, j1 = column_slab(n, world, rank)
    gb, ob = _slab_layout(config.global_b_layout, j0, j1, "B")
    gc, oc = _slab_layout(config.global_c_layout, j0, j1, "C")
    gd, od = _slab_layout(config.global_d_layout, j0, j1, "D")
    p = config.params
    block = p.block_tile if (j1 - j0) % p.block_tile[1] == 0 else None
    params = dataclasses.replace(p, gemm_shape=(m, j1 - j0, k), block_tile=block,
                                 compute_warp=p.compute_warp if block else None)
    ep = config.epilogue
    if isinstance(ep, BiasEpilogue) and ep.axis == "n":
        ep = BiasEpilogue(ep.bias[j0:j1], "n")
    slab = dataclasses.replace(config, params=params, global_b_layout=gb, global_c_layout=gc,
                               global_d_layout=gd, epilogue=ep)
    return kernel.resolve_config(slab), {"B": ob, "C": oc, "D": od}, (j0, j1)


def _view(buf, offset, size):
    return buf[offset:offset + size]


class PeerBuffers:
    """Every rank's full-D buffer mapped into this process (CUDA IPC over the process group),
    for the fused all-gather: the GEMM epilogue stores each D tile locally and into the peers'
    buffers (NVLink peer writes on an NVSwitch box).  ``full`` is this rank's flat full-D
    CUDA tensor (same size on every rank); ``close()`` unmaps the peers."""

    def __init__(self, full, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib

        self.lib = _lib.load()
        self.full = full
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        h = (ctypes.c_char * 64)()
        off = ctypes.c_int64()
        if self.lib.tk_ipc_handle(ctypes.c_void_p(full.data_ptr()), h, ctypes.byref(off)) != 0:
            raise RuntimeError(_lib.last_error())
        handles = [None] * self.world
        dist.all_gather_object(handles, (bytes(h), off.value), group=group)
        self.bases, self.mapped = [], []
        for r, (hb, offset) in enumerate(handles):
            if r == self.rank:
                self.bases.append(full.data_ptr())
                self.mapped.append(None)
                continue
            ptr = ctypes.c_void_p()
            if self.lib.tk_ipc_open(ctypes.create_string_buffer(hb, 64), ctypes.byref(ptr)) != 0:
                self.close()
                raise RuntimeError(_lib.last_error())
            self.mapped.append(ptr.value)
            self.bases.append(ptr.value + offset)  # the peer's tensor inside its allocation

    def peer_slabs(self, byte_offset):
        """Addresses of this rank's slab position inside every other rank's full D."""
        return [base + byte_offset for r, base in enumerate(self.bases) if r != self.rank]

    def close(self):
        for ptr in getattr(self, "mapped", []):
            if ptr:
                self.lib.tk_ipc_close(ptr)
        self.bases, self.mapped = [], []


def sharded_gemm(config, a, b, c, d, *, rank: int, world: int, group=None,
                 allgather_into=None, fused: bool = False, peers: "PeerBuffers" = None,
                 **run_kwargs):
    """Run this rank's column slab of ``config`` on full-problem buffers (A replicated).

    ``b``, ``c``, ``d`` are the full flat buffers (views of the rank's slab are taken);
    ``allgather_into`` (optional, flat full-D tensor) receives every rank's slab through
    ``torch.distributed.all_gather_into_tensor`` on ``group``.  With ``fused=True`` and
    ``peers`` (a ``PeerBuffers`` over each rank's ``allgather_into``) the slab is instead
    written by the GEMM itself into the local and every peer's full D (peer-memory stores from
    the epilogue, overlapping the remaining tiles).

    Ordering of the fused path (both sides are needed because peers write into memory this
    rank reads):

    * write side -- before the GEMM, every rank drains its device (so all work already queued
      that reads its ``allgather_into``, e.g. from the previous call, has finished) and the
      ranks meet at a barrier; only then may any rank's epilogue store into a peer's buffer;
    * read side -- after the GEMM, a device sync and a second barrier publish the gathered D:
      every rank's slab has landed in every buffer when ``sharded_gemm`` returns.

    Returns the slab counters.
    """
    slab, off, _ = shard_config(config, rank, world)
    sb = slab.global_b_layout.physical_size()
    sc = slab.global_c_layout.physical_size()
    sd = slab.global_d_layout.physical_size()
    if fused:
        if peers is None or allgather_into is None:
            raise ConfigError("fused all-gather needs allgather_into and its PeerBuffers")
        import torch
        import torch.distributed as dist

        dst = _view(allgather_into, off["D"], sd)
        torch.cuda.synchronize(dst.device)  # write side: no reader of the buffers is in flight
        dist.barrier(group=group)
        counters = kernel.gemm_execute(slab, a, _view(b, off["B"], sb), _view(c, off["C"], sc),
                                       dst, peers=peers.peer_slabs(off["D"] * dst.element_size()),
                                       **run_kwargs)
        torch.cuda.synchronize(dst.device)
        dist.barrier(group=group)
        if d is not None and d.data_ptr() != allgather_into.data_ptr():
            _view(d, off["D"], sd).copy_(dst)
        return counters
    counters = kernel.gemm_execute(slab, a, _view(b, off["B"], sb), _view(c, off["C"], sc),
                                   _view(d, off["D"], sd), **run_kwargs)
    if allgather_into is not None:
        import torch.distributed as dist

        dist.all_gather_into_tensor(allgather_into, _view(d, off["D"], sd).contiguous(),
                                    group=group)
    return counters
