"""Block predicates on the tensor cores (reference components.py:171-191; the predicate runs
per (output block, block-K) iteration, kernel.py:399-404).

The host evaluates the predicate into a block mask exactly like the reference's schedule
(kernel._predicate_plan); the device expands it to one bit per K=16 MMA step of every CTA-pair
tile (expand_kbits_kernel) so the producer skips k-blocks that are off and the MMA issuer
skips single steps.  Checked against the oracle's masked GEMM (the same mask over the same
block tiling): bitwise on integer inputs, and -0.0 in C survives tiles whose every iteration
was skipped (acc = g2s_c(C) untouched, as in the reference).
"""

import dataclasses

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from oracle import oracle as O
from paper_2009_12263_b200 import components, kernel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).ravel(order="F"))).cuda()


class HashPredicate:
    """An arbitrary (non-structural) predicate: iteration on iff a hash of its block and
    block-K coordinates is not 0 mod 3; blocks whose row index is 1 are switched off entirely."""

    def __call__(self, tile):
        pos = tile.absolute
        if pos["M"] // 256 == 1:
            return False
        return (pos["M"] * 7 + pos["N"] * 13 + pos["K"] * 5) // 16 % 3 != 0


@pytest.mark.parametrize("block", [(256, 256, 64), (512, 128, 16), (256, 512, 32), (256, 64, 48)])
@pytest.mark.parametrize("integer", [True, False])
def test_mask_predicate_tcgen05(cuda, block, integer):
    m, n, k = 1024, 1024, 768
    rng = np.random.default_rng(41)
    if integer:
        a = rng.integers(-4, 5, (m, k)).astype(np.float16)
        b = rng.integers(-4, 5, (k, n)).astype(np.float16)
        c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    else:
        a = rng.standard_normal((m, k)).astype(np.float16)
        b = rng.standard_normal((k, n)).astype(np.float16)
        c = rng.standard_normal((m, n)).astype(np.float32)
    c[0, :] = -0.0  # rows of block-row 0 ...
    c[300, :] = -0.0  # ... and of block-row 1 (every iteration off): -0 must survive
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16, block_tile=block),
                              predicate=HashPredicate())
    res = kernel.resolve_config(cfg)
    plan, mask, executed = kernel.lower(res)
    assert mask is not None and kernel.plan_lane(plan) == "tcgen05"
    d = torch.full((m * n,), float("nan"), device=cuda)
    cnt = tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    run = tk.last_run()
    assert run["lane"] == "tcgen05" and run["plan"]["kernel"] == "pair", run["plan"]
    assert cnt.inner_iterations_skipped == int((~executed).sum())
    want = O.gemm_real(a.astype(np.float32), b.astype(np.float32), c, kmask=mask, block=block)
    got = d.cpu().numpy().reshape((m, n), order="F")
    if integer:
        assert np.array_equal(got, want)
        assert np.array_equal(np.signbit(got[300]), np.signbit(want[300]))
    else:
        assert O.rel_err(got, want) <= O.tolerance(k)


@pytest.mark.parametrize("trans", ["nn", "tt"])
def test_diagonal_predicate_dense_a_tcgen05(cuda, trans):
    """DiagonalPredicate over a dense (stored) A: block-K iterations off the diagonal skipped on
    the tensor cores, bitwise the oracle on integer inputs."""
    m = n = k = 1024
    ta, tb = trans[0] == "t", trans[1] == "t"
    rng = np.random.default_rng(42)
    a = rng.integers(-4, 5, (m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    block = (256, 256, 64)
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16, trans_a=ta, trans_b=tb,
                                                    block_tile=block),
                              predicate=components.DiagonalPredicate())
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, _dev(a.T if ta else a), _dev(b.T if tb else b), _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    _, mask, executed = kernel.lower(kernel.resolve_config(cfg))
    run = executed.transpose(1, 0, 2).reshape(-1, executed.shape[2]).astype(np.uint8)
    want = O.gemm_real(a.astype(np.float32), b.astype(np.float32), c, kmask=run, block=block)
    assert np.array_equal(d.cpu().numpy().reshape((m, n), order="F"), want)


def test_predicate_bk8_runs_on_exact_lane(cuda):
    """bk = 8 (the reference's default operator K) splits a K=16 MMA step between two block-K
    chunks: such predicates stay on the bit-exact CUDA-core lane."""
    m = n = k = 512
    rng = np.random.default_rng(43)
    a = rng.integers(-4, 5, (m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16, block_tile=(256, 256, 8)),
                              predicate=HashPredicate())
    d = torch.zeros(m * n, device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    assert tk.last_run()["lane"] == "simt"
    _, mask, _ = kernel.lower(kernel.resolve_config(cfg))
    want = O.gemm_real(a.astype(np.float32), b.astype(np.float32), c, kmask=mask, block=(256, 256, 8))
    assert np.array_equal(d.cpu().numpy().reshape((m, n), order="F"), want)
