"""Load transforms on the A / B streams (g2s_a, g2s_b; reference kernel.py:406-418,
components.py:52-94) on the tensor cores.

The reference evaluates t(x) per element in FP32 and multiplies the transformed values.  The
B200 path evaluates the same t(x) in FP32 in one pass over the operand and hands the tensor
cores t(x) = hi + lo as two fp16 planes (3 MMAs per K step: hi*hi, hi*lo, lo*hi); exact
programs (relu, scale by +-1) need only hi.  These tests pin it against the oracle (the C
restatement of the reference) on inputs built to break an algebraic fold of the transform into
the epilogue: A close to -add_a and B close to -add_b, so (A + add_a)(B + add_b) is tiny next to
its expanded terms.
"""

import dataclasses

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from oracle import oracle as O
from paper_2009_12263_b200 import components as C

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).ravel(order="F"))).cuda()


def _host(t, shape):
    return t.cpu().numpy().reshape(shape, order="F")


def _f32(x):
    return np.asarray(x, dtype=np.float32)


@pytest.mark.parametrize("mnk,kernel", [((512, 384, 256), "single"), ((2048, 2048, 1024), "pair_ops"),
                                        ((256, 256, 8192), "single")])
def test_fused_adversarial_cancellation(cuda, mnk, kernel):
    """build_fused_config(add_a=0.1, add_b=-0.3) with A ~ -0.1, B ~ 0.3 (not on any grid): the
    transformed operands are ~1e-2 while A*B, add_a*B, ... are ~1e-1, so any expanded form
    cancels catastrophically.  C = 0 and bias = 0 keep the product term the whole result."""
    m, n, k = mnk
    rng = np.random.default_rng(31)
    a = (-0.1 + 2.0 ** -6 * rng.standard_normal((m, k))).astype(np.float16)
    b = (0.3 + 2.0 ** -6 * rng.standard_normal((k, n))).astype(np.float16)
    c = np.zeros((m, n), np.float32)
    bias = np.zeros(n, np.float32)
    cfg = tk.build_fused_config(m, n, k, np.float16, bias=bias, relu_on_c=False, relu_on_d=False,
                                add_a=0.1, add_b=-0.3)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    run = tk.last_run()
    assert run["lane"] == "tcgen05"
    assert run["plan"]["kernel"] == kernel and run["plan"]["mmas_per_k16"] == 3, run["plan"]
    want = O.fused_reference(_f32(a), _f32(b), c, bias, relu_on_c=False, relu_on_d=False,
                             add_a=0.1, add_b=-0.3)
    got = _host(d, (m, n))
    assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)
    # and against the exact product of the FP32-transformed operands
    ta = (_f32(a) + np.float32(0.1)).astype(np.float64)
    tb = (_f32(b) + np.float32(-0.3)).astype(np.float64)
    assert O.rel_err(got, ta @ tb) <= O.tolerance(k)


@pytest.mark.parametrize("mnk", [(512, 384, 320), (2048, 1536, 512)])
def test_non_affine_programs(cuda, mnk):
    """A non-affine program on A (scale, relu, add) and relu on B on the tensor cores, C and
    D transforms and a row bias on top, against the oracle."""
    m, n, k = mnk
    rng = np.random.default_rng(32)
    a = rng.standard_normal((m, k)).astype(np.float16)
    b = rng.standard_normal((k, n)).astype(np.float16)
    c = rng.standard_normal((m, n)).astype(np.float32)
    bias = rng.standard_normal(m).astype(np.float32)
    ta = C.compose(C.scale(0.3), C.relu, C.add_constant(0.1))
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16), transform_g2s_a=ta,
                              transform_g2s_b=C.relu, transform_g2s_c=C.scale(0.5),
                              epilogue=C.BiasEpilogue(torch.from_numpy(bias).cuda(), axis="m"),
                              transform_s2g_d=C.relu)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    assert tk.last_run()["plan"]["mmas_per_k16"] == 3
    want = O.gemm_real(_f32(a), _f32(b), c,
                       t_a=O.prog((O.T_SCALE, 0.3), (O.T_RELU, 0), (O.T_ADD, 0.1)),
                       t_b=O.prog((O.T_RELU, 0)), t_c=O.prog((O.T_SCALE, 0.5)),
                       t_s2g=O.prog((O.T_RELU, 0)), bias=bias, bias_axis="m")
    assert O.rel_err(_host(d, (m, n)), want) <= O.tolerance(k)


@pytest.mark.parametrize("dtype", [np.float16, "bf16"])
@pytest.mark.parametrize("mnk", [(384, 640, 320), (2048, 2048, 1024)])
def test_exact_programs_one_plane_bitwise(cuda, dtype, mnk):
    """relu / negation (exact in the storage type): one transformed plane, the ordinary real
    kernels, bitwise on integer inputs (bf16 too)."""
    dtype = tk.BFLOAT16 if dtype == "bf16" else np.dtype(dtype)
    m, n, k = mnk
    rng = np.random.default_rng(33)
    a = rng.integers(-4, 5, (m, k)).astype(np.float32)
    b = rng.integers(-4, 5, (k, n)).astype(np.float32)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, dtype), transform_g2s_a=C.relu,
                              transform_g2s_b=C.compose(C.scale(-1.0), C.relu))
    tdt = torch.float16 if dtype == np.float16 else torch.bfloat16
    dev = lambda x: _dev(x).to(tdt)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, dev(a), dev(b), _dev(c), d)
    plan = tk.last_run()["plan"]
    assert tk.last_run()["lane"] == "tcgen05" and plan["mmas_per_k16"] in (1, 2), plan
    want = O.gemm_real(a, b, c, t_a=O.prog((O.T_RELU, 0)),
                       t_b=O.prog((O.T_SCALE, -1.0), (O.T_RELU, 0)))
    assert np.array_equal(_host(d, (m, n)), want)


def test_grid_exact_split_program_skips_lo_bitwise(cuda):
    """add 0.5 on integer fp16 inputs: every transformed value is a half-integer (exact in
    fp16), so no lo plane is non-zero -- the split kernel skips those loads and MMAs -- and
    every sum stays exact: bitwise equal to the oracle."""
    m, n, k = 1024, 1024, 512
    rng = np.random.default_rng(34)
    a = rng.integers(-4, 5, (m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    bias = rng.integers(-4, 5, n).astype(np.float32)
    cfg = tk.build_fused_config(m, n, k, np.float16, bias=bias, relu_on_c=True, relu_on_d=True,
                                add_a=0.5, add_b=-0.5)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    want = O.fused_reference(_f32(a), _f32(b), c, bias, relu_on_c=True, relu_on_d=True,
                             add_a=0.5, add_b=-0.5)
    assert np.array_equal(_host(d, (m, n)), want)


@pytest.mark.slow
def test_fused_8192_random_at_size(cuda):
    """build_fused_config at 8192^3 on random fp16 inputs (add_a=0.5, add_b=-0.25, ReLU on C,
    bias; no ReLU on D, which would zero the ~ -K/8 result): whole matrix vs float64 of the
    FP32-transformed operands."""
    m = n = k = 8192
    g = torch.Generator(device=cuda)
    g.manual_seed(35)
    a = torch.randn(m * k, generator=g, device=cuda).half()
    b = torch.randn(k * n, generator=g, device=cuda).half()
    c = torch.randn(m * n, generator=g, device=cuda)
    bias = torch.randn(n, generator=g, device=cuda)
    cfg = tk.build_fused_config(m, n, k, np.float16, bias=bias, relu_on_c=True, relu_on_d=False,
                                add_a=0.5, add_b=-0.25)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, a, b, c, d)
    assert tk.last_run()["lane"] == "tcgen05"
    A = (a.float() + 0.5).double().view(k, m).t()
    B = (b.float() - 0.25).double().view(n, k).t()
    want = A @ B + torch.relu(c.double().view(n, m).t()) + bias.double()[None, :]
    got = d.view(n, m).t().double()
    assert ((got - want).abs().max() / want.abs().max()).item() <= O.tolerance(k)
