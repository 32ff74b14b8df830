"""At-size parity: the BASELINE.json configurations at the sizes the
bench and the north star quote them, through the public API on its DEFAULT dispatch (no
tuning overrides: the exact kernel, tile shape, serpentine K order and split-K policy the
bench line runs).

Yardsticks, all size-independent so they hold at 8192^3 and beyond:

* integer-valued inputs in [-4, 4]: every product and partial sum is an integer below 2^24,
  so every summation order gives the same FP32 value -- the device result must be bitwise
  equal to the exact (float64) product, and therefore to the reference's own k-ascending
  FP32 result (the oracle, tk_oracle.c);
* random fp16/bf16 inputs: normwise error vs the float64 product <= 4 * 2^-24 * sqrt(K)
  (complex 8x) over the WHOLE matrix, plus oracle blocks (the C restatement of the
  reference, k ascending in FP32) on row x column windows chosen to cover both K directions
  of the serpentine schedule and a raster-group boundary.

The float64 yardstick is computed on the GPU with torch (cuBLAS DGEMM), never by the
product path.
"""

import dataclasses

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def _ints(shape, dtype, gen, dev):
    return torch.randint(-4, 5, shape, generator=gen, device=dev, dtype=torch.int32).to(dtype)


def _cm(flat, rows, cols):
    """Logical rows x cols view of a flat column-major buffer."""
    return flat.view(cols, rows).t()


def _rel(got, want):
    return ((got.double() - want).abs().max() / want.abs().max()).item()


def _plan():
    return tk.last_run().get("plan") or {}


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_headline_8192_default_path(cuda, dtype):
    """The bench workload exactly: 8192^3, D = A*B + C, default dispatch (256 x 512 CTA-pair
    tiles with two MMAs per K step, serpentine K, grouped raster)."""
    m = n = k = 8192
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    cfg = tk.build_dense_config(m, n, k, tk.FLOAT16 if dtype == "fp16" else tk.BFLOAT16)
    g = torch.Generator(device=cuda)
    g.manual_seed(101)
    # integer inputs: bitwise equal to the exact product
    a = _ints((m * k,), tdt, g, cuda)
    b = _ints((k * n,), tdt, g, cuda)
    c = _ints((m * n,), torch.float32, g, cuda)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, a, b, c, d)
    assert tk.last_run()["lane"] == "tcgen05"
    plan = _plan()
    if plan:
        assert plan["kernel"] == "pair" and plan["nsub"] == 2 and plan["serpentine"] == 1, plan
    want = (_cm(a, m, k).double() @ _cm(b, k, n).double() + _cm(c, m, n).double()).float()
    assert torch.equal(_cm(d, m, n), want)
    del want
    # random inputs: whole matrix vs float64, oracle windows vs the reference's own order
    a = torch.randn(m * k, generator=g, device=cuda).to(tdt)
    b = torch.randn(k * n, generator=g, device=cuda).to(tdt)
    c = torch.randn(m * n, generator=g, device=cuda)
    tk.matmul(cfg, a, b, c, d)
    A, B, C, D = _cm(a, m, k), _cm(b, k, n), _cm(c, m, n), _cm(d, m, n)
    exact = A.double() @ B.double() + C.double()
    assert _rel(D, exact) <= O.tolerance(k)
    del exact
    # 512-column slab nb=4 holds tiles 64..79 of raster group 0: tiles 64-73 are the first
    # unit of clusters 64-73 (K ascending), 74-79 the second unit of clusters 0-5 (K
    # descending); rows 4096+ belong to raster group 1
    rows = torch.cat([torch.arange(0, 256), torch.arange(4096, 4352)]).to(cuda)
    cols = slice(2048, 2560)
    f32 = lambda x: np.asfortranarray(x.float().cpu().numpy())
    want = O.gemm_real(f32(A[rows]), f32(B[:, cols]), f32(C[rows][:, cols]))
    got = D[rows][:, cols].cpu().numpy()
    assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)


def test_n16384_default_path_integer_bitwise(cuda):
    """C2's top point: 16384^3 on the default dispatch, bitwise on integer inputs."""
    m = n = k = 16384
    cfg = tk.build_dense_config(m, n, k, tk.FLOAT16)
    g = torch.Generator(device=cuda)
    g.manual_seed(102)
    a = _ints((m * k,), torch.float16, g, cuda)
    b = _ints((k * n,), torch.float16, g, cuda)
    c = _ints((m * n,), torch.float32, g, cuda)
    d = torch.full((m * n,), float("nan"), device=cuda)
    tk.matmul(cfg, a, b, c, d)
    assert tk.last_run()["lane"] == "tcgen05"
    want = torch.addmm(_cm(c, m, n).double(), _cm(a, m, k).double(), _cm(b, k, n).double())
    assert torch.equal(_cm(d, m, n), want.float())


@pytest.mark.parametrize("n", [1024, 2048, 4096])
def test_sweep_default_path_integer_bitwise(cuda, n):
    """C2's lower points (single-wave and split-K shapes on the default dispatch)."""
    cfg = tk.build_dense_config(n, n, n, tk.FLOAT16)
    g = torch.Generator(device=cuda)
    g.manual_seed(103)
    a = _ints((n * n,), torch.float16, g, cuda)
    b = _ints((n * n,), torch.float16, g, cuda)
    c = _ints((n * n,), torch.float32, g, cuda)
    d = torch.full((n * n,), float("nan"), device=cuda)
    tk.matmul(cfg, a, b, c, d)
    want = torch.addmm(_cm(c, n, n).double(), _cm(a, n, n).double(), _cm(b, n, n).double())
    assert torch.equal(_cm(d, n, n), want.float())


def _c3_config(m, n, k, ta, tb, al, be, bias):
    return dataclasses.replace(
        tk.build_dense_config(m, n, k, tk.FLOAT16, trans_a=ta, trans_b=tb),
        transform_g2s_c=tk.components.scale(be / al), transform_r2s_d=tk.components.scale(al),
        epilogue=tk.components.BiasEpilogue(bias), transform_s2g_d=tk.components.relu)


@pytest.mark.parametrize("trans", ["nn", "nt", "tn", "tt"])
def test_c3_full_matrix(cuda, trans):
    """C3 at 8192: transposed layouts, alpha/beta scaling transforms, bias and ReLU epilogue,
    checked over the whole matrix.  Integer run: alpha = 2, beta = 1 keep every epilogue step
    exact, so D is bitwise relu(2 * (A B + C / 2) + bias).  Random run: alpha = 1.5,
    beta = 0.5 against the float64 relu(alpha A B + beta C + bias)."""
    m = n = k = 8192
    ta, tb = trans[0] == "t", trans[1] == "t"
    g = torch.Generator(device=cuda)
    g.manual_seed(104)
    A_of = lambda a: _cm(a, k, m).t() if ta else _cm(a, m, k)
    B_of = lambda b: _cm(b, n, k).t() if tb else _cm(b, k, n)
    for integer in (True, False):
        if integer:
            a = _ints((m * k,), torch.float16, g, cuda)
            b = _ints((k * n,), torch.float16, g, cuda)
            c = _ints((m * n,), torch.float32, g, cuda)
            bias = _ints((n,), torch.float32, g, cuda)
            al, be = 2.0, 1.0
        else:
            a = torch.randn(m * k, generator=g, device=cuda).half()
            b = torch.randn(k * n, generator=g, device=cuda).half()
            c = torch.randn(m * n, generator=g, device=cuda)
            bias = torch.randn(n, generator=g, device=cuda)
            al, be = 1.5, 0.5
        d = torch.full((m * n,), float("nan"), device=cuda)
        counters = tk.matmul(_c3_config(m, n, k, ta, tb, al, be, bias), a, b, c, d)
        assert tk.last_run()["lane"] == "tcgen05"
        assert counters.global_stores == m * n
        want = torch.relu(al * (A_of(a).double() @ B_of(b).double()) + be * _cm(c, m, n).double()
                          + bias.double()[None, :])
        if integer:
            assert torch.equal(_cm(d, m, n), want.float())
        else:
            assert _rel(_cm(d, m, n), want) <= O.tolerance(k)
        del want


def _pair_buf(p0, p1, split):
    return torch.cat([p0, p1]) if split else torch.stack([p0, p1], dim=1).reshape(-1)


def _pair_planes(buf, vol, split):
    return (buf[:vol], buf[vol:]) if split else (buf[0::2], buf[1::2])


@pytest.mark.parametrize("n", [4096, 8192])
@pytest.mark.parametrize("split", [True, False])
@pytest.mark.parametrize("kind", ["complex", "dual"])
def test_c4_c5_pair_operators_integer_bitwise(cuda, kind, split, n):
    """C4 (complex, 4 real MMAs per step) and C5's dual GEMM (3) at 4096 and 8192, split and
    interleaved layouts, default dispatch: bitwise equal to the exact product."""
    m = k = n
    g = torch.Generator(device=cuda)
    g.manual_seed(105)
    ar, ai = _ints((m * k,), torch.float16, g, cuda), _ints((m * k,), torch.float16, g, cuda)
    br, bi = _ints((k * n,), torch.float16, g, cuda), _ints((k * n,), torch.float16, g, cuda)
    cr, ci = _ints((m * n,), torch.float32, g, cuda), _ints((m * n,), torch.float32, g, cuda)
    if kind == "complex":
        cfg = tk.build_complex_config(m, n, k, tk.COMPLEX32, split=split)
    else:
        cfg = tk.build_dual_config(m, n, k, tk.DUAL16, split=split)
    cbuf = _pair_buf(cr, ci, split)
    d = torch.full_like(cbuf, float("nan"))
    tk.matmul(cfg, _pair_buf(ar, ai, split), _pair_buf(br, bi, split), cbuf, d)
    assert tk.last_run()["lane"] == "tcgen05"
    d0, d1 = (_cm(x, m, n) for x in _pair_planes(d, m * n, split))
    Ar, Ai, Br, Bi = _cm(ar, m, k).double(), _cm(ai, m, k).double(), _cm(br, k, n).double(), \
        _cm(bi, k, n).double()
    if kind == "complex":
        w0 = _cm(cr, m, n).double() + Ar @ Br - Ai @ Bi
        w1 = _cm(ci, m, n).double() + Ar @ Bi + Ai @ Br
    else:
        w0 = _cm(cr, m, n).double() + Ar @ Br
        w1 = _cm(ci, m, n).double() + Ar @ Bi + Ai @ Br
    assert torch.equal(d0, w0.float()) and torch.equal(d1, w1.float())


@pytest.mark.parametrize("split", [True, False])
def test_c4_complex_8192_random(cuda, split):
    """C4 at 8192 on random fp16 inputs: normwise within 8 * 2^-24 * sqrt(K) of the complex128
    product, both planes, whole matrix."""
    m = n = k = 8192
    g = torch.Generator(device=cuda)
    g.manual_seed(106)
    r = lambda cnt: torch.randn(cnt, generator=g, device=cuda)
    ar, ai, br, bi = r(m * k).half(), r(m * k).half(), r(k * n).half(), r(k * n).half()
    cr, ci = r(m * n), r(m * n)
    cfg = tk.build_complex_config(m, n, k, tk.COMPLEX32, split=split)
    cbuf = _pair_buf(cr, ci, split)
    d = torch.full_like(cbuf, float("nan"))
    tk.matmul(cfg, _pair_buf(ar, ai, split), _pair_buf(br, bi, split), cbuf, d)
    d0, d1 = (_cm(x, m, n) for x in _pair_planes(d, m * n, split))
    A = torch.complex(_cm(ar, m, k).double(), _cm(ai, m, k).double())
    B = torch.complex(_cm(br, k, n).double(), _cm(bi, k, n).double())
    W = A @ B + torch.complex(_cm(cr, m, n).double(), _cm(ci, m, n).double())
    scale = W.abs().max().item()
    err = max((d0.double() - W.real).abs().max().item(), (d1.double() - W.imag).abs().max().item())
    assert err / scale <= O.tolerance(k, 8.0)


@pytest.mark.parametrize("shape", [(64, 32, 2048, 2048), (64, 128, 8192, 8192)])
def test_c5_tensor_contraction_integer_bitwise(cuda, shape):
    """C5 TC: D[a,b,c] = sum_d A[b,d,a] B[d,c] at the paper shape and the large shape."""
    na, nb, nc, nd = shape
    g = torch.Generator(device=cuda)
    g.manual_seed(107)
    a = _ints((nb, nd, na), torch.float16, g, cuda)
    b = _ints((nd, nc), torch.float16, g, cuda)
    d, counters = tk.contract(a, b)
    assert tk.last_run()["lane"] == "tcgen05"
    assert counters.global_stores == na * nb * nc
    want = torch.einsum("bda,dc->abc", a.double(), b.double())
    assert torch.equal(d, want.float())


def test_c5_tensor_contraction_large_random(cuda):
    na, nb, nc, nd = 64, 128, 8192, 8192
    g = torch.Generator(device=cuda)
    g.manual_seed(108)
    a = torch.randn((nb, nd, na), generator=g, device=cuda).half()
    b = torch.randn((nd, nc), generator=g, device=cuda).half()
    d, _ = tk.contract(a, b)
    want = torch.einsum("bda,dc->abc", a.double(), b.double())
    assert _rel(d, want) <= O.tolerance(nd)


@pytest.mark.parametrize("n", [8192, 16384])
def test_c5_diagonal_at_size(cuda, n):
    """C5 diagonal: D = diag(a) B + C at 8192 and 16384 on random inputs.  One product per
    element (exact in FP32) plus C: bitwise equal to the FP32 evaluation of the same."""
    g = torch.Generator(device=cuda)
    g.manual_seed(109)
    diag = torch.randn(n, generator=g, device=cuda).half()
    b = torch.randn(n * n, generator=g, device=cuda).half()
    c = torch.randn(n * n, generator=g, device=cuda)
    d = torch.full((n * n,), float("nan"), device=cuda)
    counters = tk.matmul(tk.build_diagonal_config(n, tk.FLOAT16), diag, b, c, d)
    assert tk.last_run()["lane"] == "tcgen05"
    assert counters.global_stores == n * n
    want = diag.float()[:, None] * _cm(b, n, n).float() + _cm(c, n, n)
    assert torch.equal(_cm(d, n, n), want)
