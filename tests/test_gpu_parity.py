"""GPU parity: the device lanes against the oracle (C restatement of the reference).

Bars:
* tcgen05 lane (f16/bf16 storage, FP32 accumulation): normwise relative error vs the
  oracle <= 4 * 2^-24 * sqrt(K) (complex: 8x); integer-valued inputs: bitwise equal.
* simt lane (reference dtypes): bitwise equal -- it replays the reference's operation order.
"""

import dataclasses

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    x = np.asarray(x)
    if x.dtype == tk.BFLOAT16:
        return torch.from_numpy(np.ascontiguousarray(x.ravel(order="F")).view(np.uint16)) \
            .view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x.ravel(order="F"))).cuda()


def _host(t, shape, dtype=np.float32):
    return t.cpu().numpy().reshape(shape, order="F").astype(dtype, copy=False)


def _half(rng, shape, dtype, integer=False):
    if integer:
        return rng.integers(-4, 5, shape).astype(dtype)
    return rng.standard_normal(shape).astype(dtype)


def _f32(x):
    return np.asarray(x).astype(np.float32)


@pytest.fixture(params=["single", "pair", "pair128", "pair64", "pair64k1", "pair512", "quad", "stream",
                        "ksplit"])
def tc_kernel(request, knob):
    """Pin the single-CTA (128x256), CTA-pair (256 x 256/128/64 tiles -- the narrow ones with two
    K-blocks per ring stage, `k1` one -- or 256 x 512 with two MMAs per K step), 4-CTA multicast
    or C-streaming tcgen05 kernel; `ksplit` forces the on-chip split-K kernel wherever it is legal
    (single-wave shapes on the pair path)."""
    name = request.param
    if name == "ksplit":
        knob("TK_KSPLIT", "2")
    elif name.startswith("pair") and name != "pair":
        knob("TK_TC_KERNEL", "pair")
        if name == "pair512":
            knob("TK_PAIR_NSUB", "2")
        else:
            knob("TK_PAIR_BNI", name[4:].split("k")[0])
            if name.endswith("k1"):
                knob("TK_PAIR_KPS", "1")
    else:
        knob("TK_TC_KERNEL", name)
    return name


@pytest.mark.parametrize("dtype", [np.float16, "bf16"])
@pytest.mark.parametrize("trans", ["nn", "nt", "tn", "tt"])
def test_dense_integer_exact(cuda, dtype, trans, tc_kernel):
    dtype = tk.BFLOAT16 if dtype == "bf16" else np.dtype(dtype)
    m, n, k = 384, 640, 320
    ta, tb = trans[0] == "t", trans[1] == "t"
    rng = np.random.default_rng(0)
    a = _half(rng, (m, k), dtype, True)
    b = _half(rng, (k, n), dtype, True)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, dtype, trans_a=ta, trans_b=tb)
    abuf = _dev(a.T if ta else a) if ta else _dev(a)
    bbuf = _dev(b.T if tb else b) if tb else _dev(b)
    d = torch.zeros(m * n, dtype=torch.float32, device=cuda)
    tk.matmul(cfg, abuf, bbuf, _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    want = O.gemm_real(_f32(a), _f32(b), c)
    got = _host(d, (m, n))
    assert np.array_equal(got, want), f"max abs diff {np.max(np.abs(got - want))}"


@pytest.mark.parametrize("dtype", [np.float16, "bf16"])
@pytest.mark.parametrize("mnk", [(128, 256, 64), (1024, 1024, 1024), (384, 768, 2048),
                                 (200, 136, 72), (8, 16, 8), (1000, 520, 4104),
                                 (1024, 768, 128), (520, 1000, 256)])
def test_dense_random_within_tolerance(cuda, dtype, mnk, tc_kernel):
    dtype = tk.BFLOAT16 if dtype == "bf16" else np.dtype(dtype)
    m, n, k = mnk
    rng = np.random.default_rng(1)
    a, b = _half(rng, (m, k), dtype), _half(rng, (k, n), dtype)
    c = rng.standard_normal((m, n)).astype(np.float32)
    cfg = tk.build_dense_config(m, n, k, dtype, operator_shape=(8, 8, 8))
    d = torch.zeros(m * n, dtype=torch.float32, device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    got = _host(d, (m, n))
    want = O.gemm_real(_f32(a), _f32(b), c)
    exact = O.exact_gemm(_f32(a), _f32(b), c, beta=1.0)
    assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)
    assert O.rel_err(got, exact) <= O.tolerance(k), O.rel_err(got, exact)


@pytest.mark.parametrize("bni", ["64", "128"])
@pytest.mark.parametrize("kps", ["1", "2"])
@pytest.mark.parametrize("grid", ["3", "0"])
def test_narrow_tiles_ring_stages(cuda, bni, kps, grid, knob):
    """Narrow pair tiles with one or two K-blocks per ring stage: an odd K-block count (the last
    stage half-filled), several tiles per cluster (TK_PAIR_GRID=3: serpentine K order and ring
    phases carried across tiles), MN-major A and B -- bitwise on integers, plan as requested."""
    knob("TK_TC_KERNEL", "pair")
    knob("TK_PAIR_BNI", bni)
    knob("TK_PAIR_KPS", kps)
    if grid != "0":
        knob("TK_PAIR_GRID", grid)
    rng = np.random.default_rng(5)
    for (m, n, k, ta, tb) in [(768, 640, 7 * 64 + 24, False, False), (512, 384, 9 * 64, True, False),
                              (256, 512, 3 * 64, False, bni == "128")]:
        a = _half(rng, (m, k), np.float16, True)
        b = _half(rng, (k, n), np.float16, True)
        c = rng.integers(-4, 5, (m, n)).astype(np.float32)
        cfg = tk.build_dense_config(m, n, k, np.float16, trans_a=ta, trans_b=tb)
        d = torch.zeros(m * n, dtype=torch.float32, device=cuda)
        tk.matmul(cfg, _dev(a.T) if ta else _dev(a), _dev(b.T) if tb else _dev(b), _dev(c), d)
        plan = tk.last_run()["plan"]
        assert plan["kernel"] == "pair" and plan["mma_n"] == int(bni), plan
        assert plan["tile_k"] == 64 * int(kps), plan
        got = _host(d, (m, n))
        want = O.gemm_real(_f32(a), _f32(b), c)
        assert np.array_equal(got, want), (m, n, k, float(np.abs(got - want).max()))


@pytest.mark.parametrize("nt", ["1", "2", "w"])
@pytest.mark.parametrize("kps", ["1", "2"])
@pytest.mark.parametrize("case", [
    (1024, 1024, 1024, False, False, "f16"),      # the C2 low end: 32 tiles of 256 x 128
    (1000, 520, 4104, False, False, "bf16"),      # M / N tails, odd k-block count (65)
    (512, 768, 7 * 64 + 24, True, False, "f16"),  # K-major A, K tail inside the last block
    (768, 384, 640, False, True, "f16"),          # MN-major B
    (256, 128, 320, True, True, "bf16"),          # one cluster, 5 k-blocks (2 + 3)
    (200, 40, 1024, False, False, "f16"),         # one partial M block, N < the finalised half
])
def test_ksplit_on_chip(cuda, case, kps, nt, knob):
    """On-chip split-K (two CTA pairs per 256 x 128 tile, one K half each, partials
    reduce-scattered through distributed shared memory; 4-CTA clusters, or 8 with two tiles
    sharing multicast A atoms -- the shapes include a second tile wholly past N -- or, `w`,
    256 x 256 tiles on 4-CTA clusters, two boxes per epilogue warp): integer inputs
    bitwise equal to the oracle with bias + ReLU, random inputs within the sqrt(K) bound with the
    C3 alpha/beta scaling, and the plan really is the k-split kernel."""
    m, n, k, ta, tb, dt = case
    dtype = tk.BFLOAT16 if dt == "bf16" else np.dtype(np.float16)
    knob("TK_KSPLIT", "2")
    knob("TK_KSPLIT_KPS", kps)
    if nt == "w":
        knob("TK_KSPLIT_BNI", "256")
    else:
        knob("TK_KSPLIT_NT", nt)
    rng = np.random.default_rng(23)
    for integer in (True, False):
        a, b = _half(rng, (m, k), dtype, integer), _half(rng, (k, n), dtype, integer)
        c = (rng.integers(-4, 5, (m, n)) if integer else rng.standard_normal((m, n))).astype(np.float32)
        bias = (rng.integers(-4, 5, n) if integer else rng.standard_normal(n)).astype(np.float32)
        cfg = dataclasses.replace(tk.build_dense_config(m, n, k, dtype, trans_a=ta, trans_b=tb),
                                  epilogue=tk.components.BiasEpilogue(torch.from_numpy(bias).cuda()),
                                  transform_s2g_d=tk.components.relu)
        al, be = 1.5, 0.5
        if not integer:
            cfg = dataclasses.replace(cfg, transform_g2s_c=tk.components.scale(be / al),
                                      transform_r2s_d=tk.components.scale(al))
        d = torch.full((m * n,), float("nan"), dtype=torch.float32, device=cuda)
        tk.matmul(cfg, _dev(a.T) if ta else _dev(a), _dev(b.T) if tb else _dev(b), _dev(c), d)
        plan = tk.last_run()["plan"]
        if plan["kernel"] == "pair":  # 8-CTA clusters: only ~15 are co-resident on a B200
            assert nt == "2" and ((m + 255) // 256) * ((n + 255) // 256) >= 15, plan
        else:
            assert plan["kernel"] == "ksplit" and plan["cluster"] == (8 if nt == "2" else 4), plan
            assert plan["mma_n"] == (256 if nt == "w" else 128), plan
            assert plan["tile_k"] == 64 * int(kps), plan
        got = _host(d, (m, n))
        if integer:
            want = np.maximum(O.gemm_real(_f32(a), _f32(b), c) + bias[None, :], 0)
            assert np.array_equal(got, want), (case, float(np.abs(got - want).max()))
        else:
            prod = _f32(a).astype(np.float64) @ _f32(b).astype(np.float64)
            want = np.maximum(al * (prod + (be / al) * c) + bias[None, :], 0)
            assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)


def test_ksplit_zero_c(cuda, knob):
    """The k-split kernel with a Zero C layout (no C loads: D = A*B), integer inputs bitwise."""
    knob("TK_KSPLIT", "2")
    m, n, k = 768, 512, 1000 // 8 * 8
    rng = np.random.default_rng(29)
    a = _half(rng, (m, k), np.float16, True)
    b = _half(rng, (k, n), np.float16, True)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    cfg = dataclasses.replace(cfg, global_c_layout=tk.layouts.Zero(np.float32, ("M", "N"), (m, n)))
    d = torch.full((m * n,), float("nan"), dtype=torch.float32, device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), torch.empty(0, dtype=torch.float32, device=cuda), d)
    assert tk.last_run()["plan"]["kernel"] == "ksplit", tk.last_run()["plan"]
    want = O.gemm_real(_f32(a), _f32(b), np.zeros((m, n), np.float32))
    assert np.array_equal(_host(d, (m, n)), want)


def test_ksplit_bias_m_relu(cuda, knob):
    """k-split kernel with a bias along M and ReLU, both finalising halves: bitwise on integers."""
    knob("TK_KSPLIT", "2")
    m, n, k = 512, 384, 640
    rng = np.random.default_rng(31)
    a = _half(rng, (m, k), np.float16, True)
    b = _half(rng, (k, n), np.float16, True)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    bias = rng.integers(-4, 5, m).astype(np.float32)
    cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16),
                              epilogue=tk.components.BiasEpilogue(torch.from_numpy(bias).cuda(), axis="m"),
                              transform_s2g_d=tk.components.relu)
    d = torch.full((m * n,), float("nan"), dtype=torch.float32, device=cuda)
    tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    assert tk.last_run()["plan"]["kernel"] == "ksplit", tk.last_run()["plan"]
    want = np.maximum(O.gemm_real(_f32(a), _f32(b), c) + bias[:, None], 0)
    assert np.array_equal(_host(d, (m, n)), want)


def test_ksplit_auto_choice(cuda):
    """The default dispatch takes the on-chip split-K kernel for 1024^3 (single wave of 256 x 128
    tiles) and keeps whole-K pair tiles where there are enough of them (2048^3)."""
    for n, want in ((1024, "ksplit"), (2048, "pair")):
        a = torch.ones(n * n, dtype=torch.float16, device=cuda)
        c = torch.zeros(n * n, device=cuda)
        d = torch.empty(n * n, device=cuda)
        tk.matmul(tk.build_dense_config(n, n, n, np.float16), a, a, c, d)
        assert tk.last_run()["plan"]["kernel"] == want, (n, tk.last_run()["plan"])
        assert torch.all(d == n)


_SPLITK_WANT = {}


@pytest.mark.parametrize("mnk", [(2560, 2560, 8192), (1536, 4096, 8192), (1280, 1280, 16384)])
@pytest.mark.parametrize("splitk", ["0", "1"])
def test_split_k_last_wave(cuda, mnk, splitk, knob):
    """Pair kernel with the poorly filled last wave cut into K-parts (FP32 partials in the
    workspace, reduced in a fixed order by the last part): integer inputs stay bitwise exact,
    random inputs within tolerance, with or without the split."""
    knob("TK_SPLITK", splitk)
    knob("TK_PAIR_BNI", "256")  # 256-wide tiles: the last wave is R = T % 74 tiles
    m, n, k = mnk
    rng = np.random.default_rng(17)
    for integer in (True, False):
        a, b = _half(rng, (m, k), np.float16, integer), _half(rng, (k, n), np.float16, integer)
        c = (rng.integers(-4, 5, (m, n)) if integer else rng.standard_normal((m, n))).astype(np.float32)
        bias = rng.standard_normal(n).astype(np.float32)
        cfg = dataclasses.replace(tk.build_dense_config(m, n, k, np.float16),
                                  epilogue=tk.components.BiasEpilogue(torch.from_numpy(bias).cuda()),
                                  transform_s2g_d=tk.components.relu)
        d = torch.zeros(m * n, dtype=torch.float32, device=cuda)
        tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
        got = _host(d, (m, n))
        key = (mnk, integer)
        if key not in _SPLITK_WANT:  # the oracle is shared by the split / unsplit runs
            _SPLITK_WANT[key] = np.maximum(O.gemm_real(_f32(a), _f32(b), c) + bias[None, :], 0)
        want = _SPLITK_WANT[key]
        if integer:
            assert np.array_equal(got, want), float(np.abs(got - want).max())
        else:
            assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)


@pytest.mark.parametrize("mnk,minkb", [((2560, 2560, 8192), "64"), ((1024, 1024, 1024), "4")])
def test_split_k_ring_matches_direct(cuda, mnk, minkb, knob):
    """Split-K partials moved as TMA boxes through the C ring (default) and by per-thread
    stores/loads (TK_SK_TMA=0) sum in the same order: bitwise equal on random inputs."""
    m, n, k = mnk
    knob("TK_PAIR_BNI", "256")
    knob("TK_SPLITK_MINKB", minkb)
    g = torch.Generator(device=cuda)
    g.manual_seed(9)
    a = torch.randn(m * k, generator=g, device=cuda).half()
    b = torch.randn(k * n, generator=g, device=cuda).half()
    c = torch.randn(m * n, generator=g, device=cuda)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    outs = []
    for mode in ("1", "0"):
        knob("TK_SK_TMA", mode)
        d = torch.full((m * n,), float("nan"), device=cuda)
        tk.matmul(cfg, a, b, c, d)
        plan = tk.last_run()["plan"]
        # the split really ran, with the requested hand-off (not a silently unsplit launch)
        assert plan["kernel"] == "pair" and plan["sk_parts"] > 1, plan
        assert plan["sk_tma"] == int(mode), plan
        outs.append(d)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("mnk", [(8192, 8192, 8192), (4096, 8192 + 512, 8192)])
def test_staggered_schedule_bitwise(cuda, mnk, knob):
    """The opt-in staggered 256 x 512 schedule (half of the clusters split one tile into a
    leading and a trailing half) covers every tile exactly once: bitwise equal to the default
    schedule with serpentine K off (same k order per tile)."""
    m, n, k = mnk
    knob("TK_SERPENTINE", "0")
    knob("TK_PAIR_NSUB", "2")
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    a = torch.randn(m * k, generator=g, device=cuda).half()
    b = torch.randn(k * n, generator=g, device=cuda).half()
    c = torch.randn(m * n, generator=g, device=cuda)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    outs = []
    for stagger in ("0", "1"):
        knob("TK_STAGGER", stagger)
        d = torch.full((m * n,), float("nan"), device=cuda)
        tk.matmul(cfg, a, b, c, d)
        outs.append(d)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("trans", ["nn", "tt"])
def test_full_size_c3_tile_shapes_agree(cuda, trans, knob):
    """The bench-size (8192^3) C3 epilogue (alpha/beta, bias, ReLU) on the default 256 x 512
    pair tiles against 256 x 256 tiles (same k order with serpentine off: bitwise equal), and
    sampled rows against the float64 product (size-independent checks at full size)."""
    m = n = k = 8192
    ta, tb = trans[0] == "t", trans[1] == "t"
    g = torch.Generator(device=cuda)
    g.manual_seed(21)
    a = torch.randn(m * k, generator=g, device=cuda).half()
    b = torch.randn(k * n, generator=g, device=cuda).half()
    c = torch.randn(m * n, generator=g, device=cuda)
    bias = torch.randn(n, generator=g, device=cuda)
    al, be = 1.5, 0.5
    cfg = dataclasses.replace(
        tk.build_dense_config(m, n, k, np.float16, trans_a=ta, trans_b=tb),
        transform_g2s_c=tk.components.scale(be / al), transform_r2s_d=tk.components.scale(al),
        epilogue=tk.components.BiasEpilogue(bias), transform_s2g_d=tk.components.relu)
    knob("TK_SERPENTINE", "0")
    outs = []
    for nsub in ("2", "1"):
        knob("TK_PAIR_NSUB", nsub)
        d = torch.empty(m * n, device=cuda)
        tk.matmul(cfg, a, b, c, d)
        outs.append(d)
    assert torch.equal(outs[0], outs[1])
    # rows 0..3 and 4096..4099 against float64
    A = (a.view(m, k) if ta else a.view(k, m).t()).double()     # logical m x k
    B = (b.view(k, n) if tb else b.view(n, k).t()).double()     # logical k x n
    C = c.view(n, m).t().double()
    D = outs[0].view(n, m).t()
    for r0 in (0, 4096):
        ref = torch.relu(al * (A[r0:r0 + 4] @ B + (be / al) * C[r0:r0 + 4]) + bias.double()[None, :])
        err = ((D[r0:r0 + 4].double() - ref).abs().max() / ref.abs().max()).item()
        assert err <= O.tolerance(k), err


def test_fused_affine_bias_relu(cuda):
    m, n, k = 512, 384, 256
    rng = np.random.default_rng(2)
    # 2^-8 grid in [-4, 4]: A + 0.5 and B - 0.25 exact in fp16 (SURVEY 8d transform set)
    a = (rng.integers(-1024, 1025, (m, k)) / 256.0).astype(np.float16)
    b = (rng.integers(-1024, 1025, (k, n)) / 256.0).astype(np.float16)
    c = rng.standard_normal((m, n)).astype(np.float32)
    bias = rng.standard_normal(n).astype(np.float32)
    cfg = tk.build_fused_config(m, n, k, np.float16, bias=bias, relu_on_c=True, relu_on_d=True,
                                add_a=0.5, add_b=-0.25)
    d = torch.zeros(m * n, dtype=torch.float32, device=cuda)
    counters = tk.matmul(cfg, _dev(a), _dev(b), _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    want = O.fused_reference(_f32(a), _f32(b), c, bias, relu_on_c=True, relu_on_d=True,
                             add_a=0.5, add_b=-0.25)
    assert O.rel_err(_host(d, (m, n)), want) <= O.tolerance(k)
    assert counters.global_stores == m * n


@pytest.mark.parametrize("kernel", ["auto", "single", "pair", "pair256"])
@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("kind", ["complex", "dual"])
def test_pair_operators(cuda, split, kind, kernel, knob):
    if kernel == "pair256":  # 256-wide pair tiles, one accumulator pair
        knob("TK_TC_KERNEL", "pair")
        knob("TK_PAIROPS_BN", "256")
    elif kernel != "auto":
        knob("TK_TC_KERNEL", kernel)
    m, n, k = 512, 384, 320
    rng = np.random.default_rng(3)
    h16 = lambda s: rng.standard_normal(s).astype(np.float16)
    if kind == "complex":
        a = (h16((m, k)), h16((m, k)))
        b = (h16((k, n)), h16((k, n)))
        c = (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))).astype(np.complex64)
        half = tk.COMPLEX32
        pack = lambda x: _pack_pair(x[0], x[1], half, split)
        cfg = tk.build_complex_config(m, n, k, half, split=split)
        z = lambda x: np.asfortranarray((_f32(x[0]) + 1j * _f32(x[1])).astype(np.complex64))
        want = O.gemm_pair(z(a), z(b), np.asfortranarray(c))
        parts = lambda z: (z.real, z.imag)
        factor = 8.0
    else:
        a = (h16((m, k)), h16((m, k)))
        b = (h16((k, n)), h16((k, n)))
        c = tk.dual_array(rng.standard_normal((m, n)), rng.standard_normal((m, n)), tk.DUAL32)
        half = tk.DUAL16
        pack = lambda x: _pack_pair(x[0], x[1], half, split)
        cfg = tk.build_dual_config(m, n, k, half, split=split)
        h = lambda x: x.astype(np.float16).astype(np.float32)
        want = O.gemm_pair(np.asfortranarray(tk.dual_array(h(a[0]), h(a[1]), tk.DUAL32)),
                           np.asfortranarray(tk.dual_array(h(b[0]), h(b[1]), tk.DUAL32)),
                           np.asfortranarray(c), dual=True)
        parts = lambda z: (z["value"], z["epsilon"])
        factor = 4.0
    cbuf = _pack_pair(*parts(c), None, split)
    d = torch.zeros_like(cbuf)
    tk.matmul(cfg, pack(a), pack(b), cbuf, d)
    assert tk.last_run()["lane"] == "tcgen05"
    got = _unpack_pair(d, (m, n), split)
    w0, w1 = parts(want)
    err = max(O.rel_err(got[0], w0), O.rel_err(got[1], w1))
    assert err <= O.tolerance(k, factor), err


@pytest.mark.parametrize("bn", ["128", "256"])
@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("kind", ["complex", "dual"])
def test_pair_operators_bf16_integer_exact(cuda, kind, split, bn, knob):
    """bf16 pair storage (COMPLEXBF16 / DUALBF16) on both pair-tile widths: small-integer
    inputs make every product and sum exact, so the result is bitwise the oracle's."""
    knob("TK_TC_KERNEL", "pair")
    knob("TK_PAIROPS_BN", bn)
    m, n, k = 512, 512, 320
    rng = np.random.default_rng(8)
    ints = lambda s: rng.integers(-4, 5, s).astype(np.float32)
    a, b, c = (ints((m, k)), ints((m, k))), (ints((k, n)), ints((k, n))), (ints((m, n)), ints((m, n)))

    def bf16_pair(x):  # flat bf16 buffer, interleaved or split planes, column-major
        p0 = torch.from_numpy(np.ascontiguousarray(x[0].ravel(order="F")))
        p1 = torch.from_numpy(np.ascontiguousarray(x[1].ravel(order="F")))
        flat = torch.cat([p0, p1]) if split else torch.stack([p0, p1], dim=1).reshape(-1)
        return flat.to(torch.bfloat16).cuda()

    if kind == "complex":
        cfg = tk.build_complex_config(m, n, k, tk.COMPLEXBF16, split=split)
        z = lambda x: np.asfortranarray((x[0] + 1j * x[1]).astype(np.complex64))
        want = O.gemm_pair(z(a), z(b), z(c))
        w0, w1 = want.real, want.imag
    else:
        cfg = tk.build_dual_config(m, n, k, tk.DUALBF16, split=split)
        dd = lambda x: np.asfortranarray(tk.dual_array(x[0], x[1], tk.DUAL32))
        want = O.gemm_pair(dd(a), dd(b), dd(c), dual=True)
        w0, w1 = want["value"], want["epsilon"]
    cbuf = _pack_pair(c[0], c[1], None, split)
    d = torch.zeros_like(cbuf)
    tk.matmul(cfg, bf16_pair(a), bf16_pair(b), cbuf, d)
    assert tk.last_run()["lane"] == "tcgen05"
    got = _unpack_pair(d, (m, n), split)
    assert np.array_equal(got[0], w0) and np.array_equal(got[1], w1)


def _pack_pair(p0, p1, half, split):
    """Flat pair buffer (interleaved or split planes, column-major) as a CUDA tensor."""
    dt = np.float16 if half is not None else np.float32
    p0 = np.asarray(p0).astype(dt).ravel(order="F")
    p1 = np.asarray(p1).astype(dt).ravel(order="F")
    flat = np.concatenate([p0, p1]) if split else np.stack([p0, p1], axis=1).ravel()
    return torch.from_numpy(flat).cuda()


def _unpack_pair(t, shape, split):
    x = t.cpu().numpy()
    vol = shape[0] * shape[1]
    if split:
        p0, p1 = x[:vol], x[vol:]
    else:
        p0, p1 = x[0::2], x[1::2]
    return p0.reshape(shape, order="F"), p1.reshape(shape, order="F")


def _complex_case(rng, m, n, k, half, integer, c_zero=False):
    if integer:
        g = lambda s: rng.integers(-4, 5, s).astype(np.float32)
    else:
        g = lambda s: rng.standard_normal(s).astype(np.float32)
    q = (lambda x: x.astype(tk.BFLOAT16).astype(np.float32)) if half == "bf16" else \
        (lambda x: x.astype(np.float16).astype(np.float32))
    a = (q(g((m, k))), q(g((k, m)).T.copy()))
    b = (q(g((k, n))), q(g((k, n))))
    c = np.zeros((m, n), np.complex64) if c_zero else (g((m, n)) + 1j * g((m, n))).astype(np.complex64)
    return a, b, c


def _pack_half_pair(p0, p1, half):
    """Interleaved pair buffer of f16 / bf16 halves (column-major) on the device."""
    dt = tk.BFLOAT16 if half == "bf16" else np.float16
    flat = np.stack([p0.astype(dt).ravel(order="F"), p1.astype(dt).ravel(order="F")], axis=1).ravel()
    if half == "bf16":
        return torch.from_numpy(flat.view(np.uint16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(flat).cuda()


@pytest.mark.parametrize("half", ["f16", "bf16"])
@pytest.mark.parametrize("nsub", ["1", "2"])
@pytest.mark.parametrize("mnk", [(256, 384, 320), (512, 768, 1000), (384, 1280, 200)])
def test_complex_embedding_interleaved(cuda, half, nsub, mnk, knob):
    """Interleaved complex GEMM as the real embedding D^ = A~ B^ + C^ (tc_gemm_pair_kernel EMB):
    A~ built on chip by the transform warps, no de-interleave pass (one launch); integer inputs
    bitwise equal to the oracle and to the de-interleaving pair-operator kernel
    (TK_CPLX_EMBED=0), random inputs within the complex bound (reference operators.py:140-163)."""
    knob("TK_PAIR_NSUB", nsub)
    m, n, k = mnk
    rng = np.random.default_rng(11)
    ht = tk.COMPLEXBF16 if half == "bf16" else tk.COMPLEX32
    cfg = tk.build_complex_config(m, n, k, ht)
    for integer in (True, False):
        a, b, c = _complex_case(rng, m, n, k, half, integer)
        cbuf = _pack_pair(c.real, c.imag, None, False)
        outs = []
        for embed in ("1", "0"):
            knob("TK_CPLX_EMBED", embed)
            d = torch.zeros_like(cbuf)
            tk.matmul(cfg, _pack_half_pair(*a, half), _pack_half_pair(*b, half), cbuf, d)
            run = tk.last_run()
            assert run["lane"] == "tcgen05"
            if embed == "1":
                assert run["plan"]["kernel"] == "pair_cembed" and run["launches"] == 1, run["plan"]
            else:
                assert run["plan"]["kernel"] != "pair_cembed" and run["launches"] == 3, run["plan"]
            outs.append(_unpack_pair(d, (m, n), False))
        z = lambda x: np.asfortranarray((x[0] + 1j * x[1]).astype(np.complex64))
        want = O.gemm_pair(z(a), z(b), np.asfortranarray(c))
        got = outs[0]
        if integer:
            assert np.array_equal(got[0], want.real) and np.array_equal(got[1], want.imag)
            assert all(np.array_equal(x, y) for x, y in zip(outs[0], outs[1]))
        else:
            err = max(O.rel_err(got[0], want.real), O.rel_err(got[1], want.imag))
            assert err <= O.tolerance(k, 8.0), err


def test_complex_embedding_gemm_ex_and_edges(cuda, knob):
    """gemm_ex-style epilogues (alpha * (AB + beta/alpha * C), api.py:129-141): real alpha / beta
    scale the real-separable epilogue (still the embedding), a complex alpha does not (the
    pair-operator kernel); C / D at an 8-byte offset (the embedding's register epilogue);
    beta = 0 -- integer inputs, bitwise."""
    rng = np.random.default_rng(12)
    m, n, k = 256, 512, 192
    a, b, c = _complex_case(rng, m, n, k, "f16", True)
    z = lambda x: np.asfortranarray((x[0] + 1j * x[1]).astype(np.complex64))
    A, B = z(a), z(b)
    for alpha, beta, kern in [(2.0, 0.5, "pair_cembed"), (1.0, 0.0, "pair_cembed"),
                              (1.0 + 1.0j, 1.0, None)]:
        cdev = _pack_pair(c.real, c.imag, None, False)
        cfg = tk.build_complex_config(m, n, k, tk.COMPLEX32)
        if (alpha, beta) != (1.0, 1.0):
            cfg = dataclasses.replace(cfg, transform_g2s_c=tk.components.scale(np.complex64(beta / alpha)),
                                      transform_r2s_d=tk.components.scale(np.complex64(alpha)))
        d = torch.zeros_like(cdev)
        tk.matmul(cfg, _pack_half_pair(*a, "f16"), _pack_half_pair(*b, "f16"), cdev, d)
        plan = tk.last_run()["plan"]
        if kern:
            assert plan["kernel"] == kern, plan
        else:
            assert plan["kernel"] != "pair_cembed", plan
        got = _unpack_pair(d, (m, n), False)
        want = alpha * (A.astype(np.complex128) @ B.astype(np.complex128)) + beta * c
        assert np.array_equal(got[0], want.real.astype(np.float32)), (alpha, beta)
        assert np.array_equal(got[1], want.imag.astype(np.float32)), (alpha, beta)
    # C and D 8 bytes into their allocations: not TMA-aligned -> the embedding's register epilogue
    cfg = tk.build_complex_config(m, n, k, tk.COMPLEX32)
    cbig = torch.zeros(2 * m * n + 2, dtype=torch.float32, device=cuda)
    cbig[2:] = _pack_pair(c.real, c.imag, None, False)
    dbig = torch.zeros_like(cbig)
    tk.matmul(cfg, _pack_half_pair(*a, "f16"), _pack_half_pair(*b, "f16"), cbig[2:], dbig[2:])
    plan = tk.last_run()["plan"]
    assert plan["kernel"] == "pair_cembed" and plan["c_stream"] == 0, plan
    got = _unpack_pair(dbig[2:], (m, n), False)
    want = A.astype(np.complex128) @ B.astype(np.complex128) + c
    assert np.array_equal(got[0], want.real.astype(np.float32))
    assert np.array_equal(got[1], want.imag.astype(np.float32))


@pytest.mark.parametrize("kernel", ["auto", "single", "tensor"])
@pytest.mark.parametrize("n", [256, 1024, 640])
def test_diagonal_variant(cuda, n, kernel, knob):
    """auto: the vectorised HBM stream; single / tensor: the tcgen05 kernel with the diagonal
    tile fabricated in shared memory -- all bitwise equal to the oracle."""
    if kernel == "single":
        knob("TK_TC_KERNEL", kernel)
    elif kernel == "tensor":
        knob("TK_DIAG_STREAM", "0")
    rng = np.random.default_rng(4)
    diag = rng.standard_normal(n).astype(np.float16)
    b = rng.standard_normal((n, n)).astype(np.float16)
    c = rng.standard_normal((n, n)).astype(np.float32)
    cfg = tk.build_diagonal_config(n, np.float16, block_tile=(64, 64, 16))
    d = torch.zeros(n * n, dtype=torch.float32, device=cuda)
    counters = tk.matmul(cfg, torch.from_numpy(diag).cuda(), _dev(b), _dev(c), d)
    assert tk.last_run()["lane"] == "tcgen05"
    want = O.gemm_real(np.diag(_f32(diag)), _f32(b), c)
    # diag(a)*B + C: one product per element -> exact in FP32
    assert np.array_equal(_host(d, (n, n)), want)
    if n % 64 == 0:
        assert counters.inner_iterations_executed == (n // 64) * (n // 64) * 4


@pytest.mark.parametrize("stream", ["1", "0", "misaligned"])
def test_diagonal_epilogue_rectangular(cuda, stream, knob):
    """Diagonal A with alpha/beta scaling, a row bias and ReLU, N != M; 'misaligned' offsets
    the buffers by one element so the stream kernel takes its scalar path."""
    knob("TK_DIAG_STREAM", "0" if stream == "0" else "1")
    m, n, k = 520, 384, 520
    rng = np.random.default_rng(6)
    diag = rng.integers(-4, 5, min(m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    bias = rng.integers(-4, 5, m).astype(np.float32)
    cfg = tk.build_diagonal_config(m, np.float16)
    cfg = dataclasses.replace(
        cfg, params=dataclasses.replace(cfg.params, gemm_shape=(m, n, k)),
        global_b_layout=tk.layouts.ColMajor(np.float16, ("K", "N"), (k, n)),
        global_c_layout=tk.layouts.ColMajor(np.float32, ("M", "N"), (m, n)),
        global_d_layout=tk.layouts.ColMajor(np.float32, ("M", "N"), (m, n)),
        transform_g2s_c=tk.components.scale(0.5), transform_r2s_d=tk.components.scale(2.0),
        epilogue=tk.components.BiasEpilogue(torch.from_numpy(bias).cuda(), axis="m"),
        transform_s2g_d=tk.components.relu)
    def dev(x, off):
        t = _dev(x)
        if not off:
            return t
        buf = torch.empty(t.numel() + 1, dtype=t.dtype, device=cuda)
        buf[1:] = t
        return buf[1:]
    off = stream == "misaligned"
    dbuf = torch.zeros(m * n + 1, dtype=torch.float32, device=cuda)
    d = dbuf[1:] if off else dbuf[:-1]
    tk.matmul(cfg, dev(diag, off), dev(b, off), dev(c, off), d)
    assert tk.last_run()["lane"] == "tcgen05"
    a_full = np.zeros((m, k), np.float32)
    a_full[np.arange(min(m, k)), np.arange(min(m, k))] = diag
    want = np.maximum(2.0 * (0.5 * c + a_full @ _f32(b)) + bias[:, None], 0)
    assert np.array_equal(_host(d, (m, n)), want.astype(np.float32))


def test_gemm_ex_alpha_beta_trans(cuda):
    m, n, k = 192, 320, 256
    rng = np.random.default_rng(5)
    a = rng.standard_normal((k, m)).astype(np.float16)           # stored transposed
    b = rng.standard_normal((k, n)).astype(np.float16)
    c = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    want = O.exact_gemm(_f32(a).T, _f32(b), c, alpha=1.5, beta=0.5)
    tc = _fortran(c)
    tk.gemm_ex(True, False, 1.5, _fortran(a), _fortran(b), 0.5, tc)
    assert O.rel_err(tc.cpu().numpy(), want) <= O.tolerance(k)


def _fortran(x):
    """F-contiguous CUDA tensor view of a numpy matrix."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).T)).cuda().t()


def test_gemm_ex_raw_host_pointers():
    m, n, k = 64, 48, 32
    rng = np.random.default_rng(6)
    a = np.asfortranarray(rng.standard_normal((m, k)).astype(np.float16))
    b = np.asfortranarray(rng.standard_normal((k, n)).astype(np.float16))
    c = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    want = O.exact_gemm(_f32(a), _f32(b), c, alpha=2.0, beta=0.25)
    st = tk.gemm_ex_raw(tk.TAG_F16F32, 0, 0, m, n, k, 2.0, 0.0, a.ctypes.data, b.ctypes.data,
                        0.25, 0.0, c.ctypes.data)
    assert st == 0
    assert O.rel_err(c, want) <= O.tolerance(k)


# ---- bit-exact CUDA-core lane ------------------------------------------------------

def test_simt_f32_bitwise(cuda):
    m, n, k = 96, 80, 64
    rng = np.random.default_rng(7)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c = rng.standard_normal((m, n)).astype(np.float32)
    bias = rng.standard_normal(n).astype(np.float32)
    cfg = tk.build_fused_config(m, n, k, np.float32, bias=bias, relu_on_c=True, add_a=0.5,
                                add_b=-0.25)
    d = np.zeros(m * n, np.float32)
    tk.matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), c.ravel(order="F"), d)
    assert tk.last_run()["lane"] == "simt"
    want = O.fused_reference(a, b, c, bias, relu_on_c=True, relu_on_d=True, add_a=0.5,
                             add_b=-0.25)
    assert np.array_equal(d.reshape((m, n), order="F"), want)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("case", [(256, 256, 256, False, False), (200, 136, 72, True, False),
                                  (384, 136, 264, False, True), (136, 640, 48, True, True)])
def test_simt_dense_fast_path_bitwise(cuda, dtype, case):
    """The reference's default dtypes (build_dense_config(..., np.float32 / np.float64)) on the
    exact lane's direct-load tiled kernel: bitwise equal to the oracle (reference order, separate
    mul / add roundings) with tails in every dimension and transposed operands."""
    m, n, k, ta, tb = case
    rng = np.random.default_rng(8)
    a = rng.standard_normal((m, k)).astype(dtype)
    b = rng.standard_normal((k, n)).astype(dtype)
    c = rng.standard_normal((m, n)).astype(dtype)
    cfg = tk.build_dense_config(m, n, k, dtype, trans_a=ta, trans_b=tb)
    d = np.zeros(m * n, dtype)
    ab = (a.T if ta else a).ravel(order="F")
    bb = (b.T if tb else b).ravel(order="F")
    tk.matmul(cfg, ab, bb, c.ravel(order="F"), d)
    assert tk.last_run()["lane"] == "simt"
    want = O.gemm_real(a, b, c)
    assert np.array_equal(d.reshape((m, n), order="F"), want)


def test_simt_complex_dual_bitwise(cuda):
    m, n, k = 40, 24, 32
    rng = np.random.default_rng(8)
    mk = lambda s: np.asfortranarray((rng.standard_normal(s) + 1j * rng.standard_normal(s))
                                     .astype(np.complex64))
    a, b, c = mk((m, k)), mk((k, n)), mk((m, n))
    cfg = tk.build_complex_config(m, n, k, np.complex64)
    d = np.zeros(m * n, np.complex64)
    tk.matmul(cfg, a.ravel(order="F").view(np.float32), b.ravel(order="F").view(np.float32),
              c.ravel(order="F").view(np.float32), d.view(np.float32))
    assert np.array_equal(d.reshape((m, n), order="F"), O.gemm_pair(a, b, c))
    ints = lambda s: rng.integers(-4, 5, s).astype(np.float64)
    a = np.asfortranarray(tk.dual_array(ints((m, k)), ints((m, k))))
    b = np.asfortranarray(tk.dual_array(ints((k, n)), ints((k, n))))
    c = np.asfortranarray(tk.dual_array(ints((m, n)), ints((m, n))))
    cfg = tk.build_dual_config(m, n, k)
    d = np.zeros(m * n, tk.DUAL64)
    tk.matmul(cfg, a.ravel(order="F").view(np.float64), b.ravel(order="F").view(np.float64),
              c.ravel(order="F").view(np.float64), d.view(np.float64))
    assert np.array_equal(d.reshape((m, n), order="F"), O.gemm_pair(a, b, c, dual=True))


@pytest.mark.parametrize("shape", [(64, 32, 2048, 256), (8, 4, 256, 64), (16, 128, 512, 1024)])
def test_tensor_contraction_tcgen05(cuda, shape):
    """D[a,b,c] = sum_d A[b,d,a] B[d,c] on the tensor cores (A's M digits permuted once)."""
    na, nb, nc, nd = shape
    rng = np.random.default_rng(9)
    a = rng.standard_normal((nb, nd, na)).astype(np.float16)
    b = rng.standard_normal((nd, nc)).astype(np.float16)
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    d, counters = tk.contract(ta, tb)
    assert tk.last_run()["lane"] == "tcgen05"
    want = O.tc_reference(a.astype(np.float32), b.astype(np.float32))
    assert O.rel_err(d.cpu().numpy(), want) <= O.tolerance(nd)
    assert counters.global_stores == na * nb * nc


@pytest.mark.parametrize("spec,sizes,packs", [
    # A MN-major with two M and two K digits read in place; B's contiguous digit is a second N
    # digit, so B is packed
    ("abcd-aebf-dfce", dict(a=128, b=4, c=128, d=64, e=64, f=5), 1),
    # A K-major (K contiguous) with two M and two K digits, interleaved in memory; B plain
    ("abc-daeb-dec", dict(a=128, b=4, c=256, d=64, e=5), 0),
    # B MN-major with two N digits around the K digit (256-wide and 128-wide pair tiles)
    ("abc-ad-bdc", dict(a=512, b=128, c=4, d=320), 0),
    ("abc-ad-bdc", dict(a=256, b=128, c=2, d=320), 0),
])
def test_gett_tma_gather(cuda, spec, sizes, packs, knob):
    """Digit-mapped operands read in place through 5-D TMA maps (no pack pass): bitwise equal
    on integer inputs to the oracle and to the packed path (TK_GATHER=0), with the expected
    number of pack launches."""
    rng = np.random.default_rng(19)
    d_idx, a_idx, b_idx = spec.split("-")
    a = _half(rng, [sizes[i] for i in a_idx], np.float16, True)
    b = _half(rng, [sizes[i] for i in b_idx], np.float16, True)
    fa = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).cuda()
    fb = torch.from_numpy(np.asfortranarray(b).ravel(order="F")).cuda()
    cfg = tk.build_gett_config(spec, sizes, np.float16)
    d_size = int(np.prod([sizes[i] for i in d_idx]))
    want = O.gett_reference(spec, _f32(a), _f32(b))
    outs = {}
    for gather in ("1", "0"):
        knob("TK_GATHER", gather)
        d = torch.zeros(d_size, dtype=torch.float32, device=cuda)
        tk.matmul(cfg, fa, fb, torch.empty(0, dtype=torch.float32, device=cuda), d)
        run = tk.last_run()
        # (packed operands may take the on-chip split-K kernel: a single-wave shape)
        assert run["lane"] == "tcgen05" and run["plan"]["kernel"] in ("pair", "ksplit"), run
        assert gather == "0" or run["plan"]["kernel"] == "pair", run
        outs[gather] = (d.cpu().numpy().reshape(want.shape, order="F"), run["launches"])
    assert outs["1"][1] == 1 + packs, outs["1"][1]
    assert outs["0"][1] > outs["1"][1], (outs["0"][1], outs["1"][1])
    assert np.array_equal(outs["1"][0], want), float(np.abs(outs["1"][0] - want).max())
    assert np.array_equal(outs["1"][0], outs["0"][0])


@pytest.mark.parametrize("spec,sizes", [
    ("abcd-aebf-dfce", dict(a=32, b=8, c=16, d=24, e=16, f=24)),   # A, B gathered; D dense
    ("abc-acd-db", dict(a=64, b=96, c=8, d=136)),                 # A gathered, B TMA, D dense
    ("ab-cad-dcb", dict(a=160, b=200, c=4, d=36)),                # 2-digit K in both operands
    ("bac-abd-dc", dict(a=24, b=16, c=72, d=200)),                # D scattered (generic epilogue)
    # rank-5 maps: five M digits, four K digits, three N digits, interleaved in every tensor
    ("axbyczde-fabgchdie-xhzfigy", dict(a=4, b=8, c=4, d=2, e=4, f=4, g=8, h=4, i=8, x=8, y=16, z=8)),
])
@pytest.mark.parametrize("integer", [True, False])
def test_gett_tcgen05(cuda, spec, sizes, integer):
    """General GETT on the tensor cores: non-TMA operands are packed once into dense
    workspaces (pack_half_kernel), D leaves through the epilogue's digit maps."""
    rng = np.random.default_rng(13)
    d_idx, a_idx, b_idx = spec.split("-")
    a = _half(rng, [sizes[i] for i in a_idx], np.float16, integer)
    b = _half(rng, [sizes[i] for i in b_idx], np.float16, integer)
    d, counters = tk.gett(spec, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert tk.last_run()["lane"] == "tcgen05", tk.last_run()
    want = O.gett_reference(spec, _f32(a), _f32(b))
    got = d.cpu().numpy()
    assert got.shape == want.shape
    k = int(np.prod([sizes[i] for i in a_idx if i in b_idx]))
    if integer:
        assert np.array_equal(got, want), float(np.abs(got - want).max())
    else:
        assert O.rel_err(got, want) <= O.tolerance(k), O.rel_err(got, want)
    assert counters.global_stores == got.size


@pytest.mark.parametrize("trans_a", [0, 1])
def test_gemm_ex_raw_host_pipelined(cuda, trans_a):
    """Host-buffer tk_gemm_ex_raw above 2^30 MACs takes the 3-stream slab pipeline."""
    m, n, k = 512, 4096 + 256, 512
    rng = np.random.default_rng(10)
    a = np.asfortranarray(rng.standard_normal((k, m) if trans_a else (m, k)).astype(np.float16))
    b = np.asfortranarray(rng.standard_normal((k, n)).astype(np.float16))
    c = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    op_a = _f32(a).T if trans_a else _f32(a)
    want = O.exact_gemm(op_a, _f32(b), c, alpha=1.25, beta=-0.5)
    st = tk.gemm_ex_raw(tk.TAG_F16F32, trans_a, 0, m, n, k, 1.25, 0.0, a.ctypes.data,
                        b.ctypes.data, -0.5, 0.0, c.ctypes.data)
    assert st == 0, tk._lib.last_error()
    assert O.rel_err(c, want) <= O.tolerance(k)


def test_cuda_graph_capture(cuda):
    """gemm_execute launches are stream-ordered and capture into a CUDA graph."""
    m = n = k = 512
    rng = np.random.default_rng(11)
    a = _dev(rng.integers(-4, 5, (m, k)).astype(np.float16))
    b = _dev(rng.integers(-4, 5, (k, n)).astype(np.float16))
    c = _dev(rng.integers(-4, 5, (m, n)).astype(np.float32))
    d = torch.zeros(m * n, device=cuda)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    tk.matmul(cfg, a, b, c, d)                      # warm: plan cached, attributes set
    want = d.clone()
    d.zero_()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tk.matmul(cfg, a, b, c, d, synchronize=False)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(d, want)
