"""The device lanes on the reference's own golden vectors (tests/golden, made by running the
reference package).  The CUDA-core lane must reproduce them bit for bit; the tcgen05 lane
(half storage) within 4 * 2^-24 * sqrt(K)."""

import dataclasses
import json
import os

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from oracle import oracle as O
from paper_2009_12263_b200 import components

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return json.loads(str(z["meta"])), z


def F(x):
    return np.asarray(x).ravel(order="F")


@pytest.mark.parametrize("tag", ["nn", "nt", "tn", "tt"])
def test_dense_f32_bitwise(cuda, tag):
    meta, z = load(f"dense_f32_{tag}")
    m, n, k = meta["m"], meta["n"], meta["k"]
    a, b = z["a"], z["b"]
    cfg = tk.build_dense_config(m, n, k, np.float32, trans_a=meta["trans_a"],
                                trans_b=meta["trans_b"], operator_shape=(8, 8, 8))
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, F(a.T if meta["trans_a"] else a), F(b.T if meta["trans_b"] else b),
                    F(z["c"]), d)
    assert tk.last_run()["lane"] == "simt"
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


def test_f16_valued_on_both_lanes(cuda):
    meta, z = load("dense_f16valued")
    m, n, k = meta["m"], meta["n"], meta["k"]
    a16, b16 = z["a"].astype(np.float16), z["b"].astype(np.float16)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    d = np.zeros(m * n, np.float32)
    tk.matmul(cfg, F(a16), F(b16), F(z["c"]), d)
    assert tk.last_run()["lane"] == "tcgen05"
    assert O.rel_err(d.reshape((m, n), order="F"), z["d"]) <= O.tolerance(k)
    with tk.force_lane("simt"):   # exact widening of fp16 -> bitwise the reference on f32
        d2 = np.zeros(m * n, np.float32)
        tk.matmul(cfg, F(a16), F(b16), F(z["c"]), d2)
    assert np.array_equal(d2.reshape((m, n), order="F"), z["d"])


def test_c1_default_tiling_both_lanes(cuda):
    """BASELINE C1 (256^3, default tiling (256, 256, 8), reference-generated golden): the
    tcgen05 lane on fp16 storage within 4 * 2^-24 * sqrt(K); the exact lane bitwise."""
    meta, z = load("c1_dense_256")
    m, n, k = meta["m"], meta["n"], meta["k"]
    a16, b16 = z["a"].astype(np.float16), z["b"].astype(np.float16)
    cfg = tk.build_dense_config(m, n, k, np.float16)
    assert list(tk.kernel.resolve_config(cfg).params.block_tile) == meta["block_tile"]
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, F(a16), F(b16), F(z["c"]), d)
    assert tk.last_run()["lane"] == "tcgen05"
    assert O.rel_err(d.reshape((m, n), order="F"), z["d"]) <= O.tolerance(k)
    assert dataclasses.asdict(cnt) == meta["counters"]
    with tk.force_lane("simt"):
        d2 = np.zeros(m * n, np.float32)
        tk.matmul(cfg, F(a16), F(b16), F(z["c"]), d2)
    assert np.array_equal(d2.reshape((m, n), order="F"), z["d"])


def test_f64_and_wide_bitwise(cuda):
    meta, z = load("dense_f64_int")
    m, n, k = meta["m"], meta["n"], meta["k"]
    d = np.zeros(m * n)
    tk.matmul(tk.build_dense_config(m, n, k, np.float64, block_tile=(16, 16, 8)), F(z["a"]),
              F(z["b"]), F(z["c"]), d)
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])
    meta, z = load("dense_f32_wide")
    m, n, k = meta["m"], meta["n"], meta["k"]
    d = np.zeros(m * n, np.float32)
    tk.matmul(tk.build_dense_config(m, n, k, np.float32, wide_accumulate=True,
                                    block_tile=(32, 32, 8)), F(z["a"]), F(z["b"]), F(z["c"]), d)
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])


def test_fused_bitwise(cuda):
    meta, z = load("fused_f32")
    m, n, k = meta["m"], meta["n"], meta["k"]
    cfg = tk.build_fused_config(m, n, k, np.float32, bias=z["bias"], relu_on_c=True,
                                relu_on_d=True, add_a=0.5, add_b=-0.25, block_tile=(32, 32, 16))
    d = np.zeros(m * n, np.float32)
    cnt = tk.matmul(cfg, F(z["a"]), F(z["b"]), F(z["c"]), d)
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


def test_scaled_transposed_bias_m_relu_bitwise(cuda):
    meta, z = load("scaled_bias_m_relu")
    m, n, k = meta["m"], meta["n"], meta["k"]
    al, be = meta["alpha"], meta["beta"]
    cfg = dataclasses.replace(
        tk.build_dense_config(m, n, k, np.float32, trans_a=True, block_tile=(16, 16, 8)),
        transform_g2s_c=components.scale(be / al), transform_r2s_d=components.scale(al),
        epilogue=components.BiasEpilogue(z["bias"], axis="m"), transform_s2g_d=components.relu)
    d = np.zeros(m * n, np.float32)
    tk.matmul(cfg, F(z["a"]), F(z["b"]), F(z["c"]), d)
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])


def test_complex_gemm_ex_bitwise(cuda):
    meta, z = load("complex_gemm_ex")
    c = np.asfortranarray(z["c"].copy())
    tk.gemm_ex(False, False, complex(*meta["alpha"]), np.asfortranarray(z["a"]),
               np.asfortranarray(z["b"]), complex(*meta["beta"]), c, operator_shape=(8, 8, 8))
    assert np.array_equal(c, z["d"])


@pytest.mark.parametrize("name", ["complex_matmul", "dual32_matmul", "dual64_matmul"])
def test_pair_matmul_bitwise(cuda, name):
    meta, z = load(name)
    m, n, k = meta["m"], meta["n"], meta["k"]
    dt = z["a"].dtype
    build = tk.build_complex_config if name.startswith("complex") else tk.build_dual_config
    cfg = build(m, n, k, dt, block_tile=tuple(meta["block_tile"]))
    sc = cfg.global_a_layout.storage_dtype
    d = np.zeros(m * n, dt)
    cnt = tk.matmul(cfg, F(z["a"]).view(sc), F(z["b"]).view(sc), F(z["c"]).view(sc), d.view(sc))
    assert np.array_equal(d.reshape((m, n), order="F"), z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


def test_diagonal_bitwise(cuda):
    meta, z = load("diagonal")
    n = meta["n"]
    cfg = tk.build_diagonal_config(n, np.float32, block_tile=tuple(meta["block_tile"]))
    d = np.zeros(n * n, np.float32)
    cnt = tk.matmul(cfg, z["diag"], F(z["b"]), F(z["c"]), d)
    assert np.array_equal(d.reshape((n, n), order="F"), z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


@pytest.mark.parametrize("shape", ["2_4_8_8", "8_4_16_16", "16_8_32_32"])
def test_contract_bitwise(cuda, shape):
    meta, z = load(f"tc_{shape}")
    d, cnt = tk.contract(z["a"], z["b"])
    assert np.array_equal(d, z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


@pytest.mark.parametrize("spec", ["abcd_aebf_dfce", "abc_acd_db", "ab_cad_dcb", "axbyczde_fabgchdie_xhzfigy"])
def test_gett_bitwise(cuda, spec):
    """General contractions (f32: exact lane) against the reference's own outputs, with the
    reference's counters and resolved tiling."""
    meta, z = load(f"gett_{spec}")
    d, cnt = \
        tk.gett(meta["spec"], z["a"], z["b"])
    assert np.array_equal(d, z["d"])
    assert dataclasses.asdict(cnt) == meta["counters"]


def test_alpha_zero_bitwise(cuda):
    meta, z = load("alpha_zero")
    m, n, k = meta["m"], meta["n"], meta["k"]
    c = np.asfortranarray(z["c"].copy())
    cnt = tk.gemm_ex(False, False, 0.0, np.full((m, k), np.nan, np.float32),
                     np.full((k, n), np.inf, np.float32), meta["beta"], c,
                     operator_shape=(8, 8, 8))
    assert np.array_equal(c, z["d"])
    assert cnt.global_loads == m * n


def test_gemm_ex_raw_host_pointers_bitwise(cuda):
    meta, z = load("gemm_ex_raw_f32")
    m, n, k = meta["m"], meta["n"], meta["k"]
    a, b = np.asfortranarray(z["a"]), np.asfortranarray(z["b"])
    c = np.asfortranarray(z["c"].copy())
    st = tk.gemm_ex_raw(tk.TAG_F32, 0, 0, m, n, k, meta["alpha"], 0.0, a.ctypes.data,
                        b.ctypes.data, meta["beta"], 0.0, c.ctypes.data)
    assert st == 0
    assert np.array_equal(c, z["d"])


def _padded_cfg(m, n, k, dt, pads):
    L = tk.layouts
    return dataclasses.replace(
        tk.build_dense_config(m, n, k, dt),
        global_a_layout=L.Padded(L.ColMajor(dt, ("M", "K"), (m, k)), pads["A"]),
        global_b_layout=L.Padded(L.ColMajor(dt, ("K", "N"), (k, n)), pads["B"]),
        global_c_layout=L.Padded(L.ColMajor(np.float32, ("M", "N"), (m, n)), pads["C"]),
        global_d_layout=L.Padded(L.ColMajor(np.float32, ("M", "N"), (m, n)), pads["D"]))


def _pad_buf(x, p, dt):
    buf = np.full((x.shape[0] + p, x.shape[1]), -7.0, dt)
    buf[:x.shape[0]] = x
    return buf.ravel(order="F")


@pytest.mark.parametrize("lane", ["tcgen05", "simt"])
def test_padded_global_layouts(cuda, lane):
    """Padded global A / B / C / D (pads 8 / 3 / 4 / 5: A and C stay TMA-addressable, B is
    gathered, D leaves through the register epilogue) against the reference's own run
    (tests/golden/padded_global.npz): the padding is never read into the product nor written.
    tcgen05 on fp16 storage within 4 * 2^-24 * sqrt(K); the exact lane on f32 bitwise."""
    meta, z = load("padded_global")
    m, n, k, pads = meta["m"], meta["n"], meta["k"], meta["pads"]
    dt = np.float16 if lane == "tcgen05" else np.float32
    cfg = _padded_cfg(m, n, k, dt, pads)
    dbuf = np.full((m + pads["D"]) * n, 123.0, np.float32)
    with tk.force_lane(lane):
        cnt = tk.matmul(cfg, _pad_buf(z["a"], pads["A"], dt), _pad_buf(z["b"], pads["B"], dt),
                        _pad_buf(z["c"], pads["C"], np.float32), dbuf)
    assert tk.last_run()["lane"] == lane
    full = dbuf.reshape((m + pads["D"], n), order="F")
    want = z["d_buf"].reshape((m + pads["D"], n), order="F")
    assert np.all(full[m:] == 123.0)
    if lane == "simt":
        assert np.array_equal(dbuf, z["d_buf"])
    else:
        assert O.rel_err(full[:m], want[:m]) <= O.tolerance(k)
    assert dataclasses.asdict(cnt) == meta["counters"]


@pytest.mark.parametrize("lane", ["tcgen05", "simt"])
def test_padded_shared_builder(cuda, lane):
    """build_dense_config(shared_pad=4): on the tensor cores the 128-byte TMA swizzle replaces
    the padding (same arithmetic); the exact lane bitwise the reference's D."""
    meta, z = load("padded_shared")
    m, n, k = meta["m"], meta["n"], meta["k"]
    dt = np.float16 if lane == "tcgen05" else np.float32
    cfg = tk.build_dense_config(m, n, k, dt, shared_pad=meta["pad"])
    d = np.zeros(m * n, np.float32)
    with tk.force_lane(lane):
        cnt = tk.matmul(cfg, F(z["a"].astype(dt)), F(z["b"].astype(dt)), F(z["c"]), d)
    assert tk.last_run()["lane"] == lane
    got = d.reshape((m, n), order="F")
    if lane == "simt":
        assert np.array_equal(got, z["d"])
    else:
        assert O.rel_err(got, z["d"]) <= O.tolerance(k)
    assert dataclasses.asdict(cnt) == meta["counters"]


def test_padded_fp16_integer_bitwise_large(cuda):
    """Padded fp16 operands at a multi-tile size on the CTA-pair kernel, bitwise on integers."""
    m, n, k = 1024, 1536, 1024
    pads = {"A": 8, "B": 16, "C": 4, "D": 12}
    rng = np.random.default_rng(415)
    a = rng.integers(-4, 5, (m, k)).astype(np.float16)
    b = rng.integers(-4, 5, (k, n)).astype(np.float16)
    c = rng.integers(-4, 5, (m, n)).astype(np.float32)
    cfg = _padded_cfg(m, n, k, np.float16, pads)
    dev = lambda x: torch.from_numpy(x).cuda()
    dbuf = torch.full(((m + pads["D"]) * n,), 123.0, device=cuda)
    tk.matmul(cfg, dev(_pad_buf(a, pads["A"], np.float16)), dev(_pad_buf(b, pads["B"], np.float16)),
              dev(_pad_buf(c, pads["C"], np.float32)), dbuf)
    # (a single wave: the CTA pair, or the on-chip split-K kernel built on it)
    assert tk.last_run()["lane"] == "tcgen05" and tk.last_run()["plan"]["kernel"] in ("pair", "ksplit")
    full = dbuf.cpu().numpy().reshape((m + pads["D"], n), order="F")
    assert np.all(full[m:] == 123.0)
    assert np.array_equal(full[:m], O.gemm_real(a.astype(np.float32), b.astype(np.float32), c))
