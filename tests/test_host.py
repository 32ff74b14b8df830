"""Host-side logic of the B200 path (no GPU): tile algebra, layouts and their digit
lowering, params heuristic, transforms, planner lowering, analytic event counters against
the reference's own counters, error behaviour, and the C-ABI surface of libtk_sm100.so.
Cases mirror the reference test-suite (pkg/tests/test_tiling.py, test_layouts.py,
test_components.py, test_kernel.py, test_api.py)."""

import ctypes
import dataclasses
import json
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2009_12263_b200 as tk
from paper_2009_12263_b200 import _lib, components, kernel, layouts
from paper_2009_12263_b200.components import ConfigError
from paper_2009_12263_b200.tiling import Coord, Tile, linearise, parallelise, project, translate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return json.loads(str(z["meta"])), z


# ---- tiling (reference test_tiling.py) ------------------------------------------------------

def test_linearise_goldens():
    assert linearise(Coord.of(M=3, N=2), Coord.of(M=8, N=4)) == 19
    assert linearise(Coord.of(M=1, N=2, K=1), Coord.of(M=4, N=4, K=4)) == 1 + 2 * 4 + 16
    assert linearise(Coord.of(M=5, N=8), Coord.of(M=8, N=16)) == 69


def test_parallelise_paper_example():
    parent = Tile.of(M=4, N=4)
    seen = []
    for e in range(8):
        tiles = list(parallelise(parent, Coord.of(M=1, N=2), e, 8))
        assert len(tiles) == 1
        seen.append(tiles[0].absolute.values)
    assert sorted(seen) == sorted((m, n) for n in (0, 2) for m in range(4))
    # column-major rank order i + k*count
    assert seen[0] == (0, 0) and seen[1] == (1, 0) and seen[4] == (0, 2)


def test_parallelise_partition_and_base_offset():
    parent = Tile.of(M=128, N=128)
    covered = set()
    for e in range(8):
        it = parallelise(parent, Coord.of(M=64, N=32), e, 8)
        first = None
        for t in it:
            covered.add(t.absolute.values)
            if first is None:
                first = t.base
            assert t.base == first  # entity-dependent part stays in base
    assert len(covered) == (128 // 64) * (128 // 32)


def test_parallelise_rejects_non_divisible():
    with pytest.raises(ValueError, match="zero-pad"):
        parallelise(Tile.of(M=10, N=8), Coord.of(M=4, N=8), 0, 1)
    with pytest.raises(ValueError, match="evenly"):
        parallelise(Tile.of(M=8, N=8), Coord.of(M=4, N=4), 0, 3)


def test_project_translate():
    t = Tile.of(M=4, N=5, K=6)
    p = project(translate(t, Coord.of(M=1, N=2, K=3)), ("K", "M"))
    assert p.names == ("K", "M") and p.absolute.values == (3, 1) and p.size.values == (6, 4)


# ---- layouts (reference test_layouts.py) -----------------------------------------------------

def test_physical_sizes_and_padded_index():
    inner = layouts.ColMajor(np.float32, ("M", "K"), (128, 16))
    pad = layouts.Padded(inner, 8)
    assert pad.physical_size() == 2176
    buf = np.arange(pad.physical_size(), dtype=np.float32)
    tile = Tile(Coord.of(M=0, K=1), Coord.of(M=0, K=0), Coord.of(M=1, K=1))
    assert pad.load(buf, tile)[0] == 136  # (0,1) -> 1 * (128 + 8)
    assert pad.lower().digits == (((128, 1),), ((16, 136),))


@pytest.mark.parametrize("make", [
    lambda: layouts.ColMajor(np.float32, ("M", "K"), (8, 6)),
    lambda: layouts.RowMajor(np.float32, ("M", "K"), (8, 6)),
    lambda: layouts.Padded(layouts.ColMajor(np.float32, ("M", "K"), (8, 6)), 3),
    lambda: layouts.InterleavedComplex(np.complex64, ("M", "K"), (8, 6)),
    lambda: layouts.SplitComplex(np.complex64, ("M", "K"), (8, 6)),
    lambda: layouts.SplitComplex(tk.DUAL64, ("M", "K"), (8, 6), order="C"),
    lambda: layouts.StridedPermutation.pure(np.float32, ("M", "K"), (8, 6), ("K", "M")),
])
def test_layout_round_trip(make):
    lay = make()
    rng = np.random.default_rng(0)
    buf = np.zeros(lay.physical_size(), dtype=lay.storage_dtype)
    full = Tile.of(M=8, K=6)
    if lay.element_type.kind == "c":
        vals = (rng.standard_normal(48) + 1j * rng.standard_normal(48)).astype(lay.element_type)
    elif lay.element_type.names:
        vals = tk.dual_array(rng.standard_normal(48), rng.standard_normal(48), lay.element_type)
    else:
        vals = rng.standard_normal(48).astype(lay.element_type)
    lay.store(buf, full, vals)
    assert np.array_equal(lay.load(buf, full), vals)
    sub = Tile(Coord.of(M=2, K=1), Coord.of(M=1, K=2), Coord.of(M=4, K=2))
    assert np.array_equal(lay.load(buf, sub),
                          vals.reshape(8, 6, order="F")[3:7, 3:5].ravel(order="F"))


def test_interleaved_vs_split_images():
    vals = np.array([1 + 2j, 3 + 4j, 5 + 6j, 7 + 8j], np.complex64)
    full = Tile.of(M=2, K=2)
    il = layouts.InterleavedComplex(np.complex64, ("M", "K"), (2, 2))
    sp = layouts.SplitComplex(np.complex64, ("M", "K"), (2, 2))
    b1 = np.zeros(8, np.float32)
    b2 = np.zeros(8, np.float32)
    il.store(b1, full, vals)
    sp.store(b2, full, vals)
    assert b1.tolist() == [1, 2, 3, 4, 5, 6, 7, 8]
    assert b2.tolist() == [1, 3, 5, 7, 2, 4, 6, 8]
    assert il.lower().pair == layouts.PAIR_INTERLEAVED and sp.lower().plane_stride == 4


def test_dual_interleave_image():
    vals = tk.dual_array([1.0, 2.0], [10.0, 20.0])
    lay = layouts.InterleavedComplex(tk.DUAL64, ("M", "K"), (2, 1))
    buf = np.zeros(4)
    lay.store(buf, Tile.of(M=2, K=1), vals)
    assert buf.tolist() == [1, 10, 2, 20]


def test_diagonal_and_zero_layouts():
    d = layouts.Diagonal(np.float32, ("M", "K"), (4, 4))
    buf = np.array([1, 2, 3, 4], np.float32)
    tile = Tile(Coord.of(M=0, K=2), Coord.of(M=0, K=0), Coord.of(M=4, K=2))
    assert d.load_count(tile) == 2
    assert d.load(buf, tile).reshape(4, 2, order="F").tolist() == [[0, 0], [0, 0], [3, 0], [0, 4]]
    with pytest.raises(ValueError, match="off-diagonal"):
        d.store(buf, Tile.of(M=2, K=2), np.ones(4))
    z = layouts.Zero(np.float32, ("M", "N"), (4, 4))
    assert z.physical_size() == 0 and z.load_count(Tile.of(M=4, N=4)) == 0
    assert d.lower().kind == layouts.KIND_DIAGONAL and z.lower().kind == layouts.KIND_ZERO


def test_strided_permutation_index_and_digits():
    # (M, K) view over a (b, d, a) tensor: reference test_layouts.py:200-206 style
    lay = layouts.StridedPermutation(np.float32, ("M", "K"), (6, 4),
                                     dim_map={"M": (("b", 2), ("a", 3)), "K": (("d", 4),)},
                                     storage_order=("b", "d", "a"))
    assert lay.digits() == [[(2, 1), (3, 8)], [(4, 2)]]
    t = Tile(Coord.of(M=1, K=2), Coord.of(M=0, K=0), Coord.of(M=1, K=1))
    assert lay._flat_indices(t)[0] == 1 + 2 * 2  # b=1, a=0, d=2
    rng = np.random.default_rng(1)
    buf = rng.standard_normal(24).astype(np.float32)
    eager = buf.reshape(2, 4, 3, order="F").transpose(0, 2, 1).reshape(6, 4, order="F")
    assert np.array_equal(lay.load(buf, Tile.of(M=6, K=4)), eager.ravel(order="F"))


# ---- components (reference test_components.py) ---------------------------------------------

def _params_config(m, n, k, dtype=np.float32, **kw):
    return tk.build_dense_config(m, n, k, dtype, **kw)


def test_heuristic_matches_reference_goldens():
    data = json.load(open(os.path.join(GOLDEN, "host_logic.json")))
    for case in data["tilings"]:
        dt = np.float32 if case["dtype"] == "f32" else np.float64
        opshape = tuple(case["operator_shape"])
        cfg = _params_config(case["m"], case["n"], case["k"], dt,
                             block_tile=tuple(case["block"]) if case["block"] else None,
                             operator_shape=opshape)
        if case["budget"] is not None:
            cfg = dataclasses.replace(cfg, params=dataclasses.replace(
                cfg.params, scratch_budget=case["budget"]))
        assert list(kernel.resolve_config(cfg).params.block_tile) == case["resolved_block"], case


def test_heuristic_golden_128_16():
    cfg = _params_config(128, 128, 128, operator_shape=(8, 8, 16))
    cfg = dataclasses.replace(cfg, params=dataclasses.replace(
        cfg.params, scratch_budget=(128 * 16 + 16 * 128) * 4))
    assert kernel.resolve_config(cfg).params.block_tile == (128, 128, 16)


def test_heuristic_half_storage_doubles_the_tile_budget():
    # fp16 staging is half the bytes of f32: the same 64 KiB budget admits a larger tile
    f32 = kernel.resolve_config(_params_config(1024, 1024, 1024)).params.block_tile
    f16 = kernel.resolve_config(_params_config(1024, 1024, 1024, np.float16)).params.block_tile
    assert f32 == (1024, 1024, 8) and f16 == (1024, 1024, 8)
    small = kernel.resolve_config(_params_config(512, 512, 64, np.float16,
                                                 operator_shape=(8, 8, 32))).params.block_tile
    assert small == (512, 512, 32)


@pytest.mark.parametrize("kw,match", [
    (dict(block_tile=(24, 32, 8)), "block tile must divide"),
    (dict(block_tile=(32, 32, 8), compute_warp=(24, 16)), "compute warp must divide"),
    (dict(block_tile=(32, 32, 8), compute_warp=(16, 16), workers_per_block=3), "dealt evenly"),
])
def test_param_errors(kw, match):
    with pytest.raises(ConfigError, match=match):
        kernel.resolve_config(_params_config(64, 64, 64, **kw))


def test_k_not_divisible_and_budget_errors():
    with pytest.raises(ConfigError, match="zero-pad"):
        kernel.resolve_config(_params_config(64, 64, 60))
    cfg = _params_config(64, 64, 64)
    cfg = dataclasses.replace(cfg, params=dataclasses.replace(cfg.params, scratch_budget=16))
    with pytest.raises(ConfigError, match="budget"):
        kernel.resolve_config(cfg)


def test_transform_functors_keep_numpy_semantics():
    v = np.array([-1.5, 0.0, 2.0], np.float32)
    assert components.relu(v).tolist() == [0, 0, 2]
    assert components.add_constant(np.float32(0.5))(v).dtype == np.float32
    comp = components.compose(components.scale(2.0), components.add_constant(1.0),
                              components.relu)
    assert comp(v).tolist() == [0.0, 1.0, 5.0]
    assert [op[0] for op in comp.program()] == [components.T_SCALE, components.T_ADD,
                                                components.T_RELU]
    d = tk.dual_array([1.0, 2.0], [3.0, 4.0])
    s = components.scale(2.0)(d)
    assert s["value"].tolist() == [2, 4] and s["epsilon"].tolist() == [6, 8]
    with pytest.raises(ValueError, match="element count"):
        components.apply_transform(lambda x: x[:1], v)


def test_bias_epilogue_host_semantics():
    # reference test_components.py:186-191: out[i, j] = scratch[i, j] + bias[j]
    sl = layouts.ColMajor(np.float32, ("M", "N"), (2, 2))
    out = layouts.ColMajor(np.float32, ("M", "N"), (2, 2))
    scratch = np.array([1, 3, 2, 4], np.float32)
    dst = np.zeros(4, np.float32)
    cnt = components.run_epilogue(components.BiasEpilogue(np.array([10, 20], np.float32)), sl,
                                  scratch, out, dst, Tile.of(M=2, N=2), Tile.of(M=2, N=2))
    assert dst.reshape(2, 2, order="F").tolist() == [[11, 22], [13, 24]]
    assert cnt.global_loads == 2 and cnt.global_stores == 4


def test_diagonal_predicate():
    p = components.DiagonalPredicate()
    t = lambda m, k: Tile(Coord.of(M=m, N=0, K=k), Coord.of(M=0, N=0, K=0),
                          Coord.of(M=16, N=16, K=8))
    assert p(t(0, 8)) and p(t(16, 24)) and not p(t(0, 16)) and not p(t(32, 8))


# ---- planner / counters against the reference's own counters ------------------------------

def _golden_config(name):
    meta, z = golden(name)
    m, n, k = meta.get("m"), meta.get("n"), meta.get("k")
    bt = tuple(meta["block_tile"]) if "block_tile" in meta else None
    if name.startswith("dense_f32_") and name[-2:] in ("nn", "nt", "tn", "tt"):
        return meta, tk.build_dense_config(m, n, k, np.float32, trans_a=meta["trans_a"],
                                           trans_b=meta["trans_b"], operator_shape=(8, 8, 8))
    if name == "dense_f16valued":
        return meta, tk.build_dense_config(m, n, k, np.float16)
    if name == "dense_f64_int":
        return meta, tk.build_dense_config(m, n, k, np.float64, block_tile=bt)
    if name == "dense_f32_wide":
        return meta, tk.build_dense_config(m, n, k, np.float32, wide_accumulate=True,
                                           block_tile=bt)
    if name == "fused_f32":
        return meta, tk.build_fused_config(m, n, k, np.float32, bias=z["bias"], relu_on_c=True,
                                           relu_on_d=True, add_a=0.5, add_b=-0.25, block_tile=bt)
    if name == "complex_matmul":
        return meta, tk.build_complex_config(m, n, k, np.complex64, block_tile=bt)
    if name == "dual32_matmul":
        return meta, tk.build_dual_config(m, n, k, tk.DUAL32, block_tile=bt)
    if name == "diagonal":
        return meta, tk.build_diagonal_config(meta["n"], np.float32, block_tile=bt)
    if name.startswith("tc_"):
        return meta, tk.build_tc_config(meta["na"], meta["nb"], meta["nc"], meta["nd"],
                                        np.float32)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["dense_f32_nn", "dense_f32_tt", "dense_f16valued",
                                  "dense_f64_int", "dense_f32_wide", "fused_f32",
                                  "complex_matmul", "dual32_matmul", "diagonal", "tc_2_4_8_8",
                                  "tc_16_8_32_32"])
def test_counters_equal_reference(name):
    meta, cfg = _golden_config(name)
    res = kernel.resolve_config(cfg)
    if "block_tile" in meta:
        assert list(res.params.block_tile) == meta["block_tile"]
    _, _, executed = kernel.lower(res)
    got = dataclasses.asdict(kernel._counters(res, executed))
    assert got == meta["counters"]


def test_operator_invocation_count_128():
    cfg = kernel.resolve_config(tk.build_dense_config(128, 128, 128, np.float32,
                                                      block_tile=(64, 64, 16)))
    _, _, ex = kernel.lower(cfg)
    assert kernel._counters(cfg, ex).operator_invocations == 4096


def test_generic_predicate_mask():
    cfg = tk.build_dense_config(64, 64, 64, np.float32, block_tile=(32, 32, 16))
    cfg = dataclasses.replace(cfg, predicate=lambda t: t.absolute["K"] < 32)
    plan, mask, ex = kernel.lower(kernel.resolve_config(cfg))
    assert plan.predicate == _lib.PRED_MASK
    assert mask.shape == (4, 4) and mask[:, :2].all() and not mask[:, 2:].any()
    always = dataclasses.replace(cfg, predicate=lambda t: True)
    plan, mask, _ = kernel.lower(kernel.resolve_config(always))
    assert plan.predicate == _lib.PRED_ALWAYS and mask is None


def test_lowering_of_layouts_and_transforms():
    cfg = kernel.resolve_config(tk.build_fused_config(256, 128, 64, np.float16,
                                                      bias=np.ones(128), add_a=0.5,
                                                      relu_on_c=True, trans_a=True))
    plan, _, _ = kernel.lower(cfg)
    assert plan.a.scalar == 0 and plan.c.scalar == 2
    assert (plan.a.stride[0][0], plan.a.stride[1][0]) == (64, 1)       # row-major A
    assert (plan.b.stride[0][0], plan.b.stride[1][0]) == (1, 64)       # column-major B
    assert plan.t_a.n == 1 and plan.t_a.op[0] == components.T_ADD and plan.t_a.re[0] == 0.5
    assert plan.t_c.op[0] == components.T_RELU and plan.bias_axis == 1


def test_planner_rejects_what_cannot_run_on_device():
    cfg = tk.build_dense_config(64, 64, 64, np.float32, block_tile=(32, 32, 8))
    with pytest.raises(ConfigError, match="arbitrary Python callable"):
        kernel.lower(kernel.resolve_config(dataclasses.replace(cfg,
                                                               transform_g2s_a=lambda v: v * 2)))

    class Custom(tk.api.FmaOperator):
        def mma(self, a, b, c):
            return c

    with pytest.raises(ConfigError, match="overrides mma"):
        kernel.lower(kernel.resolve_config(dataclasses.replace(
            cfg, operator=Custom(tk.OperatorShape(8, 8, 8), np.float32))))


def test_validation_before_any_write():
    cfg = tk.build_dense_config(32, 32, 32, np.float32, block_tile=(16, 16, 8))
    a = np.zeros(32 * 32, np.float32)
    d = np.full(32 * 32, 7.0, np.float32)
    with pytest.raises(ValueError, match="buffer"):
        tk.gemm_execute(cfg, a[:-1], a, a, d)
    with pytest.raises(ConfigError, match="dtype"):
        tk.gemm_execute(cfg, a.astype(np.float64), a, a, d)
    bad = dataclasses.replace(cfg, operator=tk.api.FmaOperator(tk.OperatorShape(4, 4, 4),
                                                               np.float32))
    with pytest.raises(ConfigError, match="disagrees"):
        tk.gemm_execute(bad, a, a, a, d)
    assert np.all(d == 7.0)


def test_gemm_ex_type_errors():
    with pytest.raises(ConfigError, match="supported"):
        tk.gemm_ex(False, False, 1.0, np.zeros((8, 8), np.float32), np.zeros((8, 8)),
                   0.0, np.zeros((8, 8), np.float32))
    with pytest.raises(ConfigError, match="supported"):
        a = np.zeros((8, 8), np.int32)
        tk.gemm_ex(False, False, 1.0, a, a, 0.0, a)


# ---- the C ABI ---------------------------------------------------------------------------

def _header_symbols():
    text = open(os.path.join(ROOT, "include", "tk_sm100.h")).read()
    return set(re.findall(r"^\w[\w\s\*]*?\b(tk_\w+)\s*\(", text, flags=re.M))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert syms == set(_lib.EXPORTED)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.tk_abi_version() == _lib.ABI_VERSION


def test_struct_layout_matches_header():
    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "tk_sm100.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(TkLayout), sizeof(TkTransform),
         sizeof(TkGemmPlan), offsetof(TkGemmPlan, a), offsetof(TkGemmPlan, t_a),
         offsetof(TkGemmPlan, bias_axis), offsetof(TkLayout, ext), offsetof(TkTransform, re));
  return 0;
}'''
    tmp = "/tmp/tk_layout_check"
    with open(tmp + ".c", "w") as f:
        f.write(src)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", tmp, tmp + ".c"],
                   check=True)
    got = [int(x) for x in subprocess.run([tmp], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.TkLayout), ctypes.sizeof(_lib.TkTransform),
            ctypes.sizeof(_lib.TkGemmPlan), _lib.TkGemmPlan.a.offset, _lib.TkGemmPlan.t_a.offset,
            _lib.TkGemmPlan.bias_axis.offset, _lib.TkLayout.ext.offset, _lib.TkTransform.re.offset]
    assert got == want


@pytest.mark.parametrize("dtype,lane", [(np.float16, "tcgen05"), ("bf16", "tcgen05"),
                                        (np.float32, "simt"), (np.float64, "simt")])
def test_lane_selection_is_host_logic(dtype, lane):
    dt = tk.BFLOAT16 if dtype == "bf16" else dtype
    plan, _, _ = kernel.lower(kernel.resolve_config(tk.build_dense_config(256, 256, 256, dt)))
    assert kernel.plan_lane(plan) == lane


def test_lane_selection_variants():
    lanes = {}
    for name, cfg in {
        "complex16": tk.build_complex_config(128, 128, 64, tk.COMPLEX32),
        "complex16_split": tk.build_complex_config(128, 128, 64, tk.COMPLEX32, split=True),
        "dual16": tk.build_dual_config(128, 128, 64, tk.DUAL16),
        "diag16": tk.build_diagonal_config(512, np.float16),
        "fused16": tk.build_fused_config(256, 256, 64, np.float16, bias=np.ones(256),
                                         add_a=0.5, relu_on_c=True),
        "complex64": tk.build_complex_config(64, 64, 64, np.complex64),
        "tc16": tk.build_tc_config(64, 32, 128, 64, np.float16),
    }.items():
        lanes[name] = kernel.plan_lane(kernel.lower(kernel.resolve_config(cfg))[0])
    assert lanes == {"complex16": "tcgen05", "complex16_split": "tcgen05", "dual16": "tcgen05",
                     "diag16": "tcgen05", "fused16": "tcgen05", "complex64": "simt",
                     "tc16": "tcgen05"}
    # any A/B load transform runs on the tensor cores through the transform pass (fp16: hi +
    # lo planes when the result is not exact in fp16) ...
    prog = components.compose(components.scale(0.3), components.relu, components.add_constant(0.1))
    for t in (components.relu, prog):
        cfg = dataclasses.replace(tk.build_dense_config(256, 256, 64, np.float16),
                                  transform_g2s_a=t, transform_g2s_b=components.relu)
        assert kernel.plan_lane(kernel.lower(kernel.resolve_config(cfg))[0]) == "tcgen05"
    # ... bf16 only when the result is exact in bf16 (else it would need three planes)
    for t, lane in ((components.relu, "tcgen05"), (prog, "simt")):
        cfg = dataclasses.replace(tk.build_dense_config(256, 256, 64, tk.BFLOAT16), transform_g2s_b=t)
        assert kernel.plan_lane(kernel.lower(kernel.resolve_config(cfg))[0]) == lane
    with tk.force_lane("simt"):
        plan, _, _ = kernel.lower(kernel.resolve_config(tk.build_dense_config(256, 256, 64,
                                                                              np.float16)))
        assert kernel.plan_lane(plan) == "simt"


def test_gemm_ex_raw_config_errors_need_no_device():
    a = np.zeros((8, 8), np.float32, order="F")
    assert tk.gemm_ex_raw(99, 0, 0, 8, 8, 8, 1.0, 0.0, a.ctypes.data, a.ctypes.data, 0.0, 0.0,
                          a.ctypes.data) == 1
    bad = np.zeros((8, 3), np.float32, order="F")
    assert tk.gemm_ex_raw(tk.TAG_F32, 0, 0, 8, 8, 3, 1.0, 0.0, bad.ctypes.data, bad.ctypes.data,
                          0.0, 0.0, a.ctypes.data) == 1
    assert "block tile" in _lib.last_error() or "feasible" in _lib.last_error()


def test_gemm_ex_cfunc_is_a_c_function_pointer():
    fn = tk.gemm_ex_cfunc()
    assert isinstance(fn, tk.GEMM_EX_CFUNC)
    assert ctypes.cast(fn, ctypes.c_void_p).value == \
        ctypes.cast(_lib.load().tk_gemm_ex_raw, ctypes.c_void_p).value


def test_gett_config_wiring():
    """build_gett_config: M = A-free indices in D order, N = B-free in D order, K = contracted
    in A order; the reference's build_tc_config is the special case 'abc-bda-dc'."""
    import paper_2009_12263_b200 as tk

    cfg = tk.build_gett_config("abcd-aebf-dfce", dict(a=8, b=4, c=6, d=2, e=3, f=5), np.float16)
    assert cfg.params.gemm_shape == (32, 12, 15)
    assert cfg.global_a_layout.digits() == [[(8, 1), (4, 24)], [(3, 8), (5, 96)]]
    tc = tk.build_gett_config("abc-bda-dc", dict(a=8, b=4, c=6, d=2), np.float32)
    ref = tk.build_tc_config(8, 4, 6, 2, np.float32)
    assert tc.params.gemm_shape == ref.params.gemm_shape
    assert tc.global_a_layout.physical_size() == ref.global_a_layout.physical_size()
    for bad in ("abc-bd", "abc-bda-dcc", "ab-abc-bc", "abe-bda-dc"):
        with pytest.raises(tk.ConfigError):
            tk.build_gett_config(bad, dict(a=2, b=2, c=2, d=2, e=2), np.float32)


@pytest.mark.parametrize("spec,sizes,packed", [
    ("abc-acd-db", dict(a=64, b=96, c=8, d=136), ()),                 # chained digits merge: no gather
    ("abc-bda-dc", dict(a=64, b=32, c=128, d=256), ("A",)),          # A's M digits out of order
    ("abcd-aebf-dfce", dict(a=32, b=8, c=16, d=24, e=16, f=24), ("A", "B")),
])
def test_gett_operand_packing_plan(spec, sizes, packed):
    """Host-side planning of a GETT on the tensor cores (no GPU needed): operands whose digit
    maps normalise to one strided matrix go straight to the TMA, the others get a dense
    gather workspace of exactly rows x cols halves."""
    cfg = kernel.resolve_config(tk.build_gett_config(spec, sizes, np.float16))
    plan, _, _ = kernel.lower(cfg)
    assert kernel.plan_lane(plan) == "tcgen05"
    m, n, k = cfg.params.gemm_shape
    want = (2 * m * k if "A" in packed else 0) + (2 * k * n if "B" in packed else 0)
    assert _lib.load().tk_workspace_bytes(plan) == want


def test_fused_allgather_entry_validates_before_launch():
    """tk_gemm_peers rejects what the fused all-gather cannot do before touching the device:
    more than 7 peers, or a D that is not one dense column-major slab."""
    lib = _lib.load()
    dense = kernel.resolve_config(tk.build_dense_config(256, 256, 256, np.float16))
    plan, _, _ = kernel.lower(dense)
    peers = (ctypes.c_void_p * 8)(*([0x1000] * 8))
    rc = lib.tk_gemm_peers(ctypes.byref(plan), None, None, None, None, None, None, None, 0, None,
                           peers, 8)
    assert rc == _lib.TK_ERR_CONFIG and "peer" in _lib.last_error()
    gett = kernel.resolve_config(tk.build_gett_config("abc-acd-db", dict(a=64, b=96, c=8, d=136),
                                                      np.float16))
    plan2, _, _ = kernel.lower(gett)
    rc = lib.tk_gemm_peers(ctypes.byref(plan2), None, None, None, None, None, None, None, 0, None,
                           peers, 1)
    assert rc == _lib.TK_ERR_CONFIG and "dense column-major" in _lib.last_error()


def test_padded_shared_builder_resolves_like_reference():
    """build_dense_config(shared_pad=4): the heuristic sees the padded staging footprint, as
    the reference's (golden made by the reference, oracle/make_golden.py padded_cases)."""
    import json
    import os

    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "padded_shared.npz"))
    meta = json.loads(str(z["meta"]))
    cfg = tk.build_dense_config(meta["m"], meta["n"], meta["k"], np.float32, shared_pad=meta["pad"])
    res = kernel.resolve_config(cfg)
    assert list(res.params.block_tile) == meta["block_tile"]
    plan, _, executed = kernel.lower(res)
    assert dataclasses.asdict(kernel._counters(res, executed)) == meta["counters"]
