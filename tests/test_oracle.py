"""The oracle (C restatement of the reference arithmetic) reproduces the reference's own
outputs bit for bit.  tests/golden/*.npz were produced by running the reference package
(oracle/make_golden.py); nothing here needs a GPU."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return json.loads(str(z["meta"])), z


@pytest.mark.parametrize("tag", ["nn", "nt", "tn", "tt"])
def test_dense_f32_bitwise(tag):
    meta, z = load(f"dense_f32_{tag}")
    got = O.gemm_real(z["a"], z["b"], z["c"])
    assert np.array_equal(got, z["d"])


def test_dense_f16valued_bitwise():
    _, z = load("dense_f16valued")
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"]), z["d"])


def test_c1_default_tiling_bitwise():
    """BASELINE C1: 256^3 fp16-valued at the reference's default tiling (256, 256, 8)."""
    meta, z = load("c1_dense_256")
    assert meta["block_tile"] == [256, 256, 8]
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"]), z["d"])


def test_dense_f64_integer_bitwise():
    _, z = load("dense_f64_int")
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"]), z["d"])


def test_wide_accumulation_bitwise():
    _, z = load("dense_f32_wide")
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"], mode=1), z["d"])


def test_fused_bitwise():
    meta, z = load("fused_f32")
    got = O.fused_reference(z["a"], z["b"], z["c"], z["bias"], relu_on_c=True, relu_on_d=True,
                            add_a=meta["add_a"], add_b=meta["add_b"])
    assert np.array_equal(got, z["d"])


def test_scaled_transposed_bias_m_relu_bitwise():
    meta, z = load("scaled_bias_m_relu")
    al, be = meta["alpha"], meta["beta"]
    got = O.gemm_real(z["a"].T, z["b"], z["c"], t_c=O.prog((O.T_SCALE, be / al)),
                      t_r2s=O.prog((O.T_SCALE, al)), t_s2g=O.prog((O.T_RELU, 0)),
                      bias=z["bias"], bias_axis="m")
    assert np.array_equal(got, z["d"])


def test_complex_gemm_ex_bitwise():
    meta, z = load("complex_gemm_ex")
    alpha = complex(*meta["alpha"])
    beta = complex(*meta["beta"])
    got = O.gemm_pair(z["a"], z["b"], z["c"], t_c=O.prog((O.T_SCALE, beta / alpha)),
                      t_r2s=O.prog((O.T_SCALE, alpha)))
    assert np.array_equal(got, z["d"])


@pytest.mark.parametrize("name,dual", [("complex_matmul", False), ("dual32_matmul", True),
                                       ("dual64_matmul", True)])
def test_pair_matmul_bitwise(name, dual):
    _, z = load(name)
    got = O.gemm_pair(z["a"], z["b"], z["c"], dual=dual)
    assert np.array_equal(got, z["d"])


def test_diagonal_bitwise():
    meta, z = load("diagonal")
    n = meta["n"]
    block = tuple(meta["block_tile"])
    got = O.gemm_real(np.diag(z["diag"]), z["b"], z["c"], kmask=O.diagonal_kmask(n, block),
                      block=block)
    assert np.array_equal(got, z["d"])


@pytest.mark.parametrize("shape", ["2_4_8_8", "8_4_16_16", "16_8_32_32"])
def test_tensor_contraction_bitwise(shape):
    _, z = load(f"tc_{shape}")
    assert np.array_equal(O.tc_reference(z["a"], z["b"]), z["d"])


GETT = ["abcd_aebf_dfce", "abc_acd_db", "ab_cad_dcb", "axbyczde_fabgchdie_xhzfigy"]


@pytest.mark.parametrize("spec", GETT)
def test_general_contraction_bitwise(spec):
    """General GETT (reference StridedPermutation layouts over any index permutation)."""
    meta, z = load(f"gett_{spec}")
    assert np.array_equal(O.gett_reference(meta["spec"], z["a"], z["b"]), z["d"])


def test_alpha_zero_bitwise():
    meta, z = load("alpha_zero")
    m, n, k = meta["m"], meta["n"], meta["k"]
    zeros_a = np.zeros((m, k), np.float32)
    zeros_b = np.zeros((k, n), np.float32)
    got = O.gemm_real(zeros_a, zeros_b, z["c"], t_c=O.prog((O.T_SCALE, meta["beta"])))
    assert np.array_equal(got, z["d"])


def test_gemm_ex_raw_bitwise():
    meta, z = load("gemm_ex_raw_f32")
    assert meta["status"] == 0
    al, be = meta["alpha"], meta["beta"]
    got = O.gemm_real(z["a"], z["b"], z["c"], t_c=O.prog((O.T_SCALE, be / al)),
                      t_r2s=O.prog((O.T_SCALE, al)))
    assert np.array_equal(got, z["d"])


def test_hand_cases():
    # reference test_operators.py:31-40 / test_reference.py:26-28
    a = np.array([[1, 2], [3, 4]], np.float64)
    b = np.array([[5, 6], [7, 8]], np.float64)
    assert np.array_equal(O.gemm_real(a, b, np.eye(2)), [[20, 22], [43, 51]])
    assert np.array_equal(O.gemm_real(a, b, None), [[19, 22], [43, 50]])


def test_tolerance_bound_holds_for_reference_f32():
    # the reference's own f32 path sits well inside 4 * 2^-24 * sqrt(K) of the exact product
    _, z = load("dense_f16valued")
    exact = O.exact_gemm(z["a"], z["b"], z["c"], beta=1.0)
    assert O.rel_err(z["d"], exact) <= O.tolerance(z["a"].shape[1])


def test_padded_shared_and_global_bitwise():
    """Padded shared staging and padded global buffers (reference layouts.py:132-188) change
    no arithmetic: the oracle on the logical matrices reproduces the reference's D."""
    _, z = load("padded_shared")
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"]), z["d"])
    meta, z = load("padded_global")
    m, n, pd = meta["m"], meta["n"], meta["pads"]["D"]
    dfull = z["d_buf"].reshape((m + pd, n), order="F")
    assert np.array_equal(O.gemm_real(z["a"], z["b"], z["c"]), dfull[:m])
    assert np.all(dfull[m:] == 123.0)  # padding rows never written
