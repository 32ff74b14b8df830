"""Host-side operator contract (CPU): the fragment-level ``mma`` of each operator, checked the
way the reference checks its own (`/root/reference/pkg/tests/test_operators.py:30-127`):
values against exact products and the number of real block products per invocation (4 for
complex, 3 for dual), which is the MMA count the tensor-core kernels issue per K step
(`csrc/tk_tc_gemm2c.cuh`)."""

from unittest import mock

import numpy as np
import pytest

import paper_2009_12263_b200.operators as ops
from paper_2009_12263_b200.operators import (
    DUAL64,
    ComplexOperator,
    DualNumber,
    DualOperator,
    FmaOperator,
    Fragment,
    OperatorShape,
    dual_array,
)


def _frag(role, shape, data):
    return Fragment(role, shape, np.asarray(data, dtype=np.float64))


def test_mma_2x2x2_hand_case():
    # reference test_operators.py:31-40: A@B + I with row-major A, B
    shape = OperatorShape(2, 2, 2)
    op = FmaOperator(shape, np.float64)
    d = op.mma(_frag("A", shape, [[1, 2], [3, 4]]), _frag("B", shape, [[5, 6], [7, 8]]),
               _frag("C", shape, np.eye(2)))
    assert np.array_equal(d.data, [[20, 22], [43, 51]])


def test_mma_identity_a():
    shape = OperatorShape(4, 4, 4)
    op = FmaOperator(shape, np.float64)
    b = _frag("B", shape, np.random.default_rng(0).standard_normal((4, 4)))
    d = op.mma(_frag("A", shape, np.eye(4)), b, _frag("C", shape, np.zeros((4, 4))))
    assert np.array_equal(d.data, b.data)


@pytest.mark.parametrize("extent", [4, 8, 16])
def test_mma_integers_exact(extent):
    shape = OperatorShape(extent, extent, extent)
    op = FmaOperator(shape, np.float64)
    rng = np.random.default_rng(extent)
    a, b, c = (rng.integers(-8, 9, (extent, extent)).astype(np.float64) for _ in range(3))
    d = op.mma(_frag("A", shape, a), _frag("B", shape, b), _frag("C", shape, c))
    assert np.array_equal(d.data, a @ b + c)


def test_complex_mma_invokes_exactly_four_real_products():
    shape = OperatorShape(4, 4, 4)
    op = ComplexOperator(shape, np.complex64)
    rng = np.random.default_rng(1)
    mk = lambda: (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))).astype(np.complex64)
    a, b, c = (Fragment(r, shape, mk()) for r in "ABC")
    with mock.patch.object(ops, "real_block_product", wraps=ops.real_block_product) as spy:
        op.mma(a, b, c)
    assert spy.call_count == 4 == op.products_per_invocation


def test_complex_mma_matches_composed_real_oracle():
    shape = OperatorShape(8, 8, 8)
    op = ComplexOperator(shape, np.complex64)
    rng = np.random.default_rng(2)
    mk = lambda: (rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))).astype(np.complex64)
    a, b, c = mk(), mk(), mk()
    d = op.mma(Fragment("A", shape, a), Fragment("B", shape, b), Fragment("C", shape, c))
    want = a.astype(np.complex128) @ b.astype(np.complex128) + c
    assert np.max(np.abs(d.data - want)) / np.max(np.abs(want)) < 1e-6


def test_dual_scalar_case():
    x = DualNumber(1.0, 2.0) * DualNumber(3.0, 4.0) + DualNumber(0.0, 0.0)
    assert (x.value, x.epsilon) == (3.0, 10.0)


def test_dual_mma_epsilon_is_forward_derivative():
    shape = OperatorShape(4, 4, 4)
    op = DualOperator(shape, DUAL64)
    rng = np.random.default_rng(3)
    ints = lambda: rng.integers(-4, 5, (4, 4)).astype(np.float64)
    a0, a1, b0, b1 = ints(), ints(), ints(), ints()
    d = op.mma(Fragment("A", shape, dual_array(a0, a1)), Fragment("B", shape, dual_array(b0, b1)),
               Fragment("C", shape, dual_array(np.zeros((4, 4)), np.zeros((4, 4)))))
    assert np.array_equal(d.data["value"], a0 @ b0)
    assert np.array_equal(d.data["epsilon"], a0 @ b1 + a1 @ b0)


def test_dual_mma_uses_three_real_products():
    shape = OperatorShape(2, 2, 2)
    op = DualOperator(shape)
    zeros = dual_array(np.zeros((2, 2)), np.zeros((2, 2)))
    with mock.patch.object(ops, "real_block_product", wraps=ops.real_block_product) as spy:
        op.mma(*(Fragment(r, shape, zeros.copy()) for r in "ABC"))
    assert spy.call_count == 3 == op.products_per_invocation
