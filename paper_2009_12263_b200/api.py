"""User-facing entry points and the wiring of the shipped GEMM variants.

API parity with reference ``pkg/src/tilekit/api.py``: ``matmul`` (``api.py:37-40``),
``gemm_ex`` (``108-161``), ``gemm_ex_raw`` / ``GEMM_EX_CFUNC`` / ``gemm_ex_cfunc``
(``317-373``), the ``build_*_config`` variant builders (``166-295``) and
``contract`` (``298-312``).

Element types: everything the reference accepts (f32, f64, complex64,
complex128, DUAL32, DUAL64 -- these run on the bit-exact CUDA-core lane) plus
the tensor-core storage types float16 / bfloat16 and their complex / dual
pairs (``COMPLEX32``, ``COMPLEXBF16``, ``DUAL16``, ``DUALBF16``).  Half storage
accumulates into FP32 (C and D are float32 / complex64 / DUAL32).

``gemm_ex_raw`` keeps the reference's exact parameter list and status
convention but is the C library's own entry point (``tk_gemm_ex_raw`` in
``include/tk_sm100.h``): ``gemm_ex_cfunc()`` returns a genuine C function
pointer, not a Python callback.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib, components, dtypes, kernel, layouts
from .components import BiasEpilogue, ConfigError, DiagonalPredicate, Params, identity, scale
from .dtypes import (BFLOAT16, COMPLEX32, COMPLEXBF16, DUAL16, DUAL32, DUAL64, DUALBF16,
                     FLOAT16)
from .kernel import EventCounters, KernelConfig
from .layouts import (ColMajor, Diagonal, InterleavedComplex, RowMajor, StridedPermutation, Zero,
                      col_major, split_pairs)
from .operators import ComplexOperator, DualOperator, FmaOperator, OperatorShape


def matmul(config: KernelConfig, a, b, c, d, **kwargs) -> EventCounters:
    """Resolve, validate and execute a kernel configuration on the B200."""
    return kernel.gemm_execute(config, a, b, c, d, **kwargs)


# ---- element types -------------------------------------------------------------------

_REAL = tuple(t for t in (np.dtype(np.float32), np.dtype(np.float64), FLOAT16, BFLOAT16) if t is not None)
_COMPLEX = tuple(t for t in (np.dtype(np.complex64), np.dtype(np.complex128), COMPLEX32, COMPLEXBF16)
                 if t is not None)
_DUAL = tuple(t for t in (DUAL32, DUAL64, DUAL16, DUALBF16) if t is not None)
SUPPORTED_ELEMENT_TYPES = _REAL + _COMPLEX + _DUAL


def accumulator_dtype(dtype) -> np.dtype:
    """Element type of C/D for A/B of ``dtype``: half storage accumulates in FP32."""
    dtype = np.dtype(dtype)
    if dtype in (FLOAT16, BFLOAT16):
        return np.dtype(np.float32)
    if dtype in (COMPLEX32, COMPLEXBF16):
        return np.dtype(np.complex64)
    if dtype in (DUAL16, DUALBF16):
        return DUAL32
    return dtype


def _unsupported(dtype):
    return ConfigError(f"unsupported element type {dtype}; supported: "
                       + ", ".join(str(t) for t in SUPPORTED_ELEMENT_TYPES))


def _operator_for(dtype, shape: OperatorShape, wide_accumulate: bool):
    dtype = np.dtype(dtype)
    acc = accumulator_dtype(dtype)
    if dtype in _REAL:
        wide = wide_accumulate and acc == np.dtype(np.float32)
        return FmaOperator(shape, np.float64 if wide else acc)
    if dtype in _COMPLEX:
        return ComplexOperator(shape, acc)
    if dtype in _DUAL:
        return DualOperator(shape, acc)
    raise _unsupported(dtype)


def _element_dtype(x):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return dtypes.from_torch(x.dtype)
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x).dtype


def _flat_buffer(arr):
    """(flat scalar buffer, storage order) of a 2-D matrix, without copying."""
    try:
        import torch

        is_torch = isinstance(arr, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_torch = False
    if len(arr.shape) != 2:
        raise ConfigError(f"expected a 2-D matrix, got shape {tuple(arr.shape)}")
    if is_torch:
        r, c = arr.shape
        st = arr.stride()
        fcont = (st[0] == 1 or r == 1) and (st[1] == r or c == 1)
        ccont = (st[1] == 1 or c == 1) and (st[0] == c or r == 1)
        if fcont:
            flat, order = arr.t().reshape(-1), "F"
        elif ccont:
            flat, order = arr.reshape(-1), "C"
        else:
            raise ConfigError("matrix must be C- or F-contiguous")
        if flat.is_complex():
            flat = torch.view_as_real(flat).reshape(-1)
        return flat, order
    if arr.flags["F_CONTIGUOUS"]:
        flat, order = arr.reshape(-1, order="F"), "F"
    elif arr.flags["C_CONTIGUOUS"]:
        flat, order = arr.reshape(-1, order="C"), "C"
    else:
        raise ConfigError("matrix must be C- or F-contiguous")
    if dtypes.pair_kind(arr.dtype):
        flat = flat.view(dtypes.storage_scalar(arr.dtype))
    return flat, order


def _global_layout(arr, names, extents, trans):
    """Layout of op(arr) over its existing storage (transposition = layout flip, no copy)."""
    flat, order = _flat_buffer(arr)
    expect = tuple(extents[::-1]) if trans else tuple(extents)
    if tuple(arr.shape) != expect:
        raise ConfigError(f"matrix shape {tuple(arr.shape)} != expected {expect}")
    colmajor = (order == "F") != trans
    dt = _element_dtype(arr)
    if dtypes.pair_kind(dt):
        layout = InterleavedComplex(dt, names, extents, order="F" if colmajor else "C")
    elif colmajor:
        layout = ColMajor(dt, names, extents)
    else:
        layout = RowMajor(dt, names, extents)
    return layout, flat


def _shared_builder(dtype):
    return split_pairs(dtype) if dtypes.pair_kind(dtype) else col_major(dtype)


def _as_array(x):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)


def gemm_ex(trans_a, trans_b, alpha, a, b, beta, c, *, operator_shape=None, block_tile=None,
            wide_accumulate=False, worker_threads=1, workers_per_block=1,
            scratch_budget=components.DEFAULT_SCRATCH_BUDGET, **run_kwargs):
    """C := alpha * op(A) @ op(B) + beta * C in place (op = identity or transpose).

    Components follow from the element type: real -> FMA operator; complex -> the
    four-product operator over interleaved global / split shared layouts; dual -> the
    three-product operator.  Transposition is a layout flip; nothing is copied.
    """
    a, b, c = _as_array(a), _as_array(b), _as_array(c)
    ta, tb, tc = _element_dtype(a), _element_dtype(b), _element_dtype(c)
    if not (ta == tb and tc == accumulator_dtype(ta)):
        raise ConfigError(f"element types must agree, got {ta}/{tb}/{tc}; supported: "
                          + ", ".join(str(t) for t in SUPPORTED_ELEMENT_TYPES))
    m, k = (a.shape[1], a.shape[0]) if trans_a else tuple(a.shape)
    n = c.shape[1]
    shape = OperatorShape(*(operator_shape or components.DEFAULT_OPERATOR_SHAPE))
    op = _operator_for(ta, shape, wide_accumulate)

    if alpha == 0:
        # alpha = 0 short-circuits A and B entirely: C := beta * C
        layout_a = Zero(ta, ("M", "K"), (m, k))
        layout_b = Zero(ta, ("K", "N"), (k, n))
        buf_a = np.zeros(0, layout_a.storage_dtype)
        buf_b = np.zeros(0, layout_b.storage_dtype)
        t_c, t_d = scale(beta), identity
    else:
        layout_a, buf_a = _global_layout(a, ("M", "K"), (m, k), trans_a)
        layout_b, buf_b = _global_layout(b, ("K", "N"), (k, n), trans_b)
        q = beta / alpha
        t_c = identity if q == 1 else scale(q)
        t_d = identity if alpha == 1 else scale(alpha)
    layout_c, buf_c = _global_layout(c, ("M", "N"), (m, n), False)
    if isinstance(buf_a, np.ndarray) and not isinstance(buf_c, np.ndarray) and buf_a.size == 0:
        import torch

        buf_a = buf_b = torch.empty(0, dtype=dtypes.torch_scalar(ta), device=buf_c.device)

    config = KernelConfig(
        params=Params(gemm_shape=(m, n, k), block_tile=block_tile,
                      operator_shape=(shape.m, shape.n, shape.k), worker_threads=worker_threads,
                      workers_per_block=workers_per_block, scratch_budget=scratch_budget),
        operator=op,
        global_a_layout=layout_a, global_b_layout=layout_b,
        global_c_layout=layout_c, global_d_layout=layout_c,
        shared_a_layout=_shared_builder(ta), shared_b_layout=_shared_builder(ta),
        shared_c_layout=_shared_builder(tc), shared_d_layout=_shared_builder(tc),
        transform_g2s_c=t_c, transform_r2s_d=t_d,
    )
    return matmul(config, buf_a, buf_b, buf_c, buf_c, **run_kwargs)


# ---- variant wiring ---------------------------------------------------------------------

def _scalar_type(dtype):
    """Numpy scalar type used for transform constants of a stream of ``dtype``."""
    acc = accumulator_dtype(dtype)
    return acc.type if acc.kind == "f" else np.float32


def build_dense_config(m, n, k, dtype=np.float32, *, trans_a=False, trans_b=False,
                       wide_accumulate=False, block_tile=None, operator_shape=None,
                       shared_pad=0, worker_threads=1, workers_per_block=1,
                       compute_warp=None) -> KernelConfig:
    """Plain (mixed-precision) GEMM over dense column/row-major matrices.

    Half dtypes (float16 / bfloat16) store A and B at 16 bits and C, D in float32.
    """
    dtype = np.dtype(dtype)
    acc = accumulator_dtype(dtype)
    shape = OperatorShape(*(operator_shape or components.DEFAULT_OPERATOR_SHAPE))
    shared = col_major(dtype)
    if shared_pad:
        shared = layouts.padded(shared, shared_pad)
    return KernelConfig(
        params=Params(gemm_shape=(m, n, k), block_tile=block_tile, compute_warp=compute_warp,
                      operator_shape=(shape.m, shape.n, shape.k), worker_threads=worker_threads,
                      workers_per_block=workers_per_block),
        operator=_operator_for(dtype, shape, wide_accumulate),
        global_a_layout=(RowMajor if trans_a else ColMajor)(dtype, ("M", "K"), (m, k)),
        global_b_layout=(RowMajor if trans_b else ColMajor)(dtype, ("K", "N"), (k, n)),
        global_c_layout=ColMajor(acc, ("M", "N"), (m, n)),
        global_d_layout=ColMajor(acc, ("M", "N"), (m, n)),
        shared_a_layout=shared,
        shared_b_layout=shared,
        shared_c_layout=col_major(acc),
        shared_d_layout=col_major(acc),
    )


def build_diagonal_config(n, dtype=np.float32, *, block_tile=None, operator_shape=None,
                          worker_threads=1) -> KernelConfig:
    """GEMM with diagonal A: only diag(A) is stored and loaded; off-diagonal block-K
    iterations are skipped (on the device: the producer fabricates the diagonal tile in
    shared memory and the k-range is restricted to the intersecting blocks)."""
    base = build_dense_config(n, n, n, dtype, block_tile=block_tile,
                              operator_shape=operator_shape, worker_threads=worker_threads)
    return dataclasses.replace(base, global_a_layout=Diagonal(dtype, ("M", "K"), (n, n)),
                               predicate=DiagonalPredicate())


def build_fused_config(m, n, k, dtype=np.float32, *, bias, relu_on_c=False, relu_on_d=True,
                       add_a=None, add_b=None, block_tile=None, operator_shape=None,
                       worker_threads=1, trans_a=False, trans_b=False) -> KernelConfig:
    """Fused element-wise / bias variant: constant adds on the A/B streams, ReLU on the C
    stream and the final D store, bias[j] per output column before the D transform."""
    dtype = np.dtype(dtype)
    base = build_dense_config(m, n, k, dtype, block_tile=block_tile, trans_a=trans_a,
                              trans_b=trans_b, operator_shape=operator_shape,
                              worker_threads=worker_threads)
    const = _scalar_type(dtype)

    def stream_add(c):
        return identity if c is None else components.add_constant(const(c))

    bias_arr = bias if _is_torch(bias) else np.asarray(bias, dtype=accumulator_dtype(dtype))
    return dataclasses.replace(
        base,
        transform_g2s_a=stream_add(add_a),
        transform_g2s_b=stream_add(add_b),
        transform_g2s_c=components.relu if relu_on_c else identity,
        transform_s2g_d=components.relu if relu_on_d else identity,
        epilogue=BiasEpilogue(bias_arr),
    )


def _is_torch(x):
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def build_complex_config(m, n, k, dtype=np.complex64, *, block_tile=None, operator_shape=None,
                         worker_threads=1, split=False) -> KernelConfig:
    """Complex GEMM (4 real products per operator invocation).

    Global layouts are interleaved (re, im) by default, as in the reference; ``split=True``
    uses separate real/imaginary planes (``SplitComplex``) for A, B, C and D instead.
    """
    dtype = np.dtype(dtype)
    acc = accumulator_dtype(dtype)
    shape = OperatorShape(*(operator_shape or components.DEFAULT_OPERATOR_SHAPE))
    glob = layouts.SplitComplex if split else InterleavedComplex
    return KernelConfig(
        params=Params(gemm_shape=(m, n, k), block_tile=block_tile,
                      operator_shape=(shape.m, shape.n, shape.k), worker_threads=worker_threads),
        operator=_operator_for(dtype, shape, False),
        global_a_layout=glob(dtype, ("M", "K"), (m, k)),
        global_b_layout=glob(dtype, ("K", "N"), (k, n)),
        global_c_layout=glob(acc, ("M", "N"), (m, n)),
        global_d_layout=glob(acc, ("M", "N"), (m, n)),
        shared_a_layout=split_pairs(dtype),
        shared_b_layout=split_pairs(dtype),
        shared_c_layout=split_pairs(acc),
        shared_d_layout=split_pairs(acc),
    )


def build_dual_config(m, n, k, dtype=DUAL64, **kwargs) -> KernelConfig:
    """Dual-number GEMM (3 real products); reuses the pair layouts."""
    return build_complex_config(m, n, k, dtype, **kwargs)


def build_tc_config(na, nb, nc, nd, dtype=np.float32, *, block_tile=None, operator_shape=None,
                    worker_threads=1) -> KernelConfig:
    """Tensor contraction D[a,b,c] = sum_d A[b,d,a] * B[d,c] as a GEMM with fused
    transpositions: M = (b, a), K = d, N = c; A stays (Nb, Nd, Na) column-major, D is
    written as (Na, Nb, Nc) column-major, C is a Zero layout."""
    dtype = np.dtype(dtype)
    acc = accumulator_dtype(dtype)
    m, n, k = nb * na, nc, nd
    shape = OperatorShape(*(operator_shape or _tc_operator_shape(m, n, k)))
    layout_a = StridedPermutation(dtype, ("M", "K"), (m, k),
                                  dim_map={"M": (("b", nb), ("a", na)), "K": (("d", nd),)},
                                  storage_order=("b", "d", "a"))
    layout_d = StridedPermutation(acc, ("M", "N"), (m, n),
                                  dim_map={"M": (("b", nb), ("a", na)), "N": (("c", nc),)},
                                  storage_order=("a", "b", "c"))
    return KernelConfig(
        params=Params(gemm_shape=(m, n, k), block_tile=block_tile,
                      operator_shape=(shape.m, shape.n, shape.k), worker_threads=worker_threads),
        operator=_operator_for(dtype, shape, False),
        global_a_layout=layout_a,
        global_b_layout=ColMajor(dtype, ("K", "N"), (k, n)),
        global_c_layout=Zero(acc, ("M", "N"), (m, n)),
        global_d_layout=layout_d,
        shared_a_layout=col_major(dtype), shared_b_layout=col_major(dtype),
        shared_c_layout=col_major(acc), shared_d_layout=col_major(acc),
    )


def _tc_operator_shape(m, n, k):
    return tuple(min(e, 8) for e in (m, n, k))


def contract(a, b, *, worker_threads=1, block_tile=None, **run_kwargs):
    """Tensor contraction on (Nb, Nd, Na) x (Nd, Nc) arrays; returns (D (Na, Nb, Nc), counters).

    numpy inputs give a numpy D; torch CUDA tensors stay on the device (D as a torch tensor).
    """
    if _is_torch(a):
        import torch

        nb, nd, na = a.shape
        _, nc = b.shape
        dt = dtypes.from_torch(a.dtype)
        cfg = build_tc_config(na, nb, nc, nd, dt, worker_threads=worker_threads,
                              block_tile=block_tile)
        acc = dtypes.torch_scalar(accumulator_dtype(dt))
        d = torch.zeros(na * nb * nc, dtype=acc, device=a.device)
        fa = a.permute(2, 1, 0).reshape(-1)  # column-major flattening
        fb = b.t().reshape(-1)
        counters = matmul(cfg, fa, fb, torch.empty(0, dtype=acc, device=a.device), d,
                          **run_kwargs)
        return d.reshape(nc, nb, na).permute(2, 1, 0), counters
    a = np.asfortranarray(a)
    b = np.asfortranarray(b)
    nb, nd, na = a.shape
    _, nc = b.shape
    cfg = build_tc_config(na, nb, nc, nd, a.dtype, worker_threads=worker_threads,
                          block_tile=block_tile)
    acc = accumulator_dtype(a.dtype)
    d = np.zeros(na * nb * nc, dtype=acc)
    counters = matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), np.zeros(0, acc), d,
                      **run_kwargs)
    return d.reshape((na, nb, nc), order="F"), counters


# ---- general tensor contractions (GETT) ----------------------------------------------------

def _parse_gett(spec):
    try:
        d_idx, a_idx, b_idx = spec.replace(" ", "").split("-")
    except ValueError:
        raise ConfigError(f"GETT spec {spec!r} must read 'D-A-B', e.g. 'abc-bda-dc'") from None
    for name, idx in (("D", d_idx), ("A", a_idx), ("B", b_idx)):
        if len(set(idx)) != len(idx):
            raise ConfigError(f"GETT spec {spec!r}: repeated index in {name}")
    m_idx = tuple(i for i in d_idx if i in a_idx and i not in b_idx)
    n_idx = tuple(i for i in d_idx if i in b_idx and i not in a_idx)
    k_idx = tuple(i for i in a_idx if i in b_idx and i not in d_idx)
    if set(d_idx) != set(m_idx) | set(n_idx) or set(a_idx) != set(m_idx) | set(k_idx) or \
            set(b_idx) != set(n_idx) | set(k_idx):
        raise ConfigError(f"GETT spec {spec!r}: every index must be free in exactly one operand "
                          "and D, or contracted between A and B (no batch / trace indices)")
    if not (m_idx and n_idx and k_idx):
        raise ConfigError(f"GETT spec {spec!r}: needs free indices in A and B and a contraction")
    if max(len(m_idx), len(n_idx), len(k_idx)) > _lib.MAX_DIGITS:
        raise ConfigError(f"GETT spec {spec!r}: at most {_lib.MAX_DIGITS} indices per GEMM dimension")
    return d_idx, a_idx, b_idx, m_idx, n_idx, k_idx


def build_gett_config(spec, sizes, dtype=np.float32, *, operator_shape=None,
                      worker_threads=1) -> KernelConfig:
    """A general tensor contraction D = A . B as a GEMM with fused transpositions (GETT).

    ``spec`` is TCCG notation ``"D-A-B"`` over single-letter indices, each tensor listed in
    storage order (first index fastest, column-major like every layout here), e.g.
    ``"abc-bda-dc"`` (the case ``build_tc_config`` wires) or ``"abcd-aebf-dfce"``.  Free
    indices of A form M (ordered as in D), free indices of B form N (as in D), contracted
    indices form K (as in A); each operand is a ``StridedPermutation`` over its own storage
    order, C is Zero.  This generalises the reference's single contraction
    (``api.py:259-312``) to the StridedPermutation layouts it defines (``layouts.py:435-506``);
    on the tcgen05 lane non-TMA operands are gathered once into dense workspaces and D is
    scattered by the epilogue's digit maps.
    """
    d_idx, a_idx, b_idx, m_idx, n_idx, k_idx = _parse_gett(spec)
    missing = [i for i in set(d_idx + a_idx + b_idx) if i not in sizes]
    if missing:
        raise ConfigError(f"GETT sizes missing {sorted(missing)}")
    ext = {i: int(sizes[i]) for i in set(d_idx + a_idx + b_idx)}
    dtype = np.dtype(dtype)
    if dtypes.pair_kind(dtype):
        raise ConfigError("build_gett_config takes real element types (the reference's "
                          "StridedPermutation GETT is real); use build_complex_config / "
                          "build_dual_config for pair operators")
    acc = accumulator_dtype(dtype)
    vol = lambda idx: int(np.prod([ext[i] for i in idx]))
    m, n, k = vol(m_idx), vol(n_idx), vol(k_idx)
    group = lambda idx: tuple((i, ext[i]) for i in idx)
    layout_a = StridedPermutation(dtype, ("M", "K"), (m, k),
                                  dim_map={"M": group(m_idx), "K": group(k_idx)},
                                  storage_order=tuple(a_idx))
    layout_b = StridedPermutation(dtype, ("K", "N"), (k, n),
                                  dim_map={"K": group(k_idx), "N": group(n_idx)},
                                  storage_order=tuple(b_idx))
    layout_d = StridedPermutation(acc, ("M", "N"), (m, n),
                                  dim_map={"M": group(m_idx), "N": group(n_idx)},
                                  storage_order=tuple(d_idx))
    shape = OperatorShape(*(operator_shape or _tc_operator_shape(m, n, k)))
    return KernelConfig(
        params=Params(gemm_shape=(m, n, k), operator_shape=(shape.m, shape.n, shape.k),
                      worker_threads=worker_threads),
        operator=_operator_for(dtype, shape, False),
        global_a_layout=layout_a, global_b_layout=layout_b,
        global_c_layout=Zero(acc, ("M", "N"), (m, n)), global_d_layout=layout_d,
        shared_a_layout=col_major(dtype), shared_b_layout=col_major(dtype),
        shared_c_layout=col_major(acc), shared_d_layout=col_major(acc),
    )


def gett(spec, a, b, **run_kwargs):
    """Contract ``a`` and ``b`` per ``spec`` (see ``build_gett_config``); arrays are indexed in
    the order their spec letters are written.  numpy in -> numpy D; torch CUDA tensors stay on
    the device.  Returns (D, counters)."""
    d_idx, a_idx, b_idx, *_ = _parse_gett(spec)
    sizes = dict(zip(a_idx, a.shape))
    sizes.update(zip(b_idx, b.shape))
    for i, e in list(zip(a_idx, a.shape)) + list(zip(b_idx, b.shape)):
        if sizes[i] != e:
            raise ConfigError(f"index {i!r} has inconsistent extents")
    d_shape = tuple(sizes[i] for i in d_idx)
    if _is_torch(a):
        import torch

        dt = dtypes.from_torch(a.dtype)
        cfg = build_gett_config(spec, sizes, dt)
        accd = dtypes.torch_scalar(accumulator_dtype(dt))
        d = torch.zeros(int(np.prod(d_shape)), dtype=accd, device=a.device)
        fa = a.permute(*reversed(range(a.dim()))).reshape(-1)  # column-major flattening
        fb = b.permute(*reversed(range(b.dim()))).reshape(-1)
        counters = matmul(cfg, fa, fb, torch.empty(0, dtype=accd, device=a.device), d,
                          **run_kwargs)
        return d.reshape(tuple(reversed(d_shape))).permute(*reversed(range(len(d_shape)))), counters
    a = np.asfortranarray(a)
    b = np.asfortranarray(b)
    cfg = build_gett_config(spec, sizes, a.dtype)
    accd = accumulator_dtype(a.dtype)
    d = np.zeros(int(np.prod(d_shape)), dtype=accd)
    counters = matmul(cfg, a.ravel(order="F"), b.ravel(order="F"), np.zeros(0, accd), d,
                      **run_kwargs)
    return d.reshape(d_shape, order="F"), counters


# ---- C-compatible export ------------------------------------------------------------------

TAG_F32, TAG_F64, TAG_C64, TAG_C128, TAG_DUAL32, TAG_DUAL64 = range(6)
TAG_F16F32, TAG_BF16F32, TAG_C32C64, TAG_CBF16C64, TAG_DUAL16F32, TAG_DUALBF16F32 = range(6, 12)
_TAG_DTYPES = {
    TAG_F32: np.dtype(np.float32), TAG_F64: np.dtype(np.float64),
    TAG_C64: np.dtype(np.complex64), TAG_C128: np.dtype(np.complex128),
    TAG_DUAL32: DUAL32, TAG_DUAL64: DUAL64,
    TAG_F16F32: FLOAT16, TAG_BF16F32: BFLOAT16, TAG_C32C64: COMPLEX32,
    TAG_CBF16C64: COMPLEXBF16, TAG_DUAL16F32: DUAL16, TAG_DUALBF16F32: DUALBF16,
}

GEMM_EX_CFUNC = ctypes.CFUNCTYPE(
    ctypes.c_int,
    ctypes.c_int, ctypes.c_int, ctypes.c_int,                 # tag, transA, transB
    ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,  # m, n, k
    ctypes.c_double, ctypes.c_double,                         # alpha re/im
    ctypes.c_void_p, ctypes.c_void_p,                         # A, B
    ctypes.c_double, ctypes.c_double,                         # beta re/im
    ctypes.c_void_p,                                          # C (in/out)
)


def gemm_ex_raw(type_tag, trans_a, trans_b, m, n, k, alpha_re, alpha_im, a_ptr, b_ptr,
                beta_re, beta_im, c_ptr) -> int:
    """gemm_ex over flat column-major pointers (host or device), extents and a type tag.

    Calls ``tk_gemm_ex_raw`` of libtk_sm100.so; returns 0 on success, 1 on any
    configuration error (2 on a CUDA runtime failure).
    """
    lib = _lib.load()
    return int(lib.tk_gemm_ex_raw(int(type_tag), int(trans_a), int(trans_b), int(m), int(n),
                                  int(k), float(alpha_re), float(alpha_im), a_ptr, b_ptr,
                                  float(beta_re), float(beta_im), c_ptr))


def gemm_ex_cfunc():
    """The C library's tk_gemm_ex_raw as a GEMM_EX_CFUNC function pointer."""
    lib = _lib.load()
    return ctypes.cast(lib.tk_gemm_ex_raw, GEMM_EX_CFUNC)
