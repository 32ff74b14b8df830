"""TEST INFRASTRUCTURE ONLY -- the parity oracle.

Python face of ``tk_oracle.c`` (the C restatement of the reference arithmetic, see its
header for the reference file:line each step follows) plus composed oracles for the
variants.  Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` import this module, always as the checker or
the timed CPU baseline -- never as part of the product path.

Parity of this restatement is pinned against the reference package itself:
``tests/golden/*.npz`` hold outputs of reference ``tilekit`` runs (``make_golden.py``)
and ``tests/test_oracle.py`` requires bitwise equality with them.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_int, c_int64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

T_SCALE, T_ADD, T_RELU = 1, 2, 3


class TkoProg(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("op", ctypes.c_int32 * 8),
                ("promote", ctypes.c_int32 * 8), ("re", ctypes.c_double * 8),
                ("im", ctypes.c_double * 8)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _LIB = ctypes.CDLL(path)
        _LIB.tko_gemm_real.argtypes = [c_int, c_int64, c_int64, c_int64] + \
            [c_void_p, c_int64, c_int64] * 4 + [c_void_p] * 5 + \
            [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_int]
        _LIB.tko_gemm_pair.argtypes = [c_int, c_int, c_int64, c_int64, c_int64, c_int64] + \
            [c_void_p, c_int64, c_int64] * 4 + [c_void_p] * 5 + [c_int]
    return _LIB


def prog(*ops):
    """Op program from (code, const[, promote]) tuples, e.g. prog((T_SCALE, 2.0), (T_RELU, 0))."""
    g = TkoProg()
    g.n = len(ops)
    for i, op in enumerate(ops):
        g.op[i] = op[0]
        c = complex(op[1]) if len(op) > 1 else 0j
        g.re[i], g.im[i] = c.real, c.imag
        g.promote[i] = int(op[2]) if len(op) > 2 else 0
    return g


def _p(g):
    return ctypes.byref(g) if g is not None else None


def _strides(x):
    item = x.dtype.itemsize
    return x.strides[0] // item, x.strides[1] // item


def default_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def gemm_real(a, b, c=None, *, t_a=None, t_b=None, t_c=None, t_r2s=None, t_s2g=None,
              bias=None, bias_axis="n", mode=None, kmask=None, block=(1, 1, 1), threads=None,
              out=None):
    """D = s2g(r2s(g2s_c(C) + sum_k g2s_a(A) g2s_b(B)) + bias) with the reference order.

    a (m,k), b (k,n), c (m,n) are 2-D numpy arrays of float32 or float64 (any strides; None =
    Zero layout).  mode: 0 f32, 1 f32 storage with f64 accumulation, 2 f64 (default from dtype).
    """
    ref = next(x for x in (a, b, c) if x is not None)
    dt = np.float64 if ref.dtype == np.float64 else np.float32
    mode = (2 if dt == np.float64 else 0) if mode is None else mode
    m, k = (a.shape if a is not None else (c.shape[0], b.shape[0]))
    n = b.shape[1] if b is not None else c.shape[1]
    arrs = [None if x is None else np.asarray(x, dtype=dt) for x in (a, b, c)]
    d = out if out is not None else np.zeros((m, n), dtype=dt, order="F")
    bias_arr = None if bias is None else np.ascontiguousarray(bias, dtype=dt)
    args = []
    for x in arrs + [d]:
        if x is None:
            args += [None, 0, 0]
        else:
            rs, cs = _strides(x)
            args += [x.ctypes.data, rs, cs]
    mask = None if kmask is None else np.ascontiguousarray(kmask, dtype=np.uint8)
    lib().tko_gemm_real(mode, m, n, k, *args, _p(t_a), _p(t_b), _p(t_c), _p(t_r2s), _p(t_s2g),
                        None if bias_arr is None else bias_arr.ctypes.data,
                        0 if bias_arr is None else (1 if bias_axis == "n" else 2),
                        None if mask is None else mask.ctypes.data, block[0], block[1],
                        block[2], threads or default_threads())
    return d


def gemm_pair(a, b, c=None, *, dual=False, op_k=8, t_a=None, t_b=None, t_c=None,
              t_r2s=None, t_s2g=None, threads=None):
    """Complex (4 real products) or dual (3) GEMM in the reference's chunked order.

    a, b, c: 2-D complex64/complex128 arrays, or DUAL32/DUAL64 record arrays.
    Returns D with the same element type as the inputs.
    """
    ref = next(x for x in (a, b, c) if x is not None)
    scalar = np.float64 if ref.dtype.itemsize == 16 else np.float32
    mode = 2 if scalar == np.float64 else 0
    m, k = a.shape if a is not None else (c.shape[0], b.shape[0])
    n = b.shape[1] if b is not None else c.shape[1]
    d = np.zeros((m, n), dtype=ref.dtype, order="F")
    args = []
    for x in (a, b, c, d):
        if x is None:
            args += [None, 0, 0]
        else:
            rs, cs = (s // x.dtype.itemsize for s in x.strides)
            args += [x.ctypes.data, rs, cs]
    lib().tko_gemm_pair(mode, int(dual), m, n, k, op_k, *args, _p(t_a), _p(t_b), _p(t_c),
                        _p(t_r2s), _p(t_s2g), threads or default_threads())
    return d


# ---- composed oracles for the variants --------------------------------------------------

def fused_reference(a, b, c, bias, *, relu_on_c=False, relu_on_d=True, add_a=None,
                    add_b=None, threads=None):
    """build_fused_config semantics (reference api.py:206-230): f32, bias per column."""
    f = lambda x: np.asarray(x, dtype=np.float32)
    return gemm_real(f(a), f(b), f(c),
                     t_a=prog((T_ADD, add_a)) if add_a is not None else None,
                     t_b=prog((T_ADD, add_b)) if add_b is not None else None,
                     t_c=prog((T_RELU, 0)) if relu_on_c else None,
                     t_s2g=prog((T_RELU, 0)) if relu_on_d else None,
                     bias=f(bias), bias_axis="n", threads=threads)


def diagonal_kmask(n, block):
    """Executed block-K iterations of DiagonalPredicate (components.py:186-191)."""
    bm, bn, bk = block
    nmb, nnb, nkb = n // bm, n // bn, n // bk
    m0 = (np.arange(nmb) * bm)[:, None]
    k0 = (np.arange(nkb) * bk)[None, :]
    run = np.maximum(m0, k0) < np.minimum(m0 + bm, k0 + bk)
    full = np.broadcast_to(run[None, :, :], (nnb, nmb, nkb))
    return full.reshape(nnb * nmb, nkb).astype(np.uint8)


def tc_reference(a, b, threads=None):
    """D[a,b,c] = sum_d A[b,d,a] B[d,c] (reference api.py:259-290) via the real oracle:
    M = (b, a) b fastest, K = d; D scattered to (Na, Nb, Nc)."""
    nb, nd, na = a.shape
    _, nc = b.shape
    amk = np.asfortranarray(np.asarray(a, dtype=np.float32).transpose(0, 2, 1)
                            .reshape(nb * na, nd, order="F"))
    dmn = gemm_real(amk, np.asarray(b, dtype=np.float32), None, threads=threads)
    return dmn.reshape(nb, na, nc, order="F").transpose(1, 0, 2)


def gett_indices(spec):
    """M / N / K index groups of a TCCG spec 'D-A-B' (the wiring of oracle/make_golden.py
    gett_cases and paper_2009_12263_b200.build_gett_config)."""
    d_idx, a_idx, b_idx = spec.split("-")
    return (d_idx, a_idx, b_idx, [i for i in d_idx if i in a_idx], [i for i in d_idx if i in b_idx],
            [i for i in a_idx if i in b_idx])


def gett_matrices(spec, a, b):
    """The GEMM view (A as M x K, B as K x N, column-major digits) of a contraction."""
    d_idx, a_idx, b_idx, m_idx, n_idx, k_idx = gett_indices(spec)
    ext = dict(zip(a_idx, a.shape))
    ext.update(zip(b_idx, b.shape))
    vol = lambda idx: int(np.prod([ext[i] for i in idx]))
    amk = np.asarray(a).transpose([a_idx.index(i) for i in m_idx + k_idx]) \
        .reshape(vol(m_idx), vol(k_idx), order="F")
    bkn = np.asarray(b).transpose([b_idx.index(i) for i in k_idx + n_idx]) \
        .reshape(vol(k_idx), vol(n_idx), order="F")
    return np.asfortranarray(amk), np.asfortranarray(bkn), ext


def gett_reference(spec, a, b, threads=None):
    """D = A . B for a TCCG spec via the real oracle over the GEMM view (k ascending in the
    K-digit order, f32 multiply-then-add: the reference's generic path, layouts.py:435-506)."""
    d_idx, a_idx, b_idx, m_idx, n_idx, k_idx = gett_indices(spec)
    amk, bkn, ext = gett_matrices(spec, np.asarray(a, np.float32), np.asarray(b, np.float32))
    dmn = gemm_real(amk, bkn, None, threads=threads)
    d = dmn.reshape([ext[i] for i in m_idx + n_idx], order="F")
    return d.transpose([(m_idx + n_idx).index(i) for i in d_idx])


# ---- exact references and tolerance -----------------------------------------------------

def exact_gemm(a, b, c=None, alpha=1.0, beta=0.0):
    """alpha*A@B + beta*C in float64 / complex128 (numpy BLAS), the accuracy yardstick."""
    wide = np.complex128 if np.iscomplexobj(a) else np.float64
    d = alpha * (np.asarray(a, dtype=wide) @ np.asarray(b, dtype=wide))
    if c is not None and beta != 0:
        d = d + beta * np.asarray(c, dtype=wide)
    return d


def rel_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    wide = np.complex128 if (np.iscomplexobj(got) or np.iscomplexobj(want)) else np.float64
    got, want = got.astype(wide), want.astype(wide)
    denom = float(np.max(np.abs(want)))
    return float(np.max(np.abs(got - want)) / (denom if denom else 1.0))


def tolerance(k, factor=4.0):
    """Normwise bound for FP32 accumulation: factor * 2^-24 * sqrt(K)."""
    return factor * 2.0 ** -24 * np.sqrt(k)
