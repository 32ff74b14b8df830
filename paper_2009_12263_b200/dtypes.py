"""Element types understood by the B200 GEMM path.

The reference supports f32/f64/complex64/complex128/DUAL32/DUAL64
(reference ``api.py:45-48``).  The B200 path keeps all of them (they run on
the bit-exact CUDA-core lane) and adds the tensor-core storage types the
north star asks for: float16 / bfloat16 real, and half-precision complex and
dual pairs.  Pair types are numpy record dtypes of two scalars; complex64 /
complex128 are numpy's native complex types.
"""

from __future__ import annotations

import numpy as np

try:  # numpy has no native bfloat16; ml_dtypes ships one in this image
    import ml_dtypes as _mld

    BFLOAT16 = np.dtype(_mld.bfloat16)
except Exception:  # pragma: no cover - bf16 then only reachable via torch tensors
    BFLOAT16 = None

FLOAT16 = np.dtype(np.float16)
FLOAT32 = np.dtype(np.float32)
FLOAT64 = np.dtype(np.float64)
COMPLEX64 = np.dtype(np.complex64)
COMPLEX128 = np.dtype(np.complex128)

# Array-of-structs pair types (value, epsilon) / (real, imag).
DUAL32 = np.dtype([("value", "<f4"), ("epsilon", "<f4")])
DUAL64 = np.dtype([("value", "<f8"), ("epsilon", "<f8")])
DUAL16 = np.dtype([("value", "<f2"), ("epsilon", "<f2")])
COMPLEX32 = np.dtype([("real", "<f2"), ("imag", "<f2")])  # complex half
if BFLOAT16 is not None:
    DUALBF16 = np.dtype([("value", BFLOAT16), ("epsilon", BFLOAT16)])
    COMPLEXBF16 = np.dtype([("real", BFLOAT16), ("imag", BFLOAT16)])
else:  # pragma: no cover
    DUALBF16 = COMPLEXBF16 = None

# scalar type codes shared with the C ABI (include/tk_sm100.h TkScalar)
SCALAR_CODES = {"f16": 0, "bf16": 1, "f32": 2, "f64": 3}


def _scalar_name(dt: np.dtype) -> str:
    if dt == FLOAT16:
        return "f16"
    if BFLOAT16 is not None and dt == BFLOAT16:
        return "bf16"
    if dt == FLOAT32:
        return "f32"
    if dt == FLOAT64:
        return "f64"
    raise ValueError(f"{dt} is not a supported scalar type")


def pair_kind(dt) -> str | None:
    """'complex', 'dual' or None for a real element type."""
    dt = np.dtype(dt)
    if dt.kind == "c":
        return "complex"
    if dt.names is not None and len(dt.names) == 2:
        return "dual" if dt.names[0] == "value" else "complex"
    return None


def storage_scalar(dt) -> np.dtype:
    """Scalar dtype of the flat backing buffer of an element type."""
    dt = np.dtype(dt)
    if dt.kind == "c":
        return FLOAT32 if dt.itemsize == 8 else FLOAT64
    if dt.names is not None:
        return dt[dt.names[0]]
    return dt


def scalar_name(dt) -> str:
    return _scalar_name(storage_scalar(dt))


def is_half(dt) -> bool:
    return scalar_name(dt) in ("f16", "bf16")


def pair_planes(dt):
    """(scalar, split, combine) helpers for two-plane element types."""
    dt = np.dtype(dt)
    scalar = storage_scalar(dt)
    if dt.kind == "c":
        return scalar, (lambda v: (v.real, v.imag)), (lambda p0, p1: (p0 + 1j * p1).astype(dt))
    if dt.names is not None and len(dt.names) == 2:
        f0, f1 = dt.names

        def combine(p0, p1):
            out = np.empty(np.shape(p0), dtype=dt)
            out[f0] = p0
            out[f1] = p1
            return out

        return scalar, (lambda v: (v[f0], v[f1])), combine
    raise ValueError(f"{dt} is not a two-plane element type")


def torch_scalar(dt):
    """torch dtype of the flat backing buffer."""
    import torch

    return {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32,
            "f64": torch.float64}[scalar_name(dt)]


def from_torch(tdt):
    import torch

    table = {torch.float16: FLOAT16, torch.float32: FLOAT32, torch.float64: FLOAT64,
             torch.complex64: COMPLEX64, torch.complex128: COMPLEX128}
    if tdt == torch.bfloat16:
        if BFLOAT16 is None:  # pragma: no cover
            raise ValueError("bfloat16 needs ml_dtypes")
        return BFLOAT16
    return table[tdt]
