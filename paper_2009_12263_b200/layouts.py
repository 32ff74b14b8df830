"""Global and shared layouts: logical (M,K)/(K,N)/(M,N) tiles <-> physical storage.

Same classes and builders as the reference (``pkg/src/tilekit/layouts.py:32-506``):
``ColMajor``, ``RowMajor``, ``Padded``, ``Diagonal``, ``Zero``,
``InterleavedComplex``, ``SplitComplex``, ``StridedPermutation`` and the
``col_major / row_major / padded / interleaved_pairs / split_pairs`` builders.

B200 design: every layout is an *address map*.  A logical index along each
dimension is decomposed into "digits" ``(extent, stride)`` (fastest first);
the element offset is ``sum(digit * stride)``.  Dense column/row-major,
padding and arbitrary stride permutations (the GETT fused transposition) are
all digit lists, so a single descriptor (``lower()`` -> ``TkLayout`` in
``include/tk_sm100.h``) feeds both device lanes: the planner turns 2-D/3-D
digit lists into TMA tensor maps for the tcgen05 lane, and the CUDA-core lane
walks them directly.  ``Diagonal`` and ``Zero`` are not address maps: they
lower to dedicated producer kinds (diagonal tile fabricated in shared memory;
elided loads).

Host ``load``/``store`` are kept for API parity and inspection (values travel
as flat arrays in the tile's local column-major order, reference
``layouts.py:1-14``); they are never on the GEMM execution path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import dtypes
from .tiling import Tile

# layout kinds / pair modes, mirrored by TkLayoutKind / TkPairMode in include/tk_sm100.h
KIND_STRIDED, KIND_DIAGONAL, KIND_ZERO = 0, 1, 2
PAIR_NONE, PAIR_INTERLEAVED, PAIR_SPLIT = 0, 1, 2
MAX_DIGITS = 5  # digits per logical dimension (TK_MAX_DIGITS)


def _volume(extents) -> int:
    v = 1
    for e in extents:
        v *= int(e)
    return v


@dataclass(frozen=True)
class LayoutDesc:
    """Device-facing description of a 2-D layout (see ``TkLayout``)."""

    kind: int
    pair: int
    scalar: str
    digits: tuple  # per logical dim: tuple of (extent, stride) fastest first
    plane_stride: int
    size: int


class Layout:
    """Base class: names, extents, element type, tile bounds checks."""

    names: tuple
    extents: tuple
    element_type: np.dtype

    def physical_size(self) -> int:
        raise NotImplementedError

    @property
    def storage_dtype(self) -> np.dtype:
        return self.element_type

    def load_count(self, tile: Tile) -> int:
        return tile.volume

    def store_count(self, tile: Tile) -> int:
        return tile.volume

    # ---- address map -------------------------------------------------------
    def digits(self):
        """Per-dimension (extent, stride) digit lists, or None if not an address map."""
        return None

    def lower(self) -> LayoutDesc:
        digits = self.digits()
        if digits is None:
            raise NotImplementedError(f"{type(self).__name__} has no address map")
        return LayoutDesc(KIND_STRIDED, PAIR_NONE, dtypes.scalar_name(self.storage_dtype),
                          tuple(tuple(d) for d in digits), 0, self.physical_size())

    # ---- host-side access (API parity; not on the device path) -------------
    def _check_tile(self, tile: Tile):
        if tile.names != tuple(self.names):
            raise ValueError(f"tile dims {tile.names} do not match layout dims {self.names}")
        for name, start, size, extent in zip(self.names, tile.absolute.values,
                                             tile.size.values, self.extents):
            if start < 0 or start + size > extent:
                raise ValueError(f"tile out of bounds in {name}: [{start}, {start + size}) "
                                 f"outside [0, {extent})")

    def _check_values(self, tile: Tile, values) -> np.ndarray:
        values = np.asarray(values)
        if values.size != tile.volume:
            raise ValueError(f"value tuple length {values.size} != tile element count "
                             f"{tile.volume}")
        return values.reshape(-1)

    def _offsets(self, tile: Tile) -> np.ndarray:
        """Element offsets of a tile in local column-major order."""
        self._check_tile(tile)
        total = np.zeros((), dtype=np.int64)
        for axis, digits in enumerate(self.digits()):
            start, size = tile.absolute.values[axis], tile.size.values[axis]
            idx = np.arange(start, start + size, dtype=np.int64)
            part = np.zeros_like(idx)
            for ext, stride in digits:
                idx, r = np.divmod(idx, ext)
                part += r * stride
            shape = [1] * len(self.names)
            shape[axis] = size
            total = total + part.reshape(shape)
        return np.broadcast_to(total, tile.size.values).ravel(order="F")

    def load(self, buf, tile):
        return np.asarray(buf)[self._offsets(tile)].astype(self.element_type, copy=False)

    def store(self, buf, tile, values):
        values = self._check_values(tile, values)
        buf[self._offsets(tile)] = values.astype(self.storage_dtype, copy=False)


def alloc_buffer(layout: Layout) -> np.ndarray:
    return np.zeros(layout.physical_size(), dtype=layout.storage_dtype)


def check_buffer(layout: Layout, buf, label: str = "buffer") -> None:
    need = layout.physical_size()
    shape = tuple(buf.shape)
    if len(shape) != 1 or shape[0] != need:
        raise ValueError(f"{label}: expected flat buffer of {need} elements, got shape {shape}")


def _dense_digits(extents, order, pad_fastest=0):
    """Digits of a dense layout; ``order`` 'F' = first dim fastest."""
    n = len(extents)
    axes = range(n) if order == "F" else range(n - 1, -1, -1)
    strides = [0] * n
    stride = 1
    for i, ax in enumerate(axes):
        strides[ax] = stride
        stride *= extents[ax] + (pad_fastest if i == 0 else 0)
    return [[(int(extents[ax]), strides[ax])] for ax in range(n)]


@dataclass(frozen=True)
class ColMajor(Layout):
    """Dense column-major storage (first dimension has stride 1)."""

    element_type: np.dtype
    names: tuple
    extents: tuple

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))

    _order = "F"

    def physical_size(self) -> int:
        return _volume(self.extents)

    def digits(self):
        return _dense_digits(self.extents, self._order)


@dataclass(frozen=True)
class RowMajor(ColMajor):
    """Dense row-major storage (last dimension has stride 1)."""

    _order = "C"


@dataclass(frozen=True)
class Padded(Layout):
    """A dense layout whose fastest dimension is padded by ``pad`` elements.

    Shared-memory anti-bank-conflict padding in the reference
    (``layouts.py:132-188``).  On the device, shared staging uses the TMA
    128-byte swizzle instead, so a padded *shared* builder only changes the
    logical scratch footprint used by the block-tile heuristic; a padded
    *global* layout is an ordinary strided address map.
    """

    inner: ColMajor
    pad: int

    def __post_init__(self):
        if self.pad < 0:
            raise ValueError("padding must be >= 0")
        if not isinstance(self.inner, ColMajor):
            raise ValueError("Padded wraps a ColMajor or RowMajor layout")

    names = property(lambda self: self.inner.names)
    extents = property(lambda self: self.inner.extents)
    element_type = property(lambda self: self.inner.element_type)

    def _padded_extents(self):
        ext = list(self.extents)
        ext[0 if self.inner._order == "F" else len(ext) - 1] += self.pad
        return tuple(ext)

    def physical_size(self) -> int:
        return _volume(self._padded_extents())

    def digits(self):
        return _dense_digits(self.extents, self.inner._order, self.pad)


@dataclass(frozen=True)
class Diagonal(Layout):
    """Square matrix with only its diagonal materialised (``physical_size == n``)."""

    element_type: np.dtype
    names: tuple
    extents: tuple

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        if len(self.extents) != 2 or self.extents[0] != self.extents[1]:
            raise ValueError(f"Diagonal layout needs square extents, got {self.extents}")

    def physical_size(self) -> int:
        return self.extents[0]

    def lower(self) -> LayoutDesc:
        n = self.extents[0]
        return LayoutDesc(KIND_DIAGONAL, PAIR_NONE, dtypes.scalar_name(self.element_type),
                          (((n, 1),), ((n, 1),)), 0, n)

    def _span(self, tile: Tile):
        (r0, c0), (rn, cn) = tile.absolute.values, tile.size.values
        lo, hi = max(r0, c0), min(r0 + rn, c0 + cn)
        return lo, max(lo, hi)

    def load_count(self, tile):
        lo, hi = self._span(tile)
        return hi - lo

    store_count = load_count

    def load(self, buf, tile):
        self._check_tile(tile)
        rows, cols = tile.size.values
        r0, c0 = tile.absolute.values
        out = np.zeros((rows, cols), dtype=self.element_type)
        lo, hi = self._span(tile)
        i = np.arange(lo, hi)
        out[i - r0, i - c0] = np.asarray(buf)[lo:hi]
        return out.ravel(order="F")

    def store(self, buf, tile, values):
        self._check_tile(tile)
        grid = self._check_values(tile, values).reshape(tile.size.values, order="F")
        r0, c0 = tile.absolute.values
        lo, hi = self._span(tile)
        i = np.arange(lo, hi)
        off = np.ones(grid.shape, dtype=bool)
        off[i - r0, i - c0] = False
        if np.any(grid[off] != 0):
            raise ValueError("Diagonal layout cannot store nonzero off-diagonal values")
        buf[lo:hi] = grid[i - r0, i - c0].astype(self.storage_dtype, copy=False)


@dataclass(frozen=True)
class Zero(Layout):
    """All-zero matrix that is never materialised: no buffer, no loads, no stores."""

    element_type: np.dtype
    names: tuple
    extents: tuple

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))

    def physical_size(self) -> int:
        return 0

    @property
    def storage_dtype(self):
        return dtypes.storage_scalar(self.element_type)

    def lower(self) -> LayoutDesc:
        return LayoutDesc(KIND_ZERO, PAIR_NONE, dtypes.scalar_name(self.element_type),
                          tuple(((e, 0),) for e in self.extents), 0, 0)

    def load_count(self, tile):
        return 0

    store_count = load_count

    def load(self, buf, tile):
        self._check_tile(tile)
        return np.zeros(tile.volume, dtype=self.element_type)

    def store(self, buf, tile, values):
        self._check_tile(tile)
        self._check_values(tile, values)


class _PairLayout(Layout):
    """Shared code for two-plane (complex / dual) element types."""

    @property
    def storage_dtype(self):
        return dtypes.storage_scalar(self.element_type)

    def physical_size(self) -> int:
        return 2 * _volume(self.extents)

    def digits(self):
        return _dense_digits(self.extents, self.order)

    def _planes_of(self, buf, tile):
        raise NotImplementedError

    def load(self, buf, tile):
        off = self._offsets(tile)
        p0, p1 = self._plane_offsets(off)
        _, _, combine = dtypes.pair_planes(self.element_type)
        buf = np.asarray(buf)
        return combine(buf[p0], buf[p1])

    def store(self, buf, tile, values):
        values = self._check_values(tile, values).astype(self.element_type, copy=False)
        off = self._offsets(tile)
        p0, p1 = self._plane_offsets(off)
        _, split, _ = dtypes.pair_planes(self.element_type)
        v0, v1 = split(values)
        buf[p0] = v0
        buf[p1] = v1


@dataclass(frozen=True)
class InterleavedComplex(_PairLayout):
    """(re, im) / (value, epsilon) adjacent per element; ``order`` F or C over elements."""

    element_type: np.dtype
    names: tuple
    extents: tuple
    order: str = "F"

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        dtypes.pair_planes(self.element_type)  # validates the pair type

    def _plane_offsets(self, off):
        return 2 * off, 2 * off + 1

    def lower(self) -> LayoutDesc:
        base = super().lower()
        return LayoutDesc(KIND_STRIDED, PAIR_INTERLEAVED, base.scalar, base.digits, 1,
                          self.physical_size())


@dataclass(frozen=True)
class SplitComplex(_PairLayout):
    """Two planes in one buffer: all first components, then all second components."""

    element_type: np.dtype
    names: tuple
    extents: tuple
    order: str = "F"

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        dtypes.pair_planes(self.element_type)

    def _plane_offsets(self, off):
        return off, off + _volume(self.extents)

    def lower(self) -> LayoutDesc:
        base = super().lower()
        return LayoutDesc(KIND_STRIDED, PAIR_SPLIT, base.scalar, base.digits,
                          _volume(self.extents), self.physical_size())


@dataclass(frozen=True)
class StridedPermutation(Layout):
    """Logical dims mapped onto permuted (and optionally split) storage dims.

    ``dim_map`` sends each logical dim to an ordered (fastest-first) group of
    ``(storage_name, extent)``; ``storage_order`` lists storage dims in
    column-major order.  This is the fused-transposition (GETT) layout of
    reference ``layouts.py:435-506``; it lowers directly to a digit list.
    """

    element_type: np.dtype
    names: tuple
    extents: tuple
    dim_map: dict
    storage_order: tuple
    _strides: dict = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        object.__setattr__(self, "element_type", np.dtype(self.element_type))
        object.__setattr__(self, "names", tuple(self.names))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        object.__setattr__(self, "storage_order", tuple(self.storage_order))
        sizes = {}
        for name, extent in zip(self.names, self.extents):
            group = self.dim_map.get(name)
            if not group:
                raise ValueError(f"dim_map missing logical dimension {name!r}")
            prod = 1
            for sname, sext in group:
                sizes[sname] = int(sext)
                prod *= int(sext)
            if prod != extent:
                raise ValueError(f"storage extents for {name!r} multiply to {prod}, "
                                 f"expected {extent}")
        if set(sizes) != set(self.storage_order):
            raise ValueError("storage_order must list exactly the mapped storage dims")
        strides, s = {}, 1
        for sname in self.storage_order:
            strides[sname] = s
            s *= sizes[sname]
        object.__setattr__(self, "_strides", strides)

    @classmethod
    def pure(cls, element_type, names, extents, storage_order):
        dim_map = {n: ((n, e),) for n, e in zip(names, extents)}
        return cls(element_type, tuple(names), tuple(extents), dim_map, tuple(storage_order))

    def physical_size(self) -> int:
        return _volume(self.extents)

    def digits(self):
        return [[(int(sext), self._strides[sname]) for sname, sext in self.dim_map[name]]
                for name in self.names]

    def _flat_indices(self, tile: Tile) -> np.ndarray:
        return self._offsets(tile)


# ---- builders for shared (scratch) layouts -----------------------------------

def col_major(element_type):
    def build(names, extents):
        return ColMajor(element_type, tuple(names), tuple(extents))

    build.kind = ("col_major", np.dtype(element_type))
    return build


def row_major(element_type):
    def build(names, extents):
        return RowMajor(element_type, tuple(names), tuple(extents))

    build.kind = ("row_major", np.dtype(element_type))
    return build


def padded(inner_builder, pad: int):
    def build(names, extents):
        return Padded(inner_builder(names, extents), pad)

    build.kind = ("padded", getattr(inner_builder, "kind", None), pad)
    return build


def interleaved_pairs(element_type):
    def build(names, extents):
        return InterleavedComplex(element_type, tuple(names), tuple(extents))

    build.kind = ("interleaved_pairs", np.dtype(element_type))
    return build


def split_pairs(element_type):
    def build(names, extents):
        return SplitComplex(element_type, tuple(names), tuple(extents))

    build.kind = ("split_pairs", np.dtype(element_type))
    return build
