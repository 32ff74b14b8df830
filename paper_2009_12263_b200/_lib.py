"""ctypes binding of ``libtk_sm100.so`` (the C ABI in ``include/tk_sm100.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is
no fallback: if the shared object is missing or fails to load, every GEMM entry point
raises ``RuntimeError`` -- the product path never silently runs anywhere but the GPU.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int32, c_int64, c_longlong, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TK_SM100_LIB", os.path.join(HERE, "libtk_sm100.so"))

ABI_VERSION = 2
MAX_DIGITS = 5
MAX_TOPS = 8

LANE_AUTO, LANE_TCGEN05, LANE_SIMT = 0, 1, 2
LANE_NAMES = {LANE_TCGEN05: "tcgen05", LANE_SIMT: "simt"}
PRED_ALWAYS, PRED_DIAGONAL, PRED_MASK = 0, 1, 2
TK_OK, TK_ERR_CONFIG, TK_ERR_CUDA = 0, 1, 2


class TkLayout(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32), ("pair", c_int32), ("scalar", c_int32), ("reserved", c_int32),
        ("ndigits", c_int32 * 2),
        ("ext", (c_int64 * MAX_DIGITS) * 2),
        ("stride", (c_int64 * MAX_DIGITS) * 2),
        ("plane_stride", c_int64), ("size", c_int64),
    ]


class TkTransform(ctypes.Structure):
    _fields_ = [
        ("n", c_int32), ("op", c_int32 * MAX_TOPS), ("promote", c_int32 * MAX_TOPS),
        ("re", c_double * MAX_TOPS), ("im", c_double * MAX_TOPS),
    ]


class TkGemmPlan(ctypes.Structure):
    _fields_ = [
        ("abi_version", c_int32), ("op", c_int32), ("compute", c_int32), ("lane", c_int32),
        ("m", c_int64), ("n", c_int64), ("k", c_int64), ("op_k", c_int64),
        ("block", c_int64 * 3),
        ("a", TkLayout), ("b", TkLayout), ("c", TkLayout), ("d", TkLayout),
        ("t_a", TkTransform), ("t_b", TkTransform), ("t_c", TkTransform),
        ("t_r2s", TkTransform), ("t_s2g", TkTransform),
        ("bias_axis", c_int32), ("bias_scalar", c_int32), ("predicate", c_int32),
        ("reserved", c_int32),
    ]


class TkPlanInfo(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_char * 32)] + [(f, c_int32) for f in (
        "lane", "op", "tile_m", "tile_n", "tile_k", "mma_n", "nsub", "mmas_per_k16", "cluster",
        "stages", "stage_bytes", "cring_bytes", "smem_bytes", "tmem_cols", "grid_ctas", "tiles",
        "units", "sk_parts", "sk_tiles", "sk_tma", "serpentine", "group_m", "pdl", "c_stream",
        "d_tma", "launches", "overlap_kb")] + [("workspace_bytes", c_int64)]


GEMM_EX_ARGTYPES = [c_int, c_int, c_int, c_longlong, c_longlong, c_longlong, c_double,
                    c_double, c_void_p, c_void_p, c_double, c_double, c_void_p]

# every symbol include/tk_sm100.h declares
EXPORTED = ("tk_abi_version", "tk_plan_lane", "tk_workspace_bytes", "tk_gemm", "tk_gemm_ex_raw",
            "tk_gemm_ex_raw_async", "tk_last_launch_count", "tk_last_error", "tk_debug_pair_mhz",
            "tk_debug_pair_ts", "tk_debug_clock_probe", "tk_debug_clock_probe_mhz",
            "tk_gemm_peers", "tk_last_peer_mode", "tk_ipc_handle", "tk_ipc_open", "tk_ipc_close",
            "tk_last_plan_info", "tk_tune_set", "tk_tune_reset", "tk_tune_get")

_lib = None
_load_error = None


def load():
    """Load (once) and return the ctypes library; raise RuntimeError if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise RuntimeError(_load_error)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        _load_error = (f"libtk_sm100.so could not be loaded from {LIB_PATH} ({exc}); build it with "
                       "`python -c 'import __graft_entry__ as g; g.build()'`")
        raise RuntimeError(_load_error) from None
    lib.tk_abi_version.restype = c_int
    lib.tk_plan_lane.argtypes = [ctypes.POINTER(TkGemmPlan)]
    lib.tk_plan_lane.restype = c_int
    lib.tk_workspace_bytes.argtypes = [ctypes.POINTER(TkGemmPlan)]
    lib.tk_workspace_bytes.restype = c_int64
    lib.tk_gemm.argtypes = [ctypes.POINTER(TkGemmPlan), c_void_p, c_void_p, c_void_p, c_void_p,
                            c_void_p, c_void_p, c_void_p, c_int64, c_void_p]
    lib.tk_gemm.restype = c_int
    lib.tk_gemm_peers.argtypes = [ctypes.POINTER(TkGemmPlan), c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int]
    lib.tk_gemm_peers.restype = c_int
    lib.tk_last_peer_mode.restype = c_int
    lib.tk_ipc_handle.argtypes = [c_void_p, c_void_p, ctypes.POINTER(c_int64)]
    lib.tk_ipc_handle.restype = c_int
    lib.tk_ipc_open.argtypes = [c_void_p, ctypes.POINTER(c_void_p)]
    lib.tk_ipc_open.restype = c_int
    lib.tk_ipc_close.argtypes = [c_void_p]
    lib.tk_ipc_close.restype = c_int
    lib.tk_gemm_ex_raw.argtypes = GEMM_EX_ARGTYPES
    lib.tk_gemm_ex_raw.restype = c_int
    lib.tk_gemm_ex_raw_async.argtypes = GEMM_EX_ARGTYPES + [c_void_p]
    lib.tk_gemm_ex_raw_async.restype = c_int
    lib.tk_last_launch_count.restype = c_int
    lib.tk_last_error.restype = ctypes.c_char_p
    lib.tk_last_plan_info.argtypes = [ctypes.POINTER(TkPlanInfo)]
    lib.tk_last_plan_info.restype = c_int
    lib.tk_tune_set.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
    lib.tk_tune_set.restype = c_int
    lib.tk_tune_reset.restype = c_int
    lib.tk_tune_get.argtypes = [ctypes.c_char_p]
    lib.tk_tune_get.restype = c_int
    if lib.tk_abi_version() != ABI_VERSION:
        _load_error = f"libtk_sm100.so ABI {lib.tk_abi_version()} != expected {ABI_VERSION}"
        raise RuntimeError(_load_error)
    _lib = lib
    return lib


def last_error() -> str:
    return load().tk_last_error().decode(errors="replace")


def plan_info() -> dict:
    """The on-chip plan of the last GEMM on this thread (tk_last_plan_info) as a dict."""
    info = TkPlanInfo()
    load().tk_last_plan_info(ctypes.byref(info))
    out = {f: getattr(info, f) for f, _ in TkPlanInfo._fields_}
    out["kernel"] = info.kernel.decode()
    return out


KNOB_UNSET = -(2 ** 31)


def tune(name: str, value=None) -> None:
    """Override one tuning knob (TK_* name); None restores its default.

    Knobs are read from the environment once, when the library loads; this is the only way to
    change one afterwards (the launch path never reads the environment)."""
    rc = load().tk_tune_set(name.encode(), None if value is None else str(value).encode())
    if rc != TK_OK:
        raise ValueError(last_error())
    _drop_prepared()


def _drop_prepared() -> None:
    """Knobs can change the kernel choice and so the workspace a plan needs: forget the lowered
    configurations (kernel._PREPARED) so the next call re-queries tk_workspace_bytes."""
    from . import kernel

    kernel._PREPARED.clear()


def tune_reset() -> None:
    """Drop every override: knobs return to the values the environment gives."""
    load().tk_tune_reset()
    _drop_prepared()


def tune_get(name: str):
    v = load().tk_tune_get(name.encode())
    return None if v == KNOB_UNSET else v
