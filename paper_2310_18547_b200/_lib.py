"""ctypes binding of the C-ABI in include/lsg_sgmv.h (libsgmv_b200.so).

The library is built in-tree by ``paper_2310_18547_b200.build`` and loaded from
``paper_2310_18547_b200/lib``.  There is no fallback: if the library is missing
or a call fails, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libsgmv_b200.so")

LSG_OK, LSG_EINVAL, LSG_EUNSUPPORTED, LSG_ECUDA, LSG_ENODEVICE = 0, -1, -2, -3, -4
LSG_F16, LSG_BF16 = 0, 1
(LSG_OPT_PDL, LSG_OPT_FORCE_CLUSTER, LSG_OPT_FORCE_GENERIC, LSG_OPT_FORCE_TILE_ROWS, LSG_OPT_NO_L2_STAGING,
 LSG_OPT_NO_TENSOR_CORES, LSG_OPT_TC_SPLIT, LSG_OPT_NO_ROW_MODE, LSG_OPT_NO_MULTIROW_TILES,
 LSG_OPT_TC_MIN_ROWS, LSG_OPT_TC_LEGACY, LSG_OPT_MMA_MIN_ROWS, LSG_OPT_MMA_FUSED) = 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12
KERNEL_FUSED, KERNEL_SHRINK, KERNEL_EXPAND, KERNEL_BGMV = 0, 1, 2, 3

# Every symbol include/lsg_sgmv.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "lsg_sgmv", "lsg_sgmv_ws", "lsg_sgmv_workspace_size", "lsg_sgmv_shrink", "lsg_sgmv_expand", "lsg_bgmv",
    "lsg_build_segments_workspace", "lsg_build_segments", "lsg_gather_rows", "lsg_scatter_rows",
    "lsg_set_option", "lsg_get_option", "lsg_query_launch", "lsg_status_string",
    "lsg_last_error", "lsg_version", "lsg_set_trace", "lsg_partition_segments", "lsg_sgmv_multi",
    "lsg_dense_lora", "lsg_dense_lora_workspace_size", "lsg_sgmv_ex", "lsg_sgmv_multi_ex",
    "lsg_tp_sgmv", "lsg_tp_sgmv_nccl", "lsg_tp_nccl_workspace_size",
)


class WeightTable(C.Structure):
    """Mirror of ``lsg_weight_table``."""

    _fields_ = [
        ("a_ptr", C.c_void_p),
        ("b_ptr", C.c_void_p),
        ("a_layer_stride", C.c_int64),
        ("b_layer_stride", C.c_int64),
        ("num_slots", C.c_int32),
        ("num_layers", C.c_int32),
        ("h_in", C.c_int32),
        ("h_out", C.c_int32),
        ("rank", C.c_int32),
        ("dtype", C.c_int32),
    ]


class LaunchInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("path", "cluster", "tile_rows", "row_splits", "grid_ctas", "smem_bytes")]


class Site(C.Structure):
    """Mirror of ``lsg_sgmv_site``."""

    _fields_ = [("y", C.c_void_p), ("ldy", C.c_int64), ("x", C.c_void_p), ("ldx", C.c_int64),
                ("tbl", C.POINTER(WeightTable))]


class CallOpts(C.Structure):
    """Mirror of ``lsg_call_opts`` (-1 = process default)."""

    _fields_ = [("pdl", C.c_int32), ("tc_min_rows", C.c_int32), ("no_tensor_cores", C.c_int32),
                ("mma_min_rows", C.c_int32)]


class TpGroup(C.Structure):
    """Mirror of ``lsg_tp_group``."""

    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("y_peer", C.POINTER(C.c_void_p)),
                ("flag_peer", C.POINTER(C.c_void_p))]


class Piece(C.Structure):
    """Mirror of ``lsg_piece``."""

    _fields_ = [(n, C.c_int32) for n in ("rank", "seg", "row0", "row1")]


class LsgError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA extension must be built "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        tp = C.POINTER(WeightTable)
        L.lsg_sgmv.argtypes = [vp, i64, vp, i64, tp, vp, vp, i32, i32, i32, vp]
        L.lsg_sgmv_ws.argtypes = [vp, i64, vp, i64, tp, vp, vp, i32, i32, i32, vp, C.c_size_t, vp]
        L.lsg_sgmv_multi.argtypes = [C.POINTER(Site), i32, vp, vp, i32, i32, i32, vp]
        L.lsg_sgmv_ex.argtypes = [vp, i64, vp, i64, tp, vp, vp, i32, i32, i32, vp, C.c_size_t,
                                  C.POINTER(CallOpts), vp]
        L.lsg_sgmv_multi_ex.argtypes = [C.POINTER(Site), i32, vp, vp, i32, i32, i32, C.POINTER(CallOpts), vp]
        L.lsg_dense_lora.argtypes = [vp, i64, vp, i64, vp, i64, tp, vp, vp, i32, i32, i32, vp, C.c_size_t, vp]
        L.lsg_dense_lora_workspace_size.argtypes = [tp, i32]
        L.lsg_dense_lora_workspace_size.restype = C.c_size_t
        L.lsg_sgmv_workspace_size.argtypes = [tp, i32]
        L.lsg_sgmv_workspace_size.restype = C.c_size_t
        L.lsg_sgmv_shrink.argtypes = [vp, vp, i64, tp, vp, vp, i32, i32, i32, vp]
        L.lsg_sgmv_expand.argtypes = [vp, i64, vp, tp, vp, vp, i32, i32, i32, vp]
        L.lsg_bgmv.argtypes = [vp, i64, vp, i64, tp, vp, i32, i32, vp]
        L.lsg_build_segments_workspace.argtypes = [i32, i32]
        L.lsg_build_segments_workspace.restype = C.c_size_t
        L.lsg_build_segments.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.lsg_gather_rows.argtypes = [vp, i64, vp, i64, vp, i32, i32, vp]
        L.lsg_scatter_rows.argtypes = [vp, i64, vp, i64, vp, i32, i32, vp]
        L.lsg_set_option.argtypes = [i32, i32]
        L.lsg_get_option.argtypes = [i32]
        L.lsg_query_launch.argtypes = [tp, i32, i32, i32, C.POINTER(LaunchInfo)]
        L.lsg_status_string.argtypes = [C.c_int]
        L.lsg_status_string.restype = C.c_char_p
        L.lsg_last_error.restype = C.c_char_p
        L.lsg_version.restype = C.c_int
        L.lsg_set_trace.argtypes = [vp, i32]
        L.lsg_tp_sgmv.argtypes = [C.POINTER(TpGroup), i64, vp, i64, tp, vp, vp, i32, i32, i32, C.c_uint32, vp]
        L.lsg_tp_nccl_workspace_size.argtypes = [i32, i32, i32]
        L.lsg_tp_nccl_workspace_size.restype = C.c_size_t
        L.lsg_tp_sgmv_nccl.argtypes = [vp, i64, vp, i64, tp, vp, vp, i32, i32, i32, i32, i32, vp, vp, C.c_size_t, vp]
        L.lsg_partition_segments.argtypes = [C.POINTER(i32), C.POINTER(i32), i32, i32, i32, i32, i32, i32, i32,
                                             C.POINTER(Piece), C.POINTER(i32)]
        _lib = L
    return _lib


def check(fn: str, status: int) -> None:
    if status != LSG_OK:
        raise LsgError(fn, status, lib().lsg_last_error().decode())


def call(fn: str, *args) -> None:
    check(fn, getattr(lib(), fn)(*args))
