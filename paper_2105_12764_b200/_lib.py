"""ctypes binding of the C ABI (include/mgrg.h) -- libmgrg.so, built in-tree.

The library is the product: there is no CPU fallback.  If it is missing the
import of anything that computes fails loudly (MissingExtension)."""
from __future__ import annotations

import ctypes
import os

from . import errors

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# MGRG_LIB: an alternative in-tree build (kernel-variant experiments)
LIB_PATH = os.environ.get("MGRG_LIB") or os.path.join(PKG_DIR, "libmgrg.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "mgrg.h")

MGRG_F32 = 4
MGRG_F64 = 8

# Every function include/mgrg.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "mgrg_plan_create", "mgrg_plan_destroy", "mgrg_plan_levels",
    "mgrg_plan_class_offsets", "mgrg_plan_level_shape", "mgrg_plan_sizes",
    "mgrg_decompose", "mgrg_recompose", "mgrg_decompose_host",
    "mgrg_recompose_host", "mgrg_decompose_host_classes", "mgrg_recompose_host_classes",
    "mgrg_decompose_host_begin", "mgrg_decompose_host_end", "mgrg_recompose_host_begin",
    "mgrg_recompose_host_end", "mgrg_host_abort", "mgrg_gpk", "mgrg_masstrans", "mgrg_solve",
    "mgrg_apply_correction", "mgrg_reorder", "mgrg_last_error",
    "mgrg_coop_level", "mgrg_coop_thomas_z", "mgrg_plan_level_buffer",
    "mgrg_cooperative_decompose_host",
    "mgrg_status_name", "mgrg_plan_last_launches", "mgrg_version",
    "mgrg_plan_set_profiling", "mgrg_plan_profile_reset", "mgrg_plan_profile_read",
    "mgrg_crc32", "mgrg_class_crc32", "mgrg_write_refactored", "mgrg_read_refactored",
    "mgrg_compress", "mgrg_free", "mgrg_decompress", "mgrg_crc32_host",
    "mgrg_write_refactored_host", "mgrg_read_refactored_host", "mgrg_compress_host",
    "mgrg_decompress_host",
    "mgrg_device_count", "mgrg_coop_schedule", "mgrg_block_meta_fill",
    "mgrg_comm_unique_id", "mgrg_comm_init", "mgrg_comm_destroy", "mgrg_comm_size",
    "mgrg_comm_allgather_block_meta", "mgrg_plan_set_graphs",
)

KERNEL_KINDS = {0: "dec_level", 1: "thomas_x", 2: "thomas_y", 3: "thomas_z",
                4: "rec_load", 5: "rec_gpk"}


class MissingExtension(ImportError):
    pass


class GridDesc(ctypes.Structure):
    _fields_ = [
        ("ndims", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("shape", ctypes.c_uint64 * 4),
        ("coords", ctypes.c_void_p),
        ("levels", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


MGRG_FLAG_FAST = 1
MGRG_MAX_CLASSES = 32
MGRG_COMM_ID_BYTES = 128


class BlockMeta(ctypes.Structure):
    """mgrg_block_meta (include/mgrg.h): the fixed-size per-block record of
    the block-sharded path's one all-gather."""
    _fields_ = [
        ("block_id", ctypes.c_int64),
        ("rank", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("ndims", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("origin", ctypes.c_uint64 * 4),
        ("shape", ctypes.c_uint64 * 4),
        ("class_bytes", ctypes.c_uint64 * MGRG_MAX_CLASSES),
        ("class_crc32", ctypes.c_uint32 * MGRG_MAX_CLASSES),
        ("checksum", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("decompose_ms", ctypes.c_double),
        ("recompose_ms", ctypes.c_double),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MissingExtension(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(the refactoring path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
        u32 = ctypes.c_uint32
        sig = {
            "mgrg_plan_create": [ctypes.POINTER(GridDesc), ctypes.POINTER(vp)],
            "mgrg_plan_destroy": [vp],
            "mgrg_plan_levels": [vp, ctypes.POINTER(i32)],
            "mgrg_plan_class_offsets": [vp, vp],
            "mgrg_plan_level_shape": [vp, i32, vp],
            "mgrg_plan_sizes": [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)],
            "mgrg_decompose": [vp, vp, vp, vp],
            "mgrg_recompose": [vp, vp, i32, vp, vp],
            "mgrg_decompose_host": [vp, vp, vp],
            "mgrg_recompose_host": [vp, vp, i32, vp],
            "mgrg_decompose_host_classes": [vp, vp, vp],
            "mgrg_recompose_host_classes": [vp, vp, i32, vp],
            "mgrg_decompose_host_begin": [vp, vp],
            "mgrg_decompose_host_end": [vp, vp],
            "mgrg_recompose_host_begin": [vp, vp, i32],
            "mgrg_recompose_host_end": [vp, vp],
            "mgrg_host_abort": [vp],
            "mgrg_gpk": [vp, i32, i32, vp, vp],
            "mgrg_masstrans": [vp, i32, i32, vp, vp, i32, vp, vp],
            "mgrg_solve": [vp, i32, i32, vp, vp],
            "mgrg_apply_correction": [vp, u64, vp, vp, i32, vp],
            "mgrg_reorder": [vp, i32, i32, vp, vp, vp],
            "mgrg_coop_level": [vp, i32, u32, u32, vp, vp, vp],
            "mgrg_coop_thomas_z": [vp, i32, u32, u32, u64, u64, i32, vp, vp, vp, vp],
            "mgrg_plan_level_buffer": [vp, i32, ctypes.POINTER(ctypes.c_void_p)],
            "mgrg_cooperative_decompose_host": [ctypes.POINTER(GridDesc), i32, vp, vp, vp, vp,
                                                ctypes.POINTER(u64)],
            "mgrg_plan_last_launches": [vp, ctypes.POINTER(u64)],
            "mgrg_plan_set_profiling": [vp, i32],
            "mgrg_plan_set_graphs": [vp, i32],
            "mgrg_plan_profile_reset": [vp],
            "mgrg_plan_profile_read": [vp, u64, vp, vp, vp, vp, ctypes.POINTER(u64)],
            "mgrg_crc32": [vp, u64, ctypes.POINTER(ctypes.c_uint32), vp],
            "mgrg_class_crc32": [vp, vp, i32, vp, vp],
            "mgrg_write_refactored": [vp, vp, ctypes.c_char_p, ctypes.POINTER(u64)],
            "mgrg_read_refactored": [vp, ctypes.c_char_p, i32, vp, ctypes.POINTER(i32),
                                     ctypes.POINTER(u64)],
            "mgrg_compress": [vp, vp, ctypes.c_double, i32, ctypes.POINTER(vp),
                              ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_double)],
            "mgrg_decompress": [vp, vp, u64, vp, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)],
            "mgrg_device_count": [ctypes.POINTER(i32)],
            "mgrg_coop_schedule": [vp, i32, ctypes.POINTER(i32), vp],
            "mgrg_block_meta_fill": [vp, vp, ctypes.c_int64, i32, vp, ctypes.c_double,
                                     ctypes.c_double, ctypes.POINTER(BlockMeta), vp],
            "mgrg_comm_unique_id": [vp],
            "mgrg_comm_init": [vp, i32, i32, i32, ctypes.POINTER(vp)],
            "mgrg_comm_destroy": [vp],
            "mgrg_comm_size": [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)],
            "mgrg_comm_allgather_block_meta": [vp, ctypes.POINTER(BlockMeta), i32,
                                               ctypes.POINTER(BlockMeta), vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.mgrg_free.argtypes = [vp]
        L.mgrg_free.restype = None
        L.mgrg_last_error.restype = ctypes.c_char_p
        L.mgrg_last_error.argtypes = []
        L.mgrg_status_name.restype = ctypes.c_char_p
        L.mgrg_status_name.argtypes = [ctypes.c_int]
        L.mgrg_version.restype = ctypes.c_char_p
        L.mgrg_version.argtypes = []
        _lib = L
    return _lib


def check(status: int) -> None:
    """Raise the reference-named exception for a non-zero mgrg_status."""
    if status != 0:
        L = lib()
        msg = L.mgrg_last_error().decode() or L.mgrg_status_name(status).decode()
        raise errors.from_status(status, msg)
