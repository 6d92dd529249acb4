"""ctypes declarations of libmk.so (include/mk.h).  Argument marshalling only.

The library is built in-tree by ``paper_1904_08755_b200/build.py`` (called from
``__graft_entry__.build()``).  There is no fallback: if libmk.so is missing or cannot be
loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import os

# MK_LIBRARY overrides the library path (development builds, e.g. the MK_TRACE variant).
SO = Path(os.environ.get("MK_LIBRARY", Path(__file__).resolve().parent / "libmk.so"))

MK_MAX_REGION = 8
STATUS = {
    0: "MK_OK", 1: "MK_ERR_INVALID_ARGUMENT", 2: "MK_ERR_DIMENSION_MISMATCH", 3: "MK_ERR_SHAPE_MISMATCH",
    4: "MK_ERR_NONFINITE_INPUT", 5: "MK_ERR_COORD_RANGE", 6: "MK_ERR_STRIDE", 7: "MK_ERR_UNSUPPORTED",
    8: "MK_ERR_OUT_OF_MEMORY", 9: "MK_ERR_CUDA",
}
F32, BF16 = 0, 1
HYPERCUBE, HYPERCROSS, HYBRID, CUSTOM = 0, 1, 2, 3
POOL_MAX, POOL_AVG, POOL_SUM = 0, 1, 2


class MkRegion(ctypes.Structure):
    _fields_ = [
        ("type", ctypes.c_int32),
        ("D", ctypes.c_int32),
        ("size", ctypes.c_int32 * MK_MAX_REGION),
        ("dilation", ctypes.c_int32 * MK_MAX_REGION),
        ("temporal_axis", ctypes.c_int32),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("n_offsets", ctypes.c_int32),
    ]


EXPORTS = [
    "mk_context_create", "mk_context_destroy",
    "mk_coords_quantize", "mk_coords_quantize_deferred", "mk_coords_create", "mk_coords_info", "mk_coords_export", "mk_coords_lookup",
    "mk_coords_labels", "mk_coords_expand",
    "mk_coords_stride", "mk_coords_destroy",
    "mk_region_offsets",
    "mk_kmap_build", "mk_kmap_info", "mk_kmap_export", "mk_kmap_destroy",
    "mk_conv_forward", "mk_conv_forward_fused", "mk_conv_backward", "mk_conv_transpose_forward", "mk_conv_transpose_backward",
    "mk_pool_forward", "mk_pool_backward", "mk_global_pool", "mk_crf_infer", "mk_crf_backward",
    "mk_last_error_message", "mk_last_error_row", "mk_kernel_launch_count", "mk_debug_sort_perm",
]


def load() -> ctypes.CDLL:
    if not SO.exists():
        raise ImportError(f"{SO} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(str(SO))
    P, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "mk_context_create": [ctypes.c_int, P, P, P, PP],
        "mk_coords_quantize": [P, P, P, i64, i32, f32, P, PP, P, P],
        "mk_coords_quantize_deferred": [P, P, P, i64, i32, f32, P, PP, P, P],
        "mk_coords_create": [P, P, i64, i32, P, P, PP, P],
        "mk_coords_info": [P, P, P, P],
        "mk_coords_export": [P, P, P],
        "mk_coords_lookup": [P, P, i64, P, P],
        "mk_coords_labels": [P, P, P, i64, i64, i32, P, P],
        "mk_coords_expand": [P, P, ctypes.POINTER(MkRegion), P, P, PP],
        "mk_coords_stride": [P, P, P, P, PP],
        "mk_region_offsets": [ctypes.POINTER(MkRegion), P, P],
        "mk_kmap_build": [P, P, P, ctypes.POINTER(MkRegion), i32, P, PP],
        "mk_kmap_info": [P, P, P, P, P],
        "mk_kmap_export": [P, P, P, P, P],
        "mk_conv_forward": [P, P, P, i32, P, P, i32, ctypes.c_int, ctypes.c_int, P],
        "mk_conv_forward_fused": [P, P, P, i32, P, P, i32, ctypes.c_int, ctypes.c_int, P, P, P, i32, P],
        "mk_pool_forward": [P, P, i32, P, i32, ctypes.c_int, P, P, P],
        "mk_pool_backward": [P, P, i32, P, i32, ctypes.c_int, P, P, P],
        "mk_global_pool": [P, P, i32, P, i32, ctypes.c_int, i32, P, P],
        "mk_crf_infer": [P, P, P, P, i32, i32, P, P],
        "mk_crf_backward": [P, P, P, P, i32, i32, P, P, P, P],
        "mk_debug_sort_perm": [P, P, i64, i32, P, P],
        "mk_conv_transpose_forward": [P, P, P, i32, P, P, i32, ctypes.c_int, ctypes.c_int, P],
        "mk_conv_backward": [P, P, P, P, P, i32, i32, ctypes.c_int, P, P, P],
        "mk_conv_transpose_backward": [P, P, P, P, P, i32, i32, ctypes.c_int, P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name in ("mk_context_destroy", "mk_coords_destroy", "mk_kmap_destroy"):
        getattr(L, name).argtypes = [P]
        getattr(L, name).restype = None
    L.mk_last_error_message.restype = ctypes.c_char_p
    L.mk_last_error_message.argtypes = []
    L.mk_last_error_row.restype = ctypes.c_int64
    L.mk_last_error_row.argtypes = []
    L.mk_kernel_launch_count.restype = ctypes.c_int64
    L.mk_kernel_launch_count.argtypes = []
    return L
