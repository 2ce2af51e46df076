"""ctypes binding of libshampoo.so (include/shampoo.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  The binding
fails loudly (ImportError) if the in-tree library has not been built."""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libshampoo.so")

BLOCK_DTYPE = np.dtype([
    ("tensor_id", "<i4"), ("reserved", "<i4"), ("row0", "<i8"), ("col0", "<i8"),
    ("rows", "<i4"), ("cols", "<i4"), ("p_left", "<i4"), ("p_right", "<i4"),
    ("r_left", "<i4"), ("r_right", "<i4"), ("owner_left", "<i4"), ("owner_right", "<i4"), ("left_off", "<i8"), ("right_off", "<i8"),
    ("left_ld", "<i4"), ("right_ld", "<i4"),
])
GROUP_DTYPE = np.dtype([("owner", "<i4"), ("n", "<i4"), ("p", "<i4"), ("count", "<i4"),
                        ("offset", "<i8"), ("stride", "<i8"), ("r", "<i4"), ("reserved", "<i4")])
TENSOR_DTYPE = np.dtype([("G", "<u8"), ("D", "<u8"), ("P", "<u8"), ("ldg", "<i8"), ("ldd", "<i8"),
                         ("ldp", "<i8"), ("m", "<i8"), ("n", "<i8")])
STATE_DTYPE = np.dtype([("W", "<u8"), ("M", "<u8"), ("Pm", "<u8"), ("ldw", "<i8"), ("ldm", "<i8"), ("ldpm", "<i8")])
TTENSOR_DTYPE = np.dtype([("G", "<u8"), ("D", "<u8"), ("P", "<u8"), ("dims", "<i8", (4,)), ("order", "<i4"),
                          ("reserved", "<i4")])
TBLOCK_DTYPE = np.dtype([("tensor_id", "<i4"), ("order", "<i4"), ("origin", "<i8", (4,)), ("extent", "<i4", (4,)),
                         ("p", "<i4", (4,)), ("owner", "<i4", (4,)), ("ld", "<i4", (4,)), ("off", "<i8", (4,))])
ROOT_INFO_DTYPE = np.dtype([("iters", "<i4"), ("status", "<i4"), ("lambda_max", "<f8"), ("err", "<f8")])
assert BLOCK_DTYPE.itemsize == 80 and GROUP_DTYPE.itemsize == 40
assert TENSOR_DTYPE.itemsize == 64 and ROOT_INFO_DTYPE.itemsize == 24
assert TTENSOR_DTYPE.itemsize == 64 and TBLOCK_DTYPE.itemsize == 136

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "CUDA", 4: "WORKSPACE", 5: "CAPACITY"}

EXPORTED = [
    "shampoo_abi_version", "shampoo_last_error", "shampoo_last_launch_count", "shampoo_plan", "shampoo_plan_layers",
    "shampoo_stats_workspace_bytes", "shampoo_stats_update",
    "shampoo_root_workspace_bytes", "shampoo_inverse_pth_root_batched", "shampoo_inverse_root_rational_batched",
    "shampoo_inverse_pth_root_batched_hybrid", "shampoo_root_ozaki_workspace_bytes",
    "shampoo_inverse_pth_root_batched_ozaki", "shampoo_profile_begin", "shampoo_profile_end",
    "shampoo_profile_launch_ms", "shampoo_ozaki_iteration_slices", "shampoo_root_auto_workspace_bytes",
    "shampoo_inverse_pth_root_batched_auto",
    "shampoo_root_residual_workspace_bytes", "shampoo_root_residual_batched",
    "shampoo_precondition_workspace_bytes", "shampoo_precondition", "shampoo_precondition_split",
    "shampoo_tf32_split",
    "shampoo_momentum_workspace_bytes", "shampoo_momentum_step",
    "shampoo_tensor_plan", "shampoo_tensor_stats_workspace_bytes", "shampoo_tensor_stats_update",
    "shampoo_tensor_precondition_workspace_bytes", "shampoo_tensor_precondition",
]


class ShampooError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libshampoo {STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_sz = ctypes.c_size_t


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2002_09018_b200/build.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.shampoo_abi_version.restype = ctypes.c_int
    L.shampoo_last_error.restype = ctypes.c_char_p
    L.shampoo_last_launch_count.restype = _i64
    L.shampoo_plan.argtypes = [_vp, _i32, _i32, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp]
    L.shampoo_plan.restype = ctypes.c_int
    L.shampoo_plan_layers.argtypes = [_vp, _i32, _i32, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp,
                                      _vp]
    L.shampoo_plan_layers.restype = ctypes.c_int
    L.shampoo_stats_workspace_bytes.argtypes = [_vp, _i32, _i32]
    L.shampoo_stats_workspace_bytes.restype = _sz
    L.shampoo_stats_update.argtypes = [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _dbl, _dbl, _vp, _vp, _vp, _sz, _vp]
    L.shampoo_stats_update.restype = ctypes.c_int
    L.shampoo_root_workspace_bytes.argtypes = [_i32, _i32, _i32, _i32]
    L.shampoo_root_workspace_bytes.restype = _sz
    L.shampoo_inverse_pth_root_batched.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _dbl, _dbl,
                                                   _i32, _i32, _vp, _vp, _sz, _vp]
    L.shampoo_inverse_pth_root_batched.restype = ctypes.c_int
    L.shampoo_inverse_root_rational_batched.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _i32,
                                                        _dbl, _dbl, _i32, _i32, _vp, _vp, _sz, _vp]
    L.shampoo_inverse_root_rational_batched.restype = ctypes.c_int
    L.shampoo_inverse_pth_root_batched_hybrid.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _dbl,
                                                          _dbl, _i32, _i32, _i32, _vp, _vp, _sz, _vp]
    L.shampoo_inverse_pth_root_batched_hybrid.restype = ctypes.c_int
    L.shampoo_root_ozaki_workspace_bytes.argtypes = [_i32, _i32, _i32, _i32]
    L.shampoo_root_ozaki_workspace_bytes.restype = _sz
    L.shampoo_inverse_pth_root_batched_ozaki.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _dbl,
                                                         _dbl, _i32, _i32, _i32, _dbl, _vp, _vp, _sz, _vp]
    L.shampoo_inverse_pth_root_batched_ozaki.restype = ctypes.c_int
    L.shampoo_root_auto_workspace_bytes.argtypes = [_i32, _i32, _i32, _i32]
    L.shampoo_root_auto_workspace_bytes.restype = _sz
    L.shampoo_inverse_pth_root_batched_auto.argtypes = L.shampoo_inverse_pth_root_batched_ozaki.argtypes
    L.shampoo_inverse_pth_root_batched_auto.restype = ctypes.c_int
    L.shampoo_root_residual_workspace_bytes.argtypes = [_i32, _i32, _i32]
    L.shampoo_root_residual_workspace_bytes.restype = _sz
    L.shampoo_root_residual_batched.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i32, _dbl, _vp, _vp,
                                                _vp, _sz, _vp]
    L.shampoo_root_residual_batched.restype = ctypes.c_int
    L.shampoo_precondition_workspace_bytes.argtypes = [_vp, _i32, _vp, _i32]
    L.shampoo_precondition_workspace_bytes.restype = _sz
    L.shampoo_precondition.argtypes = [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.shampoo_precondition.restype = ctypes.c_int
    L.shampoo_precondition_split.argtypes = [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.shampoo_precondition_split.restype = ctypes.c_int
    L.shampoo_tf32_split.argtypes = [_vp, _vp, _i64, _vp]
    L.shampoo_tf32_split.restype = ctypes.c_int
    L.shampoo_momentum_workspace_bytes.argtypes = [_i32]
    L.shampoo_momentum_workspace_bytes.restype = _sz
    L.shampoo_momentum_step.argtypes = [_vp, _vp, _i32, _vp, _i32, _dbl, _dbl, _i32, _vp, _vp, _sz, _vp]
    L.shampoo_momentum_step.restype = ctypes.c_int
    L.shampoo_tensor_plan.argtypes = [_vp, _vp, _i32, _i32, _i64, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp]
    L.shampoo_tensor_plan.restype = ctypes.c_int
    L.shampoo_tensor_stats_workspace_bytes.argtypes = [_vp, _i32, _vp, _i32, _i32]
    L.shampoo_tensor_stats_workspace_bytes.restype = _sz
    L.shampoo_tensor_stats_update.argtypes = [_vp, _i32, _vp, _i32, _i32, _vp, _dbl, _dbl, _vp, _vp, _vp, _sz, _vp]
    L.shampoo_tensor_stats_update.restype = ctypes.c_int
    L.shampoo_tensor_precondition_workspace_bytes.argtypes = [_vp, _i32, _vp, _i32]
    L.shampoo_tensor_precondition_workspace_bytes.restype = _sz
    L.shampoo_tensor_precondition.argtypes = [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    L.shampoo_tensor_precondition.restype = ctypes.c_int
    L.shampoo_profile_begin.restype = ctypes.c_int
    L.shampoo_profile_end.argtypes = [ctypes.c_char_p, _vp, _vp]
    L.shampoo_profile_end.restype = ctypes.c_int
    L.shampoo_profile_launch_ms.argtypes = [ctypes.c_char_p, _vp, ctypes.c_int64, _vp]
    L.shampoo_profile_launch_ms.restype = ctypes.c_int
    L.shampoo_ozaki_iteration_slices.argtypes = [_i32, _i32, _i32, _dbl, _dbl, _i32]
    L.shampoo_ozaki_iteration_slices.restype = ctypes.c_int
    if L.shampoo_abi_version() != 4:
        raise ImportError("libshampoo ABI version mismatch")
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        raise ShampooError(rc, lib().shampoo_last_error().decode())


def last_launch_count() -> int:
    return int(lib().shampoo_last_launch_count())
