"""ctypes binding of libai3.so (include/ai3.h) -- argument marshalling only.

Every entry point here forwards to the C ABI with the same name; no arithmetic
of the convolution happens in Python.  If the shared library is missing the
import of any compute entry point raises ``Ai3LibraryMissing`` -- there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libai3.so")

# ai3_status
OK, ERR_INVALID_ARGUMENT, ERR_SHAPE, ERR_UNSUPPORTED, ERR_UNKNOWN_ALGORITHM, ERR_WORKSPACE, ERR_CUDA = range(7)
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SHAPE", 3: "UNSUPPORTED", 4: "UNKNOWN_ALGORITHM",
                5: "WORKSPACE", 6: "CUDA"}
# ai3_algo
ALGO_GUESS, ALGO_DIRECT, ALGO_GEMM, ALGO_IMPLICIT_GEMM, ALGO_WINOGRAD = 0, 1, 2, 3, 4
ALGO_IMPLICIT_PRECOMP_GEMM, ALGO_SMM, ALGO_KN2ROW, ALGO_CUSTOM, ALGO_BENCHMARK = 5, 6, 7, 8, 9
NUM_ALGOS = 10
# ai3_dtype / ai3_math / ai3_layout
F32, BF16 = 0, 1
MATH_STRICT, MATH_TF32 = 0, 1
NCHW, NHWC = 0, 1

# every symbol include/ai3.h declares (checked by tests/test_abi.py)
EXPORTS = ["ai3_version", "ai3_last_error", "ai3_algo_name", "ai3_algo_from_name", "ai3_conv2d_output_shape",
           "ai3_conv2d_supported", "ai3_conv2d_guess", "ai3_conv2d_workspace_size", "ai3_conv2d",
           "ai3_conv2d_plan_weight_bytes", "ai3_conv2d_plan_create", "ai3_conv2d_plan_algo",
           "ai3_conv2d_plan_workspace_size", "ai3_conv2d_plan_num_launches", "ai3_conv2d_plan_execute",
           "ai3_conv2d_plan_execute_host", "ai3_conv2d_plan_destroy", "ai3_register_conv2d",
           "ai3_unregister_conv2d", "ai3_custom_conv2d_count", "ai3_conv2d_resolve", "ai3_conv2d_custom",
           "ai3_conv2d_plan_set_relu", "ai3_linear_plan_weight_bytes", "ai3_linear_plan_create", "ai3_relu",
           "ai3_pool2d_output_shape", "ai3_maxpool2d", "ai3_avgpool2d", "ai3_adaptive_avgpool2d",
           "ai3_layout_copy", "ai3_conv2d_autotune_scratch_bytes", "ai3_conv2d_autotune",
           "ai3_conv2d_autotune_clear", "ai3_conv2d_plans_execute_host", "ai3_conv2d_plan_set_maxpool2x2"]


class Ai3LibraryMissing(RuntimeError):
    pass


class Params(ctypes.Structure):
    _fields_ = [("out_channels", ctypes.c_int64), ("kernel", ctypes.c_int32 * 2), ("stride", ctypes.c_int32 * 2),
                ("padding", ctypes.c_int32 * 2), ("dilation", ctypes.c_int32 * 2), ("groups", ctypes.c_int32),
                ("has_bias", ctypes.c_int32)]


class Tensor4d(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("n", ctypes.c_int64), ("c", ctypes.c_int64), ("h", ctypes.c_int64),
                ("w", ctypes.c_int64), ("dtype", ctypes.c_int32), ("layout", ctypes.c_int32)]


class PoolParams(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32 * 2), ("stride", ctypes.c_int32 * 2), ("padding", ctypes.c_int32 * 2),
                ("dilation", ctypes.c_int32 * 2), ("ceil_mode", ctypes.c_int32),
                ("count_include_pad", ctypes.c_int32), ("divisor_override", ctypes.c_int32)]


# ai3_conv2d_custom_fn (include/ai3.h)
CUSTOM_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(Tensor4d), ctypes.POINTER(Tensor4d), ctypes.c_void_p,
                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                             ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.POINTER(Tensor4d),
                             ctypes.c_void_p, ctypes.c_void_p)

_lib = None


def select_library(path: str) -> None:
    """Load `path` instead of the in-tree libai3.so (the developer build libai3_dev.so, or the
    deliberately faulty libai3_mutant.so of the mutation test).  Must precede the first load;
    no environment variable can redirect the product's library."""
    global LIB_PATH
    if _lib is not None and os.path.abspath(path) != os.path.abspath(LIB_PATH):
        raise RuntimeError(f"libai3 already loaded from {LIB_PATH}")
    LIB_PATH = path


def load():
    """Load libai3.so (building nothing).  Raises Ai3LibraryMissing if absent."""
    global _lib, LIB_PATH
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise Ai3LibraryMissing(f"{LIB_PATH} not found: build it with `python -m paper_2410_08300_b200.build` "
                                "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    i32, i64, sz, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
    i64x4 = ctypes.POINTER(ctypes.c_int64)
    pp = ctypes.POINTER(Params)
    i32x2 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "ai3_version": ([], ctypes.c_int),
        "ai3_last_error": ([], ctypes.c_char_p),
        "ai3_algo_name": ([ctypes.c_int], ctypes.c_char_p),
        "ai3_algo_from_name": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "ai3_conv2d_output_shape": ([pp, i64x4, i64x4], ctypes.c_int),
        "ai3_conv2d_supported": ([pp, i64x4, ctypes.c_int, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "ai3_conv2d_guess": ([pp, i64x4, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "ai3_conv2d_workspace_size": ([pp, i64x4, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32, i32,
                                       ctypes.POINTER(sz)], ctypes.c_int),
        "ai3_conv2d": ([ctypes.POINTER(Tensor4d), ctypes.POINTER(Tensor4d), vp, i32x2, i32x2, i32x2, i32,
                        ctypes.c_int, ctypes.c_int, ctypes.POINTER(Tensor4d), vp, sz, vp], ctypes.c_int),
        "ai3_conv2d_plan_weight_bytes": ([pp, i64x4, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(sz)],
                                         ctypes.c_int),
        "ai3_conv2d_plan_create": ([pp, i64x4, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32, i32, vp, vp, vp, sz,
                                    vp, ctypes.POINTER(vp)], ctypes.c_int),
        "ai3_conv2d_plan_algo": ([vp], ctypes.c_int),
        "ai3_conv2d_plan_workspace_size": ([vp], sz),
        "ai3_conv2d_plan_num_launches": ([vp], ctypes.c_int),
        "ai3_conv2d_plan_execute": ([vp, vp, vp, vp, sz, vp], ctypes.c_int),
        "ai3_conv2d_plan_execute_host": ([vp, vp, vp, vp, vp, vp, sz, vp], ctypes.c_int),
        "ai3_conv2d_plan_destroy": ([vp], None),
        "ai3_register_conv2d": ([ctypes.c_char_p, vp, vp, i32], ctypes.c_int),
        "ai3_unregister_conv2d": ([ctypes.c_char_p], ctypes.c_int),
        "ai3_custom_conv2d_count": ([], i32),
        "ai3_conv2d_resolve": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, sz], ctypes.c_int),
        "ai3_conv2d_custom": ([ctypes.c_char_p, ctypes.POINTER(Tensor4d), ctypes.POINTER(Tensor4d), vp, i32x2, i32x2,
                               i32x2, i32, ctypes.POINTER(Tensor4d), vp], ctypes.c_int),
        "ai3_conv2d_plan_set_relu": ([vp, i32], ctypes.c_int),
        "ai3_conv2d_plan_set_maxpool2x2": ([vp, i32], ctypes.c_int),
        "ai3_linear_plan_weight_bytes": ([i64, i64, i64, i32, ctypes.c_int, ctypes.c_int, ctypes.POINTER(sz)],
                                         ctypes.c_int),
        "ai3_linear_plan_create": ([i64, i64, i64, ctypes.c_int, ctypes.c_int, vp, vp, vp, sz, vp,
                                    ctypes.POINTER(vp)], ctypes.c_int),
        "ai3_relu": ([vp, vp, i64, i32, vp], ctypes.c_int),
        "ai3_pool2d_output_shape": ([ctypes.POINTER(PoolParams), i64x4, i64x4], ctypes.c_int),
        "ai3_maxpool2d": ([ctypes.POINTER(Tensor4d), ctypes.POINTER(PoolParams), ctypes.POINTER(Tensor4d), vp],
                          ctypes.c_int),
        "ai3_avgpool2d": ([ctypes.POINTER(Tensor4d), ctypes.POINTER(PoolParams), ctypes.POINTER(Tensor4d), vp],
                          ctypes.c_int),
        "ai3_adaptive_avgpool2d": ([ctypes.POINTER(Tensor4d), ctypes.POINTER(Tensor4d), vp], ctypes.c_int),
        "ai3_layout_copy": ([ctypes.POINTER(Tensor4d), ctypes.POINTER(Tensor4d), vp], ctypes.c_int),
        "ai3_conv2d_autotune_scratch_bytes": ([pp, i64x4, ctypes.c_int, ctypes.c_int, i32, i32, ctypes.POINTER(sz)],
                                              ctypes.c_int),
        "ai3_conv2d_autotune": ([pp, i64x4, ctypes.c_int, ctypes.c_int, i32, i32, vp, vp, vp, vp, vp, sz, i32, vp,
                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
        "ai3_conv2d_autotune_clear": ([], None),
        "ai3_conv2d_plans_execute_host": ([i32, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                           ctypes.POINTER(vp), ctypes.POINTER(vp), vp, sz, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    return load().ai3_last_error().decode()


def params(out_channels, kernel, stride, padding, dilation, groups, has_bias) -> Params:
    p = Params()
    p.out_channels = int(out_channels)
    p.kernel[:] = [int(kernel[0]), int(kernel[1])]
    p.stride[:] = [int(stride[0]), int(stride[1])]
    p.padding[:] = [int(padding[0]), int(padding[1])]
    p.dilation[:] = [int(dilation[0]), int(dilation[1])]
    p.groups = int(groups)
    p.has_bias = 1 if has_bias else 0
    return p


def shape4(s) -> ctypes.Array:
    return (ctypes.c_int64 * 4)(*[int(v) for v in s])
