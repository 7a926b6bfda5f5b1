"""ai3 on B200: fine-grain algorithm selection for forward conv2d (arXiv 2410.08300).

    import paper_2410_08300_b200 as ai3
    y = ai3.conv2d(x, w, b, stride=1, padding=1, algorithm="implicit_gemm")
    ai3.swap_conv2d(model, ["direct", "winograd"])          # in place
    m = ai3.swap_backend(model, {"conv2d": selector})        # traced model

Algorithms: "direct", "gemm" (= "im2col"),
"implicit_gemm", "winograd", "smm", "kn2row", and "guess" (= "auto"; "default" is
the registered default custom algorithm if any, else "guess").
User algorithms: ``register_conv2d(name, fn, use_as_default)``, selected by name or
"custom".  All run as
sm_100a kernels in libai3.so behind the C ABI in include/ai3.h; PyTorch only
provides device memory, streams and the module objects.
"""
from ._lib import Ai3LibraryMissing, LIB_PATH
from .conv import (ALGORITHMS, Ai3Error, ConvPlan, UnknownAlgorithm, UnsupportedConfiguration, algo_id, algo_name, autotune,
                   execute_host_many,
                   check_supported, conv2d, guess, output_shape, supported)
from .custom import register_conv2d, registered_count, unregister_conv2d
from .hooks import Conv2D, Model, swap_backend, swap_conv2d

__all__ = ["ALGORITHMS", "Ai3Error", "Ai3LibraryMissing", "autotune", "execute_host_many", "Conv2D", "ConvPlan", "LIB_PATH", "Model",
           "UnknownAlgorithm", "UnsupportedConfiguration", "algo_id", "algo_name", "check_supported", "conv2d",
           "guess", "output_shape", "register_conv2d", "registered_count", "supported", "swap_backend", "swap_conv2d",
           "unregister_conv2d", "version"]


def version() -> int:
    from . import _lib
    return int(_lib.load().ai3_version())
