"""User-defined convolution algorithms.

    ai3.register_conv2d("my_conv", fn, use_as_default=False)
    ai3.swap_conv2d(model, "my_conv")      # by name
    ai3.swap_conv2d(model, "custom")       # the unique registered algorithm
    ai3.swap_conv2d(model, "default")      # the registered default, else the `guess` rule

The registry lives in libai3 (``ai3_register_conv2d``); every custom call is
dispatched by the C ABI (``ai3_conv2d_custom``) through the registered function
pointer.  ``fn`` is either

* a native ``ai3_conv2d_custom_fn`` (a ctypes function pointer or its integer address,
  e.g. from a user's shared library -- the paper's C++ path), or
* a Python callable ``fn(x, weight, bias, stride, padding, dilation, groups, out)``
  receiving zero-copy torch views of the operands (``out`` is the caller-allocated
  result); it writes ``out`` (or returns a tensor that is copied into it).  A ctypes
  trampoline adapts it to the native signature.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib

_KEEPALIVE = {}  # name -> trampoline (a ctypes callback must outlive its registration)


class _CudaView:
    """Minimal __cuda_array_interface__ exporter for a borrowed device pointer."""

    def __init__(self, ptr: int, shape, strides_bytes, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": tuple(int(v) for v in strides_bytes)}


def _view(d: _lib.Tensor4d, device) -> torch.Tensor:
    """Zero-copy logical-NCHW torch view of an ai3_tensor4d (NCHW or NHWC storage)."""
    e = 2 if d.dtype == _lib.BF16 else 4
    n, c, h, w = d.n, d.c, d.h, d.w
    if d.layout == _lib.NHWC:
        strides = (h * w * c * e, e, w * c * e, c * e)
    else:
        strides = (c * h * w * e, h * w * e, w * e, e)
    ts = "<i2" if d.dtype == _lib.BF16 else "<f4"
    t = torch.as_tensor(_CudaView(d.data, (n, c, h, w), strides, ts), device=device)
    return t.view(torch.bfloat16) if d.dtype == _lib.BF16 else t


def _trampoline(fn):
    def call(xp, wp, bias, stride, padding, dilation, groups, yp, stream, user):
        try:
            device = torch.device("cuda", torch.cuda.current_device())
            x, w, y = _view(xp.contents, device), _view(wp.contents, device), _view(yp.contents, device)
            b = None
            if bias:
                bd = _lib.Tensor4d(data=bias, n=w.shape[0], c=1, h=1, w=1, dtype=wp.contents.dtype, layout=_lib.NCHW)
                b = _view(bd, device).reshape(-1)
            r = fn(x, w, b, (stride[0], stride[1]), (padding[0], padding[1]), (dilation[0], dilation[1]),
                   int(groups), y)
            if r is not None and r.data_ptr() != y.data_ptr():
                y.copy_(r)
            return _lib.OK
        except Exception as ex:  # surfaces as AI3_ERR_INVALID_ARGUMENT; the message is kept in Python
            _LAST_PY_ERROR[0] = f"{type(ex).__name__}: {ex}"
            return _lib.ERR_INVALID_ARGUMENT
    return _lib.CUSTOM_FN(call)


_LAST_PY_ERROR = [""]


def register_conv2d(name: str, fn, use_as_default: bool = False) -> None:
    """Register a custom conv2d algorithm under ``name`` ("a boolean which
    controls default algorithm selection using the custom algorithm")."""
    from .conv import _check
    lib = _lib.load()
    if isinstance(fn, int):
        ptr, keep = fn, None
    elif isinstance(fn, ctypes._CFuncPtr):  # native function pointer
        ptr, keep = ctypes.cast(fn, ctypes.c_void_p).value, fn
    elif callable(fn):
        keep = _trampoline(fn)
        ptr = ctypes.cast(keep, ctypes.c_void_p).value
    else:
        raise TypeError("fn must be a callable, a ctypes function pointer or an integer address")
    _check(lib.ai3_register_conv2d(name.encode(), ptr, None, 1 if use_as_default else 0))
    _KEEPALIVE[name] = keep


def unregister_conv2d(name: str) -> None:
    from .conv import _check
    _check(_lib.load().ai3_unregister_conv2d(name.encode()))
    _KEEPALIVE.pop(name, None)


def registered_count() -> int:
    return int(_lib.load().ai3_custom_conv2d_count())


def last_python_error() -> str:
    """Message of the last exception raised inside a Python custom algorithm."""
    return _LAST_PY_ERROR[0]
