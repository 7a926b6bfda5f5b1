"""ai3's implementations of the other operations of a CNN ("linear,
convolution, flatten, ReLU, and adaptive average, max, and average pooling"), used by
``swap_backend`` to replace every supported PyTorch module and function (
SURVEY §8 row f1).

Each forward is one C-ABI call (include/ai3.h) on the current stream; PyTorch only
allocates the outputs.  Activations keep their memory format: an all-ai3 model runs
NHWC (channels_last) end to end, converting once at its entry.
"""
from __future__ import annotations

import ctypes

import torch
from torch import nn

from . import _lib
from .conv import _check, _desc, _dtype_id, _math_id, _require_cuda, _stream_ptr, _WS, layout_of


def _act_layout(x: torch.Tensor) -> int:
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    return layout_of(x)


def _like(x: torch.Tensor, shape) -> torch.Tensor:
    fmt = torch.channels_last if layout_of(x) == _lib.NHWC and x.dim() == 4 else torch.contiguous_format
    return torch.empty(shape, dtype=x.dtype, device=x.device, memory_format=fmt)


def relu(x: torch.Tensor, inplace: bool = False) -> torch.Tensor:
    """torch.relu semantics (NaN propagates) via ai3_relu."""
    _require_cuda(x)
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    y = x if inplace else torch.empty_like(x)
    _check(_lib.load().ai3_relu(x.data_ptr(), y.data_ptr(), x.numel(), _dtype_id(x.dtype), _stream_ptr(x.device)))
    return y


def _pair(v):
    return (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))


def _pool_params(kernel, stride, padding, dilation, ceil_mode, count_include_pad=True, divisor_override=None):
    p = _lib.PoolParams()
    p.kernel[:] = list(_pair(kernel))
    p.stride[:] = list(_pair(stride if stride is not None and stride != [] else kernel))
    p.padding[:] = list(_pair(padding))
    p.dilation[:] = list(_pair(dilation))
    p.ceil_mode = 1 if ceil_mode else 0
    p.count_include_pad = 1 if count_include_pad else 0
    p.divisor_override = int(divisor_override or 0)
    return p


def _pool(fn_name: str, x: torch.Tensor, prm) -> torch.Tensor:
    _require_cuda(x)
    if x.dim() != 4:
        raise ValueError("ai3 pooling takes 4-D (N, C, H, W) inputs")
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    lib = _lib.load()
    out = (ctypes.c_int64 * 4)()
    _check(lib.ai3_pool2d_output_shape(ctypes.byref(prm), _lib.shape4(x.shape), out))
    y = _like(x, tuple(out))
    lay = layout_of(x)
    xd, yd = _desc(x, lay), _desc(y, lay)
    _check(getattr(lib, fn_name)(ctypes.byref(xd), ctypes.byref(prm), ctypes.byref(yd), _stream_ptr(x.device)))
    return y


def max_pool2d(x, kernel_size, stride=None, padding=0, dilation=1, ceil_mode=False):
    return _pool("ai3_maxpool2d", x, _pool_params(kernel_size, stride, padding, dilation, ceil_mode))


def avg_pool2d(x, kernel_size, stride=None, padding=0, ceil_mode=False, count_include_pad=True,
               divisor_override=None):
    return _pool("ai3_avgpool2d", x, _pool_params(kernel_size, stride, padding, 1, ceil_mode, count_include_pad,
                                                  divisor_override))


def adaptive_avg_pool2d(x: torch.Tensor, output_size) -> torch.Tensor:
    _require_cuda(x)
    if x.dim() != 4:
        raise ValueError("ai3 pooling takes 4-D (N, C, H, W) inputs")
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    oh, ow = _pair(output_size) if not isinstance(output_size, (tuple, list)) else (
        x.shape[2] if output_size[0] is None else int(output_size[0]),
        x.shape[3] if output_size[1] is None else int(output_size[1]))
    if (oh, ow) == tuple(x.shape[2:]):
        return x  # identity (e.g. VGG's 7x7 -> 7x7): no pass over memory
    y = _like(x, (x.shape[0], x.shape[1], oh, ow))
    lay = layout_of(x)
    xd, yd = _desc(x, lay), _desc(y, lay)
    _check(_lib.load().ai3_adaptive_avgpool2d(ctypes.byref(xd), ctypes.byref(yd), _stream_ptr(x.device)))
    return y


def to_layout(x: torch.Tensor, layout: int) -> torch.Tensor:
    """Copy a 4-D activation into NCHW or NHWC with ai3_layout_copy (no-op if already there)."""
    _require_cuda(x)
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    if layout_of(x) == layout and (layout == _lib.NHWC or x.is_contiguous()):
        return x
    fmt = torch.channels_last if layout == _lib.NHWC else torch.contiguous_format
    y = torch.empty(x.shape, dtype=x.dtype, device=x.device, memory_format=fmt)
    xd, yd = _desc(x, layout_of(x)), _desc(y, layout)
    _check(_lib.load().ai3_layout_copy(ctypes.byref(xd), ctypes.byref(yd), _stream_ptr(x.device)))
    return y


def flatten(x: torch.Tensor, start_dim: int = 1, end_dim: int = -1) -> torch.Tensor:
    """torch.flatten: logical (C, H, W) order; an NHWC input is transposed by ai3 first."""
    if x.dim() == 4 and layout_of(x) == _lib.NHWC and not x.is_contiguous():
        x = to_layout(x, _lib.NCHW)
    return torch.flatten(x, start_dim, end_dim)  # a view of a contiguous buffer


# ---------------------------------------------------------------------------- modules
class ReLU(nn.Module):
    def forward(self, x):
        return relu(x)


class MaxPool2D(nn.Module):
    def __init__(self, orig: nn.MaxPool2d):
        super().__init__()
        if getattr(orig, "return_indices", False):
            raise ValueError("MaxPool2d(return_indices=True) is not supported")
        self.args = (orig.kernel_size, orig.stride, orig.padding, orig.dilation, orig.ceil_mode)

    def forward(self, x):
        return max_pool2d(x, *self.args)


class AvgPool2D(nn.Module):
    def __init__(self, orig: nn.AvgPool2d):
        super().__init__()
        self.args = (orig.kernel_size, orig.stride, orig.padding, orig.ceil_mode, orig.count_include_pad,
                     orig.divisor_override)

    def forward(self, x):
        return avg_pool2d(x, *self.args)


class AdaptiveAvgPool2D(nn.Module):
    def __init__(self, orig: nn.AdaptiveAvgPool2d):
        super().__init__()
        self.output_size = orig.output_size

    def forward(self, x):
        return adaptive_avg_pool2d(x, self.output_size)


class Flatten(nn.Module):
    def __init__(self, orig: nn.Flatten | None = None, start_dim: int = 1, end_dim: int = -1):
        super().__init__()
        self.start_dim = orig.start_dim if orig is not None else start_dim
        self.end_dim = orig.end_dim if orig is not None else end_dim

    def forward(self, x):
        return flatten(x, self.start_dim, self.end_dim)


class Linear(nn.Module):
    """nn.Linear on the tcgen05 engine (ai3_linear_plan_create: a 1x1 convolution).

    Applies over the last dimension like nn.Linear.  ``relu``: fused ReLU epilogue.
    ``fused_flatten``: set by swap_backend when this layer's only input is
    torch.flatten(x, 1) of a 4-D activation.  It then takes that activation (N, C, H, W)
    itself: flatten -> linear is exactly the convolution of the (C, H, W) map with the
    weight viewed as (out, C, H, W) and an H x W kernel, so an NHWC activation is read in
    place and the plan's own weight packing (KCRS -> [K][R][S][C]) does the column
    reordering -- no transpose pass and no PyTorch data movement.
    """

    def __init__(self, orig: nn.Linear, math: str = "strict"):
        super().__init__()
        self.weight, self.bias = orig.weight, orig.bias
        self.in_features, self.out_features = orig.in_features, orig.out_features
        self.math = math
        self.relu = False
        self.fused_flatten = False
        self._plans = {}

    def _version(self):
        return (self.weight._version, None if self.bias is None else self.bias._version)

    def _check_dtype(self, x):
        if self.weight.dtype != x.dtype or (self.bias is not None and self.bias.dtype != x.dtype):
            raise TypeError(f"ai3 Linear: input dtype {x.dtype} differs from the parameters' {self.weight.dtype} "
                            "(nn.Linear raises on mixed dtypes too)")

    def _plan(self, batch: int, dtype, device):
        wv = self._version()
        key = (batch, dtype, device)
        ent = self._plans.get(key)
        if ent is not None and ent[0] == wv:
            return ent[1]
        lib = _lib.load()
        w = self.weight.detach()
        b = None if self.bias is None else self.bias.detach()
        if w.device != device:
            raise ValueError("ai3 Linear: parameters and input on different devices")
        w = w.contiguous()
        b = None if b is None else b.contiguous()
        nbytes = ctypes.c_size_t()
        _check(lib.ai3_linear_plan_weight_bytes(batch, self.in_features, self.out_features, int(b is not None),
                                                _dtype_id(dtype), _math_id(self.math), ctypes.byref(nbytes)))
        wbuf = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=device)
        h = ctypes.c_void_p()
        _check(lib.ai3_linear_plan_create(batch, self.in_features, self.out_features, _dtype_id(dtype),
                                          _math_id(self.math), w.data_ptr(), None if b is None else b.data_ptr(),
                                          wbuf.data_ptr(), wbuf.numel(), _stream_ptr(device), ctypes.byref(h)))
        if self.relu:
            _check(lib.ai3_conv2d_plan_set_relu(h, 1))
        plan = _LinearPlan(h, wbuf, (w, b), int(lib.ai3_conv2d_plan_workspace_size(h)))
        self._plans[key] = (wv, plan)
        return plan

    def _flatten_plan(self, x):
        """flatten(x, 1) -> linear as one convolution with an H x W kernel (see class doc)."""
        from .conv import ConvPlan
        N, C, H, W = (int(v) for v in x.shape)
        if C * H * W != self.in_features:
            raise ValueError(f"ai3 Linear: flatten of {tuple(x.shape)} gives {C * H * W} features, "
                             f"the layer takes {self.in_features}")
        lay = layout_of(x)
        key = ("flatten", tuple(x.shape), x.dtype, x.device, lay)
        wv = self._version()
        ent = self._plans.get(key)
        if ent is None or ent[0] != wv:
            w4 = self.weight.detach().view(self.out_features, C, H, W)  # a view: no data moves
            plan = ConvPlan(w4, self.bias, x.shape, 1, 0, 1, 1, "implicit_gemm", self.math, in_layout=lay,
                            out_layout=_lib.NHWC)
            if self.relu:
                plan.set_relu(True)
            ent = (wv, plan)
            self._plans[key] = ent
        return ent[1]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        _require_cuda(x)
        self._check_dtype(x)
        if self.fused_flatten:
            if x.dim() == 4:
                y = self._flatten_plan(x)(x)  # (N, out, 1, 1), NHWC == (N, out) row-major
                return y.view(x.shape[0], self.out_features)
            x = flatten(x, 1)
        if x.shape[-1] != self.in_features:
            raise ValueError(f"ai3 Linear: input has {x.shape[-1]} features in its last dimension, "
                             f"the layer takes {self.in_features}")
        if x.dim() != 2:
            lead = x.shape[:-1]
            return self.forward(x.reshape(-1, x.shape[-1])).reshape(*lead, self.out_features)
        x = x.contiguous()
        batch = x.shape[0]
        plan = self._plan(batch, x.dtype, x.device)
        y = torch.empty((batch, self.out_features), dtype=x.dtype, device=x.device)
        ws = _WS.get(x.device, plan.ws_bytes)
        _check(_lib.load().ai3_conv2d_plan_execute(plan.h, x.data_ptr(), y.data_ptr(),
                                                   None if ws is None else ws.data_ptr(),
                                                   0 if ws is None else ws.numel(), _stream_ptr(x.device)))
        plan.keep = None
        return y


class _LinearPlan:
    def __init__(self, h, wbuf, keep, ws_bytes):
        self.h, self.wbuf, self.keep, self.ws_bytes = h, wbuf, keep, ws_bytes

    def __del__(self):
        if self.h is not None and _lib._lib is not None:
            _lib._lib.ai3_conv2d_plan_destroy(self.h)
            self.h = None
