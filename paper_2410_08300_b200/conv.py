"""Python face of the C ABI: ``conv2d`` (stateless) and ``ConvPlan`` (prepared weights).

PyTorch supplies device memory, streams and the tensor objects; every step of
the convolution runs in libai3's kernels, called through ``_lib`` (ctypes).
Inputs must already live on a CUDA device -- there is no CPU path.
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib

ALGORITHMS = ("guess", "default", "auto", "benchmark", "direct", "gemm", "im2col", "implicit_gemm", "winograd", "smm",
              "kn2row", "implicit_precomp_gemm", "custom")


class Ai3Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{_lib.STATUS_NAMES.get(status, status)}] {msg}")
        self.status = status


class UnknownAlgorithm(ValueError):
    """Algorithm name not in the set."""


class UnsupportedConfiguration(ValueError):
    """The chosen algorithm cannot run this layer."""


def _check(status: int):
    if status != _lib.OK:
        msg = _lib.last_error()
        if status == _lib.ERR_UNKNOWN_ALGORITHM:
            raise UnknownAlgorithm(msg)
        if status == _lib.ERR_UNSUPPORTED:
            raise UnsupportedConfiguration(msg)
        raise Ai3Error(status, msg)


def algo_id(name) -> int:
    if isinstance(name, int):
        return name
    out = ctypes.c_int()
    st = _lib.load().ai3_algo_from_name(str(name).encode(), ctypes.byref(out))
    if st != _lib.OK:
        raise UnknownAlgorithm(_lib.last_error())
    return out.value


def resolve(name) -> tuple[int, str | None]:
    """Selector name -> (ai3_algo id, registered custom name or None) via ai3_conv2d_resolve
    ("custom", "default" -> a registered default first, registered names)."""
    if isinstance(name, int):
        return name, None
    out = ctypes.c_int()
    buf = ctypes.create_string_buffer(256)
    st = _lib.load().ai3_conv2d_resolve(str(name).encode(), ctypes.byref(out), buf, 256)
    if st != _lib.OK:
        _check(st)
    return out.value, (buf.value.decode() if out.value == _lib.ALGO_CUSTOM else None)


def algo_name(aid: int) -> str:
    return _lib.load().ai3_algo_name(int(aid)).decode()


def _pair(v):
    if isinstance(v, (tuple, list)):
        return int(v[0]), int(v[1])
    return int(v), int(v)


def _dtype_id(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _lib.F32
    if dt == torch.bfloat16:
        return _lib.BF16
    raise TypeError(f"ai3 supports float32 and bfloat16 tensors, got {dt}")


def _math_id(math: str) -> int:
    if math in ("strict", "fp32", "ieee"):
        return _lib.MATH_STRICT
    if math == "tf32":
        return _lib.MATH_TF32
    raise ValueError(f"math must be 'strict' or 'tf32', got {math!r}")


def layout_of(x: torch.Tensor) -> int:
    """NCHW if x is contiguous, NHWC if it is channels_last-contiguous."""
    if x.is_contiguous():
        return _lib.NCHW
    if x.is_contiguous(memory_format=torch.channels_last):
        return _lib.NHWC
    raise ValueError("input must be contiguous (NCHW) or channels_last (NHWC)")


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _raw_stream(index: int) -> int:
    """The current stream's cudaStream_t on device `index` (the hot dispatch path: no Stream
    object is built)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(index)
    return torch.cuda.current_stream(index).cuda_stream


class _Workspace(threading.local):
    """Grow-only per-(thread, device, stream) scratch buffer from torch's allocator."""

    def __init__(self):
        self.bufs = {}

    def get(self, device, nbytes: int):
        if nbytes == 0:
            return None
        key = (device, torch.cuda.current_stream(device).cuda_stream)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self.bufs[key] = buf
        return buf


_WS = _Workspace()


def _same_dtype(dt: torch.dtype, weight: torch.Tensor, bias: torch.Tensor | None):
    """Weights (and bias) must already have the activation dtype, as F.conv2d requires; the
    library converts nothing on the caller's behalf."""
    if weight.dtype != dt or (bias is not None and bias.dtype != dt):
        raise TypeError(f"input dtype {dt} differs from weight {weight.dtype}"
                        + ("" if bias is None else f" / bias {bias.dtype}") + " (torch.nn.functional.conv2d "
                        "raises on mixed dtypes too)")


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("ai3 kernels run on CUDA tensors only (there is no CPU path); move the tensors to a "
                             "CUDA device")


def output_shape(in_shape, out_channels, kernel, stride=1, padding=0, dilation=1, groups=1):
    p = _lib.params(out_channels, _pair(kernel), _pair(stride), _pair(padding), _pair(dilation), groups, False)
    out = (ctypes.c_int64 * 4)()
    _check(_lib.load().ai3_conv2d_output_shape(ctypes.byref(p), _lib.shape4(in_shape), out))
    return tuple(out)


def supported(in_shape, out_channels, kernel, stride=1, padding=0, dilation=1, groups=1, dtype=torch.float32,
              math="strict", algorithm="default") -> bool:
    p = _lib.params(out_channels, _pair(kernel), _pair(stride), _pair(padding), _pair(dilation), groups, False)
    st = _lib.load().ai3_conv2d_supported(ctypes.byref(p), _lib.shape4(in_shape), _dtype_id(dtype),
                                          _math_id(math), algo_id(algorithm))
    return st == _lib.OK


def check_supported(in_shape, out_channels, kernel, stride=1, padding=0, dilation=1, groups=1,
                    dtype=torch.float32, math="strict", algorithm="default"):
    """Raise UnsupportedConfiguration / Ai3Error naming the violated constraint."""
    p = _lib.params(out_channels, _pair(kernel), _pair(stride), _pair(padding), _pair(dilation), groups, False)
    _check(_lib.load().ai3_conv2d_supported(ctypes.byref(p), _lib.shape4(in_shape), _dtype_id(dtype),
                                            _math_id(math), algo_id(algorithm)))


def guess(in_shape, out_channels, kernel, stride=1, padding=0, dilation=1, groups=1, dtype=torch.float32,
          math="strict") -> str:
    """The algorithm the `guess` rule picks for this problem."""
    p = _lib.params(out_channels, _pair(kernel), _pair(stride), _pair(padding), _pair(dilation), groups, False)
    out = ctypes.c_int()
    _check(_lib.load().ai3_conv2d_guess(ctypes.byref(p), _lib.shape4(in_shape), _dtype_id(dtype), _math_id(math),
                                        ctypes.byref(out)))
    return algo_name(out.value)


def _desc(t: torch.Tensor, layout: int) -> _lib.Tensor4d:
    d = _lib.Tensor4d()
    d.data = t.data_ptr()
    d.n, d.c, d.h, d.w = (int(v) for v in t.shape)
    d.dtype = _dtype_id(t.dtype)
    d.layout = layout
    return d


def conv2d(input: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None, stride=1, padding=0,
           dilation=1, groups: int = 1, algorithm="default", math: str = "strict",
           out: torch.Tensor | None = None) -> torch.Tensor:
    """Forward 2-D convolution with a user-selected algorithm (north_star signature).

    Same semantics as ``torch.nn.functional.conv2d``.  ``input``
    is NCHW-contiguous or channels_last; the result has the same memory format.
    Weights are prepared on every call -- use :class:`ConvPlan` (or ``Conv2D`` /
    ``swap_conv2d``) to prepare them once.
    """
    _require_cuda(input, weight, bias)
    lib = _lib.load()
    if input.dim() != 4 or weight.dim() != 4:
        raise ValueError("input and weight must be 4-D (NCHW / KCRS)")
    if isinstance(padding, str):
        raise UnsupportedConfiguration("string padding is not supported; pass integers")
    _same_dtype(input.dtype, weight, bias)
    weight = weight.contiguous()
    if bias is not None:
        bias = bias.contiguous()
    in_layout = layout_of(input)
    s, p, d = _pair(stride), _pair(padding), _pair(dilation)
    oshape = output_shape(input.shape, weight.shape[0], weight.shape[2:], s, p, d, groups)
    fmt = torch.channels_last if in_layout == _lib.NHWC else torch.contiguous_format
    if out is None:
        out = torch.empty(oshape, dtype=input.dtype, device=input.device, memory_format=fmt)
    out_layout = layout_of(out)
    arr = lambda v: (ctypes.c_int32 * 2)(*v)  # noqa: E731
    aid, custom = resolve(algorithm)
    if aid == _lib.ALGO_CUSTOM and custom is None:
        custom = "custom"
    if custom is not None:  # a registered user algorithm, dispatched by libai3's registry
        xd, wd, yd = _desc(input, in_layout), _desc(weight, _lib.NCHW), _desc(out, out_layout)
        with torch.cuda.device(input.device):
            st = lib.ai3_conv2d_custom(custom.encode(), ctypes.byref(xd), ctypes.byref(wd),
                                       None if bias is None else bias.data_ptr(), arr(s), arr(p), arr(d),
                                       int(groups), ctypes.byref(yd), _stream_ptr(input.device))
        if st != _lib.OK:
            from .custom import last_python_error
            raise Ai3Error(st, f"custom conv2d '{custom}' failed: {_lib.last_error() or last_python_error()}")
        return out
    prm = _lib.params(weight.shape[0], weight.shape[2:], s, p, d, groups, bias is not None)
    nbytes = ctypes.c_size_t()
    _check(lib.ai3_conv2d_workspace_size(ctypes.byref(prm), _lib.shape4(input.shape), _dtype_id(input.dtype),
                                         _math_id(math), aid, in_layout, out_layout, ctypes.byref(nbytes)))
    ws = _WS.get(input.device, nbytes.value)
    xd, wd, yd = _desc(input, in_layout), _desc(weight, _lib.NCHW), _desc(out, out_layout)
    with torch.cuda.device(input.device):
        st = lib.ai3_conv2d(ctypes.byref(xd), ctypes.byref(wd), None if bias is None else bias.data_ptr(),
                            arr(s), arr(p), arr(d), int(groups), aid, _math_id(math), ctypes.byref(yd),
                            None if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                            _stream_ptr(input.device))
    _check(st)
    return out


def autotune(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None, stride=1, padding=0,
             dilation=1, groups: int = 1, math: str = "strict", reps: int = 3, out_layout=None):
    """Time every built-in algorithm that supports this convolution on these tensors
    (ai3_conv2d_autotune) and return (fastest name, {name: ms}).  The winner is cached, so
    the algorithm name "benchmark" then selects it for this problem."""
    _require_cuda(x, weight, bias)
    lib = _lib.load()
    if not (x.is_contiguous() or x.is_contiguous(memory_format=torch.channels_last)):
        x = x.contiguous()
    _same_dtype(x.dtype, weight, bias)
    weight = weight.detach().contiguous()
    if bias is not None:
        bias = bias.detach().contiguous()
    in_layout = layout_of(x)
    out_layout = in_layout if out_layout is None else out_layout
    s, p, d = _pair(stride), _pair(padding), _pair(dilation)
    prm = _lib.params(weight.shape[0], weight.shape[2:], s, p, d, groups, bias is not None)
    shp = _lib.shape4(x.shape)
    nbytes = ctypes.c_size_t()
    _check(lib.ai3_conv2d_autotune_scratch_bytes(ctypes.byref(prm), shp, _dtype_id(x.dtype), _math_id(math),
                                                 in_layout, out_layout, ctypes.byref(nbytes)))
    scratch = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=x.device)
    oshape = output_shape(x.shape, weight.shape[0], weight.shape[2:], s, p, d, groups)
    fmt = torch.channels_last if out_layout == _lib.NHWC else torch.contiguous_format
    y = torch.empty(oshape, dtype=x.dtype, device=x.device, memory_format=fmt)
    best = ctypes.c_int()
    ms = (ctypes.c_float * _lib.NUM_ALGOS)()
    with torch.cuda.device(x.device):
        _check(lib.ai3_conv2d_autotune(ctypes.byref(prm), shp, _dtype_id(x.dtype), _math_id(math), in_layout,
                                       out_layout, x.data_ptr(), weight.data_ptr(),
                                       None if bias is None else bias.data_ptr(), y.data_ptr(), scratch.data_ptr(),
                                       scratch.numel(), int(reps), _stream_ptr(x.device), ctypes.byref(best), ms))
    return algo_name(best.value), {algo_name(i): float(ms[i]) for i in range(_lib.NUM_ALGOS) if ms[i] >= 0}


def execute_host_many(plans, x_hosts, y_hosts, x_devs, y_devs):
    """Pipelined host-to-host execution of independent problems (ai3_conv2d_plans_execute_host):
    H2D copies, convolutions and D2H copies of consecutive problems overlap.  All buffers
    are torch tensors (hosts pinned, devices distinct); synchronise the current stream
    before reading the y_hosts."""
    n = len(plans)
    if not (len(x_hosts) == len(y_hosts) == len(x_devs) == len(y_devs) == n):
        raise ValueError("one buffer of each kind per plan")
    if n == 0:
        return
    dev = plans[0].device
    ws = _WS.get(dev, max(p.workspace_size for p in plans))
    arr = lambda ts: (ctypes.c_void_p * n)(*[t.data_ptr() for t in ts])  # noqa: E731
    hp = (ctypes.c_void_p * n)(*[p._h.value for p in plans])
    _check(_lib.load().ai3_conv2d_plans_execute_host(n, hp, arr(x_hosts), arr(y_hosts), arr(x_devs), arr(y_devs),
                                                     None if ws is None else ws.data_ptr(),
                                                     0 if ws is None else ws.numel(), _stream_ptr(dev)))
    for p in plans:
        p._keep = None


class ConvPlan:
    """Weights prepared once (swap time) for one input shape / layout / dtype.

    Wraps ai3_conv2d_plan_create / _execute / _destroy.  Holds the device buffer of
    the prepared weights; the original weight tensor may change or be freed after
    construction (call again to re-prepare).
    """

    def __init__(self, weight: torch.Tensor, bias: torch.Tensor | None, in_shape, stride=1, padding=0,
                 dilation=1, groups=1, algorithm="default", math="strict", in_layout=_lib.NCHW,
                 out_layout=None, dtype: torch.dtype | None = None):
        _require_cuda(weight, bias)
        lib = _lib.load()
        self.device = weight.device
        self.dtype = dtype or weight.dtype
        _same_dtype(self.dtype, weight, bias)
        weight = weight.detach().contiguous()
        if bias is not None:
            bias = bias.detach().contiguous()
        self.in_shape = tuple(int(v) for v in in_shape)
        self.stride, self.padding, self.dilation, self.groups = _pair(stride), _pair(padding), _pair(dilation), groups
        self.math = math
        self.in_layout = in_layout
        self.out_layout = in_layout if out_layout is None else out_layout
        self.out_shape = output_shape(self.in_shape, weight.shape[0], weight.shape[2:], self.stride, self.padding,
                                      self.dilation, groups)
        self.conv_shape = self.out_shape
        self.relu = False
        self.pool = False
        self._prm = _lib.params(weight.shape[0], weight.shape[2:], self.stride, self.padding, self.dilation, groups,
                                bias is not None)
        aid = algo_id(algorithm)
        nbytes = ctypes.c_size_t()
        _check(lib.ai3_conv2d_plan_weight_bytes(ctypes.byref(self._prm), _lib.shape4(self.in_shape),
                                                _dtype_id(self.dtype), _math_id(math), aid, ctypes.byref(nbytes)))
        self._wbuf = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=self.device)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.ai3_conv2d_plan_create(ctypes.byref(self._prm), _lib.shape4(self.in_shape),
                                              _dtype_id(self.dtype), _math_id(math), aid, self.in_layout,
                                              self.out_layout, weight.data_ptr(),
                                              None if bias is None else bias.data_ptr(), self._wbuf.data_ptr(),
                                              self._wbuf.numel(), _stream_ptr(self.device), ctypes.byref(handle)))
        self._keep = (weight, bias)  # alive until the prep kernels ran; released on first execute
        self._h = handle
        self.algorithm = algo_name(lib.ai3_conv2d_plan_algo(handle))
        self.workspace_size = int(lib.ai3_conv2d_plan_workspace_size(handle))
        self.num_launches = int(lib.ai3_conv2d_plan_num_launches(handle))
        self._exec = lib.ai3_conv2d_plan_execute
        self._set_out_geometry()

    def _set_out_geometry(self):
        # sizes / strides of the output in the plan's memory format (the hot path allocates it
        # with one empty_strided call)
        fmt = torch.channels_last if self.out_layout == _lib.NHWC else torch.contiguous_format
        probe = torch.empty(self.out_shape, dtype=self.dtype, device="meta", memory_format=fmt)
        self._out_size, self._out_stride = tuple(probe.shape), probe.stride()

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if tuple(x.shape) != self.in_shape or x.dtype != self.dtype:
            raise ValueError(f"plan built for {self.in_shape} {self.dtype}, got {tuple(x.shape)} {x.dtype}")
        if x.device != self.device:
            raise ValueError("input on a different device than the plan")
        fmt = torch.channels_last if self.in_layout == _lib.NHWC else torch.contiguous_format
        if not x.is_contiguous(memory_format=fmt):
            raise ValueError("input memory format differs from the plan's")
        ofmt = torch.channels_last if self.out_layout == _lib.NHWC else torch.contiguous_format
        if out is None:
            out = torch.empty(self.out_shape, dtype=self.dtype, device=self.device, memory_format=ofmt)
        elif (tuple(out.shape) != tuple(self.out_shape) or out.dtype != self.dtype or out.device != self.device
              or not out.is_contiguous(memory_format=ofmt)):
            raise ValueError(f"out must be a {self.out_shape} {self.dtype} tensor on {self.device} in the plan's "
                             f"output memory format, got {tuple(out.shape)} {out.dtype} on {out.device}")
        ws = _WS.get(self.device, self.workspace_size)
        _check(_lib.load().ai3_conv2d_plan_execute(self._h, x.data_ptr(), out.data_ptr(),
                                                   None if ws is None else ws.data_ptr(),
                                                   0 if ws is None else ws.numel(), _stream_ptr(self.device)))
        self._keep = None
        return out

    def run_checked(self, x: torch.Tensor) -> torch.Tensor:
        """The per-forward hot path of ai3.Conv2D once the module has checked that x has the
        plan's shape, dtype, device and strides (its memory format): allocate the output and
        make the one ai3_conv2d_plan_execute call (dispatch adds no overhead)."""
        dev = self.device
        out = torch.empty_strided(self._out_size, self._out_stride, dtype=self.dtype, device=dev)
        sp = _raw_stream(dev.index)
        ws = None
        if self.workspace_size:
            ws = _WS.bufs.get((dev, sp))
            if ws is None or ws.numel() < self.workspace_size:
                ws = _WS.get(dev, self.workspace_size)
        st = self._exec(self._h, x.data_ptr(), out.data_ptr(), None if ws is None else ws.data_ptr(),
                        0 if ws is None else ws.numel(), sp)
        if st:
            _check(st)
        self._keep = None
        return out

    def set_relu(self, relu: bool = True) -> "ConvPlan":
        """Fuse a ReLU into the plan's output epilogue (ai3_conv2d_plan_set_relu)."""
        _check(_lib.load().ai3_conv2d_plan_set_relu(self._h, 1 if relu else 0))
        self.relu = bool(relu)
        return self

    def set_maxpool2x2(self, pool: bool = True) -> "ConvPlan":
        """Fuse a 2x2 / stride-2 max pooling into the epilogue (ai3_conv2d_plan_set_maxpool2x2):
        the plan then outputs (N, K, P // 2, Q // 2).  Raises UnsupportedConfiguration (plan
        unchanged) when the plan's kernel mode cannot pool in its epilogue."""
        _check(_lib.load().ai3_conv2d_plan_set_maxpool2x2(self._h, 1 if pool else 0))
        n, k, p, q = self.conv_shape
        self.out_shape = (n, k, p // 2, q // 2) if pool else self.conv_shape
        self.pool = bool(pool)
        self._set_out_geometry()
        return self

    def execute_raw(self, x_ptr: int, y_ptr: int, ws_ptr: int | None, ws_bytes: int, stream_ptr: int):
        """Bare C-ABI call on raw device pointers (benchmarks, dispatch-overhead check)."""
        _check(_lib.load().ai3_conv2d_plan_execute(self._h, x_ptr, y_ptr, ws_ptr, ws_bytes, stream_ptr))

    def execute_host(self, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor):
        """Host buffers in, host buffers out (H2D + conv + D2H on the current stream)."""
        ws = _WS.get(self.device, self.workspace_size)
        _check(_lib.load().ai3_conv2d_plan_execute_host(self._h, x_host.data_ptr(), y_host.data_ptr(),
                                                        x_dev.data_ptr(), y_dev.data_ptr(),
                                                        None if ws is None else ws.data_ptr(),
                                                        0 if ws is None else ws.numel(), _stream_ptr(self.device)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.ai3_conv2d_plan_destroy(h)
            self._h = None
