"""Custom-algorithm registry.

CPU tier: registration / resolution semantics of the C ABI registry ("custom" ->
the unique entry, "default" -> the registered default else `guess`, name clashes,
ambiguity).  GPU tier: a counting wrapper around ai3's direct conv,
selected by its name, by "custom" and through "default", is invoked exactly once per
assigned layer per forward pass and reproduces the oracle; a native (ctypes
function-pointer) registration dispatches through the same ABI.
"""
import ctypes

import numpy as np
import pytest
import torch
from torch import nn

import oracle
import paper_2410_08300_b200 as ai3
from paper_2410_08300_b200 import _lib
from paper_2410_08300_b200.conv import resolve


@pytest.fixture(autouse=True)
def _clean_registry():
    yield
    for name in list(ai3.custom._KEEPALIVE):
        ai3.unregister_conv2d(name)


def _noop(x, w, b, stride, padding, dilation, groups, out):
    return None


def test_resolution_semantics():
    assert resolve("default") == (_lib.ALGO_GUESS, None)          # nothing registered: the framework picks
    with pytest.raises(ai3.UnknownAlgorithm, match="no custom conv2d"):
        resolve("custom")
    ai3.register_conv2d("my_conv", _noop)
    assert resolve("my_conv") == (_lib.ALGO_CUSTOM, "my_conv")
    assert resolve("custom") == (_lib.ALGO_CUSTOM, "my_conv")
    assert resolve("default") == (_lib.ALGO_GUESS, None)         # not registered as default
    assert resolve("direct") == (_lib.ALGO_DIRECT, None)         # built-ins unaffected
    ai3.register_conv2d("other", _noop, use_as_default=True)
    assert resolve("default") == (_lib.ALGO_CUSTOM, "other")
    with pytest.raises(ai3.Ai3Error, match="ambiguous"):
        resolve("custom")
    assert ai3.registered_count() == 2
    ai3.unregister_conv2d("other")
    assert resolve("default") == (_lib.ALGO_GUESS, None)


def test_registration_errors():
    for bad in ("direct", "custom", "default", "torch", "guess", "im2col", "smm"):
        with pytest.raises(ai3.Ai3Error, match="built-in|keyword"):
            ai3.register_conv2d(bad, _noop)
    ai3.register_conv2d("a", _noop, use_as_default=True)
    with pytest.raises(ai3.Ai3Error, match="already the default"):
        ai3.register_conv2d("b", _noop, use_as_default=True)
    ai3.register_conv2d("a", _noop, use_as_default=True)         # re-registration replaces
    assert ai3.registered_count() == 1
    with pytest.raises(ai3.UnknownAlgorithm):
        ai3.unregister_conv2d("never")
    with pytest.raises(TypeError):
        ai3.register_conv2d("c", 42.0)


def test_swap_resolves_custom_at_swap_time():
    """Swapping with a registered name binds it; unknown names still raise."""
    ai3.register_conv2d("my_conv", _noop)
    m = nn.Sequential(nn.Conv2d(3, 4, 3, padding=1), nn.ReLU(), nn.Conv2d(4, 4, 3, groups=2))
    ai3.swap_conv2d(m, ["my_conv", "custom"])
    assert [c.custom for c in m if isinstance(c, ai3.Conv2D)] == ["my_conv", "my_conv"]
    with pytest.raises(ai3.UnknownAlgorithm):
        ai3.swap_conv2d(nn.Sequential(nn.Conv2d(3, 4, 3)), "not_registered")


# ------------------------------------------------------------------ GPU: the counting wrapper
class ConvNet(nn.Module):
    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 16, 3, padding=1)
        self.conv2 = nn.Conv2d(16, 32, 3, padding=1, groups=2)  # grouped: PAPER.md:233 via a custom algorithm

    def forward(self, x):
        return self.conv2(torch.relu(self.conv1(x)))


@pytest.mark.gpu
@pytest.mark.parametrize("how", ["name", "custom", "default"])
def test_counting_wrapper_once_per_layer_per_forward(how):
    calls = []

    def counting_direct(x, w, b, stride, padding, dilation, groups, out):
        calls.append(tuple(w.shape))
        ai3.conv2d(x, w, b, stride, padding, dilation, groups, algorithm="direct", out=out)

    ai3.register_conv2d("my_conv", counting_direct, use_as_default=(how == "default"))
    torch.manual_seed(0)
    orig = ConvNet()
    x = torch.randn(2, 3, 20, 20)
    with torch.no_grad():
        ref = orig.double()(x.double()).numpy()
    sel = {"name": "my_conv", "custom": "custom", "default": "default"}[how]
    m = ai3.swap_conv2d(orig.float().cuda(), sel)
    with torch.inference_mode():
        for _ in range(3):
            y = m(x.cuda())
    assert len(calls) == 6 and calls[:2] == [(16, 3, 3, 3), (32, 8, 3, 3)]
    err = float(np.abs(y.cpu().double().numpy() - ref).max() / np.abs(ref).max())
    assert err <= 1e-5


@pytest.mark.gpu
def test_native_function_pointer_registration():
    """A native ai3_conv2d_custom_fn (here a ctypes callback that forwards to the C ABI's
    direct algorithm, as a user's C++ library would) is dispatched by libai3."""
    lib = _lib.load()
    count = [0]

    def fwd(xp, wp, bias, stride, padding, dilation, groups, yp, stream, user):
        count[0] += 1
        return _direct(xp, wp, bias, stride, padding, dilation, groups, yp, stream)

    def _direct(xp, wp, bias, stride, padding, dilation, groups, yp, stream):
        # direct needs a workspace for its prepared weights: ask for it, allocate, call
        prm = _lib.params(wp.contents.n, (wp.contents.h, wp.contents.w), (stride[0], stride[1]),
                          (padding[0], padding[1]), (dilation[0], dilation[1]), groups, bool(bias))
        nbytes = ctypes.c_size_t()
        shp = _lib.shape4((xp.contents.n, xp.contents.c, xp.contents.h, xp.contents.w))
        st = lib.ai3_conv2d_workspace_size(ctypes.byref(prm), shp, xp.contents.dtype, _lib.MATH_STRICT,
                                           _lib.ALGO_DIRECT, xp.contents.layout, yp.contents.layout,
                                           ctypes.byref(nbytes))
        if st != _lib.OK:
            return st
        ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device="cuda")
        _KEEP.append(ws)
        return lib.ai3_conv2d(xp, wp, bias, stride, padding, dilation, groups, _lib.ALGO_DIRECT, _lib.MATH_STRICT,
                              yp, ws.data_ptr(), ws.numel(), stream)

    _KEEP = []
    cb = _lib.CUSTOM_FN(fwd)
    ai3.register_conv2d("native_direct", cb)
    x = torch.randn(2, 8, 12, 12, device="cuda")
    w = torch.randn(16, 8, 3, 3, device="cuda")
    b = torch.randn(16, device="cuda")
    y = ai3.conv2d(x, w, b, 1, 1, 1, 1, algorithm="native_direct")
    y2 = ai3.conv2d(x, w, b, 1, 1, 1, 1, algorithm=_lib.ALGO_CUSTOM)
    torch.cuda.synchronize()
    ref = oracle.conv2d(x.cpu().numpy(), w.cpu().numpy(), b.cpu().numpy(), 1, 1, 1)
    for out in (y, y2):
        assert float(np.abs(out.cpu().double().numpy() - ref).max() / np.abs(ref).max()) <= 1e-5
    assert count[0] == 2
