"""GPU parity of the space-to-depth lowering of implicit_gemm (R24) and of the
32-byte-pixel halo mode it runs on.

A strided, undilated conv with few input channels (RGB stems) runs as the
stride-1 conv of ceil(R/sh) x ceil(S/sw) taps over the s2d image whose grid
starts at the padded origin.  These cases pin the corners of that rewrite
against the CPU fp64 oracle: kernel extents that are not stride multiples,
padding not a stride multiple, asymmetric strides, odd image sizes, channel
counts whose s2d width is padded (12 -> 16, 27 -> 32) or narrow (4 -> 8), and
an integer-valued stem that must be bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
from helpers import TOL, to_device, stable_seed
from synth import ConvShape, conv_inputs, integer_inputs

pytestmark = pytest.mark.gpu

# (name, N, C, H, W, K, R, S, stride (h, w), pad (h, w))
CASES = [
    ("stem7s2", 2, 3, 45, 45, 64, 7, 7, (2, 2), (3, 3)),
    ("alex11s4", 2, 3, 67, 67, 64, 11, 11, (4, 4), (2, 2)),
    ("c1s2", 3, 1, 19, 23, 16, 3, 3, (2, 2), (1, 1)),       # s2d C' = 4: narrow inner conv
    ("c4s2", 2, 4, 20, 17, 32, 3, 3, (2, 2), (1, 1)),       # C' = 16 exactly
    ("c3s3k5", 2, 3, 26, 29, 24, 5, 5, (3, 3), (2, 1)),     # C' = 27 -> 32, R % s != 0
    ("c3s2k4p0", 1, 3, 31, 30, 40, 4, 4, (2, 2), (0, 0)),   # R a stride multiple, no padding
    ("c2s4k8", 2, 2, 37, 35, 48, 8, 8, (4, 4), (3, 5)),     # C' = 32, pad > stride
    ("asym21", 2, 3, 21, 24, 32, 5, 3, (2, 1), (2, 1)),     # stride (2, 1)
    ("asym13", 2, 3, 18, 25, 16, 3, 7, (1, 3), (1, 3)),     # stride (1, 3)
    ("k200", 1, 3, 33, 33, 200, 7, 7, (2, 2), (3, 3)),      # K > 128: several N tiles
    # stride-1 layers with 9..16 channels: the 32-byte-pixel halo (two 8-channel planes) that the
    # s2d stem also runs on
    ("halo32_c12", 2, 12, 37, 29, 64, 3, 3, (1, 1), (1, 1)),
    ("halo32_c16", 3, 16, 23, 41, 48, 5, 5, (1, 1), (2, 2)),
    ("halo32_c9k128", 1, 9, 40, 19, 128, 4, 4, (1, 1), (0, 3)),
]
MODES = [("f32", "strict"), ("f32", "tf32"), ("bf16", "strict")]


def _run(x, w, b, stride, pad, dtype, math, layout, algo="implicit_gemm"):
    import paper_2410_08300_b200 as ai3
    xt = to_device(x, dtype, layout)
    wt = to_device(w, dtype)
    bt = None if b is None else to_device(b, dtype)
    oshape = ai3.output_shape(x.shape, w.shape[0], w.shape[2:], stride, pad)
    y = torch.full(oshape, float("nan"), dtype=xt.dtype, device=xt.device).contiguous(
        memory_format=torch.channels_last if layout == "nhwc" else torch.contiguous_format)  # unwritten -> NaN
    ai3.conv2d(xt, wt, bt, stride, pad, 1, 1, algo, math, out=y)
    torch.cuda.synchronize()
    return y.float().contiguous().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("dtype,math", MODES)
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_s2d_parity(case, dtype, math, layout):
    name, N, C, H, W, K, R, S, st, pd = case
    shape = ConvShape(name, N, C, H, W, K, R, S)
    x, w, b = conv_inputs(shape, seed=stable_seed(name), dtype=dtype)
    y = _run(x, w, b, st, pd, dtype, math, layout)
    r = oracle.conv2d(x, w, b, st, pd, 1, 1)
    assert y.shape == r.shape
    err = oracle.rel_err(y, r)
    assert err <= TOL[(dtype, math)], f"{name} {dtype}/{math} {layout}: rel err {err:.3e}"


@pytest.mark.parametrize("dtype,math", MODES)
def test_s2d_integer_stem_bit_exact(dtype, math):
    """Integer inputs keep every product and partial sum exact: the s2d path must match bit for bit."""
    shape = ConvShape("istem", 2, 3, 29, 27, 64, 7, 7, 2, 3)
    small = dtype == "bf16"
    x, w, b = integer_inputs(shape, seed=9, xmax=1 if small else 8, wmax=1 if small else 4)
    if small:
        w = w * (np.arange(w.size).reshape(w.shape) % 2 == 0)  # keep |y| <= 256 (bf16 output exact)
    y = _run(x, w, b, 2, 3, dtype, math, "nhwc")
    r = oracle.conv2d(x, w, b, 2, 3, 1, 1)
    assert np.abs(r).max() < (256 if small else 2 ** 24)
    np.testing.assert_array_equal(y, r)
