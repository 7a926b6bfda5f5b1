"""GPU parity of the implicit-GEMM operand modes that only some 1x1 shapes reach:

* flat mode (1x1 / stride 1 / no padding: A is the NHWC input itself, tiled TMA boxes);
* 1x1 with stride 2 (ResNet-50's downsample projections) and padded 1x1 convs, which take
  the TMA im2col traversal.
The product library reads no environment switch, so each mode is reached by its shape.
"""
import numpy as np
import pytest
import torch

import oracle
from helpers import TOL, stable_seed, to_device
from synth import ConvShape, conv_inputs

pytestmark = pytest.mark.gpu

SHAPES = [
    ConvShape("f256to64", 2, 256, 13, 17, 64, 1, 1),    # M = 442: 4 tiles + ragged tail
    ConvShape("f64to200", 3, 64, 9, 11, 200, 1, 1),     # K > 128: two N tiles, partial last
    ConvShape("f3to32", 2, 3, 15, 15, 32, 1, 1),        # C padded to a 32-byte row
    ConvShape("f512to128", 1, 512, 7, 9, 128, 1, 1, bias=False),
    ConvShape("s2_256to512", 2, 256, 15, 13, 512, 1, 1, 2, 0),  # stride-2 projection: im2col traversal
    ConvShape("p1_64to96", 2, 64, 10, 9, 96, 1, 1, 1, 1),       # padded 1x1: im2col traversal
]
MODES = [("f32", "strict"), ("f32", "tf32"), ("bf16", "strict")]


def _run(shape, x, w, b, dtype, math, layout):
    import paper_2410_08300_b200 as ai3
    xt = to_device(x, dtype, layout)
    wt = to_device(w, dtype)
    bt = None if b is None else to_device(b, dtype)
    p = ai3.ConvPlan(wt, bt, xt.shape, shape.stride, shape.pad, 1, 1, "implicit_gemm", math,
                     in_layout=1 if layout == "nhwc" else 0)
    y = torch.full(p.out_shape, float("nan"), dtype=xt.dtype, device=xt.device).contiguous(
        memory_format=torch.channels_last if layout == "nhwc" else torch.contiguous_format)
    p(xt, out=y)
    torch.cuda.synchronize()
    return y.float().contiguous().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype,math", MODES)
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_1x1_operand_modes(shape, dtype, math, layout):
    x, w, b = conv_inputs(shape, seed=stable_seed((shape.name, dtype)), dtype=dtype)
    y = _run(shape, x, w, b, dtype, math, layout)
    r = oracle.conv2d(x, w, b, shape.stride, shape.pad, 1, 1)
    err = oracle.rel_err(y, r)
    assert err <= TOL[(dtype, math)], f"{shape.name} {dtype}/{math} {layout}: rel err {err:.3e}"
