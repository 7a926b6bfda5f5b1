"""GPU parity of the implicit-GEMM operand modes that only some shapes reach, and of their
A/B switches (read when a plan is laid out):

* flat mode (1x1 / stride 1 / no padding: A is the NHWC input itself, tiled TMA boxes);
* AI3_FLAT1X1=0 (the same convs through the TMA im2col traversal);
* AI3_HALO1X1=1 (1x1 convs with K <= 128 through the halo modes, the pre-round-1-end routing);
* AI3_TC_STORE=3 (fast epilogue writing its staged rows with coalesced st.global instead of TMA stores).
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
]
MODES = [("f32", "strict"), ("f32", "tf32"), ("bf16", "strict")]


def _run(shape, x, w, b, dtype, math, layout):
    import paper_2410_08300_b200 as ai3
    xt = to_device(x, dtype, layout)
    wt = to_device(w, dtype)
    bt = None if b is None else to_device(b, dtype)
    p = ai3.ConvPlan(wt, bt, xt.shape, 1, 0, 1, 1, "implicit_gemm", math, in_layout=1 if layout == "nhwc" else 0)
    y = p(xt)
    torch.cuda.synchronize()
    return y.float().contiguous().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("env", [None, ("AI3_FLAT1X1", "0"), ("AI3_HALO1X1", "1"), ("AI3_TC_STORE", "3")],
                         ids=["flat", "im2col", "halo", "stg"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype,math", MODES)
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_1x1_operand_modes(shape, dtype, math, layout, env, monkeypatch):
    if env:
        monkeypatch.setenv(*env)
    x, w, b = conv_inputs(shape, seed=stable_seed((shape.name, dtype)), dtype=dtype)
    y = _run(shape, x, w, b, dtype, math, layout)
    r = oracle.conv2d(x, w, b, 1, 0, 1, 1)
    err = oracle.rel_err(y, r)
    assert err <= TOL[(dtype, math)], f"{shape.name} {dtype}/{math} {layout} {env}: rel err {err:.3e}"
