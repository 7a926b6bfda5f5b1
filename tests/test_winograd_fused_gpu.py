"""GPU parity of the fused Winograd kernel (TcArgs::wf: the F(2x2,3x3) output transform
Y = A^T M A applied in the tcgen05 GEMM's epilogue straight from TMEM; §V.B(d),
SURVEY §8 row a8 step (iv)) against the CPU fp64 oracle.

The fused path runs for bf16 NHWC outputs with K % 16 == 0 and K <= 64 (api.cu); these
cases pin its edges: a partial last 32-channel tile (K = 16, 48: the second epilogue
warpgroup's 16 columns lie past K), odd P / Q (cropped 2x2 tiles), a ragged last T tile
(T not a multiple of 256), bias / no bias, fused ReLU, a misaligned output view (scalar
stores), and integer-valued inputs (bit-exact: every transformed-domain value and sum is
exact in fp32, so the only rounding is the final bf16 cast of an integer below 256).
"""
import numpy as np
import pytest
import torch

import oracle
from helpers import inputs, ref, to_device, tolerance, stable_seed
from synth import ConvShape, integer_inputs

pytestmark = pytest.mark.gpu

SHAPES = [
    ConvShape("wf_k64", 3, 64, 37, 29, 64, 3, 3, 1, 1),                # T = 3*19*15 = 855: ragged last tile
    ConvShape("wf_k48_odd", 2, 32, 21, 17, 48, 3, 3, 1, 0),            # P, Q = 19, 15 odd; partial N tile
    ConvShape("wf_k16_c3", 4, 3, 33, 35, 16, 3, 3, 1, 1, bias=False),  # RGB input, one 16-channel warpgroup
    ConvShape("wf_k32", 1, 128, 14, 14, 32, 3, 3, 1, 1),               # several channel chunks per component
]


def _plan(shape, wt, bt, xt, relu=False):
    import paper_2410_08300_b200 as ai3
    p = ai3.ConvPlan(wt, bt, xt.shape, shape.stride, shape.pad, shape.dil, 1, "winograd", "strict", in_layout=1)
    if relu:
        p.set_relu(True)
    # the fused kernel replaces the GEMM + output-transform pair: input transform + one GEMM
    # launch (+ a channel-padding prep pass when C is not a multiple of 8)
    want = 2 + (1 if shape.C % 8 else 0)
    assert p.num_launches == want, f"expected {want} launches (fused), got {p.num_launches}"
    return p


def _run(shape, x, w, b, relu=False, misalign=False):
    xt = to_device(x, "bf16", "nhwc")
    wt = to_device(w, "bf16")
    bt = None if b is None else to_device(b, "bf16")
    p = _plan(shape, wt, bt, xt, relu)
    n_out = shape.N * shape.K * shape.P * shape.Q
    off = 1 if misalign else 0  # a 2-byte offset: the epilogue must fall back to scalar stores
    buf = torch.full((n_out + off,), float("nan"), dtype=torch.bfloat16, device="cuda")
    y = buf[off:].view(shape.N, shape.P, shape.Q, shape.K).permute(0, 3, 1, 2)  # NHWC strides
    p(xt, out=y)
    torch.cuda.synchronize()
    return y.float().contiguous().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("relu", [False, True])
def test_fused_winograd_matches_oracle(shape, relu):
    x, w, b = inputs(shape, stable_seed(shape.name), "bf16")
    y = _run(shape, x, w, b, relu)
    r = ref(shape, x, w, b)
    if relu:
        r = np.maximum(r, 0.0)
    err = oracle.rel_err(y, r)
    assert err <= tolerance("winograd", "bf16", "strict"), f"{shape.name}: rel err {err:.3e}"


def test_fused_winograd_misaligned_output():
    shape = SHAPES[1]
    x, w, b = inputs(shape, 11, "bf16")
    err = oracle.rel_err(_run(shape, x, w, b, misalign=True), ref(shape, x, w, b))
    assert err <= tolerance("winograd", "bf16", "strict")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
def test_fused_winograd_integer_bit_exact(shape):
    x, w, b = integer_inputs(shape, stable_seed(shape.name) + 1, xmax=2, wmax=2, bias=shape.bias)
    y = _run(shape, x, w, b)
    r = ref(shape, x, w, b)
    # integer outputs |y| <= 9 * C * 4 + 2 fit bf16 exactly only below 256: compare bf16(r)
    rb = torch.from_numpy(r).to(torch.bfloat16).double().numpy()
    assert np.array_equal(y, rb), f"{shape.name}: max |diff| {np.abs(y - rb).max()}"
