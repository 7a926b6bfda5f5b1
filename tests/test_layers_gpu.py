"""GPU parity of the all-ai3 model operations against
the fp64 oracle (oracle/ops.py, oracle.conv2d) on the same seeded inputs:

* ReLU, max pooling, layout copies: bit-exact (no arithmetic / exact max);
* average pooling: fp32 sums -> within a few fp32 ulps (fp32) / one bf16 rounding (bf16);
* linear (tcgen05 engine as a 1x1 conv) and the fused conv/linear + ReLU epilogues:
  the north_star conv tolerances (1e-5 strict fp32, 1e-3 tf32, 2e-2 bf16);
* swap_backend(VGG-16 / Listing 1 ConvNet): every supported op replaced, output vs the
  float64 PyTorch model (the paper's own check) and vs the composed oracle.
"""
import numpy as np
import pytest

from helpers import stable_seed
import torch
from torch import nn

import oracle
from oracle import ops as oops
from synth import ConvShape, conv_inputs

pytestmark = pytest.mark.gpu

TOL = {("f32", "strict"): 1e-5, ("f32", "tf32"): 1e-3, ("bf16", "strict"): 2e-2}


def _dev(a, dtype, nhwc=False):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda().to(
        torch.bfloat16 if dtype == "bf16" else torch.float32)
    return t.contiguous(memory_format=torch.channels_last) if nhwc else t


def _host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    m = np.abs(b).max()
    return float(np.abs(a - b).max() / (m if m > 0 else 1.0))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_relu_bit_exact(dtype, n):
    import paper_2410_08300_b200.layers as L
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(np.float32)
    x[::97] = np.nan
    xt = _dev(x, dtype)
    ref = oops.relu(_host(xt))
    y = _host(L.relu(xt))
    np.testing.assert_array_equal(y, ref)
    L.relu(xt, inplace=True)
    np.testing.assert_array_equal(_host(xt), ref)


def _pool_cases():
    rng = np.random.default_rng(7)
    cases = [(2, 64, 224, 224, 2, 2, 0, 1, False, True),   # VGG pool1 shape (N reduced)
             (2, 64, 112, 112, 3, 2, 1, 1, False, True),   # ResNet stem pool
             (3, 13, 17, 19, 3, 2, 1, 1, True, False),     # ragged channels, ceil_mode
             (1, 8, 9, 9, 2, 1, 1, 2, False, True)]        # dilation
    for _ in range(10):
        k = int(rng.integers(1, 5)); s = int(rng.integers(1, 4)); p = int(rng.integers(0, k // 2 + 1))
        d = int(rng.integers(1, 3)); H = int(rng.integers(d * (k - 1) + 1, 20)); W = int(rng.integers(d * (k - 1) + 1, 20))
        cases.append((int(rng.integers(1, 4)), int(rng.choice([3, 8, 16, 24])), H, W, k, s, p, d,
                      bool(rng.integers(0, 2)), bool(rng.integers(0, 2))))
    return cases


@pytest.mark.parametrize("case", _pool_cases(), ids=lambda c: "x".join(map(str, c[:4])) + f"_k{c[4]}s{c[5]}p{c[6]}d{c[7]}")
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("nhwc", [False, True])
def test_pools(case, dtype, nhwc):
    import paper_2410_08300_b200.layers as L
    N, C, H, W, k, s, p, d, cm, cip = case
    rng = np.random.default_rng(stable_seed(case))
    xt = _dev(rng.standard_normal((N, C, H, W)), dtype, nhwc)
    xh = _host(xt)
    y = L.max_pool2d(xt, k, s, p, d, cm)
    assert y.is_contiguous(memory_format=torch.channels_last if nhwc else torch.contiguous_format)
    np.testing.assert_array_equal(_host(y), oops.max_pool2d(xh, k, s, p, d, cm))
    ya = _host(L.avg_pool2d(xt, k, s, p, cm, cip))
    ra = oops.avg_pool2d(xh, k, s, p, cm, cip)
    assert _rel(ya, ra) <= (2e-6 if dtype == "f32" else 8e-3)
    oh, ow = max(1, H // 3), max(1, (W + 1) // 2)
    yd = _host(L.adaptive_avg_pool2d(xt, (oh, ow)))
    assert _rel(yd, oops.adaptive_avg_pool2d(xh, (oh, ow))) <= (2e-6 if dtype == "f32" else 8e-3)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layout_copy_and_flatten_exact(dtype):
    import paper_2410_08300_b200.layers as L
    from paper_2410_08300_b200 import _lib
    rng = np.random.default_rng(3)
    x = _dev(rng.standard_normal((3, 37, 9, 11)), dtype)
    y = L.to_layout(x, _lib.NHWC)
    assert y.is_contiguous(memory_format=torch.channels_last)
    np.testing.assert_array_equal(_host(y), _host(x))
    z = L.to_layout(y, _lib.NCHW)
    assert z.is_contiguous()
    np.testing.assert_array_equal(_host(z), _host(x))
    np.testing.assert_array_equal(_host(L.flatten(y)), oops.flatten(_host(x)))


@pytest.mark.parametrize("dtype,math", list(TOL))
@pytest.mark.parametrize("shape", [(64, 25088, 4096), (3, 100, 10), (130, 512, 1000), (2048, 4096, 4096)],
                         ids=lambda s: "x".join(map(str, s)))
def test_linear(dtype, math, shape):
    import paper_2410_08300_b200.layers as L
    B, IN, OUT = shape
    rng = np.random.default_rng(B + IN)
    x = rng.standard_normal((B, IN)).astype(np.float32)
    lin = nn.Linear(IN, OUT)
    with torch.no_grad():
        lin.weight.uniform_(-1 / IN ** 0.5, 1 / IN ** 0.5)
    lin = lin.cuda().to(torch.bfloat16 if dtype == "bf16" else torch.float32)
    m = L.Linear(lin, math)
    xt = _dev(x, dtype)
    rows = np.unique(np.r_[0, B - 1, rng.integers(0, B, 16)])
    ref = oops.linear(_host(xt)[rows], _host(lin.weight), _host(lin.bias))
    y = m(xt)
    assert y.shape == (B, OUT)
    assert _rel(_host(y)[rows], ref) <= TOL[(dtype, math)]
    m.relu, m._plans = True, {}
    assert _rel(_host(m(xt))[rows], oops.relu(ref)) <= TOL[(dtype, math)]


@pytest.mark.parametrize("nhwc", [True, False])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_flatten_linear_fused(dtype, nhwc):
    """flatten -> Linear fused: one convolution with a 7x7 kernel over the (C, 7, 7) map; the
    activation is read in place (NHWC or NCHW) and the plan's weight packing reorders columns."""
    import paper_2410_08300_b200.layers as L
    rng = np.random.default_rng(11)
    x = _dev(rng.standard_normal((4, 32, 7, 7)), dtype, nhwc=nhwc)
    lin = nn.Linear(32 * 49, 40).cuda().to(x.dtype)
    fl = L.Linear(lin)
    fl.fused_flatten = True
    y = _host(fl(x))
    ref = oops.linear(oops.flatten(_host(x)), _host(lin.weight), _host(lin.bias))
    assert y.shape == (4, 40)
    assert _rel(y, ref) <= TOL[(dtype, "strict")]


def test_linear_last_dim_and_checks():
    """nn.Linear semantics: a 4-D input is transformed over its last dimension; a wrong
    feature count or dtype raises instead of reading out of bounds."""
    import paper_2410_08300_b200.layers as L
    rng = np.random.default_rng(12)
    lin = nn.Linear(16, 24).cuda()
    m = L.Linear(lin)
    x = _dev(rng.standard_normal((2, 3, 5, 16)), "f32")
    y = _host(m(x))
    ref = oops.linear(_host(x).reshape(-1, 16), _host(lin.weight), _host(lin.bias)).reshape(2, 3, 5, 24)
    assert _rel(y, ref) <= TOL[("f32", "strict")]
    with pytest.raises(ValueError):
        m(_dev(rng.standard_normal((4, 15)), "f32"))
    with pytest.raises(TypeError):
        m(_dev(rng.standard_normal((4, 16)), "bf16"))


@pytest.mark.parametrize("algo", ["implicit_gemm", "gemm", "direct", "winograd", "smm", "kn2row"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_conv_fused_relu(algo, dtype):
    import paper_2410_08300_b200 as ai3
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 32, 19, 21))
    w = rng.uniform(-0.2, 0.2, (48, 32, 3, 3))
    b = rng.uniform(-0.2, 0.2, 48)
    xt, wt, bt = _dev(x, dtype, True), _dev(w, dtype), _dev(b, dtype)
    plan = ai3.ConvPlan(wt, bt, xt.shape, 1, 1, 1, 1, algo, in_layout=1).set_relu(True)
    y = _host(plan(xt))
    ref = oops.relu(oracle.conv2d(_host(xt), _host(wt), _host(bt), 1, 1, 1))
    assert _rel(y, ref) <= (1e-3 if algo == "winograd" and dtype == "f32" else TOL[(dtype, "strict")])
    assert (y >= 0).all()


class ConvNet(nn.Module):
    """PAPER.md:111-128 (Listing 1)."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 16, 3, padding=1)
        self.maxpool = nn.MaxPool2d(2, 2)
        self.conv2 = nn.Conv2d(16, 32, 3, padding=1)

    def forward(self, x):
        x = torch.relu(self.conv1(x))
        x = self.maxpool(x)
        x = torch.relu(self.conv2(x))
        return torch.flatten(x, 1)


def _oracle_convnet(m, x):
    y = oops.relu(oracle.conv2d(x, _host(m.conv1.weight), _host(m.conv1.bias), 1, 1))
    y = oops.max_pool2d(y, 2, 2)
    y = oops.relu(oracle.conv2d(y, _host(m.conv2.weight), _host(m.conv2.bias), 1, 1))
    return oops.flatten(y)


@pytest.mark.parametrize("graph", [False, True])
def test_swap_backend_convnet_all_ai3(graph):
    import paper_2410_08300_b200 as ai3
    torch.manual_seed(0)
    orig = ConvNet().cuda()
    x = torch.randn(10, 3, 224, 224, device="cuda")
    model = ai3.swap_backend(orig, {"conv2d": "direct"}, cuda_graph=graph)
    assert model.kept == []
    ref = _oracle_convnet(orig, _host(x))
    with torch.inference_mode():
        for _ in range(3):
            y = model(x)
    assert _rel(_host(y), ref) <= 1e-5


@pytest.mark.parametrize("sel,tol", [("direct", 1e-5), ("smm", 1e-5), ("gemm", 1e-5), ("implicit_gemm", 1e-5),
                                     ("implicit_precomp_gemm", 1e-5), ("kn2row", 1e-5), ("winograd", 1e-3),
                                     ("guess", 1e-5), (["direct", "winograd"], 1e-3)])
def test_swap_conv2d_convnet_vs_composed_oracle(sel, tol):
    """swap_conv2d: only the convolutions run in ai3, ReLU / pooling /
    flatten stay PyTorch's (fp32).  Compared with the model composed from oracle ops (fp64)
    on the same parameters and input (randn(10, 3, 224, 224))."""
    import paper_2410_08300_b200 as ai3
    torch.manual_seed(0)
    orig = ConvNet().cuda()
    x = torch.randn(10, 3, 224, 224, device="cuda")
    ref = _oracle_convnet(orig, _host(x))
    model = ai3.swap_conv2d(orig, sel)
    assert [type(model.conv1).__name__, type(model.conv2).__name__] == ["Conv2D", "Conv2D"]
    with torch.inference_mode():
        y = model(x)
    assert _rel(_host(y), ref) <= tol


def _oracle_vgg16(vgg, x):
    """VGG-16 forward composed from oracle ops (fp64), on the model's own parameters."""
    y = x
    for m in vgg.features:
        if isinstance(m, nn.Conv2d):
            y = oracle.conv2d(y, _host(m.weight), _host(m.bias), m.stride, m.padding)
        elif isinstance(m, nn.ReLU):
            y = oops.relu(y)
        elif isinstance(m, nn.MaxPool2d):
            y = oops.max_pool2d(y, m.kernel_size, m.stride)
    y = oops.flatten(oops.adaptive_avg_pool2d(y, 7))
    for m in vgg.classifier:
        if isinstance(m, nn.Linear):
            y = oops.linear(y, _host(m.weight), _host(m.bias))
        elif isinstance(m, nn.ReLU):
            y = oops.relu(y)
    return y


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_swap_backend_vgg16_all_ai3(dtype):
    """BASELINE configs[4]'s model: every VGG-16 op (13 conv + ReLU, 5 max-pool, adaptive
    avg-pool, flatten, 3 linear + ReLU, dropout = identity) runs in ai3."""
    import paper_2410_08300_b200 as ai3
    torchvision = pytest.importorskip("torchvision")
    torch.manual_seed(0)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    vgg = torchvision.models.vgg16(weights=None).eval().cuda().to(tdt)
    x = torch.randn(2, 3, 224, 224, device="cuda").to(tdt)
    model = ai3.swap_backend(vgg)
    assert model.kept == []
    kinds = [k for _, k in model.replaced]
    assert kinds.count("fused_relu") == 15 and kinds.count("flatten_fused") == 1
    assert kinds.count("fused_maxpool2x2") == 5
    with torch.inference_mode():
        y = _host(model(x))
    if dtype == "bf16":  # conv1_2 and conv2_2 (halo modes) pool in their epilogue
        pooled = [p for m in model.modules() if isinstance(m, ai3.Conv2D) for _, p in m._plans.values() if p.pool]
        assert len(pooled) >= 2
    ref = _oracle_vgg16(vgg, _host(x))
    assert _rel(y, ref) <= (1e-4 if dtype == "f32" else 5e-2)


POOL_SHAPES = [ConvShape("p64", 2, 64, 20, 22, 64, 3, 3, 1, 1),        # halo mode, ragged tiles
               ConvShape("p64odd", 1, 64, 17, 13, 64, 3, 3, 1, 1),     # odd P, Q: floor mode drops the tail
               ConvShape("p128", 2, 128, 16, 18, 128, 3, 3, 1, 1),     # chunked halo mode
               ConvShape("p64k32", 3, 64, 12, 12, 32, 3, 3, 1, 1, bias=False),
               ConvShape("p16", 2, 16, 14, 14, 64, 3, 3, 1, 1)]        # 32-byte-pixel halo


@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("shape", POOL_SHAPES, ids=lambda s: s.name)
def test_fused_maxpool2x2_matches_unfused_bitwise(shape, relu):
    """conv (+ReLU) -> 2x2 max pooling in the conv epilogue (row f1): the pooled plan's output is
    bit-identical to ai3_maxpool2d of the plain plan's output, and matches the oracle ops."""
    import paper_2410_08300_b200 as ai3
    import paper_2410_08300_b200.layers as L
    x, w, b = conv_inputs(shape, seed=stable_seed(shape.name), dtype="bf16")
    xt = _dev(x, "bf16", True)
    wt, bt = _dev(w, "bf16"), (None if b is None else _dev(b, "bf16"))
    plain = ai3.ConvPlan(wt, bt, xt.shape, 1, 1, 1, 1, "implicit_gemm", in_layout=1).set_relu(relu)
    fused = ai3.ConvPlan(wt, bt, xt.shape, 1, 1, 1, 1, "implicit_gemm", in_layout=1).set_relu(relu)
    fused.set_maxpool2x2(True)
    assert fused.out_shape == (shape.N, shape.K, shape.P // 2, shape.Q // 2)
    y = torch.full(fused.out_shape, float("nan"), dtype=torch.bfloat16, device="cuda").contiguous(
        memory_format=torch.channels_last)
    fused(xt, out=y)
    want = L.max_pool2d(plain(xt), 2, 2)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(y).any())
    assert torch.equal(y, want)
    ref = oracle.conv2d(_host(xt), _host(wt), None if bt is None else _host(bt), 1, 1, 1)
    ref = oops.max_pool2d(oops.relu(ref) if relu else ref, 2, 2)
    assert _rel(_host(y), ref) <= TOL[("bf16", "strict")]


def test_fused_maxpool2x2_unsupported_modes_raise():
    import paper_2410_08300_b200 as ai3
    x = _dev(np.zeros((2, 256, 12, 12)), "bf16", True)
    w = _dev(np.zeros((256, 256, 3, 3)), "bf16")
    p = ai3.ConvPlan(w, None, x.shape, 1, 1, 1, 1, "implicit_gemm", in_layout=1)  # K = 256: im2col mode
    with pytest.raises(ai3.UnsupportedConfiguration):
        p.set_maxpool2x2(True)
    assert p.out_shape == (2, 256, 12, 12)
    q = ai3.ConvPlan(w, None, x.shape, 1, 1, 1, 1, "direct", in_layout=1)
    with pytest.raises(ai3.UnsupportedConfiguration):
        q.set_maxpool2x2(True)
