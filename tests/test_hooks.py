"""swap_conv2d / swap_backend -- selector semantics on CPU, model
outputs on the GPU.

CPU tier: selector resolution (str / list / callable), trace order
(PAPER.md:174), "torch" keeps a layer, swap-time errors.
GPU tier: Listing 1 (ConvNet) and Listing 2 (VGG16, rule selector) analogs with
random-init weights, compared with the unswapped model run in float64 on the CPU.
"""
import numpy as np
import pytest
import torch
from torch import nn

import paper_2410_08300_b200 as ai3


class ConvNet(nn.Module):
    """PAPER.md:111-128 (Listing 1)."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(in_channels=3, out_channels=16, kernel_size=3, padding=1)
        self.maxpool = nn.MaxPool2d(kernel_size=2, stride=2)
        self.conv2 = nn.Conv2d(in_channels=16, out_channels=32, kernel_size=3, padding=1)

    def forward(self, x):
        x = torch.relu(self.conv1(x))
        x = self.maxpool(x)
        x = torch.relu(self.conv2(x))
        return torch.flatten(x, 1)


class Reordered(nn.Module):
    """Registration order differs from call order: the trace decides occurrence indices."""

    def __init__(self):
        super().__init__()
        self.late = nn.Conv2d(8, 8, 3, padding=1)
        self.early = nn.Conv2d(3, 8, 3, padding=1)

    def forward(self, x):
        return self.late(self.early(x))


def _algos(model):
    return {n: m.algorithm for n, m in model.named_modules() if isinstance(m, ai3.Conv2D)}


# ------------------------------------------------------------------ CPU: selector semantics
def test_string_selector_applies_to_all():
    m = ai3.swap_conv2d(ConvNet(), "direct")
    assert _algos(m) == {"conv1": "direct", "conv2": "direct"}


def test_list_selector_by_occurrence_and_default_past_end():
    m = ai3.swap_conv2d(ConvNet(), ["implicit_gemm"])
    assert _algos(m) == {"conv1": "implicit_gemm", "conv2": "default"}


def test_list_selector_follows_trace_order():
    m = ai3.swap_conv2d(Reordered(), ["direct", "winograd"])
    assert _algos(m) == {"early": "direct", "late": "winograd"}


def test_callable_selector_gets_original_module():
    seen = []

    def sel(conv: nn.Conv2d) -> str:
        seen.append(conv.weight.shape[1])
        return "gemm" if conv.weight.shape[1] > 8 else "direct"

    m = ai3.swap_conv2d(ConvNet(), sel)
    assert seen == [3, 16]
    assert _algos(m) == {"conv1": "direct", "conv2": "gemm"}


def test_torch_keeps_layer():
    m = ai3.swap_conv2d(ConvNet(), ["torch", "direct"])
    assert isinstance(m.conv1, nn.Conv2d) and isinstance(m.conv2, ai3.Conv2D)


def test_swap_time_errors():
    with pytest.raises(ai3.UnknownAlgorithm):
        ai3.swap_conv2d(ConvNet(), "fastest")
    bad = nn.Sequential(nn.Conv2d(3, 4, 5, stride=2))
    with pytest.raises(ai3.UnsupportedConfiguration, match="3x3"):
        ai3.swap_conv2d(bad, "winograd")
    grouped = nn.Sequential(nn.Conv2d(4, 4, 3, groups=2))
    with pytest.raises(ai3.UnsupportedConfiguration, match="groups"):
        ai3.swap_conv2d(grouped, "implicit_gemm")
    ai3.swap_conv2d(nn.Sequential(nn.Conv2d(4, 4, 3, groups=2)), "default")  # guess handles groups
    with pytest.raises(ai3.UnsupportedConfiguration):
        ai3.swap_conv2d(nn.Sequential(nn.Conv2d(3, 4, 3, padding_mode="reflect")), "direct")
    # nothing is swapped when validation fails on a later layer
    net2 = nn.Sequential(nn.Conv2d(3, 4, 3), nn.Conv2d(4, 4, 5))
    with pytest.raises(ai3.UnsupportedConfiguration):
        ai3.swap_conv2d(net2, "winograd")
    assert all(isinstance(m, nn.Conv2d) for m in net2)


def test_swap_backend_builds_model():
    model = ai3.swap_backend(ConvNet(), {"conv2d": "direct"})
    assert isinstance(model, ai3.Model)
    assert model.layers == [("conv1", "direct"), ("conv2", "direct")]
    with pytest.raises(ai3.UnknownAlgorithm):
        ai3.swap_backend(ConvNet(), {"linear": "direct"})


def test_cpu_forward_refuses():
    m = ai3.swap_conv2d(ConvNet(), "direct")
    with pytest.raises(ValueError, match="CUDA"):
        m(torch.zeros(1, 3, 8, 8))


# ------------------------------------------------------------------ GPU: model outputs
def _ref64(model, x):
    import copy
    m = copy.deepcopy(model).double().cpu()
    with torch.no_grad():
        return m(x.double().cpu()).numpy()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.gpu
@pytest.mark.parametrize("sel,tol", [("direct", 1e-5), (["direct", "implicit_gemm"], 1e-5), (["direct", "smm"], 1e-5),
                                     ("kn2row", 1e-5),
                                     ("gemm", 1e-5), ("winograd", 1e-3), ("default", 1e-5)])
def test_listing1_convnet(sel, tol):
    """randn(10,3,224,224) through swap_backend and swap_conv2d."""
    torch.manual_seed(0)
    orig = ConvNet()
    x = torch.randn(10, 3, 224, 224)
    ref = _ref64(orig, x)
    model = ai3.swap_backend(orig.cuda(), {"conv2d": sel})
    with torch.inference_mode():
        sb = model(x.cuda()).cpu().numpy()
    assert _rel(sb, ref) <= tol
    ai3.swap_conv2d(orig, sel)
    with torch.inference_mode():
        sc = orig(x.cuda()).cpu().numpy()
    assert _rel(sc, ref) <= tol


@pytest.mark.gpu
def test_listing2_vgg16_rule_selector():
    """PAPER.md:148-167 (Listing 2) with random-init VGG16: "smm" for in_channels > 200, else "direct"."""
    torchvision = pytest.importorskip("torchvision")
    torch.manual_seed(0)
    vgg = torchvision.models.vgg16(weights=None).eval()
    x = torch.randn(1, 3, 224, 224)
    ref = _ref64(vgg, x)
    chosen = []

    def selector(orig: nn.Conv2d) -> str:
        algo = "smm" if orig.weight.shape[1] > 200 else "direct"
        chosen.append(algo)
        return algo

    vgg = vgg.cuda()
    model = ai3.swap_backend(vgg, {"conv2d": selector})
    assert chosen.count("smm") == 8 and len(chosen) == 13
    with torch.inference_mode():
        out = model(x.cuda()).cpu().numpy()
    assert _rel(out, ref) <= 1e-4  # PAPER.md:163 atol=1e-4 analog (relative here)
    ai3.swap_conv2d(vgg, selector)
    with torch.inference_mode():
        out2 = vgg(x.cuda()).cpu().numpy()
    assert _rel(out2, ref) <= 1e-4


@pytest.mark.gpu
def test_bf16_channels_last_model():
    torch.manual_seed(1)
    orig = ConvNet()
    x = torch.randn(4, 3, 64, 64)
    ref = _ref64(orig, x.bfloat16().float())
    m = ai3.swap_conv2d(orig.cuda().bfloat16(), "implicit_gemm")
    with torch.inference_mode():
        y = m(x.cuda().bfloat16().contiguous(memory_format=torch.channels_last)).float().cpu().numpy()
    assert _rel(y, ref) <= 2e-2
