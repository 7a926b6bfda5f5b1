"""Full-size parity (BASELINE.json configs[1..3]) in the launch configuration bench.py times:
BF16, NHWC-resident activations, plans with algorithm "guess" (plus implicit_gemm and
winograd on the VGG-16 stack).  The oracle computes sampled outputs one by one
(oracle.conv2d_points) on the images the samples come from.

Input recipe at these sizes: x ~ N(0,1) drawn on the GPU from a seeded
torch.Generator (the host generator would dominate the test time), rounded to bf16;
w, b from synth.conv_inputs (bf16-rounded U(+-1/sqrt(fan_in))).  The GPU input is
copied back to the host so the oracle sees exactly the same bf16 values.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import conv_inputs, workload

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2  # north_star BF16 bound on max|err| / max|ref|


def _run_layer(spec, algo, seed, samples=1536):
    import paper_2410_08300_b200 as ai3
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((spec.N, spec.C, spec.H, spec.W), generator=g, device=dev).to(torch.bfloat16) \
        .contiguous(memory_format=torch.channels_last)
    _, w, b = conv_inputs(spec.with_batch(1), seed, "bf16")
    wt = torch.from_numpy(w).to(dev, torch.bfloat16)
    bt = None if b is None else torch.from_numpy(b).to(dev, torch.bfloat16)
    plan = ai3.ConvPlan(wt, bt, x.shape, spec.stride, spec.pad, spec.dil, spec.groups, algo, in_layout=1)
    y = plan(x)
    torch.cuda.synchronize()
    imgs = sorted({0, spec.N // 2, spec.N - 1})
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, len(imgs), samples)
    idx = np.stack([pick, rng.integers(0, spec.K, samples), rng.integers(0, spec.P, samples),
                    rng.integers(0, spec.Q, samples)], axis=1)
    # corners of every sampled image and channel extremes
    extra = np.array([[i, k, p, q] for i in range(len(imgs)) for k in (0, spec.K - 1)
                      for p in (0, spec.P - 1) for q in (0, spec.Q - 1)])
    idx = np.concatenate([idx, extra]).astype(np.int64)
    xs = x[imgs].float().permute(0, 1, 2, 3).contiguous().cpu().numpy()  # logical NCHW values
    ref = oracle.conv2d_points(xs, w, b, idx, spec.stride, spec.pad, spec.dil, spec.groups)
    yimg = y[imgs].float().cpu().numpy()
    got = yimg[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]]
    return oracle.rel_err(got, ref), plan.algorithm


VGG = workload("vgg16", 64)


@pytest.mark.parametrize("spec", VGG, ids=lambda s: s.name)
@pytest.mark.parametrize("algo", ["guess", "implicit_gemm", "winograd"])
def test_vgg16_fullsize_sampled(spec, algo):
    err, used = _run_layer(spec, algo, seed=2000 + VGG.index(spec))
    assert err <= TOL_BF16, f"{spec.name} {used}: {err:.3e}"


@pytest.mark.parametrize("spec", workload("alexnet", 128), ids=lambda s: s.name)
def test_alexnet_fullsize_sampled(spec):
    err, used = _run_layer(spec, "guess", seed=4000 + spec.C)
    assert err <= TOL_BF16, f"{spec.name} {used}: {err:.3e}"


@pytest.mark.parametrize("spec", workload("resnet50", 256), ids=lambda s: s.name)
def test_resnet50_fullsize_sampled(spec):
    err, used = _run_layer(spec, "guess", seed=3000 + spec.C + spec.K + spec.R)
    assert err <= TOL_BF16, f"{spec.name} {used}: {err:.3e}"


def test_vgg_conv1_2_full_image_vs_oracle():
    """One whole image of the largest VGG layer, every output element, vs the full oracle."""
    import paper_2410_08300_b200 as ai3
    spec = VGG[1].with_batch(2)
    x, w, b = conv_inputs(spec, 77, "bf16")
    xt = torch.from_numpy(x).cuda().bfloat16().contiguous(memory_format=torch.channels_last)
    plan = ai3.ConvPlan(torch.from_numpy(w).cuda().bfloat16(), torch.from_numpy(b).cuda().bfloat16(), xt.shape,
                        1, 1, 1, 1, "guess", in_layout=1)
    y = plan(xt).float().cpu().numpy()
    ref = oracle.conv2d(x, w, b, 1, 1, 1)
    assert oracle.rel_err(y, ref) <= TOL_BF16
