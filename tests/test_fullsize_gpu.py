"""Full-size parity at BASELINE.json's configurations, in the launch configuration bench.py
times (SURVEY §8d "Parity subsets"; §IV: every operation tested across its
hyperparameters and input sizes).

Coverage -- every algorithm bench.py times, on every layer it times:
* configs[1] VGG-16 conv stack, N=64: bf16 for every fixed algorithm (direct, gemm,
  implicit_gemm, implicit_precomp_gemm, winograd, kn2row, smm) and both selectors (guess,
  benchmark); fp32 `strict` and `tf32` for implicit_gemm, gemm and winograd, fp32 strict
  for direct;
* configs[2] ResNet-50 (23 unique conv shapes), N=256, and configs[3] AlexNet (5 convs),
  N=128: bf16 for every fixed algorithm that supports the layer (winograd: 3x3 stride 1
  only -- the others are not generated) and both selectors.
Launch configuration: NHWC (channels_last) activations in and out, one ConvPlan per layer;
"benchmark" first runs ai3.autotune on the layer's tensors, as bench.py does.

Checked outputs, per layer: two whole images (0 and N-1, every (k, p, q)) plus 65,536
coordinates drawn uniformly over the WHOLE batch (every image can be hit), against the CPU
fp64 oracle on the same input bits.  The oracle's values are computed once per (layer,
dtype) and shared by the algorithms.  Tolerance (north_star, on max|err| / max|ref| over the
checked set): 2e-2 bf16; 1e-5 fp32 strict; 1e-3 tf32 and fp32 Winograd.

Input recipe at these sizes: x ~ N(0,1) drawn on the GPU from a seeded torch.Generator
(bf16-rounded for bf16 runs), w, b from synth.conv_inputs (U(+-1/sqrt(fan_in))).  The GPU
input is copied back so the oracle sees exactly the same values.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import conv_inputs, workload

pytestmark = pytest.mark.gpu

NETS = {"vgg16": 64, "resnet50": 256, "alexnet": 128}
FIXED = ["direct", "gemm", "implicit_gemm", "implicit_precomp_gemm", "winograd", "kn2row", "smm"]
SELECTORS = ["guess", "benchmark"]
N_SAMPLES = 65536
TOL = {("bf16", "strict"): 2e-2, ("f32", "strict"): 1e-5, ("f32", "tf32"): 1e-3}


def _winograd_ok(s):
    return s.R == 3 and s.S == 3 and s.stride == 1 and s.dil == 1 and s.groups == 1


def _cases():
    out = []
    for net, nb in NETS.items():
        for i, spec in enumerate(workload(net, nb)):
            for algo in FIXED + SELECTORS:
                if algo == "winograd" and not _winograd_ok(spec):
                    continue
                out.append(pytest.param(net, i, algo, "bf16", "strict", id=f"{net}-{spec.name}-{algo}-bf16"))
            if net == "vgg16":
                for algo, maths in (("implicit_gemm", ("strict", "tf32")), ("gemm", ("strict", "tf32")),
                                    ("winograd", ("strict", "tf32")), ("direct", ("strict",))):
                    for m in maths:
                        out.append(pytest.param(net, i, algo, "f32", m, id=f"{net}-{spec.name}-{algo}-f32-{m}"))
    return out


_CACHE = {}


def _layer(net, i, dtype):
    """Input, weights and the oracle's reference values of one layer (cached: shared by the
    algorithms of that layer; one layer per dtype is kept)."""
    key = (net, i, dtype)
    if key in _CACHE:
        return _CACHE[key]
    for k in [k for k in _CACHE if k[2] == dtype]:
        del _CACHE[k]
    spec = workload(net, NETS[net])[i]
    seed = 7000 + 100 * list(NETS).index(net) + i
    dev = torch.device("cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((spec.N, spec.C, spec.H, spec.W), generator=g, device=dev).to(tdt) \
        .contiguous(memory_format=torch.channels_last)
    _, w, b = conv_inputs(spec.with_batch(1), seed, dtype)
    imgs = [0, spec.N - 1]
    ref_full = oracle.conv2d(x[imgs].double().cpu().numpy(), w, b, spec.stride, spec.pad, spec.dil, spec.groups)
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, spec.N, N_SAMPLES), rng.integers(0, spec.K, N_SAMPLES),
                    rng.integers(0, spec.P, N_SAMPLES), rng.integers(0, spec.Q, N_SAMPLES)], axis=1).astype(np.int64)
    ref_s = np.empty(N_SAMPLES, dtype=np.float64)
    for n in np.unique(idx[:, 0]):  # the oracle sees one image at a time (bounded host memory)
        sel = np.nonzero(idx[:, 0] == n)[0]
        loc = idx[sel].copy()
        loc[:, 0] = 0
        xn = x[int(n):int(n) + 1].double().cpu().numpy()
        ref_s[sel] = oracle.conv2d_points(xn, w, b, loc, spec.stride, spec.pad, spec.dil, spec.groups)
    ent = (spec, x, w, b, imgs, ref_full, idx, ref_s)
    _CACHE[key] = ent
    return ent


@pytest.mark.parametrize("net,i,algo,dtype,math", _cases())
def test_fullsize_parity(net, i, algo, dtype, math):
    import paper_2410_08300_b200 as ai3
    spec, x, w, b, imgs, ref_full, idx, ref_s = _layer(net, i, dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    wt = torch.from_numpy(w).cuda().to(tdt)
    bt = None if b is None else torch.from_numpy(b).cuda().to(tdt)
    if algo == "benchmark":  # bench.py: measure every algorithm once for this layer, the plan takes the winner
        ai3.autotune(x, wt, bt, spec.stride, spec.pad, spec.dil, spec.groups, math)
    plan = ai3.ConvPlan(wt, bt, x.shape, spec.stride, spec.pad, spec.dil, spec.groups, algo, math,
                        in_layout=1, out_layout=1)
    y = torch.full(plan.out_shape, float("nan"), dtype=tdt, device=x.device).contiguous(
        memory_format=torch.channels_last)  # unwritten outputs stay NaN and fail
    plan(x, out=y)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(y).any()), "some output elements were never written"
    tol = 1e-3 if (algo == "winograd" or plan.algorithm == "winograd") and dtype == "f32" else TOL[(dtype, math)]
    got_full = y[imgs].double().cpu().numpy()
    ii = torch.from_numpy(idx).cuda()
    got_s = y[ii[:, 0], ii[:, 1], ii[:, 2], ii[:, 3]].double().cpu().numpy()
    e_full = oracle.rel_err(got_full, ref_full)
    e_s = oracle.rel_err(got_s, ref_s)
    assert np.isfinite(got_full).all() and np.isfinite(got_s).all()
    assert e_full <= tol and e_s <= tol, \
        f"{net} {spec.name} {algo}({plan.algorithm}) {dtype}/{math}: whole images {e_full:.3e}, samples {e_s:.3e}"
