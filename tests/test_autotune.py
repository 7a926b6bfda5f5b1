"""The "benchmark" selector: ai3_conv2d_autotune times every built-in
algorithm that supports a problem and caches the winner; AI3_ALGO_BENCHMARK resolves to
it (to the `guess` rule before any measurement).  CPU tier: names and pre-measurement
resolution; GPU tier: measurement, caching, parity of the chosen plan with the oracle."""
import numpy as np
import pytest
import torch

import oracle
import paper_2410_08300_b200 as ai3
from paper_2410_08300_b200 import _lib


def test_benchmark_name_and_unmeasured_resolution():
    assert ai3.algo_id("benchmark") == _lib.ALGO_BENCHMARK
    assert ai3.algo_name(_lib.ALGO_BENCHMARK) == "benchmark"
    # supported wherever guess is, including grouped convs (then only direct / smm can win)
    assert ai3.supported((1, 8, 16, 16), 8, 3, padding=1, groups=2, algorithm="benchmark")
    with pytest.raises(ai3.Ai3Error):
        ai3.register_conv2d("benchmark", lambda *a: None)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(4, 64, 28, 28, 64, 3, 1, 1, 1), (2, 3, 32, 32, 16, 3, 1, 1, 1),
                                   (2, 32, 15, 15, 32, 3, 1, 1, 2), (2, 64, 14, 14, 128, 1, 2, 0, 1)],
                         ids=lambda s: "x".join(map(str, s)))
def test_autotune_measures_caches_and_matches_oracle(shape):
    N, C, H, W, K, R, st, pd, G = shape
    _lib.load().ai3_conv2d_autotune_clear()
    rng = np.random.default_rng(sum(shape))
    x = torch.from_numpy(rng.standard_normal((N, C, H, W)).astype(np.float32)).cuda().to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last)
    w = torch.from_numpy(rng.uniform(-0.3, 0.3, (K, C // G, R, R)).astype(np.float32)).cuda().to(torch.bfloat16)
    b = torch.from_numpy(rng.uniform(-0.3, 0.3, K).astype(np.float32)).cuda().to(torch.bfloat16)
    best, times = ai3.autotune(x, w, b, st, pd, 1, G)
    expect = {a for a in ("direct", "gemm", "implicit_gemm", "winograd", "smm", "kn2row")
              if ai3.supported(x.shape, K, R, st, pd, 1, G, torch.bfloat16, algorithm=a)}
    assert set(times) == expect and best in expect
    assert times[best] == min(times.values())
    plan = ai3.ConvPlan(w, b, x.shape, st, pd, 1, G, "benchmark", in_layout=1)
    assert plan.algorithm == best  # the cached winner
    y = plan(x).float().cpu().numpy()
    ref = oracle.conv2d(x.float().cpu().numpy(), w.float().cpu().numpy(), b.float().cpu().numpy(), st, pd, 1, G)
    assert oracle.rel_err(y, ref) <= 2e-2


@pytest.mark.gpu
def test_swap_with_benchmark_selector():
    from torch import nn
    _lib.load().ai3_conv2d_autotune_clear()
    torch.manual_seed(0)
    m = nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.ReLU(), nn.Conv2d(16, 32, 3, padding=1)).cuda()
    x = torch.randn(2, 3, 24, 24, device="cuda")
    ref = oracle.conv2d(np.maximum(oracle.conv2d(x.cpu().numpy(), m[0].weight.detach().cpu().numpy(),
                                                 m[0].bias.detach().cpu().numpy(), 1, 1), 0),
                        m[2].weight.detach().cpu().numpy(), m[2].bias.detach().cpu().numpy(), 1, 1)
    model = ai3.swap_backend(m, {"conv2d": "benchmark"})
    with torch.inference_mode():
        y = model(x).cpu().numpy()
    assert oracle.rel_err(y, ref) <= 1e-5
