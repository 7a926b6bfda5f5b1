"""Time one VGG layer's implicit_gemm plan with epilogue variants (plain / relu / pool / relu+pool)
plus the separate ai3 pool pass, CUDA events.  usage: python scripts/epi_variants.py conv1_2 [conv2_2 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_08300_b200 as ai3  # noqa: E402
from paper_2410_08300_b200 import layers as L  # noqa: E402
from synth import conv_inputs, workload  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for name in sys.argv[1:]:
    spec = [s for s in workload("vgg16", 64) if s.name == name][0]
    x = torch.randn(spec.N, spec.C, spec.H, spec.W, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    _, w, b = conv_inputs(spec.with_batch(1), 1, "bf16")
    wt, bt = torch.from_numpy(w).cuda().bfloat16(), torch.from_numpy(b).cuda().bfloat16()
    res = {}
    for relu in (False, True):
        for pool in (False, True):
            p = ai3.ConvPlan(wt, bt, x.shape, 1, 1, 1, 1, "implicit_gemm", in_layout=1).set_relu(relu)
            if pool:
                p.set_maxpool2x2(True)
            y = torch.empty(p.out_shape, dtype=torch.bfloat16, device="cuda").contiguous(memory_format=torch.channels_last)
            res[f"relu={int(relu)} pool={int(pool)}"] = t(lambda: p(x, out=y))
    p = ai3.ConvPlan(wt, bt, x.shape, 1, 1, 1, 1, "implicit_gemm", in_layout=1).set_relu(True)
    y = p(x)
    res["separate pool pass"] = t(lambda: L.max_pool2d(y, 2, 2))
    print(name, {k: round(v, 1) for k, v in res.items()}, flush=True)
