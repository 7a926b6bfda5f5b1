"""One execute of a VGG-16 layer's plan between cudaProfilerStart/Stop (for
`ncu --profile-from-start off`): python scripts/prof_layer.py conv3_2 winograd [--batch 64]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_08300_b200 as ai3  # noqa: E402
from synth import conv_inputs, workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("layer")
ap.add_argument("algo")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--net", default="vgg16")
a = ap.parse_args()
spec = [s for s in workload(a.net, a.batch) if s.name == a.layer][0]
x = torch.randn(spec.N, spec.C, spec.H, spec.W, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
_, w, b = conv_inputs(spec.with_batch(1), 1, "bf16")
wt = torch.from_numpy(w).cuda().bfloat16()
bt = None if b is None else torch.from_numpy(b).cuda().bfloat16()
p = ai3.ConvPlan(wt, bt, x.shape, spec.stride, spec.pad, spec.dil, 1, a.algo, in_layout=1)
y = p(x)
for _ in range(2):
    p(x, out=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
p(x, out=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
