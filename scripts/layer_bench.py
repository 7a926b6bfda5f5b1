"""Time single VGG/ResNet layers per algorithm (CUDA events); run under ncu for per-kernel times.
usage: python scripts/layer_bench.py conv4_2 [algos...] [--batch 64] [--reps 10]"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import workload, conv_inputs

ap = argparse.ArgumentParser()
ap.add_argument("layer")
ap.add_argument("algos", nargs="*", default=["implicit_gemm", "gemm"])
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--net", default="vgg16")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--lib", default=None, help="library to load (e.g. paper_2410_08300_b200/libai3_dev.so for knobs)")
a = ap.parse_args()
if a.lib:
    from paper_2410_08300_b200 import _lib
    _lib.select_library(a.lib)
import paper_2410_08300_b200 as ai3
spec = [l for l in workload(a.net, a.batch) if l.name == a.layer][0]
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
x = torch.randn(spec.N, spec.C, spec.H, spec.W, device="cuda").to(dt).contiguous(memory_format=torch.channels_last)
_, w, b = conv_inputs(spec.with_batch(1), 1, a.dtype)
wt = torch.from_numpy(w).cuda().to(dt)
bt = None if b is None else torch.from_numpy(b).cuda().to(dt)
for algo in a.algos:
    p = ai3.ConvPlan(wt, bt, x.shape, spec.stride, spec.pad, spec.dil, 1, algo, in_layout=1)
    y = p(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        p(x, out=y)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / a.reps
    print(f"{spec.name} {algo:14s} {ms*1e3:9.1f} us  {spec.flops()/ms/1e9:8.1f} TFLOP/s  launches={p.num_launches}", flush=True)
