"""Small cases for compute-sanitizer (scripts/sanitize.sh): BASELINE config 1 with every
algorithm and precision, a ragged multi-tile sweep through every engine mode, the pooling /
ReLU / layout / linear ops, and the all-ai3 model path.  Exits non-zero on a parity miss."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
if len(sys.argv) > 1 and sys.argv[1] == "--dev":  # developer build (knobs such as AI3_TC_CG=1)
    from paper_2410_08300_b200 import _lib  # noqa: E402
    _lib.select_library(os.path.join(ROOT, "paper_2410_08300_b200", "libai3_dev.so"))
import paper_2410_08300_b200 as ai3  # noqa: E402
from paper_2410_08300_b200 import layers as L  # noqa: E402
from synth import CONFIG1, ConvShape, conv_inputs  # noqa: E402

ALGOS = ["direct", "gemm", "implicit_gemm", "implicit_precomp_gemm", "winograd", "smm", "kn2row", "guess"]
SHAPES = [CONFIG1,
          ConvShape("halo64", 2, 64, 19, 21, 64, 3, 3, 1, 1),      # halo mode, ragged tiles
          ConvShape("chunk128", 1, 128, 17, 15, 96, 3, 3, 1, 1),   # chunked halo, K < 128
          ConvShape("im2col256", 2, 256, 9, 11, 192, 3, 3, 1, 1),  # im2col mode, partial N tile
          ConvShape("flat1x1", 2, 96, 13, 7, 200, 1, 1),           # flat 1x1 mode
          ConvShape("stem", 1, 3, 37, 35, 64, 7, 7, 2, 3),          # space-to-depth stem
          ConvShape("c5", 3, 512, 7, 7, 512, 3, 3, 1, 1)]           # two N sub-tiles / CTA pairs
bad = []
for s in SHAPES:
    for dt in ("f32", "bf16"):
        x, w, b = conv_inputs(s, 11, dt)
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        xt = torch.from_numpy(x).cuda().to(tdt)
        if dt == "bf16":
            xt = xt.contiguous(memory_format=torch.channels_last)
        ref = oracle.conv2d(x, w, b, s.stride, s.pad, s.dil, s.groups)
        for a in ALGOS:
            if a == "winograd" and not (s.R == 3 and s.stride == 1):
                continue
            for m in (("strict", "tf32") if dt == "f32" and a not in ("direct", "smm") else ("strict",)):
                y = torch.full((s.N, s.K, s.P, s.Q), float("nan"), dtype=tdt, device="cuda")
                if dt == "bf16":
                    y = y.contiguous(memory_format=torch.channels_last)
                ai3.conv2d(xt, torch.from_numpy(w).cuda().to(tdt), torch.from_numpy(b).cuda().to(tdt), s.stride,
                           s.pad, s.dil, s.groups, algorithm=a, math=m, out=y)
                torch.cuda.synchronize()
                e = oracle.rel_err(y.double().cpu().numpy(), ref)
                tol = 2e-2 if dt == "bf16" else (1e-5 if m == "strict" and a != "winograd" else 1e-3)
                if not e <= tol:
                    bad.append((s.name, dt, a, m, e))
# model-path ops
xm = torch.randn(2, 64, 16, 16, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
L.max_pool2d(L.relu(xm), 2, 2)
L.avg_pool2d(xm, 3, 2, 1)
L.adaptive_avg_pool2d(xm, 7)
L.to_layout(xm, 0)
lin = torch.nn.Linear(64 * 16 * 16, 40).cuda().bfloat16()
m = L.Linear(lin)
m.fused_flatten = True
m(xm)
torch.cuda.synchronize()
print("sanitize cases done; parity misses:", bad)
sys.exit(1 if bad else 0)
