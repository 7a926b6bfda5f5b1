"""3xTF32 accuracy vs reduction length (is the tensor-core accumulation the limit?)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import oracle
from synth import ConvShape, conv_inputs
from helpers import run_ai3, ref
for C in (64, 128, 256, 512):
    for R in (1, 3):
        s = ConvShape("scan", 1, C, 16, 16, 64, R, R, 1, R // 2)
        x, w, b = conv_inputs(s, 3, "f32")
        r = ref(s, x, w, b)
        errs = []
        for algo in ("implicit_gemm", "direct", "winograd" if R == 3 else "gemm"):
            y = run_ai3(s, x, w, b, algo, "f32", "strict", "nhwc")
            errs.append(f"{algo}={oracle.rel_err(y, r):.2e}")
        print(f"Kg={C*R*R:5d}", " ".join(errs), flush=True)
