"""Quick GPU probe: all shapes / modes / layouts for one algorithm (one process per
algorithm so a hang is contained by the caller's timeout).  Prints as it goes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from synth import ConvShape, conv_inputs
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import run_ai3, ref, tolerance

algo = sys.argv[1]
SHAPES = [(1, 3, 32, 32, 16, 3, 3, 1, 1), (2, 64, 23, 23, 96, 3, 3, 1, 1), (2, 3, 45, 45, 64, 7, 7, 2, 3),
          (2, 256, 14, 14, 72, 1, 1, 1, 0), (2, 128, 28, 28, 256, 3, 3, 1, 1)]
for dims in SHAPES:
    shape = ConvShape("probe", *dims)
    if algo == "winograd" and (shape.R != 3 or shape.stride != 1):
        continue
    for dtype, math in (("bf16", "strict"), ("f32", "tf32"), ("f32", "strict")):
        for layout in ("nhwc", "nchw"):
            x, w, b = conv_inputs(shape, 1, dtype)
            t = time.time()
            try:
                y = run_ai3(shape, x, w, b, algo, dtype, math, layout)
            except Exception as e:
                print(f"EXC  {algo} {dtype}/{math} {layout} {dims}: {e}", flush=True)
                continue
            r = ref(shape, x, w, b)
            e = oracle.rel_err(y, r)
            tol = tolerance(algo, dtype, math)
            print(f"{'OK  ' if e <= tol else 'FAIL'} {algo:14s} {dtype}/{math:6s} {layout} {dims} "
                  f"rel_err={e:.3e} tol={tol:.0e} ({time.time()-t:.2f}s)", flush=True)
