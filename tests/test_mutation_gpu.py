"""The parity harness has teeth: a deliberately faulty build of the library
must fail it.

``libai3_mutant.so`` is libai3 compiled with -DAI3_MUTANT_DROP_BIAS (paper_2410_08300_b200/
build.py, built by ``__graft_entry__.build()``): the plan-time bias kernel (csrc/prep.cu
bias_f32_kernel) loses the LAST output channel's bias -- an off-by-one of the kind a real
kernel bug produces, in code every algorithm's plan runs.  The same harness the parity
tests use (seeded inputs, oracle, north_star tolerance or bit-exact integer comparison)
runs once against the product library and once against the mutant, each in its own
process (the library is chosen before the first load, paper_2410_08300_b200._lib.select_library).
The product must pass every case and the mutant must fail every case.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2410_08300_b200")
ALGOS = ["direct", "gemm", "implicit_gemm", "implicit_precomp_gemm", "winograd", "smm", "kn2row"]

_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2410_08300_b200 import _lib
_lib.select_library(sys.argv[2])
import torch
import oracle
import paper_2410_08300_b200 as ai3
from synth import CONFIG1, ConvShape, conv_inputs, integer_inputs
out = {}
s = CONFIG1  # BASELINE configs[0], fp32 strict
x, w, b = conv_inputs(s, seed=1000, dtype="f32")
ref = oracle.conv2d(x, w, b, s.stride, s.pad, s.dil, s.groups)
for algo in json.loads(sys.argv[3]):
    y = ai3.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(),
                   s.stride, s.pad, s.dil, s.groups, algorithm=algo)
    out["f32/" + algo] = oracle.rel_err(y.double().cpu().numpy(), ref)
# integer-valued bf16 layer (exact on every path): bit-exact comparison
sh = ConvShape("mut_int", 2, 64, 12, 12, 64, 3, 3, 1, 1)
xi, wi, bi = integer_inputs(sh, seed=5, xmax=1, wmax=1)
wi = wi * (np.arange(wi.size).reshape(wi.shape) % 3 == 0)  # keep |y| <= 256: bf16 outputs stay exact
bi[-1] = 1.0  # the channel the mutant breaks carries a bias
ri = oracle.conv2d(xi, wi, bi, 1, 1, 1, 1)
xt = torch.from_numpy(xi.astype(np.float32)).cuda().bfloat16().contiguous(memory_format=torch.channels_last)
for algo in json.loads(sys.argv[3]):
    if algo == "winograd":
        continue  # bf16 Winograd rounds M to bf16 (DESIGN.md R26): not bit-exact; the fp32 case covers it
    p = ai3.ConvPlan(torch.from_numpy(wi.astype(np.float32)).cuda().bfloat16(),
                     torch.from_numpy(bi.astype(np.float32)).cuda().bfloat16(), xt.shape, 1, 1, 1, 1, algo,
                     in_layout=1)
    y = p(xt).double().cpu().numpy()
    out["int/" + algo] = float(np.abs(y - ri).max())
torch.cuda.synchronize()
print("RESULT " + json.dumps(out))
"""


def _run(lib_path):
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, lib_path, json.dumps(ALGOS)], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_mutant_library_fails_parity_and_product_passes():
    mutant = os.path.join(PKG, "libai3_mutant.so")
    if not os.path.exists(mutant):
        from paper_2410_08300_b200 import build
        build.build(variant="mutant")
    good = _run(os.path.join(PKG, "libai3.so"))
    bad = _run(mutant)
    for algo in ALGOS:
        tol = 1e-3 if algo == "winograd" else 1e-5
        assert good["f32/" + algo] <= tol, (algo, good)
        if algo != "winograd":
            assert good["int/" + algo] == 0.0, (algo, good)
        assert bad["f32/" + algo] > tol, f"mutant not caught by the fp32 harness on {algo}: {bad}"
        if algo != "winograd":
            assert bad["int/" + algo] > 0.0, f"mutant not caught by the bit-exact harness on {algo}: {bad}"
