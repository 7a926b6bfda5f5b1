"""Per-role pipeline-wait breakdown of one layer's tc_gemm launch (AI3_TC_TRACE=1)."""
import ctypes, os, sys
os.environ["AI3_TC_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2410_08300_b200 import _lib
_lib.select_library(os.path.join(ROOT, "paper_2410_08300_b200", "libai3_dev.so"))  # knobs (AI3_TC_TRACE) need the dev build
import paper_2410_08300_b200 as ai3
from synth import workload, conv_inputs
net = sys.argv[2] if len(sys.argv) > 2 else "vgg16"
spec = [l for l in workload(net) if l.name == sys.argv[1]][0]
x = torch.randn(spec.N, spec.C, spec.H, spec.W, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
_, w, b = conv_inputs(spec.with_batch(1), 1, "bf16")
p = ai3.ConvPlan(torch.from_numpy(w).cuda().bfloat16(), None if b is None else torch.from_numpy(b).cuda().bfloat16(), x.shape, spec.stride,
                 spec.pad, spec.dil, 1, sys.argv[3] if len(sys.argv) > 3 else "guess", in_layout=1)
y = p(x); torch.cuda.synchronize()
lib = _lib.load()
lib.ai3_debug_tc_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((296, 16), dtype=np.uint64)
lib.ai3_debug_tc_trace(buf.ctypes.data, 296)  # reset
p(x, out=y); torch.cuda.synchronize()
lib.ai3_debug_tc_trace(buf.ctypes.data, 296)
rows = buf[buf[:, 6] > 0].astype(np.float64)
names = ["prod_wait_empty", "prod_total", "mma_wait_full", "mma_wait_tempty", "mma_total", "epi_wait_tfull", "epi_total", "epi_tiles", "epi_ld_wait", "epi_tile_proc", "epi_slot_wait", "epi_fence_store", "epi_fence", "epi_release"]
print(spec.name, p.algorithm, "ctas", len(rows))
for i, n in enumerate(names):
    col = rows[:, i]
    print(f"  {n:16s} mean {col.mean():12.0f}  max {col.max():12.0f}")
