"""One swap_backend(VGG-16) forward at batch 64 after warm-up (run under ncu for the launch list)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2410_08300_b200.runner import build_vgg16, make_images  # noqa: E402

dev = torch.device("cuda", 0)
model = build_vgg16(dev, algo=sys.argv[1] if len(sys.argv) > 1 else "guess", seed=0, swap="backend")
x = make_images(0, 64, 5001, dev)
with torch.inference_mode():
    for _ in range(3):
        model(x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")
    model(x)
    torch.cuda.synchronize()
