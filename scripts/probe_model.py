"""Run swap_backend(VGG-16) node by node with a synchronize after each (locate hangs / slow ops)."""
import sys
import time

import torch
import torchvision

sys.path.insert(0, ".")
import paper_2410_08300_b200 as ai3  # noqa: E402
from paper_2410_08300_b200 import _lib  # noqa: E402
from paper_2410_08300_b200.layers import to_layout  # noqa: E402

dt = torch.float32 if sys.argv[1] == "f32" else torch.bfloat16
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.manual_seed(0)
vgg = torchvision.models.vgg16(weights=None).eval().cuda().to(dt)
model = ai3.swap_backend(vgg)
gm = model.graph_module
x = to_layout(torch.randn(batch, 3, 224, 224, device="cuda").to(dt), _lib.NHWC)
env = {}
mods = dict(gm.named_modules())
with torch.inference_mode():
    for node in gm.graph.nodes:
        t0 = time.time()
        if node.op == "placeholder":
            env[node.name] = x
            continue
        if node.op == "output":
            break
        args = torch.fx.node.map_arg(node.args, lambda n: env[n.name])
        kwargs = torch.fx.node.map_arg(node.kwargs, lambda n: env[n.name])
        if node.op == "call_module":
            m = mods[node.target]
            desc = f"{node.target} {type(m).__name__} {getattr(m, 'algorithm', '')} relu={getattr(m, 'relu', '')}"
            print("start", desc, flush=True)
            out = m(*args, **kwargs)
        else:
            desc = f"{node.name} {node.target}"
            print("start", desc, flush=True)
            out = node.target(*args, **kwargs)
        torch.cuda.synchronize()
        env[node.name] = out
        print(f"done  {desc} {tuple(out.shape)} {(time.time() - t0) * 1e3:.1f} ms", flush=True)
print("ok")
