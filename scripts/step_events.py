"""Does timing each layer with its own CUDA events slow the bench step down?  The 13-layer
VGG step (bench.py's Layer / _time_stack) timed with and without per-layer events,
alternating, on the same plans and buffers."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from synth import workload

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
layers = [bench.Layer(s, "guess", dev, seed=2000 + i) for i, s in enumerate(workload("vgg16", 64))]
stream = torch.cuda.current_stream(dev)
bench._time_stack(layers, 5, stream, per_layer=False)
for rep in range(3):
    for pl in (False, True):
        tot, lay = bench._time_stack(layers, 20, stream, per_layer=pl)
        extra = f"  sum(per-layer) {sum(lay):.4f} ms" if lay else ""
        print(f"per_layer={pl}: {tot / 20:.4f} ms/step{extra}", flush=True)
