"""The 13-layer VGG step (bench.py's Layer objects) run eagerly (one C-ABI call per layer from
Python) and as one CUDA graph of the same calls: how much of the step is launch overhead?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from synth import workload

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    layers = [bench.Layer(s, "guess", dev, seed=2000 + i) for i, s in enumerate(workload("vgg16", 64))]
    bench._time_stack(layers, 5, st, per_layer=False)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for l in layers:
            l.run(torch.cuda.current_stream().cuda_stream)
    g.replay(); st.synchronize()
    for rep in range(3):
        tot, _ = bench._time_stack(layers, 20, st, per_layer=False)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(20):
            g.replay()
        e.record(st); e.synchronize()
        print(f"eager {tot / 20:.4f} ms/step   graph {s.elapsed_time(e) / 20:.4f} ms/step", flush=True)
