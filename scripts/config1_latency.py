"""BASELINE configs[0] latency per algorithm, three ways: events around 200 back-to-back
plan executes (bench.py's leg), the same as one CUDA graph of 200 executes (no host launch
cost), and the host wall time of one execute + synchronize."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from synth import CONFIG1

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for a in ("direct", "smm", "implicit_gemm", "gemm", "winograd", "guess"):
        lay = bench.Layer(CONFIG1, a, dev, seed=1000, dtype="f32", math="strict")
        sp = st.cuda_stream
        t_ev = bench._time_fn(lambda: lay.run(sp), st, 200, warm=5) * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20):
                lay.run(torch.cuda.current_stream().cuda_stream)
        g.replay(); st.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(10):
            g.replay()
        e.record(st); e.synchronize()
        t_graph = s.elapsed_time(e) / 200 * 1e3
        walls = []
        for _ in range(50):
            t0 = time.perf_counter(); lay.run(sp); st.synchronize(); walls.append(time.perf_counter() - t0)
        walls.sort()
        print(f"{a:14s} events {t_ev:7.2f} us   graph {t_graph:7.2f} us   wall(median) {walls[25] * 1e6:7.2f} us  "
              f"launches {lay.plan.num_launches}", flush=True)
