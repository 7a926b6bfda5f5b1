#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200: conv2d TFLOP/s over the VGG-16 conv stack.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--algo guess] [--impl ours|reference] [--quick]

A step = one pass of the hot path over one batch: the 13
VGG-16 3x3 convolutions at 224x224, batch 64 per GPU (BASELINE configs[1]), BF16,
NHWC-resident activations, each layer one C-ABI plan execute (weights prepared at
plan time).  Layers run back to back on independent seeded inputs (the stack's
shapes; no pooling in between).  N GPUs: one process per GPU (under torchrun; with
--gpus N > 1 and no WORLD_SIZE in the environment bench.py launches the N ranks
itself), each with its own batch of 64 (weak scaling, no collective in the data
path); the device time is the max over ranks.

Printed (rank 0, one JSON line): value = total algorithmic TFLOP/s of all ranks;
roofline of the dominant kernel (the tcgen05 implicit-GEMM kernel on the 12
tensor-bound layers); e2e through the C ABI with pinned host buffers (H2D + conv +
D2H per layer); cpu_baseline = the fp64 oracle on host cores on a bounded sample.
Extra legs on the same line (not the metric): measured TF32 / FFMA peaks,
per-algorithm TFLOP/s with each algorithm's own roofline fraction, the fp32 (strict /
TF32) stack, per-layer algorithm tables and selector regret on VGG-16 / AlexNet /
ResNet-50, config-1 latency per algorithm, the dispatch overhead of the hooks, the
all-ai3 VGG-16 model, and BASELINE configs[4] (VGG-16 inference, global batch 2048
sharded over the N GPUs, images/s with the NCCL all-gather excluded).

--impl reference times the oracle (the only other place bench.py runs oracle/):
on the same metric/unit, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import CONFIG1, conv_inputs, workload  # noqa: E402

METRIC = "conv2d TFLOP/s per algorithm (VGG-16/ResNet-50 layers); images/s at 1/2/4/8 B200"
WORKLOAD = "vgg16_conv_stack"
BATCH = 64
FIXED = ("implicit_gemm", "implicit_precomp_gemm", "winograd", "gemm", "kn2row", "direct", "smm")
TENSOR_ALGOS = ("implicit_gemm", "implicit_precomp_gemm", "winograd", "gemm", "kn2row")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), \
            "measured (MEASURED_PEAKS.json)"
    return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def _traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def _winograd_ok(s):
    return s.R == 3 and s.S == 3 and s.stride == 1 and s.dil == 1 and s.groups == 1


def _exec_flops(spec, algo: str, math: str = "bf16") -> float:
    """FLOPs the algorithm must execute on its own pipe: the direct count, except
    Winograd F(2x2,3x3) whose batched GEMM is 16*K*C*T*2 (T = N*ceil(P/2)*ceil(Q/2)); 3xTF32
    (fp32 strict) issues three tensor-core products per term."""
    if algo == "winograd":
        f = 2.0 * 16 * spec.K * spec.C * spec.N * ((spec.P + 1) // 2) * ((spec.Q + 1) // 2)
    else:
        f = float(spec.flops())
    return 3 * f if math == "strict3" else f


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index = index
        self.samples, self.max_mhz, self.reasons = [], None, set()
        self._stop_evt = threading.Event()
        self.ready = threading.Event()  # NVML initialised and sampling (nvmlInit can take > 100 ms)
        self.ok = False

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            while not self._stop_evt.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    mask = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
                self.ready.set()
                time.sleep(0.005)
        except Exception:
            self.ok = False
            self.ready.set()

    def begin(self):
        """Wait until sampling runs, then keep only samples from the timed region on."""
        self.ready.wait(timeout=20)
        self.samples.clear()
        self.reasons.clear()

    def snapshot(self):
        """Summary of the samples since begin() (sampling continues)."""
        samples, reasons = list(self.samples), sorted(self.reasons)
        return {"sm_mhz": statistics.median(samples) if samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(samples)}

    def stop(self):
        self._stop_evt.set()
        self.join(timeout=2)
        return self.snapshot()


# ---------------------------------------------------------------------------- distributed plumbing
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: launch the N ranks (one process per GPU)
    with torch.distributed.run on 127.0.0.1 and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def _max_over_ranks(v: float, device, dist) -> float:
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_launch_check(rank: int, world: int):
    """--launch-check: the multi-rank plumbing without a GPU (gloo): every rank joins the
    process group and reports; rank 0 prints one line with the max over ranks."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    v = _max_over_ranks(float(rank), torch.device("cpu"), dist if world > 1 else None)
    ranks = torch.zeros(1, dtype=torch.int64) + (1 << rank)
    if world > 1:
        dist.all_reduce(ranks)
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "max_rank": v, "ranks_mask": int(ranks.item())}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- oracle legs
def _oracle_run(layers, k: int, seed: int = 7, images: int = 1):
    """The fp64 oracle on `images` images of every layer, first k output channels (a bounded
    sample of the step: conv is independent per image and per output channel).
    Returns (flops, secs)."""
    import oracle
    threads = oracle.host_threads()
    flops, secs = 0, 0.0
    for i, l in enumerate(layers):
        x, w, b = conv_inputs(l.with_batch(images), seed + i, "bf16")
        kk = min(k, l.K)
        t0 = time.perf_counter()
        oracle.conv2d(x, w[:kk], b[:kk], l.stride, l.pad, l.dil, l.groups, threads=threads)
        secs += time.perf_counter() - t0
        flops += 2 * images * kk * (l.C // l.groups) * l.R * l.S * l.P * l.Q
    return flops, secs


def _oracle_calibrate(layers, seconds: float):
    """Smallest sample (k output channels per layer, then whole images) taking >= `seconds`:
    returns (k, images)."""
    import oracle
    oracle.build()
    kmax = max(l.K for l in layers)
    k, images = 1, 1
    while True:
        _, dt = _oracle_run(layers, k, images=images)
        if dt >= seconds or images >= 64:
            return k, images
        grow = min(8.0, 1.2 * seconds / max(dt, 1e-3))
        if k < kmax:
            k = min(kmax, max(k + 1, int(k * grow)))
        else:
            images = min(64, max(images + 1, int(images * grow)))


def _sample_desc(layers, k: int, flops: int, threads: int, images: int = 1) -> str:
    ch = "every output channel" if k >= max(l.K for l in layers) else f"first {k} output channel(s)"
    return (f"{images} image(s) x {ch} of each of the {len(layers)} {WORKLOAD} layers "
            f"({flops / 1e9:.2f} GFLOP), fp64 oracle, {threads} threads")


def run_reference(args, rank: int, world: int):
    """Reference arm: the oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    layers = workload("vgg16", BATCH)
    per_step = max(0.5, min(2.0, 150.0 / max(1, args.steps + args.warmup)))
    k, images = _oracle_calibrate(layers, per_step)
    times, flops = [], 0
    for i in range(args.warmup + args.steps):
        flops, dt = _oracle_run(layers, k, images=images)
        if i >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    value = flops / mean / 1e12
    desc = _sample_desc(layers, k, flops, oracle.host_threads(), images)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "image": 224, "sample": desc},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": oracle.host_threads(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
class Layer:
    """One conv layer of a workload: seeded device input, a plan (weights prepared once), its
    output and workspace -- the launch configuration every timing leg uses."""

    def __init__(self, spec, algo: str, device, seed: int, dtype: str = "bf16", math: str = "strict"):
        import paper_2410_08300_b200 as ai3
        self.spec = spec
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        _, w, b = conv_inputs(spec.with_batch(1), seed, dtype)  # weights/bias: synth recipe
        g = torch.Generator(device=device).manual_seed(seed)
        self.x = torch.randn((spec.N, spec.C, spec.H, spec.W), generator=g, device=device, dtype=torch.float32) \
            .to(tdt).contiguous(memory_format=torch.channels_last)
        wt = torch.from_numpy(w).to(device=device, dtype=tdt)
        bt = None if b is None else torch.from_numpy(b).to(device=device, dtype=tdt)
        if algo == "benchmark":  # measure every algorithm once for this layer; the plan takes the winner
            ai3.autotune(self.x, wt, bt, spec.stride, spec.pad, spec.dil, spec.groups, math)
        self.plan = ai3.ConvPlan(wt, bt, self.x.shape, spec.stride, spec.pad, spec.dil, spec.groups, algo, math,
                                 in_layout=1, out_layout=1)
        self.y = torch.empty(self.plan.out_shape, dtype=tdt, device=device, memory_format=torch.channels_last)
        self.ws = torch.empty(max(self.plan.workspace_size, 256), dtype=torch.uint8, device=device)
        self.flops = spec.flops()

    def run(self, stream_ptr: int):
        self.plan.execute_raw(self.x.data_ptr(), self.y.data_ptr(), self.ws.data_ptr(), self.ws.numel(), stream_ptr)


def _time_stack(layers, steps: int, stream, per_layer: bool):
    sp = stream.cuda_stream
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in layers]
          for _ in range(steps)] if per_layer else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for s in range(steps):
        for i, l in enumerate(layers):
            if per_layer:
                ev[s][i][0].record(stream)
            l.run(sp)
            if per_layer:
                ev[s][i][1].record(stream)
    end.record(stream)
    end.synchronize()
    total_ms = start.elapsed_time(end)
    layer_ms = None
    if per_layer:
        layer_ms = [sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(steps)) / steps
                    for i in range(len(layers))]
    return total_ms, layer_ms


def _time_fn(fn, stream, reps: int, warm: int = 2) -> float:
    """Mean device ms of fn() over reps back-to-back calls (CUDA events on `stream`)."""
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps):
        fn()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / reps


def _roof_ms(spec, algo: str, peaks: dict, math: str = "bf16") -> float:
    """Roofline time of one layer for `algo`: max(F_exec / pipe peak, B_alg / HBM)."""
    if algo in ("direct", "smm"):
        pipe = peaks["ffma_tflops"]
    elif math == "tf32" or math == "strict3":
        pipe = peaks["tf32_tflops"]
    else:
        pipe = peaks["bf16_tflops"]
    elem = 2 if math == "bf16" else 4
    t_pipe = _exec_flops(spec, algo, math) / (pipe * 1e12)
    t_mem = spec.alg_bytes(elem) / (peaks["hbm_gbs"] * 1e9)
    return max(t_pipe, t_mem) * 1e3


def measure_peaks(device, stream) -> dict:
    """TF32 tensor and FP32 FFMA peaks, measured on this box (the roofline denominators the
    driver's MEASURED_PEAKS.json lacks): torch.matmul 8192^3 fp32 with allow_tf32 (best of 10,
    the same method as the driver's bf16 figure), and libai3_calib.so's FFMA microbenchmark
    (148 x 4 blocks x 512 threads x 8 independent chains; best of 5)."""
    out = {}
    a = torch.randn(8192, 8192, device=device)
    b = torch.randn(8192, 8192, device=device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        best = min(_time_fn(lambda: torch.matmul(a, b), stream, 1, warm=3 if i == 0 else 0) for i in range(10))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    out["tf32_tflops"] = 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    del a, b
    from paper_2410_08300_b200 import build as B
    lib = ctypes.CDLL(B.build_calib())
    lib.ai3_calib_ffma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.ai3_calib_ffma.restype = ctypes.c_double
    sink = torch.zeros(4096, device=device)
    blocks = torch.cuda.get_device_properties(device).multi_processor_count * 4
    flop = lib.ai3_calib_ffma(blocks, 4096, sink.data_ptr(), stream.cuda_stream)
    best = min(_time_fn(lambda: lib.ai3_calib_ffma(blocks, 4096, sink.data_ptr(), stream.cuda_stream), stream, 1,
                        warm=1) for _ in range(5))
    out["ffma_tflops"] = flop / (best * 1e-3) / 1e12
    out["how"] = ("tf32: torch.matmul 8192^3 fp32, allow_tf32, best of 10; ffma: libai3_calib.so FFMA chains "
                  f"({blocks} x 512 threads x 8 chains x 32768 FMA), best of 5; both CUDA events")
    return out


def _algo_table(specs, algos, device, stream, seed0: int, reps: int = 3):
    """Per-layer device ms of every algorithm on every layer (the launch configuration of the
    metric: bf16, NHWC), None where the algorithm does not support the layer."""
    table = {a: [] for a in algos}
    used = {a: [] for a in algos}
    for i, spec in enumerate(specs):
        for a in algos:
            if a == "winograd" and not _winograd_ok(spec):
                table[a].append(None)
                used[a].append(None)
                continue
            try:
                lay = Layer(spec, a, device, seed=seed0 + i)
            except Exception:
                table[a].append(None)
                used[a].append(None)
                continue
            r = 1 if (a in ("direct", "smm") and spec.flops() > 2e11) else reps
            table[a].append(_time_fn(lambda: lay.run(stream.cuda_stream), stream, r, warm=1))
            used[a].append(lay.plan.algorithm)
            del lay
        torch.cuda.empty_cache()
    return table, used


def _selector_quality(specs, table, fixed):
    best = []
    best_alg = []
    for i in range(len(specs)):
        cands = [(table[a][i], a) for a in fixed if table[a][i] is not None]
        t, a = min(cands)
        best.append(t * specs[i].count)
        best_alg.append(a)
    out = {"best_per_layer": dict(zip([s.name for s in specs], best_alg))}
    for sel in ("guess", "benchmark"):
        if sel in table and all(v is not None for v in table[sel]):
            out[f"{sel}_regret"] = round(sum(t * s.count for t, s in zip(table[sel], specs)) / sum(best), 4)
    return out


def _net_leg(net, nb, algos, device, stream, peaks, seed0):
    """Per-layer, per-algorithm table of one network (BASELINE configs[2] / [3]) with roofline
    fractions and selector regret; the `guess` column is the network's headline time."""
    specs = workload(net, nb)
    table, used = _algo_table(specs, algos, device, stream, seed0)
    tot = {}
    for a in algos:
        if all(v is not None for v in table[a]):
            ms = sum(t * s.count for t, s in zip(table[a], specs))
            roof = sum(_roof_ms(s, a if a not in ("guess", "benchmark") else "implicit_gemm", peaks) * s.count
                       for s in specs)
            tot[a] = {"ms": round(ms, 4), "tflops": round(sum(s.flops() * s.count for s in specs) / (ms * 1e-3) / 1e12,
                                                         1), "roofline_frac": round(roof / ms, 3)}
    g = table["guess"]
    rows = [[s.name, s.count, round(g[i] * 1e3, 1), round(s.flops() / (g[i] * 1e-3) / 1e12, 1), used["guess"][i],
             round(_roof_ms(s, used["guess"][i], peaks) / g[i], 3)] for i, s in enumerate(specs)]
    ms_g = sum(t * s.count for t, s in zip(g, specs))
    return {"batch": nb, "convs": sum(s.count for s in specs), "ms_all_convs": round(ms_g, 4),
            "tflops": round(sum(s.flops() * s.count for s in specs) / (ms_g * 1e-3) / 1e12, 1),
            "images_per_s": round(nb / (ms_g * 1e-3), 1),
            "roofline_frac": round(sum(_roof_ms(s, used["guess"][i], peaks) * s.count for i, s in enumerate(specs))
                                   / ms_g, 3),
            "layers_us_tflops_algo_frac": rows, "per_algorithm": tot,
            "per_layer_us": {a: [None if v is None else round(v * 1e3, 1) for v in table[a]] for a in algos},
            "selector_quality": _selector_quality(specs, table, [a for a in algos if a in FIXED])}


def _config1_latency(device, stream):
    """BASELINE configs[0] (N=1 C=3 32x32 K=16 3x3, fp32): device us per call of every
    algorithm's plan execute (launch-latency-bound; report us, not TF/s)."""
    out = {}
    for a in FIXED + ("guess",):
        for math in (("strict", "tf32") if a in TENSOR_ALGOS else ("strict",)):
            try:
                lay = Layer(CONFIG1, a, device, seed=1000, dtype="f32", math=math)
            except Exception as ex:
                out[f"{a}/{math}"] = f"error: {ex}"
                continue
            us = _time_fn(lambda: lay.run(stream.cuda_stream), stream, 200, warm=5) * 1e3
            out[f"{a}/{math}"] = {"us": round(us, 2), "launches": lay.plan.num_launches}
    return out


def _dispatch_overhead(device, stream):
    """Hook dispatch overhead: one
    ai3.Conv2D forward (the swapped module, as a user calls it) against the bare
    ai3_conv2d_plan_execute on the same plan, 50 back-to-back calls each, device time with
    CUDA events (what the overhead costs the GPU) and host time per call."""
    import paper_2410_08300_b200 as ai3
    from torch import nn
    res = {}
    for name, spec, dt in (("vgg_conv1_2_n64_bf16", workload("vgg16", 64)[1], torch.bfloat16),
                           ("config1_fp32", CONFIG1, torch.float32)):
        torch.manual_seed(0)
        conv = nn.Conv2d(spec.C, spec.K, spec.R, spec.stride, spec.pad, bias=True).to(device=device, dtype=dt)
        mod = ai3.Conv2D(conv, "guess")
        x = torch.randn((spec.N, spec.C, spec.H, spec.W), device=device).to(dt)
        if dt == torch.bfloat16:
            x = x.contiguous(memory_format=torch.channels_last)
        with torch.inference_mode():
            y = mod(x)
            plan = mod.plan_for(x)
            ws = torch.empty(max(plan.workspace_size, 256), dtype=torch.uint8, device=device)
            sp = stream.cuda_stream
            reps = 50
            t_bare = _time_fn(lambda: plan.execute_raw(x.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), sp),
                              stream, reps, warm=5)
            t_mod = _time_fn(lambda: mod(x), stream, reps, warm=5)
            torch.cuda.synchronize(device)
            h0 = time.perf_counter()
            for _ in range(reps):
                plan.execute_raw(x.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), sp)
            h1 = time.perf_counter()
            for _ in range(reps):
                mod(x)
            h2 = time.perf_counter()
            torch.cuda.synchronize(device)
        res[name] = {"algorithm": plan.algorithm, "device_us_bare": round(t_bare * 1e3, 2),
                     "device_us_conv2d_forward": round(t_mod * 1e3, 2),
                     "overhead_us": round((t_mod - t_bare) * 1e3, 2),
                     "overhead_pct": round(100 * (t_mod - t_bare) / t_bare, 2),
                     "host_us_per_call_bare": round((h1 - h0) / reps * 1e6, 2),
                     "host_us_per_call_conv2d_forward": round((h2 - h1) / reps * 1e6, 2)}
    return res


def _precision_leg(specs, device, stream, peaks, steps: int):
    """The paper's arithmetic (fp32 inputs) on the VGG stack: implicit_gemm in
    fp32 `strict` (3xTF32) and `tf32`, TFLOP/s (direct count) and the fraction of the measured
    TF32 peak over the executed tensor-core FLOPs (3x for strict)."""
    out = {}
    for math in ("strict", "tf32"):
        lays = [Layer(s, "implicit_gemm", device, seed=1000 * 2 + i, dtype="f32", math=math)
                for i, s in enumerate(specs)]
        _time_stack(lays, 1, stream, per_layer=False)
        reps = max(1, min(steps, 5))
        ms, lms = _time_stack(lays, reps, stream, per_layer=True)
        ms /= reps
        roof = sum(_roof_ms(s, "implicit_gemm", peaks, "strict3" if math == "strict" else "tf32") for s in specs)
        out[f"implicit_gemm/f32_{math}"] = {"ms": round(ms, 3),
                                           "tflops": round(sum(s.flops() for s in specs) / (ms * 1e-3) / 1e12, 1),
                                           "roofline_frac_of_tf32": round(roof / ms, 3),
                                           "algorithms": sorted({l.plan.algorithm for l in lays})}
        del lays
        torch.cuda.empty_cache()
    return out


def run_ours(args, rank: int, world: int, local_rank: int):
    import paper_2410_08300_b200 as ai3  # noqa: F401  (fails loudly if libai3.so is missing)
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    dist = torch.distributed if world > 1 else None
    specs = workload("vgg16", BATCH)
    layers = [Layer(s, args.algo, device, seed=1000 * 2 + i) for i, s in enumerate(specs)]
    stream = torch.cuda.current_stream(device)
    launches_per_step = sum(l.plan.num_launches for l in layers)
    step_flops = sum(l.flops for l in layers)

    # warm-up (also first-touch of every buffer)
    _time_stack(layers, max(args.warmup, 1), stream, per_layer=False)
    torch.cuda.synchronize(device)

    sampler = ClockSampler(device.index if device.index is not None else 0)
    sampler.start()
    sampler.begin()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    # the metric's timed region: K back-to-back steps between two events.  No event sits between
    # the layers here -- an event record between two kernels ends the programmatic overlap of one
    # layer's prologue with the previous layer's tail (measured: 0.04-0.26 ms per step)
    total_ms, _ = _time_stack(layers, args.steps, stream, per_layer=False)
    torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    clocks = sampler.snapshot()
    # per-layer device times (the roofline's kernel durations): the same K steps again, with
    # events around every layer (clocks sampled separately: they pick the roofline's peak)
    sampler.begin()
    _, layer_ms = _time_stack(layers, args.steps, stream, per_layer=True)
    torch.cuda.synchronize(device)
    layer_clocks = sampler.stop()
    ms_per_step = _max_over_ranks(total_ms / args.steps, device, dist)
    value = world * step_flops / (ms_per_step * 1e-3) / 1e12
    images_per_s = world * BATCH / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel: tcgen05 implicit GEMM on the tensor-bound layers.
    # Its time per step = the metric's timed step x its share of the step, the share measured
    # with per-layer events in the second pass (those events would end the programmatic
    # overlap in the timed region itself; the second pass also runs later, i.e. hotter, so its
    # absolute times are reported beside, not used).  Denominator: the burst bf16 peak when the
    # timed region held the max SM clock (a short, not power-capped region), else the
    # sustained one; the other ratio is reported beside it.
    burst, sustained, hbm, peak_src = _peaks()
    at_max = clocks["sm_mhz"] is not None and clocks["sm_max_mhz"] and clocks["sm_mhz"] >= 0.97 * clocks["sm_max_mhz"]
    peak = burst if at_max or clocks["sm_mhz"] is None else sustained
    tc_idx = [i for i, l in enumerate(layers) if l.spec.C >= 64]
    tc_flops = sum(layers[i].flops for i in tc_idx)
    tc_share = sum(layer_ms[i] for i in tc_idx) / sum(layer_ms)
    tc_ms = ms_per_step * tc_share
    achieved = tc_flops / (tc_ms * 1e-3) / 1e12
    pass_achieved = tc_flops / (sum(layer_ms[i] for i in tc_idx) * 1e-3) / 1e12
    traffic = _traffic()
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_kind": (f"bf16 {'burst' if peak == burst else 'sustained'} of {peak_src}: the timed region "
                              f"ran at {clocks['sm_mhz']} of {clocks['sm_max_mhz']} MHz"),
                "frac_of_burst": achieved / burst, "frac_of_sustained": achieved / sustained,
                "kernel": "tc_gemm_kernel (implicit GEMM, 12 tensor-bound VGG layers, 1 launch each)",
                "launches_per_step": len(tc_idx),
                "algorithmic_flops_per_launch_avg": tc_flops / len(tc_idx),
                "kernel_ms_per_step": tc_ms, "share_of_step": tc_share,
                "per_layer_pass": {"achieved": pass_achieved, "clocks": layer_clocks,
                                   "note": "the same layers timed one by one in the second pass"},
                "traffic": traffic.get("bytes_per_launch") if traffic else None}
    if traffic:
        roofline["traffic_note"] = traffic.get("note")
    per_layer = [{"layer": l.spec.name, "ms": round(layer_ms[i], 4),
                  "tflops": round(l.flops / (layer_ms[i] * 1e-3) / 1e12, 1),
                  "algorithm": l.plan.algorithm, "launches": l.plan.num_launches}
                 for i, l in enumerate(layers)]

    # ---- e2e: host buffers through the C ABI (H2D + conv + D2H per layer)
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, 5))
        hx = [torch.empty_like(l.x, device="cpu").pin_memory().copy_(l.x.cpu()) for l in layers]
        hy = [torch.empty(l.y.shape, dtype=l.y.dtype).contiguous(memory_format=torch.channels_last).pin_memory()
              for l in layers]
        plans, xd, yd = [l.plan for l in layers], [l.x for l in layers], [l.y for l in layers]
        ai3.execute_host_many(plans, hx, hy, xd, yd)  # warm
        torch.cuda.synchronize(device)
        if dist:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(e2e_steps):
            ai3.execute_host_many(plans, hx, hy, xd, yd)
        e.record(stream)
        e.synchronize()
        e2e_ms = _max_over_ranks(s.elapsed_time(e) / e2e_steps, device, dist)
        h2d = sum(x.numel() * x.element_size() for x in hx)
        d2h = sum(y.numel() * y.element_size() for y in hy)
        e2e = {"value": world * step_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "ai3_conv2d_plans_execute_host over the 13 layers (H2D / conv / D2H of consecutive layers "
                       "overlapped on copy streams), pinned host memory"}
        del hx, hy
    del layers
    torch.cuda.empty_cache()

    extras = {}
    if rank == 0 and not args.quick:
        peaks = {"bf16_tflops": burst, "hbm_gbs": hbm}
        try:
            peaks.update(measure_peaks(device, stream))
        except Exception as ex:  # report, do not hide
            peaks.update({"tf32_tflops": 1100.0, "ffma_tflops": 74.4, "error": str(ex),
                          "how": "fallback: nominal TF32 1.1 PF; FFMA 148 SM x 128 x 2 x 1.965 GHz"})
        extras["peaks"] = peaks
        # per-algorithm VGG stack, each against its own roofline (SURVEY §8d "Roofline per path")
        vgg_algos = FIXED + ("guess", "benchmark")
        table, used = _algo_table(specs, vgg_algos, device, stream, seed0=1000 * 2)
        per_algo = {}
        for a in vgg_algos:
            if any(v is None for v in table[a]):
                per_algo[a] = "unsupported on some layer"
                continue
            ms = sum(table[a])
            base = a if a in FIXED else None
            roof = sum(_roof_ms(s, base or used[a][i], peaks) for i, s in enumerate(specs))
            per_algo[a] = {"ms": round(ms, 3), "tflops": round(step_flops / (ms * 1e-3) / 1e12, 1),
                           "roofline_frac": round(roof / ms, 3),
                           "bound": "ffma" if a in ("direct", "smm") else "tensor/hbm"}
        extras["per_algorithm"] = per_algo
        extras["vgg16_per_layer_us"] = {a: [None if v is None else round(v * 1e3, 1) for v in table[a]]
                                        for a in vgg_algos}
        extras["selector_quality"] = {"vgg16": _selector_quality(specs, table, list(FIXED))}
        if not args.no_configs:
            for net, nb, seed0 in (("alexnet", 128, 4000), ("resnet50", 256, 3000)):
                try:
                    leg = _net_leg(net, nb, FIXED + ("guess", "benchmark"), device, stream, peaks, seed0)
                    extras.setdefault("other_configs", {})[net] = leg
                    extras["selector_quality"][net] = leg["selector_quality"]
                except Exception as ex:  # report, do not hide
                    extras.setdefault("other_configs", {})[net] = {"error": repr(ex)}
        try:
            extras["fp32_stack"] = _precision_leg(specs, device, stream, peaks, args.steps)
        except Exception as ex:
            extras["fp32_stack"] = {"error": repr(ex)}
        extras["config1_latency_us"] = _config1_latency(device, stream)
        extras["dispatch_overhead"] = _dispatch_overhead(device, stream)
        torch.cuda.empty_cache()

    # ---- the whole model: swap_backend(VGG-16), every op in ai3, at this rank's step batch
    if not args.no_model and rank == 0:
        from paper_2410_08300_b200.runner import build_vgg16, make_images
        try:
            model = build_vgg16(device, algo=args.algo, seed=0, swap="backend")
            xm = make_images(0, BATCH, 5001, device)
            with torch.inference_mode():
                mms = _time_fn(lambda: model(xm), stream, max(3, min(args.steps, 20)), warm=3)
            extras["vgg16_model"] = {"model": "vgg16 (torchvision, random init), swap_backend: all ops in ai3",
                                     "batch": BATCH, "ms_per_forward": mms, "images_per_s": BATCH / (mms * 1e-3),
                                     "ops_kept_in_torch": len(model.kept)}
            del model, xm
            torch.cuda.empty_cache()
        except Exception as ex:  # report, do not hide
            extras["vgg16_model"] = {"error": repr(ex)}

    # ---- BASELINE configs[4]: VGG-16 inference, global batch 2048 sharded over the N ranks
    if not args.no_config5:
        from paper_2410_08300_b200 import runner
        if dist:
            dist.barrier()
        try:
            r5 = runner.run(args.config5_batch, args.algo, steps=3, warmup=3, seed=5000, check=True,
                            swap="backend", quiet=True, finalize=False)
            extras["config5"] = r5
        except Exception as ex:  # report, do not hide
            extras["config5"] = {"error": repr(ex)}
        torch.cuda.empty_cache()

    cpu = None
    if world == 1 and not args.no_cpu:  # the oracle on host cores (rank 0, N=1 only)
        import oracle
        k, images = _oracle_calibrate(specs, args.cpu_seconds)
        flops, dt = _oracle_run(specs, k, images=images)
        cpu = {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.host_threads(), "kind": "oracle",
               "sample": _sample_desc(specs, k, flops, oracle.host_threads(), images), "seconds": round(dt, 2)}

    if dist:
        dist.barrier()  # every rank stays until rank 0's extra legs are done
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "global_batch": BATCH * world,
                           "image": 224, "layers": len(specs), "layout": "NHWC", "algorithm": args.algo,
                           "parallelism": f"dp{world} (batch-sharded, no collective in the step)",
                           "l2": "step working set ~2.9 GB of distinct per-layer buffers >> 126 MB L2; no flush"},
                "images_per_s": images_per_s, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks, "per_layer": per_layer}
        line.update(extras)
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="guess")
    ap.add_argument("--quick", action="store_true", help="metric, roofline and e2e only (no extra legs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-model", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--config5-batch", type=int, default=2048)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--launch-check", action="store_true", help="multi-rank plumbing only (gloo, no GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:
        run_launch_check(rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 and torch.distributed.is_initialized():
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
