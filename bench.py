#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200: conv2d TFLOP/s over the VGG-16 conv stack.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--algo implicit_gemm] [--impl ours|reference]

A step = one pass of the hot path over one batch: the 13
VGG-16 3x3 convolutions at 224x224, batch 64 per GPU (BASELINE configs[1]), BF16,
NHWC-resident activations, each layer one C-ABI plan execute (weights prepared at
plan time).  Layers run back to back on independent seeded inputs (the stack's
shapes; no pooling in between).  N GPUs: one process per GPU under torchrun, each
with its own batch of 64 (weak scaling, no collective in the data path); the
device time is the max over ranks.

Printed (rank 0, one JSON line): value = total algorithmic TFLOP/s of all ranks;
roofline of the dominant kernel (the tcgen05 implicit-GEMM kernel on the 12
tensor-bound layers); e2e through the C ABI with pinned host buffers (H2D + conv +
D2H per layer); cpu_baseline = the fp64 oracle on host cores on a bounded sample.

--impl reference times the oracle (the only other place bench.py runs oracle/):
on the same metric/unit, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import conv_inputs, workload  # noqa: E402

METRIC = "conv2d TFLOP/s per algorithm (VGG-16/ResNet-50 layers); images/s at 1/2/4/8 B200"
WORKLOAD = "vgg16_conv_stack"
BATCH = 64


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), \
            "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def _traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


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

    def stop(self):
        self._stop_evt.set()
        self.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- oracle legs
def _oracle_run(layers, k: int, seed: int = 7):
    """The fp64 oracle on one image of every layer, first k output channels (a bounded
    sample of the step: conv is independent per output channel).  Returns (flops, secs)."""
    import oracle
    threads = oracle.host_threads()
    flops, secs = 0, 0.0
    for i, l in enumerate(layers):
        x, w, b = conv_inputs(l.with_batch(1), seed + i, "bf16")
        kk = min(k, l.K)
        t0 = time.perf_counter()
        oracle.conv2d(x, w[:kk], b[:kk], l.stride, l.pad, l.dil, l.groups, threads=threads)
        secs += time.perf_counter() - t0
        flops += 2 * kk * (l.C // l.groups) * l.R * l.S * l.P * l.Q
    return flops, secs


def _oracle_calibrate(layers, seconds: float):
    """Smallest k (output channels per layer) whose sample takes >= `seconds`."""
    import oracle
    oracle.build()
    k = 1
    while True:
        _, dt = _oracle_run(layers, k)
        if dt >= seconds or k >= 64:
            return k
        k = min(64, max(k + 1, int(k * min(8.0, 1.2 * seconds / max(dt, 1e-3)))))


def _sample_desc(layers, k: int, flops: int, threads: int) -> str:
    return (f"1 image x first {k} output channel(s) of each of the {len(layers)} {WORKLOAD} layers "
            f"({flops / 1e9:.2f} GFLOP), fp64 oracle, {threads} threads")


def run_reference(args, rank: int, world: int):
    """Reference arm: the oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    layers = workload("vgg16", BATCH)
    per_step = max(0.5, min(2.0, 150.0 / max(1, args.steps + args.warmup)))
    k = _oracle_calibrate(layers, per_step)
    times, flops = [], 0
    for i in range(args.warmup + args.steps):
        flops, dt = _oracle_run(layers, k)
        if i >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    value = flops / mean / 1e12
    desc = _sample_desc(layers, k, flops, oracle.host_threads())
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
    def __init__(self, spec, algo: str, device, seed: int):
        import paper_2410_08300_b200 as ai3
        self.spec = spec
        _, w, b = conv_inputs(spec.with_batch(1), seed, "bf16")  # weights/bias: synth recipe
        g = torch.Generator(device=device).manual_seed(seed)
        self.x = torch.randn((spec.N, spec.C, spec.H, spec.W), generator=g, device=device, dtype=torch.float32) \
            .to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        wt = torch.from_numpy(w).to(device=device, dtype=torch.bfloat16)
        bt = None if b is None else torch.from_numpy(b).to(device=device, dtype=torch.bfloat16)
        if algo == "benchmark":  # measure every algorithm once for this layer; the plan takes the winner
            ai3.autotune(self.x, wt, bt, spec.stride, spec.pad, spec.dil, spec.groups)
        self.plan = ai3.ConvPlan(wt, bt, self.x.shape, spec.stride, spec.pad, spec.dil, spec.groups, algo,
                                 in_layout=1, out_layout=1)
        self.y = torch.empty(self.plan.out_shape, dtype=torch.bfloat16, device=device,
                             memory_format=torch.channels_last)
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
    total_ms, layer_ms = _time_stack(layers, args.steps, stream, per_layer=True)
    torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms_per_step = total_ms / args.steps
    if dist:
        t = torch.tensor([ms_per_step], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_per_step = float(t.item())
    value = world * step_flops / (ms_per_step * 1e-3) / 1e12
    images_per_s = world * BATCH / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel: tcgen05 implicit GEMM on the tensor-bound layers
    burst, sustained, hbm, peak_src = _peaks()
    tc_idx = [i for i, l in enumerate(layers) if l.spec.C >= 64]
    tc_flops = sum(layers[i].flops for i in tc_idx)
    tc_ms = sum(layer_ms[i] for i in tc_idx)
    achieved = tc_flops / (tc_ms * 1e-3) / 1e12
    traffic = _traffic()
    roofline = {"bound": "tensor", "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                "frac": achieved / sustained, "peak_kind": f"bf16 sustained ({peak_src}); burst {burst}",
                "frac_of_burst": achieved / burst,
                "kernel": "tc_gemm_kernel (implicit GEMM, 12 tensor-bound VGG layers, 1 launch each)",
                "launches_per_step": len(tc_idx),
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
        import paper_2410_08300_b200 as ai3
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
        e2e_ms = s.elapsed_time(e) / e2e_steps
        if dist:
            t = torch.tensor([e2e_ms], device=device, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = sum(x.numel() * x.element_size() for x in hx)
        d2h = sum(y.numel() * y.element_size() for y in hy)
        e2e = {"value": world * step_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "ai3_conv2d_plans_execute_host over the 13 layers (H2D / conv / D2H of consecutive layers "
                       "overlapped on copy streams), pinned host memory"}
        del hx, hy

    # ---- the other BASELINE conv configs (ResNet-50 N=256, AlexNet N=128; bf16 NHWC, `guess`):
    #      every unique layer shape timed once per rep, weighted by its count in the network
    configs = None
    if not args.no_configs and rank == 0:
        configs = {}
        for net, nb in (("resnet50", 256), ("alexnet", 128)):
            try:
                tot_ms, tot_flops, algos, launches, rows = 0.0, 0, {}, 0, []
                for i, spec in enumerate(workload(net, nb)):
                    lay = Layer(spec, args.algo, device, seed=3000 + i)
                    for _ in range(2):
                        lay.run(stream.cuda_stream)
                    reps = 10
                    s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s1.record(stream)
                    for _ in range(reps):
                        lay.run(stream.cuda_stream)
                    e1.record(stream)
                    e1.synchronize()
                    ms = s1.elapsed_time(e1) / reps
                    tot_ms += spec.count * ms
                    tot_flops += spec.count * spec.flops()
                    launches += spec.count * lay.plan.num_launches
                    algos[lay.plan.algorithm] = algos.get(lay.plan.algorithm, 0) + spec.count
                    rows.append([spec.name, spec.count, round(ms * 1e3, 1), round(spec.flops() / (ms * 1e-3) / 1e12, 1),
                                 lay.plan.algorithm])
                    del lay
                configs[net] = {"batch": nb, "convs": sum(sp.count for sp in workload(net, nb)),
                                "ms_all_convs": round(tot_ms, 4), "tflops": round(tot_flops / (tot_ms * 1e-3) / 1e12, 1),
                                "images_per_s": round(nb / (tot_ms * 1e-3), 1), "algorithms": algos,
                                "launches": launches, "layers_us_tflops": rows}
                torch.cuda.empty_cache()
            except Exception as ex:  # report, do not hide
                configs[net] = {"error": str(ex)}

    # ---- the whole model: swap_backend(VGG-16), every op in ai3 (BASELINE configs[4]'s model
    #      at this rank's batch), timed the same way; reported beside the conv-stack metric
    model_leg = None
    if not args.no_model:
        from paper_2410_08300_b200.runner import build_vgg16, make_images
        try:
            model = build_vgg16(device, algo=args.algo, seed=0, swap="backend")
            xm = make_images(0, BATCH, 5001, device)
            with torch.inference_mode():
                for _ in range(3):
                    model(xm)
                torch.cuda.synchronize(device)
                s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = max(3, min(args.steps, 20))
                s0.record(stream)
                for _ in range(reps):
                    model(xm)
                e0.record(stream)
                e0.synchronize()
            mms = s0.elapsed_time(e0) / reps
            model_leg = {"model": "vgg16 (torchvision, random init), swap_backend: all ops in ai3", "batch": BATCH,
                         "ms_per_forward": mms, "images_per_s": BATCH / (mms * 1e-3),
                         "ops_kept_in_torch": len(model.kept)}
            del model, xm
            torch.cuda.empty_cache()
        except Exception as ex:  # report, do not hide
            model_leg = {"error": str(ex)}

    # ---- per-algorithm comparison on the same stack (config: Winograd vs implicit GEMM vs direct)
    per_algo, selector = None, None
    if not args.no_compare and rank == 0:
        per_algo = {}
        layer_times = {}  # per-layer ms of every algorithm on the same stack, timed the same way
        for algo in ("implicit_gemm", "implicit_precomp_gemm", "winograd", "gemm", "kn2row", "direct", "smm",
                     "guess", "benchmark"):
            try:
                alt = [Layer(s, algo, device, seed=1000 * 2 + i) for i, s in enumerate(specs)]
                _time_stack(alt, 1, stream, per_layer=False)
                reps = 3 if algo not in ("direct", "smm") else 1
                ms, lms = _time_stack(alt, reps, stream, per_layer=True)
                per_algo[algo] = round(step_flops / (ms / reps * 1e-3) / 1e12, 1)
                layer_times[algo] = lms
                del alt
                torch.cuda.empty_cache()
            except Exception as ex:  # report, do not hide
                per_algo[algo] = f"error: {ex}"
        # selector quality: sum of the chosen algorithms' times over the sum
        # of the per-layer best among the fixed algorithms (1.0 = never picks a slower one)
        fixed = [a for a in layer_times if a not in ("guess", "benchmark")]
        if fixed:
            best = [min(layer_times[a][i] for a in fixed) for i in range(len(specs))]
            best_alg = [min(fixed, key=lambda a: layer_times[a][i]) for i in range(len(specs))]
            selector = {"best_per_layer": dict(zip([l.spec.name for l in layers], best_alg))}
            for sel in ("guess", "benchmark"):
                if sel in layer_times:
                    selector[f"{sel}_regret"] = round(sum(layer_times[sel]) / sum(best), 4)

    # ---- oracle on host cores (rank 0, N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        import oracle
        k = _oracle_calibrate(specs, args.cpu_seconds)
        flops, dt = _oracle_run(specs, k)
        cpu = {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.host_threads(), "kind": "oracle",
               "sample": _sample_desc(specs, k, flops, oracle.host_threads()), "seconds": round(dt, 2)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": WORKLOAD, "batch_per_gpu": BATCH, "global_batch": BATCH * world,
                           "image": 224, "layers": len(layers), "layout": "NHWC", "algorithm": args.algo,
                           "parallelism": f"dp{world} (batch-sharded, no collective in the step)",
                           "l2": "step working set ~2.9 GB of distinct per-layer buffers >> 126 MB L2; no flush"},
                "images_per_s": images_per_s, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks, "per_layer": per_layer,
                "per_algorithm_tflops": per_algo, "selector_quality": selector, "vgg16_model": model_leg,
                "other_configs": configs}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="guess")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-model", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
