"""Batch-sharded multi-GPU inference runner (BASELINE.json configs[4]).

    torchrun --nproc-per-node G --master-addr 127.0.0.1 -m paper_2410_08300_b200.runner \
        --global-batch 2048 --algo guess

One process per GPU.  The global batch of N images is split into G contiguous
slabs; rank r runs images [r*N/G, (r+1)*N/G) through VGG-16 whose 13 convolutions
are swapped to ai3 (swap_conv2d), with NHWC bf16 activations.
There is no communication inside the forward: images are independent, and ai3's
kernels reduce each output element in an order that does not depend on the batch
size, so the sharded result is bit-identical to the single-GPU one (pinned by
tests/test_parity_gpu.py::test_deterministic_and_batch_independent).  After the
timed forward, one NCCL all_gather_into_tensor collects the logits on every rank
for checking only; it is timed separately and excluded from images/s (north_star).

Timing: barrier -> CUDA events around the forward on each rank -> all_reduce(MAX)
-> images/s = N / t_max.

By default the model is swap_backend's all-ai3 model (SURVEY §8 row
f1): conv + ReLU fused, ai3 max-pool, flatten fused into the first linear, linear
layers on the tcgen05 engine.  --swap conv2d swaps only the convolutions
and --swap none runs PyTorch, for comparison.
"""
from __future__ import annotations

import argparse
import json
import os
import time

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slab [lo, hi) of n images for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def make_images(lo: int, hi: int, seed: int, device, dtype=torch.bfloat16, size: int = 224) -> torch.Tensor:
    """Images lo..hi-1 of the seeded synthetic global batch, generated per image so any
    rank can materialise exactly its own slab: image i ~ N(0,1) from Generator(seed + i)."""
    out = torch.empty((hi - lo, 3, size, size), device=device, dtype=torch.float32)
    g = torch.Generator(device=device)
    for i in range(lo, hi):
        g.manual_seed(seed + i)
        out[i - lo].normal_(generator=g)
    return out.to(dtype).contiguous(memory_format=torch.channels_last)


def build_vgg16(device, dtype=torch.bfloat16, algo="guess", seed: int = 0, swap: str = "backend"):
    """torchvision VGG-16 with random-init weights (no network for pretrained ones), identical
    on every rank (same seed).  swap="backend": swap_backend, every op in ai3;
    "conv2d": swap_conv2d, only the convolutions; "none": PyTorch."""
    import torchvision
    torch.manual_seed(seed)
    model = torchvision.models.vgg16(weights=None).eval()
    model = model.to(device=device, dtype=dtype).to(memory_format=torch.channels_last)
    if swap == "backend":
        from .hooks import swap_backend
        return swap_backend(model, {"conv2d": algo})
    if swap == "conv2d":
        from .hooks import swap_conv2d
        swap_conv2d(model, algo)
    return model


def gather_rows(local: torch.Tensor, world: int, counts: list[int]) -> torch.Tensor:
    """all_gather_into_tensor of per-rank row blocks (padded to the max count) -> the
    concatenation in rank order, trimmed to the true counts."""
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, pad)  # one NCCL collective over NVLink / NVSwitch
    else:  # gloo (CPU tests): same semantics through the list form
        dist.all_gather(list(out.chunk(world, dim=0)), pad)
    return torch.cat([out[r * mx: r * mx + counts[r]] for r in range(world)], dim=0)


def max_over_ranks(value: float, device) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run(global_batch: int, algo: str, steps: int, warmup: int, seed: int, check: bool, swap: str = "backend",
        quiet: bool = False, finalize: bool = True, cuda_graph: bool = False):
    """Run BASELINE configs[4] on this rank's slab; returns the result dict (rank 0 prints it
    unless quiet).  finalize=False leaves the process group up (bench.py calls this inside
    its own run)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=device)
    lo, hi = shard_bounds(global_batch, world, rank)
    x = make_images(lo, hi, seed + 1, device)
    model = build_vgg16(device, algo=algo, seed=seed, swap=swap)
    if cuda_graph and swap == "backend":
        model.cuda_graph = True
    with torch.inference_mode():
        for _ in range(warmup):
            y = model(x)
        torch.cuda.synchronize(device)
        if world > 1:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            y = model(x)
        e.record()
        e.synchronize()
    ms = s.elapsed_time(e) / steps
    if world > 1:
        ms = max_over_ranks(ms, device)
    result = {"global_batch": global_batch, "n_gpus": world, "images_per_rank": hi - lo, "ms_per_forward": ms,
              "images_per_s": global_batch / (ms * 1e-3), "algo": algo, "swap": swap,
              "timing": "CUDA events around the forward on every rank, max over ranks; the all-gather is "
                        "timed separately and excluded"}
    if world > 1:
        counts = [shard_bounds(global_batch, world, r)[1] - shard_bounds(global_batch, world, r)[0]
                  for r in range(world)]
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        logits = gather_rows(y.float(), world, counts)
        torch.cuda.synchronize(device)
        result["gather_ms"] = (time.perf_counter() - t0) * 1e3
        result["gathered_rows"] = int(logits.shape[0])
    else:
        logits = y.float()
    if check:
        # sharding changes nothing: sampled images of this rank's slab run alone give the same
        # logits, bit for bit (every ai3 kernel reduces each output in an order that does not
        # depend on the batch; ReLU / pooling are per element).
        idx = sorted({lo, (lo + hi) // 2, hi - 1})
        ok, worst = True, 0.0
        with torch.inference_mode():
            for i in idx:
                xi = make_images(i, i + 1, seed + 1, device)
                yi = model(xi).float()
                ok &= bool(torch.equal(yi, logits[i:i + 1]))
                worst = max(worst, float((yi - logits[i:i + 1]).abs().max()))
        flags = torch.tensor([1.0 if ok else 0.0, worst], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(flags[:1], op=dist.ReduceOp.MIN)
            dist.all_reduce(flags[1:], op=dist.ReduceOp.MAX)
        result["logits_bit_identical_when_sharded"] = bool(flags[0].item() == 1.0)
        result["logits_max_abs_diff_vs_single_image"] = float(flags[1].item())
    if rank == 0 and not quiet:
        print(json.dumps(result), flush=True)
    if world > 1 and finalize:
        dist.destroy_process_group()
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--global-batch", type=int, default=2048)
    ap.add_argument("--algo", default="guess")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=5000)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--swap", default="backend", choices=["backend", "conv2d", "none"])
    a = ap.parse_args()
    run(a.global_batch, a.algo, a.steps, a.warmup, a.seed, not a.no_check, a.swap)


if __name__ == "__main__":
    main()
