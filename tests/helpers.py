"""Shared helpers for the parity tests: run one conv through the C ABI (via the
Python binding) and through the CPU oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from synth import ConvShape, conv_inputs

# north_star tolerances on max|err| / max|ref|
TOL = {("f32", "strict"): 1e-5, ("f32", "tf32"): 1e-3, ("bf16", "strict"): 2e-2, ("bf16", "tf32"): 2e-2}
WINOGRAD_F32_TOL = 1e-3


def stable_seed(key) -> int:
    """A 16-bit seed from a case key that is the same in every process (hash() of a str is salted)."""
    import zlib
    return zlib.crc32(repr(key).encode()) & 0xFFFF


def tolerance(algo: str, dtype: str, math: str) -> float:
    if dtype == "f32" and algo == "winograd":
        return WINOGRAD_F32_TOL
    return TOL[(dtype, math)]


def torch_dtype(dtype: str):
    return torch.bfloat16 if dtype == "bf16" else torch.float32


def to_device(x: np.ndarray, dtype: str, layout: str = "nchw", device="cuda"):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device=device, dtype=torch_dtype(dtype))
    if layout == "nhwc":
        t = t.contiguous(memory_format=torch.channels_last)
    return t


def run_ai3(shape: ConvShape, x, w, b, algo: str, dtype: str, math: str = "strict", layout: str = "nchw",
            plan: bool = True):
    """y (fp64 numpy, NCHW) from the GPU path for host arrays x, w, b."""
    import paper_2410_08300_b200 as ai3
    xt = to_device(x, dtype, layout)
    wt = to_device(w, dtype)
    bt = None if b is None else to_device(b, dtype)
    # the output starts as NaN: an element a kernel fails to write fails the comparison
    # instead of passing on a stale value of an earlier run that reused the same memory
    fmt = torch.channels_last if layout == "nhwc" else torch.contiguous_format
    y = torch.full((shape.N, shape.K, shape.P, shape.Q), float("nan"), dtype=xt.dtype, device=xt.device) \
        .contiguous(memory_format=fmt)
    if plan:
        p = ai3.ConvPlan(wt, bt, xt.shape, shape.stride, shape.pad, shape.dil, shape.groups, algo, math,
                         in_layout=1 if layout == "nhwc" else 0)
        p(xt, out=y)
    else:
        ai3.conv2d(xt, wt, bt, shape.stride, shape.pad, shape.dil, shape.groups, algo, math, out=y)
    torch.cuda.synchronize()
    return y.float().contiguous().cpu().numpy().astype(np.float64)


def ref(shape: ConvShape, x, w, b):
    return oracle.conv2d(x, w, b, shape.stride, shape.pad, shape.dil, shape.groups)


def inputs(shape: ConvShape, seed: int, dtype: str):
    return conv_inputs(shape, seed, dtype)
