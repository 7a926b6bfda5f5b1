"""Seeded synthetic inputs and workload shape tables, shared by tests, bench and smoke.

This module holds NONE of the method's arithmetic: it draws random numbers,
rounds them to the storage dtype (input quantisation, not convolution), and
lists layer shapes.  Both the oracle side and the CUDA side consume its output;
neither imports the other (see oracle/__init__.py).

Input recipe:
  * RNG: numpy Generator(PCG64(seed)).
  * x ~ N(0, 1)   -- the paper's inputs are torch.randn.
  * w, b ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in)), fan_in = (C/groups)*R*S --
    nn.Conv2d's default init, which the paper's random-init ConvNet uses
    (PAPER.md:111-121).
  * Generated in fp32; for bf16 runs rounded to bf16 (round-to-nearest-even)
    on the host, so the GPU and the oracle see identical values.
  * Dense, no sparsity.
"""
from __future__ import annotations

from dataclasses import dataclass, asdict

import numpy as np


# ---------------------------------------------------------------------------
# bf16 helpers (storage quantisation of inputs only)
# ---------------------------------------------------------------------------

def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 value (RNE), returned as fp32 holding bf16-exact values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    # NaN/Inf are not produced by the generators; keep them as-is anyway
    bad = ~np.isfinite(a)
    if bad.any():
        out = out.copy()
        out[bad] = a[bad]
    return out


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """bf16-exact fp32 values -> uint16 bit patterns (for building bf16 tensors)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


# ---------------------------------------------------------------------------
# Layer descriptions
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ConvShape:
    name: str
    N: int
    C: int
    H: int
    W: int
    K: int
    R: int
    S: int
    stride: int = 1
    pad: int = 0
    dil: int = 1
    groups: int = 1
    bias: bool = True
    count: int = 1  # occurrences in the network (ResNet-50 repeats shapes)

    @property
    def P(self) -> int:
        return (self.H + 2 * self.pad - self.dil * (self.R - 1) - 1) // self.stride + 1

    @property
    def Q(self) -> int:
        return (self.W + 2 * self.pad - self.dil * (self.S - 1) - 1) // self.stride + 1

    def flops(self) -> int:
        """Direct-count FLOPs 2*N*K*(C/g)*R*S*P*Q."""
        return 2 * self.N * self.K * (self.C // self.groups) * self.R * self.S * self.P * self.Q

    def alg_bytes(self, elem: int) -> int:
        """Minimum bytes any algorithm moves: x + w + y (+ fp32 bias).
        A 1x1 stride>1 conv only touches N*C*P*Q inputs."""
        if self.R == 1 and self.S == 1 and self.pad == 0:
            xin = self.N * self.C * self.P * self.Q
        else:
            xin = self.N * self.C * self.H * self.W
        return (xin + self.K * (self.C // self.groups) * self.R * self.S
                + self.N * self.K * self.P * self.Q) * elem + 4 * self.K

    def with_batch(self, n: int) -> "ConvShape":
        d = asdict(self)
        d["N"] = n
        return ConvShape(**d)


def _vgg16(N: int):
    spec = [("conv1_1", 3, 64, 224), ("conv1_2", 64, 64, 224),
            ("conv2_1", 64, 128, 112), ("conv2_2", 128, 128, 112),
            ("conv3_1", 128, 256, 56), ("conv3_2", 256, 256, 56), ("conv3_3", 256, 256, 56),
            ("conv4_1", 256, 512, 28), ("conv4_2", 512, 512, 28), ("conv4_3", 512, 512, 28),
            ("conv5_1", 512, 512, 14), ("conv5_2", 512, 512, 14), ("conv5_3", 512, 512, 14)]
    return [ConvShape(n, N, c, h, h, k, 3, 3, 1, 1) for (n, c, k, h) in spec]


def _resnet50(N: int):
    # 23 unique shapes of ResNet-50 v1.5 at 224x224, with counts (53 convs)
    rows = [(3, 224, 64, 7, 2, 3, 1), (64, 56, 64, 1, 1, 0, 1), (64, 56, 64, 3, 1, 1, 3),
            (64, 56, 256, 1, 1, 0, 4), (256, 56, 64, 1, 1, 0, 2), (256, 56, 128, 1, 1, 0, 1),
            (128, 56, 128, 3, 2, 1, 1), (128, 28, 512, 1, 1, 0, 4), (256, 56, 512, 1, 2, 0, 1),
            (512, 28, 128, 1, 1, 0, 3), (128, 28, 128, 3, 1, 1, 3), (512, 28, 256, 1, 1, 0, 1),
            (256, 28, 256, 3, 2, 1, 1), (256, 14, 1024, 1, 1, 0, 6), (512, 28, 1024, 1, 2, 0, 1),
            (1024, 14, 256, 1, 1, 0, 5), (256, 14, 256, 3, 1, 1, 5), (1024, 14, 512, 1, 1, 0, 1),
            (512, 14, 512, 3, 2, 1, 1), (512, 7, 2048, 1, 1, 0, 3), (1024, 14, 2048, 1, 2, 0, 1),
            (2048, 7, 512, 1, 1, 0, 2), (512, 7, 512, 3, 1, 1, 2)]
    out = []
    for i, (c, h, k, r, s, p, cnt) in enumerate(rows):
        out.append(ConvShape(f"rn50_{i:02d}_{c}x{h}_{k}_{r}x{r}s{s}", N, c, h, h, k, r, r, s, p,
                             bias=False, count=cnt))
    return out


def _alexnet(N: int):
    return [ConvShape("conv1", N, 3, 224, 224, 64, 11, 11, 4, 2),
            ConvShape("conv2", N, 64, 27, 27, 192, 5, 5, 1, 2),
            ConvShape("conv3", N, 192, 13, 13, 384, 3, 3, 1, 1),
            ConvShape("conv4", N, 384, 13, 13, 256, 3, 3, 1, 1),
            ConvShape("conv5", N, 256, 13, 13, 256, 3, 3, 1, 1)]


CONFIG1 = ConvShape("config1", 1, 3, 32, 32, 16, 3, 3, 1, 1)


def workload(name: str, batch: int | None = None):
    """Layer list for a BASELINE.json config: 'config1', 'vgg16', 'resnet50', 'alexnet'."""
    if name == "config1":
        return [CONFIG1 if batch is None else CONFIG1.with_batch(batch)]
    if name == "vgg16":
        return _vgg16(64 if batch is None else batch)
    if name == "resnet50":
        return _resnet50(256 if batch is None else batch)
    if name == "alexnet":
        return _alexnet(128 if batch is None else batch)
    raise KeyError(name)


# ---------------------------------------------------------------------------
# Generators
# ---------------------------------------------------------------------------

def conv_inputs(shape: ConvShape, seed: int, dtype: str = "f32", bias: bool | None = None):
    """(x, w, b) as float32 numpy arrays holding values exact in `dtype` ('f32'|'bf16').

    x: (N,C,H,W), w: (K,C/g,R,S), b: (K,) or None.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    s = shape
    fan_in = (s.C // s.groups) * s.R * s.S
    bound = 1.0 / np.sqrt(fan_in)
    x = rng.standard_normal((s.N, s.C, s.H, s.W), dtype=np.float32)
    w = rng.uniform(-bound, bound, size=(s.K, s.C // s.groups, s.R, s.S)).astype(np.float32)
    use_bias = s.bias if bias is None else bias
    b = rng.uniform(-bound, bound, size=(s.K,)).astype(np.float32) if use_bias else None
    if dtype == "bf16":
        x, w = round_to_bf16(x), round_to_bf16(w)
        if b is not None:
            b = round_to_bf16(b)
    elif dtype != "f32":
        raise ValueError(dtype)
    return x, w, b


def integer_inputs(shape: ConvShape, seed: int, xmax: int = 8, wmax: int = 4, bias: bool = True):
    """Small-integer x in [-xmax, xmax], w in [-wmax, wmax], b in [-wmax, wmax]:
    every partial sum is an integer well below 2^24, so any exact-product,
    fp32-accumulating path must reproduce the fp64 result bit for bit."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = shape
    x = rng.integers(-xmax, xmax + 1, size=(s.N, s.C, s.H, s.W)).astype(np.float32)
    w = rng.integers(-wmax, wmax + 1, size=(s.K, s.C // s.groups, s.R, s.S)).astype(np.float32)
    b = rng.integers(-wmax, wmax + 1, size=(s.K,)).astype(np.float32) if bias else None
    return x, w, b


def sample_indices(n_out: tuple, count: int, seed: int) -> np.ndarray:
    """`count` random (n,k,p,q) output coordinates, always including the corners."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N, K, P, Q = n_out
    idx = np.stack([rng.integers(0, N, count), rng.integers(0, K, count),
                    rng.integers(0, P, count), rng.integers(0, Q, count)], axis=1)
    corners = np.array([[0, 0, 0, 0], [N - 1, K - 1, P - 1, Q - 1],
                        [0, K - 1, 0, Q - 1], [N - 1, 0, P - 1, 0]], dtype=np.int64)
    return np.concatenate([corners, idx.astype(np.int64)], axis=0)
