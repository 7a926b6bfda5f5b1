"""CPU fp64 oracle for the non-convolution operations of an all-ai3 model -- TEST
INFRASTRUCTURE ONLY (same import rule as the package: tests/, smoke(), bench.py's
baseline legs).

PAPER.md:80: "ai3 currently supports the following operations, linear, convolution,
flatten, ReLU, and adaptive average, max, and average pooling".  The paper states no
formulas for them; its correctness check is equality with the PyTorch model
(PAPER.md:138-139, :163), so each function below writes out PyTorch's documented
definition (reading R18), plainly, in float64:

* relu(x)              = x if x >= 0 else 0; NaN stays NaN.
* max_pool2d           : out size floor_or_ceil((L + 2p - d(k-1) - 1)/s) + 1, with the
                         ceil_mode rule that the last window starts inside input + left
                         padding; max over the taps that fall inside the input.
* avg_pool2d           : sum over taps inside the input, divided by divisor_override, or
                         by the window clipped to the padded input (count_include_pad), or
                         by the window clipped to the input.
* adaptive_avg_pool2d  : output i averages rows floor(i*L/O) .. ceil((i+1)*L/O)-1.
* linear(x, w, b)      = x @ w.T + b  (a library matmul as one step).
* flatten(x)           = x.reshape(N, -1) in logical (C, H, W) order.

Pins: tests/test_oracle_ops.py (hand-worked values, closed forms, identities against
the conv oracle, and torch.nn.functional in float64).
"""
from __future__ import annotations

import math

import numpy as np


def relu(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(x < 0, 0.0, x)


def _pair(v):
    return (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))


def pool_out_len(L: int, k: int, s: int, p: int, d: int = 1, ceil_mode: bool = False) -> int:
    if p * 2 > k:
        raise ValueError("padding must be at most half the kernel size")
    span = L + 2 * p - d * (k - 1) - 1
    if span < 0:
        raise ValueError("window larger than the padded input")
    o = (math.ceil(span / s) if ceil_mode else span // s) + 1
    if ceil_mode and (o - 1) * s >= L + p:
        o -= 1
    return o


def max_pool2d(x, kernel, stride=None, padding=0, dilation=1, ceil_mode=False):
    x = np.asarray(x, dtype=np.float64)
    N, C, H, W = x.shape
    kh, kw = _pair(kernel)
    sh, sw = _pair(stride if stride is not None else kernel)
    ph, pw = _pair(padding)
    dh, dw = _pair(dilation)
    P = pool_out_len(H, kh, sh, ph, dh, ceil_mode)
    Q = pool_out_len(W, kw, sw, pw, dw, ceil_mode)
    y = np.empty((N, C, P, Q))
    for p in range(P):
        for q in range(Q):
            best = np.full((N, C), -np.inf)
            for a in range(kh):
                h = p * sh - ph + a * dh
                if not 0 <= h < H:
                    continue
                for b in range(kw):
                    w = q * sw - pw + b * dw
                    if not 0 <= w < W:
                        continue
                    v = x[:, :, h, w]
                    best = np.where((v > best) | np.isnan(v), v, best)
            y[:, :, p, q] = best
    return y


def avg_pool2d(x, kernel, stride=None, padding=0, ceil_mode=False, count_include_pad=True, divisor_override=None):
    x = np.asarray(x, dtype=np.float64)
    N, C, H, W = x.shape
    kh, kw = _pair(kernel)
    sh, sw = _pair(stride if stride is not None else kernel)
    ph, pw = _pair(padding)
    P = pool_out_len(H, kh, sh, ph, 1, ceil_mode)
    Q = pool_out_len(W, kw, sw, pw, 1, ceil_mode)
    y = np.empty((N, C, P, Q))
    for p in range(P):
        for q in range(Q):
            h0, w0 = p * sh - ph, q * sw - pw
            h1, w1 = min(h0 + kh, H + ph), min(w0 + kw, W + pw)
            padded_count = (h1 - h0) * (w1 - w0)
            hs, ws, he, we = max(h0, 0), max(w0, 0), min(h1, H), min(w1, W)
            total = np.zeros((N, C))
            for h in range(hs, he):
                for w in range(ws, we):
                    total += x[:, :, h, w]
            if divisor_override:
                div = divisor_override
            elif count_include_pad:
                div = padded_count
            else:
                div = (he - hs) * (we - ws)
            y[:, :, p, q] = total / div
    return y


def adaptive_avg_pool2d(x, out_hw):
    x = np.asarray(x, dtype=np.float64)
    N, C, H, W = x.shape
    P, Q = _pair(out_hw)
    y = np.empty((N, C, P, Q))
    for p in range(P):
        hs, he = (p * H) // P, -((-(p + 1) * H) // P)
        for q in range(Q):
            ws, we = (q * W) // Q, -((-(q + 1) * W) // Q)
            y[:, :, p, q] = x[:, :, hs:he, ws:we].sum(axis=(2, 3)) / ((he - hs) * (we - ws))
    return y


def linear(x, w, b=None):
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    y = x @ w.T
    if b is not None:
        y = y + np.asarray(b, dtype=np.float64)[None, :]
    return y


def flatten(x):
    x = np.asarray(x, dtype=np.float64)
    return x.reshape(x.shape[0], -1)
