"""DESIGN.md R24 on the CPU: the space-to-depth lowering that `implicit_gemm` uses for strided,
few-channel convs is an exact rewrite of the definition (PAPER.md:56 / SPEC.md:130 sum).

The rewrite is written out here in numpy, independently of the CUDA code (which implements
it in prep.cu / api.cu): build the s2d image anchored at the padded origin and the s2d
filter, run the oracle's stride-1, unpadded conv on them, and compare with the oracle's
strided conv.  Integer inputs make every sum exact, so the comparison is bit-exact.
"""
import numpy as np
import pytest

import oracle
from synth import ConvShape, integer_inputs


def s2d_lowering(x, w, stride, pad):
    """x (N,C,H,W), w (K,C,R,S) -> (x', w') of the stride-1 conv (R24)."""
    (sh, sw), (ph, pw) = stride, pad
    N, C, H, W = x.shape
    K, _, R, S = w.shape
    P = (H + 2 * ph - R) // sh + 1
    Q = (W + 2 * pw - S) // sw + 1
    Th, Tw = -(-R // sh), -(-S // sw)
    H2, W2 = P + Th - 1, Q + Tw - 1
    xs = np.zeros((N, sh * sw * C, H2, W2))
    for j in range(H2):
        for l in range(W2):
            for i in range(sh):
                for u in range(sw):
                    h, ww = j * sh - ph + i, l * sw - pw + u
                    if 0 <= h < H and 0 <= ww < W:
                        xs[:, (i * sw + u) * C:(i * sw + u + 1) * C, j, l] = x[:, :, h, ww]
    ws = np.zeros((K, sh * sw * C, Th, Tw))
    for a in range(Th):
        for b in range(Tw):
            for i in range(sh):
                for u in range(sw):
                    r, s = a * sh + i, b * sw + u
                    if r < R and s < S:
                        ws[:, (i * sw + u) * C:(i * sw + u + 1) * C, a, b] = w[:, :, r, s]
    return xs, ws


CASES = [  # (N, C, H, W, K, R, S, stride, pad)
    (2, 3, 29, 27, 8, 7, 7, (2, 2), (3, 3)),    # ResNet stem shape
    (1, 3, 35, 35, 6, 11, 11, (4, 4), (2, 2)),  # AlexNet conv1 shape
    (2, 2, 17, 19, 5, 5, 3, (2, 1), (2, 1)),    # asymmetric stride
    (1, 4, 16, 16, 3, 4, 4, (2, 2), (0, 0)),    # kernel a stride multiple, no padding
    (2, 1, 23, 21, 4, 8, 8, (4, 4), (3, 5)),    # padding larger than the stride
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[5]}x{c[6]}s{c[7][0]}{c[7][1]}p{c[8][0]}{c[8][1]}")
def test_s2d_lowering_is_exact(case):
    N, C, H, W, K, R, S, st, pd = case
    shape = ConvShape("s2d", N, C, H, W, K, R, S)
    x, w, b = integer_inputs(shape, seed=11, xmax=5, wmax=3)
    xs, ws = s2d_lowering(x, w, st, pd)
    y_ref = oracle.conv2d(x, w, b, st, pd, 1, 1)
    y_s2d = oracle.conv2d(xs, ws, b, 1, 0, 1, 1)
    assert y_s2d.shape == y_ref.shape
    np.testing.assert_array_equal(y_s2d, y_ref)
