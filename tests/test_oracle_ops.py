"""Pins of oracle/ops.py (the fp64 definitions of ReLU, pooling, linear, flatten;
PAPER.md:80) against things other than itself: hand-worked values, closed forms,
identities with the independently written conv oracle, and torch.nn.functional in
float64 (the paper's own comparator).  CPU only."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from oracle import ops


def test_relu_hand_values():
    x = np.array([-2.0, -0.0, 0.0, 1.5, np.nan, -np.inf, np.inf])
    y = ops.relu(x)
    assert y[0] == 0 and y[3] == 1.5 and np.isnan(y[4]) and y[5] == 0 and y[6] == np.inf


def test_maxpool_hand_values():
    x = np.arange(16, dtype=np.float64).reshape(1, 1, 4, 4)
    np.testing.assert_array_equal(ops.max_pool2d(x, 2)[0, 0], [[5, 7], [13, 15]])
    # 3x3 stride 2 pad 1 over arange(16): windows clipped to the input
    np.testing.assert_array_equal(ops.max_pool2d(x, 3, 2, 1)[0, 0], [[5, 7], [13, 15]])


def test_maxpool_padding_never_wins():
    x = -np.ones((1, 2, 3, 3)) - np.arange(9).reshape(1, 1, 3, 3)
    y = ops.max_pool2d(x, 3, 1, 1)
    assert (y < 0).all()  # a zero from padding would win otherwise
    assert y[0, 0, 0, 0] == -1.0


def test_maxpool_identity_and_dilation():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 7, 6))
    np.testing.assert_array_equal(ops.max_pool2d(x, 1, 1), x)
    # dilation 2, kernel 2 = max of x[h], x[h+2]
    y = ops.max_pool2d(x, 2, 1, 0, 2)
    np.testing.assert_array_equal(y, np.maximum(np.maximum(x[:, :, :-2, :-2], x[:, :, 2:, :-2]),
                                                np.maximum(x[:, :, :-2, 2:], x[:, :, 2:, 2:])))


def test_maxpool_nan_propagates():
    x = np.zeros((1, 1, 2, 2))
    x[0, 0, 1, 0] = np.nan
    assert np.isnan(ops.max_pool2d(x, 2)[0, 0, 0, 0])


def test_pool_output_lengths():
    assert ops.pool_out_len(112, 2, 2, 0) == 56
    assert ops.pool_out_len(5, 2, 2, 0, ceil_mode=True) == 3
    assert ops.pool_out_len(5, 2, 2, 0) == 2
    assert ops.pool_out_len(6, 3, 2, 1, ceil_mode=True) == 4
    assert ops.pool_out_len(5, 2, 2, 1, ceil_mode=True) == 3   # a 4th window would start in the right padding
    with pytest.raises(ValueError):
        ops.pool_out_len(8, 2, 2, 2)


def test_avgpool_closed_forms():
    ones = np.ones((1, 1, 4, 4))
    np.testing.assert_array_equal(ops.avg_pool2d(ones, 2), np.ones((1, 1, 2, 2)))
    y = ops.avg_pool2d(ones, 2, 2, 1, count_include_pad=True)
    assert y[0, 0, 0, 0] == 0.25 and y[0, 0, 1, 1] == 1.0
    y = ops.avg_pool2d(ones, 2, 2, 1, count_include_pad=False)
    np.testing.assert_array_equal(y, np.ones_like(y))
    x = np.arange(16, dtype=np.float64).reshape(1, 1, 4, 4)
    np.testing.assert_array_equal(ops.avg_pool2d(x, 2)[0, 0], [[2.5, 4.5], [10.5, 12.5]])
    np.testing.assert_array_equal(ops.avg_pool2d(x, 2, divisor_override=1)[0, 0], [[10, 18], [42, 50]])


def test_adaptive_avg_identities():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 3, 12, 8))
    np.testing.assert_allclose(ops.adaptive_avg_pool2d(x, 1)[:, :, 0, 0], x.mean(axis=(2, 3)), rtol=1e-14)
    np.testing.assert_allclose(ops.adaptive_avg_pool2d(x, (6, 4)), ops.avg_pool2d(x, 2), rtol=1e-14)
    np.testing.assert_array_equal(ops.adaptive_avg_pool2d(x, (12, 8)), x)
    # 7 -> 3: bins [0,3), [2,5), [4,7)
    v = np.arange(7, dtype=np.float64).reshape(1, 1, 1, 7)
    np.testing.assert_allclose(ops.adaptive_avg_pool2d(v, (1, 3))[0, 0, 0], [1.0, 3.0, 5.0])


def test_linear_is_a_1x1_conv():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((5, 24))
    w = rng.standard_normal((7, 24))
    b = rng.standard_normal(7)
    conv = oracle.conv2d(x[:, :, None, None], w[:, :, None, None], b)[:, :, 0, 0]
    np.testing.assert_allclose(ops.linear(x, w, b), conv, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(ops.linear([[1.0, 2.0]], [[3.0, 4.0], [-1.0, 1.0]], [0.5, 0.0]), [[11.5, 1.0]])


def test_flatten_order():
    x = np.arange(24, dtype=np.float64).reshape(2, 3, 2, 2)
    np.testing.assert_array_equal(ops.flatten(x)[1], np.arange(12, 24))


@pytest.mark.parametrize("case", range(12))
def test_pools_match_torch_float64(case):
    rng = np.random.default_rng(100 + case)
    N, C = int(rng.integers(1, 3)), int(rng.integers(1, 5))
    H, W = int(rng.integers(3, 15)), int(rng.integers(3, 15))
    k = int(rng.integers(1, 4)); s = int(rng.integers(1, 4)); p = int(rng.integers(0, k // 2 + 1))
    d = int(rng.integers(1, 3)); cm = bool(rng.integers(0, 2)); cip = bool(rng.integers(0, 2))
    x = rng.standard_normal((N, C, H, W))
    xt = torch.from_numpy(x)
    if H + 2 * p >= d * (k - 1) + 1 and W + 2 * p >= d * (k - 1) + 1:
        np.testing.assert_array_equal(ops.max_pool2d(x, k, s, p, d, cm),
                                      F.max_pool2d(xt, k, s, p, d, ceil_mode=cm).numpy())
    np.testing.assert_allclose(ops.avg_pool2d(x, k, s, p, cm, cip),
                               F.avg_pool2d(xt, k, s, p, cm, cip).numpy(), rtol=1e-13, atol=1e-15)
    o = (int(rng.integers(1, H + 1)), int(rng.integers(1, W + 1)))
    np.testing.assert_allclose(ops.adaptive_avg_pool2d(x, o), F.adaptive_avg_pool2d(xt, o).numpy(), rtol=1e-13,
                               atol=1e-15)
