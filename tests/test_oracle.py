"""Pins for the CPU fp64 oracle (SURVEY §8c "What pins each part").

Each test checks the oracle against something other than itself: values the
spec/paper print (tests/golden/), closed forms, invariants, textbook routines
(matmul), an independently structured formulation (shift-and-accumulate,
the SMM formulation of PAPER.md:55), and torch.nn.functional.conv2d in fp64
(the paper's own comparator).  A dropped bias, a sign error, a
wrong index or a transposed operand fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest

from helpers import stable_seed

import oracle
from synth import ConvShape, conv_inputs, integer_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


# ---------------------------------------------------------------- printed values

@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: c["id"])
def test_spec_worked_examples(case):
    y = oracle.conv2d(case["x"], case["w"], case["b"], case["stride"], case["padding"],
                      case["dilation"], case["groups"])
    if "y" in case:
        np.testing.assert_array_equal(y, np.asarray(case["y"], dtype=np.float64))
    else:
        np.testing.assert_array_equal(y[0, :, 0, 0], np.asarray(case["y_at_00"], dtype=np.float64))


@pytest.mark.parametrize("case", _golden()["shapes"], ids=lambda c: c["cite"][:12])
def test_spec_output_shapes(case):
    P, Q = oracle.output_shape(case["in"][2:], case["kernel"], case["stride"], case["padding"],
                               case["dilation"])
    assert [case["in"][0], case["K"], P, Q] == case["out"]


def test_shape_errors():
    # kernel larger than padded input
    with pytest.raises(oracle.OracleError):
        oracle.output_shape((2, 2), (3, 3), 1, 0, 1)
    # channel mismatch
    with pytest.raises(oracle.OracleError):
        oracle.conv2d(np.zeros((1, 3, 4, 4)), np.zeros((2, 2, 3, 3)))
    # groups must divide C and K
    with pytest.raises(oracle.OracleError):
        oracle.conv2d(np.zeros((1, 4, 4, 4)), np.zeros((3, 2, 3, 3)), groups=2)


# ---------------------------------------------------------------- textbook reductions

def _triple_loop_matmul(A, B):
    M, Kd = A.shape
    Kd2, N = B.shape
    assert Kd == Kd2
    C = np.zeros((M, N))
    for i in range(M):
        for j in range(N):
            s = 0.0
            for t in range(Kd):
                s += A[i, t] * B[t, j]
            C[i, j] = s
    return C


def test_1x1_conv_equals_matmul():
    """SPEC.md:144 / S:62: a 1x1 conv is a channel matmul y[n,:,p,q] = W[KxC] x[n,:,p,q]."""
    rng = np.random.default_rng(1)
    N, C, H, W, K = 2, 5, 3, 4, 7  # K != C so a transposed W fails
    x = rng.standard_normal((N, C, H, W))
    w = rng.standard_normal((K, C, 1, 1))
    b = rng.standard_normal(K)
    y = oracle.conv2d(x, w, b)
    for n in range(N):
        X = x[n].reshape(C, H * W)
        ref = _triple_loop_matmul(w[:, :, 0, 0], X) + b[:, None]
        np.testing.assert_allclose(y[n].reshape(K, H * W), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("r0,s0,stride,pad,dil", [(0, 0, 1, 0, 1), (1, 2, 1, 1, 1), (2, 0, 2, 2, 1),
                                                  (1, 1, 3, 1, 2), (0, 2, 2, 0, 2), (2, 2, 1, 2, 2)])
def test_delta_kernels_closed_form(r0, s0, stride, pad, dil):
    """w = delta(k=c) delta(r=r0) delta(s=s0) -> y[n,k,p,q] = x[n,k,p*s-p+r0*d, q*s-p+s0*d] or 0."""
    rng = np.random.default_rng(2)
    N, C, H, W, R, S = 2, 3, 9, 8, 3, 3
    x = rng.standard_normal((N, C, H, W))
    w = np.zeros((C, C, R, S))
    for c in range(C):
        w[c, c, r0, s0] = 1.0
    y = oracle.conv2d(x, w, None, stride, pad, dil)
    P, Q = y.shape[2:]
    ref = np.zeros_like(y)
    for p in range(P):
        ih = p * stride - pad + r0 * dil
        for q in range(Q):
            iw = q * stride - pad + s0 * dil
            if 0 <= ih < H and 0 <= iw < W:
                ref[:, :, p, q] = x[:, :, ih, iw]
    np.testing.assert_array_equal(y, ref)


# ---------------------------------------------------------------- invariants / identities

def test_linearity_in_x_and_w():
    """conv is bilinear (bias-free)."""
    rng = np.random.default_rng(3)
    x1, x2 = rng.standard_normal((2, 2, 3, 7, 6))
    w1, w2 = rng.standard_normal((2, 4, 3, 3, 2))
    a, b = 0.75, -1.5
    lhs = oracle.conv2d(a * x1 + b * x2, w1, None, 2, 1, 1)
    rhs = a * oracle.conv2d(x1, w1, None, 2, 1, 1) + b * oracle.conv2d(x2, w1, None, 2, 1, 1)
    np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-12)
    lhs = oracle.conv2d(x1, a * w1 + b * w2, None, 1, 2, 2)
    rhs = a * oracle.conv2d(x1, w1, None, 1, 2, 2) + b * oracle.conv2d(x1, w2, None, 1, 2, 2)
    np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-12)


def test_padding_identity():
    """SPEC.md:44-52 zero_pad_2d: conv(x, pad p) == conv(zero_pad(x, p), pad 0)."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 3, 6, 5))
    w = rng.standard_normal((4, 3, 3, 2))
    b = rng.standard_normal(4)
    y = oracle.conv2d(x, w, b, 1, (2, 1), 1)
    xp = np.pad(x, ((0, 0), (0, 0), (2, 2), (1, 1)))
    np.testing.assert_array_equal(y, oracle.conv2d(xp, w, b, 1, 0, 1))


def test_stride_identity():
    """conv stride s == (conv stride 1)[::s, ::s]."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 2, 11, 10))
    w = rng.standard_normal((3, 2, 3, 3))
    for s in (2, 3):
        y = oracle.conv2d(x, w, None, s, 1, 1)
        y1 = oracle.conv2d(x, w, None, 1, 1, 1)
        np.testing.assert_array_equal(y, y1[:, :, ::s, ::s][:, :, :y.shape[2], :y.shape[3]])


def test_dilation_identity():
    """conv dilation d == conv with the zero-inserted kernel of size d(R-1)+1, dilation 1."""
    rng = np.random.default_rng(6)
    x = rng.standard_normal((1, 2, 12, 11))
    w = rng.standard_normal((3, 2, 3, 2))
    for d in (2, 3):
        wd = np.zeros((3, 2, d * 2 + 1, d * 1 + 1))
        wd[:, :, ::d, ::d] = w
        np.testing.assert_array_equal(oracle.conv2d(x, w, None, 1, 1, d),
                                      oracle.conv2d(x, wd, None, 1, 1, 1))


def test_group_identity():
    """grouped conv == concat over groups of independent convs on channel slices."""
    rng = np.random.default_rng(7)
    G, C, K = 3, 6, 9
    x = rng.standard_normal((2, C, 5, 5))
    w = rng.standard_normal((K, C // G, 3, 3))
    b = rng.standard_normal(K)
    y = oracle.conv2d(x, w, b, 1, 1, 1, groups=G)
    parts = [oracle.conv2d(x[:, g * 2:(g + 1) * 2], w[g * 3:(g + 1) * 3], b[g * 3:(g + 1) * 3], 1, 1, 1)
             for g in range(G)]
    np.testing.assert_array_equal(y, np.concatenate(parts, axis=1))


def test_batch_independence_and_threads():
    """conv of a batch == stack of per-image convs (also pins batch sharding); any thread
    count gives identical bits (one accumulator per output element)."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((4, 3, 7, 7))
    w = rng.standard_normal((5, 3, 3, 3))
    b = rng.standard_normal(5)
    y = oracle.conv2d(x, w, b, 1, 1, 1, threads=3)
    for n in range(4):
        np.testing.assert_array_equal(y[n:n + 1], oracle.conv2d(x[n:n + 1], w, b, 1, 1, 1, threads=1))
    np.testing.assert_array_equal(y, oracle.conv2d(x, w, b, 1, 1, 1, threads=1))


def test_points_match_full():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 3, 9, 8))
    w = rng.standard_normal((4, 3, 3, 3))
    b = rng.standard_normal(4)
    y = oracle.conv2d(x, w, b, 2, 1, 1)
    idx = np.array(list(itertools.product(range(2), range(4), range(y.shape[2]), range(y.shape[3]))))
    np.testing.assert_array_equal(oracle.conv2d_points(x, w, b, idx, 2, 1, 1), y.reshape(-1))
    with pytest.raises(oracle.OracleError):
        oracle.conv2d_points(x, w, b, [[0, 4, 0, 0]], 2, 1, 1)


# ---------------------------------------------------------------- independent formulations

def _shift_accumulate(x, w, b, stride, pad, dil, groups, dtype=np.float64):
    """SMM-style formulation: y = sum over taps (r,s) of a channel
    contraction of the shifted (strided) padded input plane.  Different loop
    structure and summation order from the oracle's nested loops."""
    N, C, H, W = x.shape
    K, Cg, R, S = w.shape
    Kg = K // groups
    xp = np.pad(x.astype(dtype), ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    P = (H + 2 * pad - dil * (R - 1) - 1) // stride + 1
    Q = (W + 2 * pad - dil * (S - 1) - 1) // stride + 1
    y = np.zeros((N, K, P, Q), dtype=dtype)
    for g in range(groups):
        xs = xp[:, g * Cg:(g + 1) * Cg]
        wg = w[g * Kg:(g + 1) * Kg].astype(dtype)
        for r in range(R):
            for s in range(S):
                plane = xs[:, :, r * dil: r * dil + stride * (P - 1) + 1: stride,
                           s * dil: s * dil + stride * (Q - 1) + 1: stride]
                y[:, g * Kg:(g + 1) * Kg] += np.einsum("kc,ncpq->nkpq", wg[:, :, r, s], plane)
    if b is not None:
        y += np.asarray(b, dtype=dtype)[None, :, None, None]
    return y


def _sweep_cases(count, seed):
    """SPEC.md:198 sweep ranges: kernel 1-5, stride 1-3, padding 0-2, dilation 1-2,
    channels 1-8, spatial 4-16, batch 1-4 (plus groups 1-2)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        R = int(rng.integers(1, 6)); S = int(rng.integers(1, 6))
        st = int(rng.integers(1, 4)); pd = int(rng.integers(0, 3)); dl = int(rng.integers(1, 3))
        G = int(rng.integers(1, 3))
        C = G * int(rng.integers(1, 5)); K = G * int(rng.integers(1, 5))
        H = int(rng.integers(4, 17)); W = int(rng.integers(4, 17)); N = int(rng.integers(1, 5))
        if H + 2 * pd < dl * (R - 1) + 1 or W + 2 * pd < dl * (S - 1) + 1:
            continue
        out.append(ConvShape("sweep", N, C, H, W, K, R, S, st, pd, dl, G, bias=bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("shape", _sweep_cases(40, 10), ids=lambda s: f"{s.N}x{s.C}x{s.H}x{s.W}_k{s.K}_{s.R}x{s.S}_s{s.stride}p{s.pad}d{s.dil}g{s.groups}")
def test_sweep_vs_shift_accumulate_and_torch(shape):
    import torch
    x, w, b = conv_inputs(shape, seed=stable_seed((shape.N, shape.C, shape.H, shape.K, shape.R)))
    y = oracle.conv2d(x, w, b, shape.stride, shape.pad, shape.dil, shape.groups)
    ref = _shift_accumulate(x, w, b, shape.stride, shape.pad, shape.dil, shape.groups)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    t = torch.nn.functional.conv2d(torch.from_numpy(x.astype(np.float64)), torch.from_numpy(w.astype(np.float64)),
                                   None if b is None else torch.from_numpy(b.astype(np.float64)),
                                   shape.stride, shape.pad, shape.dil, shape.groups).numpy()
    np.testing.assert_allclose(y, t, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("shape", [ConvShape("int3x3", 2, 64, 9, 11, 32, 3, 3, 1, 1),
                                   ConvShape("int5x5s2", 1, 16, 13, 12, 24, 5, 5, 2, 2),
                                   ConvShape("int1x1", 3, 48, 5, 5, 40, 1, 1)])
def test_integer_exact_vs_int64(shape):
    """Integer inputs: the fp64 oracle must equal exact int64 arithmetic bit for bit."""
    x, w, b = integer_inputs(shape, seed=11)
    y = oracle.conv2d(x, w, b, shape.stride, shape.pad, shape.dil)
    ref = _shift_accumulate(x.astype(np.int64), w.astype(np.int64), b.astype(np.int64),
                            shape.stride, shape.pad, shape.dil, 1, dtype=np.int64)
    np.testing.assert_array_equal(y, ref.astype(np.float64))
    assert np.abs(y).max() < 2 ** 24


def test_brute_force_tiny_by_hand():
    """A 2x2 input, 2x2 kernel, padding 1: every output written out by hand."""
    x = np.array([[[[1.0, 2.0], [3.0, 4.0]]]])
    w = np.array([[[[10.0, 20.0], [30.0, 40.0]]]])
    y = oracle.conv2d(x, w, [0.5], 1, 1, 1)
    # output (p,q) sees padded window rows p..p+1, cols q..q+1 of [[0,0,0,0],[0,1,2,0],[0,3,4,0],[0,0,0,0]]
    ref = np.array([[1 * 40 + 0.5, 1 * 30 + 2 * 40 + 0.5, 2 * 30 + 0.5],
                    [1 * 20 + 3 * 40 + 0.5, 1 * 10 + 2 * 20 + 3 * 30 + 4 * 40 + 0.5, 2 * 10 + 4 * 30 + 0.5],
                    [3 * 20 + 0.5, 3 * 10 + 4 * 20 + 0.5, 4 * 10 + 0.5]])
    np.testing.assert_array_equal(y[0, 0], ref)


def test_rel_err_metric():
    assert oracle.rel_err([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert oracle.rel_err([1.0, 2.5], [1.0, 2.0]) == pytest.approx(0.25)
    assert oracle.rel_err([0.0, 1e-3], [0.0, 0.0]) == pytest.approx(1e-3)  # absolute fallback (R7)
