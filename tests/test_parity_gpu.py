"""GPU parity: every algorithm, through the C ABI, against the CPU fp64 oracle on
the same seeded inputs (tolerances are the north_star's, see helpers.TOL).

Sizes span several 128-row tiles with a ragged tail; integer-valued cases must be
bit-exact; full-size layers are checked on sampled outputs in tests/test_fullsize_gpu.py.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
from helpers import inputs, ref, run_ai3, tolerance, to_device, stable_seed
from synth import CONFIG1, ConvShape, integer_inputs

pytestmark = pytest.mark.gpu

ALGOS = ["direct", "gemm", "implicit_gemm", "implicit_precomp_gemm", "winograd", "smm", "kn2row", "guess"]
MODES = [("f32", "strict"), ("f32", "tf32"), ("bf16", "strict")]


def _supports(shape: ConvShape, algo: str) -> bool:
    if algo in ("direct", "smm", "guess"):
        return True
    if shape.groups != 1:
        return False
    if algo == "winograd":
        return shape.R == 3 and shape.S == 3 and shape.stride == 1 and shape.dil == 1
    return True


def _expect_unsupported(shape, algo):
    """An algorithm whose preconditions the layer violates (Winograd off 3x3 / stride 1,
    tensor-core algorithms with groups, R5) must say so -- supported() is False and a call
    raises UnsupportedConfiguration -- instead of computing anything."""
    import paper_2410_08300_b200 as ai3
    x, w, b = inputs(shape, 1, "f32")
    xt, wt = to_device(x, "f32"), to_device(w, "f32")
    assert not ai3.supported(xt.shape, shape.K, (shape.R, shape.S), shape.stride, shape.pad, shape.dil, shape.groups,
                             torch.float32, algorithm=algo)
    with pytest.raises(ai3.UnsupportedConfiguration):
        ai3.conv2d(xt, wt, None, shape.stride, shape.pad, shape.dil, shape.groups, algo)


def _check(shape, algo, dtype, math, layout, seed, plan=True):
    x, w, b = inputs(shape, seed, dtype)
    y = run_ai3(shape, x, w, b, algo, dtype, math, layout, plan)
    r = ref(shape, x, w, b)
    err = oracle.rel_err(y, r)
    tol = tolerance(algo, dtype, math)
    assert err <= tol, f"{algo} {dtype}/{math} {layout}: rel err {err:.3e} > {tol:.0e}"
    return err


# ------------------------------------------------------------------ config 1 (BASELINE configs[0])
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype,math", MODES)
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_config1_all_algorithms(algo, dtype, math, layout):
    _check(CONFIG1, algo, dtype, math, layout, seed=1000)


def test_config1_stateless_call():
    for algo in ALGOS:
        _check(CONFIG1, algo, "f32", "strict", "nchw", seed=1001, plan=False)


# ------------------------------------------------------------------ multi-tile ragged shapes
RAGGED = [
    ConvShape("r3x3", 2, 64, 23, 23, 96, 3, 3, 1, 1),     # M = 1058: 9 tiles, 34-row tail
    ConvShape("r3x3_c48", 3, 48, 17, 19, 40, 3, 3, 1, 1),  # C not a multiple of 64, K < 64
    ConvShape("r3x3_k200", 1, 128, 30, 30, 200, 3, 3, 1, 1, bias=False),
    ConvShape("r1x1", 2, 256, 14, 14, 72, 1, 1),
    ConvShape("r1x1s2", 2, 96, 15, 15, 64, 1, 1, 2, 0),
    ConvShape("r5x5", 2, 32, 21, 20, 48, 5, 5, 1, 2),
    ConvShape("r7x7s2", 2, 3, 45, 45, 64, 7, 7, 2, 3),     # ResNet stem shape, small
    ConvShape("r11s4", 2, 3, 67, 67, 64, 11, 11, 4, 2),    # AlexNet conv1 shape, small
    ConvShape("r3x3d2", 2, 32, 19, 19, 32, 3, 3, 1, 2, 2),
    ConvShape("r3x3s2", 2, 128, 28, 28, 128, 3, 3, 2, 1),
    ConvShape("rodd", 1, 16, 9, 7, 24, 3, 3, 1, 0),       # odd P, Q: Winograd crop
    ConvShape("rhalo2", 2, 128, 21, 27, 96, 3, 3, 1, 1),  # chunked halo: 2 channel chunks, ragged tiles
    ConvShape("rhalo3", 1, 192, 17, 13, 64, 5, 5, 1, 2),  # chunked halo: 3 chunks, 5x5 taps
]


@pytest.mark.parametrize("shape", RAGGED, ids=lambda s: s.name)
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype,math", MODES)
def test_ragged_shapes(shape, algo, dtype, math):
    if not _supports(shape, algo):
        return _expect_unsupported(shape, algo)
    _check(shape, algo, dtype, math, "nhwc" if shape.C % 2 == 0 else "nchw", seed=stable_seed(shape.name))


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("algo", ["implicit_gemm", "implicit_precomp_gemm", "gemm", "winograd", "direct", "smm", "kn2row"])
def test_layouts_bf16(layout, algo):
    _check(RAGGED[0], algo, "bf16", "strict", layout, seed=7)


# ------------------------------------------------------------------ SPEC sweep ranges
def _sweep(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        R = int(rng.integers(1, 6)); S = int(rng.integers(1, 6))
        st = int(rng.integers(1, 4)); pd = int(rng.integers(0, 3)); dl = int(rng.integers(1, 3))
        G = int(rng.integers(1, 3)) if len(out) % 3 == 0 else 1
        C = G * int(rng.integers(1, 9)); K = G * int(rng.integers(1, 9))
        H = int(rng.integers(4, 17)); W = int(rng.integers(4, 17)); N = int(rng.integers(1, 5))
        if H + 2 * pd < dl * (R - 1) + 1 or W + 2 * pd < dl * (S - 1) + 1:
            continue
        out.append(ConvShape(f"sw{len(out)}", N, C, H, W, K, R, S, st, pd, dl, G, bias=bool(rng.integers(0, 2))))
    # make sure Winograd-eligible shapes are in the sweep
    out += [ConvShape(f"sww{i}", int(rng.integers(1, 5)), int(rng.integers(1, 9)), int(rng.integers(4, 17)),
                      int(rng.integers(4, 17)), int(rng.integers(1, 9)), 3, 3, 1, int(rng.integers(0, 3)))
            for i in range(6)]
    return out


@pytest.mark.parametrize("shape", _sweep(24, 42), ids=lambda s: s.name)
@pytest.mark.parametrize("algo", ALGOS)
def test_spec_sweep(shape, algo):
    if not _supports(shape, algo):
        return _expect_unsupported(shape, algo)
    for dtype, math in (("f32", "strict"), ("bf16", "strict")):
        _check(shape, algo, dtype, math, "nchw", seed=stable_seed((shape.name, algo)))


# ------------------------------------------------------------------ exact cases
INT_SHAPES = [ConvShape("i3x3", 2, 64, 20, 21, 80, 3, 3, 1, 1), ConvShape("i5x5s2", 2, 16, 19, 17, 32, 5, 5, 2, 2),
              ConvShape("i1x1", 3, 32, 11, 13, 48, 1, 1), ConvShape("i3x3c3", 2, 3, 33, 31, 16, 3, 3, 1, 1)]


@pytest.mark.parametrize("shape", INT_SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype,math", MODES)
def test_integer_inputs_bit_exact(shape, algo, dtype, math):
    """Integer x, w, b keep every product and partial sum exact in fp32 (and every
    operand exact in tf32 / bf16), so each path must reproduce the oracle bit for bit.
    bf16 outputs additionally need |y| <= 256: use x, w in {-1, 0, 1} there."""
    if not _supports(shape, algo):
        return _expect_unsupported(shape, algo)
    small = dtype == "bf16"
    x, w, b = integer_inputs(shape, seed=5, xmax=1 if small else 8, wmax=1 if small else 4)
    if small and shape.C * shape.R * shape.S > 250:
        x, w = x, w * (np.abs(np.arange(w.size).reshape(w.shape) % 3) == 0)  # thin out taps to keep |y| <= 256
    y = run_ai3(shape, x, w, b, algo, dtype, math, "nhwc")
    r = ref(shape, x, w, b)
    assert np.abs(r).max() < (256 if small else 2 ** 24)
    if algo == "winograd" and dtype == "bf16":
        # bf16 Winograd stores the transformed-domain products M in bf16 (R26): the
        # one inexact step; the result stays within the bf16 bound
        assert oracle.rel_err(y, r) <= 2e-2
        return
    np.testing.assert_array_equal(y, r)


# ------------------------------------------------------------------ degenerate cases
DEGEN = [ConvShape("out1x1", 2, 8, 3, 3, 5, 3, 3), ConvShape("k1", 1, 4, 6, 6, 1, 3, 3, 1, 1),
         ConvShape("c1", 2, 1, 9, 9, 16, 3, 3, 1, 1), ConvShape("hw1", 3, 32, 1, 1, 24, 1, 1),
         ConvShape("pad_only", 1, 2, 1, 1, 3, 3, 3, 1, 1), ConvShape("wide", 1, 8, 2, 130, 8, 1, 3, 1, 0)]


@pytest.mark.parametrize("shape", DEGEN, ids=lambda s: s.name)
@pytest.mark.parametrize("algo", ALGOS)
def test_degenerate(shape, algo):
    if not _supports(shape, algo):
        return _expect_unsupported(shape, algo)
    _check(shape, algo, "f32", "strict", "nchw", seed=3)
    _check(shape, algo, "bf16", "strict", "nhwc", seed=4)


# ------------------------------------------------------------------ determinism / batch independence
@pytest.mark.parametrize("algo", ["direct", "gemm", "implicit_gemm", "implicit_precomp_gemm", "winograd", "smm", "kn2row"])
def test_deterministic_and_batch_independent(algo):
    """Same plan + input -> identical bits; and image n's output does not depend on the
    batch it was computed in (pins that batch sharding across GPUs is exact)."""
    import paper_2410_08300_b200 as ai3
    shape = ConvShape("det", 6, 64, 19, 19, 64, 3, 3, 1, 1)
    x, w, b = inputs(shape, 11, "bf16")
    xt, wt, bt = to_device(x, "bf16", "nhwc"), to_device(w, "bf16"), to_device(b, "bf16")
    p = ai3.ConvPlan(wt, bt, xt.shape, 1, 1, 1, 1, algo, in_layout=1)
    y1, y2 = p(xt).clone(), p(xt).clone()
    assert torch.equal(y1, y2)
    p2 = ai3.ConvPlan(wt, bt, (2,) + tuple(xt.shape[1:]), 1, 1, 1, 1, algo, in_layout=1)
    for s in (0, 2, 4):
        part = p2(xt[s:s + 2].contiguous(memory_format=torch.channels_last))
        assert torch.equal(part, y1[s:s + 2])


@pytest.mark.parametrize("dtype,layout", [("f32", "nchw"), ("bf16", "nhwc")])
def test_direct_small_and_tiled_kernels_agree_bitwise(dtype, layout):
    """`direct` runs a one-thread-per-output kernel when the layer has fewer tiles than SMs
    (here at N = 1) and the tiled kernel otherwise (N = 96): both reduce in the same fmaf
    order, so image 0 comes out with the same bits either way (batch-size independence)."""
    import paper_2410_08300_b200 as ai3
    shape = ConvShape("smallvtiled", 96, 16, 32, 32, 32, 3, 3, 1, 1)
    x, w, b = inputs(shape, 5, dtype)
    xt, wt, bt = to_device(x, dtype, layout), to_device(w, dtype), to_device(b, dtype)
    big = ai3.conv2d(xt, wt, bt, 1, 1, 1, 1, "direct")
    one = ai3.conv2d(to_device(x[:1], dtype, layout), wt, bt, 1, 1, 1, 1, "direct")
    assert torch.equal(one, big[:1])
    ref = oracle.conv2d(x[:1], w, b, 1, 1, 1, 1)
    assert oracle.rel_err(one.double().cpu().numpy(), ref) <= (1e-5 if dtype == "f32" else 2e-2)


# (the harness has teeth: tests/test_mutation_gpu.py runs it against a faulty build)


def test_errors_surface_as_exceptions():
    import paper_2410_08300_b200 as ai3
    x = torch.zeros(1, 3, 8, 8, device="cuda")
    w = torch.zeros(4, 3, 5, 5, device="cuda")
    with pytest.raises(ai3.UnsupportedConfiguration):
        ai3.conv2d(x, w, None, 1, 0, 1, 1, "winograd")
    with pytest.raises(ai3.UnknownAlgorithm):
        ai3.conv2d(x, w, None, 1, 0, 1, 1, "nope")
    with pytest.raises(ai3.Ai3Error):
        ai3.conv2d(x, torch.zeros(4, 3, 9, 9, device="cuda"), None)  # kernel larger than input


# ------------------------------------------------------------------ host-to-host execution (bench e2e path)
def test_execute_host_single_and_pipelined_match_device():
    """ai3_conv2d_plan_execute_host and the pipelined ai3_conv2d_plans_execute_host give the
    device path's bits, and the device result matches the oracle."""
    import paper_2410_08300_b200 as ai3
    shapes = [ConvShape("h0", 3, 64, 20, 20, 64, 3, 3, 1, 1), ConvShape("h1", 2, 32, 17, 15, 48, 1, 1),
              ConvShape("h2", 1, 3, 33, 33, 16, 3, 3, 2, 1)]
    plans, xh, yh, xd, yd, want = [], [], [], [], [], []
    for i, sh in enumerate(shapes):
        x, w, b = inputs(sh, 40 + i, "bf16")
        xt = to_device(x, "bf16", "nhwc")
        p = ai3.ConvPlan(to_device(w, "bf16"), to_device(b, "bf16"), xt.shape, sh.stride, sh.pad, sh.dil, 1,
                         "guess", in_layout=1)
        y = p(xt)
        r = oracle.conv2d(xt.float().cpu().numpy(), to_device(w, "bf16").float().cpu().numpy(),
                          to_device(b, "bf16").float().cpu().numpy(), sh.stride, sh.pad, sh.dil)
        assert oracle.rel_err(y.float().cpu().numpy(), r) <= 2e-2
        plans.append(p)
        xh.append(xt.cpu().pin_memory())
        yh.append(torch.empty_like(y, device="cpu").pin_memory())
        xd.append(torch.empty_like(xt))
        yd.append(torch.empty_like(y))
        want.append(y.cpu())
    ai3.execute_host_many(plans, xh, yh, xd, yd)
    torch.cuda.synchronize()
    for a, b_ in zip(yh, want):
        assert torch.equal(a, b_)
    y1 = torch.empty_like(yh[0]).pin_memory()
    plans[0].execute_host(xh[0], y1, xd[0], yd[0])
    torch.cuda.synchronize()
    assert torch.equal(y1, want[0])

