"""C ABI tier on the CPU box: libai3.so loads without a GPU, exports every symbol
include/ai3.h declares, and its host-only entry points (names, output shape,
support checks, guess, workspace sizing, error reporting) behave as documented.
No compute call is made here."""
import ctypes
import json
import os
import re

import pytest
import torch

import paper_2410_08300_b200 as ai3
from paper_2410_08300_b200 import _lib
from synth import workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ai3.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"typedef[^;]*;", "", src, flags=re.S)  # function-pointer typedefs are not exports
    return sorted(set(re.findall(r"\b(ai3_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _header_functions()
    assert len(declared) >= 17
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_version_and_names():
    assert ai3.version() == 1000
    for name, aid in [("guess", 0), ("default", 0), ("auto", 0), ("direct", 1), ("gemm", 2), ("im2col", 2),
                      ("implicit_gemm", 3), ("winograd", 4), ("smm", 6), ("custom", 8)]:
        assert ai3.algo_id(name) == aid
    assert ai3.algo_name(3) == "implicit_gemm"
    with pytest.raises(ai3.UnknownAlgorithm, match="unknown algorithm 'fft'"):
        ai3.algo_id("fft")


def test_output_shapes_match_golden():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for s in g["shapes"]:
        assert list(ai3.output_shape(s["in"], s["K"], s["kernel"], s["stride"], s["padding"], s["dilation"])) == \
            s["out"]


def test_output_shape_matches_floor_formula_on_workloads():
    for name in ("vgg16", "resnet50", "alexnet"):
        for l in workload(name, 2):
            assert ai3.output_shape((2, l.C, l.H, l.W), l.K, (l.R, l.S), l.stride, l.pad, l.dil) == \
                (2, l.K, l.P, l.Q)


def test_shape_errors_name_the_constraint():
    with pytest.raises(ai3.Ai3Error, match="larger than the padded input"):
        ai3.output_shape((1, 3, 2, 2), 4, 3)
    with pytest.raises(ai3.Ai3Error, match="groups=2 must divide"):
        ai3.output_shape((1, 3, 8, 8), 4, 3, groups=2)
    with pytest.raises(ai3.Ai3Error, match="stride"):
        ai3.output_shape((1, 3, 8, 8), 4, 3, stride=0)


def test_winograd_preconditions():
    base = dict(in_shape=(1, 8, 16, 16), out_channels=8)
    assert ai3.supported(**base, kernel=3, padding=1, algorithm="winograd")
    for kw in (dict(kernel=5), dict(kernel=3, stride=2), dict(kernel=3, dilation=2, padding=2)):
        assert not ai3.supported(**base, **kw, algorithm="winograd")
    assert not ai3.supported((1, 8, 16, 16), 8, 3, groups=2, algorithm="winograd")


def test_smm_kn2row_preconditions():
    """smm supports every conv direct does (groups too); kn2row needs groups == 1."""
    for name in ("smm", "kn2row"):
        assert ai3.supported((1, 8, 16, 16), 8, 3, padding=1, algorithm=name)
        assert ai3.supported((2, 8, 16, 16), 8, 5, stride=2, dilation=2, padding=2, algorithm=name)
    assert ai3.supported((1, 8, 16, 16), 8, 3, groups=2, algorithm="smm")
    assert not ai3.supported((1, 8, 16, 16), 8, 3, groups=2, algorithm="kn2row")


def test_every_named_algorithm_is_built():
    """No reserved names remain: each selectable name resolves to a built algorithm."""
    for name in ("direct", "gemm", "im2col", "implicit_gemm", "implicit_precomp_gemm", "winograd", "smm", "kn2row",
                 "guess", "auto", "default", "benchmark"):
        assert ai3.supported((1, 8, 16, 16), 8, 3, padding=1, algorithm=name), name
    assert not ai3.supported((1, 8, 16, 16), 8, 3, groups=2, algorithm="implicit_precomp_gemm")


def _all_problem_shapes():
    out = []
    for name in ("vgg16", "resnet50", "alexnet", "config1"):
        out += [(l.N, l.C, l.H, l.W, l.K, l.R, l.stride, l.pad, l.dil, 1) for l in workload(name, 2)]
    out += [(2, 8, 9, 9, 8, 3, 1, 1, 1, 2), (1, 4, 5, 5, 4, 1, 1, 0, 1, 4), (3, 6, 12, 10, 9, 5, 2, 2, 2, 3)]
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_guess_is_deterministic_and_supported(dtype):
    """guess never returns an algorithm whose preconditions the spec violates."""
    for (N, C, H, W, K, R, s, p, d, g) in _all_problem_shapes():
        a = ai3.guess((N, C, H, W), K, R, s, p, d, g, dtype=dtype)
        assert a == ai3.guess((N, C, H, W), K, R, s, p, d, g, dtype=dtype)
        assert a in ("direct", "gemm", "implicit_gemm", "winograd")
        assert ai3.supported((N, C, H, W), K, R, s, p, d, g, dtype=dtype, algorithm=a)
        if g > 1:
            assert a == "direct"


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_guess_strided_rgb_stems_use_s2d_implicit_gemm(dtype):
    """DESIGN.md R24: strided RGB stems (ResNet 7x7 s2, AlexNet 11x11 s4) have a space-to-depth
    view with full K-block rows, so guess routes them to implicit_gemm; AI3_S2D=0 restores gemm
    (checked in a subprocess: the switch is read per call)."""
    assert ai3.guess((256, 3, 224, 224), 64, 7, 2, 3, 1, 1, dtype=dtype) == "implicit_gemm"
    assert ai3.guess((128, 3, 224, 224), 64, 11, 4, 2, 1, 1, dtype=dtype) == "implicit_gemm"
    # a 1x1 strided conv has no s2d benefit (kernel smaller than the stride): explicit GEMM
    assert ai3.guess((256, 3, 224, 224), 64, 1, 2, 0, 1, 1, dtype=dtype) == "gemm"


def test_guess_routes_narrow_channel_layers():
    """bf16 stride-1 layers with 9..16 channels take the 32-byte-pixel halo (implicit_gemm); the
    same layer in fp32 (64-byte pixels would need C >= 8 for a full row) stays on gemm."""
    assert ai3.guess((64, 12, 112, 112), 64, 3, 1, 1, 1, 1, dtype=torch.bfloat16) == "implicit_gemm"
    assert ai3.guess((64, 16, 112, 112), 64, 5, 1, 2, 1, 1, dtype=torch.bfloat16) == "implicit_gemm"
    assert ai3.guess((64, 3, 112, 112), 64, 3, 1, 1, 1, 1, dtype=torch.float32) == "gemm"


def test_s2d_workspace_holds_the_s2d_image():
    """R24: the implicit_gemm workspace of the ResNet stem (NHWC bf16 input) is the s2d image,
    N x (P+T-1) x (Q+T-1) x 16 channels of bf16 (P = Q = 112, T = 4) plus the prepared weights."""
    lib = _lib.load()
    prm = _lib.params(64, (7, 7), (2, 2), (3, 3), (1, 1), 1, False)
    out = ctypes.c_size_t()
    st = lib.ai3_conv2d_workspace_size(ctypes.byref(prm), _lib.shape4((8, 3, 224, 224)), _lib.BF16, _lib.MATH_STRICT,
                                       ai3.algo_id("implicit_gemm"), _lib.NHWC, _lib.NHWC, ctypes.byref(out))
    assert st == 0, _lib.last_error()
    image = 8 * 115 * 115 * 16 * 2
    weights = 64 * 16 * 16 * 2
    assert image + weights <= out.value <= image + weights + 4096


def test_workspace_sizes():
    lib = _lib.load()

    def ws(shape, K, R, algo, dtype=_lib.BF16, math=_lib.MATH_STRICT, lin=_lib.NHWC, lout=_lib.NHWC, pad=1):
        prm = _lib.params(K, (R, R), (1, 1), (pad, pad), (1, 1), 1, True)
        out = ctypes.c_size_t()
        st = lib.ai3_conv2d_workspace_size(ctypes.byref(prm), _lib.shape4(shape), dtype, math, ai3.algo_id(algo),
                                           lin, lout, ctypes.byref(out))
        assert st == 0, _lib.last_error()
        return out.value

    # implicit GEMM on NHWC bf16 with C % 16 == 0: only the prepared weights (K*R*S*C*2 + bias)
    w_only = ws((64, 256, 56, 56), 256, 3, "implicit_gemm")
    assert w_only == 256 * 9 * 256 * 2 + 256 * 4
    # explicit GEMM adds the im2col matrix
    assert ws((64, 256, 56, 56), 256, 3, "gemm") >= w_only + 64 * 56 * 56 * 9 * 256 * 2
    # NCHW input adds the layout pass
    assert ws((64, 256, 56, 56), 256, 3, "implicit_gemm", lin=_lib.NCHW) >= w_only + 64 * 56 * 56 * 256 * 2
    # Winograd: 16 transformed tiles in (V) and out (M: bf16 for bf16 runs, fp32 otherwise)
    T = 64 * 28 * 28
    assert ws((64, 256, 56, 56), 256, 3, "winograd") >= 16 * T * 256 * 2 + 16 * T * 256 * 2
    # bf16 NHWC outputs with K <= 64 run the fused kernel (M stays in TMEM): V only
    assert 16 * T * 256 * 2 <= ws((64, 256, 56, 56), 64, 3, "winograd") < 16 * T * 256 * 2 + 16 * T * 64 * 2
    assert ws((64, 256, 56, 56), 64, 3, "winograd", lout=_lib.NCHW) >= 16 * T * 256 * 2 + 16 * T * 64 * 2
    assert ws((64, 256, 56, 56), 256, 3, "winograd", dtype=_lib.F32) >= 16 * T * 256 * 4 + 16 * T * 256 * 4
    # direct needs no workspace beyond the fp32 weights [Cg][R][S][K padded to 64] and the fp32
    # bias, each region 256-byte aligned: 3*3*3*64*4 = 6912 (already aligned) + 256
    assert ws((2, 3, 32, 32), 16, 3, "direct", dtype=_lib.F32) == 6912 + 256


def test_null_and_bad_arguments():
    lib = _lib.load()
    out = (ctypes.c_int64 * 4)()
    assert lib.ai3_conv2d_output_shape(None, _lib.shape4((1, 1, 4, 4)), out) == _lib.ERR_INVALID_ARGUMENT
    assert "null" in _lib.last_error()
    assert lib.ai3_conv2d_plan_execute(None, None, None, None, 0, None) == _lib.ERR_INVALID_ARGUMENT
    lib.ai3_conv2d_plan_destroy(None)  # no-op


def test_product_never_imports_oracle():
    """The product package must not route through the oracle (there is no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2410_08300_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), fn


def test_kn2row_is_memory_lean():
    """kn2row's defining property (§II.B(b): it transforms the kernel "in order to
    decrease memory usage"): its workspace is the fp32 output accumulator, O(N*K*P*Q), below
    im2col's R*S-fold copy of the input -- and nothing for fp32 NHWC outputs (accumulated in
    place).  VGG conv3_2 at the bench batch (64 x 256 x 56 x 56, bf16)."""
    import ctypes
    lib = _lib.load()

    def ws(algo, dtype, layout):
        p = _lib.params(256, (3, 3), (1, 1), (1, 1), (1, 1), 1, True)
        n = ctypes.c_size_t()
        st = lib.ai3_conv2d_workspace_size(ctypes.byref(p), _lib.shape4((64, 256, 56, 56)), dtype, 0,
                                           ai3.algo_id(algo), layout, layout, ctypes.byref(n))
        assert st == _lib.OK
        return n.value

    out_f32 = 64 * 256 * 56 * 56 * 4
    kn, gemm = ws("kn2row", _lib.BF16, _lib.NHWC), ws("gemm", _lib.BF16, _lib.NHWC)
    assert kn < gemm / 4
    assert kn <= out_f32 + (2 << 20)  # + the packed weights (1.2 MB)
    # fp32 NHWC accumulates in place: nothing beyond what implicit_gemm needs (weights + the
    # operand-rounding pass of the input)
    assert ws("kn2row", _lib.F32, _lib.NHWC) <= ws("implicit_gemm", _lib.F32, _lib.NHWC)
