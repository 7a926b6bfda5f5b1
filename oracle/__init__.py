"""CPU fp64 oracle for the ai3 conv2d hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2410_08300_b200``) never imports it and shares no code with it.

The arithmetic lives in ``conv2d_oracle.c`` (plain C, fp64 nested loops, the
SPEC.md:130 / PAPER.md:56 definition written out -- see that file's header);
this module only marshals numpy arrays through ctypes.  Every algorithm the
paper lets a user select (direct, IM2COL/GEMM, implicit GEMM, Winograd,
PAPER.md:53-56 and :192-195) computes this same function, so one oracle
serves all of them.

Pins (tests/test_oracle.py, run with ``-m "not gpu"``): SPEC worked examples
(tests/golden/), 1x1-conv == matmul, delta kernels, linearity, padding /
stride / dilation / group / batch identities, brute force on tiny inputs,
integer-exact cases, and torch.nn.functional.conv2d in float64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv2d_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_ERRORS = {-1: "invalid argument", -2: "channels not divisible by groups",
           -3: "effective kernel larger than padded input"}


class OracleError(ValueError):
    pass


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc -O2 (no fast-math). Returns the .so path."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-fno-fast-math", "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_conv2d.argtypes = [dp, dp, dp] + [i64] * 14 + [dp, ctypes.c_int]
        lib.oracle_conv2d.restype = ctypes.c_int
        lib.oracle_conv2d_points.argtypes = [dp, dp, dp] + [i64] * 14 + [
            ctypes.POINTER(ctypes.c_int64), i64, dp]
        lib.oracle_conv2d_points.restype = ctypes.c_int
        lib.oracle_conv2d_out_shape.argtypes = [i64] * 10 + [ctypes.POINTER(i64)] * 2
        lib.oracle_conv2d_out_shape.restype = ctypes.c_int
        _lib = lib
    return _lib


def _pair(v):
    if isinstance(v, (tuple, list)):
        assert len(v) == 2
        return int(v[0]), int(v[1])
    return int(v), int(v)


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def host_threads() -> int:
    """Cores this process may run on (sched_getaffinity), the oracle's thread count."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def output_shape(in_hw, kernel_hw, stride=1, padding=0, dilation=1):
    """(P, Q) by the SPEC.md:120 floor formula; raises OracleError if < 1."""
    lib = _load()
    (H, W), (R, S) = in_hw, kernel_hw
    sh, sw = _pair(stride); ph, pw = _pair(padding); dh, dw = _pair(dilation)
    P, Q = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.oracle_conv2d_out_shape(H, W, R, S, sh, sw, ph, pw, dh, dw,
                                     ctypes.byref(P), ctypes.byref(Q))
    if rc != 0:
        raise OracleError(_ERRORS.get(rc, str(rc)))
    return P.value, Q.value


def _prep(x, w, b):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    bb = None if b is None else np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if x.ndim != 4 or w.ndim != 4:
        raise OracleError("x and w must be rank 4 (NCHW / KCRS)")
    if bb is not None and bb.shape != (w.shape[0],):
        raise OracleError("bias must have shape (K,)")
    return x, w, bb


def conv2d(x, w, b=None, stride=1, padding=0, dilation=1, groups=1, threads=None):
    """y = conv2d(x, w, b) in fp64, NCHW, exactly the SPEC.md:130 sum.

    x: (N,C,H,W); w: (K,C/groups,R,S); b: (K,) or None.  Inputs are widened
    exactly to float64 (fp32 / bf16-representable values lose nothing).
    """
    lib = _load()
    x, w, b = _prep(x, w, b)
    N, C, H, W = x.shape
    K, Cg, R, S = w.shape
    if Cg * groups != C:
        raise OracleError(f"weight has {Cg} input channels per group, input has {C} for groups={groups}")
    sh, sw = _pair(stride); ph, pw = _pair(padding); dh, dw = _pair(dilation)
    P, Q = output_shape((H, W), (R, S), stride, padding, dilation)
    y = np.empty((N, K, P, Q), dtype=np.float64)
    nt = host_threads() if threads is None else int(threads)
    rc = lib.oracle_conv2d(_dptr(x), _dptr(w), None if b is None else _dptr(b),
                           N, C, H, W, K, R, S, sh, sw, ph, pw, dh, dw, groups, _dptr(y), nt)
    if rc != 0:
        raise OracleError(_ERRORS.get(rc, str(rc)))
    return y


def conv2d_points(x, w, b, idx, stride=1, padding=0, dilation=1, groups=1):
    """Sampled outputs: idx is an (M,4) int array of (n,k,p,q); returns (M,) fp64."""
    lib = _load()
    x, w, b = _prep(x, w, b)
    N, C, H, W = x.shape
    K, Cg, R, S = w.shape
    if Cg * groups != C:
        raise OracleError("channel/group mismatch")
    sh, sw = _pair(stride); ph, pw = _pair(padding); dh, dw = _pair(dilation)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1, 4))
    out = np.empty(idx.shape[0], dtype=np.float64)
    rc = lib.oracle_conv2d_points(_dptr(x), _dptr(w), None if b is None else _dptr(b),
                                  N, C, H, W, K, R, S, sh, sw, ph, pw, dh, dw, groups,
                                  idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  idx.shape[0], _dptr(out))
    if rc != 0:
        raise OracleError(_ERRORS.get(rc, str(rc)))
    return out


def rel_err(y, ref) -> float:
    """max|y - ref| / max|ref| in fp64; absolute if max|ref| == 0
    (reading R7 in DESIGN.md)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.shape != ref.shape:
        raise OracleError(f"shape mismatch {y.shape} vs {ref.shape}")
    if ref.size == 0:
        return 0.0
    err = float(np.max(np.abs(y - ref)))
    scale = float(np.max(np.abs(ref)))
    return err / scale if scale > 0 else err
