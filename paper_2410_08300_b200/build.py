"""Build libai3.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2410_08300_b200.build        # incremental
    python -m paper_2410_08300_b200.build --force
    python -m paper_2410_08300_b200.build --dev  # developer build: A/B knobs read from the
                                                 # environment (-DAI3_DEV_KNOBS), never shipped

Each csrc/*.cu compiles to build/<name>.o in parallel; the objects link into
paper_2410_08300_b200/libai3.so with the static CUDA runtime.  The driver API
(tensor-map encoding) is resolved at run time via cudaGetDriverEntryPoint, so
the library loads on a host without a GPU driver (the CPU test tier checks
that it loads and exports every symbol include/ai3.h declares).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libai3.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "ai3.h")])


def _compile(src: str, force: bool, verbose: bool, build_dir: str = BUILD, extra=()) -> str:
    obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
    newest_dep = max(os.path.getmtime(p) for p in _deps() + [src])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """Build libai3.so.  variant="dev": the same sources with -DAI3_DEV_KNOBS into
    build_dev/ -> libai3_dev.so (environment-read A/B knobs; scripts only).
    variant="mutant": -DAI3_MUTANT_DROP_BIAS into build_mutant/ -> libai3_mutant.so, a
    deliberately faulty library (the engine epilogue drops the bias) that the mutation
    test (tests/test_mutation_gpu.py) must catch; nothing else loads it."""
    macro = {"": None, "dev": "AI3_DEV_KNOBS", "mutant": "AI3_MUTANT_DROP_BIAS"}[variant]
    bdir = BUILD if not variant else BUILD + "_" + variant
    lib = LIB if not variant else os.path.join(PKG, f"libai3_{variant}.so")
    os.makedirs(bdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if macro:  # only the sources that test the macro differ from the product objects
        build(force, verbose)
        own = [s for s in srcs if macro in open(s).read()]
    else:
        own = srcs
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, bdir, [f"-D{macro}"] if macro else [])
                           if s in own else os.path.join(BUILD, os.path.basename(s)[:-3] + ".o"), srcs))
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


def build_calib(force: bool = False) -> str:
    """libai3_calib.so: the FFMA-peak microbenchmark bench.py uses for the `direct` / `smm`
    roofline denominator (calib/ffma_peak.cu).  Not part of the convolution path."""
    src = os.path.join(PKG, "calib", "ffma_peak.cu")
    lib = os.path.join(PKG, "libai3_calib.so")
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        r = subprocess.run([NVCC, *ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", lib, src],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    v = "dev" if "--dev" in sys.argv else ("mutant" if "--mutant" in sys.argv else "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=v))
