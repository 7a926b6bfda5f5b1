#!/bin/bash
cd "$(dirname "$0")/.."
for lib in scratch_ab/libai3_dev_r2start.so paper_2410_08300_b200/libai3_dev.so; do
  AI3_TC_VERBOSE=1 timeout 60 python scripts/layer_bench.py conv3_1 implicit_gemm --reps 20 --lib $lib 2>&1 | tail -2
done
