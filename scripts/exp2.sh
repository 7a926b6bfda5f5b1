#!/bin/bash
# experiment batch 2: bn=192 product timing + parity; pipeline traces; chunked halo at K=256
cd "$(dirname "$0")/.."
DEV=paper_2410_08300_b200/libai3_dev.so
for l in conv5_2 conv1_1 conv3_2; do timeout 60 python scripts/layer_bench.py $l implicit_gemm --reps 20; done
timeout 600 python -m pytest tests/test_fullsize_gpu.py -q -x -k "conv5 or rn50_18 or rn50_21 or rn50_22 or alexnet" 2>&1 | tail -3
for l in conv1_1 conv1_2 conv2_2 conv3_2 conv5_2; do timeout 60 python scripts/trace_layer.py $l; done
for rep in 1 2; do
for cfg in "AI3_HALO_KMAX=128" "AI3_HALO_KMAX=256"; do
  for l in conv3_1 conv3_2; do
  env $cfg timeout 60 python scripts/layer_bench.py $l implicit_gemm --reps 20 --lib $DEV | sed "s|^|[$cfg] |"
  done
done
done
for cfg in "AI3_TC_CG=2" "AI3_TC_CG=1"; do
  env $cfg timeout 60 python scripts/layer_bench.py conv1_1 implicit_gemm --reps 20 --lib $DEV | sed "s|^|[$cfg] |"
done
