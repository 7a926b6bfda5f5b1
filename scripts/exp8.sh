#!/bin/bash
cd "$(dirname "$0")/.."
DEV=paper_2410_08300_b200/libai3_dev.so
timeout 120 python scripts/layer_bench.py conv3_2 implicit_precomp_gemm --reps 5; echo "rc=$?"
timeout 600 python -m pytest tests -m gpu -q -x -k "precomp" --timeout 300 2>&1 | tail -3
for cfg in "AI3_GATHER_ASYNC=0" "AI3_GATHER_ASYNC=1"; do
  for l in conv1_2 conv2_2 conv3_2 conv4_2 conv5_2; do
    env $cfg timeout 60 python scripts/layer_bench.py $l implicit_precomp_gemm --reps 10 --lib $DEV | sed "s|^|[$cfg] |"
  done
done
