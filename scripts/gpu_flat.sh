#!/bin/bash
# 1x1 flat-A A/B on the ResNet-50 1x1 layers + parity
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_layers_gpu.py -q -x 2>&1 | tail -1
for L in rn50_01_64x56_64_1x1s1 rn50_03_64x56_256_1x1s1 rn50_04_256x56_64_1x1s1 rn50_05_256x56_128_1x1s1 rn50_07_128x28_512_1x1s1 rn50_09_512x28_128_1x1s1 rn50_11_512x28_256_1x1s1 rn50_13_256x14_1024_1x1s1 rn50_15_1024x14_256_1x1s1 rn50_17_1024x14_512_1x1s1 rn50_19_512x7_2048_1x1s1 rn50_21_2048x7_512_1x1s1; do
  for f in 0 1; do AI3_FLAT1X1=$f timeout 60 python scripts/layer_bench.py $L implicit_gemm --net resnet50 --batch 256 --reps 20 | sed "s|^|[flat=$f] |"; done
done
