#!/bin/bash
# L2 prefetch distance A/B on the streaming ResNet 1x1 layers
cd "$(dirname "$0")/.."
for L in rn50_04_256x56_64_1x1s1 rn50_05_256x56_128_1x1s1 rn50_09_512x28_128_1x1s1 rn50_03_64x56_256_1x1s1 rn50_15_1024x14_256_1x1s1 rn50_21_2048x7_512_1x1s1; do
  for pf in 0 1 2 4; do AI3_PF=$pf timeout 60 python scripts/layer_bench.py $L implicit_gemm --net resnet50 --batch 256 --reps 20 | sed "s|^|[pf=$pf] |"; done
done
AI3_PF=2 timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "r1x1 or i1x1" 2>&1 | tail -1
