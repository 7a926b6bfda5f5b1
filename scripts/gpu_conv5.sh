#!/bin/bash
cd "$(dirname "$0")/.."
for v in "X=0" "AI3_BN=128" "AI3_N2=0" "AI3_TC_CG=1" "AI3_BN=128 AI3_TC_CG=1"; do
  for L in conv5_2 conv4_1 conv3_1; do env $v AI3_TC_VERBOSE=1 timeout 60 python scripts/layer_bench.py $L implicit_gemm --reps 20 2>&1 | grep -v "ai3 tc" | sed "s|^|[$v] |"; done
done
for v in "X=0" "AI3_BN=128"; do
  for L in rn50_13_256x14_1024_1x1s1 rn50_19_512x7_2048_1x1s1 rn50_21_2048x7_512_1x1s1 rn50_22_512x7_512_3x3s1 rn50_16_256x14_256_3x3s1; do env $v timeout 60 python scripts/layer_bench.py $L implicit_gemm --net resnet50 --batch 256 --reps 20 2>&1 | sed "s|^|[$v] |"; done
done
