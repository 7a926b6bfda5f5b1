#!/bin/bash
cd "$(dirname "$0")/.."
for v in "X=0" "AI3_TC_STORE=0" "AI3_TC_STORE=2" "AI3_BOX64=0" "AI3_EPI_FAST=0"; do
  for L in "conv1_1 --net vgg16 --batch 64" "rn50_00_3x224_64_7x7s2 --net resnet50 --batch 256" "rn50_04_256x56_64_1x1s1 --net resnet50 --batch 256"; do
    env $v timeout 60 python scripts/layer_bench.py ${L%% *} implicit_gemm ${L#* } --reps 20 2>&1 | grep implicit | sed "s|^|[$v] |"
  done
done
