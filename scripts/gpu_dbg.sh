#!/bin/bash
# which pipeline role limits a layer: AI3_TC_DEBUG 1 = no MMA, 2 = no TMA loads, 3 = no epilogue stores
cd "$(dirname "$0")/.."
for L in "rn50_04_256x56_64_1x1s1 --net resnet50 --batch 256" "rn50_09_512x28_128_1x1s1 --net resnet50 --batch 256" "conv1_1 --net vgg16 --batch 64" "conv3_2 --net vgg16 --batch 64"; do
  for d in 0 1 2 3; do AI3_TC_DEBUG=$d timeout 60 python scripts/layer_bench.py ${L%% *} implicit_gemm ${L#* } --reps 20 2>&1 | grep implicit | sed "s|^|[dbg=$d] |"; done
done
