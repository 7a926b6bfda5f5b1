#!/bin/bash
# store_mode 3 (coalesced st.global from the staging buffer) vs TMA stores (default)
cd "$(dirname "$0")/.."
AI3_TC_STORE=3 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_s2d_gpu.py tests/test_modes_gpu.py -q -x 2>&1 | tail -1
for L in "conv1_1 --net vgg16 --batch 64" "conv1_2 --net vgg16 --batch 64" "conv3_2 --net vgg16 --batch 64" "rn50_00_3x224_64_7x7s2 --net resnet50 --batch 256" "rn50_03_64x56_256_1x1s1 --net resnet50 --batch 256" "rn50_01_64x56_64_1x1s1 --net resnet50 --batch 256" "conv1 --net alexnet --batch 128"; do
  for m in 1 3; do AI3_TC_STORE=$m timeout 60 python scripts/layer_bench.py ${L%% *} implicit_gemm ${L#* } --reps 20 2>&1 | sed "s|^|[store=$m] |"; done
done
