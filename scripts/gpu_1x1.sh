#!/bin/bash
# 1x1 layers: flat tiled mode vs the halo modes (AI3_HALO1X1=1), with the engine configuration
cd "$(dirname "$0")/.."
for L in rn50_01_64x56_64_1x1s1 rn50_03_64x56_256_1x1s1 rn50_04_256x56_64_1x1s1 rn50_05_256x56_128_1x1s1 rn50_09_512x28_128_1x1s1; do
  for h in 1 0; do AI3_HALO1X1=$h AI3_TC_VERBOSE=1 timeout 60 python scripts/layer_bench.py $L implicit_gemm --net resnet50 --batch 256 --reps 20 2>&1 | sort -u | sed "s|^|[halo1x1=$h] |"; done
done
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_layers_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
