#!/bin/bash
# same-box A/B of the stem between an older build and the current one
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in scratch_ab/libai3_f23b91d.so paper_2410_08300_b200/libai3.so; do
    AI3_LIB=$lib timeout 60 python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 20 | sed "s|^|[$(basename $lib)] |"
  done
done


for v in "AI3_HALO32_SW=1" "AI3_S2D_SPLIT=1"; do env $v timeout 60 python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 20 | sed "s|^|[$v] |"; done
timeout 300 python -m pytest tests/test_s2d_gpu.py -q -x 2>&1 | tail -1
