#!/bin/bash
# stem A/B (32-byte halo: two planes vs one SWIZZLE_32B load) + ncu of the stem GEMM.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_s2d_gpu.py -q -x 2>&1 | tail -2
AI3_S2D_SPLIT=1 timeout 300 python -m pytest tests/test_s2d_gpu.py -q -x 2>&1 | tail -2
for sw in 0; do
  AI3_HALO32_SW=$sw timeout 120 python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 20
  AI3_HALO32_SW=$sw timeout 120 python scripts/layer_bench.py conv1 implicit_gemm --net alexnet --batch 128 --reps 20
done
AI3_S2D_SPLIT=0 timeout 120 python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 20
timeout 120 python scripts/layer_bench.py conv1_1 implicit_gemm --net vgg16 --batch 64 --reps 20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stem_launches.csv python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 2 > /dev/null 2>&1; grep -o "ai3::[a-z_0-9]*[^,]*,[^,]*,[^,]*,\"[0-9]*\"" gpurun_out/stem_launches.csv | tail -4; grep ai3 gpurun_out/stem_launches.csv | tail -3 | cut -c1-60,400-
NCUFULL=0; [ $NCUFULL = 1 ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/prof_stem -f \
  python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 1 > gpurun_out/ncu_stem.log 2>&1
echo "ncu rc=$?"
