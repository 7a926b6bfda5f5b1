#!/bin/bash
cd "$(dirname "$0")/.."
for l in conv1_2 conv2_2 conv3_2 conv4_2 conv5_2; do timeout 60 python scripts/layer_bench.py $l winograd --reps 10; done
timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --profile-from-start off python scripts/prof_layer.py conv1_2 winograd 2>&1 | grep -E "winograd|tc_gemm|duration|dram__" | head -20
