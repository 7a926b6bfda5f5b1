#!/bin/bash
# ncu source-level (SASS + stall sampling) capture of implicit_precomp_gemm on VGG conv3_2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:tc_gemm \
   -o /tmp/pc -f python scripts/prof_layer.py conv3_2 implicit_precomp_gemm > /tmp/pc.log 2>&1
echo "capture rc=$?"
ncu -i /tmp/pc.ncu-rep --page source --csv --print-source sass > gpurun_out/pc_sass.csv 2>&1
ncu -i /tmp/pc.ncu-rep --page raw --csv > gpurun_out/pc_raw.csv 2>&1
ls -la gpurun_out/pc_*
