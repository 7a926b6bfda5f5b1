#!/bin/bash
# ncu source-level (SASS + stall sampling) capture of the conv1_1 GEMM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:tc_gemm \
   -o /tmp/c11 -f python scripts/prof_layer.py conv1_1 implicit_gemm > /tmp/c11.log 2>&1
echo "capture rc=$?"; tail -3 /tmp/c11.log
ncu -i /tmp/c11.ncu-rep --page source --csv --print-source sass > gpurun_out/c11_sass.csv 2>&1
ncu -i /tmp/c11.ncu-rep --page details --csv > gpurun_out/c11_details.csv 2>&1
ls -la gpurun_out/c11_*
