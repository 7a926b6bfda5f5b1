#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/probe.txt 2>&1
for a in direct implicit_gemm gemm winograd; do
  timeout 180 python scripts/probe.py $a >> gpurun_out/probe.txt 2>&1 || echo "TIMEOUT/ERR rc=$? algo=$a" >> gpurun_out/probe.txt
done
cat gpurun_out/probe.txt
