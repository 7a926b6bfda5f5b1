#!/bin/bash
# shared-memory / L1 throughput of the engine on conv3_2 and conv1_2 (is the smem port the limit?)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for l in conv3_2 conv1_2; do
timeout 300 ncu --set full --clock-control none --profile-from-start off -k regex:tc_gemm -o /tmp/m_$l -f \
   python scripts/prof_layer.py $l implicit_gemm > /dev/null 2>&1
ncu -i /tmp/m_$l.ncu-rep --page raw --csv > gpurun_out/raw_$l.csv 2>&1
ncu -i /tmp/m_$l.ncu-rep --page details --csv > gpurun_out/details_$l.csv 2>&1
done
ls -la gpurun_out/raw_* gpurun_out/details_*
