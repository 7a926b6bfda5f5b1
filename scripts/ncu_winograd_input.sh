#!/bin/bash
# ncu full capture of the Winograd input transform (VGG conv3_2) with source-level stalls
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:winograd_input \
   -o /tmp/wi -f python scripts/prof_layer.py conv3_2 winograd > /tmp/wi.log 2>&1
echo "capture rc=$?"
ncu -i /tmp/wi.ncu-rep --page details --csv > gpurun_out/wi_details.csv 2>&1
ncu -i /tmp/wi.ncu-rep --page source --csv --print-source sass > gpurun_out/wi_sass.csv 2>&1
ls -la gpurun_out/wi_*
