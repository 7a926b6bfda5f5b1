#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,utilization.gpu --format=csv > gpurun_out/probe.txt 2>&1
python -m paper_2410_08300_b200.build > /dev/null
for a in implicit_precomp_gemm direct smm kn2row; do
  timeout 120 python scripts/smoke_new.py $a >> gpurun_out/probe.txt 2>&1; echo "$a rc=$?" >> gpurun_out/probe.txt
done
timeout 300 python -X importtime -c "import torch" 2> gpurun_out/importtime.txt
timeout 600 python -m pytest tests/test_fullsize_gpu.py -v -x --timeout 300 --durations=0 -k "conv1_1 or conv3_2" >> gpurun_out/probe.txt 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q --timeout 120 --durations=25 -k "config1" >> gpurun_out/probe.txt 2>&1
tail -60 gpurun_out/probe.txt
