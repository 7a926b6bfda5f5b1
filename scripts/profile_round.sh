#!/bin/bash
# ncu evidence for profiles/: launch list of one bench step + a full capture of the dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-compare --no-cpu --no-model --no-configs > gpurun_out/ncu_bench_stdout.txt 2>&1
echo "launch list rc=$?"
# full capture: conv4_2 (dominant-kernel class) and conv1_2 (halo) of the bench step; skip warm-up launches
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 45 -c 12 \
   -o gpurun_out/prof_step -f python bench.py --steps 1 --warmup 3 --no-e2e --no-compare --no-cpu --no-model --no-configs > gpurun_out/ncu_full_stdout.txt 2>&1
echo "full capture rc=$?"
