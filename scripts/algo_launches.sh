#!/bin/bash
# ncu launch lists (per-kernel device time, cold-cache serialised) of one VGG-16 bench step
# per algorithm: gpurun_out/launches_<algo>.csv.  ALGOS overrides the list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for a in ${ALGOS:-implicit_gemm winograd gemm kn2row implicit_precomp_gemm direct smm}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$a.csv \
     python bench.py --quick --algo $a --steps 1 --warmup 3 --no-e2e --no-cpu --no-model --no-config5 \
     > gpurun_out/ncu_$a.txt 2>&1
  echo "$a rc=$?"
done
