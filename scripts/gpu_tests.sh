#!/bin/bash
# GPU test pass with timing: quick smoke of new paths, then the whole -m gpu suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2410_08300_b200.build > /dev/null
: > gpurun_out/pytest_first.txt
for a in ${SMOKE_ALGOS:-smm}; do
  timeout 120 python scripts/smoke_new.py $a >> gpurun_out/pytest_first.txt 2>&1; echo "$a rc=$?" >> gpurun_out/pytest_first.txt
done
if [ -n "$FIRST" ]; then
  timeout ${T1:-900} python -m pytest $FIRST -m gpu -q --timeout 300 --timeout-method thread -rf --durations=15 >> gpurun_out/pytest_first.txt 2>&1
fi
tail -40 gpurun_out/pytest_first.txt
if [ "${FULL:-1}" = "1" ]; then
timeout ${T2:-2400} python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread -rf --durations=40 ${EXTRA} > gpurun_out/pytest_gpu_full.txt 2>&1
echo "full rc=$?"
tail -90 gpurun_out/pytest_gpu_full.txt > gpurun_out/pytest_gpu.txt
tail -60 gpurun_out/pytest_gpu.txt
fi
