#!/bin/bash
# GPU test pass with timing: new/changed tests first, then the whole -m gpu suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2410_08300_b200.build > /dev/null
timeout ${T1:-900} python -m pytest ${FIRST:-tests/test_custom.py tests/test_hooks.py} -m gpu -q --timeout 300 --durations=15 2>&1 | tail -40 > gpurun_out/pytest_first.txt
cat gpurun_out/pytest_first.txt
if [ "${FULL:-1}" = "1" ]; then
timeout ${T2:-2400} python -m pytest tests -m gpu -q --timeout 600 --durations=40 ${EXTRA} 2>&1 | tail -80 > gpurun_out/pytest_gpu.txt
tail -50 gpurun_out/pytest_gpu.txt
fi
